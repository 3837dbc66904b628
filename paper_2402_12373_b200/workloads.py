"""Synthetic specifications of the BASELINE shapes (planted-formula and random), plus a whole-formula
evaluator over packed traces used to classify generated traces and to check that a learned formula is sound.

The generator follows the reference's `benchgen.gen_guided` recipe (`/root/reference/pkg/src/ltllearn/
benchgen.py:116-142`: characters uniform over the powerset, a trace is kept on the side the planted formula
puts it, until both sides are full) restated on the width-generic evaluator, because the reference's own
generator refuses traces longer than 63 positions.  The evaluator follows `bitsem.eval_cm`
(`bitsem.py:168-199`) with rows of W words (SURVEY rule N4).  Host-side utilities; not on the hot path.
"""
from __future__ import annotations

import numpy as np

from .formula import (OP_AND, OP_ATOM, OP_FINALLY, OP_GLOBALLY, OP_NEXT, OP_NOT, OP_OR, OP_UNTIL, Formula,
                      parse_formula)
from .packing import TraceContext, rounds_for_words
from .traces import Alphabet, Specification


def _shl(a: np.ndarray, s: int) -> np.ndarray:
    """Row-wide logical left shift by s bits of uint64[R, W] rows (zeros enter from beyond the last word)."""
    W = a.shape[1]
    q, r = divmod(int(s), 64)
    b = np.zeros_like(a)
    if q < W:
        b[:, : W - q] = a[:, q:]
    if r:
        carry = np.zeros_like(b)
        carry[:, :-1] = b[:, 1:] >> np.uint64(64 - r)
        b = (b << np.uint64(r)) | carry
    return b


def eval_formula(f: Formula, ctx: TraceContext) -> np.ndarray:
    """Characteristic matrix uint64[R, W] of ``f`` over the packed traces."""
    rounds = rounds_for_words(ctx.words)
    memo: dict[Formula, np.ndarray] = {}

    def ev(node: Formula) -> np.ndarray:
        got = memo.get(node)
        if got is not None:
            return got
        op = node.op
        if op == OP_ATOM:
            out = ctx.atoms[node.prop].copy()
        elif op == OP_NOT:
            out = ~ev(node.kids[0]) & ctx.masks
        elif op == OP_AND:
            out = ev(node.kids[0]) & ev(node.kids[1])
        elif op == OP_OR:
            out = ev(node.kids[0]) | ev(node.kids[1])
        elif op == OP_NEXT:
            out = _shl(ev(node.kids[0]), 1)
        elif op in (OP_FINALLY, OP_GLOBALLY):
            c = ev(node.kids[0])
            c = (~c & ctx.masks) if op == OP_GLOBALLY else c.copy()
            for i in range(rounds):
                c |= _shl(c, 1 << i)
            out = (~c & ctx.masks) if op == OP_GLOBALLY else c
        elif op == OP_UNTIL:
            run, acc = ev(node.kids[0]).copy(), ev(node.kids[1]).copy()
            for i in range(rounds):
                acc |= run & _shl(acc, 1 << i)
                if i + 1 < rounds:
                    run &= _shl(run, 1 << i)
            out = acc
        else:  # pragma: no cover
            raise ValueError(f"unknown opcode {op}")
        memo[node] = out
        return out

    return ev(f)


def accepts(f: Formula, ctx: TraceContext) -> np.ndarray:
    """bool[R]: does each trace satisfy ``f`` (verdict at position 0)."""
    return (eval_formula(f, ctx)[:, 0] >> np.uint64(63)).astype(bool)


def error_count(f: Formula, spec: Specification, alphabet: Alphabet) -> int:
    """Misclassified traces of the specification (0 = the formula is sound)."""
    ctx = TraceContext.from_spec(spec, alphabet)
    ok = accepts(f, ctx)
    return int(np.count_nonzero(~ok[: spec.n_pos])) + int(np.count_nonzero(ok[spec.n_pos:]))


def planted_spec(n_props: int, n_pos: int, n_neg: int, min_len: int, max_len: int, formula: str | Formula,
                 seed: int, max_draws: int = 400) -> tuple[Specification, Alphabet, Formula]:
    """Distinct random traces classified by a planted formula: ``n_pos`` satisfying, ``n_neg`` violating."""
    alphabet = Alphabet.default(n_props)
    f = parse_formula(formula, alphabet) if isinstance(formula, str) else formula
    rng = np.random.default_rng(seed)
    pos_c, pos_l, neg_c, neg_l = [], [], [], []
    need_p, need_n = n_pos, n_neg
    earlier: list[np.ndarray] = []  # keys of the traces drawn in earlier batches
    batch = max(256, 2 * (n_pos + n_neg))
    for _ in range(max_draws):
        if need_p <= 0 and need_n <= 0:
            break
        lengths = rng.integers(min_len, max_len + 1, size=batch).astype(np.int64)
        chars = rng.integers(0, 1 << n_props, size=(batch, max_len)).astype(np.uint16)
        chars[np.arange(max_len)[None, :] >= lengths[:, None]] = 0
        # distinct traces only: first occurrence inside the batch, none that an earlier batch drew
        keyed = np.ascontiguousarray(np.concatenate([chars, lengths[:, None].astype(np.uint16)], axis=1))
        keys = keyed.view(np.dtype((np.void, keyed.shape[1] * 2))).reshape(-1)
        _, first = np.unique(keys, return_index=True)
        first.sort()
        for old in earlier:
            first = first[~np.isin(keys[first], old)]
        earlier.append(keys[first].copy())
        chars, lengths = chars[first], lengths[first]
        ok = accepts(f, _ctx_from_arrays(chars, lengths, alphabet))
        take_p = np.nonzero(ok & (lengths > 0))[0][: max(need_p, 0)]
        take_n = np.nonzero(~ok)[0][: max(need_n, 0)]
        pos_c.append(chars[take_p]); pos_l.append(lengths[take_p]); need_p -= len(take_p)  # noqa: E702
        neg_c.append(chars[take_n]); neg_l.append(lengths[take_n]); need_n -= len(take_n)  # noqa: E702
    if need_p > 0 or need_n > 0:
        raise RuntimeError("planted formula is too one-sided on random traces: could not fill both sides")
    spec = Specification.from_arrays(np.concatenate(pos_c), np.concatenate(pos_l), np.concatenate(neg_c),
                                     np.concatenate(neg_l))
    return spec, alphabet, f


def _ctx_from_arrays(chars: np.ndarray, lengths: np.ndarray, alphabet: Alphabet) -> TraceContext:
    """Pack raw (possibly duplicated) traces without building a Specification."""
    from .packing import _bits_to_words, words_for_length

    W = words_for_length(int(lengths.max()) if len(lengths) else 1)
    R = len(lengths)
    padded = np.zeros((R, W * 64), dtype=np.uint16)
    padded[:, : chars.shape[1]] = chars
    live = np.arange(W * 64)[None, :] < lengths[:, None]
    atoms = np.empty((alphabet.size, R, W), dtype=np.uint64)
    for p in range(alphabet.size):
        atoms[p] = _bits_to_words(((padded >> p) & 1).astype(bool) & live, W)
    return TraceContext(lengths.copy(), _bits_to_words(live, W), R, atoms, W)


def random_spec(n_props: int, n_pos: int, n_neg: int, min_len: int, max_len: int, seed: int):
    """Distinct uniformly random traces, arbitrarily split: the "unsolvable" variant (every level exhaustive)."""
    alphabet = Alphabet.default(n_props)
    rng = np.random.default_rng(seed)
    total = n_pos + n_neg
    lengths = rng.integers(max(min_len, 1), max_len + 1, size=total).astype(np.int64)
    chars = rng.integers(0, 1 << n_props, size=(total, max_len)).astype(np.uint16)
    chars[np.arange(max_len)[None, :] >= lengths[:, None]] = 0
    spec = Specification.from_arrays(chars[:n_pos], lengths[:n_pos], chars[n_pos:], lengths[n_pos:])
    return spec, alphabet


#: The five BASELINE.json configurations as concrete, seeded workloads.  `formula` is the planted formula,
#: `max_cost` the inclusive search bound used by bench.py / the tests.
CONFIGS = {
    "c1_tiny": dict(n_props=2, n_pos=8, n_neg=8, min_len=4, max_len=16, formula="(p0 U p1) & F(G p0)", seed=1, max_cost=10),
    "c2_planted": dict(n_props=3, n_pos=512, n_neg=512, min_len=64, max_len=64,
                       formula="(p0 U (p1 & X p2)) & X(p1 | p2)", seed=2402, max_cost=12),
    "c3_long": dict(n_props=3, n_pos=256, n_neg=256, min_len=1024, max_len=1024, formula="p0 U (p1 & X(p2 U p0))", seed=12373,
                    max_cost=8),
    "c4_many": dict(n_props=4, n_pos=1 << 20, n_neg=1 << 20, min_len=32, max_len=32, formula="p0 U (p1 & X p3)", seed=4,
                    max_cost=7),
    "c5_deep": dict(n_props=5, n_pos=4096, n_neg=4096, min_len=64, max_len=64,
                    formula="(p0 U (p1 & X p2)) & F(p3 & X(p4 | X p0))", seed=5, max_cost=20),
}


def make_config(name: str, **override):
    cfg = dict(CONFIGS[name], **override)
    spec, alphabet, f = planted_spec(cfg["n_props"], cfg["n_pos"], cfg["n_neg"], cfg["min_len"], cfg["max_len"],
                                     cfg["formula"], cfg["seed"])
    return spec, alphabet, f, cfg
