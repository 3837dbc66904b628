#!/usr/bin/env python
"""Generate tests/golden/reference_golden.json by RUNNING THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    ./oracle/build_ref.sh && python tests/golden/make_golden.py

`ltllearn` is an implicit namespace package, so putting both /root/reference/pkg/src and
oracle/_ref on sys.path gives the reference's Python modules together with its compiled core
(`ltllearn._speedups`, built from the reference's own .pyx by oracle/build_ref.sh).  Every value
below is produced by reference code; nothing from this repo's implementation is involved.
The GPU box has no /root/reference, so the parity tests read the committed JSON instead.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import warnings

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, os.path.join(ROOT, "oracle", "_ref"))

import numpy as np  # noqa: E402

from ltllearn import benchgen, bitsem, cache as rcache, enumerator as E, formula as F, kernels as K  # noqa: E402
from ltllearn import oracle as roracle  # noqa: E402
from ltllearn.traces import Alphabet, Specification, SuffixTable  # noqa: E402

assert K.BACKEND == "compiled", "run oracle/build_ref.sh first"
warnings.simplefilter("ignore")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hexs(xs):
    return [f"{int(x):#x}" for x in xs]


out: dict = {"generator": "tests/golden/make_golden.py", "reference_backend": K.BACKEND}

# ---------------------------------------------------------------- 1. known answers
out["kat"] = {
    "mix64": {str(x): f"{K.mix64(x):#x}" for x in (0, 1, 2, 0xDEADBEEF, (1 << 64) - 1)},
    "mueller": [
        {"words": hexs(w), "fp": f"{K.mueller_fingerprint(w):#x}"}
        for w in (
            [0],
            [1],
            [1 << 63, (1 << 63) - 1],
            [(i * 0x0123456789ABCDEF) & ((1 << 64) - 1) for i in range(64)],
            [(i * i * 0x9E3779B97F4A7C15 + 7) & ((1 << 64) - 1) for i in range(17)],
        )
    ],
    "fkp_bits_per_row": {str(n): K.fkp_bits_per_row(n) for n in (1, 2, 3, 16, 42, 63, 64)},
    "length_mask": {str(n): f"{bitsem.length_mask(n):#x}" for n in (0, 1, 2, 16, 62, 63, 64)},
}

# ---------------------------------------------------------------- 2. Appendix-A style traced vectors
sq = F.parse_formula  # noqa
traced = []
for width, cs in ((16, 0b0000000000000100), (8, 0b00000001), (64, 1 << 20), (64, 0x8000000000000001)):
    res, states = bitsem.finally_traced(cs, width)
    traced.append({"kind": "F", "width": width, "cs": f"{cs:#x}", "result": f"{res:#x}", "states": hexs(states)})
for width, c1, c2 in ((8, 0b11111110, 0b00000001), (16, 0xFF0F, 0x0001), (64, (1 << 64) - 2, 1), (64, 0xF0F0F0F0F0F0F0F0, 0x0101010101010101)):
    res, states = bitsem.until_traced(c1, c2, width)
    traced.append({"kind": "U", "width": width, "cs1": f"{c1:#x}", "cs2": f"{c2:#x}", "result": f"{res:#x}",
                   "states": [[k, f"{a:#x}", f"{b:#x}"] for k, a, b in states]})
out["traced"] = traced
out["rounds_for_width"] = {str(w): bitsem.rounds_for_width(w) for w in (1, 2, 3, 8, 63, 64, 65, 128, 1024)}

# ---------------------------------------------------------------- 3. operator vectors on random matrices
rng = np.random.default_rng(20240212)
opvec = []
for case in range(12):
    R = int(rng.integers(1, 65))
    n_props = int(rng.integers(1, 4))
    traces = [tuple(int(c) for c in rng.integers(0, 1 << n_props, size=int(rng.integers(0 if r else 1, 64)))) for r in range(R)]
    n_pos = int(rng.integers(1, R + 1)) if R > 1 else 1
    ctx = bitsem.TraceContext.from_traces(traces, n_props, n_pos)
    x = rng.integers(0, 1 << 63, size=R, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=R, dtype=np.uint64)
    y = rng.integers(0, 1 << 63, size=R, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=R, dtype=np.uint64)
    x &= ctx.masks
    y &= ctx.masks
    opvec.append({
        "traces": [list(t) for t in traces], "n_props": n_props, "n_pos": n_pos,
        "masks": hexs(ctx.masks), "atoms": [hexs(a) for a in ctx.atoms],
        "x": hexs(x), "y": hexs(y),
        "not": hexs(bitsem.bf_not(x, ctx.masks)), "and": hexs(bitsem.bf_and(x, y)), "or": hexs(bitsem.bf_or(x, y)),
        "next": hexs(bitsem.bf_next(x)), "finally": hexs(bitsem.bf_finally(x)),
        "globally": hexs(bitsem.bf_globally(x, ctx.masks)), "until": hexs(bitsem.bf_until(x, y)),
        "errors_x": bitsem.error_count(x, n_pos),
    })
out["opvec"] = opvec

# ---------------------------------------------------------------- 4. fingerprints through the compiled core
fpvec = []
for case in range(10):
    R = int(rng.integers(1, 65))
    lengths = [int(v) for v in rng.integers(1, 64, size=R)]
    masks = np.array([bitsem.length_mask(n) for n in lengths], dtype=np.uint64)
    cms = [(rng.integers(0, 1 << 63, size=R, dtype=np.uint64) * np.uint64(2)) & masks for _ in range(3)]
    for variant, mask_k in ((K.V_MUELLER, 0), (K.V_MUELLER, 37), (K.V_MUELLER, 90), (K.V_FKP, 0), (K.V_FKP, 64), (K.V_GATHER, 0), (K.V_GATHER, 5)):
        pr, po, fb = [], [], 0
        if variant == K.V_GATHER:
            cells = [(r, j) for r in range(R) for j in range(lengths[r])]
            pick = sorted(rng.choice(len(cells), size=min(len(cells), int(rng.integers(1, 127))), replace=False))
            pr = [cells[i][0] for i in pick]
            po = [cells[i][1] for i in pick]
        if variant == K.V_FKP:
            fb = K.fkp_bits_per_row(R)
        core = K.make_core(masks, 1, 0, variant, pr, po, fb, mask_k, 1 << 20)
        fpvec.append({
            "masks": hexs(masks), "variant": variant, "mask_k": mask_k, "proj_rows": [int(v) for v in pr],
            "proj_offs": [int(v) for v in po], "fkp_bits": fb,
            "cms": [hexs(c) for c in cms], "fps": [f"{core.fingerprint_of(c):#x}" for c in cms],
            "fps_int": [f"{K.fingerprint_int([int(w) for w in c], variant, pr, po, fb, mask_k):#x}" for c in cms],
        })
out["fpvec"] = fpvec

# ---------------------------------------------------------------- 5. learner outcomes
_captured = []
_orig_make_core = K.make_core


def _capturing_make_core(*a, **kw):
    core = _orig_make_core(*a, **kw)
    _captured.append((core, a, kw))
    return core


K.make_core = _capturing_make_core


def run_case(name, spec, alphabet, cfg_kwargs, note=""):
    kw = dict(cfg_kwargs)
    hash_kw = kw.pop("hash", None)
    cost_w = kw.pop("cost", None)
    if hash_kw:
        kw["hash"] = rcache.HashScheme(**hash_kw)
    if cost_w:
        kw["cost"] = F.CostHomomorphism(tuple(cost_w))
    cfg = E.LearnerConfig(**kw)
    _captured.clear()
    res = E.enum_learn(spec, alphabet, cfg)
    row = {
        "name": name, "note": note, "n_props": alphabet.size, "pos": [list(t) for t in spec.pos],
        "neg": [list(t) for t in spec.neg], "cfg": cfg_kwargs, "outcome": type(res).__name__,
        "stats": {k: v for k, v in res.stats.as_dict().items() if k != "levels"},
        "levels": [{k: v for k, v in lv.items() if k != "ms"} for lv in res.stats.levels],
    }
    if isinstance(res, E.Solved):
        row["formula"] = F.print_formula(res.formula)
        row["cost"] = res.cost
        assert roracle.check_separates(res.formula, spec) or cfg.noise > 0
    elif isinstance(res, E.CeilingReached):
        row["formula_sha"] = hashlib.sha256(F.print_formula(res.formula).encode()).hexdigest()
        row["formula_len"] = len(F.print_formula(res.formula))
        row["ceiling"] = res.ceiling
    if _captured:
        core, a, _ = _captured[-1]
        cms = core.export_cms()
        recs = np.array([core.get_record(i) for i in range(core.n_entries)], dtype=np.int64).reshape(-1, 3)
        row["core"] = {
            "variant": int(a[3]), "proj_rows": [int(v) for v in a[4]], "proj_offs": [int(v) for v in a[5]],
            "fkp_bits": int(a[6]), "mask_k": int(a[7]), "n_entries": int(core.n_entries), "cms_sha": sha(cms),
            "records_sha": sha(recs),
            "first_records": recs[:24].tolist(),
        }
    return row


cases = []
A2, A3 = Alphabet.default(2), Alphabet.default(3)
for seed in range(8):
    cases.append(run_case(f"simple2_k4_s{seed}", benchgen.gen_simple(A2, 4, 2, 5, seed), A2, {}))
for seed in range(4):
    cases.append(run_case(f"simple3_k6_s{seed}", benchgen.gen_simple(A3, 6, 3, 8, 100 + seed), A3, {}))
cases.append(run_case("c1_guided_seed3", benchgen.gen_guided(A2, F.parse_formula("(p0 U p1) & F(G p0)", A2), 8, 4, 16, 3), A2,
                      {"ceiling": 11}, "BASELINE config 1 (max_cost 10 => exclusive ceiling 11)"))
for seed, text in ((5, "G(p0 | X p1)"), (6, "F(p0 & X(p1 U p2))"), (7, "(p0 U p1) | G p2")):
    al = A3 if "p2" in text else A2
    cases.append(run_case(f"guided_s{seed}", benchgen.gen_guided(al, F.parse_formula(text, al), 12, 6, 20, seed), al, {"ceiling": 10}))
cases.append(run_case("nnf_simple", benchgen.gen_simple(A2, 5, 2, 6, 11), A2, {"require_nnf": True}))
cases.append(run_case("nnf_nountil", benchgen.gen_simple(A2, 5, 2, 6, 12), A2, {"require_nnf": True, "forbid_until": True}))
cases.append(run_case("nountil", benchgen.gen_simple(A3, 5, 3, 7, 13), A3, {"forbid_until": True}))
cases.append(run_case("noise10", benchgen.gen_simple(A2, 10, 3, 9, 14), A2, {"noise": 0.1}))
cases.append(run_case("noise25", benchgen.gen_simple(A2, 12, 4, 10, 15), A2, {"noise": 0.25, "ceiling": 9}))
cases.append(run_case("weights", benchgen.gen_simple(A2, 5, 2, 6, 16), A2, {"cost": [1, 2, 1, 1, 3, 2, 2, 4], "ceiling": 14}))
cases.append(run_case("weights2", benchgen.gen_simple(A3, 6, 3, 8, 17), A3, {"cost": [2, 1, 3, 3, 1, 1, 1, 2], "ceiling": 13}))
cases.append(run_case("fkp", benchgen.gen_simple(A2, 16, 8, 20, 18), A2, {"hash": {"variant": "fkp"}, "ceiling": 8}))
cases.append(run_case("mueller_mask40", benchgen.gen_simple(A2, 16, 8, 20, 19), A2, {"hash": {"variant": "mueller", "mask_bits": 40}, "ceiling": 8}))
cases.append(run_case("mueller_mask100", benchgen.gen_simple(A2, 16, 8, 20, 19), A2, {"hash": {"variant": "mueller", "mask_bits": 100}, "ceiling": 8}))
cases.append(run_case("gather_mask3", benchgen.gen_simple(A2, 4, 2, 5, 20), A2, {"hash": {"variant": "mueller", "mask_bits": 3}}))
cases.append(run_case("oom_small_budget", benchgen.gen_simple(A2, 16, 8, 20, 21), A2, {"budget_bytes": 200 * (32 * 8 + 16) + 7, "ceiling": 9}))
cases.append(run_case("oom_at_atoms", benchgen.gen_simple(A2, 16, 8, 20, 21), A2, {"budget_bytes": (32 * 8 + 16) + 3, "ceiling": 9}))
cases.append(run_case("ceiling_low", benchgen.gen_simple(A2, 16, 8, 20, 22), A2, {"ceiling": 5}))
cases.append(run_case("atom_fast", Specification(((1, 0), (1, 3)), ((0, 1), (2,))), A2, {}))
cases.append(run_case("nnf_atom_fast", Specification(((0, 1), (2, 3)), ((1, 0), (3,))), A2, {"require_nnf": True}))
cases.append(run_case("empty_negative", Specification(((1, 2), (3,)), ((), (0, 1))), A2, {}))
# exhaustive regression table from BASELINE.md: rng(1), 32+32 traces x 63, 2 props, ceiling 10
r1 = np.random.default_rng(1)
tr = [tuple(int(c) for c in r1.integers(0, 4, size=63)) for _ in range(64)]
cases.append(run_case("table_rng1_32x32x63", Specification(tuple(tr[:32]), tuple(tr[32:])), A2, {"ceiling": 10},
                      "BASELINE.md section 2 regression table"))
r2 = np.random.default_rng(2)
tr = [tuple(int(c) for c in r2.integers(0, 8, size=int(r2.integers(20, 64)))) for _ in range(40)]
cases.append(run_case("rand3_20x20", Specification(tuple(tr[:20]), tuple(tr[20:])), A3, {"ceiling": 8}))
out["learn"] = cases
K.make_core = _orig_make_core

# ---------------------------------------------------------------- 6. screening-level transcripts (core API)
transcripts = []
for seed in range(4):
    r = np.random.default_rng(900 + seed)
    R = int(r.integers(2, 65))
    lengths = [int(v) for v in r.integers(1, 64, size=R)]
    masks = np.array([bitsem.length_mask(n) for n in lengths], dtype=np.uint64)
    n_pos = int(r.integers(1, R))
    core = K.make_core(masks, n_pos, 0, K.V_MUELLER, (), (), 0, 0, 1 << 24)
    seeds = [(r.integers(0, 1 << 63, size=R, dtype=np.uint64) * np.uint64(2)) & masks for _ in range(6)]
    log = []
    for k, cm in enumerate(seeds):
        log.append(["add", core.add_entry(cm, 0, k, -1)])
    n0 = core.n_entries
    for op in (1, 4, 5, 6):
        log.append(["unary", op, list(core.screen_unary(op, 0, n0))])
    n1 = core.n_entries
    for op, tri in ((2, True), (3, True), (7, False)):
        log.append(["binary", op, list(core.screen_binary(op, 0, n0, 0, n0, tri))])
    log.append(["binary", 2, list(core.screen_binary(2, 0, n0, n0, n1, False))])
    log.append(["binary", 7, list(core.screen_binary(7, n0, n1, 0, n0, False))])
    transcripts.append({
        "masks": hexs(masks), "n_pos": n_pos, "seeds": [hexs(c) for c in seeds], "log": log,
        "counters": [int(core.n_entries), int(core.bytes_used), int(core.offered), int(core.admitted), int(core.duplicates)],
        "cms_sha": sha(core.export_cms()),
        "records_sha": sha(np.array([core.get_record(i) for i in range(core.n_entries)], dtype=np.int64).reshape(-1, 3)),
    })
out["transcripts"] = transcripts

# ---------------------------------------------------------------- 7. formula text / cost / overfit
texts = ["p0", "!p0", "!(p0 & p1)", "p0 & p1 & p2", "(p0 & p1) | p2", "p0 U (p1 U p2)", "(p0 U p1) U p2",
         "X F G !p1", "F G p0 & (p0 U p1)", "!G p1 & (p1 | X G p1)", "G(p0 | X p1)", "!(X p0 | F !p1) U G(p2 & !p0)"]
out["formula_text"] = [
    {"in": t, "printed": F.print_formula(F.parse_formula(t, A3)), "cost": F.cost(F.parse_formula(t, A3)),
     "cost_w": F.cost(F.parse_formula(t, A3), F.CostHomomorphism((1, 2, 1, 1, 3, 2, 2, 4)))}
    for t in texts
]
ov = []
for spec, al in ((Specification(((1, 0), (3,)), ((0,),)), A2), (Specification(((5, 2, 7), (0,)), ((1, 1),)), A3)):
    ov.append({"pos": [list(t) for t in spec.pos], "neg": [list(t) for t in spec.neg], "n_props": al.size,
               "text": F.print_formula(F.overfit(spec, al)), "cost": F.overfit_cost(spec, al),
               "cost_w": F.overfit_cost(spec, al, F.CostHomomorphism((1, 2, 1, 1, 3, 2, 2, 4)))})
out["overfit"] = ov

# ---------------------------------------------------------------- 8. suffix tables / scheme resolution
st = []
for seed in range(6):
    spec = benchgen.gen_simple(A2, 4 + seed, 2, 5 + seed, 300 + seed)
    table = SuffixTable.from_spec(spec)
    lengths = [len(t) for t in spec.traces]
    rs = rcache.resolve_scheme(rcache.HashScheme(), lengths, table)
    st.append({"pos": [list(t) for t in spec.pos], "neg": [list(t) for t in spec.neg], "count": table.count,
               "rows": list(table.rows), "offsets": list(table.offsets), "variant": rs.variant})
out["suffix"] = st

path = os.path.join(HERE, "reference_golden.json")
with open(path, "w") as fh:
    json.dump(out, fh, separators=(",", ":"))
print("wrote", path, os.path.getsize(path), "bytes;", len(cases), "learn cases")
for c in cases:
    print(f"  {c['name']:24s} {c['outcome']:15s} {c.get('formula', '')!s:40s} off={c['stats']['offered']} adm={c['stats']['admitted']}")
