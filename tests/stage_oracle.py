"""TEST INFRASTRUCTURE: a CPU stand-in for the multi-GPU stage API of `CudaCore` (level_size, stage_eval,
stage_file, stage_decode, stage_append, stage_purge), built on the CPU oracle, so that the sharded
orchestration (`paper_2402_12373_b200/sharded.py`) can be exercised with gloo processes on a machine without
a GPU.  Tensors are CPU torch tensors."""
from __future__ import annotations

import numpy as np
import torch

from oracle import cpu_oracle
from paper_2402_12373_b200 import errors as E

UNARY = (1, 4, 5, 6)
MASK64 = (1 << 64) - 1


def _i64(x: int) -> int:
    x &= MASK64
    return x - (1 << 64) if x >= (1 << 63) else x


def _u64(x: int) -> int:
    return x & MASK64


def seg_count(s) -> int:
    na = s.a1 - s.a0
    if s.op in UNARY:
        return max(na, 0)
    if na <= 0 or s.b1 <= s.b0:
        return 0
    if not s.tri:
        return na * (s.b1 - s.b0)
    return sum(max(0, s.b1 - max(s.b0, i + 1)) for i in range(s.a0, s.a1))


def seg_candidates(s):
    if s.op in UNARY:
        for i in range(s.a0, s.a1):
            yield s.op, i, -1
        return
    for i in range(s.a0, s.a1):
        for j in range(max(s.b0, i + 1) if s.tri else s.b0, s.b1):
            yield s.op, i, j


class OracleStageCore:
    def __init__(self, masks, n_pos, err_max, variant, proj_rows=(), proj_offs=(), fkp_bits=0, mask_k=0,
                 budget_bytes=2 << 30, *, words_per_row=1, device=None):
        self.o = cpu_oracle.OracleCore(masks, n_pos, err_max, variant, proj_rows, proj_offs, fkp_bits, mask_k,
                                       1 << 60, words_per_row=words_per_row)
        self.err_max = err_max
        self.entry_bytes = 8 * self.o.n + 16
        self.cap = int(budget_bytes) // self.entry_bytes
        self.offered = self.admitted = self.duplicates = 0
        self.table: dict[tuple[int, int], int] = {}  # this rank's shard: key -> owning global rank
        self.store = True

    # -- replicated calls
    def add_entry(self, cm, op, lhs, rhs):
        rank = self.offered
        self.offered += 1
        fp = self.o.fingerprint_of(cm)
        key = (fp >> 64, fp & MASK64)
        if key in self.table:
            self.duplicates += 1
            return -1
        if self.admitted + 1 > self.cap:
            raise E.CoreOOM
        self.table[key] = rank
        idx = self.o.add_entry(cm, op, lhs, rhs)
        assert idx == self.admitted
        self.admitted += 1
        return idx

    def get_record(self, idx):
        return self.o.get_record(idx)

    def counters(self):
        n = self.o.n_entries
        return [n, self.admitted * self.entry_bytes, self.offered, self.admitted, self.duplicates]

    def capacity_entries(self):
        return self.cap

    def set_option(self, name, value):
        pass

    # -- stages
    def level_size(self, segments):
        return sum(seg_count(s) for s in segments)

    def _candidates(self, segments, lo, hi):
        r = 0
        for s in segments:
            c = seg_count(s)
            if r + c <= lo:
                r += c
                continue
            for cand in seg_candidates(s):
                if r >= hi:
                    return
                if r >= lo:
                    yield r, cand
                r += 1

    def _eval(self, op, i, j):
        x = self.o.get_cm(i)
        return self.o.apply_unary(op, x) if j < 0 else self.o.apply_binary(op, x, self.o.get_cm(j))

    def stage_eval(self, segments, lo, hi):
        fp = torch.zeros((max(hi - lo, 0), 2), dtype=torch.int64)
        solver = -1
        for r, (op, i, j) in self._candidates(segments, lo, hi):
            cm = self._eval(op, i, j)
            f = self.o.fingerprint_of(cm)
            fp[r - lo, 0], fp[r - lo, 1] = _i64(f >> 64), _i64(f)
            if self.o.errors(cm) <= self.err_max:
                solver = r
                break
        return fp, solver

    def stage_route(self, fp, rank_base, world):
        """(hi, lo, global rank) tuples grouped by owner, in rank order inside a group, and the per-owner counts
        (`ltl_core_stage_route`)."""
        from paper_2402_12373_b200.sharded import owner_of

        keep = fp.shape[0]
        owner = owner_of(fp, world)
        order = torch.sort(owner, stable=True)[1] if keep else torch.zeros(0, dtype=torch.int64)
        counts = [int((owner == d).sum()) for d in range(world)]
        ranks = int(rank_base) + torch.arange(keep, dtype=torch.int64)
        return torch.cat([fp[order], ranks[order].unsqueeze(1)], 1).contiguous(), counts

    def stage_winners(self, send, win, rank_base, level_lo):
        """Ascending level ranks of the winners among the tuples sent (`ltl_core_stage_winners`)."""
        ranks = send[:, 2][win.to(torch.bool)] - int(rank_base) + int(level_lo)
        return torch.sort(ranks)[0]

    def stage_file(self, tuples):
        gbase = self.offered
        rows = [(_u64(int(a)), _u64(int(b)), int(c)) for a, b, c in tuples.tolist()]
        contenders = {}
        for hi, lo, rank in rows:
            old = self.table.get((hi, lo))
            if old is not None and old < gbase:
                continue
            contenders[(hi, lo)] = min(contenders.get((hi, lo), rank), rank)
        win = torch.zeros(len(rows), dtype=torch.uint8)
        for k, (hi, lo, rank) in enumerate(rows):
            if contenders.get((hi, lo)) == rank:
                win[k] = 1
                self.table[(hi, lo)] = rank
        return win

    def stage_decode(self, segments, ranks):
        want = [int(v) for v in ranks.tolist()]
        out = {}
        if want:
            lo, hi = min(want), max(want) + 1
            need = set(want)
            for r, cand in self._candidates(segments, lo, hi):
                if r in need:
                    out[r] = cand
        op = torch.tensor([out[r][0] for r in want], dtype=torch.uint8)
        lhs = torch.tensor([out[r][1] for r in want], dtype=torch.int32)
        rhs = torch.tensor([out[r][2] for r in want], dtype=torch.int32)
        return op, lhs, rhs

    def stage_append(self, op, lhs, rhs, offered_delta, duplicates_delta):
        for o, l, r in zip(op.tolist(), lhs.tolist(), rhs.tolist()):
            idx = self.o.add_entry(self._eval(int(o), int(l), int(r)), int(o), int(l), int(r))
            assert idx >= 0, "an admitted entry must be new in the replicated store"
            self.admitted += 1
        self.offered += int(offered_delta)
        self.duplicates += int(duplicates_delta)

    def stage_purge(self, cut):
        self.table = {k: v for k, v in self.table.items() if v < cut}


class OracleRowShard:
    """TEST INFRASTRUCTURE: CPU stand-in for one ROW SHARD of `CudaCore` (`set_row_shard`), on the CPU oracle's
    operator / error / fingerprint functions over this shard's rows.  Per candidate it contributes the fingerprint
    and the error count of its rows; the sums over the shards (the exchange) decide admission, identically on every
    rank.  (The sum of the shards' local fingerprints is not the device's value -- the device sums per 64-word block
    -- but admission only needs a collision-free function of all rows.)"""

    def __init__(self, masks, n_pos, err_max, variant, proj_rows=(), proj_offs=(), fkp_bits=0, mask_k=0,
                 budget_bytes=2 << 30, *, words_per_row=1, device=None):
        self.o = cpu_oracle.OracleCore(masks, n_pos, 0, variant, proj_rows, proj_offs, fkp_bits, mask_k, 1 << 60,
                                       words_per_row=words_per_row)
        self.err_max, self.budget = err_max, int(budget_bytes)
        self.cms, self.records, self.table = [], [], set()
        self.offered = self.admitted = self.duplicates = 0
        self.exchange, self.entry_bytes = None, 8 * self.o.n + 16

    def set_row_shard(self, word_base, total_words, all_reduce_sum):
        assert word_base % 64 == 0
        self.exchange, self.entry_bytes = all_reduce_sum, 8 * int(total_words) + 16

    def set_option(self, name, value):
        pass

    def close(self):
        pass

    def _sums(self, cms):
        fps = [self.o.fingerprint_of(cm) for cm in cms]
        s0 = torch.tensor([_i64(f >> 64) for f in fps], dtype=torch.int64)
        s1 = torch.tensor([_i64(f) for f in fps], dtype=torch.int64)
        err = torch.tensor([self.o.errors(cm) for cm in cms], dtype=torch.int32)
        self.exchange([s0, s1, err])
        return s0.tolist(), s1.tolist(), err.tolist()

    def _offer(self, cm, key, record):
        """First-wins admission (reference _speedups.pyx:245-262): index, -1 duplicate, -3 over budget."""
        self.offered += 1
        if key in self.table:
            self.duplicates += 1
            return -1
        if self.admitted * self.entry_bytes + self.entry_bytes > self.budget:
            return -3
        self.table.add(key)
        self.cms.append(cm)
        self.records.append(record)
        self.admitted += 1
        return self.admitted - 1

    def add_entry(self, cm, op, lhs, rhs):
        cm = np.ascontiguousarray(cm, dtype=np.uint64)
        s0, s1, _ = self._sums([cm])
        idx = self._offer(cm, (s0[0], s1[0]), (op, lhs, rhs))
        if idx == -3:
            raise E.CoreOOM
        return idx

    def _eval(self, op, i, j):
        return self.o.apply_unary(op, self.cms[i]) if j < 0 else self.o.apply_binary(op, self.cms[i], self.cms[j])

    def run_level(self, segments):
        segments = list(segments)
        cands = [(k, c) for k, s in enumerate(segments) for c in seg_candidates(s)]
        cms = [self._eval(op, i, j) for _, (op, i, j) in cands]
        s0, s1, err = self._sums(cms) if cands else ([], [], [])
        for n, (k, (op, i, j)) in enumerate(cands):
            if err[n] <= self.err_max:
                self.offered += 1  # the solving candidate is offered, never admitted (reference _speedups.pyx:347-350)
                return 1, k, i, j
            if self._offer(cms[n], (s0[n], s1[n]), (op, i, j)) == -3:
                return 2, -1, -1, -1
        return 0, -1, -1, -1

    def get_record(self, idx):
        return self.records[idx]

    def get_cm(self, idx):
        return self.cms[idx].copy()

    def counters(self):
        return [self.admitted, self.admitted * self.entry_bytes, self.offered, self.admitted, self.duplicates]

    def transfer_stats(self):
        return 0, 0
