"""One search across several GPUs of a box: candidate ranges sharded per cost level, fingerprints routed to
hash-owner GPUs, accepted delta shared before the next level (north-star multi-GPU design).

One process per GPU (`torch.distributed`, NCCL over NVLink; gloo on CPU in the tests).  Every rank holds the
same replicated entry store and counters; the uniqueness table is sharded by fingerprint owner.  Per level:

  1. every rank evaluates its contiguous slice of the level's rank range (`stage_eval`: the phase-A kernel
     in fingerprint-only mode -> (hi, lo) per candidate + the lowest solving rank of the slice);
  2. `all_reduce(min)` of the solving rank: nothing at or above it is admitted (reference `_speedups.pyx:372-374`);
  3. `(hi, lo, global rank)` tuples go to `owner = mix(fp) mod G` with one `all_to_all_single`; the owner files
     them with `atomicMin(rank)` in its table shard (`stage_file`) and answers one winner byte per tuple by the
     reverse all-to-all -- "lowest enumeration rank wins", exactly the sequential first-wins admission;
  4. winners are numbered in rank order (exclusive scan of the per-rank counts = `all_gather` of G integers),
     the budget cut is applied (reference `_speedups.pyx:252-253`), and the winners' `(op, lhs, rhs)` records are
     all-gathered: 9 bytes per admitted entry cross NVLink, never the matrices -- every rank re-derives the
     matrices from the records with its local phase-B kernel when they are first needed (HBM at ~6 TB/s beats
     receiving 7/8 of the delta at <= 0.9 TB/s);
  5. every rank appends the same records and advances the same counters (`stage_append`).

`RowShardedCore` (further down) is the second sharding: every GPU holds a slice of the ROWS of every matrix, the
per-candidate partial fingerprint sums are all-reduced, the store is partitioned instead of replicated.

Results (entry order, records, counters, statuses, formula text) are identical to the 1-GPU path and to the
CPU oracle; `tests/test_sharded_*.py` check that with G virtual ranks on threads (1 GPU) and with gloo
processes over a CPU stand-in for the stages.
"""
from __future__ import annotations

import os
import threading
from typing import Callable, Sequence

import numpy as np

S_DONE, S_SOLVED, S_OOM = 0, 1, 2
_INF = 1 << 62


# ------------------------------------------------------------------------------------------------ comms


class TorchComm:
    """torch.distributed endpoints (NCCL for CUDA tensors, gloo for CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

    def _dev(self, like=None):
        import torch

        if like is not None:
            return like.device
        return torch.device("cuda", torch.cuda.current_device()) if self.dist.get_backend(self.group) == "nccl" \
            else torch.device("cpu")

    def all_reduce_min(self, value: int, device=None) -> int:
        import torch

        t = torch.tensor([int(value)], dtype=torch.int64, device=device or self._dev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return int(t.item())

    def all_gather_ints(self, value: int, device=None) -> list[int]:
        import torch

        t = torch.tensor([int(value)], dtype=torch.int64, device=device or self._dev())
        out = torch.empty(self.world, dtype=torch.int64, device=t.device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return [int(v) for v in out.tolist()]

    def all_to_all(self, send, counts: Sequence[int]):
        """Rows of ``send`` (grouped by destination, ``counts[d]`` rows for rank d) -> rows received, grouped by
        source, and the per-source counts."""
        import torch

        counts_t = torch.tensor(list(counts), dtype=torch.int64, device=send.device)
        recv_counts_t = torch.empty_like(counts_t)
        self.dist.all_to_all_single(recv_counts_t, counts_t, group=self.group)
        recv_counts = [int(v) for v in recv_counts_t.tolist()]
        recv = torch.empty((sum(recv_counts),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(recv, send.contiguous(), output_split_sizes=recv_counts,
                                    input_split_sizes=list(counts), group=self.group)
        return recv, recv_counts

    def all_gather_cat(self, t):
        """Concatenation of every rank's rows, in rank order (row counts may differ)."""
        import torch

        sizes = self.all_gather_ints(t.shape[0], device=t.device)
        width = max(sizes) if sizes else 0
        padded = torch.zeros((width,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        padded[: t.shape[0]] = t
        out = torch.empty((self.world * width,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, padded.contiguous(), group=self.group)
        return torch.cat([out[r * width: r * width + sizes[r]] for r in range(self.world)], 0)

    def all_reduce_sum(self, tensors):
        """In-place wrapping integer sums over the ranks; returns once the results are visible to the device."""
        import torch

        for t in tensors:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        if tensors and tensors[0].is_cuda:
            torch.cuda.current_stream(tensors[0].device).synchronize()

    def barrier(self):
        self.dist.barrier(group=self.group)


class ThreadComm:
    """G virtual ranks on threads of one process (tests: exercises the exchange logic on one GPU or on CPU
    without NCCL).  Create with `ThreadComm.group(G)`."""

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared, rank):
        self._s, self.rank, self.world = shared, rank, shared.world

    @staticmethod
    def group(world: int):
        shared = ThreadComm._Shared(world)
        return [ThreadComm(shared, r) for r in range(world)]

    def _exchange(self, value):
        s = self._s
        s.slots[self.rank] = value
        s.barrier.wait()
        got = list(s.slots)
        s.barrier.wait()
        return got

    def all_reduce_min(self, value: int, device=None) -> int:
        return min(self._exchange(int(value)))

    def all_gather_ints(self, value: int, device=None) -> list[int]:
        return self._exchange(int(value))

    def all_to_all(self, send, counts):
        import torch

        offs = np.concatenate([[0], np.cumsum(counts)])
        parts = [send[int(offs[d]): int(offs[d + 1])] for d in range(self.world)]
        everything = self._exchange(parts)
        mine = [everything[src][self.rank] for src in range(self.world)]
        recv_counts = [int(p.shape[0]) for p in mine]
        return torch.cat([p.to(send.device) for p in mine], 0), recv_counts

    def all_gather_cat(self, t):
        import torch

        return torch.cat([p.to(t.device) for p in self._exchange(t)], 0)

    def all_reduce_sum(self, tensors):
        import torch

        everything = self._exchange(tensors)  # every rank sees every rank's tensors (same device or CPU)
        totals = []
        for k, mine in enumerate(tensors):
            acc = torch.zeros_like(mine)
            for r in range(self.world):
                acc += everything[r][k].to(mine.device)
            totals.append(acc)
        if tensors and tensors[0].is_cuda:
            torch.cuda.synchronize()
        self._s.barrier.wait()  # nobody overwrites an input another rank is still reading
        for mine, acc in zip(tensors, totals):
            mine.copy_(acc)
        if tensors and tensors[0].is_cuda:
            torch.cuda.synchronize()

    def barrier(self):
        self._s.barrier.wait()


# ------------------------------------------------------------------------------------------------ the sharded core


def owner_of(fp, world: int):
    """Owner rank of each fingerprint (int64[N, 2] bit patterns): a multiplicative mix of hi ^ lo, reduced
    mod the world size.  Pure integer arithmetic, identical on every rank and device."""
    x = (fp[:, 0] ^ fp[:, 1]) * (-7046029254386353131)  # 0x9E3779B97F4A7C15 as int64; wraps
    return ((x >> 33) & 0x7FFFFFFF) % world


class ShardedCore:
    """The screening-core contract (`add_entry`, `run_level`, `get_record`, `counters`, ...) over G ranks.
    ``local`` is this rank's stage backend (a `CudaCore`, or a CPU stand-in in the gloo tests)."""

    def __init__(self, local, comm):
        self.local, self.comm = local, comm
        self.stage_ms = {} if os.environ.get("LTL_SHARDED_TIMERS") else None  # per-stage wall time (device-synchronised)

    def _tick(self, name, t0):
        """Profiling aid (LTL_SHARDED_TIMERS=1): synchronise the device and add the time since t0 to `name`."""
        import time

        if self.stage_ms is None:
            return 0.0
        import torch

        if torch.cuda.is_available():
            torch.cuda.synchronize()
        t1 = time.perf_counter()
        self.stage_ms[name] = self.stage_ms.get(name, 0.0) + 1e3 * (t1 - t0)
        return t1

    # replicated single-matrix calls: every rank performs the same call on its replica
    def add_entry(self, cm, op, lhs, rhs):
        return self.local.add_entry(cm, op, lhs, rhs)

    def get_record(self, idx):
        return self.local.get_record(idx)

    def export_records(self, first=0, count=None):
        return self.local.export_records(first, count)

    def counters(self):
        return self.local.counters()

    n_entries = property(lambda s: s.local.counters()[0])

    def set_option(self, name, value):
        if name == "deadline_ms":
            return  # ranks must take every decision together: the deadline stays a per-level check of the caller
        if hasattr(self.local, "set_option"):
            self.local.set_option(name, value)

    def transfer_stats(self):
        return self.local.transfer_stats() if hasattr(self.local, "transfer_stats") else (0, 0)

    def close(self):
        close = getattr(self.local, "close", None)
        if close:
            close()

    def _segment_of(self, segments, rank: int) -> int:
        lo, hi = 0, len(segments) - 1
        while lo < hi:  # first prefix whose size exceeds the rank
            mid = (lo + hi) // 2
            if self.local.level_size(segments[: mid + 1]) > rank:
                hi = mid
            else:
                lo = mid + 1
        return lo

    def run_level(self, segments):
        import torch

        segments = list(segments)
        local, comm = self.local, self.comm
        G, g = comm.world, comm.rank
        total = local.level_size(segments)
        if total == 0:
            return S_DONE, -1, -1, -1
        n_entries, _, gbase, _, _ = local.counters()
        lo, hi = total * g // G, total * (g + 1) // G

        # 1-2: evaluate the slice, agree on the first solver
        import time

        tk = time.perf_counter() if self.stage_ms is not None else 0.0
        fp, solver_local = local.stage_eval(segments, lo, hi)
        tk = self._tick("eval", tk)
        dev = fp.device
        solver = comm.all_reduce_min(solver_local if solver_local >= 0 else _INF, device=dev)
        limit = min(total, solver)
        keep = max(0, min(hi, limit) - lo)
        fp = fp[:keep]
        tk = self._tick("solver_allreduce", tk)

        # 3: route to hash owners, file, route the verdicts back.  Grouping by owner (a stable counting sort) and the
        # extraction of the winners' ranks run in the library (`ltl_core_stage_route` / `_winners`), not as tensor ops
        send, counts = local.stage_route(fp, gbase + lo, G)
        tk = self._tick("route_sort", tk)
        recv, recv_counts = comm.all_to_all(send, counts)
        tk = self._tick("all_to_all", tk)
        win_recv = local.stage_file(recv)
        tk = self._tick("file", tk)
        win_sorted, _ = comm.all_to_all(win_recv, recv_counts)
        tk = self._tick("all_to_all_back", tk)
        winners = local.stage_winners(send, win_sorted, gbase + lo, lo)  # ascending level ranks
        tk = self._tick("winners", tk)

        # 4: global numbering in rank order, budget cut
        n_local = int(winners.shape[0])
        all_n = comm.all_gather_ints(n_local, device=dev)
        total_w, base = sum(all_n), sum(all_n[:g])
        room = max(0, local.capacity_entries() - n_entries)
        oom = total_w > room
        oom_rank = _INF
        if oom:
            mine = int(winners[room - base].item()) if base <= room < base + n_local else _INF
            oom_rank = comm.all_reduce_min(mine, device=dev)
            winners = winners[: max(0, min(n_local, room - base))]
        op, lhs, rhs = local.stage_decode(segments, winners)
        tk = self._tick("decode", tk)
        packed = torch.stack([op.to(torch.int32), lhs, rhs], 1)
        packed = comm.all_gather_cat(packed)
        tk = self._tick("all_gather", tk)
        count = min(total_w, room)
        assert packed.shape[0] == count, (packed.shape, count)

        # 5: identical append on every rank
        status, cut = S_DONE, None
        if oom:
            status, cut = S_OOM, oom_rank
            offered_delta, dup_delta = oom_rank + 1, oom_rank - count
        elif solver < _INF:
            status, cut = S_SOLVED, solver
            offered_delta, dup_delta = solver + 1, solver - count
        else:
            offered_delta, dup_delta = total, total - count
        local.stage_append(packed[:, 0].to(torch.uint8), packed[:, 1].contiguous(), packed[:, 2].contiguous(),
                           offered_delta, dup_delta)
        tk = self._tick("append", tk)
        if status == S_DONE:
            return S_DONE, -1, -1, -1
        local.stage_purge(gbase + cut)
        if status == S_OOM:
            return S_OOM, -1, -1, -1
        sop, sl, sr = local.stage_decode(segments, torch.tensor([solver], dtype=torch.int64, device=dev))
        return S_SOLVED, self._segment_of(segments, solver), int(sl.item()), int(sr.item())


# ------------------------------------------------------------------------------------------------ row shards


def row_slices(n_rows: int, words_per_row: int, world: int, half_width: bool = False):
    """Row range of every shard: equal slices whose word offsets are multiples of 64 (fingerprint blocks must not
    straddle shards); trailing shards may be short or -- if there are too few rows -- empty (then: ValueError).
    ``half_width``: the core stores two rows per word (variant NH32), so a fingerprint block is 128 rows."""
    import math

    unit = 128 if half_width else 64 // math.gcd(64, words_per_row)  # rows per whole number of 64-word blocks
    per = -(-n_rows // world)
    per = -(-per // unit) * unit
    out = [(min(n_rows, g * per), min(n_rows, (g + 1) * per)) for g in range(world)]
    if any(a == b for a, b in out):
        raise ValueError(f"{n_rows} rows x {words_per_row} words cannot be cut into {world} shards of whole 64-word blocks")
    return out


class RowShardedCore:
    """The screening-core contract over G GPUs that each hold a slice of the ROWS of every characteristic matrix
    (the alternative for many-row specifications; `include/ltl_core.h: ltl_core_set_row_shard`).

    Every rank enumerates every candidate on its rows (1/G of the words), the per-candidate partial fingerprint sums
    and error counts are all-reduced (20 bytes per candidate over NVLink), and every rank then takes identical
    decisions: same winners, same entry order, same records and counters as one core over all rows.  Unlike the
    candidate-sharded core the entry store is partitioned, not replicated: G GPUs hold G times the language cache,
    and phase B (writing the new matrices) scales with G as well."""

    def __init__(self, local, comm, r0: int, r1: int, n_rows: int, words_per_row: int):
        self.local, self.comm = local, comm
        self.r0, self.r1, self.n_rows, self.W = r0, r1, n_rows, words_per_row
        self.stage_ms = None

    def _mine(self, cm):
        a = np.ascontiguousarray(cm, dtype=np.uint64).reshape(-1)
        if len(a) != self.n_rows * self.W:
            raise ValueError(f"expected {self.n_rows * self.W} words, got {len(a)}")
        return a[self.r0 * self.W: self.r1 * self.W]

    def _gather_rows(self, local_rows):
        import torch

        t = torch.from_numpy(np.ascontiguousarray(local_rows).view(np.int64).reshape(-1))
        dev = self.comm._dev() if hasattr(self.comm, "_dev") else t.device
        out = self.comm.all_gather_cat(t.to(dev))
        return out.cpu().numpy().view(np.uint64)

    # collective calls: every rank makes the same call at the same time
    def add_entry(self, cm, op, lhs, rhs):
        return self.local.add_entry(self._mine(cm), op, lhs, rhs)

    def run_level(self, segments):
        return self.local.run_level(segments)

    def screen_unary(self, op, c0, c1):
        return self.local.screen_unary(op, c0, c1)

    def screen_binary(self, op, a0, a1, b0, b1, tri):
        return self.local.screen_binary(op, a0, a1, b0, b1, tri)

    def contains(self, cm):
        return self.local.contains(self._mine(cm))

    def fingerprint_of(self, cm):
        return self.local.fingerprint_of(self._mine(cm))

    def get_cm(self, idx):
        return self._gather_rows(self.local.get_cm(idx))

    # replicated state
    def get_record(self, idx):
        return self.local.get_record(idx)

    def export_records(self, first=0, count=None):
        return self.local.export_records(first, count)

    def counters(self):
        return self.local.counters()

    n_entries = property(lambda s: s.local.counters()[0])

    def set_option(self, name, value):
        if name == "deadline_ms":
            return  # every pass is collective: a rank that stopped alone would leave the others in the all-reduce
        self.local.set_option(name, value)

    def transfer_stats(self):
        return self.local.transfer_stats()

    def kernel_stats(self):
        return self.local.kernel_stats()

    def level_size(self, segments):
        return self.local.level_size(segments)

    def close(self):
        self.local.close()


def row_sharded_core_factory(comm, local_factory: Callable | None = None, shard_table: bool = True, **options):
    """A `core_factory` for `learner.Enumeration` / `learn`: this rank's `CudaCore` over its slice of the rows
    (``local_factory``: a CPU stand-in with the same `set_row_shard` contract, for the gloo tests).
    ``shard_table``: the uniqueness table is sharded by fingerprint owner too (`ltl_core_set_table_shard`), so that its
    memory and the filing of keys scale with the GPUs; False keeps a replica of the whole table on every GPU."""

    def make(masks, n_pos, err_max, variant, proj_rows, proj_offs, fkp_bits, mask_k, budget_bytes, *,
             words_per_row=1, device=0):
        W = int(words_per_row)
        m = np.ascontiguousarray(masks, dtype=np.uint64).reshape(-1)
        n_rows = len(m) // W
        try:
            r0, r1 = row_slices(n_rows, W, comm.world, half_width=int(variant) == 4)[comm.rank]
        except ValueError:
            if int(variant) != 4:
                raise
            # too few rows for whole 128-row blocks of the half-width store on every shard: full-width NH instead
            # (search results do not depend on which collision-free fingerprint is used, DESIGN 3)
            variant = 3
            r0, r1 = row_slices(n_rows, W, comm.world)[comm.rank]
        if local_factory is None:
            from .core import make_core as factory
        else:
            factory = local_factory
        local = factory(m[r0 * W: r1 * W], max(0, min(int(n_pos), r1) - r0), err_max, variant, proj_rows, proj_offs,
                        fkp_bits, mask_k, budget_bytes, words_per_row=W, device=device, **options)
        local.set_row_shard(r0 * W, n_rows * W, comm.all_reduce_sum)
        if shard_table and comm.world > 1 and hasattr(local, "set_table_shard"):
            local.set_table_shard(comm.rank, comm.world)
        # A solver is only known after the exchange, so a pass cannot stop early inside a chunk: keep chunks at 2^22
        # candidates (the search stops after the first chunk that holds a solver; the level it ends in is the largest)
        if "chunk_candidates" not in options:
            local.set_option("chunk_candidates", 1 << 22)
        return RowShardedCore(local, comm, r0, r1, n_rows, W)

    return make


def sharded_core_factory(comm, local_factory: Callable | None = None, **options):
    """A `core_factory` for `learner.Enumeration` / `learn`: this rank's `CudaCore` behind `ShardedCore`."""

    def make(masks, n_pos, err_max, variant, proj_rows, proj_offs, fkp_bits, mask_k, budget_bytes, *,
             words_per_row=1, device=0):
        if local_factory is None:
            from .core import make_core

            local = make_core(masks, n_pos, err_max, variant, proj_rows, proj_offs, fkp_bits, mask_k, budget_bytes,
                              words_per_row=words_per_row, device=device, **options)
        else:
            local = local_factory(masks, n_pos, err_max, variant, proj_rows, proj_offs, fkp_bits, mask_k,
                                  budget_bytes, words_per_row=words_per_row, device=device)
        return ShardedCore(local, comm)

    return make


# ------------------------------------------------------------------------------------------------ bench (N > 1)


def bench_main(args, spec, alphabet, planted, cfg_desc, sampler=None, peaks=None, cpu_baseline_fn=None):
    """`bench.py --gpus N` under torchrun: every rank runs the same search, sharded; device time of the K
    level loops, max over ranks; rank 0 prints the JSON line."""
    import json
    import time

    import torch
    import torch.distributed as dist

    from . import workloads as Wl
    from .formula import print_formula
    from .learner import Enumeration, LearnerConfig, Solved

    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    if not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    comm = TorchComm()
    max_cost = cfg_desc["max_cost"]
    from .scheme import HashScheme

    lcfg = LearnerConfig(ceiling=max_cost + 1, budget_bytes=int(args.budget_gb * (1 << 30)), device=local_rank,
                         pack_on_device=True, hash=HashScheme(getattr(args, "hash", "mueller")))
    mode = getattr(args, "sharding", "auto")
    if mode == "auto":
        try:
            row_slices(spec.size, -(-spec.max_len // 64), comm.world, half_width=spec.max_len <= 32)
            mode = "rows"
        except ValueError:
            mode = "candidates"
    make = row_sharded_core_factory if mode == "rows" else sharded_core_factory
    factory = make(comm, profile=True)

    def search():
        en = Enumeration(spec, alphabet, lcfg, core_factory=factory)
        en.keep_core = True
        return en

    res = None
    for _ in range(max(args.warmup, 3)):
        en = search()
        res = en.run()
        en.core.close()
    assert isinstance(res, Solved)
    text = print_formula(res.formula, alphabet)
    assert Wl.error_count(res.formula, spec, alphabet) == 0
    offered = res.stats.offered
    dev_ms = 0.0
    launches = 0
    kstats = []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    if sampler is not None and comm.rank == 0:
        sampler.start()
    for _ in range(args.steps):
        en = search()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        comm.barrier()
        torch.cuda.synchronize()
        ev0.record()
        en.run()
        ev1.record()
        comm.barrier()
        torch.cuda.synchronize()
        dev_ms += ev0.elapsed_time(ev1)
        kstats.append(en.core.local.kernel_stats())
        launches += sum(v["launches"] for v in kstats[-1].values())
        flush.fill_(1)  # L2 flush between timed iterations
        if getattr(en.core, "stage_ms", None) is not None and comm.rank == 0:
            import sys

            print("stage ms:", {k: round(v, 2) for k, v in en.core.stage_ms.items()},
                  {k: round(v["ms"], 2) for k, v in en.core.local.kernel_stats().items() if v["launches"]}, file=sys.stderr)
        en.core.close()
    clocks = sampler.stop() if sampler is not None and comm.rank == 0 else None
    # end to end: host trace arrays in (every rank packs and uploads its replica), formula text out
    from .traces import Specification

    pos_c, pos_l = spec.chars[: spec.n_pos].copy(), spec.lengths[: spec.n_pos].copy()
    neg_c, neg_l = spec.chars[spec.n_pos:].copy(), spec.lengths[spec.n_pos:].copy()
    e2e_factory = make(comm)

    def e2e_once():
        s = Specification.from_arrays(pos_c, pos_l, neg_c, neg_l)
        out = Enumeration(s, alphabet, lcfg, core_factory=e2e_factory).run()
        assert isinstance(out, Solved) and print_formula(out.formula, alphabet) == text
        return out

    e2e_once()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    comm.barrier()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        out = e2e_once()
    e1.record()
    comm.barrier()
    torch.cuda.synchronize()
    t = torch.tensor([dev_ms, e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, e2e_ms = float(t[0].item()), float(t[1].item())
    if comm.rank == 0:
        value = offered * args.steps / (total_ms / 1e3)
        cfg_desc = dict(cfg_desc, parallelism=(
            f"rows sharded over {comm.world} GPUs ({spec.size // comm.world} rows each), per-candidate partial fingerprints "
            f"all-reduced, entry store partitioned" if mode == "rows" else
            f"candidate ranges sharded over {comm.world} GPUs, hash-owner all-to-all, entry store replicated"))
        # roofline of rank 0's phase-A kernel (its share of the rows / candidates), same definition as at N = 1
        roofline = None
        scr_ms = sum(ks["screen"]["ms"] for ks in kstats)
        if scr_ms > 0:
            peak, peak_src = peaks if peaks else (6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)")
            scr_bytes = sum(ks["screen"]["alg_bytes"] for ks in kstats)
            scr_launch = sum(ks["screen"]["launches"] for ks in kstats)
            ach = scr_bytes / (scr_ms / 1e3) / 1e9
            roofline = {"bound": "hbm", "kernel": "k_screen (rank 0)", "achieved": ach, "peak": peak, "unit": "GB/s",
                        "frac": ach / peak, "traffic": None, "peak_source": peak_src,
                        "alg_bytes_per_launch": scr_bytes / max(scr_launch, 1), "ms_per_launch": scr_ms / max(scr_launch, 1),
                        "kernel_ms_by_class": {k: round(sum(ks[k]["ms"] for ks in kstats), 3) for k in kstats[0]}}
        cpu = cpu_baseline_fn() if cpu_baseline_fn is not None else None  # rank 0's host cores, after the timed regions
        print(json.dumps({
            "clocks": clocks, "roofline": roofline, "cpu_baseline": cpu,
            "metric": "candidates_per_sec", "value": value, "unit": "candidates/s", "n_gpus": comm.world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": cfg_desc, "gpu_launches": launches, "formula": text, "cost": res.cost,
            "e2e": {"value": offered * args.steps / (e2e_ms / 1e3), "unit": "candidates/s",
                    "ms_per_step": e2e_ms / args.steps, "h2d_bytes_per_step": out.stats.h2d_bytes,
                    "d2h_bytes_per_step": out.stats.d2h_bytes,
                    "note": "host trace arrays -> device packing -> sharded search -> formula text, per rank bytes"},
            "candidates_per_step": offered, "unique_cs_per_step": res.stats.admitted,
        }))
    dist.barrier()
    dist.destroy_process_group()
