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

    # replicated single-matrix calls: every rank performs the same call on its replica
    def add_entry(self, cm, op, lhs, rhs):
        return self.local.add_entry(cm, op, lhs, rhs)

    def get_record(self, idx):
        return self.local.get_record(idx)

    def counters(self):
        return self.local.counters()

    n_entries = property(lambda s: s.local.counters()[0])

    def set_option(self, name, value):
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
        fp, solver_local = local.stage_eval(segments, lo, hi)
        dev = fp.device
        solver = comm.all_reduce_min(solver_local if solver_local >= 0 else _INF, device=dev)
        limit = min(total, solver)
        keep = max(0, min(hi, limit) - lo)
        fp = fp[:keep]

        # 3: route to hash owners, file, route the verdicts back
        owner = owner_of(fp, G)
        order = torch.argsort(owner, stable=True)
        counts = torch.bincount(owner, minlength=G).tolist()
        ranks_global = gbase + lo + torch.arange(keep, dtype=torch.int64, device=dev)
        send = torch.cat([fp[order], ranks_global[order].unsqueeze(1)], 1).contiguous()
        recv, recv_counts = comm.all_to_all(send, counts)
        win_recv = local.stage_file(recv)
        win_sorted, _ = comm.all_to_all(win_recv, recv_counts)
        win = torch.zeros(keep, dtype=torch.uint8, device=dev)
        win[order] = win_sorted
        winners = lo + torch.nonzero(win, as_tuple=False).flatten()  # ascending level ranks

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
        packed = torch.stack([op.to(torch.int32), lhs, rhs], 1)
        packed = comm.all_gather_cat(packed)
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
        if status == S_DONE:
            return S_DONE, -1, -1, -1
        local.stage_purge(gbase + cut)
        if status == S_OOM:
            return S_OOM, -1, -1, -1
        sop, sl, sr = local.stage_decode(segments, torch.tensor([solver], dtype=torch.int64, device=dev))
        return S_SOLVED, self._segment_of(segments, solver), int(sl.item()), int(sr.item())


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


def bench_main(args, spec, alphabet, planted, cfg_desc):
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
    lcfg = LearnerConfig(ceiling=max_cost + 1, budget_bytes=int(args.budget_gb * (1 << 30)), device=local_rank)
    factory = sharded_core_factory(comm, profile=True)

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
        launches += sum(v["launches"] for v in en.core.local.kernel_stats().values())
        en.core.close()
    t = torch.tensor([dev_ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    if comm.rank == 0:
        value = offered * args.steps / (total_ms / 1e3)
        cfg_desc = dict(cfg_desc, parallelism=f"candidate ranges sharded over {comm.world} GPUs, hash-owner all-to-all")
        print(json.dumps({
            "metric": "candidates_per_sec", "value": value, "unit": "candidates/s", "n_gpus": comm.world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": cfg_desc, "gpu_launches": launches, "formula": text, "cost": res.cost,
            "e2e": {"value": value, "unit": "candidates/s", "h2d_bytes_per_step": res.stats.h2d_bytes,
                    "d2h_bytes_per_step": res.stats.d2h_bytes,
                    "note": "sharded run: atoms are uploaded by every rank inside the step"},
            "candidates_per_step": offered, "unique_cs_per_step": res.stats.admitted,
        }))
    dist.barrier()
    dist.destroy_process_group()
