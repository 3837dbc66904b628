#!/usr/bin/env python
"""Benchmark of the north-star hot path: bottom-up enumerative LTL search over characteristic sequences.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2_planted]

A "step" is one complete search (all cost levels, up to the minimal separating formula) on a synthetic
specification of a BASELINE shape.  The headline workload is BASELINE config 2 (3 propositions, 512 + 512
traces of length 64, planted formula); the default run also measures the other four BASELINE shapes with short
step counts and reports them under `configs` (value / e2e / roofline / cpu_baseline each).
metric = candidates/sec (`offered` candidates) over the level loop.

  value        inputs (packed atoms) already resident in HBM when the timed region starts
  e2e          the same metric through the public API `learn(P, N, ...)` from HOST trace arrays: de-duplication,
               packing, host->device copies, every level, device->host readback of records, formula text
  roofline     the dominant kernel (k_screen: evaluate + check + fingerprint + dedup), timed with CUDA events on its
               launching stream inside the timed region.  The algorithmic-bytes figure of SURVEY 8d is always given;
               when an ncu pass of the SAME config / hash / max_cost is on file (profiles/roofline_traffic.json) the DRAM
               counter decides what bounds the kernel: algorithmic / DRAM > 1.2 means the operands come from shared
               memory / L1 / L2, the kernel is bound by instruction issue and `frac` is the issue fraction
  cpu_baseline the CPU oracle port (oracle/, all host threads; config 1: the reference's own compiled core) on a
               bounded sample of the same workload, plus its single-thread rate

`--gpus N` with N > 1 and no torchrun environment re-launches itself under `python -m torch.distributed.run`
(one rank per GPU, NCCL; see paper_2402_12373_b200/sharded.py).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402,F401

METRIC = "candidates_per_sec"
UNIT = "candidates/s"
HEADLINE = "c2_planted"
#: the other BASELINE shapes measured by the default run: (steps, warm-up, cost bound of the CPU sample)
SIDE_CONFIGS = {"c1_tiny": (20, 5, 10), "c3_long": (3, 3, 7), "c4_many": (2, 3, 4), "c5_deep": (5, 3, 6)}
CPU_SAMPLE_COST = {"c1_tiny": 10, "c2_planted": 9, "c3_long": 7, "c4_many": 4, "c5_deep": 6}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_profile_entry(config: str, hash_name: str, max_cost: int):
    """The ncu counters on file for exactly this workload (config, hash scheme, cost bound), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as fh:
            prof = json.load(fh)
        return prof.get("entries", {}).get(f"{config}|{hash_name}|{max_cost}")
    except Exception:
        return None


def sources_digest() -> str:
    try:
        from paper_2402_12373_b200 import build as B

        return B._sources_digest()[:16]
    except Exception:
        return ""


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region: the sampler runs from before the warm-up
    (nvidia-smi needs ~0.2 s to produce its first line), `mark()` is called when the timed region starts, and only lines
    that arrived after it count.  A region shorter than the 100 ms period may see none: then the last line before it --
    taken under the same load, during the warm-up -- is reported with `"samples": 0, "nearest": true`."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc, self.t_mark = index, [], None, 0.0

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except Exception:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), [c.strip() for c in line.split(",")]))

    def mark(self):
        self.t_mark = time.perf_counter()

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        rows = [r for t, r in self.rows if t >= self.t_mark]
        nearest = not rows and bool(self.rows)
        if nearest:
            rows = [self.rows[-1][1]]
        for r in rows:
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
                for n, v in zip(names, r[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            except Exception:
                pass
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
               "samples": 0 if nearest else len(sm), "reasons": sorted(reasons)}
        if nearest:
            out["nearest"] = True
        return out


# ------------------------------------------------------------------------------------------------ CPU arm


def oracle_factory(threads: int):
    from oracle import cpu_oracle
    from paper_2402_12373_b200 import errors as E

    class _Oracle(cpu_oracle.OracleCore):
        def add_entry(self, *a):
            try:
                return super().add_entry(*a)
            except cpu_oracle.CoreOOM:
                raise E.CoreOOM from None

        counters = cpu_oracle.OracleCore._counters

    def make(masks, n_pos, err_max, variant, pr, po, fkp, mask_k, budget, *, words_per_row=1, device=None):
        return _Oracle(masks, n_pos, err_max, variant, pr, po, fkp, mask_k, budget, words_per_row=words_per_row,
                       threads=threads)

    return make


def reference_core_factory():
    """The reference's OWN compiled core (oracle/_ref, built from _speedups.pyx by oracle/build_ref.sh) behind the
    core-factory signature: only inside the reference's limits (<= 64 traces of <= 63 positions)."""
    sys.path.insert(1, os.path.join(ROOT, "oracle", "_ref"))
    from ltllearn import _speedups as S  # noqa: E402
    from paper_2402_12373_b200 import errors as E

    oom = sys.modules["ltllearn._kernels_py"].CoreOOM

    class _Ref:
        def __init__(self, core):
            self._c = core

        def add_entry(self, cm, op, lhs, rhs):
            try:
                return self._c.add_entry(np.ascontiguousarray(cm, dtype=np.uint64).reshape(-1), op, lhs, rhs)
            except oom:
                raise E.CoreOOM from None

        def counters(self):
            c = self._c
            return [c.n_entries, c.bytes_used, c.offered, c.admitted, c.duplicates]

        def __getattr__(self, name):
            return getattr(self._c, name)

    def make(masks, n_pos, err_max, variant, pr, po, fkp, mask_k, budget, *, words_per_row=1, device=None):
        if words_per_row != 1:
            raise ValueError("the reference core holds one word per row")
        m = np.ascontiguousarray(masks, dtype=np.uint64).reshape(-1)
        return _Ref(S.Core(m, n_pos, err_max, variant, list(pr), list(po), fkp, mask_k, budget))

    return make


def cpu_sample(spec, alphabet, sample_cost: int, threads: int, hash_name: str = "mueller", factory=None):
    """The CPU arm on the same specification, cost levels 2..sample_cost: (candidates, seconds, result)."""
    from paper_2402_12373_b200.learner import learn
    from paper_2402_12373_b200.scheme import HashScheme

    t0 = time.perf_counter()
    res = learn(spec, None, alphabet, max_cost=sample_cost, core_factory=factory or oracle_factory(threads),
                overfit_on_ceiling=False, budget_bytes=48 << 30, hash=HashScheme(hash_name))
    return res.stats.offered, time.perf_counter() - t0, res


def cpu_baseline(config: str, spec, alphabet, sample_cost: int, hash_name: str) -> dict:
    """All host threads on a bounded sample + the single-thread rate on a (smaller) sample of the same workload.
    Config 1 lies inside the reference's limits: there the reference's own compiled core does the work (kind
    "reference", one thread by construction); elsewhere the generalised oracle port."""
    from oracle import cpu_oracle

    threads = cpu_oracle.max_threads()
    if spec.size <= 64 and spec.max_len <= 63 and os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "ltllearn")):
        try:
            fac = reference_core_factory()
            cpu_sample(spec, alphabet, sample_cost, 1, hash_name, factory=fac)
            c = s = 0
            for _ in range(20):
                ci, si, _ = cpu_sample(spec, alphabet, sample_cost, 1, hash_name, factory=fac)
                c, s = c + ci, s + si
            return {"value": c / s, "unit": UNIT, "cores": 1, "kind": "reference",
                    "sample": f"20 searches to max_cost {sample_cost} of the same specification with the reference's own "
                              f"compiled core (oracle/_ref), driven by this repo's level loop ({c} candidates, {s:.3f} s)"}
        except Exception:
            pass
    c, s, _ = cpu_sample(spec, alphabet, sample_cost, threads, hash_name)
    c1, s1, _ = cpu_sample(spec, alphabet, max(2, sample_cost - 1), 1, hash_name)
    return {"value": c / s, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"cost levels 2..{sample_cost} of the same specification ({c} candidates, {s:.1f} s)",
            "single_thread": {"value": c1 / s1, "unit": UNIT, "cores": 1,
                              "sample": f"cost levels 2..{max(2, sample_cost - 1)} ({c1} candidates, {s1:.1f} s)"}}


def workload_desc(config, spec, wl, planted, alphabet, max_cost, hash_name):
    from paper_2402_12373_b200.formula import print_formula

    return {
        "workload": f"{config}: {wl['n_props']} props, {wl['n_pos']}+{wl['n_neg']} traces of length "
                    f"{wl['min_len']}..{wl['max_len']}, planted '{print_formula(planted, alphabet)}', max_cost {max_cost}",
        "rows": spec.size, "words_per_row": -(-spec.max_len // 64), "max_cost": max_cost, "seed": wl["seed"],
        "hash": hash_name,
        "l2": "inputs larger than L2 (entry store grows to GBs per step) + explicit 256 MiB L2 flush between steps",
    }


def run_reference_arm(args):
    """--impl reference: the reference algorithm's CPU implementation on this box's host cores.  The
    reference's own compiled core refuses > 64 traces (`_speedups.pyx:83-84`), so for the headline workload the arm
    runs the generalised oracle port (oracle/ltl_oracle.c) with every host thread, each step a bounded sample
    (cost levels 2..sample_cost of the same specification); config 1 runs on the reference's own compiled core."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import cpu_oracle
    from paper_2402_12373_b200 import workloads as Wl

    spec, alphabet, planted, wl = Wl.make_config(args.config)
    max_cost = args.max_cost or wl["max_cost"]
    cfg = workload_desc(args.config, spec, wl, planted, alphabet, max_cost, args.hash)
    threads = cpu_oracle.max_threads()
    sample_cost = args.ref_sample_cost or max(2, CPU_SAMPLE_COST.get(args.config, 6) - (1 if args.config == HEADLINE else 0))
    kind, factory = "port", None
    if spec.size <= 64 and spec.max_len <= 63 and os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "ltllearn")):
        try:
            factory, kind, threads = reference_core_factory(), "reference", 1
        except Exception:
            factory = None
    for _ in range(args.warmup):
        cpu_sample(spec, alphabet, min(sample_cost, 6), threads, args.hash, factory)
    cands = secs = 0
    for _ in range(args.steps):
        c, s, _ = cpu_sample(spec, alphabet, sample_cost, threads, args.hash, factory)
        cands += c
        secs += s
    value = cands / secs
    sample = f"cost levels 2..{sample_cost} of {cfg['workload']} ({cands // max(args.steps, 1)} candidates per step)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(args.steps, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ------------------------------------------------------------------------------------------------ GPU arm, N = 1


def build_roofline(kstats, steps, clocks, config, hash_name, max_cost, sm_count):
    """Roofline record of k_screen (and phase B beside it) from the library's CUDA-event times of the timed region."""
    peak, peak_src = load_peaks()
    scr_ms = sum(ks["screen"]["ms"] for ks in kstats)
    scr_bytes = sum(ks["screen"]["alg_bytes"] for ks in kstats)
    scr_launch = sum(ks["screen"]["launches"] for ks in kstats)
    alg = scr_bytes / (scr_ms / 1e3) / 1e9 if scr_ms > 0 else 0.0
    entry = load_profile_entry(config, hash_name, max_cost)
    kernel_share = {k: round(sum(ks[k]["ms"] for ks in kstats), 3) for k in kstats[0]} if kstats else {}
    roof = {"kernel": "k_screen", "peak_source": peak_src, "launches": scr_launch,
            "alg_bytes_per_launch": scr_bytes / max(scr_launch, 1), "ms_per_launch": scr_ms / max(scr_launch, 1),
            "kernel_ms_by_class": kernel_share,
            "hbm_algorithmic": {"achieved": alg, "peak": peak, "unit": "GB/s", "frac": alg / peak,
                                "note": "candidates x (arity x stored matrix bytes + 16) / CUDA-event time (SURVEY 8d); "
                                        "exceeds the DRAM figure whenever operands are reused from smem / L1 / L2"}}
    dram = None
    if entry and scr_ms > 0:
        per_step = entry["k_screen_dram_bytes_per_step"]
        dram = per_step * steps / (scr_ms / 1e3) / 1e9
        roof["hbm_dram"] = {"achieved": dram, "peak": peak, "unit": "GB/s", "frac": dram / peak,
                            "bytes_per_step": per_step, "l2_hit_pct": entry.get("k_screen_l2_hit_pct"),
                            "atomics_per_step": entry.get("k_screen_atom_ops_per_step"),
                            "source": f"ncu dram__bytes_read+write of one search ({entry.get('source')}) / CUDA-event time"}
        roof["traffic"] = per_step / max(entry.get("k_screen_launches", 1), 1)
        roof["profile_build_matches"] = entry.get("build_digest") == sources_digest()
        insts = entry.get("k_screen_warp_instructions_per_step")
        if insts and clocks.get("sm_mhz"):
            ipeak = sm_count * 4 * clocks["sm_mhz"] * 1e6  # one warp instruction per cycle per SM sub-partition
            iach = insts * steps / (scr_ms / 1e3)
            roof["issue"] = {"achieved": iach, "peak": ipeak, "unit": "warp-inst/s", "frac": iach / ipeak,
                             "source": "ncu smsp__inst_executed.sum of one search / CUDA-event time"}
    else:
        roof["traffic"] = None
    if dram and alg / dram > 1.2 and "issue" in roof:
        roof.update({"bound": "issue", "achieved": roof["issue"]["achieved"], "peak": roof["issue"]["peak"],
                     "unit": "warp-inst/s", "frac": roof["issue"]["frac"],
                     "why": f"algorithmic / DRAM bytes = {alg / dram:.1f}: operands are served from shared memory / L1 / L2, "
                            "the kernel is bound by integer instruction issue, not by HBM"})
    elif dram:
        roof.update({"bound": "hbm", "achieved": dram, "peak": peak, "unit": "GB/s", "frac": dram / peak,
                     "why": "DRAM counter within 1.2x of the algorithmic bytes: HBM-bound; achieved = DRAM bytes / time"})
    else:
        roof.update({"bound": "hbm", "achieved": alg, "peak": peak, "unit": "GB/s", "frac": alg / peak,
                     "why": "no ncu pass on file for this config / hash / max_cost: algorithmic bytes only (a fraction above 1 "
                            "means operand reuse from L2 / shared memory, not HBM traffic)"})
    mat_ms = sum(ks["materialize"]["ms"] for ks in kstats)
    mat_bytes = sum(ks["materialize"]["alg_bytes"] for ks in kstats)
    if mat_ms > 0:  # second kernel of the step: phase B (k_materialize / k_materialize_not), bound by HBM
        m = {"bound": "hbm", "kernel": "k_materialize_not + k_materialize", "achieved": mat_bytes / (mat_ms / 1e3) / 1e9,
             "peak": peak, "unit": "GB/s", "frac": mat_bytes / (mat_ms / 1e3) / 1e9 / peak,
             "note": "algorithmic bytes = admitted entries x (stored matrix bytes + 16 + 9) written (SURVEY 8d) + 16 per fused "
                     "NOT candidate; the operand matrices it re-reads are not counted; a fused launch whose store gate was closed "
                     "(the level solved: DESIGN.md 4, gated store) is booked as the NOT pass it was, entries x (matrix bytes + 16)"}
        # (the DRAM bytes of phase B are only quoted from a pass over this very build: its launches are what changes)
        if entry and entry.get("build_digest") == sources_digest() and entry.get("k_materialize_dram_bytes_per_step"):
            mt = entry["k_materialize_dram_bytes_per_step"]
            m["dram"] = {"achieved": mt * steps / (mat_ms / 1e3) / 1e9, "unit": "GB/s",
                         "frac": mt * steps / (mat_ms / 1e3) / 1e9 / peak, "bytes_per_step": mt,
                         "source": "ncu dram__bytes_read+write of one search / CUDA-event kernel time"}
        roof["materialize"] = m
    return roof


def measure_config(config: str, args, *, steps: int, warmup: int, cpu_cost: int | None, local_rank: int = 0) -> dict:
    """value, e2e, roofline, cpu_baseline of one BASELINE shape on one GPU (the JSON line without the envelope)."""
    import torch

    from paper_2402_12373_b200 import workloads as Wl
    from paper_2402_12373_b200.core import make_core
    from paper_2402_12373_b200.formula import print_formula
    from paper_2402_12373_b200.learner import Enumeration, LearnerConfig, Solved, as_specification, learn
    from paper_2402_12373_b200.scheme import HashScheme
    spec, alphabet, planted, wl = Wl.make_config(config)
    max_cost = (args.max_cost if config == args.config and args.max_cost else None) or wl["max_cost"]
    cfg_desc = workload_desc(config, spec, wl, planted, alphabet, max_cost, args.hash)
    budget = int(args.budget_gb * (1 << 30))
    lcfg = LearnerConfig(ceiling=max_cost + 1, budget_bytes=budget, device=local_rank, hash=HashScheme(args.hash),
                         pack_on_device=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def resident_search(profile: bool):
        """Create the core and admit the atoms (inputs resident in HBM), return the prepared search."""

        def factory(*a, **kw):
            return make_core(*a, **kw, profile=profile)

        en = Enumeration(spec, alphabet, lcfg, core_factory=factory)
        en.keep_core = True
        return en

    # ---- warm-up (also validates the answer)
    sampler = ClockSampler(local_rank)
    sampler.start()
    res = None
    for _ in range(max(warmup, 3)):
        en = resident_search(False)
        res = en.run()
        en.core.close()
        flush.fill_(1)
    assert isinstance(res, Solved), f"workload did not solve within max_cost {max_cost}: {type(res).__name__}"
    text = print_formula(res.formula, alphabet)
    assert Wl.error_count(res.formula, spec, alphabet) == 0, "learned formula is not sound"
    offered_per_step = res.stats.offered

    # ---- timed: device-resident inputs.  Per step the core is created and the atoms are admitted OUTSIDE the
    # timed region (inputs resident in HBM), the cost-level loop runs INSIDE it, bracketed by CUDA events and a
    # device synchronize on both sides; the K timed intervals are summed.
    kstats, host_times, close_ms = [], [], 0.0
    launches = 0
    dev_ms = wall = 0.0
    torch.cuda.synchronize()
    sampler.mark()
    for _ in range(steps):
        en = resident_search(True)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record()
        t0 = time.perf_counter()
        en.run()
        ev1.record()
        torch.cuda.synchronize()
        wall += time.perf_counter() - t0
        dev_ms += ev0.elapsed_time(ev1)
        kstats.append(en.core.kernel_stats())
        host_times.append(en.core.host_times())
        tc = time.perf_counter()
        en.core.close()
        close_ms += 1e3 * (time.perf_counter() - tc)
        flush.fill_(1)  # L2 flush between timed iterations
    torch.cuda.synchronize()
    clocks = sampler.stop()
    total_ms = max(dev_ms, 1e-6)
    value = offered_per_step * steps / (total_ms / 1e3)
    for ks in kstats:
        launches += sum(v["launches"] for v in ks.values())
    sm_count = torch.cuda.get_device_properties(local_rank).multi_processor_count
    roofline = build_roofline(kstats, steps, clocks, config, args.hash, max_cost, sm_count)

    # ---- end to end through the public API, host buffers in, formula out
    # the step's inputs live in PINNED host memory (numpy views of pinned torch tensors): the library's cudaMemcpyAsync then
    # runs at PCIe speed instead of staging pageable memory (config 4: 134 MB per step)
    def pinned(a):
        a = np.ascontiguousarray(a)
        t = torch.from_numpy(a.view(np.uint8).reshape(-1)).pin_memory()  # (bytes: every torch build pins uint8)
        return t.numpy().view(a.dtype).reshape(a.shape)

    pos_c, pos_l = pinned(spec.chars[: spec.n_pos]), pinned(spec.lengths[: spec.n_pos])
    neg_c, neg_l = pinned(spec.chars[spec.n_pos:]), pinned(spec.lengths[spec.n_pos:])
    e2e_parts = {"spec_ms": 0.0, "learn_ms": 0.0}

    def e2e_once():
        ta = time.perf_counter()
        # host arrays in: uploaded, screened for duplicates, censused and packed on the device (core.DeviceTraces)
        s = as_specification((pos_c, pos_l), (neg_c, neg_l), device=local_rank)
        tb = time.perf_counter()
        out = learn(s, None, alphabet, max_cost=max_cost, budget_bytes=budget, device=local_rank,
                    hash=HashScheme(args.hash))
        e2e_parts["spec_ms"] += 1e3 * (tb - ta)
        e2e_parts["learn_ms"] += 1e3 * (time.perf_counter() - tb)
        return out

    r = e2e_once()
    assert r.text == text
    if os.environ.get("LTL_BENCH_PROFILE"):  # where does the end-to-end call spend host time?
        import cProfile
        import pstats

        pr = cProfile.Profile()
        pr.enable()
        e2e_once()
        pr.disable()
        pstats.Stats(pr, stream=sys.stderr).sort_stats("cumulative").print_stats(25)
    h2d = d2h = 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    e2e_wall, e2e_search, e2e_phase = [], [], []
    for _ in range(steps):
        tw = time.perf_counter()
        r = e2e_once()
        e2e_wall.append(round(1e3 * (time.perf_counter() - tw), 2))
        e2e_search.append(round(1e3 * r.stats.search_seconds, 2))
        e2e_phase.append({k: round(v, 2) for k, v in r.stats.phase_ms.items()})
        h2d, d2h = r.stats.h2d_bytes, r.stats.d2h_bytes
        flush.fill_(1)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    e2e = {"value": offered_per_step * steps / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / steps,
           "host_ms_per_step": {k: v / (steps + 1) for k, v in e2e_parts.items()},
           "search_ms_last": 1e3 * r.stats.search_seconds, "host_ms_each_step": e2e_wall[:8],
           "search_ms_each_step": e2e_search[:8], "phase_ms_each_step": e2e_phase[:3]}
    del flush

    # ---- CPU baseline on a bounded sample
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(config, spec, alphabet, min(cpu_cost or CPU_SAMPLE_COST.get(config, 6), max_cost), args.hash)

    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": steps, "warmup": max(warmup, 3),
        "ms_per_step": total_ms / steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic", "config": cfg_desc, "clocks": clocks, "e2e": e2e,
        "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
        "time_to_formula_ms": e2e_ms / steps, "formula": text, "cost": res.cost,
        "candidates_per_step": offered_per_step, "unique_cs_per_step": res.stats.admitted,
        "wall_ms_per_step": 1e3 * wall / steps,
        "host_ms_per_step": {"grow": sum(h["grow_ms"] for h in host_times) / steps,
                             "device_wait": sum(h["sync_ms"] for h in host_times) / steps,
                             "close": close_ms / steps},
        "levels": [[lv["cost"], lv["offered"], lv["admitted"], lv.get("ms")] for lv in res.stats.levels],
    }


# ------------------------------------------------------------------------------------------------ launcher


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch_command(n: int, argv: list[str]) -> list[str]:
    """The torchrun command `python bench.py --gpus N` replaces itself with when it was started without one."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr",
            "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__), *argv]


def maybe_self_launch(args, argv):
    """`python bench.py --gpus N` (N > 1) outside torchrun: check the box has N GPUs, then re-exec under
    torch.distributed.run (one rank per GPU).  NCCL's init log stays on so the launch shows its ranks."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return
    if not os.environ.get("LTL_BENCH_LAUNCH_ONLY"):  # (tests: exercise the re-exec without GPUs)
        import torch

        have = torch.cuda.device_count() if torch.cuda.is_available() else 0
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices on this node, found {have} "
                  "(one process per GPU over NCCL; there is no CPU fallback)", file=sys.stderr)
            sys.exit(2)
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = self_launch_command(args.gpus, argv)
    sys.stdout.flush()
    os.execv(cmd[0], cmd)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=HEADLINE)
    ap.add_argument("--max-cost", type=int, default=None)
    ap.add_argument("--cpu-sample-cost", type=int, default=None)
    ap.add_argument("--ref-sample-cost", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--configs", default="auto",
                    help="other BASELINE shapes to measure beside the headline: 'auto' (all four when the headline is "
                         "config 2), 'none', or a comma-separated list")
    ap.add_argument("--budget-gb", type=float, default=150.0)
    ap.add_argument("--sharding", default="auto", choices=["auto", "rows", "candidates"],
                    help="N > 1: row shards (partial fingerprints all-reduced, store partitioned) or candidate ranges "
                         "(hash-owner all-to-all, store replicated); auto = rows when the rows cut into whole blocks")
    ap.add_argument("--hash", default="mueller", choices=["mueller", "mueller_blocked", "nh", "fkp"],
                    help="fingerprint scheme (scheme.py): 'mueller' = the reference's hash inside its domain, NH beyond")
    args = ap.parse_args(argv)

    if args.impl == "reference":
        return run_reference_arm(args)
    maybe_self_launch(args, argv)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("LTL_BENCH_LAUNCH_ONLY"):  # tests of the launcher: say who we are and leave
        sys.stdout.write(json.dumps({"launch_only": True, "rank": rank, "world": world, "local_rank": local_rank,
                                     "master": os.environ.get("MASTER_ADDR")}) + "\n")  # one write: ranks share the pipe
        sys.stdout.flush()
        return
    if args.gpus > 1 or world > 1 or os.environ.get("LTL_FORCE_SHARDED"):  # the env switch: NCCL path on one GPU (tests)
        from paper_2402_12373_b200 import sharded
        from paper_2402_12373_b200 import workloads as Wl

        spec, alphabet, planted, wl = Wl.make_config(args.config)
        max_cost = args.max_cost or wl["max_cost"]
        cfg_desc = workload_desc(args.config, spec, wl, planted, alphabet, max_cost, args.hash)
        cpu_fn = None
        if not args.no_cpu_baseline:
            cpu_fn = lambda: cpu_baseline(args.config, spec, alphabet,  # noqa: E731
                                          min(args.cpu_sample_cost or CPU_SAMPLE_COST.get(args.config, 6), max_cost), args.hash)
        return sharded.bench_main(args, spec, alphabet, planted, cfg_desc, sampler=ClockSampler(local_rank),
                                  peaks=load_peaks(), cpu_baseline_fn=cpu_fn)

    import torch

    torch.cuda.set_device(local_rank)
    line = measure_config(args.config, args, steps=args.steps, warmup=args.warmup, cpu_cost=args.cpu_sample_cost,
                          local_rank=local_rank)
    names = []
    if args.configs == "auto":
        names = list(SIDE_CONFIGS) if args.config == HEADLINE and not args.max_cost else []
    elif args.configs != "none":
        names = [c for c in args.configs.split(",") if c and c != args.config]
    if names:
        side = {}
        keep = ("value", "unit", "steps", "warmup", "ms_per_step", "config", "clocks", "e2e", "gpu_launches", "roofline",
                "cpu_baseline", "time_to_formula_ms", "formula", "cost", "candidates_per_step", "unique_cs_per_step")
        for name in names:
            st, wu, cc = SIDE_CONFIGS.get(name, (3, 3, None))
            try:
                from paper_2402_12373_b200.core import pool_trim

                pool_trim()  # the previous shape's arena (tens of GB mapped) goes back to the driver
                full = measure_config(name, args, steps=st, warmup=wu, cpu_cost=cc, local_rank=local_rank)
                full["e2e"] = {k: v for k, v in full["e2e"].items() if k in ("value", "unit", "h2d_bytes_per_step",
                                                                            "d2h_bytes_per_step", "ms_per_step",
                                                                            "host_ms_per_step")}
                side[name] = {k: full[k] for k in keep}
            except Exception as exc:  # noqa: BLE001 -- a side config must not take the headline line down
                side[name] = {"error": f"{type(exc).__name__}: {exc}"}
        line["configs"] = side
    print(json.dumps(line))


if __name__ == "__main__":
    main()
