#!/usr/bin/env python
"""Benchmark of the north-star hot path: bottom-up enumerative LTL search over characteristic sequences.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2_planted]

A "step" is one complete search (all cost levels, up to the minimal separating formula) on the synthetic
planted-formula specification of BASELINE config 2 (3 propositions, 512 + 512 traces of length 64).
metric = candidates/sec (`offered` candidates) over the level loop.

  value        inputs (packed atoms) already resident in HBM when the timed region starts
  e2e          the same metric through the public API `learn(P, N, ...)` from HOST trace arrays: packing,
               host->device copies, every level, device->host readback of records, formula text
  roofline     the dominant kernel (k_screen: evaluate + check + fingerprint + dedup), timed with CUDA events
               on its launching stream inside the timed region
  cpu_baseline the CPU oracle port (oracle/, all host threads) on a bounded sample of the same workload

One rank per GPU under torchrun for N > 1 (see paper_2402_12373_b200/sharded.py).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "candidates_per_sec"
UNIT = "candidates/s"


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except Exception:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
                for n, v in zip(names, r[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            except Exception:
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


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


def cpu_sample(spec, alphabet, sample_cost: int, threads: int, hash_name: str = "mueller"):
    """The CPU oracle port on the same specification, levels 2..sample_cost: (candidates, seconds)."""
    from paper_2402_12373_b200.learner import learn
    from paper_2402_12373_b200.scheme import HashScheme

    t0 = time.perf_counter()
    res = learn(spec, None, alphabet, max_cost=sample_cost, core_factory=oracle_factory(threads),
                overfit_on_ceiling=False, budget_bytes=48 << 30, hash=HashScheme(hash_name))
    return res.stats.offered, time.perf_counter() - t0, res


def run_reference_arm(args, spec, alphabet, cfg):
    """--impl reference: the reference algorithm's CPU implementation on this box's host cores.  The
    reference's own compiled core refuses > 64 traces (`_speedups.pyx:83-84`), so for this workload the arm
    runs the generalised oracle port (oracle/ltl_oracle.c) with every host thread, each step a bounded sample
    (cost levels 2..sample_cost of the same specification)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import cpu_oracle

    threads = cpu_oracle.max_threads()
    sample_cost = args.ref_sample_cost
    for _ in range(args.warmup):
        cpu_sample(spec, alphabet, min(sample_cost, 6), threads, args.hash)
    cands = secs = 0
    for _ in range(args.steps):
        c, s, _ = cpu_sample(spec, alphabet, sample_cost, threads, args.hash)
        cands += c
        secs += s
    value = cands / secs
    sample = f"cost levels 2..{sample_cost} of {cfg['workload']} ({cands // max(args.steps, 1)} candidates per step)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(args.steps, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2_planted")
    ap.add_argument("--max-cost", type=int, default=None)
    ap.add_argument("--cpu-sample-cost", type=int, default=9)
    ap.add_argument("--ref-sample-cost", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--budget-gb", type=float, default=150.0)
    ap.add_argument("--sharding", default="auto", choices=["auto", "rows", "candidates"],
                    help="N > 1: row shards (partial fingerprints all-reduced, store partitioned) or candidate ranges "
                         "(hash-owner all-to-all, store replicated); auto = rows when the rows cut into whole blocks")
    ap.add_argument("--hash", default="mueller", choices=["mueller", "mueller_blocked", "nh", "fkp"],
                    help="fingerprint scheme (scheme.py): 'mueller' = the reference's hash inside its domain, NH beyond")
    args = ap.parse_args()

    from paper_2402_12373_b200 import workloads as Wl
    from paper_2402_12373_b200.formula import print_formula
    from paper_2402_12373_b200.learner import Enumeration, LearnerConfig, Solved, learn

    spec, alphabet, planted, wl = Wl.make_config(args.config)
    max_cost = args.max_cost or wl["max_cost"]
    cfg_desc = {
        "workload": f"{args.config}: {wl['n_props']} props, {wl['n_pos']}+{wl['n_neg']} traces of length "
                    f"{wl['min_len']}..{wl['max_len']}, planted '{print_formula(planted, alphabet)}', max_cost {max_cost}",
        "rows": spec.size, "words_per_row": -(-spec.max_len // 64), "max_cost": max_cost, "seed": wl["seed"],
        "hash": args.hash,
        "l2": "inputs larger than L2 (entry store grows to GBs per step) + explicit 256 MiB L2 flush between steps",
    }
    if args.impl == "reference":
        return run_reference_arm(args, spec, alphabet, cfg_desc)

    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 or world > 1 or os.environ.get("LTL_FORCE_SHARDED"):  # the env switch: NCCL path on one GPU (tests)
        from paper_2402_12373_b200 import sharded

        return sharded.bench_main(args, spec, alphabet, planted, cfg_desc, sampler=ClockSampler(local_rank),
                                  peaks=load_peaks())

    torch.cuda.set_device(local_rank)
    budget = int(args.budget_gb * (1 << 30))
    from paper_2402_12373_b200.scheme import HashScheme

    lcfg = LearnerConfig(ceiling=max_cost + 1, budget_bytes=budget, device=local_rank, hash=HashScheme(args.hash),
                         pack_on_device=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def resident_search(profile: bool):
        """Create the core and admit the atoms (inputs resident in HBM), return the prepared search."""
        from paper_2402_12373_b200.core import make_core

        def factory(*a, **kw):
            return make_core(*a, **kw, profile=profile)

        en = Enumeration(spec, alphabet, lcfg, core_factory=factory)
        en.keep_core = True
        return en

    # ---- warm-up (also validates the answer)
    res = None
    for _ in range(max(args.warmup, 3)):
        en = resident_search(False)
        out = en.run()
        res = out
        en.core.close()
        flush.fill_(1)
    assert isinstance(res, Solved), f"workload did not solve within max_cost {max_cost}: {type(res).__name__}"
    text = print_formula(res.formula, alphabet)
    assert Wl.error_count(res.formula, spec, alphabet) == 0, "learned formula is not sound"
    offered_per_step = res.stats.offered

    # ---- timed: device-resident inputs.  Per step the core is created and the atoms are admitted OUTSIDE the
    # timed region (inputs resident in HBM), the cost-level loop runs INSIDE it, bracketed by CUDA events and a
    # device synchronize on both sides; the K timed intervals are summed.
    sampler = ClockSampler(local_rank)
    kstats, host_times, close_ms = [], [], 0.0
    launches = 0
    dev_ms = wall = 0.0
    torch.cuda.synchronize()
    sampler.start()
    for _ in range(args.steps):
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
    value = offered_per_step * args.steps / (total_ms / 1e3)
    for ks in kstats:
        launches += sum(v["launches"] for v in ks.values())

    # ---- roofline of the dominant kernel (k_screen), from the library's CUDA events on its launching stream
    peak, peak_src = load_peaks()
    scr_ms = sum(ks["screen"]["ms"] for ks in kstats)
    scr_bytes = sum(ks["screen"]["alg_bytes"] for ks in kstats)
    scr_launch = sum(ks["screen"]["launches"] for ks in kstats)
    achieved = scr_bytes / (scr_ms / 1e3) / 1e9 if scr_ms > 0 else 0.0
    traffic = insts = None
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as fh:
            prof = json.load(fh)
        traffic = prof.get("k_screen_dram_bytes_per_launch")
        if args.config == "c2_planted" and args.hash in ("mueller", "nh") and max_cost == wl["max_cost"]:
            insts = prof.get("k_screen_warp_instructions_per_step")  # deterministic for this workload (ncu count)
    except Exception:
        pass
    kernel_share = {k: round(sum(ks[k]["ms"] for ks in kstats), 3) for k in kstats[0]} if kstats else {}
    roofline = {"bound": "hbm", "kernel": "k_screen", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "alg_bytes_per_launch": scr_bytes / max(scr_launch, 1), "ms_per_launch": scr_ms / max(scr_launch, 1),
                "kernel_ms_by_class": kernel_share,
                "note": "algorithmic bytes = candidates x (arity x 8n + 16) (SURVEY 8d); operand lines are reused from "
                        "shared memory / L1 across the 128 candidates of a warp tile, so DRAM traffic is a fraction of "
                        "it and frac can exceed 1: the kernel is bound by integer issue, see `issue`"}
    if traffic and scr_ms > 0:
        dram = traffic * scr_launch / (scr_ms / 1e3) / 1e9
        roofline["dram"] = {"achieved": dram, "unit": "GB/s", "frac": dram / peak,
                            "source": "ncu dram__bytes_read+write per launch (profiles/roofline_traffic.json)"}
    mat_ms = sum(ks["materialize"]["ms"] for ks in kstats)
    mat_bytes = sum(ks["materialize"]["alg_bytes"] for ks in kstats)
    if mat_ms > 0:  # second kernel of the step: phase B (k_materialize / k_materialize_not), bound by HBM
        roofline["materialize"] = {"bound": "hbm", "kernel": "k_materialize_not + k_materialize",
                                   "achieved": mat_bytes / (mat_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                                   "frac": mat_bytes / (mat_ms / 1e3) / 1e9 / peak,
                                   "note": "algorithmic bytes = admitted entries x (8n + 16 + 9) written (SURVEY 8d) + "
                                           "16 per fused NOT candidate; the operand matrices it re-reads are not counted"}
        try:
            mt = prof.get("k_materialize_dram_bytes_per_step")
            if mt and args.config == "c2_planted" and max_cost == wl["max_cost"]:
                roofline["materialize"]["dram"] = {"achieved": mt * args.steps / (mat_ms / 1e3) / 1e9, "unit": "GB/s",
                                                   "frac": mt * args.steps / (mat_ms / 1e3) / 1e9 / peak,
                                                   "source": "ncu dram__bytes_read+write of one search "
                                                             "(profiles/roofline_traffic.json) / CUDA-event kernel time"}
        except Exception:
            pass
    if insts and scr_ms > 0 and clocks.get("sm_mhz"):
        sm_count = torch.cuda.get_device_properties(local_rank).multi_processor_count
        ipeak = sm_count * 4 * clocks["sm_mhz"] * 1e6  # one warp instruction per cycle per SM sub-partition
        iach = insts * args.steps / (scr_ms / 1e3)
        roofline["issue"] = {"bound": "warp-instruction issue", "achieved": iach, "peak": ipeak, "unit": "warp-inst/s",
                             "frac": iach / ipeak, "source": "ncu smsp__inst_executed.sum of one search "
                                                             "(profiles/roofline_traffic.json) / CUDA-event kernel time"}

    # ---- end to end through the public API, host buffers in, formula out
    pos_c, pos_l = spec.chars[: spec.n_pos].copy(), spec.lengths[: spec.n_pos].copy()
    neg_c, neg_l = spec.chars[spec.n_pos:].copy(), spec.lengths[spec.n_pos:].copy()
    from paper_2402_12373_b200.traces import Specification

    e2e_parts = {"spec_ms": 0.0, "learn_ms": 0.0}

    def e2e_once():
        ta = time.perf_counter()
        s = Specification.from_arrays(pos_c, pos_l, neg_c, neg_l)
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
    for _ in range(args.steps):
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
    e2e = {"value": offered_per_step * args.steps / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.steps,
           "host_ms_per_step": {k: v / (args.steps + 1) for k, v in e2e_parts.items()},
           "search_ms_last": 1e3 * r.stats.search_seconds, "host_ms_each_step": e2e_wall,
           "search_ms_each_step": e2e_search, "phase_ms_each_step": e2e_phase}

    # ---- CPU baseline on a bounded sample
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import cpu_oracle

        threads = cpu_oracle.max_threads()
        c, s, _ = cpu_sample(spec, alphabet, min(args.cpu_sample_cost, max_cost - 1), threads, args.hash)
        cpu = {"value": c / s, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"cost levels 2..{min(args.cpu_sample_cost, max_cost - 1)} of the same specification "
                         f"({c} candidates, {s:.1f} s)"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic", "config": cfg_desc, "clocks": clocks, "e2e": e2e,
        "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
        "time_to_formula_ms": e2e_ms / args.steps, "formula": text, "cost": res.cost,
        "candidates_per_step": offered_per_step, "unique_cs_per_step": res.stats.admitted,
        "wall_ms_per_step": 1e3 * wall / args.steps,
        "host_ms_per_step": {"grow": sum(h["grow_ms"] for h in host_times) / args.steps,
                             "device_wait": sum(h["sync_ms"] for h in host_times) / args.steps,
                             "close": close_ms / args.steps},
        "levels": [[lv["cost"], lv["offered"], lv["admitted"], lv.get("ms")] for lv in res.stats.levels],
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
