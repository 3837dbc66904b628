"""`learn` command line (the reference specifies it, `/root/reference/SPEC.md:569-608`, but ships none).

    python -m paper_2402_12373_b200.cli learn TRACE_FILE [--max-cost N] [--hash mueller|fkp|mueller_blocked|nh] [--mask-bits K]
        [--nnf] [--no-until] [--noise EPS] [--budget BYTES] [--costs a,n,c,d,x,f,g,u] [--timeout SECS]
        [--device D] [--json PATH] [--verify] [--dnc --window N --strategy det|rand --seed S --min-window M]
    torchrun --nproc-per-node G -m paper_2402_12373_b200.cli learn TRACE_FILE ... [--sharding auto|rows|candidates]

Reads a trace file (format `traces.py`, reference `traces.py:180-253`), runs the enumerative learner on the
B200 core and writes the JSON report of `SPEC.md:158`: {formula, cost, wall_ms, mode, hash, stats}.  Only the
`learn` subcommand is in scope (component 13).  With `--dnc` the specification is learned by divide
and conquer (`dnc.py`, reference `dnc.py:205-224`); without it by one enumeration (the reference needs D&C above
64 traces, this core does not).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

from .errors import BackendUnavailable, TimeoutExceeded
from .formula import parse_formula, print_formula
from .learner import learn
from .scheme import HashScheme
from .traces import TraceFormatError, load_spec


def cmd_learn(args) -> int:
    try:
        spec, alphabet = load_spec(args.trace_file)
    except (OSError, TraceFormatError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    costs = None if args.costs is None else [int(v) for v in args.costs.split(",")]
    t0 = time.perf_counter()
    report = {"input": args.trace_file, "n_pos": spec.n_pos, "n_neg": spec.n_neg, "max_len": spec.max_len,
              "config": {"max_cost": args.max_cost, "hash": args.hash, "mask_bits": args.mask_bits, "nnf": args.nnf,
                         "no_until": args.no_until, "noise": args.noise, "budget": args.budget, "costs": costs}}
    if args.dnc:
        return _learn_dnc(args, spec, alphabet, costs, report, t0)
    try:
        core_factory, device, rank = _distributed_factory(args, spec)
        report["config"]["gpus"] = int(os.environ.get("WORLD_SIZE", "1"))
        res = learn(spec, None, alphabet, max_cost=args.max_cost, costs=costs, require_nnf=args.nnf,
                    forbid_until=args.no_until, noise=args.noise,
                    hash=HashScheme(args.hash, args.mask_bits), budget_bytes=args.budget, deadline_s=args.timeout,
                    device=device, **({} if core_factory is None else {"core_factory": core_factory}))
        if rank != 0:  # every rank holds the same result; rank 0 reports it
            return 0 if res.status in ("solved", "ceiling") else 1
    except BackendUnavailable as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    except TimeoutExceeded:
        report.update(status="timeout", wall_ms=round(1e3 * (time.perf_counter() - t0), 3))
        _emit(report, args)
        return 4
    report.update(status=res.status, formula=res.text, cost=res.cost,
                  wall_ms=round(1e3 * (time.perf_counter() - t0), 3),
                  mode="precise" if res.stats.precise else "hashed", hash=args.hash, overfit_cost=res.stats.ceiling,
                  ratio=None if res.cost is None else res.cost / max(res.stats.ceiling, 1), stats=res.stats.as_dict())
    rc = 0 if res.status in ("solved", "ceiling") else 1
    if args.verify and res.formula is not None:
        from .workloads import error_count

        reparsed = parse_formula(print_formula(res.formula, alphabet), alphabet)
        errs = error_count(reparsed, spec, alphabet)
        report["verified_errors"] = errs
        allowed = int(args.noise * spec.size + 1e-9)
        if errs > allowed:
            print(f"error: learned formula misclassifies {errs} traces (allowed {allowed})", file=sys.stderr)
            rc = 5
    _emit(report, args)
    return rc


def _distributed_factory(args, spec):
    """Under torchrun (WORLD_SIZE > 1): one process per GPU, the search sharded over them (`sharded.py`).
    Returns (core_factory or None, device index, rank)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world <= 1 and not os.environ.get("LTL_FORCE_SHARDED"):  # the env switch: NCCL path on one GPU (tests)
        return None, args.device, 0
    import torch
    import torch.distributed as dist

    from . import sharded

    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    if not dist.is_initialized():
        import atexit

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        atexit.register(lambda: dist.is_initialized() and dist.destroy_process_group())
    comm = sharded.TorchComm()
    mode = args.sharding
    if mode == "auto":
        try:
            sharded.row_slices(spec.size, -(-spec.max_len // 64), world)
            mode = "rows"
        except ValueError:
            mode = "candidates"
    make = sharded.row_sharded_core_factory if mode == "rows" else sharded.sharded_core_factory
    return make(comm), local_rank, comm.rank


def _learn_dnc(args, spec, alphabet, costs, report, t0) -> int:
    """--dnc: divide and conquer (reference `dnc.py`) with every leaf on the device."""
    from . import dnc
    from .formula import CostHomomorphism, UNIFORM, cost as formula_cost, overfit_cost
    from .learner import LearnerConfig

    h = UNIFORM if costs is None else CostHomomorphism(tuple(costs))
    cfg = LearnerConfig(cost=h, require_nnf=args.nnf, forbid_until=args.no_until, noise=args.noise,
                        hash=HashScheme(args.hash, args.mask_bits), device=args.device,
                        ceiling=None if args.max_cost is None else args.max_cost + 1,
                        deadline=None if args.timeout is None else time.monotonic() + args.timeout,
                        **({} if args.budget is None else {"budget_bytes": args.budget}))
    split = dnc.SplitConfig(args.strategy, args.window, min(args.min_window, args.window), args.seed)
    report["config"].update(dnc=True, window=args.window, strategy=args.strategy, seed=args.seed)
    try:
        res = dnc.dnc_learn(spec, alphabet, cfg, split)
    except BackendUnavailable as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    except TimeoutExceeded:
        report.update(status="timeout", wall_ms=round(1e3 * (time.perf_counter() - t0), 3))
        _emit(report, args)
        return 4
    except dnc.WindowExhausted as exc:
        report.update(status="oom", error=str(exc), wall_ms=round(1e3 * (time.perf_counter() - t0), 3))
        _emit(report, args)
        return 1
    c, oc = formula_cost(res.formula, h), overfit_cost(spec, alphabet, h)
    report.update(status="solved", formula=print_formula(res.formula, alphabet), cost=c, overfit_cost=oc,
                  ratio=c / max(oc, 1), wall_ms=round(1e3 * (time.perf_counter() - t0), 3), hash=args.hash,
                  dnc={"nodes": res.nodes, "enum_calls": res.enum_calls})
    rc = 0
    if args.verify:
        reparsed = parse_formula(report["formula"], alphabet)
        ok = dnc.separates(reparsed, spec, alphabet)
        report["verified"] = ok
        if not ok and args.noise == 0.0:
            print("error: the recombined formula does not separate the input", file=sys.stderr)
            rc = 5
    _emit(report, args)
    return rc


def _emit(report, args):
    text = json.dumps(report, sort_keys=True)
    if args.json:
        with open(args.json, "w", encoding="utf-8") as fh:
            fh.write(text + "\n")
    else:
        print(text)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2402_12373_b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    lp = sub.add_parser("learn", help="learn a minimal separating LTL formula from a trace file")
    lp.add_argument("trace_file")
    lp.add_argument("--max-cost", type=int, default=None, help="inclusive cost bound (default: up to the overfit cost)")
    lp.add_argument("--hash", choices=["mueller", "fkp", "mueller_blocked", "nh"], default="mueller")
    lp.add_argument("--mask-bits", type=int, default=0)
    lp.add_argument("--nnf", action="store_true")
    lp.add_argument("--no-until", action="store_true")
    lp.add_argument("--noise", type=float, default=0.0)
    lp.add_argument("--budget", type=int, default=None, help="logical memory budget in bytes")
    lp.add_argument("--costs", default=None, help="8 weights: atom,not,and,or,next,finally,globally,until")
    lp.add_argument("--timeout", type=float, default=None)
    lp.add_argument("--device", type=int, default=0)
    lp.add_argument("--sharding", choices=["auto", "rows", "candidates"], default="auto",
                    help="under torchrun with several GPUs: row shards or candidate ranges (DESIGN.md section 8)")
    lp.add_argument("--json", default=None, help="write the report here instead of stdout")
    lp.add_argument("--verify", action="store_true", help="re-evaluate the learned formula on the input")
    lp.add_argument("--dnc", action="store_true", help="divide and conquer over windows of --window traces")
    lp.add_argument("--window", type=int, default=64)
    lp.add_argument("--min-window", type=int, default=4)
    lp.add_argument("--strategy", choices=["det", "rand"], default="rand")
    lp.add_argument("--seed", type=int, default=0)
    lp.set_defaults(fn=cmd_learn)
    args = ap.parse_args(argv)
    return args.fn(args)


if __name__ == "__main__":
    sys.exit(main())
