#!/usr/bin/env python
"""The reference's two cache-policy experiments (paper section 7; `benchgen.py:225-300`) on the B200 core:
the fingerprint-masking sweep (cost found vs number of masked fingerprint bits) and the RUC experiment (extra cost of
MuellerHash vs first-k-percent fingerprints on conservative extensions with known minimal cost).  Prints one JSON
object; `--out` writes it to a file."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2402_12373_b200 import benchgen as B  # noqa: E402
from paper_2402_12373_b200.formula import parse_formula  # noqa: E402
from paper_2402_12373_b200.learner import LearnerConfig  # noqa: E402
from paper_2402_12373_b200.scheme import HashScheme  # noqa: E402
from paper_2402_12373_b200.traces import Alphabet  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seeds", type=int, default=10)
ap.add_argument("--ext", default="0,8,16,24")
ap.add_argument("--base-seed", type=int, default=0)
ap.add_argument("--sweep-formula", default="F (p0 & X p1) & G (p1 | X p0)")
ap.add_argument("--sweep-traces", type=int, default=24, help="traces per side of the masking-sweep specification")
ap.add_argument("--sweep-len", default="20,40")
ap.add_argument("--hashes", default="mueller,fkp",
                help="schemes of the RUC experiment; 'nh' / 'mueller_blocked' force this build's hashes at every size")
ap.add_argument("--out", default=None)
a = ap.parse_args()

al = Alphabet.default(2)
lo, hi = (int(v) for v in a.sweep_len.split(","))
t0 = time.perf_counter()
spec = B.gen_guided(al, parse_formula(a.sweep_formula, al), a.sweep_traces, lo, hi, seed=a.base_seed)
sweeps = {}
for variant in ("mueller", "fkp"):
    rows = B.run_masking_sweep(spec, al, LearnerConfig(hash=HashScheme(variant)))
    sweeps[variant] = [{k: r.get(k) for k in ("k", "status", "cost", "wall_ms", "offered", "admitted")} for r in rows]
t1 = time.perf_counter()
ruc = B.run_ruc_experiment(a.seeds, ext_sizes=tuple(int(v) for v in a.ext.split(",")), base_seed=a.base_seed,
                           skip_failed_generations=True, hashes=tuple(a.hashes.split(",")))
t2 = time.perf_counter()
report = {"masking_sweep": {"formula": a.sweep_formula, "traces_per_side": a.sweep_traces, "lengths": [lo, hi],
                            "rows": sweeps, "wall_s": round(t1 - t0, 3)},
          "ruc": {"seeds": a.seeds, "summary": ruc["summary"], "runs": len(ruc["rows"]), "skipped": ruc["skipped"],
                  "wall_s": round(t2 - t1, 3)}}
text = json.dumps(report)
if a.out:
    with open(a.out, "w") as fh:
        fh.write(text + "\n")
print(text)
