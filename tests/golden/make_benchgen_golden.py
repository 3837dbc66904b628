#!/usr/bin/env python
"""Generate tests/golden/benchgen_golden.json by RUNNING THE REFERENCE's generators and experiments
(`/root/reference/pkg/src/ltllearn/benchgen.py`) with its own compiled core (oracle/_ref, see make_golden.py).
Every recorded value is produced by reference code.  Run in the build container:

    ./oracle/build_ref.sh && python tests/golden/make_benchgen_golden.py
"""
from __future__ import annotations

import json
import os
import sys
import warnings
from dataclasses import replace

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, os.path.join(ROOT, "oracle", "_ref"))

from ltllearn import benchgen, enumerator as E, formula as F, kernels as K  # noqa: E402
from ltllearn.cache import HashScheme  # noqa: E402
from ltllearn.traces import Alphabet  # noqa: E402

assert K.BACKEND == "compiled", "run oracle/build_ref.sh first"
warnings.simplefilter("ignore")


def spec_json(s):
    return {"pos": [list(t) for t in s.pos], "neg": [list(t) for t in s.neg]}


a2, a3 = Alphabet.default(2), Alphabet.default(3)
out = {"simple": [], "guided": [], "hamming": [], "samplebench": [], "masking": [], "ruc": None}

for n_props, k, lo, hi, seed in [(2, 4, 2, 5, 0), (2, 10, 0, 6, 7), (3, 25, 3, 9, 11), (1, 6, 1, 4, 3), (2, 40, 5, 12, 99)]:
    s = benchgen.gen_simple(Alphabet.default(n_props), k, lo, hi, seed)
    out["simple"].append(dict(n_props=n_props, k=k, lo=lo, hi=hi, seed=seed, **spec_json(s)))

for n_props, text, k, lo, hi, seed in [(2, "(p0 U p1) & F G p0", 8, 4, 16, 3), (3, "G (p0 | X p2) & F p1", 20, 5, 14, 5),
                                       (2, "F (p0 & X (p1 & X p0))", 12, 3, 10, 8), (2, "G p0", 6, 6, 9, 2),
                                       (2, "X X X p1 | (p0 U G p1)", 10, 63, 63, 13), (3, "!p0 & F (p1 & !p2)", 15, 1, 7, 21)]:
    al = Alphabet.default(n_props)
    s = benchgen.gen_guided(al, F.parse_formula(text, al), k, lo, hi, seed)
    out["guided"].append(dict(n_props=n_props, formula=text, k=k, lo=lo, hi=hi, seed=seed, **spec_json(s)))

for n_props, l, delta, seed in [(2, 5, 1, 0), (2, 6, 2, 4), (3, 4, 2, 9), (1, 7, 3, 1), (2, 3, 3, 6)]:
    s = benchgen.gen_hamming(Alphabet.default(n_props), l, delta, seed)
    out["hamming"].append(dict(n_props=n_props, l=l, delta=delta, seed=seed, **spec_json(s)))

for i, k, conservative, seed in [(3, 4, True, 1), (4, 6, False, 2), (8, 8, True, 1009), (5, 0, True, 17), (6, 10, True, 5)]:
    sb = benchgen.gen_samplebench(i, k, conservative, seed)
    out["samplebench"].append(dict(i=i, k=k, conservative=conservative, seed=seed, seed_formula=F.print_formula(sb.seed_formula, a2),
                                   seed_cost=sb.seed_cost, seed_spec=spec_json(sb.seed_spec), **spec_json(sb.spec)))

# masking sweeps: a precise-mode specification (masking is ignored: exact fingerprints) and two hashed ones
sweeps = [("simple2_k6", benchgen.gen_simple(a2, 6, 3, 8, 42), a2, {}, "mueller"),
          ("guided_len20", benchgen.gen_guided(a2, F.parse_formula("F (p0 & X p1) & G (p1 | X p0)", a2), 10, 14, 20, 4), a2, {}, "mueller"),
          ("guided_len20_fkp", benchgen.gen_guided(a2, F.parse_formula("F (p0 & X p1) & G (p1 | X p0)", a2), 10, 14, 20, 4), a2,
           {"require_nnf": True}, "fkp")]
for name, spec, al, kw, variant in sweeps:
    cfg = E.LearnerConfig(hash=HashScheme(variant), **kw)
    rows = benchgen.run_masking_sweep(spec, al, cfg)
    out["masking"].append(dict(name=name, n_props=al.size, cfg=kw, hash=variant, **spec_json(spec),
                               rows=[{k: r.get(k) for k in ("k", "status", "cost", "precise")} for r in rows]))

ruc = benchgen.run_ruc_experiment(2, ext_sizes=(0, 8, 16), base_seed=3)
out["ruc"] = dict(n_seeds=2, ext_sizes=[0, 8, 16], base_seed=3,
                  rows=[{k: r.get(k) for k in ("seed", "ext", "hash", "status", "cost", "precise", "minimal", "n_pos", "n_neg", "extra")}
                        for r in ruc["rows"]],
                  summary=ruc["summary"])

path = os.path.join(HERE, "benchgen_golden.json")
with open(path, "w") as fh:
    json.dump(out, fh, separators=(",", ":"))
print(path, os.path.getsize(path), "bytes;", {k: (len(v) if isinstance(v, list) else 1) for k, v in out.items()})
