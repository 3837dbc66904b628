#!/usr/bin/env python
"""Generate tests/golden/dnc_golden.json by RUNNING THE REFERENCE's divide-and-conquer learner
(`/root/reference/pkg/src/ltllearn/dnc.py`) with its own compiled core (oracle/_ref, see make_golden.py).
Every recorded value is produced by reference code.  Run in the build container:

    ./oracle/build_ref.sh && python tests/golden/make_dnc_golden.py
"""
from __future__ import annotations

import json
import os
import sys
import warnings

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, os.path.join(ROOT, "oracle", "_ref"))

from ltllearn import benchgen, dnc, enumerator as E, formula as F, kernels as K  # noqa: E402
from ltllearn.traces import Alphabet  # noqa: E402

assert K.BACKEND == "compiled", "run oracle/build_ref.sh first"
warnings.simplefilter("ignore")


def run(name, spec, alphabet, cfg_kw, split_kw):
    cfg = E.LearnerConfig(**cfg_kw)
    checked = []

    def check(f, pos, neg):
        checked.append(1)
        return True

    try:
        res = dnc.dnc_learn(spec, alphabet, cfg, dnc.SplitConfig(**split_kw), debug_check=check)
    except dnc.WindowExhausted as exc:
        return {"name": name, "n_props": alphabet.size, "pos": [list(t) for t in spec.pos], "neg": [list(t) for t in spec.neg],
                "cfg": cfg_kw, "split": split_kw, "raises": "WindowExhausted", "message": str(exc)}
    return {
        "name": name, "n_props": alphabet.size, "pos": [list(t) for t in spec.pos], "neg": [list(t) for t in spec.neg],
        "cfg": cfg_kw, "split": split_kw, "formula": F.print_formula(res.formula, alphabet),
        "cost": F.cost(res.formula, cfg.cost), "nodes": res.nodes, "enum_calls": res.enum_calls,
        "enum_offered": [s["offered"] for s in res.enum_stats], "recombinations": len(checked),
    }


cases = []
OOM_BUDGETS = (20000, 400000)
a2, a3 = Alphabet.default(2), Alphabet.default(3)
f_plant = F.parse_formula("(p0 U p1) & F G p0", a2)
g_plant = F.parse_formula("G (p0 | X p2) & F p1", a3)

s = benchgen.gen_guided(a2, f_plant, 40, 4, 12, seed=11)
cases.append(run("guided40_rand_w16", s, a2, {}, {"strategy": "rand", "window": 16, "seed": 3}))
cases.append(run("guided40_det_w16", s, a2, {}, {"strategy": "det", "window": 16}))
cases.append(run("guided40_rand_w64", s, a2, {}, {"strategy": "rand", "window": 64, "seed": 1}))
s = benchgen.gen_guided(a3, g_plant, 100, 5, 14, seed=5)
cases.append(run("guided100_rand_w32", s, a3, {}, {"strategy": "rand", "window": 32, "seed": 7}))
cases.append(run("guided100_det_w64", s, a3, {}, {"strategy": "det", "window": 64}))
s = benchgen.gen_simple(a2, 60, 3, 9, seed=21)
cases.append(run("simple60_rand_w8", s, a2, {"ceiling": 9}, {"strategy": "rand", "window": 8, "seed": 2}))
cases.append(run("simple60_det_w8", s, a2, {"ceiling": 9}, {"strategy": "det", "window": 8}))
# window halving: a budget so small that the first leaves run out of memory
s = benchgen.gen_guided(a2, f_plant, 16, 4, 12, seed=23)
for budget in OOM_BUDGETS:
    cases.append(run(f"guided16_oom_rand_{budget}", s, a2, {"budget_bytes": budget}, {"strategy": "rand", "window": 32, "min_window": 4, "seed": 9}))
    cases.append(run(f"guided16_oom_det_{budget}", s, a2, {"budget_bytes": budget}, {"strategy": "det", "window": 32, "min_window": 4}))
cases.append(run("guided16_exhausted", s, a2, {"budget_bytes": 600}, {"strategy": "det", "window": 16, "min_window": 8}))
# noise, NNF, weighted costs flow through the leaves
s = benchgen.gen_guided(a2, f_plant, 30, 4, 10, seed=17)
cases.append(run("guided30_nnf_rand", s, a2, {"require_nnf": True}, {"strategy": "rand", "window": 16, "seed": 5}))
cases.append(run("guided30_nountil_det", s, a2, {"forbid_until": True}, {"strategy": "det", "window": 16}))

out = {"generator": "tests/golden/make_dnc_golden.py", "cases": cases}
with open(os.path.join(HERE, "dnc_golden.json"), "w") as fh:
    json.dump(out, fh, separators=(",", ":"))
for c in cases:
    kinds = [n["kind"] for n in c.get("nodes", [])]
    print(c["name"], (c.get("formula") or c.get("raises"))[:60], c.get("cost"), c.get("enum_calls"), len(kinds), "oom-nodes", kinds.count("enum-oom"))
