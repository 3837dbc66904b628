"""CPU: the C-ABI library loads without a GPU and exports every symbol include/ltl_core.h declares; without
a device the product path fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

from paper_2402_12373_b200 import build as B
from paper_2402_12373_b200 import core as K
from paper_2402_12373_b200.errors import BackendUnavailable

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ltl_core.h")).read()
    return sorted(set(re.findall(r"LTL_API\s+[\w\s\*]+?\b(ltl_\w+)\s*\(", text)))


def test_library_builds_and_exports_every_declared_symbol():
    lib = ctypes.CDLL(B.build())
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert lib.ltl_abi_version() == 1


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import numpy as np

    with pytest.raises(BackendUnavailable):
        K.make_core(np.full(4, 2**64 - 1, dtype=np.uint64), 2, 0, K.V_MUELLER)
    from paper_2402_12373_b200.learner import learn

    with pytest.raises(BackendUnavailable):
        learn([(1, 0), (0, 1)], [(0, 0), (1, 1)], 2, max_cost=5)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2402_12373_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", text, re.M), f
                assert "liboracle" not in text, f


def test_level_planner_of_the_device_resident_levels_follows_the_learner():
    """`ltl_plan_level` is the planner `csrc/levels.cuh` runs on the device (same function, compiled for the host): its
    pieces must be the learner's segments (`learner.level_segments`, reference `enumerator.py:254-296`) with triangular
    segments cut as `_speedups.pyx:364-368` enumerates them -- for uniform and non-uniform costs, fragments, empty
    buckets and a bucket that exists before its level (negated atoms of the NNF fragment)."""
    import numpy as np

    from paper_2402_12373_b200 import learner as Ln
    from paper_2402_12373_b200.cache import LanguageCache
    from paper_2402_12373_b200.formula import COMMUTATIVE_OPS, UNARY_OPS, CostHomomorphism

    lib = ctypes.CDLL(B.build())
    i32p, i64p = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)
    lib.ltl_plan_level.argtypes = [i32p, ctypes.c_uint32, i64p, i64p, i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, i32p, i32p, i64p, i64p,
                                   ctypes.POINTER(ctypes.c_int), i64p]
    lib.ltl_plan_level.restype = ctypes.c_int
    rng = np.random.default_rng(7)
    for trial in range(200):
        costs = [1] * 8 if trial % 3 == 0 else [int(v) for v in rng.integers(1, 4, size=8)]
        cfg = Ln.LearnerConfig(cost=CostHomomorphism(costs), require_nnf=bool(trial % 5 == 1), forbid_until=bool(trial % 7 == 2))
        ops = Ln.enabled_ops(cfg)
        # a random bucket table: consecutive entry ranges by cost, some costs empty
        cache = LanguageCache.__new__(LanguageCache)
        cache._buckets = {}
        first = 0
        for c in range(1, int(rng.integers(2, 10))):
            size = int(rng.choice([0, 1, 2, 5, 40]))
            cache._buckets[c] = [first, first + size]
            first += size
        level = max(cache._buckets) + 1
        segs = Ln.level_segments(cache, cfg, ops, level)
        want = []
        for s in segs:
            if s.op in UNARY_OPS:
                want.append((s.op, 0, s.a0, s.a1, -1, -1, s.a1 - s.a0))
            elif not s.tri:
                want.append((s.op, 1, s.a0, s.a1, s.b0, s.b1, (s.a1 - s.a0) * (s.b1 - s.b0)))
            else:
                assert s.op in COMMUTATIVE_OPS and (s.a0, s.a1) == (s.b0, s.b1)
                k = s.a1 - s.a0
                if k >= 2:
                    want.append((s.op, 2, s.a0, s.a1 - 1, -1, s.b1, k * (k - 1) // 2))
        bc = np.array(sorted(cache._buckets), dtype=np.int64)
        bf = np.array([cache._buckets[int(c)][0] for c in bc], dtype=np.int64)
        be = np.array([cache._buckets[int(c)][1] for c in bc], dtype=np.int64)
        oc = np.array([cfg.cost.of(op) for op in range(8)], dtype=np.int32)
        cap = 96
        op_o, kind_o = np.zeros(cap, np.int32), np.zeros(cap, np.int32)
        rng_o, cnt_o = np.zeros(4 * cap, np.int64), np.zeros(cap, np.int64)
        n_p, total = ctypes.c_int(), ctypes.c_int64()
        rc = lib.ltl_plan_level(oc.ctypes.data_as(i32p), sum(1 << op for op in ops), bc.ctypes.data_as(i64p), bf.ctypes.data_as(i64p),
                                be.ctypes.data_as(i64p), len(bc), level, cap, op_o.ctypes.data_as(i32p), kind_o.ctypes.data_as(i32p),
                                rng_o.ctypes.data_as(i64p), cnt_o.ctypes.data_as(i64p), ctypes.byref(n_p), ctypes.byref(total))
        assert rc == 0
        got = [(int(op_o[k]), int(kind_o[k]), *(int(v) for v in rng_o[4 * k: 4 * k + 4]), int(cnt_o[k])) for k in range(n_p.value)]
        # (unary pieces carry j0 = j1 = -1, triangles j0 = -1)
        assert got == want, (trial, costs, cache._buckets)
        assert total.value == sum(w[-1] for w in want)
