"""The reference's OWN learner driving the CUDA core through the drop-in boundary.

`ltllearn.enumerator.enum_learn` (reference `enumerator.py:159-251`) -- its validation, packing (`bitsem.py:73-88`),
scheme resolution (`cache.py:64-91`), level loop and chunked dispatch (`enumerator.py:271-296`), language cache
(`cache.py:101-213`) and D&C (`dnc.py`) -- runs unmodified; only `kernels.make_core` (`kernels.py:140-172`) is replaced
by the binding of INTEGRATION.md section 2, written here in full over the C ABI of `include/ltl_core.h` (ctypes on
`libltlcore.so`, nothing of this repository's Python host side in between).  Outcomes must equal the fixtures recorded
from the reference running its own compiled core (`tests/golden/reference_golden.json`, `dnc_golden.json`): formula
text, cost, counters, per-level rows, and the SHA-256 of every stored matrix and record.

The reference travels to the GPU box as binaries only: `oracle/build_ref.sh` compiles its modules where they lie
(Cython -> gcc) into the git-ignored `oracle/_ref/ltllearn/`.
"""
import ctypes as C
import hashlib
import json
import os
import sys
import warnings

import numpy as np
import pytest

from helpers import ROOT, golden, sha

REF_DIR = os.path.join(ROOT, "oracle", "_ref")
LIB = os.path.join(ROOT, "paper_2402_12373_b200", "csrc", "libltlcore.so")


@pytest.fixture(scope="module", params=[pytest.param("cuda", marks=pytest.mark.gpu), "compiled"])
def ref(request):
    """The reference package (compiled copies under oracle/_ref) with `kernels.make_core` bound to the CUDA library
    ("cuda"); "compiled" keeps the reference's own core behind the same harness -- the CPU check that the harness
    itself reproduces the fixtures, so that the CUDA runs differ from it by the core alone."""
    if not os.path.exists(os.path.join(REF_DIR, "ltllearn")) or not any(
            f.startswith("enumerator.") for f in os.listdir(os.path.join(REF_DIR, "ltllearn"))):
        pytest.fail("oracle/_ref/ltllearn is not built: run oracle/build_ref.sh where /root/reference exists")
    sys.path.insert(0, REF_DIR)
    try:
        from ltllearn import cache as rcache, dnc as rdnc, enumerator as E, formula as F, kernels as K
        from ltllearn._kernels_py import CoreOOM
        from ltllearn.traces import Alphabet, Specification
    finally:
        sys.path.remove(REF_DIR)

    made = []
    original = K.make_core
    ns = dict(E=E, F=F, K=K, rcache=rcache, rdnc=rdnc, Alphabet=Alphabet, Specification=Specification, made=made)
    if request.param == "compiled":
        assert K.BACKEND == "compiled"

        def capture(*a, **kw):
            core = original(*a, **kw)
            made.append((core, a))
            return core

        K.make_core = capture
        yield type("Ref", (), ns)
        K.make_core = original
        return

    lib = C.CDLL(LIB)
    u64p, i32p, vp = C.POINTER(C.c_uint64), C.POINTER(C.c_int32), C.c_void_p
    lib.ltl_core_last_error.restype = C.c_char_p
    lib.ltl_core_last_error.argtypes = [vp]
    lib.ltl_core_destroy.argtypes = [vp]
    lib.ltl_core_destroy.restype = None

    def ptr(a):
        return a.ctypes.data_as(u64p)

    class CudaCore:  # INTEGRATION.md section 2, every member (same members as reference `_speedups.Core`)
        def __init__(self, masks, n_pos, err_max, variant, proj_rows, proj_offs, fkp_bits, mask_k, budget_bytes):
            m = np.ascontiguousarray(masks, np.uint64)
            pr, po = (np.ascontiguousarray(list(v), np.int32) for v in (proj_rows, proj_offs))
            self._h, self.R = vp(), len(m)
            rc = lib.ltl_core_create(ptr(m), C.c_int(len(m)), 1, int(n_pos), int(err_max), int(variant),
                                     pr.ctypes.data_as(i32p), po.ctypes.data_as(i32p), len(pr), int(fkp_bits), int(mask_k),
                                     C.c_uint64(budget_bytes), 0, C.byref(self._h))
            if rc:
                raise ValueError(lib.ltl_core_last_error(None).decode())  # reference `_speedups.pyx:83-84, 92-93`

        def __del__(self):
            if getattr(self, "_h", None):
                lib.ltl_core_destroy(self._h)
                self._h = None

        def _ok(self, rc):
            if rc == -3:
                raise CoreOOM("memory budget exhausted")  # reference `_speedups.pyx:275-276`
            if rc == -1:
                raise ValueError(lib.ltl_core_last_error(self._h).decode())
            if rc:
                raise RuntimeError(lib.ltl_core_last_error(self._h).decode())

        def _cm(self, cm):
            a = np.ascontiguousarray(cm, np.uint64).reshape(-1)
            if len(a) != self.R:
                raise ValueError("wrong matrix size")
            return a

        def _counter(self, k):
            out = np.zeros(5, np.uint64)
            self._ok(lib.ltl_core_counters(self._h, ptr(out)))
            return int(out[k])

        n_entries = property(lambda s: s._counter(0))    # reference `_speedups.pyx:113-115`
        bytes_used = property(lambda s: s._counter(1))
        offered = property(lambda s: s._counter(2))      # reference `_speedups.pyx:68`
        admitted = property(lambda s: s._counter(3))
        duplicates = property(lambda s: s._counter(4))

        def add_entry(self, cm, op, lhs, rhs):           # reference `_speedups.pyx:264-277`
            idx = C.c_int64()
            self._ok(lib.ltl_core_add_entry(self._h, ptr(self._cm(cm)), int(op), int(lhs), int(rhs), C.byref(idx)))
            return idx.value

        def contains(self, cm):                          # reference `_speedups.pyx:279-287`
            found = C.c_int()
            self._ok(lib.ltl_core_contains(self._h, ptr(self._cm(cm)), C.byref(found)))
            return bool(found.value)

        def fingerprint_of(self, cm):                    # reference `_speedups.pyx:233-241`
            hi, lo = C.c_uint64(), C.c_uint64()
            self._ok(lib.ltl_core_fingerprint_of(self._h, ptr(self._cm(cm)), C.byref(hi), C.byref(lo)))
            return (hi.value << 64) | lo.value

        def get_cm(self, idx):                           # reference `_speedups.pyx:117-122`
            out = np.empty(self.R, np.uint64)
            rc = lib.ltl_core_get_cm(self._h, C.c_int64(idx), ptr(out))
            if rc == -1:
                raise IndexError(idx)
            self._ok(rc)
            return out

        def get_record(self, idx):                       # reference `_speedups.pyx:124-129`
            op, lhs, rhs = C.c_int(), C.c_int(), C.c_int()
            rc = lib.ltl_core_get_record(self._h, C.c_int64(idx), C.byref(op), C.byref(lhs), C.byref(rhs))
            if rc == -1:
                raise IndexError(idx)
            self._ok(rc)
            return op.value, lhs.value, rhs.value

        def export_cms(self):                            # reference `_speedups.pyx:131-137`
            n = self.n_entries
            out = np.empty((n, self.R), np.uint64)
            if n:
                self._ok(lib.ltl_core_export_cms(self._h, C.c_int64(0), C.c_int64(n), ptr(out)))
            return out

        def screen_unary(self, op, c0, c1):              # reference `_speedups.pyx:337-355`
            st, li, ri = C.c_int(), C.c_int64(), C.c_int64()
            self._ok(lib.ltl_core_screen_unary(self._h, int(op), C.c_int64(c0), C.c_int64(c1), C.byref(st), C.byref(li),
                                               C.byref(ri)))
            return st.value, li.value, ri.value

        def screen_binary(self, op, a0, a1, b0, b1, tri):  # reference `_speedups.pyx:357-380`
            st, li, ri = C.c_int(), C.c_int64(), C.c_int64()
            self._ok(lib.ltl_core_screen_binary(self._h, int(op), C.c_int64(a0), C.c_int64(a1), C.c_int64(b0), C.c_int64(b1),
                                                int(bool(tri)), C.byref(st), C.byref(li), C.byref(ri)))
            return st.value, li.value, ri.value

    def make_core(masks, n_pos, err_max, variant, proj_rows=(), proj_offs=(), fkp_bits=0, mask_k=0,
                  budget_bytes=2 << 30, backend=None):  # the `chosen == "cuda"` arm of reference `kernels.py:160-172`
        core = CudaCore(masks, n_pos, err_max, variant, proj_rows, proj_offs, fkp_bits, mask_k, budget_bytes)
        made.append((core, (masks, n_pos, err_max, variant, proj_rows, proj_offs, fkp_bits, mask_k, budget_bytes)))
        return core

    K.make_core = make_core
    yield type("Ref", (), ns)
    K.make_core = original


LEARN_CASES = golden()["learn"]


@pytest.mark.parametrize("case", LEARN_CASES, ids=[c["name"] for c in LEARN_CASES])
def test_reference_enum_learn_on_the_cuda_core(ref, case):
    kw = dict(case["cfg"])
    if "hash" in kw:
        kw["hash"] = ref.rcache.HashScheme(**kw["hash"])
    if "cost" in kw:
        kw["cost"] = ref.F.CostHomomorphism(tuple(kw["cost"]))
    alphabet = ref.Alphabet.default(case["n_props"])
    spec = ref.Specification(tuple(tuple(t) for t in case["pos"]), tuple(tuple(t) for t in case["neg"]))
    ref.made.clear()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = ref.E.enum_learn(spec, alphabet, ref.E.LearnerConfig(**kw))
    assert type(res).__name__ == case["outcome"]
    assert {k: v for k, v in res.stats.as_dict().items() if k != "levels"} == case["stats"]
    assert [{k: v for k, v in lv.items() if k != "ms"} for lv in res.stats.levels] == case["levels"]
    if case["outcome"] == "Solved":
        assert ref.F.print_formula(res.formula) == case["formula"] and res.cost == case["cost"]
    elif case["outcome"] == "CeilingReached":
        text = ref.F.print_formula(res.formula)
        assert hashlib.sha256(text.encode()).hexdigest() == case["formula_sha"] and res.ceiling == case["ceiling"]
    if "core" in case:
        core, args = ref.made[-1]
        want = case["core"]
        assert (int(args[3]), [int(v) for v in args[4]], [int(v) for v in args[5]], int(args[6]), int(args[7])) == (
            want["variant"], want["proj_rows"], want["proj_offs"], want["fkp_bits"], want["mask_k"])
        assert core.n_entries == want["n_entries"]
        recs = np.array([core.get_record(i) for i in range(core.n_entries)], dtype=np.int64).reshape(-1, 3)
        assert sha(recs) == want["records_sha"]
        assert sha(core.export_cms()) == want["cms_sha"]
    else:
        assert not ref.made  # atom fast paths never build a core


def _dnc_cases():
    with open(os.path.join(ROOT, "tests", "golden", "dnc_golden.json")) as fh:
        return json.load(fh)["cases"]


@pytest.mark.parametrize("case", _dnc_cases(), ids=[c["name"] for c in _dnc_cases()])
def test_reference_dnc_on_the_cuda_core(ref, case):
    """The reference's divide-and-conquer learner (`dnc.py:55-224`) over the same binding: formula text, cost, node log
    and per-leaf candidate counts of the runs recorded with the reference's own core."""
    alphabet = ref.Alphabet.default(case["n_props"])
    spec = ref.Specification(tuple(tuple(t) for t in case["pos"]), tuple(tuple(t) for t in case["neg"]))
    cfg = ref.E.LearnerConfig(**case["cfg"])
    checked = []

    def check(f, pos, neg):
        checked.append(1)
        return True

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        if case.get("raises") == "WindowExhausted":
            with pytest.raises(ref.rdnc.WindowExhausted) as exc:
                ref.rdnc.dnc_learn(spec, alphabet, cfg, ref.rdnc.SplitConfig(**case["split"]), debug_check=check)
            assert str(exc.value) == case["message"]
            return
        res = ref.rdnc.dnc_learn(spec, alphabet, cfg, ref.rdnc.SplitConfig(**case["split"]), debug_check=check)
    assert ref.F.print_formula(res.formula, alphabet) == case["formula"]
    assert ref.F.cost(res.formula, cfg.cost) == case["cost"]
    assert res.nodes == case["nodes"] and res.enum_calls == case["enum_calls"]
    assert [s["offered"] for s in res.enum_stats] == case["enum_offered"] and len(checked) == case["recombinations"]
