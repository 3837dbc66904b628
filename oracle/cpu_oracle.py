"""ctypes face of oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY (parity status: pinned, see
ltl_oracle.c header).

``OracleCore`` has the screening-core contract of the reference
(`/root/reference/pkg/src/ltllearn/_kernels_py.py:32-281`, "the contract" per `kernels.py:152`),
generalised to R rows x W words: characteristic matrices are ``uint64[R*W]`` (row-major,
``cm[r*W + w]``); for ``W == 1`` that is exactly the reference's ``uint64[R]``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

S_DONE, S_SOLVED, S_OOM = 0, 1, 2
V_GATHER, V_MUELLER, V_FKP, V_NH, V_NH32 = 0, 1, 2, 3, 4


class CoreOOM(Exception):
    """Budget exhausted in add_entry (reference: _kernels_py.py:28-29)."""


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "ltl_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-C", _HERE, "liboracle.so"], stdout=subprocess.DEVNULL)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        u64p = C.POINTER(C.c_uint64)
        i32p = C.POINTER(C.c_int)
        lp = C.POINTER(C.c_long)
        L.oracle_create.restype = C.c_void_p
        L.oracle_create.argtypes = [u64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, i32p, i32p, C.c_int,
                                    C.c_int, C.c_int, C.c_uint64]
        L.oracle_destroy.argtypes = [C.c_void_p]
        L.oracle_set_threads.argtypes = [C.c_void_p, C.c_int]
        L.oracle_add_entry.restype = C.c_long
        L.oracle_add_entry.argtypes = [C.c_void_p, u64p, C.c_int, C.c_int, C.c_int]
        L.oracle_contains.argtypes = [C.c_void_p, u64p]
        L.oracle_fingerprint_of.argtypes = [C.c_void_p, u64p, u64p, u64p]
        L.oracle_apply_unary.argtypes = [C.c_void_p, C.c_int, u64p, u64p]
        L.oracle_apply_binary.argtypes = [C.c_void_p, C.c_int, u64p, u64p, u64p]
        L.oracle_errors.argtypes = [C.c_void_p, u64p]
        L.oracle_get_cm.argtypes = [C.c_void_p, C.c_long, u64p]
        L.oracle_get_record.argtypes = [C.c_void_p, C.c_long, i32p, i32p, i32p]
        L.oracle_export_cms.argtypes = [C.c_void_p, C.c_long, C.c_long, u64p]
        L.oracle_export_records.argtypes = [C.c_void_p, C.c_long, C.c_long, C.POINTER(C.c_int8),
                                            C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.oracle_counters.argtypes = [C.c_void_p, u64p]
        L.oracle_screen_unary.argtypes = [C.c_void_p, C.c_int, C.c_long, C.c_long, lp, lp]
        L.oracle_screen_binary.argtypes = [C.c_void_p, C.c_int, C.c_long, C.c_long, C.c_long, C.c_long, C.c_int, lp, lp]
        L.oracle_max_threads.restype = C.c_int
        L.oracle_set_store_results.argtypes = [C.c_void_p, C.c_int]
        L.oracle_unstored_from.argtypes = [C.c_void_p]
        L.oracle_unstored_from.restype = C.c_long
        _lib = L
    return _lib


def _u64(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


class OracleCore:
    """Generalised CPU screening core; same members as the reference cores."""

    def __init__(self, masks, n_pos, err_max, variant, proj_rows=(), proj_offs=(), fkp_bits=0, mask_k=0,
                 budget_bytes=2 << 30, *, words_per_row=1, threads=1, device=None):
        m = np.ascontiguousarray(masks, dtype=np.uint64).reshape(-1)
        W = int(words_per_row)
        if len(m) % W:
            raise ValueError("masks length must be a multiple of words_per_row")
        self.R, self.W, self.n = len(m) // W, W, len(m)
        pr = np.ascontiguousarray(list(proj_rows), dtype=np.int32)
        po = np.ascontiguousarray(list(proj_offs), dtype=np.int32)
        if len(pr) > 126:
            raise ValueError("projection wider than the fingerprint")
        ip = C.POINTER(C.c_int)
        self._h = lib().oracle_create(_u64(m), self.R, W, int(n_pos), int(err_max), int(variant),
                                      pr.ctypes.data_as(ip), po.ctypes.data_as(ip), len(pr), int(fkp_bits),
                                      int(mask_k), int(budget_bytes))
        if not self._h:
            raise ValueError("oracle_create rejected the arguments")
        if threads != 1:
            lib().oracle_set_threads(self._h, int(threads))

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:
            _lib.oracle_destroy(h)

    close = __del__

    def _cm(self, cm):
        a = np.ascontiguousarray(cm, dtype=np.uint64).reshape(-1)
        if len(a) != self.n:
            raise ValueError(f"expected {self.n} words, got {len(a)}")
        return a

    # -- counters ----------------------------------------------------------
    def _counters(self):
        out = np.zeros(5, dtype=np.uint64)
        lib().oracle_counters(self._h, _u64(out))
        return [int(v) for v in out]

    n_entries = property(lambda s: s._counters()[0])
    bytes_used = property(lambda s: s._counters()[1])
    offered = property(lambda s: s._counters()[2])
    admitted = property(lambda s: s._counters()[3])
    duplicates = property(lambda s: s._counters()[4])

    # -- contract ----------------------------------------------------------
    def add_entry(self, cm, op, lhs, rhs):
        res = lib().oracle_add_entry(self._h, _u64(self._cm(cm)), int(op), int(lhs), int(rhs))
        if res == -3:
            raise CoreOOM
        if res == -4:
            raise MemoryError("oracle host allocation failed")
        return int(res)

    def contains(self, cm):
        return bool(lib().oracle_contains(self._h, _u64(self._cm(cm))))

    def fingerprint_of(self, cm):
        hi, lo = C.c_uint64(), C.c_uint64()
        lib().oracle_fingerprint_of(self._h, _u64(self._cm(cm)), C.byref(hi), C.byref(lo))
        return int(hi.value) << 64 | int(lo.value)

    def get_cm(self, idx):
        self._check_stored(int(idx), 1)
        out = np.empty(self.n, dtype=np.uint64)
        lib().oracle_get_cm(self._h, int(idx), _u64(out))
        return out

    def get_record(self, idx):
        op, l, r = C.c_int(), C.c_int(), C.c_int()
        lib().oracle_get_record(self._h, int(idx), C.byref(op), C.byref(l), C.byref(r))
        return op.value, l.value, r.value

    def export_cms(self, first=0, count=None):
        n = self.n_entries
        count = n - first if count is None else count
        out = np.empty((count, self.n), dtype=np.uint64)
        self._check_stored(int(first), int(count))
        if count:
            lib().oracle_export_cms(self._h, int(first), int(count), _u64(out))
        return out

    def export_records(self, first=0, count=None):
        n = self.n_entries
        count = n - first if count is None else count
        op = np.empty(count, dtype=np.int8)
        lhs = np.empty(count, dtype=np.int32)
        rhs = np.empty(count, dtype=np.int32)
        if count:
            lib().oracle_export_records(self._h, int(first), int(count), op.ctypes.data_as(C.POINTER(C.c_int8)),
                                        lhs.ctypes.data_as(C.POINTER(C.c_int32)),
                                        rhs.ctypes.data_as(C.POINTER(C.c_int32)))
        return op, lhs, rhs

    def screen_unary(self, op, c0, c1):
        self._check_stored(0, int(c1))
        li, ri = C.c_long(), C.c_long()
        st = lib().oracle_screen_unary(self._h, int(op), int(c0), int(c1), C.byref(li), C.byref(ri))
        return st, li.value, ri.value

    def screen_binary(self, op, a0, a1, b0, b1, tri):
        self._check_stored(0, max(int(a1), int(b1)))
        li, ri = C.c_long(), C.c_long()
        st = lib().oracle_screen_binary(self._h, int(op), int(a0), int(a1), int(b0), int(b1), int(bool(tri)),
                                        C.byref(li), C.byref(ri))
        return st, li.value, ri.value

    def set_option(self, name, value):
        """Only ``store_results`` (same meaning as the device core's option): 0 = entries admitted from now on
        keep record and fingerprint but no matrix."""
        if name != "store_results":
            raise ValueError(f"unknown option {name}")
        if lib().oracle_set_store_results(self._h, int(value)):
            raise ValueError("matrices were already skipped: storing cannot resume")

    def _check_stored(self, first, count):
        u = lib().oracle_unstored_from(self._h)
        if u >= 0 and first + count > u:
            raise ValueError("matrices of these entries were not stored")

    # -- pure operator access (op-level parity tests) ------------------------
    def apply_unary(self, op, x):
        out = np.empty(self.n, dtype=np.uint64)
        lib().oracle_apply_unary(self._h, int(op), _u64(self._cm(x)), _u64(out))
        return out

    def apply_binary(self, op, x, y):
        out = np.empty(self.n, dtype=np.uint64)
        lib().oracle_apply_binary(self._h, int(op), _u64(self._cm(x)), _u64(self._cm(y)), _u64(out))
        return out

    def errors(self, cm):
        return int(lib().oracle_errors(self._h, _u64(self._cm(cm))))
