"""ctypes face of `csrc/libltlcore.so` -- the B200 screening core behind the reference's core contract.

`CudaCore` has the members of the reference's interchangeable cores (`_speedups.Core`,
`/root/reference/pkg/src/ltllearn/_speedups.pyx:61-380`; contract `_kernels_py.py:32-281`):
``add_entry, contains, fingerprint_of, get_cm, get_record, export_cms, screen_unary, screen_binary`` and the
counters ``n_entries, bytes_used, offered, admitted, duplicates`` -- same argument meaning, same status
codes, same exceptions (`ValueError` for misuse, `CoreOOM` from ``add_entry``) -- plus ``run_level``
(one call per cost level instead of one per chunk, reference `enumerator.py:271-296`).
`make_core` mirrors `kernels.make_core` (`kernels.py:140-172`).

There is no CPU fallback: if the shared library is missing or no CUDA device is visible, `make_core`
raises `BackendUnavailable`.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

import numpy as np

from .errors import BackendUnavailable, CoreError, CoreOOM

S_DONE, S_SOLVED, S_OOM = 0, 1, 2
V_GATHER, V_MUELLER, V_FKP, V_NH, V_NH32 = 0, 1, 2, 3, 4
MAX_WORDS_PER_ROW = 16

ERR_ARG, ERR_CUDA, ERR_BUDGET, ERR_DEVICE_OOM, ERR_INVARIANT = -1, -2, -3, -4, -5
KERNEL_CLASSES = ("screen", "finalize", "resolve", "scan", "emit", "materialize", "rehash", "purge", "misc", "levels")

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LTL_CORE_LIB") or os.path.join(_HERE, "csrc", "libltlcore.so")  # override: A/B builds


class Segment(C.Structure):
    _fields_ = [("op", C.c_int32), ("tri", C.c_int32), ("a0", C.c_int64), ("a1", C.c_int64), ("b0", C.c_int64),
                ("b1", C.c_int64)]


class LevelStats(C.Structure):
    _fields_ = [("cost", C.c_int32), ("status", C.c_int32), ("offered", C.c_uint64), ("admitted", C.c_uint64),
                ("duplicates", C.c_uint64), ("bytes", C.c_uint64), ("first_entry", C.c_int64), ("end_entry", C.c_int64),
                ("ms", C.c_double)]


#: row-shard exchange callback (include/ltl_core.h: ltl_exchange_fn)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64)

_lib = None


def load_library():
    """Load libltlcore.so (never builds it: `python -m paper_2402_12373_b200.build` does)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise BackendUnavailable(f"{LIB_PATH} is missing: run `python -m paper_2402_12373_b200.build` "
                                 "(there is no CPU fallback)")
    try:
        L = C.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover
        raise BackendUnavailable(f"cannot load {LIB_PATH}: {exc}") from None
    u64p, i32p, i64p, ip = C.POINTER(C.c_uint64), C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int)
    vp = C.c_void_p
    L.ltl_abi_version.restype = C.c_int
    L.ltl_device_count.restype = C.c_int
    L.ltl_core_create.argtypes = [u64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, i32p, i32p, C.c_int, C.c_int,
                                  C.c_int, C.c_uint64, C.c_int, C.POINTER(vp)]
    L.ltl_core_destroy.argtypes = [vp]
    L.ltl_core_destroy.restype = None
    L.ltl_core_last_error.argtypes = [vp]
    L.ltl_core_last_error.restype = C.c_char_p
    L.ltl_core_add_entry.argtypes = [vp, u64p, C.c_int, C.c_int, C.c_int, i64p]
    L.ltl_core_screen_unary.argtypes = [vp, C.c_int, C.c_int64, C.c_int64, ip, i64p, i64p]
    L.ltl_core_screen_binary.argtypes = [vp, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int, ip, i64p,
                                         i64p]
    L.ltl_core_run_level.argtypes = [vp, C.POINTER(Segment), C.c_int, ip, ip, i64p, i64p]
    L.ltl_core_run_search.argtypes = [vp, i32p, C.c_uint32, i64p, i64p, i64p, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(LevelStats), C.c_int, ip, ip, ip, i64p, i64p, ip]
    L.ltl_core_run_search.restype = C.c_int
    L.ltl_core_contains.argtypes = [vp, u64p, ip]
    L.ltl_core_fingerprint_of.argtypes = [vp, u64p, u64p, u64p]
    L.ltl_core_get_cm.argtypes = [vp, C.c_int64, u64p]
    L.ltl_core_get_record.argtypes = [vp, C.c_int64, ip, ip, ip]
    L.ltl_core_get_subtree.argtypes = [vp, C.c_int64, C.c_int, i32p, ip]
    L.ltl_core_get_subtree.restype = C.c_int
    L.ltl_core_export_cms.argtypes = [vp, C.c_int64, C.c_int64, u64p]
    L.ltl_core_export_records.argtypes = [vp, C.c_int64, C.c_int64, C.POINTER(C.c_int8), i32p, i32p]
    L.ltl_core_entry_fingerprints.argtypes = [vp, C.c_int64, C.c_int64, u64p, u64p]
    L.ltl_core_counters.argtypes = [vp, u64p]
    L.ltl_core_set_option.argtypes = [vp, C.c_char_p, C.c_int64]
    L.ltl_core_set_row_shard.argtypes = [vp, C.c_int64, C.c_int64, EXCHANGE_FN, vp]
    L.ltl_core_set_table_shard.argtypes = [vp, C.c_int, C.c_int]
    L.ltl_core_set_table_shard.restype = C.c_int
    L.ltl_core_kernel_stats.argtypes = [vp, C.c_int, u64p, C.POINTER(C.c_double), C.POINTER(C.c_double), u64p]
    L.ltl_core_reset_kernel_stats.argtypes = [vp]
    L.ltl_core_info.argtypes = [vp, u64p]
    L.ltl_core_stream.argtypes = [vp, C.POINTER(vp)]
    L.ltl_core_transfer_stats.argtypes = [vp, u64p]
    L.ltl_core_host_times.argtypes = [vp, C.POINTER(C.c_double)]
    L.ltl_core_host_times.restype = C.c_int
    L.ltl_pool_trim.restype = C.c_uint64
    L.ltl_pack_traces.argtypes = [C.POINTER(C.c_uint16), i64p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, u64p, u64p]
    L.ltl_pack_traces.restype = C.c_int
    u16p = C.POINTER(C.c_uint16)
    L.ltl_traces_create.argtypes = [u16p, i64p, C.c_int64, u16p, i64p, C.c_int64, C.c_int, C.c_int, C.POINTER(vp)]
    L.ltl_traces_destroy.argtypes = [vp]
    L.ltl_traces_destroy.restype = None
    L.ltl_traces_last_error.argtypes = [vp]
    L.ltl_traces_last_error.restype = C.c_char_p
    L.ltl_traces_pack.argtypes = [vp, C.c_int]
    L.ltl_traces_info.argtypes = [vp, u64p]
    L.ltl_traces_suspects.argtypes = [vp, i64p, C.c_int64]
    L.ltl_traces_export.argtypes = [vp, u64p, u64p]
    L.ltl_core_create_on_traces.argtypes = [vp, C.c_int, C.c_int, i32p, i32p, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                            C.POINTER(vp)]
    L.ltl_core_add_atom.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, i64p]
    for name in ("ltl_traces_create", "ltl_traces_pack", "ltl_traces_info", "ltl_traces_suspects", "ltl_traces_export",
                 "ltl_core_create_on_traces", "ltl_core_add_atom"):
        getattr(L, name).restype = C.c_int
    L.ltl_trace_file_scan.argtypes = [C.c_char_p, C.c_uint64, i64p, ip, ip, ip, i64p]
    L.ltl_trace_file_fill.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_int, u16p, i64p, u16p, i64p]
    L.ltl_trace_file_scan.restype = L.ltl_trace_file_fill.restype = C.c_int
    L.ltl_core_level_size.argtypes = [vp, C.POINTER(Segment), C.c_int, i64p]
    L.ltl_core_stage_eval.argtypes = [vp, C.POINTER(Segment), C.c_int, C.c_int64, C.c_int64, vp, i64p]
    L.ltl_core_stage_file.argtypes = [vp, vp, C.c_int64, vp, i64p]
    L.ltl_core_stage_route.argtypes = [vp, vp, C.c_int64, C.c_uint64, C.c_int, vp, i64p]
    L.ltl_core_stage_winners.argtypes = [vp, vp, vp, C.c_int64, C.c_uint64, C.c_int64, vp, i64p]
    L.ltl_core_stage_route.restype = L.ltl_core_stage_winners.restype = C.c_int
    L.ltl_core_stage_decode.argtypes = [vp, C.POINTER(Segment), C.c_int, vp, C.c_int64, vp, vp, vp]
    L.ltl_core_stage_append.argtypes = [vp, vp, vp, vp, C.c_int64, C.c_uint64, C.c_uint64]
    L.ltl_core_stage_purge.argtypes = [vp, C.c_uint64]
    for name in ("ltl_core_level_size", "ltl_core_stage_eval", "ltl_core_stage_file", "ltl_core_stage_decode",
                 "ltl_core_stage_append", "ltl_core_stage_purge"):
        getattr(L, name).restype = C.c_int
    for name in ("ltl_core_create", "ltl_core_add_entry", "ltl_core_screen_unary", "ltl_core_screen_binary",
                 "ltl_core_run_level", "ltl_core_contains", "ltl_core_fingerprint_of", "ltl_core_get_cm",
                 "ltl_core_get_record", "ltl_core_export_cms", "ltl_core_export_records",
                 "ltl_core_entry_fingerprints", "ltl_core_counters", "ltl_core_set_option", "ltl_core_set_row_shard", "ltl_core_kernel_stats",
                 "ltl_core_reset_kernel_stats", "ltl_core_info", "ltl_core_stream", "ltl_core_transfer_stats"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def pool_trim() -> int:
    """Return pooled device memory of released cores to the driver; bytes freed."""
    return int(load_library().ltl_pool_trim())


def device_count() -> int:
    n = load_library().ltl_device_count()
    return max(n, 0)


def _u64(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def pack_traces(chars: np.ndarray, lengths: np.ndarray, n_props: int, words_per_row: int, device: int = 0):
    """Pack a padded character matrix ``uint16[R, L]`` into length masks ``uint64[R, W]`` and per-proposition
    characteristic sequences ``uint64[n_props, R, W]`` on the device (`k_pack`; replaces the reference's
    `TraceContext.from_traces` triple loop, `bitsem.py:73-88`)."""
    L = load_library()
    if device_count() <= 0:
        raise BackendUnavailable("no CUDA device visible (there is no CPU fallback)")
    chars = np.ascontiguousarray(chars, dtype=np.uint16)
    lengths = np.ascontiguousarray(lengths, dtype=np.int64)
    R, width = chars.shape if chars.ndim == 2 else (len(lengths), 0)
    W = int(words_per_row)
    if width > 64 * W:
        chars, width = np.ascontiguousarray(chars[:, : 64 * W]), 64 * W
    masks = np.empty((R, W), dtype=np.uint64)
    atoms = np.empty((int(n_props), R, W), dtype=np.uint64)
    rc = L.ltl_pack_traces(chars.ctypes.data_as(C.POINTER(C.c_uint16)), lengths.ctypes.data_as(C.POINTER(C.c_int64)), R,
                           int(width), int(n_props), W, int(device), _u64(masks), _u64(atoms))
    if rc != 0:
        msg = (L.ltl_core_last_error(None) or b"").decode()
        if rc == ERR_ARG:
            raise ValueError(msg)
        raise CoreError(f"ltl_pack_traces failed ({rc}): {msg}")
    return masks, atoms


def parse_trace_file(data: bytes):
    """Canonical-form trace file bytes -> ``(pos_chars, pos_lengths, neg_chars, neg_lengths, width, extra_sections)``
    through the library's two-pass reader (`ltl_trace_file_scan` / `_fill`; host code, no device needed), or None when the
    file is not in canonical form (the line-by-line reader then owns the error message)."""
    L = load_library()
    counts = (C.c_int64 * 2)()
    max_len, width, extra = C.c_int(), C.c_int(), C.c_int()
    bad = C.c_int64()
    if L.ltl_trace_file_scan(data, len(data), counts, C.byref(max_len), C.byref(width), C.byref(extra), C.byref(bad)):
        return None
    if width.value < 1:
        return None
    n_pos, n_neg, width_l = int(counts[0]), int(counts[1]), max(int(max_len.value), 1)
    pc, nc = np.zeros((n_pos, width_l), dtype=np.uint16), np.zeros((n_neg, width_l), dtype=np.uint16)
    pl, nl = np.zeros(n_pos, dtype=np.int64), np.zeros(n_neg, dtype=np.int64)
    u16p, i64p = C.POINTER(C.c_uint16), C.POINTER(C.c_int64)
    if L.ltl_trace_file_fill(data, len(data), width.value, width_l, pc.ctypes.data_as(u16p), pl.ctypes.data_as(i64p),
                             nc.ctypes.data_as(u16p), nl.ctypes.data_as(i64p)):
        return None
    return pc, pl, nc, nl, int(width.value), int(extra.value)


class DeviceTraces:
    """A specification resident in HBM (`include/ltl_core.h: ltl_traces_*`): the padded character matrices are uploaded
    once; duplicate screening (reference `traces.py:64-106`), the census of the overfit cost (`formula.py:230-250`),
    trace packing (`bitsem.py:73-88`) and the atom fast path's error counts (`enumerator.py:182-192`) run on the device
    and only counters come back.  `CudaCore.on_traces` / `CudaCore.add_atom` consume the packed masks / atoms in place."""

    INFO_WORDS = 48

    def __init__(self, pos_chars, pos_lengths, neg_chars, neg_lengths, device: int = 0):
        L = load_library()
        if device_count() <= 0:
            raise BackendUnavailable("no CUDA device visible (there is no CPU fallback)")
        pl = np.ascontiguousarray(pos_lengths, dtype=np.int64).reshape(-1)
        nl = np.ascontiguousarray(neg_lengths, dtype=np.int64).reshape(-1)
        pc = np.ascontiguousarray(pos_chars, dtype=np.uint16).reshape(len(pl), -1)
        nc = np.ascontiguousarray(neg_chars, dtype=np.uint16).reshape(len(nl), -1)
        width = max(pc.shape[1] if len(pl) else 0, nc.shape[1] if len(nl) else 0)
        longest = max(int(pl.max()) if len(pl) else 0, int(nl.max()) if len(nl) else 0)
        if 0 <= longest < width:  # columns no trace reaches: words per row follow the longest trace, as on the host
            pc, nc, width = np.ascontiguousarray(pc[:, :longest]), np.ascontiguousarray(nc[:, :longest]), longest
        if len(pl) and pc.shape[1] != width:
            pc = np.ascontiguousarray(np.pad(pc, ((0, 0), (0, width - pc.shape[1]))))
        if len(nl) and nc.shape[1] != width:
            nc = np.ascontiguousarray(np.pad(nc, ((0, 0), (0, width - nc.shape[1]))))
        if (len(pl) and (int(pl.min()) < 0 or int(pl.max()) > width)) or (len(nl) and (int(nl.min()) < 0 or int(nl.max()) > width)):
            raise ValueError("trace lengths must lie in [0, row width]")
        self._L, self._h = L, C.c_void_p()
        self.device_index = int(device)
        u16p, i64p = C.POINTER(C.c_uint16), C.POINTER(C.c_int64)
        rc = L.ltl_traces_create(pc.ctypes.data_as(u16p), pl.ctypes.data_as(i64p), len(pl), nc.ctypes.data_as(u16p),
                                 nl.ctypes.data_as(i64p), len(nl), int(width), int(device), C.byref(self._h))
        if rc:
            msg = (L.ltl_traces_last_error(None) or b"").decode()
            self._h = None
            if rc == ERR_ARG:
                raise ValueError(msg)
            if rc == ERR_CUDA:
                raise BackendUnavailable(f"CUDA core unavailable: {msg} (there is no CPU fallback)")
            raise CoreError(msg)

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._L.ltl_traces_destroy(h)

    __del__ = close

    def _check(self, rc):
        if rc == 0:
            return
        msg = (self._L.ltl_traces_last_error(self._h) or b"").decode()
        if rc == ERR_ARG:
            raise ValueError(msg)
        raise CoreError(f"[{rc}] {msg}")

    def info(self) -> dict:
        out = np.zeros(self.INFO_WORDS, dtype=np.uint64)
        self._check(self._L.ltl_traces_info(self._h, _u64(out)))
        keys = ("rows", "n_pos", "words", "max_len", "min_len", "non_empty", "char_or", "pos_positions", "pos_bits",
                "suspects", "empty_pos", "n_props", "h2d_bytes", "d2h_bytes")
        d = {k: int(v) for k, v in zip(keys, out)}
        d["atom_errors"] = [int(v) for v in out[16:32]]
        d["neg_atom_errors"] = [int(v) for v in out[32:48]]
        return d

    def suspects(self) -> np.ndarray:
        """int64[k, 2]: (row, first row with the same 128-bit hash) -- candidates for being duplicate traces."""
        n = self.info()["suspects"]
        pairs = np.zeros((max(n, 1), 2), dtype=np.int64)
        got = self._L.ltl_traces_suspects(self._h, pairs.ctypes.data_as(C.POINTER(C.c_int64)), n)
        if got < 0:
            self._check(got)
        return pairs[:got]

    def pack(self, n_props: int):
        self._check(self._L.ltl_traces_pack(self._h, int(n_props)))

    def export(self):
        """Host copies of the packed masks ``uint64[R, W]`` and atoms ``uint64[n_props, R, W]`` (tools, tests)."""
        i = self.info()
        R, W, n_props = i["rows"], i["words"], i["n_props"]
        masks = np.empty((R, W), dtype=np.uint64)
        atoms = np.empty((max(n_props, 1), R, W), dtype=np.uint64)
        self._check(self._L.ltl_traces_export(self._h, _u64(masks), _u64(atoms)))
        return masks, atoms[:n_props]


class CudaCore:
    """Device-resident screening core (matrices, records, uniqueness table live in HBM)."""

    def __init__(self, masks, n_pos, err_max, variant, proj_rows: Sequence[int] = (), proj_offs: Sequence[int] = (),
                 fkp_bits=0, mask_k=0, budget_bytes=2 << 30, *, words_per_row=1, device=0, chunk_candidates=None,
                 profile=False, traces: "DeviceTraces | None" = None):
        L = load_library()
        if traces is not None:  # masks are in HBM already (DeviceTraces.pack): `masks` is ignored
            ti = traces.info()
            W, n_words = ti["words"], ti["rows"] * ti["words"]
            n_pos, device = ti["n_pos"], traces.device_index
        else:
            m = np.ascontiguousarray(masks, dtype=np.uint64).reshape(-1)
            W, n_words = int(words_per_row), len(m)
        if W < 1 or W > MAX_WORDS_PER_ROW:
            raise ValueError(f"words_per_row must lie in [1, {MAX_WORDS_PER_ROW}]")
        if n_words == 0 or n_words % W:
            raise ValueError("masks length must be a positive multiple of words_per_row")
        pr = np.ascontiguousarray(list(proj_rows), dtype=np.int32)
        po = np.ascontiguousarray(list(proj_offs), dtype=np.int32)
        if len(pr) != len(po):
            raise ValueError("proj_rows and proj_offs differ in length")
        if len(pr) > 126:
            raise ValueError("projection wider than the fingerprint")  # reference `_speedups.pyx:92-93`
        self.R, self.W, self.n = n_words // W, W, n_words
        self.device_index = int(device)
        self._L = L
        self._h = C.c_void_p()
        i32p = C.POINTER(C.c_int32)
        if traces is not None:
            rc = L.ltl_core_create_on_traces(traces._h, int(err_max), int(variant), pr.ctypes.data_as(i32p),
                                             po.ctypes.data_as(i32p), len(pr), int(fkp_bits), int(mask_k),
                                             int(budget_bytes), C.byref(self._h))
        else:
            rc = L.ltl_core_create(_u64(m), self.R, W, int(n_pos), int(err_max), int(variant), pr.ctypes.data_as(i32p),
                                   po.ctypes.data_as(i32p), len(pr), int(fkp_bits), int(mask_k), int(budget_bytes),
                                   int(device), C.byref(self._h))
        if rc:
            msg = (L.ltl_core_last_error(None) or b"").decode()
            self._h = None
            if rc == ERR_ARG:
                raise ValueError(msg)
            if rc == ERR_CUDA:
                raise BackendUnavailable(f"CUDA core unavailable: {msg} (there is no CPU fallback)")
            raise CoreError(msg)
        if chunk_candidates is not None:
            self.set_option("chunk_candidates", chunk_candidates)
        if profile:
            self.set_option("profile", 1)
        for kv in filter(None, os.environ.get("LTL_CORE_OPTIONS", "").split(",")):  # A/B switches: "name=value,..."
            name, _, value = kv.partition("=")
            self.set_option(name.strip(), int(value))

    # -- lifetime ----------------------------------------------------------------------
    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._L.ltl_core_destroy(h)

    __del__ = close

    def _check(self, rc):
        if rc == 0:
            return
        exc, self._exchange_error = getattr(self, "_exchange_error", None), None
        if exc is not None:  # raised inside the row-shard exchange callback
            raise exc
        msg = (self._L.ltl_core_last_error(self._h) or b"").decode()
        if rc == ERR_BUDGET:
            raise CoreOOM(msg)
        if rc == ERR_ARG:
            raise ValueError(msg)
        if rc == ERR_INVARIANT:  # LTLLEARN_DEBUG_MASKS / option debug_masks: the reference raises AssertionError (bitsem.py:58-61)
            raise AssertionError(msg)
        raise CoreError(f"[{rc}] {msg}")

    def _cm(self, cm) -> np.ndarray:
        a = np.ascontiguousarray(cm, dtype=np.uint64).reshape(-1)
        if len(a) != self.n:
            raise ValueError(f"expected {self.n} words, got {len(a)}")
        return a

    # -- counters ----------------------------------------------------------------------
    def counters(self):
        """(n_entries, bytes_used, offered, admitted, duplicates) -- reference `_speedups.pyx:68, 113-115`."""
        out = np.zeros(5, dtype=np.uint64)
        self._check(self._L.ltl_core_counters(self._h, _u64(out)))
        return [int(v) for v in out]

    n_entries = property(lambda s: s.counters()[0])
    bytes_used = property(lambda s: s.counters()[1])
    offered = property(lambda s: s.counters()[2])
    admitted = property(lambda s: s.counters()[3])
    duplicates = property(lambda s: s.counters()[4])

    # -- contract ----------------------------------------------------------------------
    def add_entry(self, cm, op, lhs, rhs) -> int:
        idx = C.c_int64()
        self._check(self._L.ltl_core_add_entry(self._h, _u64(self._cm(cm)), int(op), int(lhs), int(rhs), C.byref(idx)))
        return int(idx.value)

    def add_atom(self, traces: DeviceTraces, prop: int, negated: bool, op, lhs, rhs) -> int:
        """`add_entry` of a proposition's characteristic matrix (``negated``: its negation inside the length mask) taken
        from the device-resident packed traces -- no host round trip."""
        idx = C.c_int64()
        self._check(self._L.ltl_core_add_atom(self._h, traces._h, int(prop), int(bool(negated)), int(op), int(lhs),
                                              int(rhs), C.byref(idx)))
        return int(idx.value)

    def contains(self, cm) -> bool:
        found = C.c_int()
        self._check(self._L.ltl_core_contains(self._h, _u64(self._cm(cm)), C.byref(found)))
        return bool(found.value)

    def fingerprint_of(self, cm) -> int:
        hi, lo = C.c_uint64(), C.c_uint64()
        self._check(self._L.ltl_core_fingerprint_of(self._h, _u64(self._cm(cm)), C.byref(hi), C.byref(lo)))
        return int(hi.value) << 64 | int(lo.value)

    def get_cm(self, idx) -> np.ndarray:
        out = np.empty(self.n, dtype=np.uint64)
        rc = self._L.ltl_core_get_cm(self._h, int(idx), _u64(out))
        if rc == ERR_ARG:
            raise IndexError((self._L.ltl_core_last_error(self._h) or b"").decode())
        self._check(rc)
        return out

    def get_record(self, idx):
        op, lhs, rhs = C.c_int(), C.c_int(), C.c_int()
        rc = self._L.ltl_core_get_record(self._h, int(idx), C.byref(op), C.byref(lhs), C.byref(rhs))
        if rc == ERR_ARG:
            raise IndexError((self._L.ltl_core_last_error(self._h) or b"").decode())
        self._check(rc)
        return op.value, lhs.value, rhs.value

    def get_subtree(self, idx, cap: int = 1024) -> dict:
        """``{entry: (op, lhs, rhs)}`` for every entry reachable from ``idx`` (`ltl_core_get_subtree`)."""
        nodes = np.empty((int(cap), 4), dtype=np.int32)
        n = C.c_int()
        rc = self._L.ltl_core_get_subtree(self._h, int(idx), int(cap), nodes.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(n))
        if rc == ERR_ARG:
            raise IndexError((self._L.ltl_core_last_error(self._h) or b"").decode())
        self._check(rc)
        return {int(e): (int(op), int(lhs), int(rhs)) for e, op, lhs, rhs in nodes[: n.value]}

    def export_cms(self, first=0, count=None) -> np.ndarray:
        n = self.n_entries
        count = n - first if count is None else count
        out = np.empty((count, self.n), dtype=np.uint64)
        if count:
            self._check(self._L.ltl_core_export_cms(self._h, int(first), int(count), _u64(out)))
        return out

    def export_records(self, first=0, count=None):
        n = self.n_entries
        count = n - first if count is None else count
        op = np.empty(count, dtype=np.int8)
        lhs = np.empty(count, dtype=np.int32)
        rhs = np.empty(count, dtype=np.int32)
        if count:
            self._check(self._L.ltl_core_export_records(self._h, int(first), int(count),
                                                        op.ctypes.data_as(C.POINTER(C.c_int8)),
                                                        lhs.ctypes.data_as(C.POINTER(C.c_int32)),
                                                        rhs.ctypes.data_as(C.POINTER(C.c_int32))))
        return op, lhs, rhs

    def entry_fingerprints(self, first=0, count=None):
        n = self.n_entries
        count = n - first if count is None else count
        hi = np.empty(count, dtype=np.uint64)
        lo = np.empty(count, dtype=np.uint64)
        if count:
            self._check(self._L.ltl_core_entry_fingerprints(self._h, int(first), int(count), _u64(hi), _u64(lo)))
        return hi, lo

    def screen_unary(self, op, c0, c1):
        st, li, ri = C.c_int(), C.c_int64(), C.c_int64()
        self._check(self._L.ltl_core_screen_unary(self._h, int(op), int(c0), int(c1), C.byref(st), C.byref(li),
                                                  C.byref(ri)))
        return st.value, li.value, ri.value

    def screen_binary(self, op, a0, a1, b0, b1, tri):
        st, li, ri = C.c_int(), C.c_int64(), C.c_int64()
        self._check(self._L.ltl_core_screen_binary(self._h, int(op), int(a0), int(a1), int(b0), int(b1),
                                                   int(bool(tri)), C.byref(st), C.byref(li), C.byref(ri)))
        return st.value, li.value, ri.value

    def run_level(self, segments):
        """Screen a whole cost level.  ``segments``: iterable of objects with ``op, a0, a1, b0, b1, tri``
        in enumeration order.  Returns ``(status, segment_index, li, ri)``."""
        segments = list(segments)
        arr = (Segment * max(1, len(segments)))()
        for k, s in enumerate(segments):
            arr[k] = Segment(int(s.op), int(bool(s.tri)), int(s.a0), int(s.a1), int(s.b0), int(s.b1))
        st, seg, li, ri = C.c_int(), C.c_int(), C.c_int64(), C.c_int64()
        self._check(self._L.ltl_core_run_level(self._h, arr, len(segments), C.byref(st), C.byref(seg), C.byref(li),
                                               C.byref(ri)))
        return st.value, seg.value, li.value, ri.value

    def run_search(self, op_cost, op_mask: int, buckets, first_cost: int, ceiling: int, store_last_level: bool = False):
        """The whole cost-level loop in the library (`ltl_core_run_search`; reference `enumerator.py:234-251`).
        ``op_cost``: 8 connective costs by opcode; ``buckets``: ``{cost: (first, end)}`` admitted so far.
        Returns ``(status, op, li, ri, end_cost, rows)`` with one dict per level that ended."""
        oc = np.ascontiguousarray(list(op_cost), dtype=np.int32)
        bc = np.ascontiguousarray([c for c in buckets], dtype=np.int64)
        bf = np.ascontiguousarray([buckets[c][0] for c in buckets], dtype=np.int64)
        be = np.ascontiguousarray([buckets[c][1] for c in buckets], dtype=np.int64)
        n_levels = max(0, int(ceiling) - int(first_cost))
        rows = (LevelStats * max(1, n_levels))()
        n_rows, st, op, end_cost = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        li, ri = C.c_int64(), C.c_int64()
        i32p, i64p = C.POINTER(C.c_int32), C.POINTER(C.c_int64)
        self._check(self._L.ltl_core_run_search(self._h, oc.ctypes.data_as(i32p), int(op_mask), bc.ctypes.data_as(i64p),
                                                bf.ctypes.data_as(i64p), be.ctypes.data_as(i64p), len(bc), int(first_cost),
                                                int(ceiling), int(bool(store_last_level)), rows, n_levels, C.byref(n_rows),
                                                C.byref(st), C.byref(op), C.byref(li), C.byref(ri), C.byref(end_cost)))
        out = [{"cost": r.cost, "offered": r.offered, "admitted": r.admitted, "duplicates": r.duplicates, "bytes": r.bytes,
                "ms": round(r.ms, 3), "entries": (r.first_entry, r.end_entry), "status": r.status}
               for r in rows[: n_rows.value]]
        return st.value, op.value, li.value, ri.value, end_cost.value, out

    # -- row shard (see sharded.RowShardedCore) --------------------------------------------
    def set_row_shard(self, word_base: int, total_words: int, all_reduce_sum):
        """Make this core one row shard of a larger specification.  ``all_reduce_sum(tensors)`` must add, in place
        and across all shards, the given device tensors (one int64 tensor of 3 words per candidate: wrapping sums) and
        return once the result is visible to the device.  It is called for up to ``exchange_parts`` consecutive
        candidate ranges of a pass, each while the next range is still being evaluated on the core's own stream."""
        import torch

        dev = torch.device("cuda", self.device_index)

        class _Dev:  # zero-copy view of a device array of the library (CUDA array interface)
            def __init__(self, ptr, n, typestr):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (int(ptr), False), "version": 2}

        def hook(_ctx, sums, count):
            try:
                all_reduce_sum([torch.as_tensor(_Dev(sums, 3 * int(count), "<i8"), device=dev)])
                return 0
            except BaseException as exc:  # noqa: BLE001 -- no exception may cross the C ABI
                self._exchange_error = exc
                return 1

        self._exchange_error = None
        self._exchange_cb = EXCHANGE_FN(hook)  # keep the trampoline alive as long as the core
        self._check(self._L.ltl_core_set_row_shard(self._h, int(word_base), int(total_words), self._exchange_cb, None))

    def set_table_shard(self, shard: int, n_shards: int):
        """Row shards: also shard the uniqueness table by fingerprint owner (`ltl_core_set_table_shard`)."""
        self._check(self._L.ltl_core_set_table_shard(self._h, int(shard), int(n_shards)))

    # -- multi-GPU stages (device tensors in / out; see sharded.py) -----------------------
    @staticmethod
    def _segments(segments):
        segments = list(segments)
        arr = (Segment * max(1, len(segments)))()
        for k, s in enumerate(segments):
            arr[k] = Segment(int(s.op), int(bool(s.tri)), int(s.a0), int(s.a1), int(s.b0), int(s.b1))
        return arr, len(segments)

    def level_size(self, segments) -> int:
        arr, n = self._segments(segments)
        total = C.c_int64()
        self._check(self._L.ltl_core_level_size(self._h, arr, n, C.byref(total)))
        return int(total.value)

    def stage_eval(self, segments, lo: int, hi: int):
        """Fingerprints of level ranks [lo, hi): int64[hi - lo, 2] device tensor (hi, lo bit patterns), and the
        lowest solving level rank of the slice or -1."""
        import torch

        dev = torch.device("cuda", self.device_index)
        fp = torch.empty((max(hi - lo, 0), 2), dtype=torch.int64, device=dev)
        arr, n = self._segments(segments)
        solver = C.c_int64(-1)
        torch.cuda.current_stream(dev).synchronize()
        self._check(self._L.ltl_core_stage_eval(self._h, arr, n, int(lo), int(hi), C.c_void_p(fp.data_ptr()),
                                                C.byref(solver)))
        return fp, int(solver.value)

    def stage_file(self, tuples):
        """Owner side: file int64[N, 3] (hi, lo, global rank) device tuples; uint8[N] winner flags."""
        import torch

        tuples = tuples.contiguous()
        win = torch.zeros(tuples.shape[0], dtype=torch.uint8, device=tuples.device)
        n_win = C.c_int64()
        torch.cuda.current_stream(tuples.device).synchronize()
        self._check(self._L.ltl_core_stage_file(self._h, C.c_void_p(tuples.data_ptr()), tuples.shape[0],
                                                C.c_void_p(win.data_ptr()), C.byref(n_win)))
        return win

    def stage_route(self, fp, rank_base: int, world: int):
        """Fingerprints int64[N, 2] of consecutive candidates (global ranks ``rank_base ..``) -> int64[N, 3] tuples
        ``(hi, lo, global rank)`` grouped by owner rank, and the number of tuples per owner (`ltl_core_stage_route`: a
        stable counting sort by owner on the device)."""
        import torch

        fp = fp.contiguous()
        n = fp.shape[0]
        send = torch.empty((n, 3), dtype=torch.int64, device=fp.device)
        counts = (C.c_int64 * int(world))()
        torch.cuda.current_stream(fp.device).synchronize()
        self._check(self._L.ltl_core_stage_route(self._h, C.c_void_p(fp.data_ptr()), n, int(rank_base) & 0xFFFFFFFFFFFFFFFF,
                                                 int(world), C.c_void_p(send.data_ptr()), counts))
        return send, [int(v) for v in counts]

    def stage_winners(self, send, win, rank_base: int, level_lo: int):
        """Verdict bytes ``win`` (uint8[N], in the order of the tuples ``send``) -> ascending level ranks of the winners
        (int64 device tensor; `ltl_core_stage_winners`)."""
        import torch

        win = win.contiguous()
        n = send.shape[0]
        out = torch.empty(n, dtype=torch.int64, device=send.device)
        n_out = C.c_int64()
        torch.cuda.current_stream(send.device).synchronize()
        self._check(self._L.ltl_core_stage_winners(self._h, C.c_void_p(send.data_ptr()), C.c_void_p(win.data_ptr()), n,
                                                   int(rank_base) & 0xFFFFFFFFFFFFFFFF, int(level_lo),
                                                   C.c_void_p(out.data_ptr()), C.byref(n_out)))
        return out[: int(n_out.value)]

    def stage_decode(self, segments, ranks):
        """Level ranks (int64 device tensor) -> (op uint8, lhs int32, rhs int32) device tensors."""
        import torch

        ranks = ranks.contiguous()
        n = ranks.shape[0]
        op = torch.empty(n, dtype=torch.uint8, device=ranks.device)
        lhs = torch.empty(n, dtype=torch.int32, device=ranks.device)
        rhs = torch.empty(n, dtype=torch.int32, device=ranks.device)
        arr, ns = self._segments(segments)
        torch.cuda.current_stream(ranks.device).synchronize()
        self._check(self._L.ltl_core_stage_decode(self._h, arr, ns, C.c_void_p(ranks.data_ptr()), n,
                                                  C.c_void_p(op.data_ptr()), C.c_void_p(lhs.data_ptr()),
                                                  C.c_void_p(rhs.data_ptr())))
        return op, lhs, rhs

    def stage_append(self, op, lhs, rhs, offered_delta: int, duplicates_delta: int):
        import torch

        op, lhs, rhs = op.contiguous(), lhs.contiguous(), rhs.contiguous()
        torch.cuda.current_stream(op.device).synchronize()
        self._check(self._L.ltl_core_stage_append(self._h, C.c_void_p(op.data_ptr()), C.c_void_p(lhs.data_ptr()),
                                                  C.c_void_p(rhs.data_ptr()), op.shape[0], int(offered_delta),
                                                  int(duplicates_delta)))

    def stage_purge(self, global_rank_cut: int):
        self._check(self._L.ltl_core_stage_purge(self._h, int(global_rank_cut)))

    def capacity_entries(self) -> int:
        return self.info()["capacity_entries"]

    def stage_device(self):
        import torch

        return torch.device("cuda", self.device_index)

    # -- tuning / measurement ------------------------------------------------------------
    def set_option(self, name: str, value: int):
        self._check(self._L.ltl_core_set_option(self._h, name.encode(), int(value)))

    def kernel_stats(self) -> dict:
        out = {}
        for k, name in enumerate(KERNEL_CLASSES):
            launches, units = C.c_uint64(), C.c_uint64()
            ms, nbytes = C.c_double(), C.c_double()
            self._check(self._L.ltl_core_kernel_stats(self._h, k, C.byref(launches), C.byref(ms), C.byref(nbytes),
                                                      C.byref(units)))
            out[name] = {"launches": int(launches.value), "ms": float(ms.value), "alg_bytes": float(nbytes.value),
                         "units": int(units.value)}
        return out

    def reset_kernel_stats(self):
        self._check(self._L.ltl_core_reset_kernel_stats(self._h))

    def stream_handle(self) -> int:
        """The cudaStream_t all work of this core is issued on (for CUDA-event timing by the caller)."""
        out = C.c_void_p()
        self._check(self._L.ltl_core_stream(self._h, C.byref(out)))
        return int(out.value or 0)

    def host_times(self) -> dict:
        """Host wall milliseconds: growing the store, waiting for the device, planning."""
        out = (C.c_double * 3)()
        self._check(self._L.ltl_core_host_times(self._h, out))
        return {"grow_ms": out[0], "sync_ms": out[1], "plan_ms": out[2]}

    def transfer_stats(self) -> tuple[int, int]:
        """(host->device bytes, device->host bytes) copied so far."""
        out = np.zeros(2, dtype=np.uint64)
        self._check(self._L.ltl_core_transfer_stats(self._h, _u64(out)))
        return int(out[0]), int(out[1])

    def info(self) -> dict:
        out = np.zeros(6, dtype=np.uint64)
        self._check(self._L.ltl_core_info(self._h, _u64(out)))
        keys = ("capacity_entries", "matrix_bytes_mapped", "table_slots", "chunk_candidates", "flags", "words_per_matrix")
        d = {k: int(v) for k, v in zip(keys, out)}
        d["vmm"], d["device_oom"], d["gated_skips"] = bool(d["flags"] & 1), bool(d["flags"] & 2), d["flags"] >> 8
        return d


def make_core(masks, n_pos, err_max, variant, proj_rows=(), proj_offs=(), fkp_bits=0, mask_k=0,
              budget_bytes=2 << 30, *, words_per_row=1, device=0, **options) -> CudaCore:
    """The drop-in for reference `kernels.make_core` (`kernels.py:140-172`): always the CUDA core.
    ``traces=DeviceTraces`` (keyword): a core over a specification already packed in HBM (``masks`` may be None)."""
    return CudaCore(masks, n_pos, err_max, variant, proj_rows, proj_offs, fkp_bits, mask_k, budget_bytes,
                    words_per_row=words_per_row, device=device, **options)
