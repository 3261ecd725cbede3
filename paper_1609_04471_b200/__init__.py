"""sr_sort: a B200-native adaptive comparison sort (after arXiv 1609.04471, "Sort Race").

Thin ctypes binding over libsr_sort.so (include/sr_sort.h).  Argument
marshalling only: every step of the sort runs in the CUDA kernels of csrc/.
PyTorch supplies device memory and streams.  There is no CPU fallback: if the
library cannot be loaded, every call raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

SR_INT32, SR_INT64, SR_FLOAT32, SR_FLOAT64 = 0, 1, 2, 3  # include/sr_sort.h
STATUS = {0: "ok", 1: "invalid argument", 2: "unsupported dtype", 3: "size out of range", 4: "misaligned pointer",
          5: "out of device memory", 6: "CUDA error", 7: "internal error"}
ROUTES = {0: "none", 1: "sorted", 2: "reversed", 3: "merge", 4: "partition", 5: "tile", 6: "outlier", 7: "distance"}
ROUTE_MERGE, ROUTE_PARTITION, ROUTE_OUTLIER = 3, 4, 6
OPT_FORCE_ROUTE, OPT_PROFILE, OPT_MERGE_ROUTE, OPT_RESIDENT, OPT_RESIDENT_CAP, OPT_OUTLIER_ROUTE, OPT_WS_LIMIT = (
    0, 1, 2, 3, 4, 5, 6)
OPT_DISTANCE_ROUTE = 7
OPT_TUNE = 16  # + 0 fused second level, + 1 level-1 buckets (n >= 2^26), + 2 fused mean sub-bucket

EXPORTS = [
    "sr_sort_keys", "sr_sort_pairs", "sr_sort_host", "sr_sort_host_batch", "sr_sort_records", "sr_presortedness", "sr_last_plan", "sr_status_string", "sr_last_error",
    "sr_set_option", "sr_last_profile", "sr_presort_scan", "sr_reverse_range", "sr_tile_sort", "sr_merge_path",
    "sr_merge", "sr_splitters", "sr_partition_level", "sr_generate",
]


class SrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"sr_sort error {status} ({STATUS.get(status, '?')}): {msg}")
        self.status = status


class Plan(ctypes.Structure):
    _fields_ = [("route", ctypes.c_int32), ("levels", ctypes.c_int32), ("n", ctypes.c_int64),
                ("descents", ctypes.c_int64), ("asc_breaks", ctypes.c_int64), ("long_runs", ctypes.c_int64),
                ("desc_runs_reversed", ctypes.c_int64), ("equal_keys", ctypes.c_int64),
                ("bytes_planned", ctypes.c_int64), ("workspace_bytes", ctypes.c_int64),
                ("launches", ctypes.c_int32), ("host_syncs", ctypes.c_int32)]


class PresortStats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in
                ("n", "descents", "asc_breaks", "n_asc_runs", "n_desc_runs", "asc_cover", "desc_cover")]


_lib = None


def lib():
    """Load (building in-tree if the sources are newer) libsr_sort.so, or with
    SR_CHECKED_LIB=1 the checked build libsr_sort_checked.so (device-side index
    checks, build.py --checked)."""
    global _lib
    if _lib is None:
        checked = os.environ.get("SR_CHECKED_LIB", "0") not in ("", "0")
        path = _build.LIB_CHECKED if checked else _build.LIB
        if _build.needs_build(checked):
            _build.build(checked=checked)
        if not os.path.exists(path):
            raise ImportError(f"libsr_sort.so missing at {path}; run paper_1609_04471_b200/build.py")
        L = ctypes.CDLL(path)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        L.sr_sort_keys.argtypes = [vp, i64, i32, vp]
        L.sr_sort_pairs.argtypes = [vp, vp, i64, i32, vp]
        L.sr_sort_host.argtypes = [vp, vp, i64, i32, vp]
        L.sr_sort_host_batch.argtypes = [vp, vp, vp, i32, i32, vp]
        L.sr_sort_records.argtypes = [vp, i64, i32, vp]
        L.sr_presortedness.argtypes = [vp, i64, i32, ctypes.POINTER(Measures), vp]
        L.sr_last_plan.argtypes = [ctypes.POINTER(Plan)]
        L.sr_generate.argtypes = [vp, i64, i32, i32, ctypes.c_uint64, i64, vp]
        L.sr_status_string.argtypes = [i32]
        L.sr_status_string.restype = ctypes.c_char_p
        L.sr_last_error.argtypes = []
        L.sr_last_error.restype = ctypes.c_char_p
        L.sr_set_option.argtypes = [i32, i64]
        L.sr_last_profile.argtypes = [vp, vp, vp, i32]
        L.sr_presort_scan.argtypes = [vp, i64, i32, i32, i32, ctypes.POINTER(PresortStats), vp, i64, vp]
        L.sr_reverse_range.argtypes = [vp, vp, i64, i32, i64, i64, vp]
        L.sr_tile_sort.argtypes = [vp, vp, i64, i32, i32, vp]
        L.sr_merge_path.argtypes = [vp, i64, vp, i64, i32, vp, vp, i64, vp]
        L.sr_merge.argtypes = [vp, vp, i64, vp, vp, i64, vp, vp, i32, vp]
        L.sr_splitters.argtypes = [vp, i64, i32, i32, vp, vp, ctypes.POINTER(i32), vp]
        L.sr_partition_level.argtypes = [vp, vp, i64, i32, i32, vp, vp, vp, vp]
        for name in EXPORTS:
            if name not in ("sr_status_string", "sr_last_error"):
                getattr(L, name).restype = i32
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise SrError(rc, lib().sr_last_error().decode())


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.int32:
        return SR_INT32
    if t.dtype == torch.int64:
        return SR_INT64
    if t.dtype == torch.float32:
        return SR_FLOAT32
    if t.dtype == torch.float64:
        return SR_FLOAT64
    raise TypeError(f"keys must be int32, int64, float32 or float64, got {t.dtype}")


def _stream(t):
    """The tensor's device's current CUDA stream (raw handle; the private
    accessor skips building a torch.cuda.Stream object, ~2 us per call)."""
    import torch
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return ctypes.c_void_p(raw(t.device.index))
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _dev(t, name):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _vals_ok(v):
    import torch
    if v.element_size() != 4:
        raise TypeError("vals must have 4-byte elements")


# ----------------------------------------------------------------------------- sort

def sort_keys(keys):
    """Sort a CUDA int32/int64 (signed order) or float32/float64 (IEEE totalOrder)
    tensor ascending in place (sr_sort_keys)."""
    _dev(keys, "keys")
    _check(lib().sr_sort_keys(_ptr(keys), keys.numel(), _dtype_code(keys), _stream(keys)))
    return keys


def sort_pairs(keys, vals):
    """Stable key-value sort in place (sr_sort_pairs); vals: any 4-byte dtype."""
    _dev(keys, "keys")
    _dev(vals, "vals")
    _vals_ok(vals)
    if vals.numel() != keys.numel():
        raise ValueError("keys and vals differ in length")
    _check(lib().sr_sort_pairs(_ptr(keys), _ptr(vals), keys.numel(), _dtype_code(keys), _stream(keys)))
    return keys, vals


class Measures(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in ["n", "runs", "inversions", "mono", "max_dis", "misplaced"]]


def presortedness(keys) -> dict:
    """Presortedness measures of a CUDA int32/int64 tensor (sr_presortedness,
    PAPER.md:62-85): runs, inversions, mono, max_dis, misplaced."""
    _dev(keys, "keys")
    m = Measures()
    _check(lib().sr_presortedness(_ptr(keys), keys.numel(), _dtype_code(keys), ctypes.byref(m), _stream(keys)))
    return {f: getattr(m, f) for f, _ in Measures._fields_}


def sort_records(recs):
    """Sort the rows of a CUDA int32 tensor of shape (n, words) ascending in
    lexicographic order, in place (sr_sort_records; record keys, the paper's
    16-/64-/256-int lists)."""
    import torch
    _dev(recs, "recs")
    if recs.dtype != torch.int32 or recs.dim() != 2:
        raise TypeError("recs must be a 2-D int32 tensor (n, words)")
    _check(lib().sr_sort_records(_ptr(recs), recs.shape[0], recs.shape[1], _stream(recs)))
    return recs


def sort_host(keys: np.ndarray, vals: np.ndarray | None = None, stream: int = 0):
    """End-to-end sort of HOST numpy arrays in place (sr_sort_host)."""
    codes = {np.dtype(np.int32): SR_INT32, np.dtype(np.int64): SR_INT64,
             np.dtype(np.float32): SR_FLOAT32, np.dtype(np.float64): SR_FLOAT64}
    if keys.dtype not in codes:
        raise TypeError("keys must be int32, int64, float32 or float64")
    code = codes[keys.dtype]
    assert keys.flags.c_contiguous and (vals is None or (vals.flags.c_contiguous and vals.itemsize == 4))
    vp = None if vals is None else vals.ctypes.data_as(ctypes.c_void_p)
    _check(lib().sr_sort_host(keys.ctypes.data_as(ctypes.c_void_p), vp, keys.size, code, ctypes.c_void_p(stream)))
    return keys if vals is None else (keys, vals)


def sort_host_batch(keys: list, vals: list | None = None, stream: int = 0):
    """End-to-end sort of a batch of HOST numpy arrays of one dtype in place,
    uploads and downloads overlapped with the sorts (sr_sort_host_batch)."""
    codes = {np.dtype(np.int32): SR_INT32, np.dtype(np.int64): SR_INT64,
             np.dtype(np.float32): SR_FLOAT32, np.dtype(np.float64): SR_FLOAT64}
    count = len(keys)
    if count == 0:
        return keys
    if keys[0].dtype not in codes or any(k.dtype != keys[0].dtype for k in keys):
        raise TypeError("keys must all be int32, int64, float32 or float64 arrays of one dtype")
    assert all(k.flags.c_contiguous for k in keys)
    assert vals is None or (len(vals) == count and all(
        v is None or (v.flags.c_contiguous and v.itemsize == 4 and v.size == k.size) for k, v in zip(keys, vals)))
    kp = (ctypes.c_void_p * count)(*[k.ctypes.data for k in keys])
    vp = None if vals is None else (ctypes.c_void_p * count)(*[None if v is None else v.ctypes.data for v in vals])
    ns = (ctypes.c_int64 * count)(*[k.size for k in keys])
    _check(lib().sr_sort_host_batch(kp, vp, ns, count, codes[keys[0].dtype], ctypes.c_void_p(stream)))
    return keys if vals is None else (keys, vals)


GEN_ORDERS = {"random": 0, "sorted": 1, "reversed": 2, "swaps": 3, "few_unique": 4, "runs": 5, "last": 6,
              "sharp_teeth": 7, "equal_teeth": 8, "even_teeth": 9, "distance": 10, "all_equal": 11, "extremes": 12}


def generate(out, order: str, seed: int, param: int = 0):
    """Fill the CUDA int32/int64 tensor `out` with an input of class `order`
    on the device (sr_generate; bit-identical to workloads/gen.py for the same
    seed; see include/sr_sort.h for `param`)."""
    _dev(out, "out")
    code = _dtype_code(out)
    if code not in (SR_INT32, SR_INT64):
        raise TypeError("generate: int32 or int64 tensors only")
    _check(lib().sr_generate(_ptr(out), out.numel(), code, GEN_ORDERS[order], seed & (2**64 - 1), int(param),
                             _stream(out)))
    return out


def last_plan() -> dict:
    p = Plan()
    _check(lib().sr_last_plan(ctypes.byref(p)))
    d = {f: getattr(p, f) for f, _ in Plan._fields_}
    d["route_name"] = ROUTES.get(d["route"], "?")
    return d


def set_option(key: int, value: int):
    _check(lib().sr_set_option(key, value))


def last_profile():
    """[(kernel name, device ms, algorithmic bytes)] of the last call (needs OPT_PROFILE)."""
    n = lib().sr_last_profile(None, None, None, 0)
    if n <= 0:
        return []
    names = (ctypes.c_char_p * n)()
    ms = (ctypes.c_float * n)()
    by = (ctypes.c_int64 * n)()
    lib().sr_last_profile(names, ms, by, n)
    return [(names[i].decode(), float(ms[i]), int(by[i])) for i in range(n)]


# ----------------------------------------------------------------------------- step-level entry points

def presort_scan(keys, strict: bool = False, tile: int = 4096):
    """H1: (stats dict, [(start, len, dir)]) for runs >= tile (dir 0 asc, 1 desc)."""
    _dev(keys, "keys")
    st = PresortStats()
    cap = keys.numel() // tile + 4
    rows = np.zeros((cap * 2, 4), np.int64)
    _check(lib().sr_presort_scan(_ptr(keys), keys.numel(), _dtype_code(keys), int(strict), tile, ctypes.byref(st),
                                 rows.ctypes.data_as(ctypes.c_void_p), cap * 2, _stream(keys)))
    stats = {f: getattr(st, f) for f, _ in PresortStats._fields_}
    nr = stats["n_asc_runs"] + stats["n_desc_runs"]
    return stats, [tuple(int(x) for x in r[:3]) for r in rows[:nr]]


def reverse_range(keys, s: int, e: int, vals=None):
    """H2: reverse keys[s:e] (and vals) in place."""
    _dev(keys, "keys")
    _check(lib().sr_reverse_range(_ptr(keys), _ptr(vals), keys.numel(), _dtype_code(keys), s, e, _stream(keys)))


def tile_sort(keys, tile: int, vals=None):
    """H4: stable sort of every tile of `tile` elements independently (in place)."""
    _dev(keys, "keys")
    _check(lib().sr_tile_sort(_ptr(keys), _ptr(vals), keys.numel(), _dtype_code(keys), tile, _stream(keys)))


def merge_path(a, b, diags):
    """H5: #A among the first d outputs of the stable merge, for each d in diags."""
    d = np.ascontiguousarray(np.asarray(diags, dtype=np.int64))
    out = np.zeros_like(d)
    _check(lib().sr_merge_path(_ptr(a), a.numel(), _ptr(b), b.numel(), _dtype_code(a),
                               d.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p), d.size,
                               _stream(a)))
    return out


def merge(a, b, va=None, vb=None):
    """H6: stable merge of two sorted CUDA tensors (A wins ties) -> out (, vout)."""
    import torch
    out = torch.empty(a.numel() + b.numel(), dtype=a.dtype, device=a.device)
    vout = None if va is None else torch.empty(out.numel(), dtype=va.dtype, device=a.device)
    _check(lib().sr_merge(_ptr(a), _ptr(va), a.numel(), _ptr(b), _ptr(vb), b.numel(), _ptr(out), _ptr(vout),
                          _dtype_code(a), _stream(a)))
    return out if vout is None else (out, vout)


def splitters(keys, nbuckets: int):
    """H7: (splitters int64[m], equality flags uint8[m])."""
    _dev(keys, "keys")
    spl = np.zeros(nbuckets, np.int64)
    eq = np.zeros(nbuckets, np.uint8)
    m = ctypes.c_int32(0)
    _check(lib().sr_splitters(_ptr(keys), keys.numel(), _dtype_code(keys), nbuckets,
                              spl.ctypes.data_as(ctypes.c_void_p), eq.ctypes.data_as(ctypes.c_void_p),
                              ctypes.byref(m), _stream(keys)))
    return spl[:m.value], eq[:m.value]


def partition_level(keys, nbuckets: int, vals=None):
    """H8-H10: one stable partition level -> (out keys, out vals|None, counts[2*nbuckets+1])."""
    import torch
    _dev(keys, "keys")
    out = torch.empty_like(keys)
    vout = None if vals is None else torch.empty_like(vals)
    counts = np.zeros(2 * nbuckets + 1, np.int64)
    _check(lib().sr_partition_level(_ptr(keys), _ptr(vals), keys.numel(), _dtype_code(keys), nbuckets, _ptr(out),
                                    _ptr(vout), counts.ctypes.data_as(ctypes.c_void_p), _stream(keys)))
    return out, vout, counts
