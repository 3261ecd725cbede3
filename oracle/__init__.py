"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, single-threaded C (oracle.c, built with gcc -O2) behind numpy
wrappers.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package; the product package
(paper_1609_04471_b200) never does and shares no code with it.
Each wrapper cites the passage its C function follows (see oracle.c header).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc -O2; no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, c64, c32, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int
        L.or_sort.argtypes = [vp, vp, c64, ci]
        L.or_sort.restype = ci
        L.or_descents.argtypes = [vp, c64, ci]
        L.or_descents.restype = c64
        L.or_asc_runs.argtypes = [vp, c64, ci, vp, vp, c64]
        L.or_asc_runs.restype = c64
        L.or_desc_runs.argtypes = [vp, c64, ci, ci, vp, vp, c64]
        L.or_desc_runs.restype = c64
        L.or_reverse.argtypes = [vp, vp, c64, c64, ci]
        L.or_reverse.restype = None
        L.or_merge.argtypes = [vp, vp, c64, vp, vp, c64, vp, vp, ci]
        L.or_merge.restype = None
        L.or_merge_path.argtypes = [vp, c64, vp, c64, c64, ci]
        L.or_merge_path.restype = c64
        L.or_sample_pos.argtypes = [c64, c64, c64, c64]
        L.or_sample_pos.restype = c64
        L.or_splitters.argtypes = [vp, c64, c64, c32, c32, ci, vp, vp]
        L.or_splitters.restype = c32
        L.or_classify.argtypes = [vp, c64, ci, vp, vp, c32, vp]
        L.or_classify.restype = None
        L.or_stable_partition.argtypes = [vp, c64, c32, vp, vp, vp, vp, vp, ci]
        L.or_stable_partition.restype = ci
        L.or_count.argtypes = [vp, c64, ci, c64, i64p]
        L.or_count.restype = c64
        L.or_stable_rank.argtypes = [vp, c64, ci, c64]
        L.or_stable_rank.restype = c64
        L.or_sort_float.argtypes = [vp, vp, c64, ci]
        L.or_sort_float.restype = ci
        L.or_sort_records.argtypes = [vp, c64, ci, vp]
        L.or_sort_records.restype = ci
        L.or_measures.argtypes = [vp, c64, ci, vp]
        L.or_measures.restype = ci
        _lib = L
    return _lib


def _ks(a: np.ndarray) -> int:
    if a.dtype == np.int32:
        return 4
    if a.dtype == np.int64:
        return 8
    raise TypeError(f"oracle keys must be int32 or int64, got {a.dtype}")


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _fs(a: np.ndarray) -> int:
    return {np.dtype(np.float32): 4, np.dtype(np.float64): 8}.get(a.dtype, 0)


def sort_keys(keys: np.ndarray) -> np.ndarray:
    """Ascending sort (plain stable mergesort): signed order for integers,
    IEEE 754 totalOrder for float32/float64.  Returns a new array."""
    out = np.ascontiguousarray(keys).copy()
    rc = lib().or_sort_float(_p(out), None, out.size, _fs(out)) if _fs(out) else \
        lib().or_sort(_p(out), None, out.size, _ks(out))
    if rc != 0:
        raise MemoryError("oracle sort: out of host memory")
    return out


def sort_pairs(keys: np.ndarray, vals: np.ndarray):
    """Stable key-value sort: equal keys keep input order."""
    k = np.ascontiguousarray(keys).copy()
    v = np.ascontiguousarray(vals).view(np.uint32).copy()
    assert k.size == v.size
    rc = lib().or_sort_float(_p(k), _p(v), k.size, _fs(k)) if _fs(k) else lib().or_sort(_p(k), _p(v), k.size, _ks(k))
    if rc != 0:
        raise MemoryError("oracle sort: out of host memory")
    return k, v.view(vals.dtype)


def sort_records(recs: np.ndarray, with_perm: bool = False):
    """Records (rows of an (n, words) int32 array) in ascending lexicographic
    order by a plain stable mergesort (PAPER.md:58 lists).  Returns a new array
    (and the input row of every output row with with_perm)."""
    r = np.ascontiguousarray(recs, dtype=np.int32).copy()
    n, words = r.shape
    perm = np.zeros(n, np.int64)
    if lib().or_sort_records(_p(r), n, words, _p(perm)) != 0:
        raise MemoryError("oracle sort: out of host memory")
    return (r, perm) if with_perm else r


def measures(keys: np.ndarray) -> dict:
    """Presortedness measures: Run, Inv, Mono, Dis (max
    |rank - i|, k-distance) and the number of misplaced elements (k-exchange)."""
    k = np.ascontiguousarray(keys)
    out = np.zeros(5, np.int64)
    if lib().or_measures(_p(k), k.size, _ks(k), _p(out)) != 0:
        raise MemoryError("oracle measures: out of host memory")
    return dict(zip(["runs", "inversions", "mono", "max_dis", "misplaced"], out.tolist()))


def descents(keys: np.ndarray) -> int:
    """D = |{i: a_i > a_{i+1}}| = Run(A) - 1."""
    k = np.ascontiguousarray(keys)
    return int(lib().or_descents(_p(k), k.size, _ks(k)))


def _runs(fn, keys, *extra):
    k = np.ascontiguousarray(keys)
    cap = max(1, k.size)
    st = np.zeros(cap, np.int64)
    ln = np.zeros(cap, np.int64)
    cnt = fn(_p(k), k.size, _ks(k), *extra, _p(st), _p(ln), cap)
    return [(int(s), int(l)) for s, l in zip(st[:cnt], ln[:cnt])]


def asc_runs(keys: np.ndarray):
    """Maximal ascending (non-decreasing) runs as (start, len)."""
    return _runs(lib().or_asc_runs, keys)


def desc_runs(keys: np.ndarray, strict: bool):
    """Maximal descending runs: non-increasing (keys-only) or strictly decreasing
    (pairs)."""
    return _runs(lib().or_desc_runs, keys, 1 if strict else 0)


def reverse(keys: np.ndarray, s: int, e: int, vals: np.ndarray | None = None):
    """Reverse a[s..e) in place."""
    lib().or_reverse(_p(keys), _p(vals), s, e, _ks(keys))


def merge(a, b, va=None, vb=None):
    """Stable merge of two sorted runs, A wins ties."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.dtype == b.dtype
    out = np.empty(a.size + b.size, a.dtype)
    vout = np.empty(out.size, np.uint32) if va is not None else None
    va = None if va is None else np.ascontiguousarray(va).view(np.uint32)
    vb = None if vb is None else np.ascontiguousarray(vb).view(np.uint32)
    lib().or_merge(_p(a), _p(va), a.size, _p(b), _p(vb), b.size, _p(out), _p(vout), _ks(a))
    return out if vout is None else (out, vout)


def merge_path(a, b, d: int) -> int:
    """# of A elements among the first d outputs of merge(a, b)."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return int(lib().or_merge_path(_p(a), a.size, _p(b), b.size, d, _ks(a)))


def sample_pos(start: int, length: int, S: int, k: int) -> int:
    return int(lib().or_sample_pos(start, length, S, k))


def splitters(keys, start: int, length: int, nbuckets: int, oversample: int):
    """(splitters int64[m], eq uint8[m]) for segment [start, start+length)."""
    k = np.ascontiguousarray(keys)
    spl = np.zeros(max(1, nbuckets), np.int64)
    eq = np.zeros(max(1, nbuckets), np.uint8)
    m = lib().or_splitters(_p(k), start, length, nbuckets, oversample, _ks(k), _p(spl), _p(eq))
    return spl[:m].astype(k.dtype), eq[:m].copy()


def classify(keys, spl, eq) -> np.ndarray:
    """Bucket ids 2i + [x == t_i and eq_i], i = #{t_j < x}."""
    k = np.ascontiguousarray(keys)
    s = np.ascontiguousarray(spl).astype(np.int64)
    e = np.ascontiguousarray(eq).astype(np.uint8)
    bins = np.empty(k.size, np.int32)
    lib().or_classify(_p(k), k.size, _ks(k), _p(s), _p(e), s.size, _p(bins))
    return bins


def stable_partition(bins, nbins: int, keys, vals=None):
    """Stable counting distribution by bucket -> (keys, vals|None, counts)."""
    k = np.ascontiguousarray(keys)
    b = np.ascontiguousarray(bins).astype(np.int32)
    v = None if vals is None else np.ascontiguousarray(vals).view(np.uint32)
    ok = np.empty_like(k)
    ov = np.empty(k.size, np.uint32) if v is not None else None
    counts = np.zeros(nbins, np.int64)
    lib().or_stable_partition(_p(b), k.size, nbins, _p(k), _p(v), _p(ok), _p(ov), _p(counts), _ks(k))
    return ok, ov, counts


def count(keys, v: int):
    """(#{x < v}, #{x <= v}) -- the value at sorted position p satisfies lt <= p < le."""
    k = np.ascontiguousarray(keys)
    le = ctypes.c_int64(0)
    lt = lib().or_count(_p(k), k.size, _ks(k), int(v), ctypes.byref(le))
    return int(lt), int(le.value)


def stable_rank(keys, i: int) -> int:
    """#{j: k_j < k_i} + #{j < i: k_j = k_i}."""
    k = np.ascontiguousarray(keys)
    return int(lib().or_stable_rank(_p(k), k.size, _ks(k), i))
