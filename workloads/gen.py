"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds NO sorting arithmetic: it only builds input arrays. It is
shared by the oracle tests, the GPU parity tests and bench.py (the one thing
the oracle and the CUDA path may share).

PRNG: splitmix64 used as a counter-based generator -- draw i of stream `seed`
is mix64(seed + (i+1)*GAMMA).  SPEC.md:147 allows "any seedable generator with
>= 64-bit state and published algorithm"; the paper names none.

Orders (§2, lines 56-87; BASELINE.json configs):
  random        uniform int32/int64 over the full range       (G1)
  reversed      a[i] = n-1-i                                   (k-sharp teeth k=1)
  swaps(k)      ramp 0..n-1 then k random position swaps      (k-exchange)
  few_unique(m) m distinct uniform values, a[i] = v[U[0,m)]    (k-limited analogue)
  runs(L)       ramp cut into blocks of L, blocks shuffled    (BASELINE configs[2])
  last_pct(p)   ramp, last p% of positions uniform random     (BASELINE configs[2])
  alternating(L) sections of L sorted random keys, odd sections descending (configs[2], primary)
  sharp_teeth(k) ramp, 1-based odd sections reversed
  even_teeth(k)  k sections each ramp 1..n/k, 1-based odd reversed
  equal_teeth(k) k sections each ramp 1..n/k
  distance(k)   ramp, blocks of k+1 shuffled
  organ_pipe    even_teeth(2)
  bsd(m)        reversed 1..m, m+1, reversed m+2..2m+1
  all_equal     constant                                       (k=0)
  extremes      INT_MIN / INT_MAX / 0 / -1 mix
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK32 = np.uint64(0xFFFFFFFF)


def seed_for(config: int, order: int, instance: int) -> int:
    """Per-instance seed (SURVEY.md §8(d) "Per-instance seed")."""
    return (0x5EED000000000000 ^ (config << 40) ^ (order << 32) ^ instance) & (2**64 - 1)


def draws(seed: int, count: int, start: int = 0) -> np.ndarray:
    """uint64 draws start..start+count-1 of the counter-based splitmix64 stream."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_below(d: np.ndarray, m: int) -> np.ndarray:
    """U[0,m) = (draw * m) >> 64 (multiply-high), for 1 <= m < 2**32."""
    assert 1 <= m < 2**32
    mm = np.uint64(m)
    with np.errstate(over="ignore"):
        dh = d >> np.uint64(32)
        dl = d & _MASK32
        t = dh * mm + ((dl * mm) >> np.uint64(32))
    return (t >> np.uint64(32)).astype(np.int64)


def _u_scalar(seed: int, idx: int, m: int) -> int:
    return int(uniform_below(draws(seed, 1, idx), m)[0])


def random_keys(n: int, dtype, seed: int) -> np.ndarray:
    d = draws(seed, n)
    if np.dtype(dtype) == np.int32:
        return (d >> np.uint64(32)).astype(np.uint32).view(np.int32)
    return d.view(np.int64).copy()


def ramp(n: int, dtype) -> np.ndarray:
    return np.arange(n, dtype=dtype)


def reversed_ramp(n: int, dtype) -> np.ndarray:
    return np.arange(n - 1, -1, -1, dtype=dtype)


def swaps(n: int, k: int, dtype, seed: int) -> np.ndarray:
    """Ramp with k random position swaps applied in draw order (p then q)."""
    a = ramp(n, dtype)
    if n == 0 or k == 0:
        return a
    u = uniform_below(draws(seed, 2 * k), n)
    p = u[0::2].tolist()
    q = u[1::2].tolist()
    for x, y in zip(p, q):
        a[x], a[y] = a[y], a[x]
    return a


def few_unique(n: int, m: int, dtype, seed: int) -> np.ndarray:
    """m distinct uniform values (repeats rejected), a[i] = v[U[0,m)]."""
    vals: list[int] = []
    seen = set()
    idx = 0
    bits32 = np.dtype(dtype) == np.int32
    while len(vals) < m:
        d = int(draws(seed, 1, idx)[0])
        idx += 1
        v = (d >> 32) if bits32 else d
        v = v - (1 << 32) if bits32 and v >= (1 << 31) else v
        if not bits32 and v >= (1 << 63):
            v -= 1 << 64
        if v not in seen:
            seen.add(v)
            vals.append(v)
    table = np.array(vals, dtype=dtype)
    sel = uniform_below(draws(seed ^ 0xF00D, n), m)
    return table[sel]


def shuffled_runs(n: int, L: int, dtype, seed: int) -> np.ndarray:
    """Ramp cut into blocks of L (last may be short), block order Fisher-Yates shuffled."""
    nb = (n + L - 1) // L
    order = list(range(nb))
    if nb > 1:
        d = draws(seed, nb)
        for i in range(nb - 1, 0, -1):
            j = int(uniform_below(d[nb - 1 - i: nb - i], i + 1)[0])
            order[i], order[j] = order[j], order[i]
    a = ramp(n, dtype)
    parts = [a[b * L: min(n, (b + 1) * L)] for b in order]
    return np.concatenate(parts) if parts else a


def last_pct(n: int, pct: float, dtype, seed: int) -> np.ndarray:
    a = ramp(n, dtype)
    t = int(n * pct / 100.0)
    if t:
        a[n - t:] = random_keys(t, dtype, seed)
    return a


def alternating(n: int, L: int, dtype, seed: int) -> np.ndarray:
    """Sections of L uniform keys; section j sorted ascending if j even, descending if odd."""
    a = random_keys(n, dtype, seed)
    for j, s in enumerate(range(0, n, L)):
        sec = np.sort(a[s: s + L], kind="stable")  # input construction, not the method
        a[s: s + L] = sec if j % 2 == 0 else sec[::-1]
    return a


def sharp_teeth(n: int, k: int, dtype) -> np.ndarray:
    """ramp 0..n-1, k equal sections, 1-based odd sections reversed."""
    a = ramp(n, dtype)
    bounds = [(j * n) // k for j in range(k + 1)]
    for j in range(k):
        if j % 2 == 0:  # 1-based odd
            a[bounds[j]: bounds[j + 1]] = a[bounds[j]: bounds[j + 1]][::-1].copy()
    return a


def equal_teeth(n: int, k: int, dtype) -> np.ndarray:
    """k sections, each a sorted ramp 1..n/k."""
    bounds = [(j * n) // k for j in range(k + 1)]
    parts = [np.arange(1, bounds[j + 1] - bounds[j] + 1, dtype=dtype) for j in range(k)]
    return np.concatenate(parts) if parts else np.zeros(0, dtype)


def even_teeth(n: int, k: int, dtype) -> np.ndarray:
    """equal teeth with 1-based odd sections reversed."""
    bounds = [(j * n) // k for j in range(k + 1)]
    a = equal_teeth(n, k, dtype)
    for j in range(k):
        if j % 2 == 0:
            a[bounds[j]: bounds[j + 1]] = a[bounds[j]: bounds[j + 1]][::-1].copy()
    return a


def distance(n: int, k: int, dtype, seed: int) -> np.ndarray:
    """ramp, blocks of k+1 each Fisher-Yates shuffled."""
    a = ramp(n, dtype)
    B = k + 1
    d = draws(seed, n)
    di = 0
    for s in range(0, n, B):
        e = min(n, s + B)
        for i in range(e - s - 1, 0, -1):
            j = int(uniform_below(d[di: di + 1], i + 1)[0])
            di += 1
            a[s + i], a[s + j] = a[s + j], a[s + i]
    return a


def bsd_adversarial(m: int, dtype) -> np.ndarray:
    """reversed 1..m, then m+1, then reversed m+2..2m+1."""
    return np.concatenate([np.arange(m, 0, -1), [m + 1], np.arange(2 * m + 1, m + 1, -1)]).astype(dtype)


def extremes(n: int, dtype, seed: int) -> np.ndarray:
    info = np.iinfo(dtype)
    table = np.array([info.min, info.max, 0, -1, 1, info.min + 1, info.max - 1], dtype=dtype)
    return table[uniform_below(draws(seed, n), len(table))]


# Named orders used by tests and bench (order id -> builder).  Order ids feed seed_for().
ORDERS = {
    "random": 0, "reversed": 1, "nearly": 2, "few_unique": 3,
    "swaps_1e4": 4, "swaps_1e3": 5, "swaps_1e2": 6, "swaps_1e1": 7,
    "runs1024": 8, "last1pct": 9, "alternating": 10, "sharp_teeth": 11,
    "sorted": 12, "all_equal": 13, "organ_pipe": 14, "extremes": 15,
    "even_teeth": 16, "equal_teeth": 17, "distance256": 18, "few100": 19,
    "swaps_1e3b": 20,
}


def make(order: str, n: int, dtype=np.int32, config: int = 0, instance: int = 0) -> np.ndarray:
    """Build one input of a named order (see ORDERS)."""
    dtype = np.dtype(dtype)
    s = seed_for(config, ORDERS[order], instance)
    if order == "random":
        return random_keys(n, dtype, s)
    if order == "reversed":
        return reversed_ramp(n, dtype)
    if order == "sorted":
        return ramp(n, dtype)
    if order == "nearly":  # configs[1](c): n/100 swaps
        return swaps(n, n // 100, dtype, s)
    if order == "few_unique":
        return few_unique(n, 10, dtype, s)
    if order == "few100":
        return few_unique(n, 100, dtype, s)
    if order.startswith("swaps_1e"):
        e = int(order[len("swaps_1e"):].rstrip("b"))
        return swaps(n, n // (10 ** e), dtype, s)
    if order == "runs1024":
        return shuffled_runs(n, 1024, dtype, s)
    if order == "last1pct":
        return last_pct(n, 1.0, dtype, s)
    if order == "alternating":
        return alternating(n, 65536, dtype, s)
    if order == "sharp_teeth":
        return sharp_teeth(n, max(1, n // 65536), dtype)
    if order == "all_equal":
        return np.full(n, 7, dtype=dtype)
    if order == "organ_pipe":
        return even_teeth(n, 2, dtype)
    if order == "even_teeth":
        return even_teeth(n, 8, dtype)
    if order == "equal_teeth":
        return equal_teeth(n, 8, dtype)
    if order == "distance256":
        return distance(n, 256, dtype, s)
    if order == "extremes":
        return extremes(n, dtype, s)
    raise KeyError(order)


# ---- floating-point keys (the paper's "random double"
# class).  Orders: "fbits" = uniformly random bit patterns (every
# class: normals, subnormals, +-0, +-inf, NaNs with payloads, both signs);
# "funiform" = uniform [0, 1) from the top 53 (24) bits of a draw (the paper's
# random doubles); "fspecial" = a mix drawn from the special values and a few
# ordinary numbers, with many ties; "fsorted" / "freversed" = ramps.
FLOAT_ORDERS = {"fbits": 32, "funiform": 33, "fspecial": 34, "fsorted": 35, "freversed": 36}


def make_float(order: str, n: int, dtype=np.float64, config: int = 0, instance: int = 0) -> np.ndarray:
    dtype = np.dtype(dtype)
    assert dtype in (np.float32, np.float64)
    s = seed_for(config, FLOAT_ORDERS[order], instance)
    d = draws(s, n)
    if order == "fbits":
        return (d >> np.uint64(32)).astype(np.uint32).view(np.float32) if dtype == np.float32 else d.view(np.float64)
    if order == "funiform":
        if dtype == np.float64:
            return (d >> np.uint64(11)).astype(np.float64) * 2.0**-53
        return ((d >> np.uint64(40)).astype(np.float64) * 2.0**-24).astype(np.float32)
    if order == "fspecial":
        it = np.uint32 if dtype == np.float32 else np.uint64
        if dtype == np.float32:
            bits = [0x7fc00000, 0x7fc00001, 0x7f800001, 0xffc00000, 0xffc00001, 0xff800001, 0x7f800000, 0xff800000,
                    0x00000000, 0x80000000, 0x00000001, 0x80000001, 0x3f800000, 0xbf800000, 0x7f7fffff, 0xff7fffff]
        else:
            bits = [0x7ff8000000000000, 0x7ff8000000000001, 0x7ff0000000000001, 0xfff8000000000000,
                    0xfff8000000000001, 0xfff0000000000001, 0x7ff0000000000000, 0xfff0000000000000,
                    0x0, 0x8000000000000000, 0x1, 0x8000000000000001, 0x3ff0000000000000, 0xbff0000000000000,
                    0x7fefffffffffffff, 0xffefffffffffffff]
        table = np.array(bits, dtype=it).view(dtype)
        return table[uniform_below(d, len(table))]
    if order == "fsorted":
        return np.arange(n, dtype=dtype) * dtype.type(0.5) - dtype.type(n // 4)
    if order == "freversed":
        return (np.arange(n, dtype=dtype) * dtype.type(0.5) - dtype.type(n // 4))[::-1].copy()
    raise KeyError(order)


# ---- record keys: n lists of `words` int32, the
# paper's "random 16-/64-/256-list" classes.  "lrandom" = uniform
# words; "lprefix" = the first words drawn from `vals` values (long shared
# prefixes, many refinement rounds); "lequal" = every record identical except
# a few; "ldup" = random records, each repeated ~4 times.
LIST_ORDERS = {"lrandom": 48, "lprefix": 49, "lequal": 50, "ldup": 51}


def make_list(order: str, n: int, words: int, config: int = 0, instance: int = 0, vals: int = 3) -> np.ndarray:
    s = seed_for(config, LIST_ORDERS[order], instance)
    d = draws(s, n * words)
    r = (d >> np.uint64(32)).astype(np.uint32).view(np.int32).reshape(n, words).copy()
    if order == "lprefix":
        few = uniform_below(draws(s ^ 1, n * words), vals).reshape(n, words).astype(np.int32) - 1
        keep = max(1, words - 1)  # all but the last word from {-1, 0, 1}
        r[:, :keep] = few[:, :keep]
    elif order == "lequal":
        base = r[0].copy()
        r[:] = base
        k = max(1, n // 100)
        pos = uniform_below(draws(s ^ 2, k), n)
        r[pos, -1] = (draws(s ^ 3, k) >> np.uint64(33)).astype(np.int32)
    elif order == "ldup":
        m = max(1, n // 4)
        r = r[uniform_below(draws(s ^ 4, n), m)].copy()
    elif order != "lrandom":
        raise KeyError(order)
    return r


def index_payload(n: int) -> np.ndarray:
    """configs[3]: payload = original index (int32, stored as 4-byte opaque)."""
    return np.arange(n, dtype=np.uint32)
