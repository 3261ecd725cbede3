"""Parity of record keys (-m gpu): n lists of `words`
int32 compared lexicographically -- the paper's "random 16-/64-/256-list"
classes (Table 2) -- sorted by sr_sort_records,
bit-exact against the oracle's plain lexicographic mergesort."""
import numpy as np
import pytest
import torch

import oracle
import paper_1609_04471_b200 as sr
from workloads import gen

pytestmark = pytest.mark.gpu


def _check(r):
    d = torch.from_numpy(r.copy()).cuda()
    sr.sort_records(d)
    torch.cuda.synchronize()
    got, exp = d.cpu().numpy(), oracle.sort_records(r)
    assert np.array_equal(got, exp), f"first mismatching row {int(np.argmax((got != exp).any(axis=1)))}"
    return sr.last_plan()


@pytest.mark.parametrize("words", [1, 2, 3, 16])
@pytest.mark.parametrize("order", ["lrandom", "lprefix", "lequal", "ldup"])
@pytest.mark.parametrize("n", [2, 1000, 8193, 65537])
def test_records_parity(order, words, n):
    _check(gen.make_list(order, n, words, config=60))


@pytest.mark.parametrize("words", [16, 64])
def test_records_paper_lists(words):
    """The paper's random 16-/64-int lists at 100K records (64 / 256 bytes each)."""
    p = _check(gen.make_list("lrandom", 100_000, words, config=61))
    assert p["levels"] == 1  # distinct (w0, w1) prefixes: one round


@pytest.mark.parametrize("order", ["lrandom", "lprefix", "ldup", "lequal"])
def test_records_256_int_lists(order):
    """The paper's random 256-int lists (1024-byte records; Table 2
    row PAPER.md:128-130): 20K records, every list class; lprefix shares 255
    words from {-1, 0, 1}, so the refinement runs deep."""
    _check(gen.make_list(order, 20_000, 256, config=63))


def test_records_deep_prefix_rounds():
    """Prefixes from {-1, 0, 1} over 7 words and a random last word: the
    ternary words take 2-bit fields, so ONE packed round decides (14 + 32 bits)."""
    p = _check(gen.make_list("lprefix", 50_000, 8, config=62))
    assert p["levels"] == 1


def test_records_refinement_rounds():
    """Full-range words with ties: round 0 packs w0, w1 (64 bits) and leaves
    ties; round 1 sorts by (segment id, w2); constant words are skipped."""
    rng = np.random.default_rng(64)
    n = 60_000
    pool = rng.integers(-2**31, 2**31, 8, dtype=np.int64).astype(np.int32)
    r = np.empty((n, 5), np.int32)
    r[:, 0] = pool[rng.integers(0, 4, n)]
    r[:, 1] = pool[4 + rng.integers(0, 4, n)]
    r[:, 2] = 7  # constant
    r[:, 3] = rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    r[:, 4] = rng.integers(-5, 5, n).astype(np.int32)
    p = _check(r)
    assert p["levels"] == 2
    same = np.repeat(rng.integers(-9, 9, (1, 6)).astype(np.int32), 1000, axis=0)
    assert _check(same)["levels"] == 0  # every word constant: nothing to sort
    ext = np.zeros((4000, 3), np.int32)
    ext[:, 0] = np.where(rng.integers(0, 2, 4000) == 1, np.iinfo(np.int32).max, np.iinfo(np.int32).min)
    ext[:, 1] = rng.integers(-2**31, 2**31, 4000, dtype=np.int64).astype(np.int32)
    _check(ext)  # a word spanning the whole int32 range (32-bit field)


def test_records_errors():
    d = torch.zeros((10, 3), dtype=torch.int32, device="cuda")
    lib = sr.lib()
    import ctypes
    assert lib.sr_sort_records(ctypes.c_void_p(d.data_ptr()), 10, 0, None) == 1  # words out of range
    assert lib.sr_sort_records(ctypes.c_void_p(d.data_ptr()), 10, 1025, None) == 1
    assert lib.sr_sort_records(None, 10, 3, None) == 1
    assert lib.sr_sort_records(ctypes.c_void_p(d.data_ptr() + 2), 10, 3, None) == 4  # misaligned
