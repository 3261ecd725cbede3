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


def test_records_deep_prefix_rounds():
    """Prefixes from {-1, 0, 1} over 7 words: several refinement rounds."""
    p = _check(gen.make_list("lprefix", 50_000, 8, config=62))
    assert p["levels"] >= 3


def test_records_errors():
    d = torch.zeros((10, 3), dtype=torch.int32, device="cuda")
    lib = sr.lib()
    import ctypes
    assert lib.sr_sort_records(ctypes.c_void_p(d.data_ptr()), 10, 0, None) == 1  # words out of range
    assert lib.sr_sort_records(ctypes.c_void_p(d.data_ptr()), 10, 1025, None) == 1
    assert lib.sr_sort_records(None, 10, 3, None) == 1
    assert lib.sr_sort_records(ctypes.c_void_p(d.data_ptr() + 2), 10, 3, None) == 4  # misaligned
