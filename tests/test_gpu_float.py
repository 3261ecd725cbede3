"""Parity of floating-point keys (-m gpu, the paper's
"random double" class): float32 / float64 keys sorted by IEEE 754
totalOrder through sr_sort_keys / sr_sort_pairs / sr_sort_host, bit-exact
against the CPU oracle (whose comparator is written from the totalOrder
definition; the GPU path maps the bit patterns to signed integer order, so the
two share no code).  Sizes span the tile / resident / multi-kernel ranges and
ragged tails."""
import numpy as np
import pytest
import torch

import oracle
import paper_1609_04471_b200 as sr
from workloads import gen

pytestmark = pytest.mark.gpu

TORCH = {np.float32: torch.float32, np.float64: torch.float64}
UINT = {np.float32: np.uint32, np.float64: np.uint64}


def _gpu_sort(k):
    d = torch.from_numpy(k.copy()).cuda()
    sr.sort_keys(d)
    torch.cuda.synchronize()
    return d.cpu().numpy()


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("order", ["fbits", "funiform", "fspecial", "fsorted", "freversed"])
@pytest.mark.parametrize("n", [2, 3, 1000, 8192, 8193, 65537, 300_007])
def test_float_keys_parity(order, dtype, n):
    k = gen.make_float(order, n, dtype, config=40)
    got, exp = _gpu_sort(k), oracle.sort_keys(k)
    u = UINT[dtype]
    assert np.array_equal(got.view(u), exp.view(u)), f"first mismatch at {int(np.argmax(got.view(u) != exp.view(u)))}"


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("order", ["fbits", "funiform"])
def test_float_keys_large(order, dtype):
    n = 2_000_000 if dtype == np.float64 else 4_000_003  # resident range and the multi-kernel path
    k = gen.make_float(order, n, dtype, config=41)
    got, exp = _gpu_sort(k), oracle.sort_keys(k)
    u = UINT[dtype]
    assert np.array_equal(got.view(u), exp.view(u))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [5, 8193, 300_007])
def test_float_pairs_stable_parity(dtype, n):
    k = gen.make_float("fspecial", n, dtype, config=42)
    v = gen.index_payload(n)
    dk, dv = torch.from_numpy(k.copy()).cuda(), torch.from_numpy(v.view(np.int32).copy()).cuda()
    sr.sort_pairs(dk, dv)
    torch.cuda.synchronize()
    ek, ev = oracle.sort_pairs(k, v)
    u = UINT[dtype]
    assert np.array_equal(dk.cpu().numpy().view(u), ek.view(u))
    assert np.array_equal(dv.cpu().numpy().view(np.uint32), ev)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_float_sort_host(dtype):
    k = gen.make_float("fbits", 100_003, dtype, config=43)
    h = k.copy()
    sr.sort_host(h)
    u = UINT[dtype]
    assert np.array_equal(h.view(u), oracle.sort_keys(k).view(u))


def test_float_step_entry_points_reject():
    d = torch.zeros(100, dtype=torch.float32, device="cuda")
    with pytest.raises(sr.SrError):
        sr.tile_sort(d, 64)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [100_003, 3_000_000])  # resident (one launch) and multi-kernel paths
@pytest.mark.parametrize("pairs", [False, True])
def test_float_oom_leaves_keys_untouched(dtype, n, pairs):
    """SR_ERR_OUT_OF_MEMORY from the first workspace reservation (injected
    with SR_OPT_WS_LIMIT) leaves float keys bit-identical (include/sr_sort.h
    "Error behaviour"): the in-place totalOrder map is undone."""
    k = gen.make_float("fbits", n, dtype, config=41)
    d = torch.from_numpy(k.copy()).cuda()
    v = torch.arange(n, dtype=torch.int32, device="cuda")
    sr.set_option(sr.OPT_WS_LIMIT, 4096)
    try:
        with pytest.raises(sr.SrError) as ei:
            sr.sort_pairs(d, v) if pairs else sr.sort_keys(d)
    finally:
        sr.set_option(sr.OPT_WS_LIMIT, 0)
    assert ei.value.status == 5
    torch.cuda.synchronize()
    u = UINT[dtype]
    assert np.array_equal(d.cpu().numpy().view(u), k.view(u))
    assert torch.equal(v, torch.arange(n, dtype=torch.int32, device="cuda"))
    got = d.clone()  # and the library still works afterwards
    sr.sort_keys(got)
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy().view(u), oracle.sort_keys(k).view(u))
