"""End-to-end parity (-m gpu): the CUDA path (through the C ABI) against the
CPU oracle, element by element, bit-exact, on seeded synthetic inputs.

Every case runs under the automatic route and with the merge and partition
routes forced (SR_OPT_FORCE_ROUTE), because the planner exercises only one
route per input.  Sizes span several tiles and ragged tails (kCap = 8192).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1609_04471_b200 as sr
from workloads import gen

pytestmark = pytest.mark.gpu

SIZES = [0, 1, 2, 3, 31, 33, 1000, 8191, 8192, 8193, 16383, 16385, 100_003]
ORDERS = ["random", "reversed", "nearly", "few_unique", "sorted", "all_equal", "organ_pipe", "extremes",
          "runs1024", "last1pct", "sharp_teeth", "even_teeth", "equal_teeth", "distance256", "few100", "swaps_1e1"]
ROUTES = {"auto": 0, "merge": sr.ROUTE_MERGE, "partition": sr.ROUTE_PARTITION}


@pytest.fixture(autouse=True)
def _reset_route():
    yield
    sr.set_option(sr.OPT_FORCE_ROUTE, 0)


def run_case(order, n, dtype, pairs, route, config=7, instance=0):
    k = gen.make(order, n, dtype, config=config, instance=instance)
    sr.set_option(sr.OPT_FORCE_ROUTE, ROUTES[route])
    dk = torch.from_numpy(k.copy()).cuda()
    if pairs:
        v = gen.index_payload(n)
        dv = torch.from_numpy(v.view(np.int32).copy()).cuda()
        sr.sort_pairs(dk, dv)
        torch.cuda.synchronize()
        ek, ev = oracle.sort_pairs(k, v)
        gk, gv = dk.cpu().numpy(), dv.cpu().numpy().view(np.uint32)
        assert np.array_equal(gk, ek), f"keys differ: {order} n={n} {route}"
        assert np.array_equal(gv, ev), f"payload order differs: {order} n={n} {route}"
    else:
        sr.sort_keys(dk)
        torch.cuda.synchronize()
        assert np.array_equal(dk.cpu().numpy(), oracle.sort_keys(k)), f"keys differ: {order} n={n} {route}"
    return sr.last_plan()


@pytest.mark.parametrize("route", list(ROUTES))
@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("order", ORDERS)
def test_parity_small(order, dtype, pairs, route):
    for n in SIZES:
        run_case(order, n, dtype, pairs, route)


@pytest.mark.parametrize("route", list(ROUTES))
@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("order", ["random", "reversed", "nearly", "few_unique"])
def test_parity_c2_size(order, pairs, route):
    """configs[1] size: n = 2,000,000 int32, the four orders."""
    run_case(order, 2_000_000, np.int32, pairs, route, config=1)


@pytest.mark.parametrize("order", ["random", "nearly", "few_unique", "runs1024", "last1pct", "alternating",
                                   "swaps_1e4", "swaps_1e3", "sharp_teeth"])
def test_parity_multilevel(order):
    """~4.2M keys: enough for a second partition level on part of the buckets."""
    run_case(order, 4_200_007, np.int32, False, "auto", config=2)


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_parity_int64_and_pairs_multilevel(dtype):
    run_case("random", 3_000_001, dtype, True, "partition", config=3)
    run_case("few100", 3_000_001, dtype, True, "auto", config=3)


def test_bsd_adversarial_and_worked_example():
    for m in [1, 2, 3, 100, 5000, 70000]:
        k = gen.bsd_adversarial(m, np.int32)
        for route in ROUTES:
            sr.set_option(sr.OPT_FORCE_ROUTE, ROUTES[route])
            dk = torch.from_numpy(k.copy()).cuda()
            sr.sort_keys(dk)
            assert np.array_equal(dk.cpu().numpy(), np.sort(k))
    w = np.array([1, 15, 18, 19, 20, 16, 11, 10, 9, 8, 7, 6, 5, 4, 3, 2], np.int32)
    dk = torch.from_numpy(w.copy()).cuda()
    sr.set_option(sr.OPT_FORCE_ROUTE, 0)
    sr.sort_keys(dk)
    assert dk.cpu().tolist() == [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 15, 16, 18, 19, 20]
    assert sr.last_plan()["descents"] == 11


def test_route_selection():
    """H3: the planner's exits and routes on the classic orders."""
    n = 2_000_000
    assert run_case("sorted", n, np.int32, False, "auto")["route_name"] == "sorted"
    p = run_case("reversed", n, np.int32, False, "auto")
    assert p["route_name"] == "reversed" and p["descents"] == n - 1
    p = run_case("few_unique", n, np.int32, False, "auto")
    assert p["route_name"] == "partition" and p["equal_keys"] == n
    assert run_case("random", n, np.int32, False, "auto")["route_name"] == "partition"
    p = run_case("all_equal", n, np.int32, True, "auto")
    assert p["route_name"] == "sorted"
    # a strictly decreasing array with pairs is reversed; with equal neighbours it is not
    p = run_case("reversed", n, np.int32, True, "auto")
    assert p["route_name"] == "reversed"


def test_sorted_input_is_not_written():
    """is_sorted exit: sorted input is read once and never written."""
    n = 1 << 20
    k = torch.arange(n, dtype=torch.int32, device="cuda")
    sr.sort_keys(k)
    p = sr.last_plan()
    assert p["route_name"] == "sorted" and p["host_syncs"] == 1
    assert p["bytes_planned"] < 2 * n * 4


def test_host_api_roundtrip():
    n = 1_000_003
    k = gen.make("random", n, np.int32, config=11)
    v = gen.index_payload(n)
    hk, hv = k.copy(), v.copy()
    sr.sort_host(hk, hv)
    ek, ev = oracle.sort_pairs(k, v)
    assert np.array_equal(hk, ek) and np.array_equal(hv, ev)
    hk = k.astype(np.int64)
    sr.sort_host(hk)
    assert np.array_equal(hk, oracle.sort_keys(k.astype(np.int64)))


@pytest.mark.parametrize("pinned", [True, False])
def test_host_batch_keys(pinned):
    """sr_sort_host_batch: instances of mixed size and order (resident, tile,
    multi-kernel, empty, single) pipelined over the ring of four buffers, more
    instances than ring slots; each bit-exact with the oracle."""
    specs = [("random", 2_000_000), ("reversed", 2_000_000), ("nearly", 2_000_000), ("few_unique", 2_000_000),
             ("random", 0), ("sorted", 1), ("random", 5000), ("distance256", 300_007), ("random", 3_000_001),
             ("runs1024", 100_003), ("random", 2)]
    src = [gen.make(o, n, np.int32, config=13, instance=i) for i, (o, n) in enumerate(specs)]
    if pinned:
        hold = [torch.from_numpy(k.copy()).pin_memory() for k in src]
        bufs = [h.numpy() for h in hold]
    else:
        bufs = [k.copy() for k in src]
    stream = torch.cuda.Stream()
    sr.sort_host_batch(bufs, stream=stream.cuda_stream)
    for k, b, (o, n) in zip(src, bufs, specs):
        assert np.array_equal(b, oracle.sort_keys(k)), (o, n)


def test_host_batch_pairs_and_int64():
    ns = [700_001, 8193, 1_500_000, 33, 2_000_000, 100]
    ks = [gen.make("few100" if i % 2 else "random", n, np.int64, config=14, instance=i) for i, n in enumerate(ns)]
    vs = [gen.index_payload(n) for n in ns]
    hk, hv = [k.copy() for k in ks], [v.copy() for v in vs]
    hv[3] = None  # a keys-only instance inside a pair batch
    sr.sort_host_batch(hk, hv)
    for i, (k, v) in enumerate(zip(ks, vs)):
        if hv[i] is None:
            assert np.array_equal(hk[i], oracle.sort_keys(k))
        else:
            ek, ev = oracle.sort_pairs(k, v)
            assert np.array_equal(hk[i], ek) and np.array_equal(hv[i], ev), i


def test_host_batch_errors():
    k = gen.make("random", 1000, np.int32, config=15)
    assert sr.sort_host_batch([]) == []
    with pytest.raises(TypeError):
        sr.sort_host_batch([k.copy(), k.astype(np.int64)])
    import ctypes
    L = sr.lib()
    ns = (ctypes.c_int64 * 1)(-1)
    kp = (ctypes.c_void_p * 1)(k.ctypes.data)
    assert L.sr_sort_host_batch(kp, None, ns, 1, sr.SR_INT32, None) == 1   # SR_ERR_INVALID_ARGUMENT
    ns[0] = 1000
    assert L.sr_sort_host_batch(kp, None, ns, 1, 99, None) == 2            # SR_ERR_UNSUPPORTED_DTYPE
    assert L.sr_sort_host_batch(None, None, ns, 1, sr.SR_INT32, None) == 1
    assert L.sr_sort_host_batch(kp, None, ns, -1, sr.SR_INT32, None) == 1
    kp[0] = None
    assert L.sr_sort_host_batch(kp, None, ns, 1, sr.SR_INT32, None) == 1


def test_streams_and_concurrency():
    """Work is enqueued on the caller's stream; two streams sort independently."""
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    a = gen.make("random", 500_000, np.int32, config=12)
    b = gen.make("few_unique", 700_001, np.int64, config=12)
    with torch.cuda.stream(s1):
        da = torch.from_numpy(a.copy()).cuda(non_blocking=False)
        sr.sort_keys(da)
    with torch.cuda.stream(s2):
        db = torch.from_numpy(b.copy()).cuda(non_blocking=False)
        sr.sort_keys(db)
    torch.cuda.synchronize()
    assert np.array_equal(da.cpu().numpy(), oracle.sort_keys(a))
    assert np.array_equal(db.cpu().numpy(), oracle.sort_keys(b))


def test_error_paths_leave_buffers_untouched():
    k = torch.arange(1000, 0, -1, dtype=torch.int32, device="cuda")
    before = k.clone()
    L = sr.lib()
    import ctypes
    # host pointer
    h = np.arange(100, dtype=np.int32)
    assert L.sr_sort_keys(h.ctypes.data_as(ctypes.c_void_p), 100, 0, None) == 1
    # overlapping keys / vals
    assert L.sr_sort_pairs(ctypes.c_void_p(k.data_ptr()), ctypes.c_void_p(k.data_ptr() + 8), 500, 0, None) == 1
    # misaligned
    assert L.sr_sort_keys(ctypes.c_void_p(k.data_ptr() + 2), 100, 0, None) == 4
    assert L.sr_sort_keys(ctypes.c_void_p(k.data_ptr()), 100, 9, None) == 2
    torch.cuda.synchronize()
    assert torch.equal(k, before)
