"""Parity of the resident path (-m gpu): keys-only sorts of 8192 < n <= 2^22
run as ONE cooperative launch (resident.cuh), checked bit-exact against the
CPU oracle, with the multi-kernel path as a second witness.

The in-kernel finishing caps are lowered through SR_OPT_RESIDENT_CAP so that
the CTA-finished buckets and the hand-off of oversized buckets to the host's
next partition level (Appendix B recursion) are exercised
on ordinary inputs.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1609_04471_b200 as sr
from workloads import gen

pytestmark = pytest.mark.gpu

ORDERS = ["random", "reversed", "nearly", "few_unique", "sorted", "all_equal", "organ_pipe", "extremes",
          "runs1024", "last1pct", "sharp_teeth", "even_teeth", "equal_teeth", "distance256", "few100", "swaps_1e1"]
SIZES = [8193, 12345, 65537, 300_007]
RES_MAX = 1 << 22


@pytest.fixture(autouse=True)
def _reset():
    yield
    sr.set_option(sr.OPT_RESIDENT, 1)
    sr.set_option(sr.OPT_RESIDENT_CAP, 16384)
    sr.set_option(sr.OPT_FORCE_ROUTE, 0)
    sr.set_option(sr.OPT_OUTLIER_ROUTE, 1)


def check(k, expect=None):
    d = torch.from_numpy(k.copy()).cuda()
    sr.sort_keys(d)
    torch.cuda.synchronize()
    e = oracle.sort_keys(k) if expect is None else expect
    got = d.cpu().numpy()
    assert np.array_equal(got, e), f"n={k.size}: first mismatch at {int(np.argmax(got != e))}"
    return sr.last_plan()


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("order", ORDERS)
def test_resident_parity(order, dtype):
    for n in SIZES:
        k = gen.make(order, n, dtype, config=8)
        p = check(k)
        one = p["route_name"] in ("sorted", "reversed") or (
            p["route_name"] == "partition" and p["long_runs"] == 0)
        if one:
            assert p["launches"] == 1, p  # the whole sort was the one cooperative launch


@pytest.mark.parametrize("order", ["random", "nearly", "few_unique", "few100", "organ_pipe", "reversed"])
def test_resident_c2_and_limits(order):
    for n in [1_000_000, 2_000_000, RES_MAX, RES_MAX + 1]:
        k = gen.make(order, n, np.int32, config=1)
        p = check(k)
        if n > RES_MAX:
            assert p["launches"] > 1  # beyond the resident limit: multi-kernel path


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_resident_reversal_vector_and_scalar(dtype):
    """REVERSED route in the one launch: 16-byte vector
    swaps when the keys are 16-byte aligned and n is a whole number of vectors
    (even and odd vector counts: the middle vector reverses in place), the
    scalar loop otherwise (ragged n, or a base pointer off the 16-byte grid)."""
    v = 16 // np.dtype(dtype).itemsize
    for n in [8192 + v, 8192 + 2 * v, 8192 + 3 * v, 8193 + v, 100_000, 100_000 + v, 1_000_003, 2_000_000, 2_000_000 + v]:
        for off in (0, 1):
            k = gen.make("reversed", n, dtype, config=1)
            buf = torch.empty(n + off, dtype=torch.int32 if dtype == np.int32 else torch.int64, device="cuda")
            d = buf[off:]
            d.copy_(torch.from_numpy(k))
            sr.sort_keys(d)
            torch.cuda.synchronize()
            p = sr.last_plan()
            assert p["route_name"] == "reversed" and p["launches"] == 1, (n, off, p)
            assert np.array_equal(d.cpu().numpy(), oracle.sort_keys(k)), (n, off)


@pytest.mark.parametrize("cap", [1, 37, 300, 1024, 2000])
@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_resident_lowered_caps(cap, dtype):
    """Buckets above the cap leave the kernel in the workspace and finish in the
    host-driven next level; buckets in (min(cap, 1024), cap] are CTA-finished."""
    sr.set_option(sr.OPT_RESIDENT_CAP, cap)
    for order in ["random", "few100", "nearly", "organ_pipe"]:
        for n in [9000, 200_003]:
            k = gen.make(order, n, dtype, config=9)
            p = check(k)
            if order == "random" and cap <= 300:
                assert p["levels"] >= 2, p


def test_resident_matches_multikernel():
    # the outlier route's threshold differs by design between the two paths
    sr.set_option(sr.OPT_OUTLIER_ROUTE, 0)
    for order in ORDERS:
        k = gen.make(order, 1 << 20, np.int32, config=10)
        sr.set_option(sr.OPT_RESIDENT, 0)
        a = torch.from_numpy(k.copy()).cuda()
        sr.sort_keys(a)
        pa = sr.last_plan()
        sr.set_option(sr.OPT_RESIDENT, 1)
        b = torch.from_numpy(k.copy()).cuda()
        sr.sort_keys(b)
        pb = sr.last_plan()
        torch.cuda.synchronize()
        assert torch.equal(a, b), order
        assert pa["route_name"] == pb["route_name"], (order, pa, pb)
        assert pa["descents"] == pb["descents"] and pa["long_runs"] == pb["long_runs"], order


def test_resident_forced_routes():
    for route in [sr.ROUTE_MERGE, sr.ROUTE_PARTITION]:
        sr.set_option(sr.OPT_FORCE_ROUTE, route)
        for order in ["random", "reversed", "runs1024", "few_unique"]:
            k = gen.make(order, 500_000, np.int32, config=11)
            p = check(k)
            if order != "reversed" or route == sr.ROUTE_MERGE:
                assert p["route"] == route or p["route_name"] == "sorted", (order, p)


def test_resident_stream_and_repeat():
    """Back-to-back calls on a side stream (the workspace is stream-ordered)."""
    s = torch.cuda.Stream()
    ks = [gen.make("random", 1 << 20, np.int32, config=12, instance=i) for i in range(4)]
    ds = [torch.from_numpy(k.copy()).cuda() for k in ks]
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        for d in ds:
            sr.sort_keys(d)
    s.synchronize()
    for k, d in zip(ks, ds):
        assert np.array_equal(d.cpu().numpy(), oracle.sort_keys(k))


def test_resident_host_threads_concurrent():
    """Resident sorts from several host threads at once, each on its own stream:
    every thread has its own completion record and arrival counters (and the
    GPU may run only one cooperative launch at a time: they serialise, never
    interleave their barriers)."""
    import threading
    ks = [gen.make(o, 700_001, np.int32, config=13, instance=i)
          for i, o in enumerate(["random", "reversed", "few_unique", "sorted", "nearly", "organ_pipe"])]
    outs = [None] * len(ks)
    errs = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(3):
                    d = torch.from_numpy(ks[i].copy()).cuda()
                    sr.sort_keys(d)
                s.synchronize()
                outs[i] = d.cpu().numpy()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(ks))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for k, o in zip(ks, outs):
        assert np.array_equal(o, oracle.sort_keys(k))


def test_resident_many_calls_counters():
    """Hundreds of consecutive resident calls: the persistent arrival counters
    advance by a fixed amount per launch and never desynchronise."""
    k = gen.make("random", 20_000, np.int32, config=14)
    e = oracle.sort_keys(k)
    d = torch.empty(k.size, dtype=torch.int32, device="cuda")
    src = torch.from_numpy(k).cuda()
    for _ in range(300):
        d.copy_(src)
        sr.sort_keys(d)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), e)
    assert sr.last_plan()["launches"] == 1


@pytest.mark.parametrize("dtype,limit", [(np.int32, 2 * 144 * 8192), (np.int64, 2 * 144 * 8192)])
def test_resident_size_limits(dtype, limit):
    """At the resident limit (every tile-holding CTA full) the sort is one launch;
    one key more goes to the multi-kernel path; both bit-exact."""
    for n in (limit, limit + 1):
        k = gen.make("random", n, dtype, config=15)
        p = check(k)
        if n == limit:
            assert p["launches"] == 1, p
        else:
            assert p["launches"] > 1, p


@pytest.mark.parametrize("n", [8193, 9000, 20_000, 70_001])
def test_resident_few_tiles(n):
    """Small resident sizes: fewer tiles than CTAs (most CTAs scan nothing)."""
    for order in ["random", "reversed", "sorted", "few_unique", "organ_pipe"]:
        check(gen.make(order, n, np.int32, config=16))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_two_devices_same_thread():
    """One host thread sorting on two devices alternately: the resident path's
    per-thread state (arena, arrival counter, completion record, graphs, the
    shared-memory attribute) is kept per device, and the call runs on the
    device that owns the keys even when another device is current."""
    n = 1_000_000
    k = gen.make("random", n, np.int32, config=1)
    exp = oracle.sort_keys(k)
    torch.cuda.set_device(0)
    for rep in range(3):
        for d in (0, 1):
            t = torch.from_numpy(k.copy()).to(f"cuda:{d}")
            sr.sort_keys(t)  # device 0 stays current; keys on device d
            torch.cuda.synchronize(d)
            assert np.array_equal(t.cpu().numpy(), exp), (rep, d)
            assert sr.last_plan()["route_name"] == "partition"
