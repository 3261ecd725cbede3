"""Parity of the outlier route (-m gpu): nearly-sorted keys (k-exchange,
PAPER.md:85) sorted by extracting the endpoints of every descent, sorting
them and merging them back (outlier.cuh), bit-exact against the CPU oracle.
Forcing the route on inputs that are not nearly sorted exercises the second
round and the fallback to the partition."""
import numpy as np
import pytest
import torch

import oracle
import paper_1609_04471_b200 as sr
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _reset():
    yield
    sr.set_option(sr.OPT_FORCE_ROUTE, 0)
    sr.set_option(sr.OPT_OUTLIER_ROUTE, 1)
    sr.set_option(sr.OPT_RESIDENT, 1)


def check(k):
    d = torch.from_numpy(k.copy()).cuda()
    sr.sort_keys(d)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), oracle.sort_keys(k)), f"n={k.size}"
    return sr.last_plan()


def swaps(n, k, dtype, seed):
    return gen.swaps(n, k, dtype, seed)


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("n", [8193, 100_003, 2_000_000, 5_000_011])
def test_outlier_auto_on_exchanges(n, dtype):
    for k in [1, n // 10000, n // 1000, n // 100]:
        if k < 1:
            continue
        p = check(swaps(n, k, dtype, 1000 + k))
        if k <= max(1, n // 10000) or (n > 1 << 22 and k <= n // 1000):  # isolated exchanges: outlier route
            assert p["route_name"] == "outlier", p


@pytest.mark.parametrize("resident", [0, 1])
@pytest.mark.parametrize("order", ["random", "runs1024", "few_unique", "nearly", "sharp_teeth", "organ_pipe",
                                   "distance256", "swaps_1e1", "last1pct", "extremes"])
def test_outlier_forced(order, resident):
    """Forced on every order: either one or two rounds leave a sorted
    remainder, or the partition takes over from the permuted keys."""
    sr.set_option(sr.OPT_RESIDENT, resident)
    sr.set_option(sr.OPT_FORCE_ROUTE, sr.ROUTE_OUTLIER)
    for n in [8193, 65537, 1_000_003]:
        k = gen.make(order, n, np.int32, config=13)
        p = check(k)
        if p["descents"] > 0 and p["route_name"] not in ("reversed",):
            assert p["route_name"] in ("outlier", "partition"), p


def test_outlier_disabled_and_pairs():
    k = swaps(1_000_000, 1000, np.int32, 77)
    sr.set_option(sr.OPT_OUTLIER_ROUTE, 0)
    assert check(k)["route_name"] != "outlier"
    sr.set_option(sr.OPT_OUTLIER_ROUTE, 1)
    # pairs never take the outlier route (stability across the merge is not defined for it)
    v = gen.index_payload(k.size)
    dk, dv = torch.from_numpy(k.copy()).cuda(), torch.from_numpy(v.view(np.int32).copy()).cuda()
    sr.set_option(sr.OPT_FORCE_ROUTE, sr.ROUTE_OUTLIER)
    sr.sort_pairs(dk, dv)
    torch.cuda.synchronize()
    ek, ev = oracle.sort_pairs(k, v)
    assert np.array_equal(dk.cpu().numpy(), ek) and np.array_equal(dv.cpu().numpy().view(np.uint32), ev)
    assert sr.last_plan()["route_name"] != "outlier"


def test_outlier_adjacent_and_overlapping_exchanges():
    """Exchanges at distance 1-3 and chains of exchanges sharing positions."""
    n = 300_000
    rng = np.random.default_rng(5)
    for trial in range(6):
        a = np.arange(n, dtype=np.int32)
        for _ in range(200):
            p = int(rng.integers(0, n - 4))
            q = p + int(rng.integers(1, 4)) if trial % 2 == 0 else int(rng.integers(0, n))
            a[p], a[q] = a[q], a[p]
        check(a)
