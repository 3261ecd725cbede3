"""On-device generator (sr_generate, the paper's input
classes PAPER.md:56-87) against the host builders of workloads/gen.py, bit for
bit, for every class, both key widths, sizes with ragged tails."""
import numpy as np
import pytest
import torch

import paper_1609_04471_b200 as sr
from workloads import gen

pytestmark = pytest.mark.gpu

SIZES = [1, 7, 1000, 65_537, 1_000_003]


def _host(order, n, dt, seed, param):
    if order == "random":
        return gen.random_keys(n, dt, seed)
    if order == "sorted":
        return gen.ramp(n, dt)
    if order == "reversed":
        return gen.reversed_ramp(n, dt)
    if order == "swaps":
        return gen.swaps(n, param, dt, seed)
    if order == "few_unique":
        return gen.few_unique(n, param, dt, seed)
    if order == "runs":
        return gen.shuffled_runs(n, param, dt, seed)
    if order == "last":  # gen.last_pct with t = param positions
        a = gen.ramp(n, dt)
        if param:
            a[n - param:] = gen.random_keys(param, dt, seed)
        return a
    if order == "sharp_teeth":
        return gen.sharp_teeth(n, param, dt)
    if order == "equal_teeth":
        return gen.equal_teeth(n, param, dt)
    if order == "even_teeth":
        return gen.even_teeth(n, param, dt)
    if order == "distance":
        return gen.distance(n, param, dt, seed)
    if order == "all_equal":
        return np.full(n, param, dtype=dt)
    if order == "extremes":
        return gen.extremes(n, dt, seed)
    raise KeyError(order)


CASES = [("random", 0), ("sorted", 0), ("reversed", 0), ("swaps", 0), ("swaps", 3), ("swaps", 997),
         ("few_unique", 1), ("few_unique", 10), ("few_unique", 100), ("runs", 1), ("runs", 64), ("runs", 1024),
         ("last", 0), ("last", 1), ("sharp_teeth", 1), ("sharp_teeth", 8), ("equal_teeth", 8), ("even_teeth", 2),
         ("even_teeth", 7), ("distance", 1), ("distance", 256), ("all_equal", 7), ("extremes", 0)]


@pytest.mark.parametrize("dt", [np.int32, np.int64])
@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("order,param", CASES)
def test_generate_matches_host(order, param, n, dt):
    if order in ("runs", "sharp_teeth", "equal_teeth", "even_teeth") and param > n:
        pytest.skip("more sections than keys")
    if order == "last":
        param = min(n, max(param, n // 100))
    if order == "distance" and n > 100_000 and param == 1:
        param = 2
    seed = gen.seed_for(7, gen.ORDERS.get(order, 30), n % 97)
    want = _host(order, n, dt, seed, param)
    t = torch.empty(n, dtype=torch.int32 if dt == np.int32 else torch.int64, device="cuda")
    sr.generate(t, order, seed, param)
    torch.cuda.synchronize()
    got = t.cpu().numpy()
    assert got.dtype == want.dtype and np.array_equal(got, want), (order, param, n, int(np.argmax(got != want)))


def test_generate_bench_inputs():
    """The bench's configs[4] inputs (nearly sorted = n/1000 swaps) at 16M keys."""
    n = 1 << 24
    seed = gen.seed_for(4, 2, 0)
    t = torch.empty(n, dtype=torch.int32, device="cuda")
    sr.generate(t, "swaps", seed, n // 1000)
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy(), gen.swaps(n, n // 1000, np.int32, seed))


def test_generate_errors():
    t = torch.empty(10, dtype=torch.int32, device="cuda")
    with pytest.raises(sr.SrError):
        sr.generate(t, "runs", 1, 0)
    with pytest.raises(sr.SrError):
        sr.generate(t, "few_unique", 1, 0)
    with pytest.raises(TypeError):
        sr.generate(torch.empty(10, dtype=torch.float32, device="cuda"), "random", 1)
