"""Parity of the fused second partition level (k_bucket_sort, bucket_sort.cuh)
against the oracle, element by element.

The fused level runs on the large keys-only path (level-1 buckets of the
multi-kernel partition, PAPER.md:397-403 recursion) -- by default only above
~16M keys.  SR_OPT_TUNE + 3 caps the level-1 bucket count so that small inputs
reach it with level-1 buckets of tens of thousands of keys; SR_OPT_TUNE + 2
raises the mean sub-bucket so that the skew paths (bins above one warp's
network -> the CTA finishing kernel; above kCap -> the host's next level) run
too.  Every case is compared bit-exact with oracle.sort_keys.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1609_04471_b200 as sr
from workloads import gen

pytestmark = pytest.mark.gpu

T = sr.OPT_TUNE


@pytest.fixture
def tune():
    saved = []

    def set_(i, v, default):
        saved.append((i, default))
        sr.set_option(T + i, v)
    yield set_
    for i, d in reversed(saved):
        sr.set_option(T + i, d)
    sr.set_option(sr.OPT_RESIDENT, 1)


def _check(k):
    d = torch.from_numpy(k.copy()).cuda()
    sr.sort_keys(d)
    torch.cuda.synchronize()
    got = d.cpu().numpy()
    exp = oracle.sort_keys(k)
    assert np.array_equal(got, exp)
    return sr.last_plan()


@pytest.mark.parametrize("dt", [np.int32, np.int64])
@pytest.mark.parametrize("order", ["random", "few_unique", "few100", "swaps_1e1", "runs1024", "extremes",
                                   "organ_pipe", "equal_teeth"])
@pytest.mark.parametrize("n", [3_000_001, 4_194_304])
def test_fused_level_exact(tune, dt, order, n):
    sr.set_option(sr.OPT_RESIDENT, 0)
    tune(0, 1, 0)   # the fused level on (default off)
    tune(3, 64, 0)  # level-1 buckets of ~n/64 (47K-66K keys): the fused level takes them all
    p = _check(gen.make(order, n, dt, config=5))
    if order == "random":
        assert p["route_name"] == "partition" and p["levels"] == 2


@pytest.mark.parametrize("dt", [np.int32, np.int64])
@pytest.mark.parametrize("target", [16, 1500, 4096])
def test_fused_level_skew_paths(tune, dt, target):
    # target 1500 / 4096: most bins exceed one warp's network (CTA items), some exceed
    # kCap (host's next level); 16: the deepest trees with many empty bins
    sr.set_option(sr.OPT_RESIDENT, 0)
    tune(0, 1, 0)
    tune(3, 16, 0)
    tune(2, target, 256)
    _check(gen.make("random", 2_500_003, dt, config=6))


def test_fused_level_off_matches(tune):
    sr.set_option(sr.OPT_RESIDENT, 0)
    tune(3, 64, 0)
    tune(0, 0, 0)
    _check(gen.make("random", 3_000_001, np.int32, config=7))
