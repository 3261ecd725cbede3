"""Parity of the presortedness measures (-m gpu; SURVEY.md §8(f) NEXT #4,
PAPER.md:62-85): sr_presortedness against the oracle's plain definitions on the
paper's input classes, sizes spanning single and many CTAs and ragged tails."""
import numpy as np
import pytest
import torch

import oracle
import paper_1609_04471_b200 as sr
from workloads import gen

pytestmark = pytest.mark.gpu

ORDERS = ["random", "reversed", "nearly", "few_unique", "sorted", "all_equal", "organ_pipe", "runs1024",
          "sharp_teeth", "even_teeth", "equal_teeth", "distance256", "swaps_1e3"]


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("order", ORDERS)
@pytest.mark.parametrize("n", [2, 3, 1000, 16385, 300_007])
def test_measures_parity(order, dtype, n):
    k = gen.make(order, n, dtype, config=71)
    d = torch.from_numpy(k.copy()).cuda()
    got = sr.presortedness(d)
    exp = oracle.measures(k)
    assert {f: got[f] for f in exp} == exp
    assert np.array_equal(d.cpu().numpy(), k)  # the input is not modified


def test_measures_large():
    k = gen.make("nearly", 2_000_000, np.int32, config=72)
    assert sr.presortedness(torch.from_numpy(k).cuda()) == {"n": k.size, **oracle.measures(k)}


def test_measures_trivial_sizes():
    for n in [0, 1]:
        m = sr.presortedness(torch.zeros(n, dtype=torch.int32, device="cuda"))
        assert m["n"] == n and m["runs"] == n and m["mono"] == n and m["inversions"] == 0
