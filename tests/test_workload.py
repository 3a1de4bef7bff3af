"""Host trace generation (CPU): the product's generator reproduces the
reference's build_workload (experiment.hpp:291-305) bit for bit, and the
Table 1 statistics (test_workload.cpp:226-244 style)."""
import numpy as np
import pytest

import oracles as O
from paper_2408_13510_b200 import abi, engine

pytestmark = pytest.mark.skipif(not O.have_ref(), reason="reference driver unavailable")


@pytest.mark.parametrize("seed,n,rate,weights,process", [
    (1, 2000, 20.0, None, 0),
    (777, 12, 12.0, None, 0),
    (31337, 500, 40.0, None, 1),
    (5, 3000, 40.0, (0, 3, 1, 2, 0), 0),   # BASELINE c5 heavy-decode mixture
    (2**40 + 3, 64, 7.5, (1, 1, 1, 1, 1), 0),
])
def test_generator_bit_identical(lib, seed, n, rate, weights, process):
    ref = O.ref_generate(seed, n, rate, weights, process)
    tb = engine.build_workload([seed], n, rate, weights, process)
    assert np.array_equal(tb.prompt, ref.prompt)
    assert np.array_equal(tb.decode, ref.decode)
    assert np.array_equal(tb.task, ref.task)
    assert np.array_equal(tb.arrival.view(np.uint64), ref.arrival.view(np.uint64))


def test_batch_generation_matches_single(lib):
    seeds = [3, 4, 5, 6]
    tb = engine.build_workload(seeds, 300, 20.0, threads=3)
    for r, s in enumerate(seeds):
        one = engine.build_workload([s], 300, 20.0)
        sl = tb.replay(r)
        assert np.array_equal(tb.arrival[sl], one.arrival)
        assert np.array_equal(tb.prompt[sl], one.prompt)


def test_table1_statistics(lib):
    # Overall means of the 5-task mix over 31,329 requests (Table 1 weights).
    tb = engine.build_workload([1], 31329, 20.0)
    assert 1 <= tb.prompt.min() and tb.prompt.max() <= 1000
    assert 1 <= tb.decode.min() and tb.decode.max() <= 4096
    assert abs(tb.prompt.mean() - 89.0) < 6.0
    assert abs(tb.decode.mean() - 176.0) < 12.0
    assert np.all(np.diff(tb.arrival) >= 0)
    counts = np.bincount(tb.task, minlength=5) / tb.task.size
    want = np.array(abi.DATASET_SAMPLES) / sum(abi.DATASET_SAMPLES)
    assert np.allclose(counts, want, atol=0.01)
