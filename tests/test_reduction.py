"""Contention microbenchmark: segmented extremes.

CPU part: the oracle restatement (oracle/lp2d_oracle.c) against the compiled
reference (reduction.hpp:46-129) and the reference's own test cases
(test_reduction.cpp, test_acceptance.cpp criterion 6, test_bench.cpp
"contention runs cover the requested grid"). GPU part: every GPU strategy
(include/lp2d_b200.h LP2D_REDUCE_*) bit-identical to the oracle."""
import numpy as np
import pytest

from conftest import requires_ref

LEVELS = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512]






@requires_ref
@pytest.mark.parametrize("strategy", [0, 1, 2])
def test_oracle_matches_reference(O, strategy):
    v = O.uniform(808, 1, -1e9, 1e9, 1 << 14)
    for c in LEVELS + [35, 3, 1000]:
        vv = v[: len(v) // c * c]
        a = O.segmented_extremes(vv, c, strategy)
        b = O.segmented_extremes(vv, c, strategy, ref=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert np.array_equal(a[0], vv.reshape(-1, c).min(1))
        assert np.array_equal(a[1], vv.reshape(-1, c).max(1))


@requires_ref
def test_contention_inputs_match_reference(O, P):
    assert np.array_equal(P.reduction.contention_values(5, 4096), O.uniform(5, 0xC0, -1e6, 1e6, 4096, ref=True))


def test_bad_shapes_rejected(O, P):
    """test_reduction.cpp:76-90 and bench.hpp:249-255."""
    v = np.zeros(16)
    for c in (0, 3):
        with pytest.raises(ValueError):
            O.segmented_extremes(v, c, 0)
        with pytest.raises(ValueError):
            P.segmented_extremes(v, c)
    for bad in ([48], [1024], [0]):
        with pytest.raises(ValueError):
            P.contention_bench([P.ReduceStrategy.tree_reduction], bad, 1, 5, 2048)


GPU_STRATEGIES = ["serialized_shared_update", "tree_reduction", "private_then_merge",
                  "global_atomic", "cub_segmented_reduce"]


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", GPU_STRATEGIES)
def test_gpu_strategies_bit_identical(O, P, strategy):
    s = getattr(P.ReduceStrategy, strategy)
    v = O.uniform(606, 0, -1e9, 1e9, 10240)  # test_acceptance.cpp:244-270 shape
    for c in LEVELS + [35, 5, 1000, 10240]:
        vv = v[: len(v) // c * c]
        mn, mx = P.segmented_extremes(vv, c, s)
        omn, omx = O.segmented_extremes(vv, c, 0)
        assert np.array_equal(mn, omn) and np.array_equal(mx, omx), (strategy, c)


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", GPU_STRATEGIES)
def test_gpu_nan_handling_like_fmin(O, P, strategy):
    s = getattr(P.ReduceStrategy, strategy)
    v = O.uniform(7, 0, -1.0, 1.0, 64 * 16)
    v[::7] = np.nan
    v[16 * 3:16 * 4] = np.nan  # one all-NaN group
    mn, mx = P.segmented_extremes(v, 16, s)
    omn, omx = O.segmented_extremes(v, 16, 0)
    assert np.array_equal(mn, omn, equal_nan=True) and np.array_equal(mx, omx, equal_nan=True)
    assert np.isnan(mn[3]) and np.isnan(mx[3])


@pytest.mark.gpu
def test_contention_bench_grid(P):
    """test_bench.cpp "contention runs cover the requested grid"."""
    strategies = [P.ReduceStrategy.serialized_shared_update, P.ReduceStrategy.tree_reduction]
    recs = P.contention_bench(strategies, [1, 8, 512], 2, 5, 512 * 8)
    assert len(recs) == 2 * 3 * 2
    assert all(r.wall_time_ns >= 0 for r in recs)
