"""lane_stats with the reference's block semantics (batch.hpp:84-120,
run_block :149-294, merge :357-371), rebuilt from a per-(block, insertion
step) violation histogram (rebuild_lane_stats, the C++ shim's twin). CPU: the
oracle's histogram + results rebuild exactly the unmodified reference's own
lane_stats; GPU: the kernels' histogram equals the oracle's, and acceptance
criterion 5 (test_acceptance.cpp:189-242) holds on the GPU solve."""
import numpy as np
import pytest

from conftest import load_batch, requires_ref


@requires_ref
@pytest.mark.parametrize("name", ["c1", "mixed", "verify"])
@pytest.mark.parametrize("W", [512, 64, 7])
@pytest.mark.parametrize("balanced", [True, False])
def test_rebuilt_lane_stats_equal_the_reference(P, O, name, W, balanced):
    pk = load_batch(name)
    o = O.solve_batch(pk)
    hist = O.iter_hist(pk, W)
    sched = P.SchedulerKind.balanced if balanced else P.SchedulerKind.naive
    st = P.lp2d.rebuild_lane_stats(pk.m, o["status"], o["pair"], pk.perm, pk.offset,
                                   o["work_units"], hist, W, sched, True)
    lane_wu, tot, recs = O.ref_lane_stats(pk, W, balanced, record=True)
    assert st.blocks == int(tot[4])
    assert np.array_equal(st.lane_wu, lane_wu)
    assert st.total_wu == int(tot[0]) and st.violation_events == int(tot[1])
    assert st.masked_lane_iterations == int(tot[2])
    assert st.idle_wu_steps == int(tot[3])
    assert len(st.iterations) == int(tot[5])
    got = np.array([[r.block, r.iteration, r.active_lanes, r.masked_lanes, r.wu_count, r.idle_steps]
                    for r in st.iterations], np.uint64).reshape(-1, 6)
    assert np.array_equal(got, recs)
    ref_imb = float(lane_wu.max()) / (float(tot[0]) / len(lane_wu))
    assert P.lane_imbalance(st) == pytest.approx(ref_imb, rel=1e-12)


@pytest.mark.gpu
def test_gpu_histogram_and_criterion5(P, O):
    """The GPU's iter_hist equals the oracle's, so solve_batch's lane_stats
    are the reference's; criterion 5 on sizes {16, 1024} in one 512-lane
    block: balanced imbalance <= 1.5, naive >= 5, balanced faster."""
    import time

    b = P.gen_mixed([16, 1024], 512, 2026)
    pk = P.PackedBatch.from_batch(b)
    for W in (512, 100):
        hist = np.zeros(((pk.n + W - 1) // W) * (int(pk.m.max()) + 1), np.uint32)
        P.solve_packed(pk, P.BlockConfig(block_width=W), iter_hist=hist)
        assert np.array_equal(hist, O.iter_hist(pk, W))
    cfg_b = P.BlockConfig(block_width=512, scheduler=P.SchedulerKind.balanced, workers=1)
    cfg_n = P.BlockConfig(block_width=512, scheduler=P.SchedulerKind.naive, workers=1)
    P.solve_batch(b, cfg_b)  # warm
    P.solve_batch(b, cfg_n)
    tb = tn = 0.0
    for _ in range(3):
        t0 = time.perf_counter()
        rn = P.solve_batch(b, cfg_n)
        t1 = time.perf_counter()
        rb = P.solve_batch(b, cfg_b)
        t2 = time.perf_counter()
        tn += t1 - t0
        tb += t2 - t1
    imb_b, imb_n = P.lane_imbalance(rb.stats), P.lane_imbalance(rn.stats)
    lane_wu, tot, _ = O.ref_lane_stats(pk, 512, True)
    assert np.array_equal(rb.stats.lane_wu, lane_wu)
    assert imb_b <= 1.5 and imb_n >= 5.0, (imb_b, imb_n)
    assert tn > tb, (tn, tb)
