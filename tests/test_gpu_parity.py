"""Parity of the CUDA path (through the C ABI) with the reference and the
oracle. Bit-exact everywhere: fp64-stored results equal the UNMODIFIED
reference's (committed fixtures) and the fp64 oracle's; fp32-stored results
equal the unmodified reference run on the same fp32-rounded instance (double
arithmetic on the stored values: the ref32_* fixtures and the oracle's f
path). "Equal" is IEEE value equality (== ; -0 == +0) for x, y, value and
exact integer equality for status, defining pair, violation_events and
work_units. The north-star tolerances (1e-5 rel fp32, 1e-12 rel fp64) are
therefore met with zero error."""
import numpy as np
import pytest

from conftest import load_batch, load_npz

pytestmark = pytest.mark.gpu

SCHEDS = ("balanced", "naive")


def _cfg(P, sched):
    return P.BlockConfig(scheduler=getattr(P.SchedulerKind, sched))


def assert_same_as_oracle(r, o, O, what=""):
    st = r.status.astype(np.int32)
    bad = np.nonzero((st != o["status"]) | (r.pair != o["pair"]).any(axis=1))[0]
    assert bad.size == 0, f"{what}: status/pair differ at LPs {bad[:8]}"
    feas = o["status"] != O.INFEASIBLE
    for k in ("x", "y", "value"):
        g = getattr(r, k)[feas].astype(np.float64)
        # (NaN == NaN here: overflowing inputs give NaN in both)
        assert np.array_equal(g, o[k][feas], equal_nan=True), f"{what}: {k} differs"
    assert np.array_equal(r.violation_events.astype(np.uint64), o["violation_events"]), what
    assert np.array_equal(r.work_units, o["work_units"]), what


@pytest.mark.parametrize("sched", SCHEDS)
@pytest.mark.parametrize("name", ["c1", "mixed", "verify", "m1024"])
def test_fp64_equals_reference_fixture(P, O, name, sched):
    pk = load_batch(name)
    ref = load_npz(f"ref_{name}.npz")
    g = load_npz(f"oracle_{name}.npz")
    r = P.solve_packed(pk.with_perm_bits(16), _cfg(P, sched))
    feas = r.status.astype(np.int32) != O.INFEASIBLE
    assert np.array_equal(feas, ref["feasible"].astype(bool))
    for k in ("x", "y", "value"):
        assert np.array_equal(getattr(r, k)[feas], ref[k][feas]), k
    assert np.array_equal(r.violation_events.astype(np.uint64), ref["violation_events"])
    assert np.array_equal(r.work_units, ref["work_units"])
    assert np.array_equal(r.status.astype(np.int32), g["status64"])
    assert np.array_equal(r.pair, g["pair64"])


@pytest.mark.parametrize("sched", SCHEDS)
@pytest.mark.parametrize("name", ["c1", "mixed", "verify", "m1024"])
def test_fp32_equals_reference_fixture(P, O, name, sched):
    """fp32 storage: the UNMODIFIED reference's results on the fp32-rounded
    instance (ref32_* fixtures), bit for bit; status/pair as the oracle."""
    pk = load_batch(name).astype(np.float32)
    ref = load_npz(f"ref32_{name}.npz")
    g = load_npz(f"oracle_{name}.npz")
    r = P.solve_packed(pk, _cfg(P, sched))
    feas = r.status.astype(np.int32) != O.INFEASIBLE
    assert np.array_equal(feas, ref["feasible"].astype(bool))
    for k in ("x", "y", "value"):
        assert np.array_equal(getattr(r, k)[feas], ref[k][feas]), k
    assert np.array_equal(r.violation_events.astype(np.uint64), ref["violation_events"])
    assert np.array_equal(r.work_units, ref["work_units"])
    assert np.array_equal(r.status.astype(np.int32), g["status32"])
    assert np.array_equal(r.pair, g["pair32"])


def test_headline_config_full_size(P, O):
    """BASELINE configs[1]: 16384 x 1024 fp32, every LP against the oracle."""
    pb = P.PackedBatch.generate(np.full(16384, 1024, np.int32), 2).astype(np.float32)
    r = P.solve_packed(pb)
    assert_same_as_oracle(r, O.solve_batch(pb, threads=16), O, "c2")


def test_orca_config_full_size(P, O):
    """BASELINE configs[2] shape: 2^20 x 128 fp32 (one GPU's worth here)."""
    n = 1 << 20
    kind = np.zeros(n, np.uint8)
    kind[::10] = 1  # every 10th LP infeasible
    pb = P.PackedBatch.generate(np.full(n, 128, np.int32), 3, kind=kind,
                                bscale=2e-7).astype(np.float32)
    r = P.solve_packed(pb)
    o = O.solve_batch(pb, threads=16)
    assert_same_as_oracle(r, o, O, "c3")
    assert (o["status"] == O.INFEASIBLE).sum() >= n // 10


def test_fp64_mixed_status_config(P, O):
    """BASELINE configs[4] shape (2^16 subset): 256 constraints fp64 with
    10% infeasible and 10% unbounded kinds."""
    n = 1 << 16
    kind = np.zeros(n, np.uint8)
    kind[3::10] = 1
    kind[7::10] = 3
    pb = P.PackedBatch.generate(np.full(n, 256, np.int32), 5, kind=kind)
    r = P.solve_packed(pb)
    o = O.solve_batch(pb, threads=16)
    assert_same_as_oracle(r, o, O, "c5")
    st = r.status.astype(np.int32)
    assert (st[3::10] == O.INFEASIBLE).all() and (st[7::10] == O.UNBOUNDED).all()


def pareto_sizes(P, seed, total):
    L = P.lp2d.N.lib()
    out = np.zeros(total // 8 + 1, np.int32)
    n = L.lp2dgen_pareto_sizes(seed, 8.0, 1.0, 8192, total, len(out), out.ctypes.data)
    return out[:n]


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_heavy_tailed_mixed_batch(P, O, dt):
    """BASELINE configs[3] shape (2^20-constraint subset): Pareto sizes 8..8192
    exercise every size class, the device-side binning and the large-LP
    kernel."""
    m = pareto_sizes(P, 4, 1 << 20)
    pb = P.PackedBatch.generate(m, 4)
    if dt == np.float32:
        pb = pb.astype(np.float32)
    r = P.solve_packed(pb)
    assert_same_as_oracle(r, O.solve_batch(pb, threads=16), O, "c4")


def test_large_lps_both_precisions(P, O):
    m = np.array([1053, 2000, 541, 4100, 8192, 70000, 12], np.int32)
    for dt in (np.float32, np.float64):
        pb = P.PackedBatch.generate(m, 12, perm_bits=32)
        if dt == np.float32:
            pb = pb.astype(np.float32)
        for sched in SCHEDS:
            assert_same_as_oracle(P.solve_packed(pb, _cfg(P, sched)), O.solve_batch(pb), O, sched)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_size_class_edges(P, O, dt):
    cap = 1052
    sizes = np.array([0, 1, 2, 3, 4, 27, 28, 29, 31, 32, 60, 61, 92, 93, 156, 157, 284, 285,
                      540, 541 if dt == np.float32 else 539, cap], np.int32)
    pb = P.PackedBatch.generate(np.repeat(sizes, 3), 21).astype(dt)
    assert_same_as_oracle(P.solve_packed(pb), O.solve_batch(pb), O, "edges")


def test_u32_permutations_and_naive(P, O):
    pb = P.PackedBatch.generate(np.full(300, 200, np.int32), 4, perm_bits=32).astype(np.float32)
    o = O.solve_batch(pb)
    for sched in SCHEDS:
        assert_same_as_oracle(P.solve_packed(pb, _cfg(P, sched)), o, O, sched)


def test_invalid_permutation_is_flagged(P):
    pb = P.PackedBatch.generate(np.full(8, 40, np.int32), 4)
    pb.perm[int(pb.offset[3]) + 5] = 60000
    r = P.solve_packed(pb)
    assert r.status[3] == 255 and (r.status[[0, 1, 2, 4, 5, 6, 7]] != 255).all()


def test_hand_cases_and_parallel_constraints(P, O):
    """Axis-aligned and duplicated constraints exercise the exact parallel
    path (test_serial.cpp:57-86 shapes)."""
    probs = [
        ([[1, 0, 1], [0, 1, 1]], (1, 1), 10),
        ([[1, 0, 0], [-1, 0, -1]], (1, 1), 10),            # contradictory
        ([[0, 1, 1], [0, 1, 1], [0, 2, 2], [1, 0, 2]], (1, 1), 10),  # parallel/duplicate
        ([[0, 1, 1], [0, -1, -2]], (0, 1), 10),            # parallel infeasible
        ([[1, 1, 2], [1, -1, 0], [-1, 0, 0]], (0, 1), 10),  # ties
        ([], (-1, -1), 5),
    ]
    batch = P.Batch([P.Problem(c, np.array(cons, float).reshape(-1, 3), M) for cons, c, M in probs],
                    [P.identity_permutation(len(cons)) for cons, _, _ in probs])
    for dt in (np.float64, np.float32):
        pb = P.PackedBatch.from_batch(batch, dtype=dt)
        for sched in SCHEDS:
            assert_same_as_oracle(P.solve_packed(pb, _cfg(P, sched)), O.solve_batch(pb), O, sched)


def test_wild_magnitudes_take_the_exact_path(P, O):
    rng = np.random.default_rng(5)
    pb = P.PackedBatch.generate(np.full(64, 50, np.int32), 8).astype(np.float32)
    pb.ax[: int(pb.offset[8])] *= np.float32(1e20)  # |a| >= 2^61: exact path
    pb.b[int(pb.offset[16]):int(pb.offset[24])] *= np.float32(1e-30)
    pb.ay[int(pb.offset[30]):int(pb.offset[31])] = 0.0
    assert_same_as_oracle(P.solve_packed(pb), O.solve_batch(pb), O, "wild")


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_tiny_lps_lane_kernel(P, O, dt):
    """m <= 28 runs one LP per lane (k_solve_lanes): all generator kinds,
    every size 0..28, wild magnitudes (exact fold per lane), an invalid
    permutation, alone (uniform launch) and mixed with larger LPs (binned,
    lane class sorted by m), host and device mode."""
    import torch

    rng = np.random.default_rng(11)
    m = rng.integers(0, 29, 3000).astype(np.int32)
    kind = rng.choice([P.GenKind.feasible_random, P.GenKind.infeasible,
                       P.GenKind.unbounded_random], 3000).astype(np.uint8)
    kind[m < 1] = P.GenKind.feasible_random  # (infeasible needs m >= 1)
    pb = P.PackedBatch.generate(m, 31, kind=kind).astype(dt)
    e = int(pb.offset[100])
    pb.ax[:e] *= dt(1e20) if dt == np.float32 else dt(1e160)
    pb.b[int(pb.offset[200]):int(pb.offset[260])] *= dt(1e-30)
    pb.ay[int(pb.offset[300]):int(pb.offset[340])] = 0.0
    o = O.solve_batch(pb)
    r = P.solve_packed(pb)
    assert_same_as_oracle(r, o, O, "tiny")
    bad = pb.subset(0, 64)
    j = int(np.nonzero(bad.m > 3)[0][0])
    bad.perm = bad.perm.copy()
    bad.perm[int(bad.offset[j]) + 1] = 1000
    rb = P.solve_packed(bad)
    assert rb.status[j] == 255 and (np.delete(rb.status, j) != 255).all()
    # mixed with larger LPs: the binned path with per-m sub-bins
    mix = P.PackedBatch.generate(np.concatenate([m[:1500], rng.integers(29, 400, 500)]).astype(np.int32),
                                 32).astype(dt)
    om = O.solve_batch(mix)
    assert_same_as_oracle(P.solve_packed(mix), om, O, "tiny+mixed")
    db = P.DeviceBatch(mix)
    out = db.empty_result()
    P.solve_device(db, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.status.cpu().numpy().astype(np.int32), om["status"])
    assert np.array_equal(out.work_units.cpu().numpy(), om["work_units"])


def test_batch_api_matches_serial_semantics(P, O):
    """test_batch.cpp:55-74: both schedulers == serial, stats equal."""
    base = P.gen(128, 77)
    b = P.replicate(base, 96, 5)
    pb = P.PackedBatch.from_batch(b)
    o = O.solve_batch(pb)
    for sched in SCHEDS:
        res = P.solve_batch(b, _cfg(P, sched))
        assert res.stats.violation_events == int(o["violation_events"].sum())
        assert res.stats.total_wu == int(o["work_units"].sum())
        for j, s in enumerate(res.solutions):
            assert s.feasible == (o["status"][j] != O.INFEASIBLE)
            assert s.point == (o["x"][j], o["y"][j]) and s.value == o["value"][j]


def test_device_mode_matches_host_mode(P):
    import torch

    pb = P.PackedBatch.generate(np.full(2048, 300, np.int32), 6).astype(np.float32)
    host = P.solve_packed(pb)
    db = P.DeviceBatch(pb)
    out = db.empty_result()
    P.solve_device(db, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.status.cpu().numpy(), host.status)
    assert np.array_equal(out.x.cpu().numpy(), host.x)
    assert np.array_equal(out.pair.cpu().numpy(), host.pair)
    # repeated launches reuse the self-resetting ticket counters
    for _ in range(5):
        P.solve_device(db, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.value.cpu().numpy(), host.value)


def test_kernel_launch_counter(P):
    import torch

    uni = P.DeviceBatch(P.PackedBatch.generate(np.full(512, 200, np.int32), 3).astype(np.float32))
    mixed = P.DeviceBatch(P.PackedBatch.generate(np.array([8, 40, 100, 700, 3000], np.int32)
                                                 .repeat(64), 3).astype(np.float32))
    # uniform fp32 warp class: one K4 launch; mixed: 2 binning + 5 widening
    # (the lane/CTA classes read double copies) + <= 11 class launches
    for db, lo, hi in ((uni, 1, 1), (mixed, 3, 2 + 5 + 11)):
        out = db.empty_result()
        k0 = P.kernel_launches()
        P.solve_device(db, out)
        k = P.kernel_launches() - k0
        torch.cuda.synchronize()
        assert lo <= k <= hi, k


def test_device_shuffle_matches_host(P):
    import ctypes as C

    import torch

    m = np.array([1, 2, 10, 16, 1000, 4096], np.int32)
    off = P.lp2d.pack_offsets(m)
    seeds = np.array([P.derive_seed(7, j) for j in range(len(m))], np.uint64)
    dev = torch.device("cuda", 0)
    for bits, tdt in ((16, torch.int16), (32, torch.int32)):
        perm = torch.zeros(int(off[-1]), dtype=tdt, device=dev)
        dm, doff = torch.from_numpy(m).to(dev), torch.from_numpy(off).to(dev)
        ds = torch.from_numpy(seeds.view(np.int64)).to(dev)
        rc = P.lp2d.N.lib().lp2dgpu_shuffle_device(len(m), dm.data_ptr(), doff.data_ptr(), ds.data_ptr(),
                                                    perm.data_ptr(), bits, 0, None)
        assert rc == 0
        torch.cuda.synchronize()
        got = perm.cpu().numpy().view(np.uint16 if bits == 16 else np.uint32)
        for j in range(len(m)):
            o = int(off[j])
            assert np.array_equal(got[o:o + m[j]], P.shuffle(int(m[j]), int(seeds[j])).order)


def test_smoke_entry_point():
    import __graft_entry__

    __graft_entry__.smoke()


def test_cpp_drop_in_against_reference_headers():
    """tests/cpp/shim_test.cpp: the reference's own types and solver, compiled
    with include/lp2d_b200/solve_batch.hpp (built where /root/reference is)."""
    import os
    import subprocess

    from conftest import ROOT

    exe = os.path.join(ROOT, "tests", "cpp", "build", "shim_test")
    if not os.path.exists(exe):
        pytest.skip("shim_test not built (needs the reference headers)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_adversarial_inputs_every_warp_class(P, O, dt):
    """Every warp-kernel size class (register classes, the register+tail
    class) under inputs that defeat each fast-path shortcut and must take the
    exact reference operations instead: duplicated and parallel constraints
    (parallel-bound refolds), huge coefficients (infinite per-lane bound),
    tiny right-hand sides (line through the fast sqrt/div range check),
    zero normals (NaN lines), NaN and infinite entries. Bit-identical to the
    oracle in both precisions."""
    rng = np.random.default_rng(21)
    sizes = np.repeat(np.array([40, 100, 150, 180, 250, 300, 500, 700, 1000, 1500, 2076],
                               np.int32), 6)
    pb = P.PackedBatch.generate(sizes, 77).astype(dt)
    ax, ay, b = pb.ax, pb.ay, pb.b
    for j in range(pb.n):
        o, mj = int(pb.offset[j]), int(pb.m[j])
        sel = j % 6
        k = rng.integers(0, mj, 8)
        if sel == 0:    # duplicates and scaled (parallel) copies
            src = rng.integers(0, mj, 8)
            ax[o + k], ay[o + k], b[o + k] = ax[o + src], ay[o + src], b[o + src]
            ax[o + k[:4]] *= dt(2)
            ay[o + k[:4]] *= dt(2)
            b[o + k[:4]] *= dt(2)
        elif sel == 1:  # huge coefficients, late in the permutation too
            ax[o + k] *= dt(1e20) if dt == np.float32 else dt(1e160)
        elif sel == 2:  # tiny right-hand sides
            b[o + k] *= dt(1e-30) if dt == np.float32 else dt(1e-300)
        elif sel == 3:  # zero normals, violated (b < 0) or not
            ax[o + k] = 0
            ay[o + k] = 0
            b[o + k[:4]] = -1
        elif sel == 4:  # NaN entry
            ay[o + k[0]] = np.nan
        else:           # infinite right-hand sides and nearly parallel pairs
            b[o + k[:3]] = np.inf
            ax[o + k[3:]] = ax[o + k[2]] * (dt(1) + dt(2) ** -20)
            ay[o + k[3:]] = ay[o + k[2]]
    o = O.solve_batch(pb)
    for sched in SCHEDS:
        assert_same_as_oracle(P.solve_packed(pb, _cfg(P, sched)), o, O, f"adversarial {sched}")


def test_device_generator_streams_and_parity(P, O):
    """lp2dgpu_generate_device: the integer streams
    (permutations, and hence every draw) are bit-identical to the host
    generator; the trigonometry is the device's, within a few ulps of glibc;
    a solve over the device-generated batch is bit-identical to the oracle
    run on the downloaded instance (fp64 and fp32, all kinds)."""
    rng = np.random.default_rng(3)
    m = rng.integers(1, 1100, 600).astype(np.int32)
    kind = rng.choice([P.GenKind.feasible_random, P.GenKind.infeasible,
                       P.GenKind.unbounded_random], 600).astype(np.uint8)
    host = P.PackedBatch.generate(m, 99, kind=kind, first=7)
    for dt in (np.float64, np.float32):
        db = P.DeviceBatch.generate(m, 99, kind=kind, first=7, dtype=dt)
        dv = db.to_packed()
        assert np.array_equal(dv.perm, host.perm)
        assert np.array_equal(dv.offset, host.offset)
        hx = host.astype(dt)
        eps = np.finfo(dt).eps
        for a, h in ((dv.ax, hx.ax), (dv.ay, hx.ay), (dv.c, hx.c)):  # unit vectors
            assert np.allclose(a, h, rtol=0, atol=4 * eps)
        # b = a.interior + slack with |interior| <= 5e6: a 1-ulp cos/sin
        # difference moves b by <= ~1e7 ulps of 1 (then float rounding)
        assert np.allclose(dv.b, hx.b, rtol=0, atol=1e7 * 8 * np.finfo(np.float64).eps + 2 * eps * 1.5e7)
        assert np.array_equal(dv.M, hx.M)
        out = db.empty_result()
        P.solve_device(db, out)
        o = O.solve_batch(dv)
        st = out.status.cpu().numpy().astype(np.int32)
        assert np.array_equal(st, o["status"])
        assert np.array_equal(out.pair.cpu().numpy(), o["pair"])
        feas = o["status"] != O.INFEASIBLE
        assert np.array_equal(out.x.cpu().numpy()[feas].astype(np.float64), o["x"][feas])
        assert np.array_equal(out.work_units.cpu().numpy().astype(np.uint64), o["work_units"])


def test_small_lps_class(P, O):
    """29 <= m <= 60 in fp32 storage (K4 by default; K6 lane groups with
    LP2D_B200_GRP=2, test_k6_lane_groups_small_class): all generator kinds,
    every size of the class, wild magnitudes (exact refolds), an invalid
    permutation (status 255 for that LP only), uniform and binned launches."""
    rng = np.random.default_rng(12)
    m = rng.integers(29, 61, 2000).astype(np.int32)
    kind = rng.choice([P.GenKind.feasible_random, P.GenKind.infeasible,
                       P.GenKind.unbounded_random], 2000).astype(np.uint8)
    pb = P.PackedBatch.generate(m, 41, kind=kind).astype(np.float32)
    pb.ax[:int(pb.offset[50])] *= np.float32(1e20)
    pb.b[int(pb.offset[100]):int(pb.offset[150])] *= np.float32(1e-30)
    pb.ay[int(pb.offset[200]):int(pb.offset[230])] = 0.0
    assert_same_as_oracle(P.solve_packed(pb), O.solve_batch(pb), O, "k6")
    bad = pb.subset(0, 64)
    bad.perm = bad.perm.copy()
    bad.perm[int(bad.offset[5]) + 7] = 1000
    rb = P.solve_packed(bad)
    assert rb.status[5] == 255 and (np.delete(rb.status, 5) != 255).all()
    mix = P.PackedBatch.generate(np.concatenate([m[:800], rng.integers(1, 400, 400)]).astype(np.int32),
                                 42).astype(np.float32)
    assert_same_as_oracle(P.solve_packed(mix), O.solve_batch(mix), O, "k6+mixed")


def test_k6_lane_groups_small_class():
    """The same class through K6 (4 lanes per LP, 8 LPs per warp), in a fresh
    process because the library reads LP2D_B200_GRP once."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, LP2D_B200_GRP="2")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(here, "test_gpu_parity.py") + "::test_small_lps_class"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
