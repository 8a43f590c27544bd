"""Edge cases of the GPU path the reference's own tests pin (SURVEY.md
§8(c)): adversarial_ordered instances (test_generate.cpp:62-88: every
constraint violates in file order, so the 1D re-solves run over the whole
prefix, O(m^2)), the defining pair (each optimum is exactly the intersection
the pair names, recomputed with the reference's operations), and the
reference's brute-force vertex oracle (oracle.hpp:38-70) for m <= 512.
fp64 and fp32 storage (the reference's double arithmetic on the stored
values)."""
import numpy as np
import pytest

from conftest import requires_ref

pytestmark = pytest.mark.gpu


def _adversarial_batch(O, sizes, seed0, shuffled):
    ref = O.ref_lib()
    n = len(sizes)
    m = np.asarray(sizes, np.int32)
    off = O.pack_offsets(m)
    E = int(off[-1])
    ax = np.zeros(E); ay = np.zeros(E); b = np.zeros(E)
    perm = np.zeros(E, np.uint32); c = np.zeros(2 * n); M = np.zeros(n)
    for j, mj in enumerate(sizes):
        o = int(off[j])
        tax, tay, tb = np.zeros(mj), np.zeros(mj), np.zeros(mj)
        cc, mm = np.zeros(2), np.zeros(1)
        assert ref.ref_gen(mj, seed0 + j, 2, 1.0, tax.ctypes.data, tay.ctypes.data, tb.ctypes.data,
                           cc.ctypes.data, mm.ctypes.data) == 0
        ax[o:o + mj], ay[o:o + mj], b[o:o + mj] = tax, tay, tb
        c[2 * j:2 * j + 2], M[j] = cc, mm[0]
        perm[o:o + mj] = O.shuffle(mj, seed0 + j) if shuffled else np.arange(mj, dtype=np.uint32)
    return O.RefPacked(m, off, ax, ay, b, perm, c, M)


def _packed(P, rp, dt):
    q = rp.astype(dt) if dt != np.float64 else rp
    return P.PackedBatch(q.m, q.offset, q.ax, q.ay, q.b, q.perm.astype(np.uint16), q.c, q.M)


def _same(r, o, O, what):
    st = r.status.astype(np.int32)
    assert np.array_equal(st, o["status"]), what
    assert np.array_equal(r.pair, o["pair"]), what
    feas = o["status"] != O.INFEASIBLE
    for k in ("x", "y", "value"):
        assert np.array_equal(getattr(r, k)[feas], o[k][feas]), (what, k)
    assert np.array_equal(r.violation_events.astype(np.uint64), o["violation_events"]), what
    assert np.array_equal(r.work_units, o["work_units"]), what


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_adversarial_ordered_every_step_violates(P, O, dt):
    sizes = [16, 40, 60, 64, 100, 300, 700, 1000, 2048]
    rp = _adversarial_batch(O, sizes, 3, shuffled=False)
    pb = _packed(P, rp, dt)
    o = O.solve_batch(pb)
    for sched in ("balanced", "naive"):
        r = P.solve_packed(pb, P.BlockConfig(scheduler=getattr(P.SchedulerKind, sched)))
        _same(r, o, O, f"adversarial {sched} {np.dtype(dt)}")
    if dt == np.float64:  # test_generate.cpp:62-88 (in file order: m events)
        assert np.array_equal(o["violation_events"], np.asarray(sizes, np.uint64))
    # shuffled order breaks the chain (logarithmic events), same answers
    rs = _adversarial_batch(O, sizes, 3, shuffled=True)
    ps = _packed(P, rs, dt)
    _same(P.solve_packed(ps), O.solve_batch(ps), O, "adversarial shuffled")


def _exact_point(h, q, M):
    """serial.hpp:95-111 / core.hpp:70-109 with the reference's operation
    order in float64 (numpy scalars are IEEE doubles, no contraction)."""
    hx, hy, hb = (np.float64(v) for v in h)
    len2 = hx * hx + hy * hy
    ln = np.sqrt(len2)
    s = hb / len2
    r = np.float64(1.0) / ln
    ox, oy, dx, dy = s * hx, s * hy, r * (-hy), r * hx
    qx, qy, qb = (np.float64(v) for v in q)
    t = (qb - (qx * ox + qy * oy)) / (qx * dx + qy * dy)
    return ox + t * dx, oy + t * dy


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_defining_pair_reproduces_the_optimum(P, O, dt):
    """For every solved LP the optimum is, bit for bit, the intersection of
    the defining pair's lines computed with the reference's operations."""
    pb = P.PackedBatch.generate(np.array([64, 200, 1024, 40, 500], np.int32).repeat(40), 17)
    pb = pb.astype(dt) if dt != np.float64 else pb
    r = P.solve_packed(pb)
    box = {-1: (1.0, 0.0), -2: (-1.0, 0.0), -3: (0.0, 1.0), -4: (0.0, -1.0)}

    def con(j, k):
        if k < 0:
            return (*box[k], float(pb.M[j]))
        o = int(pb.offset[j]) + k
        return (float(pb.ax[o]), float(pb.ay[o]), float(pb.b[o]))

    checked = 0
    for j in range(pb.n):
        if r.status[j] == O.INFEASIBLE:
            continue
        k0, k1 = int(r.pair[j, 0]), int(r.pair[j, 1])
        if k0 < 0:  # no event: the start corner
            M = float(pb.M[j])
            assert abs(r.x[j]) == M and abs(r.y[j]) == M
            continue
        x, y = _exact_point(con(j, k0), con(j, k1), pb.M[j])
        assert (x, y) == (r.x[j], r.y[j]), j
        checked += 1
    assert checked > pb.n // 2


@requires_ref
def test_against_the_reference_bruteforce_oracle(P, O):
    """The unmodified reference's solve_bruteforce (oracle.hpp:38-70, vertex
    enumeration, m <= 512, oracle/_ref): same feasibility and
    the optimum value to the reference's own agreement rule (5 significant
    figures, core.hpp:120-125); fp64."""
    kind = np.zeros(160, np.uint8)
    kind[::7] = 1
    pb = P.PackedBatch.generate(np.array([8, 30, 64, 150, 300], np.int32).repeat(32), 23, kind=kind)
    r = P.solve_packed(pb)
    for j in range(pb.n):
        o, mj = int(pb.offset[j]), int(pb.m[j])
        bf_feas, _, _, bf_value = O.ref_bruteforce(pb.ax[o:o + mj], pb.ay[o:o + mj], pb.b[o:o + mj],
                                                   pb.c[2 * j:2 * j + 2], pb.M[j])
        feas = r.status[j] != O.INFEASIBLE
        assert feas == bf_feas, j
        if feas:
            assert P.lp2d.agree_sig_figs(float(r.value[j]), bf_value, 5), (j, r.value[j], bf_value)


def test_perm_seed_device_mode_fills_the_generator_permutations(P):
    """Device mode with perm_from_seed: the library writes shuffle(m,
    derive_seed(seed, 2g+1)) for global LP g = first + j into the caller's
    buffer (the PackedBatch generator's streams), then solves."""
    import torch

    sizes = np.array([0, 1, 7, 64, 300, 1024, 5000, 70000], np.int32)
    pb = P.PackedBatch.generate(sizes, 17, first=1000, perm_bits=32)
    db = P.DeviceBatch(pb)
    db.perm.zero_()
    out = db.empty_result()
    s = P.lp2d.N.BatchSoA(db.n, db.m.data_ptr(), db.offset.data_ptr(), db.ax.data_ptr(),
                          db.ay.data_ptr(), db.b.data_ptr(), db.perm.data_ptr(), 32,
                          P.lp2d.N.MEM_DEVICE, db.c.data_ptr(), db.M.data_ptr(), db.max_m, db.min_m)
    s.perm_from_seed, s.perm_mul, s.perm_add, s.perm_seed, s.perm_first = 1, 2, 1, 17, 1000
    o = P.lp2d._opts(P.BlockConfig(), P.Tolerance(), device=0,
                     stream=torch.cuda.current_stream().cuda_stream)
    r = P.lp2d.N.Out(out.status.data_ptr(), out.x.data_ptr(), out.y.data_ptr(),
                     out.value.data_ptr(), out.pair.data_ptr(), out.violation_events.data_ptr(),
                     out.work_units.data_ptr())
    import ctypes as C

    assert P.lp2d.N.lib().lp2dgpu_solve_f64(C.byref(s), C.byref(o), C.byref(r)) == 0
    torch.cuda.synchronize()
    got = db.perm.cpu().numpy().view(np.uint32)
    for j in range(pb.n):
        a, b = int(pb.offset[j]), int(pb.offset[j]) + int(sizes[j])
        assert np.array_equal(got[a:b], pb.perm[a:b]), j
    ref = P.solve_packed(pb)
    assert np.array_equal(out.status.cpu().numpy(), ref.status)
    assert np.array_equal(out.x.cpu().numpy(), ref.x)
