"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes bindings for the restated CPU oracle (oracle/build/liblp2d_oracle.so)
and for the unmodified reference wrapped as oracle/_ref/liblp2d_ref.so.
Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg; the product never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "build", "liblp2d_oracle.so")
REF_SO = os.path.join(_HERE, "_ref", "liblp2d_ref.so")

OPTIMAL, INFEASIBLE, UNBOUNDED = 0, 1, 2
NONE = -(2**31)


class OracleResult(C.Structure):
    _fields_ = [
        ("x", C.c_double),
        ("y", C.c_double),
        ("value", C.c_double),
        ("violation_events", C.c_uint64),
        ("work_units", C.c_uint64),
        ("pair", C.c_int32 * 2),
        ("status", C.c_int32),
        ("pad", C.c_int32),
    ]


RESULT_DTYPE = np.dtype(
    [
        ("x", "<f8"),
        ("y", "<f8"),
        ("value", "<f8"),
        ("violation_events", "<u8"),
        ("work_units", "<u8"),
        ("pair", "<i4", (2,)),
        ("status", "<i4"),
        ("pad", "<i4"),
    ]
)
assert RESULT_DTYPE.itemsize == C.sizeof(OracleResult)


def build():
    """Compile oracle/ (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_oracle = None
_ref = None


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = C.CDLL(ORACLE_SO)
        lib.lp2d_oracle_derive_seed.restype = C.c_uint64
        lib.lp2d_oracle_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.lp2d_oracle_shuffle.argtypes = [C.c_int64, C.c_uint64, C.c_void_p]
        lib.lp2d_oracle_xoshiro_first.argtypes = [C.c_uint64, C.c_int, C.c_void_p]
        lib.lp2d_oracle_gen.argtypes = [C.c_int64, C.c_uint64, C.c_int, C.c_double] + [C.c_void_p] * 6
        for suf in ("d", "f"):
            fn = getattr(lib, "lp2d_oracle_solve_batch_" + suf)
            fn.argtypes = [C.c_int64] + [C.c_void_p] * 8 + [C.c_double, C.c_double, C.c_int, C.c_void_p]
        lib.lp2d_oracle_iter_hist_d.argtypes = [C.c_int64] + [C.c_void_p] * 8 + [C.c_double, C.c_double,
                                                                                  C.c_int64, C.c_int64, C.c_void_p]
        lib.lp2d_oracle_bruteforce.argtypes = [C.c_void_p] * 3 + [C.c_int64] + [C.c_double] * 5 + [C.c_void_p]
        lib.lp2d_oracle_segmented_extremes.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                                       C.c_void_p, C.c_void_p]
        lib.lp2d_oracle_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_int64,
                                            C.c_void_p]
        _oracle = lib
    return _oracle


def ref_available():
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError("oracle/_ref/liblp2d_ref.so missing (build it where /root/reference exists)")
        lib = C.CDLL(REF_SO)
        lib.ref_derive_seed.restype = C.c_uint64
        lib.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.ref_xoshiro_first.argtypes = [C.c_uint64, C.c_int, C.c_void_p]
        lib.ref_shuffle.argtypes = [C.c_int64, C.c_uint64, C.c_void_p]
        lib.ref_gen.argtypes = [C.c_int64, C.c_uint64, C.c_int, C.c_double] + [C.c_void_p] * 5
        lib.ref_gen_mixed.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_uint64, C.c_int, C.c_double] + [C.c_void_p] * 7
        lib.ref_solve.argtypes = [C.c_void_p] * 4 + [C.c_int64] + [C.c_double] * 5 + [C.c_void_p] * 6
        lib.ref_bruteforce.restype = C.c_int
        lib.ref_bruteforce.argtypes = [C.c_void_p] * 3 + [C.c_int64] + [C.c_double] * 5 + [C.c_void_p] * 4
        lib.ref_batch_create.restype = C.c_void_p
        lib.ref_batch_create.argtypes = [C.c_int64] + [C.c_void_p] * 8
        lib.ref_batch_free.argtypes = [C.c_void_p]
        lib.ref_batch_solve.restype = C.c_int64
        lib.ref_batch_solve.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_uint, C.c_double, C.c_double] + [C.c_void_p] * 6
        lib.ref_batch_solve_serial_threads.restype = C.c_int64
        lib.ref_batch_solve_serial_threads.argtypes = [C.c_void_p, C.c_uint, C.c_double, C.c_double] + [C.c_void_p] * 4
        lib.ref_verify.restype = C.c_int64
        lib.ref_verify.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_int64]
        lib.ref_segmented_extremes.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
        lib.ref_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_int64, C.c_void_p]
        lib.ref_contention_ns.restype = C.c_int64
        lib.ref_contention_ns.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_uint64, C.c_int64]
        lib.ref_batch_lane_stats.restype = C.c_int
        lib.ref_batch_lane_stats.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int] + [C.c_void_p] * 3
        lib.ref_fill.restype = C.c_int
        lib.ref_fill.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_double, C.c_double] + [C.c_void_p] * 6
        lib.ref_pareto_sizes.restype = C.c_int64
        lib.ref_pareto_sizes.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_int32, C.c_int64,
                                         C.c_int64, C.c_void_p]
        _ref = lib
    return _ref


# ---- oracle wrappers -------------------------------------------------------

def derive_seed(base: int, stream: int) -> int:
    return int(oracle_lib().lp2d_oracle_derive_seed(base & (2**64 - 1), stream & (2**64 - 1)))


def shuffle(m: int, seed: int) -> np.ndarray:
    out = np.empty(m, dtype=np.uint32)
    oracle_lib().lp2d_oracle_shuffle(m, seed & (2**64 - 1), _p(out))
    return out


def xoshiro_first(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    oracle_lib().lp2d_oracle_xoshiro_first(seed, n, _p(out))
    return out


def gen(m: int, seed: int, kind: int = 0, margin: float = 1.0):
    """generate.hpp gen() restated; returns (ax, ay, b, c[2], M, witness[2])."""
    ax = np.empty(max(m, 1)); ay = np.empty(max(m, 1)); b = np.empty(max(m, 1))
    c = np.empty(2); M = np.empty(1); w = np.empty(2)
    rc = oracle_lib().lp2d_oracle_gen(m, seed & (2**64 - 1), kind, margin, _p(ax), _p(ay), _p(b), _p(c), _p(M), _p(w))
    if rc:
        raise ValueError("oracle gen failed")
    return ax[:m], ay[:m], b[:m], c, float(M[0]), w


def solve_batch(packed, eps_par=1e-12, eps_feas=1e-9, threads=1) -> np.ndarray:
    """Serial-solver restatement over a packed batch (see PackedBatch fields:
    n, offset, m, ax, ay, b, perm, c, M). fp32 or fp64 per packed.ax.dtype."""
    lib = oracle_lib()
    out = np.zeros(packed.n, dtype=RESULT_DTYPE)
    perm = np.ascontiguousarray(packed.perm, dtype=np.uint32)
    fn = lib.lp2d_oracle_solve_batch_d if packed.ax.dtype == np.float64 else lib.lp2d_oracle_solve_batch_f
    rc = fn(packed.n, _p(packed.offset), _p(packed.m), _p(packed.ax), _p(packed.ay), _p(packed.b), _p(perm),
            _p(packed.c), _p(packed.M), eps_par, eps_feas, threads, _p(out))
    if rc:
        raise ValueError("oracle: invalid permutation")
    return out


def bruteforce(ax, ay, b, c, M, eps_par=1e-12, eps_feas=1e-9):
    out = OracleResult()
    ax = np.ascontiguousarray(ax, np.float64); ay = np.ascontiguousarray(ay, np.float64); b = np.ascontiguousarray(b, np.float64)
    rc = oracle_lib().lp2d_oracle_bruteforce(_p(ax), _p(ay), _p(b), len(ax), float(c[0]), float(c[1]), float(M),
                                            eps_par, eps_feas, C.byref(out))
    if rc:
        raise ValueError("bruteforce: instance larger than the oracle cap")
    return out


# ---- contention microbenchmark (reduction.hpp, bench.hpp:244-274) ----------

def segmented_extremes(values, contention, strategy, ref=False):
    """(mins, maxs) of consecutive groups; strategy 0 serialized, 1 tree,
    2 private-then-merge. ref=True runs the compiled reference."""
    v = np.ascontiguousarray(values, np.float64)
    g = len(v) // contention if contention > 0 else 0
    mn = np.zeros(max(g, 1)); mx = np.zeros(max(g, 1))
    fn = ref_lib().ref_segmented_extremes if ref else oracle_lib().lp2d_oracle_segmented_extremes
    if fn(_p(v), len(v), contention, strategy, _p(mn), _p(mx)):
        raise ValueError("segmented_extremes: bad shape")
    return mn[:g], mx[:g]


def uniform(seed, stream, lo, hi, n, ref=False):
    out = np.zeros(n)
    fn = ref_lib().ref_uniform if ref else oracle_lib().lp2d_oracle_uniform
    fn(seed & (2**64 - 1), stream & (2**64 - 1), lo, hi, n, _p(out))
    return out


# ---- the reference's own generator / solver over packed batches ------------

class RefPacked:
    """Packed SoA batch (the product layout) built by the reference's
    generator (ref_fill), with no dependency on the product library."""

    def __init__(self, m, offset, ax, ay, b, perm, c, M):
        self.m, self.offset, self.ax, self.ay, self.b = m, offset, ax, ay, b
        self.perm, self.c, self.M = perm, c, M
        self.n = len(m)

    def astype(self, dt):
        return RefPacked(self.m, self.offset, self.ax.astype(dt), self.ay.astype(dt),
                         self.b.astype(dt), self.perm, self.c.astype(dt), self.M.astype(dt))


def pack_offsets(m):
    cap = (np.asarray(m, np.int64) + 7) // 8 * 8
    off = np.zeros(len(m) + 1, np.int64)
    off[1:] = np.cumsum(cap)
    return off


def ref_fill(m, seed, kind=None, margin=1.0, bscale=1.0, first=0):
    m = np.ascontiguousarray(m, np.int32)
    n = len(m)
    off = pack_offsets(m)
    E = int(off[-1])
    ax = np.zeros(E); ay = np.zeros(E); b = np.zeros(E)
    perm = np.zeros(E, np.uint32); c = np.zeros(2 * n); M = np.zeros(n)
    kd = None if kind is None else np.ascontiguousarray(np.broadcast_to(np.asarray(kind, np.uint8), (n,)))
    rc = ref_lib().ref_fill(n, first, seed & (2**64 - 1), _p(m), _p(off), _p(kd), margin, bscale,
                            _p(ax), _p(ay), _p(b), _p(perm), _p(c), _p(M))
    if rc:
        raise ValueError("ref_fill failed")
    return RefPacked(m, off, ax, ay, b, perm, c, M)


def ref_pareto_sizes(seed, total, xmin=8.0, alpha=1.0, xmax=8192):
    out = np.zeros(int(total // xmin) + 1, np.int32)
    k = ref_lib().ref_pareto_sizes(seed, xmin, alpha, xmax, total, len(out), _p(out))
    return out[:k]


def ref_solve_batch(packed, threads=0, block_width=512, balanced=True):
    """lp2d::solve_batch (the unmodified reference) over a packed batch; float
    storage is widened exactly (the fp32 configs' semantics). Returns
    (feasible u8, x, y, value, stats[5] = total_wu, violation_events, ...)."""
    ref = ref_lib()
    f64 = lambda a: np.ascontiguousarray(a, np.float64)
    ax, ay, b, c, M = (f64(a) for a in (packed.ax, packed.ay, packed.b, packed.c, packed.M))
    perm = np.ascontiguousarray(packed.perm, np.uint32)
    off = np.ascontiguousarray(packed.offset, np.int64)
    mm = np.ascontiguousarray(packed.m, np.int32)
    n = len(mm)
    h = ref.ref_batch_create(n, _p(off), _p(mm), _p(ax), _p(ay), _p(b), _p(perm), _p(c), _p(M))
    fe = np.zeros(n, np.uint8); x = np.zeros(n); y = np.zeros(n); v = np.zeros(n)
    st = np.zeros(5, np.uint64)
    try:
        ref.ref_batch_solve(h, block_width, 1 if balanced else 0, threads, 1e-12, 1e-9, _p(fe), _p(x),
                            _p(y), _p(v), _p(st), None)
    finally:
        ref.ref_batch_free(h)
    return fe, x, y, v, st


def iter_hist(packed, W):
    """Oracle violation histogram per (block of W LPs, insertion step)."""
    f64 = lambda a: np.ascontiguousarray(a, np.float64)
    n = packed.n
    stride = int(np.max(packed.m, initial=0)) + 1
    hist = np.zeros(((n + W - 1) // W) * stride, np.uint32)
    perm = np.ascontiguousarray(packed.perm, np.uint32)
    rc = oracle_lib().lp2d_oracle_iter_hist_d(n, _p(np.ascontiguousarray(packed.offset, np.int64)),
                                              _p(np.ascontiguousarray(packed.m, np.int32)),
                                              _p(f64(packed.ax)), _p(f64(packed.ay)), _p(f64(packed.b)),
                                              _p(perm), _p(f64(packed.c)), _p(f64(packed.M)), 1e-12, 1e-9,
                                              W, stride, _p(hist))
    if rc:
        raise ValueError("iter_hist failed")
    return hist


def ref_lane_stats(packed, W, balanced=True, record=False):
    """The unmodified reference's lane_stats (lane_wu, [total_wu,
    violation_events, masked, idle, blocks, n_iter], iteration records)."""
    ref = ref_lib()
    f64 = lambda a: np.ascontiguousarray(a, np.float64)
    ax, ay, b, c, M = (f64(a) for a in (packed.ax, packed.ay, packed.b, packed.c, packed.M))
    perm = np.ascontiguousarray(packed.perm, np.uint32)
    off = np.ascontiguousarray(packed.offset, np.int64)
    mm = np.ascontiguousarray(packed.m, np.int32)
    n = len(mm)
    h = ref.ref_batch_create(n, _p(off), _p(mm), _p(ax), _p(ay), _p(b), _p(perm), _p(c), _p(M))
    nb = (n + W - 1) // W
    lane_wu = np.zeros(nb * W, np.uint64)
    st = np.zeros(6, np.uint64)
    it = np.zeros(6 * nb * (int(mm.max(initial=0)) + 1), np.uint64) if record else None
    try:
        if ref.ref_batch_lane_stats(h, W, 1 if balanced else 0, 1 if record else 0, _p(lane_wu), _p(st),
                                    _p(it)):
            raise ValueError("ref lane stats failed")
    finally:
        ref.ref_batch_free(h)
    recs = it[:6 * int(st[5])].reshape(-1, 6) if record else None
    return lane_wu, st, recs


def ref_bruteforce(ax, ay, b, c, M, eps_par=1e-12, eps_feas=1e-9):
    """The unmodified reference's solve_bruteforce (oracle.hpp:38-70, vertex
    enumeration, m <= 512): (feasible, x, y, value)."""
    ax = np.ascontiguousarray(ax, np.float64); ay = np.ascontiguousarray(ay, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    fe = np.zeros(1, np.uint8); x = np.zeros(1); y = np.zeros(1); v = np.zeros(1)
    rc = ref_lib().ref_bruteforce(_p(ax), _p(ay), _p(b), len(ax), float(c[0]), float(c[1]), float(M),
                                  eps_par, eps_feas, _p(fe), _p(x), _p(y), _p(v))
    if rc:
        raise ValueError("ref_bruteforce failed")
    return bool(fe[0]), float(x[0]), float(y[0]), float(v[0])
