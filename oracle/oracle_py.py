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
