"""ctypes binding of the product library lib/liblp2d_b200.so (include/*.h).

The library is built in-tree by `make -C paper_1902_04995_b200/csrc` (see
__graft_entry__.build). There is no CPU fallback: if the library is missing
or no CUDA device is visible, solving raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# LP2D_B200_LIB overrides the in-tree build (A/B experiments of kernel variants).
LIB_PATH = os.environ.get("LP2D_B200_LIB", os.path.join(_HERE, "lib", "liblp2d_b200.so"))
CSRC = os.path.join(_HERE, "csrc")

# include/lp2d_b200.h
LP2D_OK = 0
ERR_EMPTY_BATCH = -1
ERR_PERM_COUNT = -2
ERR_PERM_LENGTH = -3
ERR_BLOCK_WIDTH = -4
ERR_LAYOUT = -5
ERR_BAD_PERM = -6
ERR_ARG = -7
ERR_UNSUPPORTED = -8
ERR_CUDA = -9

OPTIMAL, INFEASIBLE, UNBOUNDED, INVALID = 0, 1, 2, 255
PAIR_NONE = -(2**31)
MEM_HOST, MEM_DEVICE = 0, 1
SCHED_NAIVE, SCHED_BALANCED = 0, 1

GEN_FEASIBLE, GEN_INFEASIBLE, GEN_UNBOUNDED = 0, 1, 3
(REDUCE_SHARED_ATOMIC, REDUCE_TREE, REDUCE_PRIVATE_MERGE, REDUCE_GLOBAL_ATOMIC,
 REDUCE_CUB) = range(5)


class BatchSoA(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("m", C.c_void_p),
        ("offset", C.c_void_p),
        ("ax", C.c_void_p),
        ("ay", C.c_void_p),
        ("b", C.c_void_p),
        ("perm", C.c_void_p),
        ("perm_bits", C.c_int32),
        ("mem", C.c_int32),
        ("c", C.c_void_p),
        ("bound_m", C.c_void_p),
        ("max_m", C.c_int64),
        ("min_m", C.c_int64),
        ("perm_from_seed", C.c_int32),
        ("perm_mul", C.c_int32),
        ("perm_add", C.c_int32),
        ("_pad", C.c_int32),
        ("perm_seed", C.c_uint64),
        ("perm_first", C.c_int64),
    ]


class Opts(C.Structure):
    _fields_ = [
        ("scheduler", C.c_int32),
        ("block_width", C.c_int32),
        ("n_gpus", C.c_int32),
        ("device", C.c_int32),
        ("stream", C.c_void_p),
        ("eps_parallel", C.c_double),
        ("eps_feas", C.c_double),
    ]


class Out(C.Structure):
    _fields_ = [
        ("status", C.c_void_p),
        ("x", C.c_void_p),
        ("y", C.c_void_p),
        ("value", C.c_void_p),
        ("pair", C.c_void_p),
        ("violation_events", C.c_void_p),
        ("work_units", C.c_void_p),
        ("iter_hist", C.c_void_p),
    ]


# Every symbol include/lp2d_b200.h and include/lp2d_b200_gen.h declare.
EXPORTS = (
    "lp2dgpu_default_opts",
    "lp2dgpu_solve_f32",
    "lp2dgpu_solve_f64",
    "lp2dgpu_pack_offsets",
    "lp2dgpu_partition",
    "lp2dgpu_shuffle_device",
    "lp2dgpu_generate_device",
    "lp2dgpu_device_count",
    "lp2dgpu_fx_stats",
    "lp2dgpu_kernel_launches",
    "lp2dgpu_segmented_extremes",
    "lp2dgpu_last_error",
    "lp2dgpu_version",
    "lp2dgen_derive_seed",
    "lp2dgen_shuffle",
    "lp2dgen_gen",
    "lp2dgen_fill",
    "lp2dgen_pareto_sizes",
    "lp2dgen_uniform",
)

_lib = None


def build(verbose: bool = False) -> None:
    import subprocess

    subprocess.run(["make", "-s", "-C", CSRC], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)


def lib():
    """Load the library (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `make -C {CSRC}` "
            "(the solver has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.lp2dgpu_default_opts.argtypes = [C.POINTER(Opts)]
    for name in ("lp2dgpu_solve_f32", "lp2dgpu_solve_f64"):
        fn = getattr(L, name)
        fn.argtypes = [C.POINTER(BatchSoA), C.POINTER(Opts), C.POINTER(Out)]
        fn.restype = C.c_int
    L.lp2dgpu_pack_offsets.argtypes = [C.c_int64, C.c_void_p, C.c_void_p]
    L.lp2dgpu_pack_offsets.restype = C.c_int64
    if hasattr(L, "lp2dgpu_partition"):
        L.lp2dgpu_partition.argtypes = [C.c_int64, C.c_void_p, C.c_int32, C.c_void_p]
        L.lp2dgpu_partition.restype = C.c_int
    L.lp2dgpu_shuffle_device.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
    L.lp2dgpu_shuffle_device.restype = C.c_int
    L.lp2dgpu_generate_device.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                          C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                          C.c_int32, C.c_void_p]
    L.lp2dgpu_generate_device.restype = C.c_int
    L.lp2dgpu_device_count.restype = C.c_int
    L.lp2dgpu_fx_stats.argtypes = [C.c_void_p, C.c_int]
    L.lp2dgpu_fx_stats.restype = C.c_int
    L.lp2dgpu_kernel_launches.restype = C.c_uint64
    L.lp2dgpu_segmented_extremes.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int32,
                                             C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
    L.lp2dgpu_segmented_extremes.restype = C.c_int
    L.lp2dgpu_last_error.restype = C.c_char_p
    L.lp2dgpu_version.restype = C.c_char_p
    L.lp2dgen_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_int64,
                                  C.c_void_p]
    L.lp2dgen_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
    L.lp2dgen_derive_seed.restype = C.c_uint64
    L.lp2dgen_shuffle.argtypes = [C.c_int64, C.c_uint64, C.c_void_p]
    L.lp2dgen_gen.argtypes = [C.c_int64, C.c_uint64, C.c_int, C.c_double] + [C.c_void_p] * 5
    L.lp2dgen_gen.restype = C.c_int
    L.lp2dgen_fill.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_double, C.c_double] + [C.c_void_p] * 6 + [C.c_int]
    L.lp2dgen_fill.restype = C.c_int
    L.lp2dgen_pareto_sizes.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_int32,
                                       C.c_int64, C.c_int64, C.c_void_p]
    L.lp2dgen_pareto_sizes.restype = C.c_int64
    _lib = L
    return L


def last_error() -> str:
    return lib().lp2dgpu_last_error().decode()
