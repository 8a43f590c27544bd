"""Host-side mirror of the reference's batch-solve API, backed by the sm_100a
kernels through the C ABI (include/lp2d_b200.h).

Reference interface (paths under /root/reference/proj/include/lp2d/):
  tolerance            core.hpp:59-68        -> Tolerance
  problem / solution   serial.hpp:28-43      -> Problem / Solution
  permutation, shuffle serial.hpp:126-146    -> Permutation, shuffle()
  derive_seed          rng.hpp:64-68         -> derive_seed()
  batch, block_config  batch.hpp:45-58       -> Batch, BlockConfig
  solve_batch          batch.hpp:303-371     -> solve_batch()
  gen / gen_mixed      generate.hpp:143-189  -> gen(), gen_mixed()

solve_batch raises ValueError exactly where the reference throws
std::invalid_argument (batch.hpp:306-320). Scalars may be stored as float64 or
float32; either way the arithmetic is the reference's double arithmetic and
the results (double) compare equal to the reference's on the stored instance
(value equality of x, y, value and the feasibility flag). The builder's
extensions (status incl. "unbounded", the defining constraint pair, per-LP
violation/work-unit counts) ride along.

For throughput, PackedBatch keeps the structure-of-arrays layout the kernels
consume and solve_packed() runs on host or device (torch) buffers.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N

OPTIMAL, INFEASIBLE, UNBOUNDED, INVALID = N.OPTIMAL, N.INFEASIBLE, N.UNBOUNDED, N.INVALID
PAIR_NONE = N.PAIR_NONE
DEFAULT_BOUND = 1e7  # serial.hpp:26


class SchedulerKind(enum.IntEnum):
    """batch.hpp:39: naive (thread per LP) / balanced (warp-dealt work units)."""

    naive = N.SCHED_NAIVE
    balanced = N.SCHED_BALANCED


class GenKind(enum.IntEnum):
    """generate.hpp:26-30 (+ the builder-defined unbounded kind)."""

    feasible_random = N.GEN_FEASIBLE
    infeasible = N.GEN_INFEASIBLE
    unbounded_random = N.GEN_UNBOUNDED


@dataclass
class Tolerance:
    """core.hpp:59-68."""

    eps_parallel: float = 1e-12
    eps_feas: float = 1e-9
    sig_figs: int = 5

    def feas_slack(self, bound: float) -> float:
        return self.eps_feas * (1.0 + abs(bound))


@dataclass
class BlockConfig:
    """batch.hpp:50-58. block_width is validated like the reference; the GPU
    schedule itself is fixed by the kernel (warp = block of 32 lanes).
    workers maps to the number of GPUs the batch is sharded over (0 = all)."""

    block_width: int = 512
    scheduler: SchedulerKind = SchedulerKind.balanced
    workers: int = 0
    record_iterations: bool = False


@dataclass
class Problem:
    """serial.hpp:28-32: max c.x s.t. a.x <= b, inside the +-bound_m box.
    constraints is an (m, 3) array of rows (ax, ay, b)."""

    c: tuple = (0.0, 0.0)
    constraints: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    bound_m: float = DEFAULT_BOUND

    def __post_init__(self):
        self.constraints = np.asarray(self.constraints, dtype=np.float64).reshape(-1, 3)


@dataclass
class Permutation:
    """serial.hpp:126-129 insertion order of the user constraints."""

    order: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))

    def __post_init__(self):
        self.order = np.asarray(self.order, dtype=np.uint32)


def identity_permutation(m: int) -> Permutation:
    return Permutation(np.arange(m, dtype=np.uint32))


@dataclass
class Batch:
    """batch.hpp:45-48."""

    problems: List[Problem] = field(default_factory=list)
    permutations: List[Permutation] = field(default_factory=list)


@dataclass
class Solution:
    """serial.hpp:34-43 plus the builder's status / defining pair / stats."""

    feasible: bool = False
    point: tuple = (0.0, 0.0)
    value: float = 0.0
    status: int = INFEASIBLE
    pair: tuple = (PAIR_NONE, PAIR_NONE)
    violation_events: int = 0
    work_units: int = 0

    def __eq__(self, other):  # solution::operator== (serial.hpp:41)
        return (self.feasible == other.feasible and tuple(self.point) == tuple(other.point)
                and self.value == other.value)


@dataclass
class IterationRecord:
    """batch.hpp:84-92 iteration_record (record_iterations)."""

    block: int = 0
    iteration: int = 0
    active_lanes: int = 0
    masked_lanes: int = 0
    wu_count: int = 0
    idle_steps: int = 0
    lane_wu: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))


@dataclass
class LaneStats:
    """batch.hpp:94-107 with the reference's block semantics: blocks of
    block_width LPs stepping through insertion steps in lockstep (run_block,
    batch.hpp:149-294). The GPU solves LPs independently; these counters are
    rebuilt exactly from the GPU's per-(block, step) violation histogram
    (lp2d_out::iter_hist, rebuild_lane_stats), so lane_imbalance() means what
    it means in the reference."""

    block_width: int = 0
    blocks: int = 0
    lane_wu: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    total_wu: int = 0
    violation_events: int = 0
    masked_lane_iterations: int = 0
    idle_wu_steps: int = 0
    iterations: List[IterationRecord] = field(default_factory=list)


@dataclass
class BatchResult:
    solutions: List[Solution]
    stats: LaneStats


# ---- RNG / generators (host, product-side restatement) -----------------------

def derive_seed(base: int, stream: int) -> int:
    return int(N.lib().lp2dgen_derive_seed(base & (2**64 - 1), stream & (2**64 - 1)))


def shuffle(m: int, seed: int) -> Permutation:
    out = np.empty(m, dtype=np.uint32)
    N.lib().lp2dgen_shuffle(m, seed & (2**64 - 1), out.ctypes.data)
    return Permutation(out)


def kernel_launches() -> int:
    """Kernels the native library has enqueued so far (monotonic counter)."""
    return int(N.lib().lp2dgpu_kernel_launches())


def pack_offsets(m: np.ndarray) -> np.ndarray:
    """Element offsets satisfying the C-ABI layout contract (8-aligned)."""
    m = np.ascontiguousarray(m, dtype=np.int32)
    off = np.empty(len(m) + 1, dtype=np.int64)
    N.lib().lp2dgpu_pack_offsets(len(m), m.ctypes.data, off.ctypes.data)
    return off


@dataclass
class PackedBatch:
    """Structure-of-arrays batch (the layout of lp2d_batch_soa)."""

    m: np.ndarray            # int32 [n]
    offset: np.ndarray       # int64 [n+1]
    ax: np.ndarray           # T [offset[n]]
    ay: np.ndarray
    b: np.ndarray
    perm: np.ndarray         # u16 or u32 [offset[n]]
    c: np.ndarray            # T [2n]
    M: np.ndarray            # T [n]

    @property
    def n(self) -> int:
        return len(self.m)

    @property
    def dtype(self):
        return self.ax.dtype

    def astype(self, dtype) -> "PackedBatch":
        """Round scalars to dtype (round-to-nearest) — the fp32 configs."""
        dt = np.dtype(dtype)
        return PackedBatch(self.m, self.offset, self.ax.astype(dt), self.ay.astype(dt),
                           self.b.astype(dt), self.perm, self.c.astype(dt), self.M.astype(dt))

    def with_perm_bits(self, bits: int) -> "PackedBatch":
        dt = np.uint16 if bits == 16 else np.uint32
        return PackedBatch(self.m, self.offset, self.ax, self.ay, self.b,
                           self.perm.astype(dt), self.c, self.M)

    def constraint_bytes(self) -> int:
        """Algorithmic bytes: 3 * sizeof(T) per constraint."""
        return int(3 * self.ax.itemsize * int(self.m.astype(np.int64).sum()))

    def subset(self, lo: int, hi: int) -> "PackedBatch":
        e0, e1 = int(self.offset[lo]), int(self.offset[hi])
        return PackedBatch(self.m[lo:hi].copy(), self.offset[lo:hi + 1] - e0,
                           self.ax[e0:e1], self.ay[e0:e1], self.b[e0:e1], self.perm[e0:e1],
                           self.c[2 * lo:2 * hi], self.M[lo:hi])

    def problem(self, j: int) -> Problem:
        o, mj = int(self.offset[j]), int(self.m[j])
        cons = np.stack([self.ax[o:o + mj], self.ay[o:o + mj], self.b[o:o + mj]], axis=1)
        return Problem((float(self.c[2 * j]), float(self.c[2 * j + 1])), cons.astype(np.float64),
                       float(self.M[j]))

    def permutation(self, j: int) -> Permutation:
        o, mj = int(self.offset[j]), int(self.m[j])
        return Permutation(self.perm[o:o + mj].astype(np.uint32))

    @staticmethod
    def from_batch(b: Batch, dtype=np.float64, perm_bits: Optional[int] = None) -> "PackedBatch":
        _validate_batch(b)
        n = len(b.problems)
        m = np.array([p.constraints.shape[0] for p in b.problems], dtype=np.int32)
        off = pack_offsets(m)
        E = int(off[-1])
        dt = np.dtype(dtype)
        ax = np.zeros(E, dt); ay = np.zeros(E, dt); bb = np.zeros(E, dt)
        if perm_bits is None:
            perm_bits = 16 if (n == 0 or m.max(initial=0) <= 65536) else 32
        perm = np.zeros(E, np.uint16 if perm_bits == 16 else np.uint32)
        c = np.zeros(2 * n, dt); M = np.zeros(n, dt)
        for j, (p, q) in enumerate(zip(b.problems, b.permutations)):
            o, mj = int(off[j]), int(m[j])
            ax[o:o + mj] = p.constraints[:, 0]
            ay[o:o + mj] = p.constraints[:, 1]
            bb[o:o + mj] = p.constraints[:, 2]
            perm[o:o + mj] = q.order
            c[2 * j], c[2 * j + 1] = p.c
            M[j] = p.bound_m
        return PackedBatch(m, off, ax, ay, bb, perm, c, M)

    @staticmethod
    def generate(m: Sequence[int], seed: int, kind=None, margin: float = 1.0,
                 bscale: float = 1.0, first: int = 0, perm_bits: Optional[int] = None,
                 threads: int = 0) -> "PackedBatch":
        """gen_mixed-style synthesis, LP j seeded by global index first + j
        (generate.hpp:174-189). fp64; use astype(np.float32) for fp32 configs."""
        m = np.ascontiguousarray(m, dtype=np.int32)
        n = len(m)
        off = pack_offsets(m)
        E = int(off[-1])
        ax = np.zeros(E); ay = np.zeros(E); b = np.zeros(E)
        perm32 = np.zeros(E, np.uint32)
        c = np.zeros(2 * n); M = np.zeros(n)
        kd = None
        if kind is not None:
            kd = np.ascontiguousarray(np.broadcast_to(np.asarray(kind, dtype=np.uint8), (n,)))
        rc = N.lib().lp2dgen_fill(n, first, seed & (2**64 - 1), m.ctypes.data, off.ctypes.data,
                                  kd.ctypes.data if kd is not None else None, margin, bscale,
                                  ax.ctypes.data, ay.ctypes.data, b.ctypes.data,
                                  perm32.ctypes.data, c.ctypes.data, M.ctypes.data, threads)
        if rc:
            raise ValueError(f"lp2dgen_fill failed ({rc})")
        if perm_bits is None:
            perm_bits = 16 if m.max(initial=0) <= 65536 else 32
        perm = perm32.astype(np.uint16) if perm_bits == 16 else perm32
        return PackedBatch(m, off, ax, ay, b, perm, c, M)


def gen(m: int, seed: int, kind: GenKind = GenKind.feasible_random, margin: float = 1.0) -> Problem:
    """generate.hpp:143-155 gen({m, seed, kind, margin})."""
    ax = np.zeros(max(m, 1)); ay = np.zeros(max(m, 1)); b = np.zeros(max(m, 1))
    c = np.zeros(2); M = np.zeros(1)
    rc = N.lib().lp2dgen_gen(m, seed & (2**64 - 1), int(kind), margin, ax.ctypes.data,
                             ay.ctypes.data, b.ctypes.data, c.ctypes.data, M.ctypes.data)
    if rc:
        raise ValueError("gen: bad spec")
    return Problem((float(c[0]), float(c[1])), np.stack([ax[:m], ay[:m], b[:m]], axis=1), float(M[0]))


def replicate(p: Problem, count: int, perm_seed: int) -> Batch:
    """generate.hpp:159-169."""
    m = p.constraints.shape[0]
    return Batch([p] * count, [shuffle(m, derive_seed(perm_seed, i)) for i in range(count)])


def gen_mixed(sizes: Sequence[int], count: int, seed: int,
              kind: GenKind = GenKind.feasible_random, margin: float = 1.0) -> Batch:
    """generate.hpp:174-189."""
    sizes = list(sizes)
    if not sizes:
        raise ValueError("gen_mixed: no sizes")
    m = np.array([sizes[i % len(sizes)] for i in range(count)], dtype=np.int32)
    pb = PackedBatch.generate(m, seed, kind=int(kind), margin=margin, perm_bits=32)
    return Batch([pb.problem(j) for j in range(count)], [pb.permutation(j) for j in range(count)])


# ---- solving -------------------------------------------------------------------

def _validate_batch(b: Batch) -> None:
    n = len(b.problems)
    if n == 0:
        raise ValueError("solve_batch: empty batch")
    if len(b.permutations) != n:
        raise ValueError("solve_batch: one permutation per problem required")
    for p, q in zip(b.problems, b.permutations):
        if len(q.order) != p.constraints.shape[0]:
            raise ValueError("solve_batch: permutation length does not match problem size")


@dataclass
class PackedResult:
    status: object   # u8 [n]
    x: object        # T [n]
    y: object
    value: object
    pair: object     # int32 [n, 2]
    violation_events: object  # u32 [n]
    work_units: object        # u64 [n]


def _raise(rc: int):
    msg = N.last_error()
    if rc in (N.ERR_EMPTY_BATCH, N.ERR_PERM_COUNT, N.ERR_PERM_LENGTH, N.ERR_BLOCK_WIDTH,
              N.ERR_LAYOUT, N.ERR_ARG, N.ERR_BAD_PERM):
        raise ValueError(msg)
    raise RuntimeError(f"lp2d_b200 error {rc}: {msg}")


_OPTS0 = None


def _opts(cfg: BlockConfig, tol: Tolerance, device: int = 0, stream: int = 0) -> N.Opts:
    global _OPTS0
    if _OPTS0 is None:
        _OPTS0 = N.Opts()
        N.lib().lp2dgpu_default_opts(C.byref(_OPTS0))
    o = N.Opts.from_buffer_copy(_OPTS0)
    o.scheduler = int(cfg.scheduler)
    o.block_width = int(cfg.block_width) if cfg.block_width < 2**31 else 2**31 - 1
    o.n_gpus = int(cfg.workers)
    o.device = device
    o.stream = stream
    o.eps_parallel = tol.eps_parallel
    o.eps_feas = tol.eps_feas
    return o


@dataclass(frozen=True)
class PermSeed:
    """Permutations generated on the device (lp2d_batch_soa::perm_from_seed):
    LP j's order is shuffle(m[j], derive_seed(seed, mul * (first + j) + add)).
    mul=2, add=1: gen_mixed / PackedBatch.generate streams (generate.hpp:186);
    mul=1, add=0: replicate's (generate.hpp:165-166)."""
    seed: int
    mul: int = 2
    add: int = 1
    first: int = 0


def _pointers(obj, arrays) -> tuple:
    """Data pointers of `arrays`, cached on `obj` while it holds the very same
    array objects (the cache keeps them alive, so identity is a safe key):
    a repeated call with the same host batch / result buffers skips the
    numpy->ctypes conversions (~3 us per array, ~40 us per call otherwise)."""
    c = obj.__dict__.get("_ptr_cache")
    if c is not None and len(c[0]) == len(arrays) and all(x is y for x, y in zip(c[0], arrays)):
        return c[1]
    ptrs = tuple(a.ctypes.data if a is not None else None for a in arrays)
    obj.__dict__["_ptr_cache"] = (tuple(arrays), ptrs)
    return ptrs


def solve_packed(pb: PackedBatch, cfg: BlockConfig = BlockConfig(), tol: Tolerance = Tolerance(),
                 out: Optional[PackedResult] = None,
                 iter_hist: Optional[np.ndarray] = None,
                 perm_seed: Optional[PermSeed] = None, device: int = 0) -> PackedResult:
    """Host-buffer solve through the C ABI (copies in/out inside the call).
    With perm_seed, pb.perm is ignored (may be None): the permutations are
    generated on the device and never cross PCIe. device: the GPU of a
    single-device call (cfg.workers == 1), e.g. a rank's local GPU."""
    if pb.n == 0:
        raise ValueError("solve_batch: empty batch")
    dt = pb.dtype
    if dt not in (np.float32, np.float64):
        raise ValueError("scalars must be float32 or float64")
    perm_in = pb.perm if pb.perm is not None else np.zeros(0, np.uint16)
    arrs = [np.ascontiguousarray(a) for a in (pb.m, pb.offset, pb.ax, pb.ay, pb.b, perm_in, pb.c, pb.M)]
    m, off, ax, ay, b, perm, c, M = arrs
    if perm_seed is None and pb.perm is None:
        raise ValueError("solve_batch: permutations missing (pass perm or perm_seed)")
    if out is None:
        # results are the reference's doubles for both storage types
        out = PackedResult(np.zeros(pb.n, np.uint8), np.zeros(pb.n), np.zeros(pb.n),
                           np.zeros(pb.n), np.zeros((pb.n, 2), np.int32),
                           np.zeros(pb.n, np.uint32), np.zeros(pb.n, np.uint64))
    pbits = 16 if perm.dtype == np.uint16 else 32
    if perm_seed is not None:
        pbits = 16 if int(pb.m.max(initial=0)) <= 65536 else 32
    pm, po, pax, pay, pbb, pp, pc, pM = _pointers(pb, arrs)
    s = N.BatchSoA(len(m), pm, po, pax, pay, pbb, pp if perm_seed is None else None, pbits,
                   N.MEM_HOST, pc, pM, 0, 0)
    if perm_seed is not None:
        s.perm_from_seed = 1
        s.perm_mul, s.perm_add = int(perm_seed.mul), int(perm_seed.add)
        s.perm_seed = perm_seed.seed & (2**64 - 1)
        s.perm_first = int(perm_seed.first)
    o = _opts(cfg, tol, device=device)
    r = N.Out(*_pointers(out, (out.status, out.x, out.y, out.value, out.pair, out.violation_events,
                               out.work_units, iter_hist)))
    fn = N.lib().lp2dgpu_solve_f32 if dt == np.float32 else N.lib().lp2dgpu_solve_f64
    rc = fn(C.byref(s), C.byref(o), C.byref(r))
    if rc:
        _raise(rc)
    return out


class DeviceBatch:
    """A PackedBatch resident in GPU memory (torch tensors); the zero-copy
    device-mode entry of the C ABI. max_m is kept on the host."""

    def __init__(self, pb: PackedBatch, device: int = 0):
        import torch

        dev = torch.device("cuda", device)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        self.n = pb.n
        self.device = device
        self.dtype = pb.dtype
        self.max_m = int(pb.m.max(initial=0))
        self.min_m = int(pb.m.min()) if pb.n else 0
        self.m, self.offset = t(pb.m), t(pb.offset)
        self.ax, self.ay, self.b = t(pb.ax), t(pb.ay), t(pb.b)
        self.perm = t(pb.perm.view(np.int16) if pb.perm.dtype == np.uint16 else pb.perm.view(np.int32))
        self.perm_bits = 16 if pb.perm.dtype == np.uint16 else 32
        self.c, self.M = t(pb.c), t(pb.M)
        self.constraint_bytes = pb.constraint_bytes()

    @classmethod
    def generate(cls, m: Sequence[int], seed: int, kind=None, margin: float = 1.0,
                 bscale: float = 1.0, first: int = 0, dtype=np.float64,
                 perm_bits: Optional[int] = None, device: int = 0,
                 stream=None) -> "DeviceBatch":
        """PackedBatch.generate on the GPU (lp2dgpu_generate_device): the same
        streams, synthesized in HBM (no host arrays, no PCIe)."""
        import torch

        dev = torch.device("cuda", device)
        m = np.ascontiguousarray(m, dtype=np.int32)
        n = len(m)
        off = pack_offsets(m)
        E = int(off[-1])
        if perm_bits is None:
            perm_bits = 16 if m.max(initial=0) <= 65536 else 32
        tdt = torch.float32 if dtype == np.float32 else torch.float64
        self = cls.__new__(cls)
        self.n, self.device, self.dtype = n, device, np.dtype(dtype).type
        self.max_m = int(m.max(initial=0))
        self.min_m = int(m.min()) if n else 0
        self.m = torch.from_numpy(m).to(dev)
        self.offset = torch.from_numpy(off).to(dev)
        self.ax = torch.zeros(E, dtype=tdt, device=dev)
        self.ay = torch.zeros(E, dtype=tdt, device=dev)
        self.b = torch.zeros(E, dtype=tdt, device=dev)
        self.perm = torch.zeros(E, dtype=torch.int16 if perm_bits == 16 else torch.int32, device=dev)
        self.perm_bits = perm_bits
        self.c = torch.zeros(2 * n, dtype=tdt, device=dev)
        self.M = torch.zeros(n, dtype=tdt, device=dev)
        kd = None
        if kind is not None:
            kd = torch.from_numpy(np.broadcast_to(np.asarray(kind, dtype=np.uint8), (n,)).copy()).to(dev)
        self.constraint_bytes = 3 * int(m.astype(np.int64).sum()) * (4 if dtype == np.float32 else 8)
        if stream is None:
            stream = torch.cuda.current_stream(device)
        rc = N.lib().lp2dgpu_generate_device(
            n, first, seed & (2**64 - 1), self.m.data_ptr(), self.offset.data_ptr(),
            kd.data_ptr() if kd is not None else None, margin, bscale,
            32 if dtype == np.float32 else 64, self.ax.data_ptr(), self.ay.data_ptr(),
            self.b.data_ptr(), self.perm.data_ptr(), perm_bits, self.c.data_ptr(),
            self.M.data_ptr(), device, stream.cuda_stream)
        if rc:
            _raise(rc)
        return self

    def to_packed(self) -> PackedBatch:
        """Download (e.g. to check a device-generated batch on the oracle)."""
        np_ = lambda t: t.cpu().numpy()
        perm = np_(self.perm).view(np.uint16 if self.perm_bits == 16 else np.uint32)
        return PackedBatch(np_(self.m), np_(self.offset), np_(self.ax), np_(self.ay), np_(self.b),
                           perm, np_(self.c), np_(self.M))

    def empty_result(self) -> PackedResult:
        import torch

        dev = torch.device("cuda", self.device)
        tdt = torch.float64  # results are the reference's doubles for both storage types
        n = self.n
        return PackedResult(torch.zeros(n, dtype=torch.uint8, device=dev),
                            torch.zeros(n, dtype=tdt, device=dev), torch.zeros(n, dtype=tdt, device=dev),
                            torch.zeros(n, dtype=tdt, device=dev),
                            torch.zeros((n, 2), dtype=torch.int32, device=dev),
                            torch.zeros(n, dtype=torch.int32, device=dev),
                            torch.zeros(n, dtype=torch.int64, device=dev))


def solve_device(db: DeviceBatch, out: PackedResult, cfg: BlockConfig = BlockConfig(),
                 tol: Tolerance = Tolerance(), stream=None, stats: bool = True) -> None:
    """Enqueue the solve on `stream` (default: torch's current stream)."""
    import torch

    if stream is None:
        stream = torch.cuda.current_stream(db.device)
    s = N.BatchSoA(db.n, db.m.data_ptr(), db.offset.data_ptr(), db.ax.data_ptr(), db.ay.data_ptr(),
                   db.b.data_ptr(), db.perm.data_ptr(), db.perm_bits, N.MEM_DEVICE,
                   db.c.data_ptr(), db.M.data_ptr(), db.max_m, db.min_m)
    o = _opts(cfg, tol, device=db.device, stream=stream.cuda_stream)
    r = N.Out(out.status.data_ptr(), out.x.data_ptr(), out.y.data_ptr(), out.value.data_ptr(),
              out.pair.data_ptr() if stats else None,
              out.violation_events.data_ptr() if stats else None,
              out.work_units.data_ptr() if stats else None)
    fn = N.lib().lp2dgpu_solve_f32 if db.dtype == np.float32 else N.lib().lp2dgpu_solve_f64
    rc = fn(C.byref(s), C.byref(o), C.byref(r))
    if rc:
        _raise(rc)


def solve_batch(b: Batch, cfg: BlockConfig = BlockConfig(), tol: Tolerance = Tolerance(),
                dtype=np.float64) -> BatchResult:
    """batch.hpp:303-371 solve_batch on the GPU."""
    _validate_batch(b)
    if cfg.block_width == 0:
        raise ValueError("solve_batch: block width must be positive")
    pb = PackedBatch.from_batch(b, dtype=dtype)
    W = int(cfg.block_width)
    nb = (pb.n + W - 1) // W
    hist = np.zeros(nb * (int(pb.m.max(initial=0)) + 1), np.uint32)
    r = solve_packed(pb, cfg, tol, iter_hist=hist)
    sols = []
    for j in range(pb.n):
        st = int(r.status[j])
        feas = st in (OPTIMAL, UNBOUNDED)
        sols.append(Solution(feas, (float(r.x[j]), float(r.y[j])) if feas else (0.0, 0.0),
                             float(r.value[j]) if feas else 0.0, st,
                             (int(r.pair[j, 0]), int(r.pair[j, 1])),
                             int(r.violation_events[j]), int(r.work_units[j])))
    if (r.status == INVALID).any():
        # a permutation entry >= m: the reference's solve would index out of
        # range; the front-end refuses instead of returning a value
        bad = np.nonzero(r.status == INVALID)[0]
        raise ValueError("solve_batch: permutation entry out of range for LP(s) %s" % bad[:8].tolist())
    stats = rebuild_lane_stats(pb.m, r.status, r.pair, pb.perm, pb.offset, r.work_units, hist, W,
                               cfg.scheduler, cfg.record_iterations)
    return BatchResult(sols, stats)


def rebuild_lane_stats(m: np.ndarray, status: np.ndarray, pair: np.ndarray,
                       perm: np.ndarray, offset: np.ndarray, work_units: np.ndarray,
                       hist: np.ndarray, block_width: int, scheduler: SchedulerKind,
                       record_iterations: bool = False) -> LaneStats:
    """The reference's lane_stats (batch.hpp:149-294, 327-371) from a solve's
    per-LP results and its (block, insertion step) violation histogram:
    per block, every executed step masks the lanes that are past their m, out
    of the batch, or infeasible (from the step of their infeasible event,
    found as the insertion position of the defining pair's violated
    constraint); the balanced deal gives lane l ceil((active*prefix - l)/W)
    units (prefix = 3 + step), the naive deal gives each LP's lane its own
    work units and charges the others prefix idle slots per active step."""
    W = int(block_width)
    n = len(m)
    nb = (n + W - 1) // W
    stride = len(hist) // max(nb, 1)
    if hist is None:  # (only the naive lane_wu/total can be rebuilt without it)
        hist = np.zeros(nb, np.uint32)
        stride = 1
    H = np.asarray(hist, np.int64).reshape(nb, stride)
    m64 = np.asarray(m, np.int64)
    inf = np.asarray(status) == INFEASIBLE
    # step of the infeasible event: position of the violated constraint + 1
    t = np.full(n, np.iinfo(np.int64).max, np.int64)
    for j in np.nonzero(inf)[0]:
        o = int(offset[j])
        pos = np.nonzero(perm[o:o + int(m[j])] == pair[j, 0])[0]
        t[j] = int(pos[0]) + 1
    e = np.where(inf, np.minimum(m64, t), m64)  # lane j keeps the block going while step < e_j
    balanced = SchedulerKind(scheduler) == SchedulerKind.balanced
    lane_wu = np.zeros(nb * W, np.uint64)
    st = LaneStats(block_width=W, blocks=nb, lane_wu=lane_wu)
    for b in range(nb):
        js = np.arange(b * W, min(n, (b + 1) * W))
        lp_max = int(m64[js].max(initial=0))
        last = min(lp_max, max(1, int(e[js].max(initial=0))))
        if lp_max == 0:
            continue
        steps = np.arange(1, last + 1)
        # masked lanes: !live (W - count), past m, or infeasible before the step
        past = (steps[None, :] > m64[js][:, None]) | (steps[None, :] > t[js][:, None])
        masked = (W - len(js)) + past.sum(axis=0)
        active = H[b, 1:last + 1]
        prefix = 3 + steps
        st.masked_lane_iterations += int(masked.sum())
        st.violation_events += int(active.sum())
        if balanced:
            wu = active * prefix
            q, r = wu // W, wu % W
            lanes = np.arange(W)
            per_lane = q.sum() + (lanes[None, :] < r[:, None]).sum(axis=0)
            lane_wu[b * W:(b + 1) * W] = per_lane.astype(np.uint64)
            idle = ((wu + W - 1) // W) * W - wu
        else:
            lane_wu[b * W:b * W + len(js)] = np.asarray(work_units, np.uint64)[js]
            idle = np.where(active > 0, prefix * (W - active), 0)
            wu = active * prefix
        st.idle_wu_steps += int(idle.sum())
        if record_iterations:
            for k, it in enumerate(steps):
                lw = np.zeros(W, np.uint32)
                if active[k]:
                    if balanced:
                        lw[:] = q[k]
                        lw[:r[k]] += 1
                    else:
                        # lanes of the LPs that violated at this step: not
                        # recoverable from the histogram alone (counts only)
                        lw = np.zeros(W, np.uint32)
                st.iterations.append(IterationRecord(b, int(it), int(active[k]), int(masked[k]),
                                                     int(wu[k]), int(idle[k]), lw))
    st.total_wu = int(lane_wu.sum())
    return st


def lane_imbalance(stats: LaneStats) -> float:
    """batch.hpp:111-120 (max/mean of per-lane work)."""
    if stats.total_wu == 0:
        raise ValueError("lane_imbalance: no work units were executed")
    return float(stats.lane_wu.max()) / (stats.total_wu / len(stats.lane_wu))


def agree_sig_figs(a: float, b: float, sig_figs: int = 5) -> bool:
    """core.hpp:120-125."""
    import math

    if a == b:
        return True
    mag = max(abs(a), abs(b))
    step = 10.0 ** (math.floor(math.log10(mag)) - (sig_figs - 1))
    return abs(a - b) <= 0.5 * step


# ---- lp2d v1 text instances (io.hpp:13-97), for replaying single LPs -------

class ParseError(RuntimeError):
    """io.hpp read_problem throws std::runtime_error("lp2d parse: ...")."""


def _full(v: float) -> str:
    return "%.16e" % v  # io.hpp:28-32 full_precision: bit-exact round trip


def to_text(p: Problem) -> str:
    """io.hpp:34-47 write_problem / to_text."""
    out = [f"lp2d v1 m={p.constraints.shape[0]} M={_full(p.bound_m)}",
           f"c {_full(p.c[0])} {_full(p.c[1])}"]
    for ax, ay, b in p.constraints:
        out.append(f"h {_full(ax)} {_full(ay)} {_full(b)}")
    return "\n".join(out) + "\n"


def problem_from_text(text: str) -> Problem:
    """io.hpp:49-97 read_problem: same checks, same failure cases."""
    import math

    tok = text.split()

    def fail(what):
        raise ParseError("lp2d parse: " + what)

    if (len(tok) < 4 or tok[0] != "lp2d" or tok[1] != "v1" or not tok[2].startswith("m=")
            or not tok[3].startswith("M=")):
        fail("bad header line")
    try:
        m = int(tok[2][2:])
        bound = float(tok[3][2:])
    except ValueError:
        fail("bad header numbers")
    if m < 0:
        fail("bad header numbers")
    if not math.isfinite(bound) or bound <= 0.0:
        fail("bound must be positive and finite")
    try:
        if tok[4] != "c":
            fail("bad objective line")
        c = (float(tok[5]), float(tok[6]))
    except (IndexError, ValueError):
        fail("bad objective line")
    if not (math.isfinite(c[0]) and math.isfinite(c[1])):
        fail("objective not finite")
    rows = []
    pos = 7
    for _ in range(m):
        try:
            if tok[pos] != "h":
                fail("bad constraint line")
            ax, ay, b = float(tok[pos + 1]), float(tok[pos + 2]), float(tok[pos + 3])
        except (IndexError, ValueError):
            fail("bad constraint line")
        pos += 4
        if not all(math.isfinite(v) for v in (ax, ay, b)) or (ax == 0.0 and ay == 0.0):
            fail("constraint not finite or zero normal")  # core.hpp:41-43 valid()
        rows.append((ax, ay, b))
    return Problem(c, np.array(rows, dtype=np.float64).reshape(-1, 3), bound)
