"""Contention microbenchmark on the GPU.

Mirror of the reference's reduction.hpp / bench.hpp contention API:

* ``ReduceStrategy``          reduction.hpp:18-22 (+ the paper's GPU arms)
* ``segmented_extremes``      reduction.hpp:46-129
* ``contention_bench``        bench.hpp:244-274 (``ContentionRecord`` :237-241)

The reference models three CPU update disciplines for combining lanes'
classifications into one interval; the paper (Fig. atomicComp) measured the
GPU choices: shared-memory atomics, global atomics and CUB's segmented
reduce. All run here as CUDA kernels behind ``lp2dgpu_segmented_extremes``
(include/lp2d_b200.h) and return the reference's values bit for bit — min and
max are exact. There is no CPU path: without a GPU the calls raise.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

from . import _native as N


class ReduceStrategy(enum.IntEnum):
    """reduction.hpp:18-22 names for the first three; the GPU disciplines they
    become are in lp2d_reduce.cuh."""

    serialized_shared_update = N.REDUCE_SHARED_ATOMIC  # shared-memory atomics
    tree_reduction = N.REDUCE_TREE
    private_then_merge = N.REDUCE_PRIVATE_MERGE
    global_atomic = N.REDUCE_GLOBAL_ATOMIC             # the paper's global atomics
    cub_segmented_reduce = N.REDUCE_CUB                # the paper's library baseline


def to_string(s: ReduceStrategy) -> str:  # reduction.hpp:24-34
    return {
        ReduceStrategy.serialized_shared_update: "serialized-shared-update",
        ReduceStrategy.tree_reduction: "tree-reduction",
        ReduceStrategy.private_then_merge: "per-lane-private-then-merge",
        ReduceStrategy.global_atomic: "global-atomic",
        ReduceStrategy.cub_segmented_reduce: "cub-segmented-reduce",
    }[ReduceStrategy(s)]


def _check(rc: int):
    if rc == N.ERR_ARG:
        raise ValueError(N.lib().lp2dgpu_last_error().decode())
    if rc != 0:
        raise RuntimeError(N.lib().lp2dgpu_last_error().decode())


def _stream_ptr(torch, stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def segmented_extremes_device(values, contention: int, strategy: ReduceStrategy,
                              out_min, out_max, stream=None) -> None:
    """Device form: float64 CUDA tensors, enqueued on ``stream``."""
    import torch

    n = values.numel()
    rc = N.lib().lp2dgpu_segmented_extremes(
        C.c_void_p(values.data_ptr()), n, int(contention), int(strategy),
        C.c_void_p(out_min.data_ptr()), C.c_void_p(out_max.data_ptr()),
        values.device.index or 0, _stream_ptr(torch, stream))
    _check(rc)


def segmented_extremes(values, contention: int,
                       strategy: ReduceStrategy = ReduceStrategy.serialized_shared_update
                       ) -> Tuple[np.ndarray, np.ndarray]:
    """Host form (reduction.hpp:46): min and max of every consecutive group of
    ``contention`` values. Errors as the reference: contention < 1 or a size
    that does not split into groups -> ValueError."""
    import torch

    v = np.ascontiguousarray(values, dtype=np.float64)
    if contention < 1:
        raise ValueError("segmented_extremes: contention must be >= 1")
    if len(v) % contention:
        raise ValueError("segmented_extremes: input size must be a multiple of contention")
    g = len(v) // contention
    dev = torch.device("cuda", torch.cuda.current_device())
    dv = torch.from_numpy(v).to(dev)
    mn = torch.empty(g, dtype=torch.float64, device=dev)
    mx = torch.empty(g, dtype=torch.float64, device=dev)
    segmented_extremes_device(dv, contention, strategy, mn, mx)
    torch.cuda.synchronize(dev)
    return mn.cpu().numpy(), mx.cpu().numpy()


@dataclass
class ContentionRecord:  # bench.hpp:237-241
    strategy: ReduceStrategy
    contention: int
    wall_time_ns: int


def contention_values(seed: int, values: int) -> np.ndarray:
    """bench.hpp:256-257 inputs: xoshiro256pp(derive_seed(seed, 0xC0)).in_range(-1e6, 1e6)."""
    out = np.empty(values, dtype=np.float64)
    N.lib().lp2dgen_uniform(seed & (2**64 - 1), 0xC0, -1e6, 1e6, values, out.ctypes.data)
    return out


def contention_bench(strategies: Sequence[ReduceStrategy], contentions: Sequence[int],
                     reps: int, seed: int, values: int = 512 * 2048,
                     inner: int = 10) -> List[ContentionRecord]:
    """bench.hpp:244-274 on the GPU: one record per (contention, strategy, rep),
    wall_time_ns = device time of one segmented-extremes pass: `inner`
    back-to-back passes are captured in a CUDA graph and the replay is timed
    with CUDA events, so host launch latency is excluded."""
    import torch

    for c in contentions:  # bench.hpp:249-255
        if c == 0 or c > 512 or (c & (c - 1)) != 0:
            raise ValueError("contention_bench: contention levels must be powers of two in [1, 512]")
    dev = torch.device("cuda", torch.cuda.current_device())
    dv = torch.from_numpy(contention_values(seed, values)).to(dev)
    mn = torch.empty(values, dtype=torch.float64, device=dev)
    mx = torch.empty(values, dtype=torch.float64, device=dev)
    out: List[ContentionRecord] = []
    for c in contentions:
        g = values // c
        src, omn, omx = dv[: g * c], mn[:g], mx[:g]
        for s in strategies:
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                segmented_extremes_device(src, c, s, omn, omx, stream=side)  # warm-up
            side.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=side):
                for _ in range(inner):
                    segmented_extremes_device(src, c, s, omn, omx, stream=side)
            graph.replay()
            torch.cuda.synchronize(dev)
            for _ in range(reps):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                graph.replay()
                e1.record()
                e1.synchronize()
                out.append(ContentionRecord(ReduceStrategy(s), c,
                                            int(e0.elapsed_time(e1) * 1e6 / inner)))
    return out
