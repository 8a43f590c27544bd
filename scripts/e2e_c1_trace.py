"""Host-mode timeline of one config-1 call (LP2D_B200_TRACE=1): where the
~100 us of a 1024-LP end-to-end solve go."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1902_04995_b200 as P  # noqa: E402
import torch  # noqa: E402

pb = bench.make_batch("c1", 0, np.float32)
pin = lambda a: bench._pinned_copy(torch, a)
hp = P.PackedBatch(pin(pb.m), pin(pb.offset), pin(pb.ax), pin(pb.ay), pin(pb.b), pin(pb.perm), pin(pb.c), pin(pb.M))
n = pb.n
hout = P.PackedResult(*(pin(np.zeros(sh, d)) for sh, d in (
    (n, np.uint8), (n, np.float64), (n, np.float64), (n, np.float64), ((n, 2), np.int32), (n, np.uint32), (n, np.uint64))))
cfg = P.BlockConfig(workers=1)
for _ in range(5):
    P.solve_packed(hp, cfg, out=hout)
print("---- last call ----", file=sys.stderr, flush=True)
P.solve_packed(hp, cfg, out=hout)
