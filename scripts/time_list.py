"""Solve-kernel time of a device batch with config 4's sizes in [lo, hi]
(class tuning aid): python scripts/time_list.py lo hi"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1902_04995_b200 as P  # noqa: E402

lo, hi = int(sys.argv[1]), int(sys.argv[2])
s = bench.pareto_sizes(4)
s = s[(s >= lo) & (s <= hi)].astype(np.int32)
db = P.DeviceBatch.generate(s, 4, dtype=np.float32)
out = db.empty_result()
for _ in range(3):
    P.solve_device(db, out)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(10):
    ev[0].record()
    P.solve_device(db, out)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
print("m in [%d, %d]: n=%d  min %.1f us  median %.1f us" % (lo, hi, len(s), 1e3 * min(ts), 1e3 * np.median(ts)))
