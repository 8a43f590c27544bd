"""Solve-kernel time of uniform device batches (class tuning aid):
python scripts/time_sizes.py f64 500 131072 [m n ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_04995_b200 as P  # noqa: E402

dt = np.float64 if sys.argv[1] == "f64" else np.float32
args = [int(a) for a in sys.argv[2:]]
for m, n in zip(args[0::2], args[1::2]):
    db = P.DeviceBatch.generate(np.full(n, m, np.int32), 5, dtype=dt)
    out = db.empty_result()
    for _ in range(3):
        P.solve_device(db, out)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(5):
        ev[0].record()
        P.solve_device(db, out)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    print("%s m=%d n=%d: %.1f us (%.2f ns/LP)" % (sys.argv[1], m, n, 1e3 * min(ts), 1e6 * min(ts) / n))
