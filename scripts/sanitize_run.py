"""Small solves over every size class and both precisions, for
compute-sanitizer (memcheck / racecheck) runs on the GPU box."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1902_04995_b200 as P  # noqa: E402
import oracle_py as O  # noqa: E402

sizes = np.array([0, 3, 28, 29, 60, 100, 150, 180, 250, 300, 500, 572, 700, 1024, 1052, 1500,
                  2076, 3000], np.int32)
for dt in (np.float32, np.float64):
    for sz in (sizes, np.full(40, 1024, np.int32), np.full(40, 256, np.int32)):
        pb = P.PackedBatch.generate(np.repeat(sz, 2), 11).astype(dt)
        r = P.solve_packed(pb)
        o = O.solve_batch(pb)
        assert np.array_equal(r.status.astype(np.int32), o["status"]), (dt, len(sz))
        assert np.array_equal(r.pair, o["pair"]), (dt, len(sz))
print("sanitize run ok")
