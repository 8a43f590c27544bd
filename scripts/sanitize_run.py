"""Small solves over every size class and both storage types, for
compute-sanitizer (memcheck / synccheck / racecheck) runs on the GPU box.
Run it once per kernel selection, e.g. LP2D_B200_FS=all (K5 for every fp32
warp class) and LP2D_B200_CHUNK_ELEMS=3000 (many host-mode chunks); every
run also covers permutations generated from seeds."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1902_04995_b200 as P  # noqa: E402
import oracle_py as O  # noqa: E402

sizes = np.array([0, 3, 28, 29, 60, 100, 150, 180, 250, 300, 500, 572, 700, 1024, 1052, 1500,
                  2076, 3000, 5000], np.int32)
for dt in (np.float32, np.float64):
    for sz in (sizes, np.full(40, 1024, np.int32), np.full(40, 256, np.int32)):
        base = P.PackedBatch.generate(np.repeat(sz, 2), 11)
        pb = base.astype(dt) if dt == np.float32 else base
        o = O.solve_batch(pb)
        r = P.solve_packed(pb)
        assert np.array_equal(r.status.astype(np.int32), o["status"]), (dt, len(sz))
        assert np.array_equal(r.pair, o["pair"]), (dt, len(sz))
        noperm = P.PackedBatch(pb.m, pb.offset, pb.ax, pb.ay, pb.b, None, pb.c, pb.M)
        r = P.solve_packed(noperm, perm_seed=P.PermSeed(11))
        assert np.array_equal(r.pair, o["pair"]), (dt, len(sz), "perm_seed")
print("sanitize run ok (%s)" % ", ".join(f"{k}={v}" for k, v in os.environ.items()
                                          if k.startswith("LP2D_B200_")))
