"""K4 path statistics and timing per config (run on a GPU box with
LP2D_B200_FX_STATS=1): events, certified, reshifts, exact events, flags."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1902_04995_b200 as P  # noqa: E402

NAMES = ["events", "cert_first", "reshift", "exact_events", "test_flags", "lazy_points", "wild_lps",
         "cert_after_reshift"]


def main():
    import torch

    cfgs = sys.argv[1:] or ["c2"]
    L = P.lp2d.N.lib()
    st = np.zeros(8, np.uint64)
    for cfg in cfgs:
        dt = bench.config_dtype(cfg, None)
        pb = bench.make_batch(cfg, 0, dt)
        db = P.DeviceBatch(pb)
        out = db.empty_result()
        P.solve_device(db, out)
        torch.cuda.synchronize()
        L.lp2dgpu_fx_stats(st.ctypes.data, 1)
        P.solve_device(db, out)
        torch.cuda.synchronize()
        n = L.lp2dgpu_fx_stats(st.ctypes.data, 1)
        s = {k: int(v) for k, v in zip(NAMES, st)} if n else {}
        s["events"] = int(out.violation_events.sum().item())  # (counted by the outputs)
        s.pop("cert_first", None)
        s.pop("cert_after_reshift", None)
        ev = max(s["events"], 1)
        print(cfg, pb.n, "LPs", s, {k: "%.3f%%" % (100 * v / ev) for k, v in s.items() if k != "events"})


if __name__ == "__main__":
    main()
