"""Debug: per-LP K4 path counts (library variant built with -DLP2D_FX_TIMELINE
-DLP2D_FX_LPSTATS: pair[2j+1] = reshifts | exact events << 10 | exact tests << 20,
pair[2j] = duration ns) of a config's slowest LPs."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["LP2D_B200_LIB"] = os.path.join(ROOT, "paper_1902_04995_b200", "lib", "variants",
                                           sys.argv[2] if len(sys.argv) > 2 else "st.so")
import bench  # noqa: E402
import paper_1902_04995_b200 as P  # noqa: E402
import torch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
pb = bench.make_batch(cfg, 0, bench.config_dtype(cfg, None))
db = P.DeviceBatch(pb)
out = db.empty_result()
for _ in range(3):
    P.solve_device(db, out)
torch.cuda.synchronize()
w = out.pair.cpu().numpy()[:, 1].astype(np.int64)
dur = out.pair.cpu().numpy()[:, 0].astype(np.int64) / 1e3
viol = out.violation_events.cpu().numpy()
res, exe, tst = w & 1023, (w >> 10) & 1023, (w >> 20) & 1023
print("all LPs: dur mean %.1f us; reshifts %.2f exact events %.3f exact tests %.2f per LP"
      % (dur.mean(), res.mean(), exe.mean(), tst.mean()))
for q in (50, 90, 99, 99.9):
    k = dur >= np.percentile(dur, q)
    print("dur >= p%g (%.1f us): n=%d reshifts %.2f exact events %.2f exact tests %.2f events %.1f"
          % (q, np.percentile(dur, q), k.sum(), res[k].mean(), exe[k].mean(), tst[k].mean(), viol[k].mean()))
for j in np.argsort(-dur)[:10]:
    print("LP %6d dur %6.1f us events %3d reshifts %d exact events %d exact tests %d"
          % (j, dur[j], viol[j], res[j], exe[j], tst[j]))
