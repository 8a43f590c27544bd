"""Debug: per-LP solve durations of the K4 kernel (library variant built with
-DLP2D_FX_TIMELINE: wu = start ns, pair[2j] = duration ns)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["LP2D_B200_LIB"] = os.path.join(ROOT, "paper_1902_04995_b200", "lib", "variants", "tl.so")
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
start = out.work_units.cpu().numpy().astype(np.int64)
dur = out.pair.cpu().numpy()[:, 0].astype(np.int64)
viol = out.violation_events.cpu().numpy()
t0 = start.min()
end = start + dur
print("span %.1f us, LP duration mean %.2f us, p50 %.2f p99 %.2f max %.2f us" % (
    (end.max() - t0) / 1e3, dur.mean() / 1e3, np.percentile(dur, 50) / 1e3, np.percentile(dur, 99) / 1e3,
    dur.max() / 1e3))
order = np.argsort(-dur)[:12]
for j in order:
    print("LP %6d start %8.1f us dur %8.1f us events %d" % (j, (start[j] - t0) / 1e3, dur[j] / 1e3, viol[j]))
# completion profile
ends = np.sort(end - t0) / 1e3
for q in (0.5, 0.9, 0.99, 0.999, 1.0):
    print("LPs done by %.1f%%: %.1f us" % (100 * q, ends[min(len(ends) - 1, int(q * len(ends)))]))
np.save("gpurun_out/slow_lps_%s.npy" % cfg, order)
