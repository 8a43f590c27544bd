import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
import paper_1902_04995_b200 as P
cfg = sys.argv[1]
pb = bench.make_batch(cfg, 0, bench.CONFIGS[cfg][2])
pin = lambda a: bench._pinned_copy(torch, a)
hp = P.PackedBatch(pin(pb.m), pin(pb.offset), pin(pb.ax), pin(pb.ay), pin(pb.b), pin(pb.perm), pin(pb.c), pin(pb.M))
n = pb.n; f8 = np.float64
hout = P.PackedResult(*(pin(np.zeros(sh, d)) for sh, d in ((n, np.uint8), (n, f8), (n, f8), (n, f8), ((n, 2), np.int32), (n, np.uint32), (n, np.uint64))))
arrs = [hp.m, hp.offset, hp.ax, hp.ay, hp.b, hp.perm, hp.c, hp.M]
tot = sum(a.nbytes for a in arrs)
dev = [torch.empty(a.nbytes, dtype=torch.uint8, device='cuda') for a in arrs]
src = [torch.from_numpy(a.view(np.uint8).reshape(-1)) for a in arrs]
for _ in range(2):
    for d, s in zip(dev, src): d.copy_(s, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    for d, s in zip(dev, src): d.copy_(s, non_blocking=True)
torch.cuda.synchronize()
h2d = (time.perf_counter() - t) / 5
cfgb = P.BlockConfig(workers=1)
if len(sys.argv) > 2 and sys.argv[2] == "seed":  # permutations generated on the device
    hp = P.PackedBatch(hp.m, hp.offset, hp.ax, hp.ay, hp.b, None, hp.c, hp.M)
    _ps = P.PermSeed(bench.CONFIGS[cfg][3], 2, 1, 0)
    _solve = P.solve_packed
    P.solve_packed = lambda a, b, out: _solve(a, b, out=out, perm_seed=_ps)
P.solve_packed(hp, cfgb, out=hout)
ts = []
for _ in range(5):
    t = time.perf_counter(); P.solve_packed(hp, cfgb, out=hout); ts.append(time.perf_counter() - t)
print("%s n=%d bytes=%.1f MB  h2d-only %.3f ms (%.1f GB/s)  e2e %.3f ms (min %.3f)  -> overhead %.3f ms" % (
    cfg, n, tot / 1e6, h2d * 1e3, tot / h2d / 1e9, np.median(ts) * 1e3, min(ts) * 1e3, (min(ts) - h2d) * 1e3))
