"""Host-pipeline ordering check: alternate two different batches through the
chunked host path and compare every result with a device-mode solve of the
same batch (stale results from the other batch would show as mismatches)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1902_04995_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
dt = bench.CONFIGS[cfg][2]
pbs = [bench.make_batch(cfg, 0, dt), bench.make_batch(cfg, 1, dt)]  # rank 0 / rank 1 shards
pin = lambda a: bench._pinned_copy(torch, a)
exp = []
for pb in pbs:
    db = P.DeviceBatch(pb)
    out = db.empty_result()
    P.solve_device(db, out)
    torch.cuda.synchronize()
    exp.append((out.status.cpu().numpy(), out.x.cpu().numpy(), out.y.cpu().numpy()))
hps = [P.PackedBatch(pin(pb.m), pin(pb.offset), pin(pb.ax), pin(pb.ay), pin(pb.b), pin(pb.perm),
                     pin(pb.c), pin(pb.M)) for pb in pbs]
bad = 0
for it in range(8):
    i = it % 2
    n = pbs[i].n
    f8 = np.float64
    hout = P.PackedResult(*(pin(np.zeros(sh, d)) for sh, d in (
        (n, np.uint8), (n, f8), (n, f8), (n, f8), ((n, 2), np.int32), (n, np.uint32), (n, np.uint64))))
    if len(sys.argv) > 2 and sys.argv[2] == "seed":  # permutations generated on the device
        hb = hps[i]
        nop = P.PackedBatch(hb.m, hb.offset, hb.ax, hb.ay, hb.b, None, hb.c, hb.M)
        P.solve_packed(nop, P.BlockConfig(workers=1), out=hout,
                       perm_seed=P.PermSeed(bench.CONFIGS[cfg][3], 2, 1, i * pbs[0].n))
    else:
        P.solve_packed(hps[i], P.BlockConfig(workers=1), out=hout)
    st, x, y = exp[i]
    nb = int(np.sum((hout.status != st) | ~((hout.x == x) | (np.isnan(hout.x) & np.isnan(x)))))
    bad += nb
    print("iter %d batch %d: %d mismatches of %d" % (it, i, nb, n))
print("RACE" if bad else "ok")
