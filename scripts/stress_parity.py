"""Randomised parity stress (GPU): many seeds of perturbed instances over every
size class and both storage types, each solve compared with the oracle.
python scripts/stress_parity.py [seeds] [kernel-selection env is inherited]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_py as O  # noqa: E402
import paper_1902_04995_b200 as P  # noqa: E402


def perturb(pb, dt, rng):
    ax, ay, b = pb.ax, pb.ay, pb.b
    for j in range(pb.n):
        o, mj = int(pb.offset[j]), int(pb.m[j])
        if mj == 0:
            continue
        sel = int(rng.integers(0, 9))
        k = rng.integers(0, mj, max(1, mj // 16))
        if sel == 0:    # duplicates / scaled copies
            src = rng.integers(0, mj, len(k))
            s = dt(rng.choice([1.0, 2.0, 0.5, 3.0]))
            ax[o + k], ay[o + k], b[o + k] = ax[o + src] * s, ay[o + src] * s, b[o + src] * s
        elif sel == 1:  # tight slacks: constraints through a common point
            px, py = rng.uniform(-5e6, 5e6, 2)
            b[o + k] = (ax[o + k].astype(np.float64) * px + ay[o + k] * py).astype(dt)
        elif sel == 2:  # nearly parallel bundles
            ax[o + k] = ax[o + k[0]] * (dt(1) + dt(rng.uniform(-1e-6, 1e-6)))
            ay[o + k] = ay[o + k[0]]
        elif sel == 3:  # axis-aligned
            ax[o + k] = dt(0)
            ay[o + k] = dt(1)
        elif sel == 4:  # rescaled LP (small coordinates)
            b[o:o + mj] *= dt(rng.choice([1e-6, 1e-3, 1e3]))
        elif sel == 5:  # objective along a constraint normal
            pass
        # sel >= 6: unperturbed
    return pb


def main():
    seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    bad = 0
    for seed in range(seeds):
        rng = np.random.default_rng(1000 + seed)
        sizes = rng.choice([0, 3, 20, 28, 29, 45, 60, 61, 100, 124, 125, 150, 188, 189, 250, 316,
                            317, 500, 572, 573, 1024, 1052, 1053, 2000, 2076, 2077, 3000, 5000],
                           int(os.environ.get("STRESS_N", "96"))).astype(np.int32)
        for dt in (np.float32, np.float64):
            base = P.PackedBatch.generate(sizes, 500 + seed)
            pb = base.astype(dt) if dt == np.float32 else base
            pb = perturb(pb, dt, rng)
            if seed % 3 == 0:
                c = pb.c.reshape(-1, 2)
                for j in range(pb.n):  # objective along some constraint's normal
                    if pb.m[j] > 0:
                        q = int(pb.offset[j])
                        c[j] = (pb.ax[q], pb.ay[q])
                pb.c = c.reshape(-1).astype(pb.c.dtype)
            o = O.solve_batch(pb, threads=16)
            for sched in (P.SchedulerKind.balanced, P.SchedulerKind.naive):
                r = P.solve_packed(pb, P.BlockConfig(scheduler=sched))
                st = r.status.astype(np.int32)
                feas = o["status"] != O.INFEASIBLE
                ok = (np.array_equal(st, o["status"]) and np.array_equal(r.pair, o["pair"]) and
                      all(np.array_equal(getattr(r, k)[feas].astype(np.float64), o[k][feas],
                                         equal_nan=True) for k in ("x", "y", "value")) and
                      np.array_equal(r.work_units, o["work_units"]))
                if not ok:
                    bad += 1
                    diff = np.nonzero((st != o["status"]) | (r.pair != o["pair"]).any(axis=1))[0]
                    print("MISMATCH seed", seed, dt.__name__, sched, "LPs", diff[:8],
                          "m", pb.m[diff[:8]])
    print("stress: %d seeds x 2 storage types x 2 schedulers, %d mismatching solves" % (seeds, bad))
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
