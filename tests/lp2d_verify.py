"""verify / replay for the GPU drop-in (test infrastructure: it uses the
oracle as the checker). Mirrors the reference's cross-solver check
(`bench::verify`, /root/reference/proj/include/lp2d/bench.hpp:291-378) and its
CLI subcommand (`lp2d-bench verify`, tools/lp2d_bench.cpp:173-183; exit codes
0 ok / 1 disagreements / 2 bad arguments, :21-23):

  python tests/lp2d_verify.py verify [--count 1000] [--max-size 128]
         [--seed 20260822] [--dtype f64|f32] [--block-width 512] [--dump DIR]
  python tests/lp2d_verify.py replay FILE.lp2d [--perm-seed S] [--dtype ...]

verify draws the reference's instance stream (sizes 1 + below(max_size) from
derive_seed(seed, 0xA0), every fourth instance infeasible by construction,
problem i seeded derive_seed(seed, 2i), insertion order shuffle(m,
derive_seed(seed, 2i+1))), solves the whole mixed-size batch on the GPU with
BOTH schedulers through the C ABI, and checks per instance, in the
reference's order: naive == serial and balanced == serial bit for bit
(serial = the unmodified reference's solve when oracle/_ref is built, else
the oracle restatement), feasibility against the brute-force vertex oracle
(oracle.hpp:38-70), the value to tolerance.sig_figs, and that the reported
optimum satisfies every constraint. Each disagreement is written to DIR as
`lp2d v1` text (io.hpp:34-47) named instance_<i>_perm<seed>.lp2d, which
`replay` reads back (io.hpp:49-97) and solves again on the GPU, printing the
oracle / serial / naive / balanced lines of the reference's single-instance
log (bench.hpp:352-369)."""
from __future__ import annotations

import argparse
import os
import re
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

M64 = (1 << 64) - 1


class Xoshiro:
    """rng.hpp:13-60 (splitmix64 seeding, xoshiro256++, Lemire below)."""

    def __init__(self, seed: int):
        def sm(st):
            st = (st + 0x9E3779B97F4A7C15) & M64
            z = st
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
            return st, z ^ (z >> 31)

        st = seed & M64
        self.s = []
        for _ in range(4):
            st, v = sm(st)
            self.s.append(v)

    def next(self) -> int:
        s0, s1, s2, s3 = self.s
        rot = lambda x, k: ((x << k) | (x >> (64 - k))) & M64
        r = (rot((s0 + s3) & M64, 23) + s0) & M64
        t = (s1 << 17) & M64
        s2 ^= s0
        s3 ^= s1
        s1 ^= s2
        s0 ^= s3
        s2 ^= t
        s3 = rot(s3, 45)
        self.s = [s0, s1, s2, s3]
        return r

    def below(self, n: int) -> int:
        x = self.next()
        p = x * n
        lo = p & M64
        if lo < n:
            thr = ((1 << 64) - n) % n
            while lo < thr:
                x = self.next()
                p = x * n
                lo = p & M64
        return p >> 64


def verify_batch(P, count: int, max_size: int, seed: int):
    rng = Xoshiro(P.derive_seed(seed, 0xA0))
    sizes = np.array([1 + rng.below(max_size) for _ in range(count)], np.int32)
    kind = np.array([1 if i % 4 == 3 else 0 for i in range(count)], np.uint8)
    # problem i: gen({m, derive_seed(seed, 2i), kind}); order: shuffle(m, derive_seed(seed, 2i+1))
    return P.PackedBatch.generate(sizes, seed, kind=kind)


def fmt(feasible, x, y, v):
    return "(%.17g, %.17g) value %.17g" % (x, y, v) if feasible else "infeasible"


def cmd_verify(a) -> int:
    import oracle_py as O
    import paper_1902_04995_b200 as P

    if a.count <= 0 or a.max_size <= 0:
        print("verify: count and max size must be positive", file=sys.stderr)
        return 2
    if a.max_size > 512:  # oracle.hpp oracle_cap
        print("verify: max size above the oracle cap", file=sys.stderr)
        return 2
    pb = verify_batch(P, a.count, a.max_size, a.seed)
    if a.dtype == "f32":
        pb = pb.astype(np.float32)
    tol = P.Tolerance()
    naive = P.solve_packed(pb, P.BlockConfig(block_width=a.block_width,
                                             scheduler=P.SchedulerKind.naive))
    bal = P.solve_packed(pb, P.BlockConfig(block_width=a.block_width))
    serial_is_ref = O.ref_available()
    if serial_is_ref:
        fe, sx, sy, sval, _ = O.ref_solve_batch(pb, threads=0)
        sfe = fe.astype(bool)
    else:
        o = O.solve_batch(pb, threads=16)
        sfe, sx, sy, sval = o["status"] != O.INFEASIBLE, o["x"], o["y"], o["value"]
    bad = 0
    for i in range(pb.n):
        p = pb.problem(i)
        sv = (bool(sfe[i]), float(sx[i]), float(sy[i]), float(sval[i]))
        gn = (naive.status[i] in (0, 2), naive.x[i], naive.y[i], naive.value[i])
        gb = (bal.status[i] in (0, 2), bal.x[i], bal.y[i], bal.value[i])
        same = lambda g: g[0] == sv[0] and (not sv[0] or (g[1] == sv[1] and g[2] == sv[2]
                                                          and g[3] == sv[3]))
        ob = O.ref_bruteforce(p.constraints[:, 0], p.constraints[:, 1], p.constraints[:, 2],
                              p.c, p.bound_m) if serial_is_ref else None
        why = ""
        if not same(gn):
            why = "naive scheduler differs from serial"
        elif not same(gb):
            why = "balanced scheduler differs from serial"
        elif ob is not None and ob[0] != sv[0]:
            why = "oracle and serial disagree on feasibility"
        elif ob is not None and sv[0] and not P.lp2d.agree_sig_figs(sv[3], ob[3], tol.sig_figs):
            why = "oracle and serial values disagree"
        elif sv[0]:
            for ax, ay, b in p.constraints:  # core.hpp:111-113 satisfied
                if not (ax * sv[1] + ay * sv[2] <= b + tol.feas_slack(b)):
                    why = "reported optimum violates a constraint"
                    break
        if why or a.dump_all:
            if why:
                bad += 1
                print(f"instance {i}: {why}")
            if a.dump:
                os.makedirs(a.dump, exist_ok=True)
                ps = P.derive_seed(a.seed, 2 * i + 1)
                with open(os.path.join(a.dump, f"instance_{i}_perm{ps}.lp2d"), "w") as f:
                    f.write(P.to_text(p))
    print(f"verify: {pb.n} instances ({'reference' if serial_is_ref else 'oracle'} serial, "
          f"{a.dtype} storage), {bad} disagreements")
    return 1 if bad else 0


def cmd_replay(a) -> int:
    import oracle_py as O
    import paper_1902_04995_b200 as P

    try:
        with open(a.file) as f:
            p = P.problem_from_text(f.read())
    except (OSError, P.ParseError) as e:
        print(f"replay: {e}", file=sys.stderr)
        return 2
    m = p.constraints.shape[0]
    ps = a.perm_seed
    if ps is None:
        g = re.search(r"_perm(\d+)\.lp2d$", a.file)
        ps = int(g.group(1)) if g else None
    perm = P.shuffle(m, ps) if ps is not None else P.identity_permutation(m)
    b = P.Batch([p], [perm])
    dt = np.float32 if a.dtype == "f32" else np.float64
    res = {}
    for name, sched in (("naive", P.SchedulerKind.naive), ("balanced", P.SchedulerKind.balanced)):
        r = P.solve_batch(b, P.BlockConfig(scheduler=sched), dtype=dt)
        s = r.solutions[0]
        res[name] = (bool(s.feasible), float(s.point[0]), float(s.point[1]), float(s.value))
    pk = P.PackedBatch.from_batch(b, dtype=dt)
    if O.ref_available():
        fe, x, y, v, _ = O.ref_solve_batch(pk, threads=1)
        res["serial"] = (bool(fe[0]), float(x[0]), float(y[0]), float(v[0]))
        res["oracle"] = O.ref_bruteforce(p.constraints[:, 0], p.constraints[:, 1],
                                         p.constraints[:, 2], p.c, p.bound_m) if m <= 512 else None
    else:
        r = O.solve_batch(pk)
        res["serial"] = (bool(r["status"][0] != O.INFEASIBLE), float(r["x"][0]), float(r["y"][0]),
                         float(r["value"][0]))
        res["oracle"] = None
    print(P.to_text(p), end="")
    for name in ("oracle", "serial", "naive", "balanced"):
        if res.get(name) is not None:
            print(f"{name}: {fmt(*res[name])}")
    agree = res["naive"] == res["serial"] and res["balanced"] == res["serial"]
    return 0 if agree else 1


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="lp2d_verify")
    sub = ap.add_subparsers(dest="cmd", required=True)
    v = sub.add_parser("verify")
    v.add_argument("--count", type=int, default=1000)
    v.add_argument("--max-size", type=int, default=128)
    v.add_argument("--seed", type=int, default=20260822)
    v.add_argument("--dtype", choices=["f64", "f32"], default="f64")
    v.add_argument("--block-width", type=int, default=512)
    v.add_argument("--dump", default=None)
    v.add_argument("--dump-all", action="store_true", help="write every instance (replay tests)")
    r = sub.add_parser("replay")
    r.add_argument("file")
    r.add_argument("--perm-seed", type=int, default=None)
    r.add_argument("--dtype", choices=["f64", "f32"], default="f64")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    return cmd_verify(a) if a.cmd == "verify" else cmd_replay(a)


if __name__ == "__main__":
    sys.exit(main())
