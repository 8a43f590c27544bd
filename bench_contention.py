"""Contention microbenchmark (the paper's Fig.
atomicComp; reference bench.hpp:244-274 contention_bench).

Times one segmented min/max pass over 512*2048 doubles (the reference's
default) for every GPU update discipline at contention 1..512, on the device
(CUDA events, median of reps), next to the reference's own CPU
contention_bench (oracle/_ref, 1 thread) for its three strategies.
Prints one JSON object per line: {"strategy", "contention", "gpu_us" | "cpu_us", ...}.

usage: python bench_contention.py [--reps 20] [--values 1048576] [--no-cpu]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--values", type=int, default=512 * 2048)
    ap.add_argument("--seed", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    import paper_1902_04995_b200 as P

    levels = [1 << k for k in range(10)]
    recs = P.contention_bench(list(P.ReduceStrategy), levels, args.reps, args.seed, args.values)
    for s in P.ReduceStrategy:
        for c in levels:
            t = [r.wall_time_ns for r in recs if r.strategy == s and r.contention == c]
            us = float(np.median(t)) / 1e3
            print(json.dumps({"impl": "b200", "strategy": P.reduction.to_string(s), "contention": c,
                              "gpu_us": us, "values": args.values,
                              "gvalues_per_s": args.values / us / 1e3}), flush=True)
    if args.no_cpu:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py as O  # baseline only: the reference's own CPU timing

    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    names = ["serialized-shared-update", "tree-reduction", "per-lane-private-then-merge"]
    for s in range(3):
        for c in levels:
            ns = O.ref_lib().ref_contention_ns(s, c, max(3, args.reps // 4), args.seed, args.values)
            print(json.dumps({"impl": "reference-cpu", "strategy": names[s], "contention": c,
                              "cpu_us": ns / 1e3, "values": args.values, "threads": 1}), flush=True)


if __name__ == "__main__":
    main()
