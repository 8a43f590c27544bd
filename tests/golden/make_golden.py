"""Regenerate the golden fixtures in tests/golden/ from the UNMODIFIED
reference (oracle/_ref/liblp2d_ref.so, built from /root/reference by
oracle/Makefile). Run here, where /root/reference exists:

    python tests/golden/make_golden.py

Fixtures (all small):
  kat.json          RNG / shuffle / generator / solver known answers, incl.
                    the reference's pinned frozen_value_seed42_m32
                    (proj/tests/test_generate.cpp:20) recomputed here.
  ref_<name>.npz    reference fp64 results (feasible, x, y, value, per-LP
                    violation_events and work_units from serial solve with
                    solve_stats) for the instance batches below.
  ref32_<name>.npz  the same reference results for the fp32-rounded copy of
                    each batch (the fp32 configs: float storage, the
                    reference's double arithmetic on the widened values).
  oracle_<name>.npz the restated oracle's status / defining pair for the same
                    batches (fp64) and for their fp32-rounded copies — the
                    builder extension has no reference counterpart, so these
                    pin the restatement against regressions.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle_py as O  # noqa: E402


class Packed:
    def __init__(self, m, offset, ax, ay, b, perm, c, M):
        self.m, self.offset, self.ax, self.ay, self.b = m, offset, ax, ay, b
        self.perm, self.c, self.M = perm, c, M
        self.n = len(m)

    def astype(self, dt):
        return Packed(self.m, self.offset, self.ax.astype(dt), self.ay.astype(dt),
                      self.b.astype(dt), self.perm, self.c.astype(dt), self.M.astype(dt))


def offsets(m):
    cap = (np.asarray(m, np.int64) + 7) // 8 * 8
    off = np.zeros(len(m) + 1, np.int64)
    off[1:] = np.cumsum(cap)
    return off


def ref_gen_mixed(sizes, count, seed, kind=0, margin=1.0):
    ref = O.ref_lib()
    sizes = np.asarray(sizes, np.int64)
    m = np.array([sizes[i % len(sizes)] for i in range(count)], np.int32)
    off = offsets(m)
    E = int(off[-1])
    ax = np.zeros(E); ay = np.zeros(E); b = np.zeros(E)
    perm = np.zeros(E, np.uint32); c = np.zeros(2 * count); M = np.zeros(count)
    rc = ref.ref_gen_mixed(sizes.ctypes.data, len(sizes), count, seed, kind, margin, off.ctypes.data,
                           ax.ctypes.data, ay.ctypes.data, b.ctypes.data, perm.ctypes.data,
                           c.ctypes.data, M.ctypes.data)
    assert rc == 0
    return Packed(m, off, ax, ay, b, perm, c, M)


def ref_single(pk, j):
    ref = O.ref_lib()
    o, mj = int(pk.offset[j]), int(pk.m[j])
    ax = np.ascontiguousarray(pk.ax[o:o + mj]); ay = np.ascontiguousarray(pk.ay[o:o + mj])
    b = np.ascontiguousarray(pk.b[o:o + mj]); perm = np.ascontiguousarray(pk.perm[o:o + mj])
    fe = np.zeros(1, np.uint8); x = np.zeros(1); y = np.zeros(1); v = np.zeros(1)
    vi = np.zeros(1, np.uint64); wu = np.zeros(1, np.uint64)
    ref.ref_solve(ax.ctypes.data, ay.ctypes.data, b.ctypes.data, perm.ctypes.data, mj,
                  float(pk.c[2 * j]), float(pk.c[2 * j + 1]), float(pk.M[j]), 1e-12, 1e-9,
                  fe.ctypes.data, x.ctypes.data, y.ctypes.data, v.ctypes.data, vi.ctypes.data,
                  wu.ctypes.data)
    return bool(fe[0]), x[0], y[0], v[0], int(vi[0]), int(wu[0])


def ref_results(pk):
    res = [ref_single(pk, j) for j in range(pk.n)]
    return {"feasible": np.array([r[0] for r in res], np.uint8),
            "x": np.array([r[1] for r in res]), "y": np.array([r[2] for r in res]),
            "value": np.array([r[3] for r in res]),
            "violation_events": np.array([r[4] for r in res], np.uint64),
            "work_units": np.array([r[5] for r in res], np.uint64)}


def verify_batch(count, max_size, seed):
    """bench.hpp:291-312 verify() instance stream: sizes 1 + below(max_size)
    from derive_seed(seed, 0xA0), every 4th infeasible, problem seed
    derive_seed(seed, 2i), permutation shuffle(m, derive_seed(seed, 2i+1))."""
    ref = O.ref_lib()
    draws = np.zeros(count, np.uint64)
    O.oracle_lib().lp2d_oracle_below.restype = None
    import ctypes as C
    O.oracle_lib().lp2d_oracle_below.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_void_p]
    O.oracle_lib().lp2d_oracle_below(O.derive_seed(seed, 0xA0), max_size, count, draws.ctypes.data)
    m = (1 + draws).astype(np.int32)
    off = offsets(m)
    E = int(off[-1])
    ax = np.zeros(E); ay = np.zeros(E); b = np.zeros(E)
    perm = np.zeros(E, np.uint32); c = np.zeros(2 * count); M = np.zeros(count)
    for i in range(count):
        o, mj = int(off[i]), int(m[i])
        kind = 1 if i % 4 == 3 else 0
        cc = np.zeros(2); mm = np.zeros(1)
        tax = np.zeros(mj); tay = np.zeros(mj); tb = np.zeros(mj)
        assert ref.ref_gen(mj, O.derive_seed(seed, 2 * i), kind, 1.0, tax.ctypes.data,
                           tay.ctypes.data, tb.ctypes.data, cc.ctypes.data, mm.ctypes.data) == 0
        ax[o:o + mj], ay[o:o + mj], b[o:o + mj] = tax, tay, tb
        c[2 * i:2 * i + 2] = cc
        M[i] = mm[0]
        tp = np.zeros(mj, np.uint32)
        ref.ref_shuffle(mj, O.derive_seed(seed, 2 * i + 1), tp.ctypes.data)
        perm[o:o + mj] = tp
    return Packed(m, off, ax, ay, b, perm, c, M)


BATCHES = {
    # name: builder
    "c1": lambda: ref_gen_mixed([64], 1024, 1),             # BASELINE configs[0]
    "mixed": lambda: ref_gen_mixed([3, 40, 150], 300, 123),  # test_batch.cpp:76-98 shape
    "verify": lambda: verify_batch(400, 128, 20260822),      # acceptance criterion 1 stream
    "m1024": lambda: ref_gen_mixed([1024], 48, 2),           # headline shape, small count
}


def main():
    ref = O.ref_lib()
    kat = {}
    x = np.zeros(3, np.uint64)
    ref.ref_xoshiro_first(0, 3, x.ctypes.data)
    kat["xoshiro_seed0_first3"] = [int(v) for v in x]
    kat["derive_seed_1_0"] = int(ref.ref_derive_seed(1, 0))
    kat["derive_seed_1_1"] = int(ref.ref_derive_seed(1, 1))
    for m, s in ((10, 5), (16, 42)):
        o = np.zeros(m, np.uint32)
        ref.ref_shuffle(m, s, o.ctypes.data)
        kat[f"shuffle_{m}_{s}"] = [int(v) for v in o]
    # frozen oracle value of gen({32, 42}) (test_generate.cpp:20, :90-101)
    ax = np.zeros(32); ay = np.zeros(32); b = np.zeros(32); c = np.zeros(2); M = np.zeros(1)
    ref.ref_gen(32, 42, 0, 1.0, ax.ctypes.data, ay.ctypes.data, b.ctypes.data, c.ctypes.data, M.ctypes.data)
    fe = np.zeros(1, np.uint8); px = np.zeros(1); py = np.zeros(1); v = np.zeros(1)
    ref.ref_bruteforce(ax.ctypes.data, ay.ctypes.data, b.ctypes.data, 32, c[0], c[1], M[0], 1e-12, 1e-9,
                       fe.ctypes.data, px.ctypes.data, py.ctypes.data, v.ctypes.data)
    kat["bruteforce_gen32_42_value"] = float(v[0])
    kat["gen32_42_first_constraint"] = [float(ax[0]), float(ay[0]), float(b[0])]
    kat["gen32_42_objective"] = [float(c[0]), float(c[1])]
    # gen_mixed checksums (SURVEY.md §8(c) probe KATs)
    for sizes, count, seed in (([64], 1024, 1), ([128], 4096, 3)):
        pk = ref_gen_mixed(sizes, count, seed)
        h = ref.ref_batch_create(pk.n, pk.offset.ctypes.data, pk.m.ctypes.data, pk.ax.ctypes.data,
                                 pk.ay.ctypes.data, pk.b.ctypes.data, pk.perm.ctypes.data,
                                 pk.c.ctypes.data, pk.M.ctypes.data)
        fe = np.zeros(pk.n, np.uint8); xx = np.zeros(pk.n); yy = np.zeros(pk.n); vv = np.zeros(pk.n)
        st = np.zeros(5, np.uint64)
        ref.ref_batch_solve(h, 512, 1, 0, 1e-12, 1e-9, fe.ctypes.data, xx.ctypes.data, yy.ctypes.data,
                            vv.ctypes.data, st.ctypes.data, None)
        ref.ref_batch_free(h)
        checksum = 0.0
        for j in range(pk.n):  # bench.hpp:76-82 sequential checksum
            if fe[j]:
                checksum += vv[j]
        kat[f"gen_mixed_{sizes[0]}_{count}_{seed}"] = {
            "checksum": checksum, "violation_events": int(st[1]), "total_wu": int(st[0])}
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1)

    for name, build in BATCHES.items():
        pk = build()
        np.savez_compressed(os.path.join(HERE, f"batch_{name}.npz"), m=pk.m, offset=pk.offset,
                            ax=pk.ax, ay=pk.ay, b=pk.b, perm=pk.perm, c=pk.c, M=pk.M)
        np.savez_compressed(os.path.join(HERE, f"ref_{name}.npz"), **ref_results(pk))
        np.savez_compressed(os.path.join(HERE, f"ref32_{name}.npz"),
                            **ref_results(pk.astype(np.float32).astype(np.float64)))
        o64 = O.solve_batch(pk)
        o32 = O.solve_batch(pk.astype(np.float32))
        np.savez_compressed(os.path.join(HERE, f"oracle_{name}.npz"),
                            status64=o64["status"], pair64=o64["pair"],
                            status32=o32["status"], pair32=o32["pair"], x32=o32["x"], y32=o32["y"],
                            value32=o32["value"], viol32=o32["violation_events"],
                            wu32=o32["work_units"])
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
