"""Parity of one fp32-storage kernel variant, run in a fresh process because
the library reads its kernel-selection knobs (LP2D_B200_FS, LP2D_B200_GRP) once:
    LP2D_B200_FS=all python tests/variant_check.py
Every fp32 fixture against the UNMODIFIED reference's results on the rounded
instance, the size-class edges and a heavy-tailed batch against the oracle."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from conftest import load_batch, load_npz  # noqa: E402

import oracle_py as O  # noqa: E402
import paper_1902_04995_b200 as P  # noqa: E402


def same(r, o, what):
    st = r.status.astype(np.int32)
    bad = np.nonzero((st != o["status"]) | (r.pair != o["pair"]).any(axis=1))[0]
    assert bad.size == 0, f"{what}: status/pair differ at LPs {bad[:8]}"
    feas = o["status"] != O.INFEASIBLE
    for k in ("x", "y", "value"):
        assert np.array_equal(getattr(r, k)[feas].astype(np.float64), o[k][feas], equal_nan=True), \
            f"{what}: {k}"
    assert np.array_equal(r.violation_events.astype(np.uint64), o["violation_events"]), what
    assert np.array_equal(r.work_units, o["work_units"]), what


def main():
    for name in ("c1", "mixed", "verify", "m1024"):
        pk = load_batch(name).astype(np.float32)
        ref = load_npz(f"ref32_{name}.npz")
        r = P.solve_packed(pk)
        feas = r.status.astype(np.int32) != O.INFEASIBLE
        assert np.array_equal(feas, ref["feasible"].astype(bool)), name
        for k in ("x", "y", "value"):
            assert np.array_equal(getattr(r, k)[feas], ref[k][feas]), (name, k)
        assert np.array_equal(r.work_units, ref["work_units"]), name
    sizes = np.array([29, 31, 32, 60, 61, 92, 93, 124, 125, 156, 157, 188, 189, 284, 285, 316,
                      317, 540, 572, 573, 1000, 1024, 1052], np.int32)
    pb = P.PackedBatch.generate(np.repeat(sizes, 40), 31).astype(np.float32)
    same(P.solve_packed(pb), O.solve_batch(pb, threads=16), "edges")
    for m, n, seed in ((128, 4096, 3), (500, 2048, 7), (1024, 1024, 2)):
        pb = P.PackedBatch.generate(np.full(n, m, np.int32), seed).astype(np.float32)
        same(P.solve_packed(pb), O.solve_batch(pb, threads=16), f"m={m}")
    print("variant FS=%s GRP=%s ok" % (os.environ.get("LP2D_B200_FS", "default"),
                                        os.environ.get("LP2D_B200_GRP", "default")))


if __name__ == "__main__":
    main()
