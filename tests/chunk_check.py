"""Host-mode chunk pipeline on the GPU (run in a fresh process with a small
LP2D_B200_CHUNK_ELEMS): results of pageable and pinned host buffers, fp32 and
fp64 storage, with the lane_stats histogram, equal the oracle's."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import conftest  # noqa: F401,E402  (paths)
import oracle_py as O  # noqa: E402
import paper_1902_04995_b200 as P  # noqa: E402
import torch  # noqa: E402


def pinned(a):
    t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
    v = t.numpy().view(a.dtype).reshape(a.shape)
    v[...] = a
    return v


def check(r, o, what):
    st = r.status.astype(np.int32)
    assert np.array_equal(st, o["status"]), what
    assert np.array_equal(r.pair, o["pair"]), what
    feas = o["status"] != O.INFEASIBLE
    for k in ("x", "y", "value"):
        assert np.array_equal(getattr(r, k)[feas], o[k][feas]), (what, k)
    assert np.array_equal(r.work_units, o["work_units"]), what


def main():
    rng = np.random.default_rng(3)
    sizes = np.concatenate([rng.integers(0, 1100, 600), [5000, 20, 9000]]).astype(np.int32)
    base = P.PackedBatch.generate(sizes, 9)
    for dt in (np.float32, np.float64):
        pb = base.astype(dt) if dt == np.float32 else base
        o = O.solve_batch(pb, threads=16)
        W = 64
        rows = (pb.n + W - 1) // W
        h1 = np.zeros(rows * (int(sizes.max()) + 1), np.uint32)
        r1 = P.solve_packed(pb, P.BlockConfig(block_width=W), iter_hist=h1)
        check(r1, o, f"pageable {dt.__name__}")
        # permutations generated on the device from the generator's seeds
        noperm = P.PackedBatch(pb.m, pb.offset, pb.ax, pb.ay, pb.b, None, pb.c, pb.M)
        r3 = P.solve_packed(noperm, P.BlockConfig(block_width=W), perm_seed=P.PermSeed(9))
        check(r3, o, f"perm_seed {dt.__name__}")
        pp = P.PackedBatch(*(pinned(a) for a in (pb.m, pb.offset, pb.ax, pb.ay, pb.b, pb.perm,
                                                  pb.c, pb.M)))
        out = P.PackedResult(*(pinned(np.zeros(sh, d)) for sh, d in (
            (pb.n, np.uint8), (pb.n, np.float64), (pb.n, np.float64), (pb.n, np.float64),
            ((pb.n, 2), np.int32), (pb.n, np.uint32), (pb.n, np.uint64))))
        h2 = np.zeros_like(h1)
        r2 = P.solve_packed(pp, P.BlockConfig(block_width=W), out=out, iter_hist=h2)
        check(r2, o, f"pinned {dt.__name__}")
        assert np.array_equal(h1, h2)
        # the histogram accounts for every violation event
        assert int(h1.sum()) == int(o["violation_events"].sum())
    print("chunks ok")


if __name__ == "__main__":
    main()
