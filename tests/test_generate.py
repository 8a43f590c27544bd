"""Product-side host instance synthesis (lp2d_generate.cpp) == the reference's
generators bit for bit (the oracle restatement and, when present, the
compiled reference). CPU only."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_batch

KAT = json.load(open(os.path.join(GOLDEN, "kat.json")))


def test_rng_and_shuffle_match_reference(P):
    assert P.derive_seed(1, 0) == KAT["derive_seed_1_0"]
    assert P.derive_seed(1, 1) == KAT["derive_seed_1_1"]
    assert list(P.shuffle(10, 5).order) == KAT["shuffle_10_5"]
    assert list(P.shuffle(16, 42).order) == KAT["shuffle_16_42"]


def test_gen_matches_oracle_and_reference(P, O):
    p = P.gen(32, 42)
    assert [p.constraints[0, 0], p.constraints[0, 1], p.constraints[0, 2]] == KAT["gen32_42_first_constraint"]
    assert list(p.c) == KAT["gen32_42_objective"]
    for m, seed, kind in ((64, 1, 0), (24, 5, 1), (1, 17, 1), (200, 9, 0)):
        q = P.gen(m, seed, P.GenKind(kind))
        ax, ay, b, c, M, _ = O.gen(m, seed, kind)
        assert np.array_equal(q.constraints[:, 0], ax) and np.array_equal(q.constraints[:, 2], b)
        assert tuple(q.c) == tuple(c) and q.bound_m == M


@pytest.mark.parametrize("name,sizes,count,seed", [
    ("c1", [64], 1024, 1), ("mixed", [3, 40, 150], 300, 123), ("m1024", [1024], 48, 2)])
def test_packed_generation_matches_reference_gen_mixed(P, name, sizes, count, seed):
    ref = load_batch(name)  # made by the reference's gen_mixed
    m = np.array([sizes[i % len(sizes)] for i in range(count)], np.int32)
    pb = P.PackedBatch.generate(m, seed, perm_bits=32)
    assert np.array_equal(pb.offset, ref.offset)
    for k in ("ax", "ay", "b", "c", "M"):
        assert np.array_equal(getattr(pb, k), getattr(ref, k)), k
    for j in range(count):
        o, mj = int(pb.offset[j]), int(pb.m[j])
        assert np.array_equal(pb.perm[o:o + mj], ref.perm[o:o + mj])


def test_generation_is_shard_invariant(P):
    m = np.full(100, 33, np.int32)
    full = P.PackedBatch.generate(m, 9)
    part = P.PackedBatch.generate(m[40:], 9, first=40)
    e0 = int(full.offset[40])
    assert np.array_equal(full.ax[e0:], part.ax) and np.array_equal(full.perm[e0:], part.perm)


def test_gen_mixed_batch_api(P):
    b = P.gen_mixed([16, 1024], 6, 55)
    assert [p.constraints.shape[0] for p in b.problems] == [16, 1024] * 3
    assert not np.array_equal(b.problems[0].constraints, b.problems[2].constraints)


def test_unbounded_kind_points_away_from_objective(P):
    p = P.gen(64, 3, P.GenKind.unbounded_random)
    a = p.constraints[:, :2]
    assert np.all(a @ np.asarray(p.c) <= -0.5 + 1e-12)


def test_pareto_sizes(P):
    import ctypes as C

    L = P.lp2d.N.lib()
    out = np.zeros(1 << 20, np.int32)
    n = L.lp2dgen_pareto_sizes(4, 8.0, 1.0, 8192, 1 << 24, len(out), out.ctypes.data)
    s = out[:n]
    assert s.min() >= 8 and s.max() <= 8192 and s.sum() >= 1 << 24
    assert 200_000 < n < 330_000  # E[m] = 8(1 + ln 1024) ~ 63.5
