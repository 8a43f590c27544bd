"""The CPU oracle (oracle/) pinned against the reference's known answers and
the committed golden fixtures made from the unmodified reference
(tests/golden/make_golden.py). CPU only."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_batch, load_npz

KAT = json.load(open(os.path.join(GOLDEN, "kat.json")))


def test_rng_known_answers(O):
    # rng.hpp:13-68 (SURVEY.md §8(c) probe KATs)
    assert [int(v) for v in O.xoshiro_first(0, 3)] == KAT["xoshiro_seed0_first3"]
    assert O.derive_seed(1, 0) == KAT["derive_seed_1_0"]
    assert O.derive_seed(1, 1) == KAT["derive_seed_1_1"]
    assert list(O.shuffle(10, 5)) == KAT["shuffle_10_5"]
    assert list(O.shuffle(16, 42)) == KAT["shuffle_16_42"]


def test_shuffle_is_a_permutation(O):
    # test_serial.cpp:142-160
    a, b, c = O.shuffle(1000, 5), O.shuffle(1000, 5), O.shuffle(1000, 6)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert np.array_equal(np.sort(a), np.arange(1000))


def test_frozen_oracle_value(O):
    # test_generate.cpp:20,90-101: frozen_value_seed42_m32 = -5161588.8190740123
    ax, ay, b, c, M, _ = O.gen(32, 42)
    assert [ax[0], ay[0], b[0]] == KAT["gen32_42_first_constraint"]
    direct = O.bruteforce(ax, ay, b, c, M)
    assert direct.status == O.OPTIMAL
    assert abs(direct.value - (-5161588.8190740123)) <= 1e-12 * 5161588.8190740123
    assert direct.value == KAT["bruteforce_gen32_42_value"]


def _solve_one(O, ax, ay, b, perm, c, M, dtype=np.float64):
    from types import SimpleNamespace

    m = len(ax)
    cap = (m + 7) // 8 * 8
    pad = lambda a: np.concatenate([np.asarray(a, dtype), np.zeros(cap - m, dtype)])
    pk = SimpleNamespace(n=1, offset=np.array([0, cap], np.int64), m=np.array([m], np.int32),
                         ax=pad(ax), ay=pad(ay), b=pad(b),
                         perm=np.concatenate([np.asarray(perm, np.uint32), np.zeros(cap - m, np.uint32)]),
                         c=np.asarray(c, dtype), M=np.asarray([M], dtype))
    return O.solve_batch(pk)[0]


def test_hand_cases(O):
    # test_serial.cpp:57-86, :129-140
    r = _solve_one(O, [1.0, 0.0], [0.0, 1.0], [1.0, 1.0], [0, 1], [1.0, 1.0], 10.0)
    assert r["status"] == O.OPTIMAL and (r["x"], r["y"], r["value"]) == (1.0, 1.0, 2.0)
    assert r["violation_events"] == 2 and r["work_units"] == 4 + 5
    assert sorted(r["pair"]) == [0, 1]
    r = _solve_one(O, [], [], [], [], [1.0, 1.0], 10.0)  # no constraints: box corner
    assert (r["x"], r["y"]) == (10.0, 10.0) and r["status"] == O.UNBOUNDED
    assert list(r["pair"]) == [-1, -3]
    for perm in ([0, 1], [1, 0]):  # contradictory x <= 0, x >= 1
        r = _solve_one(O, [1.0, -1.0], [0.0, 0.0], [0.0, -1.0], perm, [1.0, 1.0], 10.0)
        assert r["status"] == O.INFEASIBLE


@pytest.mark.parametrize("name", ["c1", "mixed", "verify", "m1024"])
def test_oracle_matches_reference_fixtures(O, name):
    """fp64 restatement == unmodified reference, bit for bit (incl. stats)."""
    pk = load_batch(name)
    ref = load_npz(f"ref_{name}.npz")
    o = O.solve_batch(pk)
    feas = o["status"] != O.INFEASIBLE
    assert np.array_equal(feas, ref["feasible"].astype(bool))
    for k in ("x", "y", "value"):
        assert np.array_equal(o[k][feas], ref[k][feas]), k
    assert np.array_equal(o["violation_events"], ref["violation_events"])
    assert np.array_equal(o["work_units"], ref["work_units"])


@pytest.mark.parametrize("name", ["c1", "mixed", "verify", "m1024"])
def test_oracle_extension_and_fp32_pinned(O, name):
    pk = load_batch(name)
    g = load_npz(f"oracle_{name}.npz")
    o64 = O.solve_batch(pk)
    assert np.array_equal(o64["status"], g["status64"]) and np.array_equal(o64["pair"], g["pair64"])
    o32 = O.solve_batch(pk.astype(np.float32))
    assert np.array_equal(o32["status"], g["status32"]) and np.array_equal(o32["pair"], g["pair32"])
    for k, gk in (("x", "x32"), ("y", "y32"), ("value", "value32"),
                  ("violation_events", "viol32"), ("work_units", "wu32")):
        assert np.array_equal(o32[k], g[gk]), k


def test_oracle_agrees_with_bruteforce(O):
    # bench.hpp:291-378 verify protocol on the committed verify stream
    pk = load_batch("verify")
    o = O.solve_batch(pk)
    for j in range(0, pk.n, 7):
        s, e = int(pk.offset[j]), int(pk.offset[j]) + int(pk.m[j])
        bf = O.bruteforce(pk.ax[s:e], pk.ay[s:e], pk.b[s:e], pk.c[2 * j:2 * j + 2], pk.M[j])
        assert (bf.status == O.INFEASIBLE) == (o[j]["status"] == O.INFEASIBLE)
        if bf.status != O.INFEASIBLE:
            a, b = bf.value, o[j]["value"]
            mag = max(abs(a), abs(b))
            step = 10.0 ** (np.floor(np.log10(mag)) - 4) if mag > 0 else 0
            assert a == b or abs(a - b) <= 0.5 * step


def test_unbounded_status_means_box_pair(O):
    pk = load_batch("mixed")
    o = O.solve_batch(pk)
    unb = o["status"] == O.UNBOUNDED
    assert unb.any()
    assert np.all((o["pair"][unb] < 0).any(axis=1))
    opt = o["status"] == O.OPTIMAL
    assert np.all(o["pair"][opt] >= 0)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(GOLDEN), "..", "oracle", "_ref", "liblp2d_ref.so")),
                    reason="reference build absent")
def test_reference_gen_mixed_kats(O):
    k = KAT["gen_mixed_64_1024_1"]
    assert k["violation_events"] == 7227 and k["total_wu"] == 147079
    assert k["checksum"] == pytest.approx(16797174.362085555, rel=1e-15)


@pytest.mark.parametrize("name", ["c1", "mixed", "verify", "m1024"])
def test_fp32_oracle_is_reference_on_rounded_instance(O, name):
    """fp32 configs: float storage, the reference's double arithmetic. The
    oracle's float entry point == the unmodified reference run on the
    fp32-rounded instance (widened to double), bit for bit incl. stats."""
    pk = load_batch(name).astype(np.float32)
    ref = load_npz(f"ref32_{name}.npz")
    o = O.solve_batch(pk)
    feas = o["status"] != O.INFEASIBLE
    assert np.array_equal(feas, ref["feasible"].astype(bool))
    for k in ("x", "y", "value"):
        assert np.array_equal(o[k][feas], ref[k][feas]), k
    assert np.array_equal(o["violation_events"], ref["violation_events"])
    assert np.array_equal(o["work_units"], ref["work_units"])
    g = load_npz(f"oracle_{name}.npz")
    assert np.array_equal(o["status"], g["status32"]) and np.array_equal(o["pair"], g["pair32"])
