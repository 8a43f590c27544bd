"""The host-mode multi-device driver (C ABI, one host thread per device,
chunked H2D/solve pipeline per shard) exercised on CPU through the library's
test-only mock devices (LP2D_B200_MOCK_DEVICES): every LP is visited exactly
once, its result lands in its own slot, shards are contiguous LP ranges
balanced by sum(m + 4) exactly as lp2dgpu_partition cuts them (batch.hpp:335-
351's worker split, re-expressed per device), and chunks respect the element
budget."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def run_mock(sizes, n_gpus, mock, chunk, dt="f32"):
    env = dict(os.environ, LP2D_B200_MOCK_DEVICES=str(mock), LP2D_B200_CHUNK_ELEMS=str(chunk))
    r = subprocess.run([sys.executable, os.path.join(HERE, "mock_driver_check.py"),
                        ",".join(map(str, sizes)), str(n_gpus), dt], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("n_gpus,mock,chunk", [(0, 4, 1000), (2, 8, 64), (8, 8, 5000),
                                               (3, 3, 1 << 24)])
def test_mock_shards_and_chunks(P, n_gpus, mock, chunk):
    rng = np.random.default_rng(7)
    sizes = rng.integers(0, 700, 97).astype(np.int32)
    d = run_mock(sizes, n_gpus, mock, chunk)
    n = len(sizes)
    use = min(n_gpus if n_gpus > 0 else mock, mock, n)
    assert all(s == 254 for s in d["status"])  # LP2D_MOCK
    assert d["x"] == list(range(n))            # each LP's result in its own slot
    assert d["wu"] == sizes.tolist()
    # shards: contiguous, in device order, the partition's cuts
    cut = np.zeros(use + 1, np.int64)
    P.lp2d.N.lib().lp2dgpu_partition(n, sizes.ctypes.data, use, cut.ctypes.data)
    shard = np.asarray(d["shard"], np.int64)
    for g in range(use):
        assert (shard[cut[g]:cut[g + 1]] == g).all()
    # chunks: contiguous runs inside a shard, each within the element budget
    # (or a single LP), covering the shard; greedy except that the shard's
    # last greedy chunk may be cut in two (the taper)
    off = np.asarray(d["offset"], np.int64)
    first = np.asarray(d["chunk"], np.int64)
    for g in range(use):
        lo, hi = cut[g], cut[g + 1]
        runs = []
        j = lo
        while j < hi:
            c0 = first[j]
            assert c0 == j
            k = j
            while k < hi and first[k] == c0:
                k += 1
            assert k - j == 1 or off[k] - off[j] <= chunk
            runs.append((j, k))
            j = k
        for i, (j, k) in enumerate(runs[:-1]):
            tapered = i == len(runs) - 2 and off[hi] - off[j] <= chunk
            if not tapered:  # greedy: the next LP would have overflowed the chunk
                assert off[k + 1] - off[j] > chunk


def test_partition_balances_work(P):
    sizes = np.array([8192] + [8] * 500 + [1024] * 20, np.int32)
    for parts in (2, 3, 8):
        cut = np.zeros(parts + 1, np.int64)
        P.lp2d.N.lib().lp2dgpu_partition(len(sizes), sizes.ctypes.data, parts, cut.ctypes.data)
        assert cut[0] == 0 and cut[-1] == len(sizes) and (np.diff(cut) >= 0).all()
        w = np.array([(sizes[cut[g]:cut[g + 1]] + 4).sum() for g in range(parts)])
        # every boundary is the first index at which the prefix reaches k/parts of the total
        tot = (sizes + 4).sum()
        pre = np.concatenate([[0], np.cumsum(sizes + 4)])
        for k in range(1, parts):
            assert pre[cut[k]] >= tot * k / parts and (cut[k] == 0 or pre[cut[k] - 1] < tot * k / parts)
        assert w.sum() == tot
