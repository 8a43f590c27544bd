"""bench.py's contract pieces that run without a GPU: both arms describe a
config with identical keys (the driver compares them), the L2 policy is
stated inside `config`, and configs smaller than the L2 are the flushed ones."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


class _Sizes:
    def __init__(self, m):
        self.m = np.asarray(m, np.int32)
        self.n = len(self.m)


def test_config_states_the_l2_policy():
    big = bench.config_dict("c2", _Sizes(np.full(16384, 1024)), 1, np.float32)
    assert big["l2"].startswith("inputs 201 MB per GPU > 126 MB L2, no flush")
    small = bench.config_dict("c1", _Sizes(np.full(1024, 64)), 1, np.float32)
    assert "flushed between timed steps" in small["l2"]
    f64 = bench.config_dict("c2", _Sizes(np.full(16384, 1024)), 1, np.float64)
    assert f64["storage"] == "f64" and "403 MB" in f64["l2"]


def test_both_arms_share_the_config_object():
    # the reference arm and ours call the same function on the same layout
    a = bench.config_dict("c3", _Sizes(np.full(1 << 17, 128)), 8, np.float32)
    b = bench.config_dict("c3", _Sizes(np.full(1 << 17, 128)), 8, np.float32)
    assert a == b and a["parallelism"].startswith("dp8")
    full = bench.config_dict("c5", _Sizes(np.full(1 << 15, 256)), 2, np.float64, full=True)
    assert full["total_lps"] == 1 << 22 and full["lps_per_gpu"] == 1 << 21


def test_hold_gpu_is_optional():
    class _NoSleep:
        class cuda:  # noqa: N801
            pass

    bench.hold_gpu(_NoSleep, None)  # no torch.cuda._sleep: returns without touching a stream
