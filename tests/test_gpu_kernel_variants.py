"""Every fp32-storage kernel variant (K4 register/tail classes, K5
insertion-order classes; the library picks per size class, the A/B knob
LP2D_B200_FS forces either) is bit-identical to the reference on the same
inputs. Each variant runs in its own process (the knob is read once)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("knobs", [{"LP2D_B200_FS": "0"}, {"LP2D_B200_FS": "all"},
                                   {"LP2D_B200_GRP": "6"}, {"LP2D_B200_GRP": "2"},
                                   {"LP2D_B200_ORDER": "0"}],
                         ids=["k4", "k5-all", "k6-all", "k6-small", "order-largest-first"])
def test_fp32_kernel_variant_parity(knobs):
    """K4 (the default warp classes), K5 for every warp class, K6 lane groups
    for every class up to m = 188 or for m <= 60 only, and the mixed-batch
    class launches in the largest-first order."""
    env = dict(os.environ, **knobs)
    r = subprocess.run([sys.executable, os.path.join(HERE, "variant_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("chunk", ["4096", "70000"])
def test_host_mode_chunk_pipeline(chunk):
    """Many chunks per shard (two device slots reused in turn, pinned and
    pageable buffers, the lane_stats histogram accumulated over chunks)."""
    env = dict(os.environ, LP2D_B200_CHUNK_ELEMS=chunk)
    r = subprocess.run([sys.executable, os.path.join(HERE, "chunk_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]


def test_randomised_stress_parity():
    """scripts/stress_parity.py: perturbed instances (duplicates, scaled
    copies, constraints through a common point, nearly parallel bundles,
    axis-aligned rows, rescaled LPs, objectives along a constraint normal)
    over every size class, both storage types and both schedulers, each solve
    bit-identical to the oracle. (The committed run used 350 seeds.)"""
    root = os.path.dirname(HERE)
    r = subprocess.run([sys.executable, os.path.join(root, "scripts", "stress_parity.py"), "12"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
