"""The verify / replay tool (tests/lp2d_verify.py), the drop-in's version of
`lp2d-bench verify` (bench.hpp:291-378, lp2d_bench.cpp:173-183)."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
TOOL = os.path.join(HERE, "lp2d_verify.py")


def run(*args):
    return subprocess.run([sys.executable, TOOL, *args], capture_output=True, text=True,
                          timeout=600)


def test_bad_arguments_exit_2():
    assert run("verify", "--count", "0").returncode == 2
    assert run("verify", "--max-size", "600").returncode == 2
    assert run("nonsense").returncode == 2
    assert run("replay", "/nonexistent.lp2d").returncode == 2


def test_xoshiro_matches_the_reference_kats():
    sys.path.insert(0, HERE)
    import json

    import lp2d_verify as V

    kat = json.load(open(os.path.join(HERE, "golden", "kat.json")))
    r = V.Xoshiro(0)
    assert [r.next() for _ in range(3)] == kat["xoshiro_seed0_first3"]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_verify_and_replay_on_the_gpu(tmp_path, dtype):
    r = run("verify", "--count", "400", "--max-size", "128", "--dtype", dtype,
            "--dump", str(tmp_path), "--dump-all")
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 disagreements" in r.stdout
    files = sorted(os.listdir(tmp_path))
    assert len(files) == 400
    rr = run("replay", str(tmp_path / files[7]), "--dtype", dtype)
    assert rr.returncode == 0, rr.stdout + rr.stderr
    assert "balanced:" in rr.stdout and "serial:" in rr.stdout
