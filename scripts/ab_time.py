"""A/B timing of library variants (paper_1902_04995_b200/lib/variants/*.so)
on one config: each variant in its own process (LP2D_B200_LIB), device
kernel time of the default solve."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1]
names = sys.argv[2:]
for n in names:
    env = dict(os.environ)
    if n != "base":
        env["LP2D_B200_LIB"] = os.path.join(ROOT, "paper_1902_04995_b200", "lib", "variants", n + ".so")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--no-cpu-baseline",
                        "--steps", "10", "--e2e-steps", "1"], capture_output=True, text=True, env=env)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        print("%-8s %s kernel %.4f ms  pipelined %.4f ms/step  frac %.3f" % (
            n, cfg, d["roofline"]["kernel_ms"], d["ms_per_step"], d["roofline"]["frac"]), flush=True)
    except Exception:
        print(n, "FAILED", r.stderr[-600:], flush=True)
