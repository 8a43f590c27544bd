"""Copy a gpu_final.sh run (gpurun_out/) into profiles/r02_* and print the
DESIGN.md §6 measurement table."""
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, PR = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
rows = [("c1", "c1 1024×64 fp32"), ("c2", "**c2 16384×1024 fp32 (headline)**"),
        ("c2f64", "c2 16384×1024, fp64 storage"), ("c3", "c3 2^17×128 fp32 (1/8 of config 3)"),
        ("c3full", "c3 FULL 2^20×128 fp32, 1 GPU"), ("c4", "c4 Pareto mixed, Σm≈2^24 fp32"),
        ("c5", "c5 2^19×256 fp64 (1/8 of config 5)"), ("c5full", "c5 FULL 2^22×256 fp64, 1 GPU")]
for k, _ in rows:
    shutil.copy(os.path.join(G, f"bench_{k}.json"), os.path.join(PR, f"r02_bench_{k}.json"))
    shutil.copy(os.path.join(G, f"ref_{k}.json"), os.path.join(PR, f"r02_reference_{k}.json"))
for f in os.listdir(G):
    if f.startswith("r02_") and f.endswith(".txt"):
        shutil.copy(os.path.join(G, f), os.path.join(PR, f))
shutil.copy(os.path.join(G, "c2_launches.csv"), os.path.join(PR, "r02_c2_launches.csv"))
shutil.copy(os.path.join(G, "c4_kernels.txt"), os.path.join(PR, "r02_c4_kernels.txt"))
shutil.copy(os.path.join(G, "pytest_gpu.log"), os.path.join(PR, "r02_pytest_gpu.log"))
traffic = {}
for line in open(os.path.join(G, "traffic_r02.txt")):
    t, b = line.split()
    traffic[{"c2f64": "c2-f64"}.get(t, t)] = int(b)
traffic["note"] = ("dram__bytes_read.sum + dram__bytes_write.sum of one launch of the config's dominant "
                   "solve kernel, ncu --set full (profiles/r02_<tag>_ncu_summary.txt); keys: config, or "
                   "config-dtype for a non-default storage type")
json.dump(traffic, open(os.path.join(PR, "traffic.json"), "w"), indent=1)
out = ["| config | value (LP/s, device, 3-stream pipelined) | ms/step pipelined / isolated kernel | "
       "roofline frac (isolated kernel) | e2e LP/s (pinned host buffers, H2D+D2H in region) | e2e, "
       "permutations from seeds | reference arm LP/s (16 host threads) | e2e / reference |",
       "|---|---|---|---|---|---|---|---|"]
for k, name in rows:
    d = json.loads(open(os.path.join(PR, f"r02_bench_{k}.json")).read().strip().splitlines()[-1])
    r = json.loads(open(os.path.join(PR, f"r02_reference_{k}.json")).read().strip().splitlines()[-1])
    assert d["config"] == r["config"], k
    assert not d["clocks"]["reasons"], (k, d["clocks"])
    out.append("| %s | %.3g | %.4g / %.4g | %.3f | %.3g | %.3g | %.3g | %.1f× |" % (
        name, d["value"], d["ms_per_step"], d["roofline"]["kernel_ms"], d["roofline"]["frac"],
        d["e2e"]["value"], d["e2e_perm_seed"]["value"], r["value"], d["e2e"]["value"] / r["value"]))
print("\n".join(out))
