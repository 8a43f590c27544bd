#!/bin/bash
# Round-end measurement: parity tests, smoke, bench lines for every config and
# the reference arm, the c2 launch list, one ncu --set full capture per config.
cd "${GRAFT_REPO_ROOT:-.}"
bash scripts/gpu_measure.sh
for c in c2 c3 c5; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve_warp -c 1 -s 2 \
    -o gpurun_out/full_$c -f python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_$c.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve_lanes -c 1 -s 1 \
  -o gpurun_out/full_c4lanes -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_c4lanes.log 2>&1
bash scripts/ncu_launches.sh c4 > gpurun_out/c4_kernels.txt 2>&1
echo final-done
