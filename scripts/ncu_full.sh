#!/bin/bash
# One ncu --set full capture of the solve kernel of a config (default c2),
# with source; the report comes back in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${1:-x}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:${3:-k_solve_fx} -c 1 -s 2 \
  -o gpurun_out/full_$TAG -f python bench.py --config ${2:-c2} --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -n 3 gpurun_out/ncu_full_$TAG.log
ls -la gpurun_out/full_$TAG.ncu-rep
