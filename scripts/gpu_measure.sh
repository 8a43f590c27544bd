#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench lines for every config (and
# the full-size / fp64-storage variants), the reference arm on the same
# configs, and the ncu launch list of the default bench. Outputs: gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
run() {  # name, args...
  local name=$1; shift
  timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err
  timeout 900 python bench.py --impl reference "$@" > gpurun_out/ref_$name.json 2> gpurun_out/ref_$name.err
}
run c2
run c1 --config c1
run c3 --config c3
run c4 --config c4
run c5 --config c5
run c2f64 --config c2 --dtype f64
run c3full --config c3 --full --steps 5
run c5full --config c5 --full --steps 5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/c2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_bench.log 2>&1
echo done
