#!/bin/bash
# Iteration call: GPU parity tests, bench lines for the given configs, and one
# ncu --set full capture of the first config's solve kernel (regex $KERN).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-it}
KERN=${KERN:-k_solve_fs}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -n 2 gpurun_out/${TAG}_pytest.log; grep -E "^E |FAILED" gpurun_out/${TAG}_pytest.log | head -8
for c in ${@:-c2}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench_$c.json').read().strip().splitlines()[-1])
print('$c', 'ms/step %.4f' % d['ms_per_step'], 'kernel_ms %.4f' % d['roofline']['kernel_ms'], 'frac %.3f' % d['roofline']['frac'])" || tail -5 gpurun_out/${TAG}_bench_$c.err
done
if [ -z "$NONCU" ]; then
  c=${1:-c2}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$KERN -c 1 -s 2 \
    -o gpurun_out/full_${TAG} -f python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_${TAG}.log 2>&1
  tail -n 1 gpurun_out/ncu_full_${TAG}.log
fi
