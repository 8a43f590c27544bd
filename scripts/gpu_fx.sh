#!/bin/bash
# K4 iteration: path statistics + timings for the given configs, then GPU tests.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
LP2D_B200_FX_STATS=1 timeout 600 python scripts/fx_stats.py ${@:-c2} 2>&1 | tail -n 8
for c in ${@:-c2}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/q_bench_$c.json 2> gpurun_out/q_bench_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/q_bench_$c.json').read().strip().splitlines()[-1])
print('$c', 'ms/step %.4f' % d['ms_per_step'], 'kernel_ms %.4f' % d['roofline']['kernel_ms'], 'frac %.3f' % d['roofline']['frac'])" || tail -5 gpurun_out/q_bench_$c.err
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
tail -n 3 gpurun_out/q_pytest.log
grep -E "^E |FAILED" gpurun_out/q_pytest.log | head -8
