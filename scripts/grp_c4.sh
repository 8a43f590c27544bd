#!/bin/bash
# config 4 with K6 on the m <= 60 class (LP2D_B200_GRP=2) against K4 (default), alternating
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for g in 0 2 0 2; do
  LP2D_B200_GRP=$g timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 20 > gpurun_out/g.json 2> gpurun_out/g.err
  python -c "
import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1])
print('c4 GRP=$g', 'ms/step %.4f' % d['ms_per_step'], 'kernel_ms %.4f' % d['roofline']['kernel_ms'])" || tail -5 gpurun_out/g.err
done
