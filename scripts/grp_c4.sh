#!/bin/bash
# config 4 with K6 on class 1 only (LP2D_B200_GRP=2; G = 8 or 4) against K4 everywhere
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for v in "0 8" "2 8" "2 4" "0 8" "2 8"; do
  set -- $v
  LP2D_B200_GRP=$1 LP2D_B200_GRP_G=$2 timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 20 > gpurun_out/g.json 2> gpurun_out/g.err
  python -c "
import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1])
print('c4 GRP=$1 G=$2', 'ms/step %.4f' % d['ms_per_step'], 'kernel_ms %.4f' % d['roofline']['kernel_ms'])" || tail -5 gpurun_out/g.err
done
