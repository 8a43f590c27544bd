#!/bin/bash
# K6 (lane groups) A/B: parity of the default selection, per-size timing with
# K6 on every class up to m = 188 (LP2D_B200_GRP=6) and off (=0, the default), config 3/4 bench lines.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python tests/variant_check.py > gpurun_out/grp_variant.log 2>&1; echo "variant rc=$?"; tail -3 gpurun_out/grp_variant.log
SIZES=${SIZES:-"40 131072 60 131072 100 65536 128 131072 150 65536 180 65536"}
for mode in 6 0; do
  echo "== LP2D_B200_GRP=$mode"
  LP2D_B200_GRP=$mode timeout 300 python scripts/time_sizes.py f32 $SIZES 2>&1 | tail -8
done
for c in ${CFGS:-c3 c4}; do
  for mode in 6 0; do
    LP2D_B200_GRP=$mode timeout 600 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/grp_${c}_${mode}.json 2> gpurun_out/grp_${c}_${mode}.err
    python -c "
import json; d=json.loads(open('gpurun_out/grp_${c}_${mode}.json').read().strip().splitlines()[-1])
print('$c GRP=$mode', 'ms/step %.4f' % d['ms_per_step'], 'kernel_ms %.4f' % d['roofline']['kernel_ms'], 'frac %.3f' % d['roofline']['frac'])" || tail -5 gpurun_out/grp_${c}_${mode}.err
  done
done
