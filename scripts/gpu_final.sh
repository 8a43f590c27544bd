#!/bin/bash
# Round-end measurement: scripts/gpu_measure.sh plus one ncu --set full
# capture of the dominant solve kernel per config and the c4 launch list.
cd "${GRAFT_REPO_ROOT:-.}"
bash scripts/gpu_measure.sh
cap() {  # tag, kernel regex, config args...
  local tag=$1 k=$2; shift 2
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -s 2 \
    -o gpurun_out/full_$tag -f python bench.py "$@" --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_$tag.log 2>&1
}
# (reports are summarised here and deleted: gpurun returns at most 64 MiB)
cap c2 k_solve_fx --config c2
cap c3 k_solve_fx --config c3
cap c5 k_solve_warp --config c5
cap c2f64 k_solve_warp --config c2 --dtype f64
cap c4lanes k_solve_lanes --config c4
bash scripts/ncu_launches.sh c4 > gpurun_out/c4_kernels.txt 2>&1
for r in gpurun_out/full_*.ncu-rep; do
  t=$(basename $r .ncu-rep); t=${t#full_}
  n=16384; case $t in c3) n=131072;; c5) n=524288;; c4*) n=0;; esac
  python profiles/ncu_summary.py $r > gpurun_out/r02_${t}_ncu_summary.txt 2>&1
  [ $n -gt 0 ] && python profiles/ncu_hotspots.py $r $n > gpurun_out/r02_${t}_sass_hotspots.txt 2>&1
  python scripts/ncu_traffic.py $r $t >> gpurun_out/traffic_r02.txt 2>&1
done
[ -n "${KEEP_REPS:-}" ] || rm -f gpurun_out/full_*.ncu-rep
echo final-done
