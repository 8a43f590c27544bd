#!/bin/bash
# one ncu --set full capture of K6 (lane groups) on a uniform m = 128 batch
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_solve_grp -c 1 -s 2 \
  -o gpurun_out/full_grp -f env LP2D_B200_GRP=6 python scripts/time_sizes.py f32 128 131072 > gpurun_out/ncu_grp.log 2>&1
python profiles/ncu_summary.py gpurun_out/full_grp.ncu-rep > gpurun_out/grp_ncu_summary.txt 2>&1
python profiles/ncu_hotspots.py gpurun_out/full_grp.ncu-rep 131072 > gpurun_out/grp_hotspots.txt 2>&1
rm -f gpurun_out/full_grp.ncu-rep
cat gpurun_out/grp_ncu_summary.txt; head -45 gpurun_out/grp_hotspots.txt
