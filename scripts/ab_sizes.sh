#!/bin/bash
# A/B of the fp32-storage kernels over uniform sizes: K5 (default) vs K4 (LP2D_B200_FS=0).
cd "${GRAFT_REPO_ROOT:-.}"
S="40 131072 100 131072 128 131072 150 131072 180 131072 250 65536 300 65536 500 32768 1000 16384 1024 16384"
echo "== K5"; timeout 300 python scripts/time_sizes.py f32 $S
echo "== K4"; LP2D_B200_FS=0 timeout 300 python scripts/time_sizes.py f32 $S
