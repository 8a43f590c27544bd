#!/bin/bash
# K6 group width sweep: per-size timing for LP2D_B200_GRP_G in $GS.
cd "${GRAFT_REPO_ROOT:-.}"
SIZES=${SIZES:-"40 131072 60 131072 100 65536 128 131072 150 65536 180 65536"}
for gw in ${GS:-4 16}; do
  echo "== G=$gw"; LP2D_B200_GRP_G=$gw timeout 300 python scripts/time_sizes.py f32 $SIZES 2>&1 | tail -8
done
