#!/bin/bash
# compute-sanitizer over scripts/sanitize_run.py for each kernel selection.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
out=gpurun_out/sanitizer.txt
: > $out
for env in "" "LP2D_B200_FS=all" "LP2D_B200_FS=0 LP2D_B200_CHUNK_ELEMS=3000"; do
  for tool in memcheck synccheck racecheck; do
    echo "== $tool ${env:-default}" >> $out
    env $env timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_run.py 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize run|Error|Invalid|Warning: Race" | sort | uniq -c | head -20 >> $out
  done
done
cat $out
