#!/bin/bash
# Per-kernel durations (ncu, serialised, cold) of one solve of a config.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
C=${1:-c4}
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__grid_size,launch__registers_per_thread --clock-control none -c 60 --csv \
  --log-file gpurun_out/launches_$C.csv python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python3 - "$C" <<'PY'
import csv,sys,collections
txt=open("gpurun_out/launches_%s.csv"%sys.argv[1]).read(); import io; rows=list(csv.DictReader(io.StringIO(txt[txt.index(chr(34)+"ID"):])))
d=collections.OrderedDict()
for r in rows:
    k=(r['ID'],r['Kernel Name'][:70])
    d.setdefault(k,{})[r['Metric Name']]=r['Metric Value']
for (i,n),m in list(d.items())[:60]:
    print(i,n,m.get('gpu__time_duration.sum'),m.get('smsp__inst_executed.sum'),m.get('launch__grid_size'),m.get('launch__registers_per_thread'))
PY
