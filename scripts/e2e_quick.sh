#!/bin/bash
# e2e legs of bench.py for the given configs (host-pipeline tuning aid).
cd "${GRAFT_REPO_ROOT:-.}"
for c in ${@:-c1 c2 c3 c4 c5}; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', 'e2e %.4g' % d['e2e']['value'], 'perm_seed %.4g' % d['e2e_perm_seed']['value'], 'dev %.4g' % d['value'])"
done
