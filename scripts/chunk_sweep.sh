cd "${GRAFT_REPO_ROOT:-.}"
for c in c4 c3 c2; do for ce in 1048576 2097152 4194304 8388608 33554432; do
  LP2D_B200_CHUNK_ELEMS=$ce timeout 300 python bench.py --config $c --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', $ce, '%.4g' % d['e2e']['value'], '%.4g' % d['e2e_perm_seed']['value'])"
done; done
