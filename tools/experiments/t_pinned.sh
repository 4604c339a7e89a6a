# e2e with library-allocated pinned Grids (tvs_host_alloc) vs registered numpy pages
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "pinned or drop_in" -p no:cacheprovider 2>&1 | tail -2
for host in register alloc; do
  for c in 3 5 1; do
    echo "== $host config $c"
    TVS_BENCH_HOST=$host timeout 300 python bench.py --config $c --no-all --no-cpu --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"
  done
done
