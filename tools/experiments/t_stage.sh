# 2D drop-in: contiguous band copies through host-layout staging rows vs pitched 2D copies
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pinned or drop_in or e2e or plan or concurrent" -p no:cacheprovider 2>&1 | tail -2
for st in 0 1; do
  echo "== TVS_E2E_STAGE=$st"
  TVS_E2E_STAGE=$st timeout 300 python tools/e2e_pipe_probe.py 2>&1 | grep -v "^pipe\|^bulk"
  TVS_E2E_STAGE=$st timeout 300 python bench.py --config 3 --no-all --no-cpu --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d['gpu_launches'])"
done
