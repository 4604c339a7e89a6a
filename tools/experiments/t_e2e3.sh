# skewed-band pipelined drop-in path (config 3 e2e): parity, then band sweep with timeline
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "e2e_bands or jacobi2d_depths or slab" 2>&1 | tail -2
for b in 256 512 1024 2048; do
  TVS_E2E_TRACE=1 TVS_E2E_BANDS=$b timeout 300 python -c "
import bench, statistics
t, nb, _ = bench.e2e_time(bench.CONFIGS[3], 3, 1)
print('band $b e2e ms', [round(x,1) for x in t], 'GSt/s', round(16384*16384*200/statistics.mean(t)/1e6,1))
" 2>&1 | tail -3
done
