set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py tests/test_acceptance_gpu.py tests/test_full_grid.py -m gpu -x -q -k "1d or heat1d or golden or acceptance or fma or pinned or jacobi1d or config1 or graph or repeated or thread" 2>&1 | tail -2
timeout 300 python tools/profile_run.py --config 1 --reps 3 2>&1 | tail -2
timeout 300 python -c "
import bench, statistics
t, nb, _ = bench.e2e_time(bench.CONFIGS[1], 20, 5)
print('config 1 e2e ms', round(statistics.mean(t), 4), 'GSt/s', round(2**20 * 1000 / statistics.mean(t) / 1e6, 1))
"
