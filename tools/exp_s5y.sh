set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py tests/test_acceptance_gpu.py -m gpu -x -q -k "1d or heat1d or golden or acceptance or fma or pinned or jacobi1d or config1" 2>&1 | tail -2
timeout 300 python tools/profile_run.py --config 1 --reps 4 2>&1 | tail -3
