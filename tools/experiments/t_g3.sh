timeout 200 python tools/parity_quick.py gs2d9p | tail -2; timeout 200 python -m pytest tests/test_gpu_parity.py -q -x -k "gauss_seidel_orders or golden or plan" -p no:cacheprovider 2>&1 | tail -2
timeout 60 python tools/profile_run.py --config 4 --reps 2 | tail -1
