timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gs1d or gs2d or golden" -p no:cacheprovider 2>&1 | tail -2
timeout 120 python tools/profile_run.py --config 4 --reps 2 | tail -1
timeout 60 python tools/profile_run.py --config 2 --reps 2 | tail -1
