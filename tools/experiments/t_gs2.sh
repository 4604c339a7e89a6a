timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -k "gauss_seidel_orders or golden" -p no:cacheprovider 2>&1 | tail -4
timeout 60 python tools/profile_run.py --config 4 --reps 3
for w in 1 2 4; do TVS_GS1D_WARPS=$w timeout 60 python tools/profile_run.py --config 2 --reps 2 | tail -1; done
