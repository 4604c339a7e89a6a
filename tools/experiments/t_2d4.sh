timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "jacobi2d or golden or slab or plan" -p no:cacheprovider 2>&1 | tail -2
timeout 120 python tools/parity_quick.py heat2d | tail -1
for d in 3 4 5 6 7 8 9; do timeout 60 python tools/profile_run.py --config 3 --T 48 --depth $d --reps 3 | tail -1; done
