timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "jacobi2d or golden or fma or slab or plan" -p no:cacheprovider 2>&1 | tail -2
for d in 2 3 4 5 6 8 10; do timeout 60 python tools/profile_run.py --config 3 --T 48 --depth $d --reps 2 | tail -1; done
