timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -3
for d in 2 4 6 8; do python tools/profile_run.py --config 3 --T 48 --depth $d --reps 2 | tail -1; done
python tools/profile_run.py --config 2 --T 128 --reps 2
python tools/profile_run.py --config 2 --reps 2
