timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sizes or gauss_seidel_orders or golden" -p no:cacheprovider 2>&1 | tail -2
for s in "8192 8192" "8192 2048" "4096 4096"; do timeout 120 python tools/shape_run.py gs2d9p $s --T 100 2>&1 | tail -1; done
timeout 120 python tools/profile_run.py --config 5 --T 4 --reps 2 | tail -1; timeout 120 python tools/profile_run.py --config 5 --T 4 --fma allow --reps 2 | tail -1
