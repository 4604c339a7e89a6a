timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sizes or gauss_seidel_orders or golden or plan_api or matrix" -p no:cacheprovider 2>&1 | tail -2
for s in "8192 8192" "8192 2048"; do timeout 120 python tools/shape_run.py gs2d9p $s --T 100 2>&1 | tail -1; done
timeout 120 python tools/shape_run.py gs2d9p 8192 8192 --T 128 2>&1 | tail -1
