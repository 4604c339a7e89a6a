timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sizes or gauss_seidel_orders" -p no:cacheprovider 2>&1 | tail -15
for c in 1 2 4 8; do echo "== CS=$c"; TVS_GS2D_CLUSTER=$c timeout 120 python tools/profile_run.py --config 4 --reps 2 | tail -1; TVS_GS2D_CLUSTER=$c timeout 120 python tools/shape_run.py gs2d9p 8192 2048 --T 100 | tail -1; done
