timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sizes or gauss_seidel_orders" -p no:cacheprovider 2>&1 | tail -2
for c in 1 4 8; do for s in "8192 8192" "8192 2048"; do echo -n "CS=$c "; TVS_GS2D_CLUSTER=$c timeout 120 python tools/shape_run.py gs2d9p $s --T 100 2>&1 | tail -1; done; done
TVS_GS2D_CLUSTER=1 timeout 120 build/var/gs2d_trace 8192 8192 100 | sed -n 3,6p
