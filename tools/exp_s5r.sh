set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_shard.py -m gpu -x -q -k "3d or jac3d or shard" 2>&1 | tail -3
echo "== frame 32"; TVS_J3D_FRAME=32 timeout 300 python tools/c5_time.py 2>&1 | tail -2
echo "== frame 64"; TVS_J3D_FRAME=64 timeout 300 python tools/c5_time.py 2>&1 | tail -2
