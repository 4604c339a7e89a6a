set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_acceptance_gpu.py tests/test_shard.py -m gpu -x -q -k "2d or heat2d or jacobi2d or golden or acceptance or shard or pipelined or staged or fma" 2>&1 | tail -2
timeout 300 python tools/c3_depth.py 8 2>&1 | tail -1
timeout 300 python tools/c3_depth.py 8 2>&1 | tail -1
