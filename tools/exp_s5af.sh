set -x
timeout 600 python tools/gs2d_lane_check.py 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_acceptance_gpu.py -m gpu -x -q -k "gs2d or lane or gs or acceptance or repeat" 2>&1 | tail -2
