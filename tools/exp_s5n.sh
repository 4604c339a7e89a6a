set -x
timeout 600 python tools/gs2d_lane_check.py 2>&1 | tail -3
