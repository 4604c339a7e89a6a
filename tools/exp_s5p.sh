set -x
echo "== uniform warp index (slack 0)"; timeout 600 python tools/gs2d_lane_check.py 2>&1 | tail -3
echo "== slack 1 (lag / skew 3, prefetch)"; TVSTENCIL_LIB=build/var/gsl_slack1/libtvstencil.so timeout 600 python tools/gs2d_lane_check.py 2>&1 | tail -3
