set -x
echo "== default (first block requested with the prologue)"; timeout 600 python tools/gs2d_lane_check.py 2>&1 | tail -3
echo "== G=4"; TVSTENCIL_LIB=build/var/gsl_g4/libtvstencil.so timeout 600 python tools/gs2d_lane_check.py 2>&1 | tail -3
