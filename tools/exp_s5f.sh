set -x
echo "== v3"; timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
echo "== v3 weak"; TVSTENCIL_LIB=build/var/gsl_v3_weak/libtvstencil.so timeout 300 python tools/gs2d_lane_check.py 2>&1 | tail -4
