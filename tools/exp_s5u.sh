set -x
echo "== rp2"; TVSTENCIL_LIB=build/var/gsl_rp2/libtvstencil.so timeout 600 python tools/gs2d_lane_check.py 2>&1 | tail -8
echo "== rp2 noup"; TVSTENCIL_LIB=build/var/gsl_rp2_noup/libtvstencil.so timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
echo "== default"; timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
