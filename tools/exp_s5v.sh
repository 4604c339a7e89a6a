set -x
echo "== rp1 noup nobar"; TVSTENCIL_LIB=build/var/gsl_nobar/libtvstencil.so timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
echo "== rp2 noup nobar"; TVSTENCIL_LIB=build/var/gsl_rp2_nobar/libtvstencil.so timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
