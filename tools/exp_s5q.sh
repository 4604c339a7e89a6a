set -x
echo "== slack 0 noup"; TVSTENCIL_LIB=build/var/gsl_s0_noup/libtvstencil.so timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
echo "== slack 1 noup"; TVSTENCIL_LIB=build/var/gsl_s1_noup/libtvstencil.so timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
