set -x
echo "== gate 0"; timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
for gt in 16 32 48; do echo "== gate $gt"; TVSTENCIL_LIB=build/var/gsl_gate$gt/libtvstencil.so timeout 600 python tools/gs2d_lane_check.py 2>&1 | tail -3; done
