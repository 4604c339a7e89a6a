set -x
for v in b2d2 b2d3 d1; do echo "== $v"; TVSTENCIL_LIB=build/var/gsl_$v/libtvstencil.so timeout 600 python tools/gs2d_lane_check.py 2>&1 | tail -3; done
