set -x
echo "== default"; timeout 600 python tools/c3_depth.py 8 2>&1 | tail -1
echo "== ring0 (register prefetch)"; TVSTENCIL_LIB=build/var/j2d_ring0/libtvstencil.so timeout 600 python tools/c3_depth.py 8 2>&1 | tail -1
