set -x
echo "== seg 128 (default)"; timeout 300 python tools/c5_time.py 2>&1 | tail -2
for sg in 64 256; do echo "== seg $sg"; TVSTENCIL_LIB=build/var/j3d_seg$sg/libtvstencil.so timeout 300 python tools/c5_time.py 2>&1 | tail -2; done
