TVSTENCIL_LIB=build/var/lib_g5.so timeout 120 python tools/gs2d_case.py 97 64 100
TVSTENCIL_LIB=build/var/lib_g5.so timeout 120 python tools/gs2d_case.py 300 500 128
TVSTENCIL_LIB=build/var/lib_g5.so timeout 120 python tools/gs2d_case.py 61 300 129
for s in "8192 8192" "8192 2048"; do TVSTENCIL_LIB=build/var/lib_g5.so timeout 120 python tools/shape_run.py gs2d9p $s --T 100 2>&1 | tail -1; done
