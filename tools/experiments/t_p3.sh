TVSTENCIL_LIB=build/var/lib_p3.so timeout 120 python tools/parity_quick.py heat2d | tail -1
TVSTENCIL_LIB=build/var/lib_p3.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "jacobi2d" -p no:cacheprovider 2>&1 | tail -1
for d in 6 7 8; do echo -n "P3 "; TVSTENCIL_LIB=build/var/lib_p3.so timeout 60 python tools/profile_run.py --config 3 --depth $d --reps 3 | tail -1; done
echo -n "P4 "; timeout 60 python tools/profile_run.py --config 3 --depth 8 --reps 3 | tail -1
