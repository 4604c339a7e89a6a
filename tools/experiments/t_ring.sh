timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "jacobi2d or golden or slab or plan" -p no:cacheprovider 2>&1 | tail -2
timeout 120 python tools/parity_quick.py heat2d | tail -1
echo "== ring"; for d in 2 4; do timeout 60 python tools/profile_run.py --config 3 --T 48 --depth $d --reps 3 | tail -1; done
echo "== regs"; TVS_J2D_RING=0 timeout 60 python tools/profile_run.py --config 3 --T 48 --depth 4 --reps 3 | tail -1
echo "== mb4"; TVSTENCIL_LIB=build/var/lib_mb4.so timeout 120 python tools/parity_quick.py heat2d | tail -1; TVSTENCIL_LIB=build/var/lib_mb4.so timeout 60 python tools/profile_run.py --config 3 --T 48 --depth 4 --reps 3 | tail -1
