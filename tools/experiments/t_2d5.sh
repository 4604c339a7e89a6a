timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "jacobi2d or golden or slab or plan" -p no:cacheprovider 2>&1 | tail -2
timeout 120 python tools/parity_quick.py heat2d | tail -1
echo "== ring8"; for d in 4 6 8; do timeout 60 python tools/profile_run.py --config 3 --T 48 --depth $d --reps 3 | tail -1; done
for r in 4 16; do echo "== ring$r"; for d in 4 6 8; do TVSTENCIL_LIB=build/var/lib_r$r.so timeout 60 python tools/profile_run.py --config 3 --T 48 --depth $d --reps 3 | tail -1; done; done
echo "== regs"; for d in 4 6 8; do TVS_J2D_RING=0 timeout 60 python tools/profile_run.py --config 3 --T 48 --depth $d --reps 3 | tail -1; done
