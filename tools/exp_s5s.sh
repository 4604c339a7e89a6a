set -x
echo "== base"; TVSTENCIL_LIB=build/var/gs1d_base/libtvstencil.so timeout 300 python tools/profile_run.py --config 2 --reps 3 2>&1 | tail -2
echo "== uniform"; timeout 300 python tools/profile_run.py --config 2 --reps 3 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gs1d or gs_1d or golden or acceptance" 2>&1 | tail -2
