timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gs1d or golden or known" -p no:cacheprovider 2>&1 | tail -2
for W in 2 4; do for T in 128 512 1000 1024 4096; do TVS_GS1D_WARPS=$W timeout 60 python tools/profile_run.py --config 2 --T $T --reps 2 | tail -1; done; done
