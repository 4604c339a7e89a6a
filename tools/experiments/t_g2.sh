timeout 120 python tools/parity_quick.py gs2d9p | tail -1; timeout 60 python tools/profile_run.py --config 4 --reps 2 | tail -1
timeout 120 ./build/var/gs2d_trace 2>&1 | tail -16
