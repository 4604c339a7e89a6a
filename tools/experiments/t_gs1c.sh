for T in 128 256 512 1000 2048 4096; do timeout 60 python tools/profile_run.py --config 2 --T $T --reps 2 | tail -1; done
