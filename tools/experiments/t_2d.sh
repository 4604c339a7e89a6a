timeout 60 python tools/profile_run.py --config 4 --reps 3
for d in 3 4 5 6 8 10 12; do timeout 60 python tools/profile_run.py --config 3 --T 48 --depth $d --reps 2 | tail -1; done
