set -x
python tools/profile_run.py --config 1 --reps 2 && python tools/profile_run.py --config 2 --reps 2 && python tools/profile_run.py --config 3 --T 16 && python tools/profile_run.py --config 4 --T 4 && python tools/profile_run.py --config 5 --T 2 > gpurun_out/prof_plain.log 2>&1
cat gpurun_out/prof_plain.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python tools/profile_run.py --config 1 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi1d -s 3 -c 1 -o gpurun_out/prof_c1 python tools/profile_run.py --config 1 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi2d -s 2 -c 1 -o gpurun_out/prof_c3 python tools/profile_run.py --config 3 --T 16 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi3d -c 1 -o gpurun_out/prof_c5 python tools/profile_run.py --config 5 --T 1 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gs1d -c 1 -o gpurun_out/prof_c2 python tools/profile_run.py --config 2 --T 128 --reps 1 > /dev/null 2>&1
ls -la gpurun_out
