# ncu --set full of K4b (fma allow and exact), one launch each
python tools/profile_run.py --config 5 --T 2 --reps 1 --fma allow > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:jacobi3d_tb -c 1 -o gpurun_out/tb3d_fma python tools/profile_run.py --config 5 --T 2 --reps 1 --fma allow > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi3d_tb -c 1 -o gpurun_out/tb3d_exact python tools/profile_run.py --config 5 --T 2 --reps 1 > /dev/null 2>&1
ls gpurun_out
