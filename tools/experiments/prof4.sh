python tools/profile_run.py --config 4 --T 100 --reps 1 > gpurun_out/p4plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gs2d_pipe -c 1 -o gpurun_out/prof_c4 python tools/profile_run.py --config 4 --T 100 --reps 1 > gpurun_out/ncu4.log 2>&1
tail -3 gpurun_out/ncu4.log; cat gpurun_out/p4plain.log
