# ncu --set full (with source) of the GS-2D pipeline kernel, config 4
python tools/profile_run.py --config 4 --reps 1 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gs2d_pipe -c 1 -o gpurun_out/full_c4 python tools/profile_run.py --config 4 --reps 1 > gpurun_out/ncu_c4.log 2>&1
ls -la gpurun_out/full_c4.ncu-rep
