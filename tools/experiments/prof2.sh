set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "jacobi3d or golden or fma or plan or slab" -p no:cacheprovider 2>&1 | tail -3
python tools/profile_run.py --config 5 --T 2 --reps 2 && python tools/profile_run.py --config 2 --T 128 --reps 2 > gpurun_out/p2plain.log 2>&1
cat gpurun_out/p2plain.log
ncu --set full --clock-control none --import-source on -k regex:jacobi3d -c 1 -o gpurun_out/prof_c5b python tools/profile_run.py --config 5 --T 1 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gs1d -c 1 -o gpurun_out/prof_c2b python tools/profile_run.py --config 2 --T 128 --reps 1 > /dev/null 2>&1
ls gpurun_out
