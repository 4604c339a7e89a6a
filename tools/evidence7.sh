# session-3 final evidence: full GPU suite, bench line, reference arm, smoke,
# launch lists (config 3, integer), ncu --set full of the 2D Jacobi and Life
# kernels after the interior-warp loops
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_s3.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_s3b.json 2> gpurun_out/bench_s3b.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_s3.json 2> gpurun_out/ref_s3.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s3b.log 2>&1; echo "smoke rc=$?"
python tools/profile_run.py --config 3 --T 16 --reps 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_s3b_c3.csv python tools/profile_run.py --config 3 --T 16 --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_s3b_integer.csv python tools/int_prof.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi2d -c 1 -o gpurun_out/full_s3_c3 python tools/profile_run.py --config 3 --T 8 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:life2d_tb -c 1 -o gpurun_out/full_s3_life python tools/int_prof.py > /dev/null 2>&1
ls -la gpurun_out | tail -12
