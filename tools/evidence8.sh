# session-3 closing evidence: full GPU suite, bench line, smoke, GS-1D launch list
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_s3c.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_s3c.json 2> gpurun_out/bench_s3c.err; echo "bench rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s3c.log 2>&1; echo "smoke rc=$?"
python tools/profile_run.py --config 2 --reps 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_s3c_c2.csv python tools/profile_run.py --config 2 --reps 1 > /dev/null 2>&1
tail -2 gpurun_out/pytest_gpu_s3c.log
