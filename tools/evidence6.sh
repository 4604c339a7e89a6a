# session-3 evidence: bench line after the GS-1D sub-chunk and drop-in copy
# changes, smoke, GS-1D / config-3 launch lists, ncu --set full of gs1d_kernel
set -x
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err; echo "bench rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s3.log 2>&1; echo "smoke rc=$?"
for c in 2 3; do
  T=""; [ $c = 3 ] && T="--T 16"
  python tools/profile_run.py --config $c $T --reps 1 > gpurun_out/plain_s3_c$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_s3_c$c.csv python tools/profile_run.py --config $c $T --reps 1 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:gs1d_kernel -c 1 -o gpurun_out/full_s3_gs1d python tools/profile_run.py --config 2 --reps 1 > /dev/null 2>&1
ls -la gpurun_out | tail -20
