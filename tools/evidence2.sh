# round-1 evidence refresh (session 2): GPU tests, bench line, reference arm,
# long-run 3D depth check, ncu launch lists per config + untiled kernel, one
# ncu --set full capture per dominant kernel
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
for d in 1 2; do timeout 200 python tools/power_probe.py jac3d27p 1024 1024 1024 --T 100 --depth $d; done > gpurun_out/probe3d.log 2>&1
for c in 1 2 3 4 5; do
  T=""; [ $c = 3 ] && T="--T 16"; [ $c = 5 ] && T="--T 2"; [ $c = 4 ] && T="--T 100"
  python tools/profile_run.py --config $c $T --reps 1 > gpurun_out/plain_c$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c$c.csv python tools/profile_run.py --config $c $T --reps 1 > /dev/null 2>&1
done
python tools/profile_run.py --config 3 --T 4 --algo naive --reps 1 > gpurun_out/plain_u3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/launches_untiled_c3.csv python tools/profile_run.py --config 3 --T 4 --algo naive --reps 1 > /dev/null 2>&1
python tools/profile_run.py --config 3 --T 8 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:jacobi2d -c 1 -o gpurun_out/full_c3 python tools/profile_run.py --config 3 --T 8 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi3d_tb -c 1 -o gpurun_out/full_c5 python tools/profile_run.py --config 5 --T 2 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi_naive -c 1 -o gpurun_out/full_untiled_c3 python tools/profile_run.py --config 3 --T 1 --algo naive --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi1d -s 2 -c 1 -o gpurun_out/full_c1 python tools/profile_run.py --config 1 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gs1d -c 1 -o gpurun_out/full_c2 python tools/profile_run.py --config 2 --reps 1 > /dev/null 2>&1
ls -la gpurun_out
