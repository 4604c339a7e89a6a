# round-1 evidence: bench line, launch lists per config, one full ncu capture per dominant kernel
set -x
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?"
for c in 1 2 3 4 5; do
  T=""; [ $c = 3 ] && T="--T 16"; [ $c = 5 ] && T="--T 2"; [ $c = 4 ] && T="--T 100"
  python tools/profile_run.py --config $c $T --reps 1 > gpurun_out/plain_c$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c$c.csv python tools/profile_run.py --config $c $T --reps 1 > /dev/null 2>&1
done
python tools/profile_run.py --config 3 --T 8 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:jacobi2d -c 1 -o gpurun_out/full_c3 python tools/profile_run.py --config 3 --T 8 --reps 1 > /dev/null 2>&1
python tools/profile_run.py --config 5 --T 1 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:jacobi3d -c 1 -o gpurun_out/full_c5 python tools/profile_run.py --config 5 --T 1 --reps 1 > /dev/null 2>&1
python tools/profile_run.py --config 1 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:jacobi1d -s 2 -c 1 -o gpurun_out/full_c1 python tools/profile_run.py --config 1 --reps 1 > /dev/null 2>&1
python tools/profile_run.py --config 2 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gs1d -c 1 -o gpurun_out/full_c2 python tools/profile_run.py --config 2 --reps 1 > /dev/null 2>&1
python tools/profile_run.py --config 4 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gs2d -c 1 -o gpurun_out/full_c4 python tools/profile_run.py --config 4 --reps 1 > /dev/null 2>&1
ls -la gpurun_out
