# final round-1 evidence (session 2): full GPU suite, bench line, reference arm,
# launch lists per config, ncu --set full of the kernels changed since evidence2-4
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_final.json 2> gpurun_out/ref_final.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for c in 1 2 3 4 5; do
  T=""; [ $c = 3 ] && T="--T 16"; [ $c = 5 ] && T="--T 2"; [ $c = 4 ] && T="--T 100"
  python tools/profile_run.py --config $c $T --reps 1 > gpurun_out/plain_c$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c$c.csv python tools/profile_run.py --config $c $T --reps 1 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:jacobi3d_tb -c 1 -o gpurun_out/full_c5 python tools/profile_run.py --config 5 --T 2 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi2d -c 1 -o gpurun_out/full_c3 python tools/profile_run.py --config 3 --T 8 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:life2d_tb -c 1 -o gpurun_out/full_life python tools/int_prof.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:lcs_kernel -c 1 -o gpurun_out/full_lcs python tools/int_prof.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_integer.csv python tools/int_prof.py > /dev/null 2>&1
ls -la gpurun_out
