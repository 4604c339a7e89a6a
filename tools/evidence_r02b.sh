# round-2 final evidence (session 5): bench line, reference arm, smoke, per-config launch lists,
# ncu --set full of the dominant kernels of configs 3, 4 (both orders) and 5 (bit-exact and fma allow)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02b_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02b_gpu_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02b_reference_arm.json 2> gpurun_out/r02b_ref.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; echo "smoke rc=$?"
for c in 1 2 3 4 5; do
  python tools/profile_run.py --config $c --reps 1 > gpurun_out/r02b_profile_run_c$c.txt 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02b_launches_c$c.csv python tools/profile_run.py --config $c --reps 1 > /dev/null 2>&1
  echo "launches c$c rc=$?"
done
