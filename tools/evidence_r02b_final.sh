# round-2 final evidence, last refresh (after the last K2 / K6v3 changes): GPU suite, bench line, reference arm, smoke,
# launch lists and ncu captures of configs 1 and 4 (the other configs' lists / captures of evidence_r02b*.sh are unchanged)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02b_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02b_gpu_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02b_reference_arm.json 2> gpurun_out/r02b_ref.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; echo "smoke rc=$?"
for c in 1 4; do
  python tools/profile_run.py --config $c --reps 1 > gpurun_out/r02b_profile_run_c$c.txt 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02b_launches_c$c.csv python tools/profile_run.py --config $c --reps 1 > /dev/null 2>&1; echo "launches c$c rc=$?"
done
timeout 600 ncu --set full --clock-control none -k regex:jacobi1d_kernel -s 4 -c 1 -o gpurun_out/r02b_full_c1 \
  python tools/profile_run.py --config 1 --reps 1 > /dev/null 2>&1; echo "full c1 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs2d_lane_kernel -c 1 -o gpurun_out/r02b_full_c4 \
  python tools/gsl_ncu.py > /dev/null 2>&1; echo "full c4 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs2d_lane_kernel -c 1 -o gpurun_out/r02b_full_c4_ref \
  python tools/gsl_ncu.py reference > /dev/null 2>&1; echo "full c4 ref rc=$?"
