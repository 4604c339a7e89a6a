# round-2 final evidence (session 5): bench line, reference arm, smoke, per-config launch lists,
# ncu --set full of the dominant kernels of configs 3, 4 (both orders) and 5 (bit-exact and fma allow)
set -x
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02b_reference_arm.json 2> gpurun_out/r02b_ref.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; echo "smoke rc=$?"
for c in 1 2 3 4 5; do
  python tools/profile_run.py --config $c --reps 1 > gpurun_out/r02b_profile_run_c$c.txt 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02b_launches_c$c.csv python tools/profile_run.py --config $c --reps 1 > /dev/null 2>&1
  echo "launches c$c rc=$?"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi2d_kernel -s 2 -c 1 -o gpurun_out/r02b_full_c3 \
  python tools/profile_run.py --config 3 --T 16 --reps 1 > /dev/null 2>&1; echo "full c3 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs2d_lane_kernel -c 1 -o gpurun_out/r02b_full_c4 \
  python tools/gsl_ncu.py > /dev/null 2>&1; echo "full c4 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs2d_lane_kernel -c 1 -o gpurun_out/r02b_full_c4_ref \
  python tools/gsl_ncu.py reference > /dev/null 2>&1; echo "full c4 ref rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi3d_tma_kernel -s 3 -c 1 -o gpurun_out/r02b_full_c5 \
  python tools/profile_run.py --config 5 --T 8 --reps 1 > /dev/null 2>&1; echo "full c5 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi3d_tma_kernel -s 3 -c 1 -o gpurun_out/r02b_full_c5_fma \
  python tools/profile_run.py --config 5 --T 8 --reps 1 --fma allow > /dev/null 2>&1; echo "full c5 fma rc=$?"
