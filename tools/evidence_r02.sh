# round-2 evidence: bench line, reference arm, smoke, per-config launch lists,
# ncu --set full of the config-3 and config-4 dominant kernels
set -x
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_reference_arm.json 2> gpurun_out/r02_ref.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"
for c in 1 2 3 4 5; do
  python tools/profile_run.py --config $c --reps 1 > gpurun_out/r02_profile_run_c$c.txt 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02_launches_c$c.csv python tools/profile_run.py --config $c --reps 1 > /dev/null 2>&1
  echo "launches c$c rc=$?"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi2d_kernel -s 2 -c 1 -o gpurun_out/r02_full_c3 \
  python tools/profile_run.py --config 3 --T 16 --reps 1 > /dev/null 2>&1; echo "full c3 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs2d_lane_kernel -c 1 -o gpurun_out/r02_full_c4 \
  python tools/profile_run.py --config 4 --reps 1 > /dev/null 2>&1; echo "full c4 rc=$?"
