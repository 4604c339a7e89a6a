# round-2 final evidence, part 2: ncu --set full captures of the dominant kernels (run after evidence_r02b.sh;
# kept under 64 MiB of output per gpurun call)
set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi2d_kernel -s 1 -c 1 -o gpurun_out/r02b_full_c3 \
  python tools/profile_run.py --config 3 --T 16 --reps 1 > /dev/null 2>&1; echo "full c3 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs2d_lane_kernel -c 1 -o gpurun_out/r02b_full_c4 \
  python tools/gsl_ncu.py > /dev/null 2>&1; echo "full c4 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs2d_lane_kernel -c 1 -o gpurun_out/r02b_full_c4_ref \
  python tools/gsl_ncu.py reference > /dev/null 2>&1; echo "full c4 ref rc=$?"
