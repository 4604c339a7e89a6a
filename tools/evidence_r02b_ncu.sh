# round-2 final evidence, part 2: ncu --set full captures of the dominant kernels (run after evidence_r02b.sh;
# kept under 64 MiB of output per gpurun call)
set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi2d_kernel -s 1 -c 1 -o gpurun_out/r02b_full_c3 \
  python tools/profile_run.py --config 3 --T 16 --reps 1 > /dev/null 2>&1; echo "full c3 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs2d_lane_kernel -c 1 -o gpurun_out/r02b_full_c4 \
  python tools/gsl_ncu.py > /dev/null 2>&1; echo "full c4 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs2d_lane_kernel -c 1 -o gpurun_out/r02b_full_c4_ref \
  python tools/gsl_ncu.py reference > /dev/null 2>&1; echo "full c4 ref rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi3d_tma_kernel -s 3 -c 1 -o gpurun_out/r02b_full_c5 \
  python tools/profile_run.py --config 5 --T 8 --reps 1 > /dev/null 2>&1; echo "full c5 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi3d_tma_kernel -s 3 -c 1 -o gpurun_out/r02b_full_c5_fma \
  python tools/profile_run.py --config 5 --T 8 --reps 1 --fma allow > /dev/null 2>&1; echo "full c5 fma rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi1d_kernel -s 4 -c 1 -o gpurun_out/r02b_full_c1 \
  python tools/profile_run.py --config 1 --reps 1 > /dev/null 2>&1; echo "full c1 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs1d_kernel -c 1 -o gpurun_out/r02b_full_c2 \
  python tools/profile_run.py --config 2 --reps 1 > /dev/null 2>&1; echo "full c2 rc=$?"
