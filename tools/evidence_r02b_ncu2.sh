# round-2 final evidence, part 3: ncu --set full of configs 5 (both FMA modes), 1 and 2
set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi3d_tma_kernel -s 3 -c 1 -o gpurun_out/r02b_full_c5 \
  python tools/profile_run.py --config 5 --T 8 --reps 1 > /dev/null 2>&1; echo "full c5 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi3d_tma_kernel -s 3 -c 1 -o gpurun_out/r02b_full_c5_fma \
  python tools/profile_run.py --config 5 --T 8 --reps 1 --fma allow > /dev/null 2>&1; echo "full c5 fma rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:jacobi1d_kernel -s 4 -c 1 -o gpurun_out/r02b_full_c1 \
  python tools/profile_run.py --config 1 --reps 1 > /dev/null 2>&1; echo "full c1 rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:gs1d_kernel -c 1 -o gpurun_out/r02b_full_c2 \
  python tools/profile_run.py --config 2 --reps 1 > /dev/null 2>&1; echo "full c2 rc=$?"
