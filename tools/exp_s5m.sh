set -x
echo "== default"; timeout 600 python tools/c3_depth.py 6 7 8 2>&1 | tail -3
echo "== p4"; TVSTENCIL_LIB=build/var/j2d_p4/libtvstencil.so timeout 600 python tools/c3_depth.py 5 6 7 2>&1 | tail -3
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi2d_kernel -s 1 -c 1 -o gpurun_out/r02b_full_c3 python tools/profile_run.py --config 3 --T 16 --reps 1 > /dev/null 2>&1; echo "full c3 rc=$?"
