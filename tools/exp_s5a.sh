# session-5 experiment A: 3D one-barrier kernel parity + A/B; GS-2D lane trace / no-hand-off / ncu
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_shard.py -m gpu -x -q -k "3d or jac3d or shard" > gpurun_out/s5a_3d_tests.log 2>&1; echo "3d tests rc=$?"; tail -3 gpurun_out/s5a_3d_tests.log
timeout 300 python tools/c5_time.py > gpurun_out/s5a_c5_lag1.txt 2>&1; cat gpurun_out/s5a_c5_lag1.txt
TVSTENCIL_LIB=build/var/j3d_lag0/libtvstencil.so timeout 300 python tools/c5_time.py > gpurun_out/s5a_c5_lag0.txt 2>&1; cat gpurun_out/s5a_c5_lag0.txt
TVSTENCIL_LIB=build/var/gsl_trace/libtvstencil.so timeout 300 python tools/gsl_trace.py > gpurun_out/s5a_gsl_trace.txt 2>&1; cat gpurun_out/s5a_gsl_trace.txt
TVSTENCIL_LIB=build/var/gsl_noup/libtvstencil.so timeout 300 python tools/gsl_ncu.py > gpurun_out/s5a_gsl_noup.txt 2>&1; cat gpurun_out/s5a_gsl_noup.txt
timeout 300 python tools/gsl_ncu.py > gpurun_out/s5a_gsl_plain.txt 2>&1; cat gpurun_out/s5a_gsl_plain.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs2d_lane_kernel -c 1 -o gpurun_out/s5a_full_c4 python tools/gsl_ncu.py > /dev/null 2>&1; echo "ncu c4 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi3d_tb_kernel -s 3 -c 1 -o gpurun_out/s5a_full_c5fma python tools/profile_run.py --config 5 --T 8 --reps 1 --fma allow > /dev/null 2>&1; echo "ncu c5 rc=$?"
