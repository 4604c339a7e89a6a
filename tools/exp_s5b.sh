# session-5 experiment B: packed GS-2D lane groups (G=4 / G=5); TMA 3D kernel parity + timing
set -x
timeout 600 python tools/gs2d_lane_check.py > gpurun_out/s5b_gsl_g4.txt 2>&1; cat gpurun_out/s5b_gsl_g4.txt
TVSTENCIL_LIB=build/var/gsl_g5/libtvstencil.so timeout 600 python tools/gs2d_lane_check.py > gpurun_out/s5b_gsl_g5.txt 2>&1; cat gpurun_out/s5b_gsl_g5.txt
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_shard.py -m gpu -x -q -k "3d or jac3d or shard" > gpurun_out/s5b_3d_tests.log 2>&1; echo "3d tests rc=$?"; tail -5 gpurun_out/s5b_3d_tests.log
timeout 300 python tools/c5_time.py > gpurun_out/s5b_c5_tma.txt 2>&1; cat gpurun_out/s5b_c5_tma.txt
TVS_J3D=cpasync timeout 300 python tools/c5_time.py > gpurun_out/s5b_c5_cpasync.txt 2>&1; cat gpurun_out/s5b_c5_cpasync.txt
