set -x
timeout 900 python tools/gs2d_lane_check.py > gpurun_out/s5j_gsl_v3.txt 2>&1; cat gpurun_out/s5j_gsl_v3.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5j_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/s5j_gpu_tests.log
