set -x
timeout 600 python tools/gs2d_lane_check.py 2>&1 | tail -3
TVSTENCIL_LIB=build/var/gsl_v3_trace/libtvstencil.so timeout 300 python tools/gsl_trace.py > gpurun_out/s5l_gsl_trace.txt 2>&1; cat gpurun_out/s5l_gsl_trace.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gs2d or gs" 2>&1 | tail -2
