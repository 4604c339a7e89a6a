set -x
echo "== old"; TVSTENCIL_LIB=build/var/old/libtvstencil.so timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
timeout 900 python tools/gs2d_lane_check.py > gpurun_out/s5d_gsl_v3.txt 2>&1; cat gpurun_out/s5d_gsl_v3.txt
echo "== v3 noup"; TVSTENCIL_LIB=build/var/gsl_v3_noup/libtvstencil.so timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
echo "== v3 g4"; TVSTENCIL_LIB=build/var/gsl_v3_g4/libtvstencil.so timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
TVSTENCIL_LIB=build/var/gsl_v3_trace/libtvstencil.so timeout 300 python tools/gsl_trace.py > gpurun_out/s5d_gsl_trace.txt 2>&1; cat gpurun_out/s5d_gsl_trace.txt
