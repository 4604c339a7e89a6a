set -x
echo "== old"; TVSTENCIL_LIB=build/var/old/libtvstencil.so timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
timeout 900 python tools/gs2d_lane_check.py > gpurun_out/s5i_gsl_v3.txt 2>&1; cat gpurun_out/s5i_gsl_v3.txt
echo "== v3 noup"; TVSTENCIL_LIB=build/var/gsl_v3_noup/libtvstencil.so timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
echo "== v3 nl4"; TVSTENCIL_LIB=build/var/gsl_v3_nl4/libtvstencil.so timeout 300 python tools/gs2d_lane_check.py 2>&1 | tail -3
