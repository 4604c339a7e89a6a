set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs2d_lane_kernel -c 1 -o gpurun_out/s5e_full_c4_v3 python tools/gsl_ncu.py > /dev/null 2>&1; echo "ncu rc=$?"
TVSTENCIL_LIB=build/var/gsl_v3_noup/libtvstencil.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs2d_lane_kernel -c 1 -o gpurun_out/s5e_full_c4_v3_noup python tools/gsl_ncu.py > /dev/null 2>&1; echo "ncu rc=$?"
