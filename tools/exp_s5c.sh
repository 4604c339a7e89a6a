set -x
for v in nopack nopack_noup pack4_noup pack5_noup pack5; do
  echo "== $v"; TVSTENCIL_LIB=build/var/gsl_$v/libtvstencil.so timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
done
echo "== default (pack4)"; timeout 300 python tools/gsl_ncu.py 2>&1 | tail -1
TVSTENCIL_LIB=build/var/gsl_pack4_trace/libtvstencil.so timeout 300 python tools/gsl_trace.py > gpurun_out/s5c_gsl_trace_pack4.txt 2>&1; cat gpurun_out/s5c_gsl_trace_pack4.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs2d_lane_kernel -c 1 -o gpurun_out/s5c_full_c4_pack4 python tools/gsl_ncu.py > /dev/null 2>&1; echo "ncu rc=$?"
