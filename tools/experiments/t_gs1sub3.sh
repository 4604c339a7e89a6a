# GS-1D sub-chunk 128 (default) vs 256 (writer stores split into 128-runs)
for v in default sub256; do
  if [ $v = default ]; then unset TVSTENCIL_LIB; else export TVSTENCIL_LIB=build/var/$v/libtvstencil.so; fi
  echo "== $v"
  timeout 300 python tools/parity_quick.py gs1d_w343 | tail -1
  for i in 1 2; do timeout 120 python tools/profile_run.py --config 2 --reps 3 2>&1 | tail -1; done
done
unset TVSTENCIL_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py tests/test_integer_kernels.py -q -x -k "gs1d or gauss or 1d or cid" -p no:cacheprovider 2>&1 | tail -2
