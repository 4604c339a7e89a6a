# GS-1D with 128-position sub-chunks: chunk 256 (default) vs 512 vs 1024 (dynamic smem ring); measured 128: 61.5, 256: 65.1, 1024: 62.1
for v in ch512; do
  if [ $v = default ]; then unset TVSTENCIL_LIB; else export TVSTENCIL_LIB=build/var/$v/libtvstencil.so; fi
  echo "== $v"
  timeout 300 python tools/parity_quick.py gs1d_w343 | tail -1
  for i in 1 2; do timeout 120 python tools/profile_run.py --config 2 --reps 3 2>&1 | tail -1; done
done
unset TVSTENCIL_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -q -x -k "gs1d or gauss or 1d or cid" -p no:cacheprovider 2>&1 | tail -3
