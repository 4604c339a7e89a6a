# GS-1D: separate all-steady sub-chunk loop (new) vs per-sub-chunk variant branch (previous)
for v in gs1old default gs1old default; do
  if [ $v = default ]; then unset TVSTENCIL_LIB; else export TVSTENCIL_LIB=build/var/$v/libtvstencil.so; fi
  echo "== $v"
  timeout 120 python tools/profile_run.py --config 2 --reps 3 2>&1 | tail -1
done
unset TVSTENCIL_LIB
timeout 300 python tools/parity_quick.py gs1d_w343 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -q -x -k "gs1d or gauss or 1d or cid" -p no:cacheprovider 2>&1 | tail -2
