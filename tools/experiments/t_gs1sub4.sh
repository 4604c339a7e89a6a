# GS-1D sub-chunk 256 on the dedicated all-steady loop
for v in default sub256b; do
  if [ $v = default ]; then unset TVSTENCIL_LIB; else export TVSTENCIL_LIB=build/var/$v/libtvstencil.so; fi
  echo "== $v"
  timeout 300 python tools/parity_quick.py gs1d_w343 | tail -1
  timeout 120 python tools/profile_run.py --config 2 --reps 3 2>&1 | tail -1
done
