# GS-1D unrolled sub-chunk length 32 (default) vs 64 vs 128: parity + config 2 time
for v in default sub64 sub128 sub256; do
  if [ $v = default ]; then unset TVSTENCIL_LIB; else export TVSTENCIL_LIB=build/var/$v/libtvstencil.so; fi
  echo "== $v"
  timeout 300 python tools/parity_quick.py gs1d_w343 | tail -1
  for i in 1 2; do timeout 120 python tools/profile_run.py --config 2 --reps 3 | tail -1; done
done
