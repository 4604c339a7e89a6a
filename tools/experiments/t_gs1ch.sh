# GS-1D: chunk length (sync granularity) 256 / 512 / 1024
for v in base ch512 ch1024; do
  L=build/var/$v/libtvstencil.so; [ $v = base ] && L=paper_2010_04868_b200/libtvstencil.so
  TVSTENCIL_LIB=$L timeout 300 python tools/parity_quick.py gs1d_w343 | tail -1
  TVSTENCIL_LIB=$L timeout 120 python tools/profile_run.py --config 2 --reps 3 | tail -1 | sed "s/^/$v /"
done
