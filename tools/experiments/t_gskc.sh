# GS-2D: chunk size (sync granularity) and the lags it allows
for v in base c2a c2b c8; do
  L=build/var/$v/libtvstencil.so; [ $v = base ] && L=paper_2010_04868_b200/libtvstencil.so
  TVSTENCIL_LIB=$L timeout 300 python tools/parity_quick.py gs2d9p | tail -1
  TVSTENCIL_LIB=$L timeout 120 python tools/shape_run.py gs2d9p 8192 8192 --T 100 --reps 3 | sed "s/^/$v /"
  TVSTENCIL_LIB=$L timeout 120 python tools/shape_run.py gs2d9p 8192 4096 --T 100 --reps 3 | sed "s/^/$v /"
done
