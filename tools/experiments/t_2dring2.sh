# 2D Jacobi: ring depth 2/4 and segment length with the ring, config 3
for v in r4 r4s512 r4s384 r2; do
  L=build/var/$v/libtvstencil.so
  for d in 7 8 9; do TVSTENCIL_LIB=$L timeout 60 python tools/shape_run.py heat2d 16384 16384 --T 200 --depth $d | sed "s/^/$v d$d /"; done
done
