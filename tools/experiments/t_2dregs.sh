# 2D Jacobi: register cap 128 (16 warps/SM, some spills) vs 160 (12 warps/SM)
for v in base m14; do
  L=build/var/$v/libtvstencil.so; [ $v = base ] && L=paper_2010_04868_b200/libtvstencil.so
  TVSTENCIL_LIB=$L timeout 120 python tools/parity_quick.py heat2d | tail -1
  for d in 6 8; do TVSTENCIL_LIB=$L timeout 60 python tools/shape_run.py heat2d 16384 16384 --T 200 --depth $d --reps 3 | sed "s/^/$v d$d /"; done
done
