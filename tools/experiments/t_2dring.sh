# 2D Jacobi: cp.async row ring (depth 4/8/16) and 4-row register prefetch vs default, config 3
for v in base r4 r8 r16 pf4; do
  L=build/var/$v/libtvstencil.so; [ $v = base ] && L=paper_2010_04868_b200/libtvstencil.so
  TVSTENCIL_LIB=$L timeout 120 python tools/parity_quick.py heat2d | tail -1
  for d in 6 8 10; do TVSTENCIL_LIB=$L timeout 60 python tools/shape_run.py heat2d 16384 16384 --T 200 --depth $d | sed "s/^/$v /"; done
done
