# 2D Jacobi: two-row skew between levels (independent level updates) vs one-row skew
TVSTENCIL_LIB=build/var/skew2/libtvstencil.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "jacobi2d_depths or e2e_bands or slab or ranged" 2>&1 | tail -2
for v in base skew2; do
  L=build/var/$v/libtvstencil.so; [ $v = base ] && L=paper_2010_04868_b200/libtvstencil.so
  for d in 4 5 6 8; do TVSTENCIL_LIB=$L timeout 60 python tools/shape_run.py heat2d 16384 16384 --T 200 --depth $d --reps 3 | sed "s/^/$v d$d /"; done
done
