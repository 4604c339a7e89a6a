# 2D Jacobi: interior-warp row loop without per-row checks (new default) vs previous kernel
for v in j2dold default j2dold default; do
  if [ $v = default ]; then unset TVSTENCIL_LIB; else export TVSTENCIL_LIB=build/var/$v/libtvstencil.so; fi
  echo "== $v"
  timeout 120 python tools/profile_run.py --config 3 --reps 3 2>&1 | tail -1
  timeout 120 python tools/profile_run.py --config 3 --T 16 --reps 3 2>&1 | tail -1
done
unset TVSTENCIL_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py tests/test_halo_cpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
