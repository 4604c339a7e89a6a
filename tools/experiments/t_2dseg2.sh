# 2D Jacobi after the interior-warp loop: row segment 256 (default) vs 512 / 128, ring depth 4 vs 2
for v in default seg512 seg128 ring2 default; do
  if [ $v = default ]; then unset TVSTENCIL_LIB; else export TVSTENCIL_LIB=build/var/$v/libtvstencil.so; fi
  echo "== $v"
  timeout 120 python tools/profile_run.py --config 3 --reps 3 2>&1 | tail -1
done
