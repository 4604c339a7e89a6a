# 2D Jacobi depth sweep after the interior-warp row loop
for d in 6 7 8 9 10 12; do
  echo "== depth $d"
  timeout 120 python tools/profile_run.py --config 3 --depth $d --reps 3 2>&1 | tail -1
done
