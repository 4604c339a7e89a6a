# Life temporally blocked kernel: interior-warp loop without boundary selects (new) vs previous
for v in intold default intold default; do
  if [ $v = default ]; then unset TVSTENCIL_LIB; else export TVSTENCIL_LIB=build/var/$v/libtvstencil.so; fi
  echo "== $v"
  timeout 300 python tools/int_prof.py 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip()); print({k:round(v['value'],1) for k,v in d.items()})"
done
unset TVSTENCIL_LIB
timeout 900 python -m pytest tests/test_integer_kernels.py tests/test_tiling.py -q -x -p no:cacheprovider 2>&1 | tail -2
