# 3D K4b: output planes per block (plane-overlap overhead vs parallelism)
for v in base s32 s128 s256; do
  L=build/var/$v/libtvstencil.so; [ $v = base ] && L=paper_2010_04868_b200/libtvstencil.so
  for f in exact allow; do TVSTENCIL_LIB=$L timeout 120 python tools/power_probe.py jac3d27p 1024 1024 1024 --T 20 --fma $f | sed "s/^/$v /"; done
done
