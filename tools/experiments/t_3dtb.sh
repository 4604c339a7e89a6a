# K4b two-level 3D blocking: parity, then throughput vs depth 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "jacobi3d or slab or fma_policies or equivalence_matrix_gpu or golden" 2>&1 | tail -3
P="timeout 120 python tools/power_probe.py"
for d in 1 2; do
$P jac3d27p 1024 1024 1024 --T 10 --depth $d
$P jac3d27p 1024 1024 1024 --T 10 --depth $d --fma allow
$P heat3d 1024 1024 1024 --T 10 --depth $d
done
$P jac3d27p 1024 1024 1024 --T 100 --fma allow
