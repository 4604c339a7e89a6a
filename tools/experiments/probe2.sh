# single-step (untiled) kernels after the bandwidth rewrite
P="timeout 120 python tools/power_probe.py"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "naive or slab or jacobi2d_depths or jacobi3d_streaming or equivalence_matrix_gpu" 2>&1 | tail -3
$P heat2d 16384 16384 --T 20 --algo naive
$P jac2d9p 16384 16384 --T 20 --algo naive
$P heat1d 268435456 --T 10 --algo naive
$P heat3d 1024 1024 1024 --T 10 --algo naive
$P heat3d 1024 1024 1024 --T 10
$P jac3d27p 1024 1024 1024 --T 10 --algo naive
