# session 4 batch A: K4b lean loop (parity + timing), GS-2D lane trace + no-hand-off floor
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_shard.py -m gpu -x -q -k "3d or jac3 or shard or golden or matrix" > gpurun_out/s4a_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s4a_tests.log
timeout 300 python tools/c5_time.py > gpurun_out/s4a_c5.txt 2>&1; cat gpurun_out/s4a_c5.txt
TVSTENCIL_LIB=build/var/gsl_trace/libtvstencil.so timeout 300 python tools/gsl_trace.py > gpurun_out/s4a_trace.txt 2>&1; cat gpurun_out/s4a_trace.txt
TVSTENCIL_LIB=build/var/gsl_noup/libtvstencil.so timeout 300 python - > gpurun_out/s4a_noup.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
import bench, numpy as np
for order in ("lexicographic", "reference"):
    t, l = bench.device_time(bench.CONFIGS[4], 3, 3, order=order)
    print("no-hand-off", order, [round(x, 2) for x in t])
PY
cat gpurun_out/s4a_noup.txt
