for c in 1 4; do for s in "2048 2048" "2048 8192" "2048 32768" "512 32768"; do echo -n "CS=$c "; TVS_GS2D_CLUSTER=$c timeout 120 python tools/shape_run.py gs2d9p $s --T 100 | tail -1; done; done
python - <<'PY'
import ctypes
from cuda.bindings import runtime as rt
err, prop = rt.cudaGetDeviceProperties(0)
print("SMs", prop.multiProcessorCount, "smem/block optin", prop.sharedMemPerBlockOptin)
PY
