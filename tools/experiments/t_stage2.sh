# 2D drop-in tail: hardware connections (CUDA_DEVICE_MAX_CONNECTIONS) x staging
for conn in 8 32; do for st in 0 1; do
  echo "== connections $conn stage $st"
  CUDA_DEVICE_MAX_CONNECTIONS=$conn TVS_E2E_STAGE=$st timeout 300 python tools/e2e_pipe_probe.py 2>&1 | grep -v "^pipe\|^bulk" | tail -4
done; done
