for b in 1024 1500 0; do TVS_E2E_BAND1=$b timeout 300 python tests/e2e_band1_check.py 2>&1 | grep -c "^ok" | sed "s/^/band $b ok count: /"; done
# pinned (registered) buffers: graph path, repeated calls, then changed contents with the same buffers
timeout 300 python - <<'PY'
import numpy as np, sys
sys.path.insert(0, ".")
from oracle import cref
from paper_2010_04868_b200 import Grid, _native
from paper_2010_04868_b200.catalog import get
from paper_2010_04868_b200.kernels import heat1d_temporal
spec = get("heat1d").spec
g = Grid.random((1 << 20,), seed=0); out = g.copy()
_native.host_register(g.data); _native.host_register(out.data)
ok = True
for rep in range(4):
    g.set_interior(np.random.default_rng(rep).uniform(-1, 1, 1 << 20))
    heat1d_temporal(g, 1000, out=out) if False else None
    from paper_2010_04868_b200.kernels._common import execute
    execute(spec, g, 1000, out=out)
    want = cref.scalar_reference(spec, g, 1000, threads=8)
    ok &= np.array_equal(out.interior, want.interior)
print("graph replay parity", ok)
PY
for b in 65536 131072 262144; do TVS_E2E_BAND1=$b timeout 300 python -c "
import bench, statistics
t, nb, _ = bench.e2e_time(bench.CONFIGS[1], 20, 3)
print(\"band $b config 1 e2e ms\", round(statistics.mean(t),3), \"GSt/s\", round(2**20*1000/statistics.mean(t)/1e6,1))
" 2>&1 | tail -1; done
