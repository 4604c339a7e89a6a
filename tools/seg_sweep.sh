#!/bin/bash
# config-3 device time vs 2D segment rows (TVS_J2D_SEG; 0 = auto wave fill)
for s in 0 256 0 228 0 256; do
  echo "seg=$s $(TVS_J2D_SEG=$s python bench.py --no-all --no-cpu --steps 5 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],1), d["clocks"]["sm_mhz"], round(d["e2e"]["value"],1))')"
done
