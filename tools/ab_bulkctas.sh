#!/bin/bash
# A/B: bulk motion kernel CTAs per SM under the step overlap (C5)
cd "$(dirname "$0")/.."
for rep in 1 2; do for kv in "TRB_MOTION_BULK_CTAS=3" "TRB_MOTION_BULK_CTAS=2" "TRB_MOTION_BULK_CTAS=1" "TRB_MOTION_BULK_CTAS=4"; do
  env $kv timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 0 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$kv', round(d['value']), round(d['ms_per_step'],3), round(d['config']['stage_ms_per_step']['motion'],3))"
done; done
