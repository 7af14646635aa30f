#!/bin/bash
# A/B: queue-order knobs with the decaying iteration hint (C5)
cd "$(dirname "$0")/.."
for rep in 1 2 3; do for kv in "TRB_ITER_FLOOR=6" "TRB_ITER_FLOOR=3" "TRB_ITER_FLOOR=10" "TRB_ORDER_FIX=2500" "TRB_ORDER_FIX=10000" "TRB_SPLIT_US=150"; do
  env $kv timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 0 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$kv', round(d['value']), round(d['ms_per_step'],3))"
done; done
