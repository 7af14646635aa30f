#!/bin/bash
cd "$(dirname "$0")/.."
for kv in "TRB_SPLIT_US=200" "TRB_SPLIT_US=120" "TRB_SPLIT_US=300" "TRB_ORDER_FIX=2500" "TRB_ORDER_FIX=10000" "TRB_ITER_FLOOR=3" "TRB_ITER_FLOOR=10" "TRB_SPLIT_US=200"; do
  env $kv timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 0 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$kv', round(d['value']), round(d['ms_per_step'],3))"
done
