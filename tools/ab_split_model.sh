#!/bin/bash
# A/B: split-mode cost model (single-CTA us per kpx) and threshold on C5
cd "$(dirname "$0")/.."
for rep in 1 2; do
for kv in "TRB_SPLIT_US=200" "TRB_SPLIT_PERKPX=6.5 TRB_SPLIT_US=200" "TRB_SPLIT_PERKPX=6.5 TRB_SPLIT_US=400" \
          "TRB_SPLIT_PERKPX=6.5 TRB_SPLIT_FIX=75 TRB_SPLIT_US=300" "TRB_SPLIT_US=100"; do
  env $kv timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 0 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$kv', round(d['value']), round(d['ms_per_step'],3))"
done; done
