#!/bin/bash
# bench meanshift time for engine / split-threshold variants (each under a timeout)
cd "$(dirname "$0")/.."
for cfg in "2 200" "2 400" "2 800" "2 100" "1 200"; do
  set -- $cfg
  TRB_ENGINE=$1 TRB_SPLIT_US=$2 timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
    --verify-streams 0 > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print('engine $1 split $2', round(d['value']), round(d['config']['stage_ms_per_step']['track_meanshift'],3))"
done
