#!/bin/bash
# C1..C4 single-stream configs under both exact-sum engines
cd "$(dirname "$0")/.."
for cfg in C1 C2 C3 C4; do
  for eng in 1 2; do
    TRB_ENGINE=$eng timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
      --verify-streams 1 > gpurun_out/ec.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/ec.json').read().strip().splitlines()[-1]); print('$cfg engine $eng', round(d['value']), round(d['config']['stage_ms_per_step']['track_meanshift'],4), d.get('verify',{}).get('identical_to_reference'))"
  done
done
