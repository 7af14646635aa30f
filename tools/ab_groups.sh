#!/bin/bash
cd "$(dirname "$0")/.."
for rep in 1 2; do for g in 1 2 4; do
  TRB_STREAM_GROUPS=$g timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 1 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('groups=$g', round(d['value']), round(d['ms_per_step'],3), d['verify']['identical_to_reference'])"
done; done
