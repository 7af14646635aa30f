#!/bin/bash
cd "$(dirname "$0")/.."
for cfg in C1 C2; do for sp in 200 600 2000 20000; do
  TRB_SPLIT_US=$sp timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
    --verify-streams 1 > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg split_us=$sp', round(d['value']), round(d['ms_per_step'],3), d['verify']['identical_to_reference'])"
done; done
