#!/bin/bash
# A/B: priority of the internal tracker stream (step overlap) on C5 / C5MODE
cd "$(dirname "$0")/.."
for cfg in C5 C5MODE; do for rep in 1 2; do for kv in "TRB_TRK_PRIO=0" "TRB_TRK_PRIO=1" "TRB_TRK_PRIO=-1"; do
  env $kv timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --verify-streams 0 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg $kv', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']))"
done; done; done
