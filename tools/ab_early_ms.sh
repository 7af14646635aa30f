#!/bin/bash
# A/B: mean-shift of step t waits for the step's motion only (gate waits for its CCL) vs for the CCL
cd "$(dirname "$0")/.."
for cfg in C5 C5MODE C3 C4; do for rep in 1 2; do for kv in "TRB_EARLY_MS=0" "TRB_EARLY_MS=1"; do
  env $kv timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --verify-streams 2 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg $kv', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), d.get('verify',{}).get('identical_to_reference'))"
done; done; done
