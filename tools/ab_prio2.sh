#!/bin/bash
# A/B: tracker stream priority on the single-stream configs
cd "$(dirname "$0")/.."
for cfg in C1 C2 C3 C4; do for rep in 1 2; do for kv in "TRB_TRK_PRIO=0" "TRB_TRK_PRIO=1"; do
  env $kv timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --verify-streams 1 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg $kv', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), d.get('verify',{}).get('identical_to_reference'))"
done; done; done
