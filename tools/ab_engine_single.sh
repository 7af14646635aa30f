#!/bin/bash
# A/B: mean-shift engine on the single-stream full-HD / 4K configs
cd "$(dirname "$0")/.."
for cfg in C3 C4; do for rep in 1 2; do for kv in "TRB_ENGINE=1" "TRB_ENGINE=2" "TRB_ENGINE=2 TRB_CLUSTER=16" "TRB_ENGINE=2 TRB_CLUSTER=12"; do
  env $kv timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 1 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg $kv', round(d['value']), round(d['ms_per_step'],3), round(d['config']['stage_ms_per_step']['track_meanshift'],3), d.get('verify',{}).get('identical_to_reference'))"
done; done; done
