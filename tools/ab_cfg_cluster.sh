#!/bin/bash
# cluster size per config (engine auto), driver bench settings
cd "$(dirname "$0")/.."
for cfg in ${CFGS:-C3 C4}; do for g in ${GS:-8 12 16}; do
  TRB_CLUSTER=$g timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
    --verify-streams 1 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "$cfg G=$g :: $(python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],3), round(d['config']['stage_ms_per_step']['track_meanshift'],3), d.get('verify',{}).get('identical_to_reference'))" 2>&1 | tail -1)"
done; done
