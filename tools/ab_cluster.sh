#!/bin/bash
# cluster size x engine at the driver's bench settings (C5, steps 20, warmup 5)
cd "$(dirname "$0")/.."
for g in ${GS:-8 4 2}; do for eng in ${ENGS:-1 2}; do
  TRB_CLUSTER=$g TRB_ENGINE=$eng timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
    --verify-streams 1 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "G=$g engine $eng :: $(python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],3), round(d['config']['stage_ms_per_step']['track_meanshift'],3), d.get('verify',{}).get('identical_to_reference'))" 2>&1 | tail -1)"
done; done
