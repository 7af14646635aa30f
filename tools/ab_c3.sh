#!/bin/bash
# A/B of the step machinery on the single-stream 1080p config (C3)
cd "$(dirname "$0")/.."
for rep in 1 2; do for kv in "TRB_OVERLAP=1" "TRB_OVERLAP=0" "TRB_CLUSTER=16" "TRB_CLUSTER=8" "TRB_TRK_PRIO=0"; do
  env $kv timeout 300 python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 0 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);c=d['config']['stage_ms_per_step'];print('$kv', round(d['value']), round(d['ms_per_step'],3), {k:round(v,3) for k,v in c.items()})"
done; done
