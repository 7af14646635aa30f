#!/bin/bash
# A/B: incremental Mode kernel, 2 strided px/thread vs 4 consecutive (vector) px/thread
cd "$(dirname "$0")/.."
for rep in 1 2; do for pix in 2 0; do
  TRB_MODE_PIX=$pix timeout 300 python bench.py --config C5MODE --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 2 \
    > gpurun_out/abm.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/abm.json').read().strip().splitlines()[-1]);c=d['config']['stage_ms_per_step'];print('pix=$pix', round(d['value']), round(d['ms_per_step'],3), 'motion', round(c['motion'],3), d.get('verify',{}).get('identical_to_reference'))"
done; done
