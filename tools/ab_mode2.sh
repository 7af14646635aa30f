#!/bin/bash
# A/B of incremental-Mode kernel variants (C5MODE motion stage)
cd "$(dirname "$0")/.."
for rep in 1 2; do for v in cur idiv off64 both; do
  lib=paper_1310_3322_b200/libtrb.so; [ $v != cur ] && lib=paper_1310_3322_b200/variants/libtrb_$v.so
  for pix in 1 2; do
  TRB_LIB=$lib TRB_MODE_PIX=$pix timeout 300 python bench.py --config C5MODE --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 0 \
    > gpurun_out/abm.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/abm.json').read().strip().splitlines()[-1]);c=d['config']['stage_ms_per_step'];print('$v pix=$pix', round(d['value']), round(d['ms_per_step'],3), 'motion', round(c['motion'],3))"
done; done; done
