#!/bin/bash
# A/B of libtrb variants on the e2e (host-frame) leg: cur vs base
cd "$(dirname "$0")/.."
for cfg in C2 C1 C5; do for rep in 1 2; do for v in cur base; do
  lib=paper_1310_3322_b200/libtrb.so; [ $v != cur ] && lib=paper_1310_3322_b200/variants/libtrb_$v.so
  TRB_LIB=$lib timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --verify-streams 1 \
    > gpurun_out/abe.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/abe.json').read().strip().splitlines()[-1]);print('$cfg $v', round(d['value']), 'e2e', round(d['e2e']['value']), d.get('verify',{}).get('identical_to_reference'))"
done; done; done
