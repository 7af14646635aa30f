#!/bin/bash
# A/B of libtrb variants (paper_1310_3322_b200/variants/libtrb_NAME.so) on a config
#   CFG=C5 tools/ab_variants.sh cur nt128b4 ...
cd "$(dirname "$0")/.."
CFG=${CFG:-C5}
for rep in 1 2; do for v in "$@"; do
  lib=paper_1310_3322_b200/libtrb.so; [ $v != cur ] && lib=paper_1310_3322_b200/variants/libtrb_$v.so
  TRB_VERBOSE=1 TRB_LIB=$lib timeout 300 python bench.py --config $CFG --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 2 \
    > gpurun_out/abv.json 2>gpurun_out/abv_$v.err
  python -c "import json;d=json.loads(open('gpurun_out/abv.json').read().strip().splitlines()[-1]);c=d['config']['stage_ms_per_step'];print('$CFG $v', round(d['value']), round(d['ms_per_step'],3), 'ms', round(c['track_meanshift'],3), d.get('verify',{}).get('identical_to_reference'))"
  grep -m1 "tracker:" gpurun_out/abv_$v.err
done; done
