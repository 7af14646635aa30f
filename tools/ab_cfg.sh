#!/bin/bash
# A/B over configs: tools/ab_cfg.sh "C2 C3 C4" lib1 lib2 ... (engine auto)
cd "$(dirname "$0")/.."
cfgs=$1; shift
for lib in "$@"; do
  [ "$lib" = "default" ] && lib=""
  if [ -n "$lib" ]; then export TRB_LIB=$PWD/paper_1310_3322_b200/variants/libtrb_$lib.so; else unset TRB_LIB; fi
  for cfg in $cfgs; do
    timeout 300 python bench.py --config $cfg --steps ${STEPS:-20} --warmup ${WARM:-5} --no-cpu-baseline --no-e2e \
      --verify-streams 1 > gpurun_out/ab.json 2> gpurun_out/ab.err
    echo "${lib:-default} $cfg :: $(python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],3), round(d['config']['stage_ms_per_step']['track_meanshift'],3), d.get('verify',{}).get('identical_to_reference'))" 2>&1 | tail -1)"
  done
done
