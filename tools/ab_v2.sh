#!/bin/bash
# A/B: v2 engine on the default library vs variants (TRB_LIB), C5 and C1
cd "$(dirname "$0")/.."
for lib in "$@"; do
  [ "$lib" = "default" ] && lib=""
  if [ -n "$lib" ]; then export TRB_LIB=$PWD/paper_1310_3322_b200/variants/libtrb_$lib.so; else unset TRB_LIB; fi
  for cfg in C5 C1; do for eng in 2 1; do
    TRB_ENGINE=$eng timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
      --verify-streams 1 > gpurun_out/ab.json 2> gpurun_out/ab.err
    echo "${lib:-default} $cfg engine $eng :: $(python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['config']['stage_ms_per_step']['track_meanshift'],3), d.get('verify',{}).get('identical_to_reference'))" 2>&1 | tail -1)"
  done; done
done
