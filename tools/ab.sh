#!/bin/bash
# A/B: bench the default library and each variant (TRB_LIB) in turn.
for lib in "$@"; do
  [ "$lib" = "default" ] && lib=""
  if [ -n "$lib" ]; then export TRB_LIB=$PWD/paper_1310_3322_b200/variants/libtrb_$lib.so; else unset TRB_LIB; fi
  TRB_VERBOSE=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "${lib:-default} $(grep -o 'tracker: .*' gpurun_out/ab.err | head -1) :: $(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(round(d['value']), round(d['config']['stage_ms_per_step']['track_meanshift'],3))" 2>&1 | tail -1)"
done
