#!/bin/bash
# v2 correctness (tracker + streams tests under TRB_ENGINE=2) and speed (C5, C1, C3) vs v1
cd "$(dirname "$0")/.."
TRB_ENGINE=2 timeout 300 python -m pytest tests/test_gpu_tracker.py tests/test_gpu_streams.py -x -q 2>&1 | tail -2
for cfg in C5 C1 C3; do for eng in 2 1; do
  TRB_ENGINE=$eng timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
    --verify-streams 1 > gpurun_out/ec.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ec.json').read().strip().splitlines()[-1]); print('$cfg engine $eng', round(d['value']), round(d['config']['stage_ms_per_step']['track_meanshift'],4), d.get('verify',{}).get('identical_to_reference'))"
done; done
