#!/bin/bash
# HISTORICAL: the experiment this script A/B-tested was reverted (DESIGN.md lists the result);
# its knob no longer exists in the library.
# serial sums for tiny windows: correctness + threshold sweep
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_tracker.py tests/test_gpu_streams.py -x -q 2>&1 | tail -2
TRB_SERIAL_MAX=100000 timeout 600 python -m pytest tests/test_gpu_tracker.py -x -q 2>&1 | tail -2
for cfg in C1 C2 C5; do for m in 0 1024 2048 4096; do
  TRB_SERIAL_MAX=$m timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
    --verify-streams 1 > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg serial_max=$m', round(d['value']), round(d['ms_per_step'],3), d['verify']['identical_to_reference'])"
done; done
