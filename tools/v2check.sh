#!/bin/bash
# A/B the v2 exact-sum engine (TRB_ENGINE=2) on the GPU box, every step under
# its own timeout (a hung kernel must not hold the box).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export TRB_ENGINE=2
timeout 300 python -m pytest tests/test_gpu_tracker.py -x -q 2>&1 | tail -8
timeout 300 python -m pytest tests/test_gpu_streams.py -x -q 2>&1 | tail -8
timeout 120 python -c "
from paper_1310_3322_b200 import api; print(api.debug_stats())"
for eng in 2 1; do
  TRB_ENGINE=$eng timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --verify-streams 4 \
    > gpurun_out/v2_e$eng.json 2> gpurun_out/v2_e$eng.err
  echo "engine $eng rc=$?"
  timeout 60 python -c "
import json,sys; d=json.loads(open('gpurun_out/v2_e$eng.json').read().strip().splitlines()[-1]); print(d['value'], d['config']['stage_ms_per_step'], d.get('verify'))"
  tail -2 gpurun_out/v2_e$eng.err
done
