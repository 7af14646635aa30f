#!/bin/bash
# ncu full captures (one launch each, after the tracker's first steady steps)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:track_meanshift_kernel -s 5 -c 1 \
  -o gpurun_out/r02_meanshift python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --verify-streams 0 \
  > gpurun_out/r02_ncu_ms.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ccl_local|ccl_merge" -s 8 -c 2 \
  -o gpurun_out/r02_c4_ccl python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --verify-streams 0 \
  > gpurun_out/r02_ncu_c4.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"track_meanshift_kernel|motion_mean_bulk" -s 10 -c 4 --csv --log-file gpurun_out/r02_dram.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --verify-streams 0 > gpurun_out/r02_ncu_dram.log 2>&1
# v2 engine with the lean 3-lane centroid walk (C1 / C5)
for eng in 2; do for cfg in C1 C5; do
  TRB_ENGINE=$eng timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
    --verify-streams 1 > gpurun_out/ec.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ec.json').read().strip().splitlines()[-1]); print('$cfg engine $eng', round(d['value']), round(d['config']['stage_ms_per_step']['track_meanshift'],4), d.get('verify',{}).get('identical_to_reference'))"
done; done
ls gpurun_out/*.ncu-rep
