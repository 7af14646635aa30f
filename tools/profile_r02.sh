#!/bin/bash
# Round-2 measurement set: bench lines (C5 default + every config + the
# reference arm), the C5 steady launch list and ncu full captures of the
# dominant kernels (mean-shift, bulk motion; C4 CCL).  Bench numbers never
# come from a run under ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_c5.json 2> gpurun_out/r02_c5.err
timeout 1500 python bench.py --config all --steps 20 --warmup 5 --no-e2e > gpurun_out/r02_all.json 2> gpurun_out/r02_all.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02_launches_c5.csv \
  python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --verify-streams 0 > gpurun_out/r02_ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:track_meanshift_kernel -s 96 -c 1 \
  -o gpurun_out/r02_meanshift python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --verify-streams 0 \
  > gpurun_out/r02_ncu_ms.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:motion_mean_bulk -s 96 -c 1 \
  -o gpurun_out/r02_motion_bulk python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --verify-streams 0 \
  > gpurun_out/r02_ncu_motion.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ccl_local|ccl_merge" -s 190 -c 2 \
  -o gpurun_out/r02_c4_ccl python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --verify-streams 0 \
  > gpurun_out/r02_ncu_c4.log 2>&1
ls -la gpurun_out | tail -20
