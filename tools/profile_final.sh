#!/bin/bash
# Round-end measurement set at HEAD: the driver-style C5 bench line, every
# config, the reference arm, the C5 steady launch list (ncu, durations only)
# and one ncu --set full capture of the mean-shift kernel.  Bench numbers
# never come from a run under ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err
timeout 1500 python bench.py --config all --steps 20 --warmup 5 > gpurun_out/final_all.json 2> gpurun_out/final_all.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/final_launches_c5.csv \
  python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --verify-streams 0 > gpurun_out/final_ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:track_meanshift_kernel -s 5 -c 1 \
  -o gpurun_out/final_meanshift python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --verify-streams 0 \
  > gpurun_out/final_ncu_ms.log 2>&1
ls -la gpurun_out | grep final
