# Round profile set (one GPU): bench line, full launch list (steady steps are
# cut out offline), ncu full capture of the top kernel (mean-shift).
set -x
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
    --log-file gpurun_out/launches_all.csv python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l.log 2>&1
ncu --set full --import-source on --clock-control none -k track_meanshift_kernel --launch-skip 6 -c 1 \
    -o gpurun_out/ms_full python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ms.log 2>&1
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
