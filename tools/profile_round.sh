# Round profile set (one GPU): bench line, steady-state launch list, ncu full
# capture of the top kernel (mean-shift) and of motion / ccl_local.
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 700 -c 80 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l.log 2>&1
ncu --set full --import-source on --clock-control none -k track_meanshift_kernel --launch-skip 6 -c 1 \
    -o gpurun_out/ms_full python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ms.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"motion_mean_kernel|ccl_local_kernel" --launch-skip 100 -c 2 \
    -o gpurun_out/mc_full python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_mc.log 2>&1
