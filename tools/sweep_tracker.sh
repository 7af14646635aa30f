for cfg in "TRB_CLUSTER=8 TRB_SPLIT_US=300" "TRB_CLUSTER=8 TRB_SPLIT_US=600" "TRB_CLUSTER=8 TRB_SPLIT_US=1200" "TRB_CLUSTER=8 TRB_SPLIT_US=150" "TRB_CLUSTER=16 TRB_SPLIT_US=300" "TRB_CLUSTER=16 TRB_SPLIT_US=1200" "TRB_CLUSTER=4 TRB_SPLIT_US=300" "TRB_CLUSTER=4 TRB_SPLIT_US=1000"; do
  env $cfg python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw.json 2>/dev/null
  echo "$cfg $(python -c "import json;d=json.load(open('gpurun_out/sw.json'));print(round(d['value']), d['config']['stage_ms_per_step']['track_meanshift'])")"
done
