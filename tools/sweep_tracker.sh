# sweep the tracker's scheduling knobs (same box); prints fps and tracker ms
for cfg in "$@"; do
  env $cfg python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw.json 2>/dev/null
  echo "$cfg $(python -c "import json;d=json.load(open('gpurun_out/sw.json'));print(round(d['value']), round(d['config']['stage_ms_per_step']['track_meanshift'],3))")"
done
