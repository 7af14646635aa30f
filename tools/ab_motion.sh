# motion kernel variants (TRB_LIB): roofline_motion from bench (stage profile)
for lib in "$@"; do
  if [ "$lib" = default ]; then unset TRB_LIB; else export TRB_LIB=$PWD/paper_1310_3322_b200/variants/libtrb_$lib.so; fi
  timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/b.json 2>/dev/null
  echo "$lib $(python -c "import json;d=json.load(open('gpurun_out/b.json'));print(round(d['value']), round(d['roofline_motion']['achieved']), round(d['roofline_motion']['frac'],3))")"
done
