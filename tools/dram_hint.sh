#!/bin/bash
# DRAM bytes of the mean-shift kernel with / without the L2 evict_last hint
# on its scratch stores (variant libtrb_nohint.so), and the bench line
cd "$(dirname "$0")/.."
for v in cur nohint; do
  lib=paper_1310_3322_b200/libtrb.so; [ $v != cur ] && lib=paper_1310_3322_b200/variants/libtrb_$v.so
  TRB_LIB=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:track_meanshift_kernel -s 5 -c 2 --csv --log-file gpurun_out/dramh_$v.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --verify-streams 0 > /dev/null 2>&1
  python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/dramh_$v.csv')))
h=None
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print('$v', d['ID'], d['Metric Name'], d['Metric Value'], d['Metric Unit'])
PY
done
for rep in 1 2; do for v in cur nohint; do
  lib=paper_1310_3322_b200/libtrb.so; [ $v != cur ] && lib=paper_1310_3322_b200/variants/libtrb_$v.so
  TRB_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 2 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$v', round(d['value']), d['config']['stage_ms_per_step'], d['verify']['identical_to_reference'])"
done; done
