#!/bin/bash
# HISTORICAL: the experiment this script A/B-tested was reverted (DESIGN.md lists the result);
# its knob no longer exists in the library.
# DRAM bytes of the mean-shift kernel with / without the L2 discard of dead scratch, and the bench line
cd "$(dirname "$0")/.."
for dc in 1 0; do
  TRB_DISCARD=$dc timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:track_meanshift_kernel -s 5 -c 2 --csv --log-file gpurun_out/dram_$dc.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --verify-streams 0 > /dev/null 2>&1
  python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/dram_$dc.csv')))
h=None
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print('discard=$dc', d['ID'], d['Metric Name'], d['Metric Value'], d['Metric Unit'])
PY
  TRB_DISCARD=$dc timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 2 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('discard=$dc', round(d['value']), d['verify']['identical_to_reference'])"
done
