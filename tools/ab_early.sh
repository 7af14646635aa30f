#!/bin/bash
# HISTORICAL: the experiment this script A/B-tested was reverted (DESIGN.md lists the result);
# its knob no longer exists in the library.
# A/B of the split-mode knobs (early split clusters, split threshold) on C5
cd "$(dirname "$0")/.."
CFG=${CFG:-C5}
for rep in 1 2; do
for kv in "TRB_SPLIT_EARLY=0 TRB_SPLIT_US=200" "TRB_SPLIT_EARLY=1 TRB_SPLIT_US=200" "TRB_SPLIT_EARLY=1 TRB_SPLIT_US=600" \
          "TRB_SPLIT_EARLY=1 TRB_SPLIT_US=1200" "TRB_SPLIT_EARLY=1 TRB_SPLIT_US=2000" "TRB_SPLIT_EARLY=0.7 TRB_SPLIT_US=1200" \
          "TRB_SPLIT_EARLY=1.3 TRB_SPLIT_US=1200"; do
  env $kv timeout 300 python bench.py --config $CFG --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 2 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$kv', round(d['value']), round(d['ms_per_step'],3), d.get('verify',{}).get('identical_to_reference'))"
done; done
