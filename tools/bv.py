"""Print value / e2e / stage ms of bench.py JSON lines read from stdin."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    st = d.get("config", {}).get("stage_ms_per_step", {})
    e2e = d.get("e2e", {}).get("value")
    print(f"value {d.get('value', 0):.1f}  e2e {e2e if e2e is None else round(e2e, 1)}  ms/step {d.get('ms_per_step', 0):.3f}  "
          + " ".join(f"{k} {v:.3f}" for k, v in st.items()))
