"""Top source lines (cuda,sass view) of an ncu report by warp-stall samples."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
f = None
hdr = None
res = []
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] != "" and len(r) == len(hdr):
        try:
            s = int(r[4])
        except ValueError:
            continue
        st = {k: int(v) for k, v in zip(hdr, r) if k.startswith("stall_") and "(Not" not in k and v.isdigit()}
        top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        res.append((s, f, r[0], r[1].strip()[:64], int(r[7]) if r[7].isdigit() else 0, top))
tot = sum(o[0] for o in res)
print("total samples (lines, inlined frames double-count)", tot)
for o in sorted(res, key=lambda o: -o[0])[:n]:
    top = " ".join(f"{k[6:]}={v}" for k, v in o[5])
    print(f"{o[0]:7d} {o[1]}:{o[2]:5s} inst={o[4]/1e6:8.2f}M {o[3]:64s} {top}")
