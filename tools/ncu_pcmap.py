"""Map SASS PCs of an ncu report to (file:line) and show the source lines
around given hot instructions (by stall samples).  Diagnostics only.
python tools/ncu_pcmap.py rep.ncu-rep [n_top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 20
both = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                      capture_output=True, text=True).stdout
pc2src = {}
f = None
line = None
for r in csv.reader(both.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif r[0] and r[0] not in ("Line No", "Function Name"):
        line = (f, r[0], r[1].strip()[:70])
    elif len(r) > 3 and r[2].startswith("0x"):
        pc2src.setdefault(r[2], []).append(line)
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(sass.splitlines()))
hdr, R = rows[1], rows[2:]
isam = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[isam]) for r in R)
top = sorted(range(len(R)), key=lambda i: -int(R[i][isam]))[:ntop]
for i in top:
    r = R[i]
    # first following instruction with a non-helper source line
    ctx = None
    for j in range(i + 1, min(len(R), i + 40)):
        for s in pc2src.get(R[j][0], []):
            if s and s[0] not in ("helpers.h", "sm_90_rt.hpp", "cooperative_groups.h", "trb_exact.cuh") and "sync()" not in s[2]:
                ctx = s
                break
        if ctx:
            break
    own = [s for s in pc2src.get(r[0], []) if s]
    print(f"{int(r[isam]):7d} {100*int(r[isam])/tot:5.1f}% #{i:6d} {r[1].strip()[:34]:34s} own={own[-1][0]+':'+own[-1][1] if own else '-':22s} next={ctx[0]+':'+ctx[1]+' '+ctx[2] if ctx else '-'}")
