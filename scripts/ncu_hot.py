"""Top SASS instructions of an ncu report by warp-stall samples (dev aid):
python scripts/ncu_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = csv.reader(io.StringIO(raw))
h = next(r)
next(r)
d = dict(zip(h, next(r)))
st = []
for k, v in d.items():
    if "issue_stalled" in k and k.endswith(".ratio") and v:
        try:
            st.append((float(v.replace(",", "")), k))
        except ValueError:
            pass
print("stall reasons (cycles per issued instruction):")
for v, k in sorted(st, reverse=True)[:12]:
    print(f"  {v:8.2f} {k}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
lines = src.splitlines()
r = csv.reader(io.StringIO("\n".join(lines[1:])))
h = next(r)
rows = [dict(zip(h, row)) for row in r]
tot = sum(int(x["Warp Stall Sampling (All Samples)"] or 0) for x in rows)
print(f"total samples {tot}")
for x in sorted(rows, key=lambda x: -int(x["Warp Stall Sampling (All Samples)"] or 0))[:top]:
    s = int(x["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{s:7d} {100.0 * s / max(tot, 1):5.1f}%  {x['Address'][-5:]}  {x['Source'].strip()[:70]}")
