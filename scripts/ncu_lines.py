"""Per-CUDA-source-line stall attribution from an ncu report (needs -lineinfo)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep] + (["-k", sys.argv[3]] if len(sys.argv) > 3 else []) + [ "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
agg, ins, src = collections.Counter(), collections.Counter(), {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or not r[0]:
        continue
    try:
        ln = int(r[0])
        s = float(r[4])
        e = float(r[7])
    except (ValueError, IndexError):
        continue
    agg[(cur, ln)] += s
    ins[(cur, ln)] += e
    src[(cur, ln)] = r[1]
tot = sum(agg.values()) or 1
print(f"total stall samples {tot:.0f}, warp instructions {sum(ins.values()):.3g}")
for (f, l), v in agg.most_common(top):
    print(f"{100 * v / tot:5.1f}% {ins[(f, l)] / 1e6:9.1f}M  {f}:{l}  {src[(f, l)].strip()[:90]}")
