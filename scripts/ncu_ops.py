"""Executed warp instructions and stall samples per SASS opcode from an ncu
report's source page (the dynamic instruction mix of one kernel launch)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
i_src, i_s, i_e = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
ins, stall = collections.Counter(), collections.Counter()
for x in rows[2:]:
    s = x[i_src].split()
    if not s:
        continue
    op = s[1] if s[0].startswith("@") and len(s) > 1 else s[0]
    op = op.split(".")[0]
    ins[op] += float(x[i_e] or 0)
    stall[op] += float(x[i_s] or 0)
ti, ts = sum(ins.values()) or 1, sum(stall.values()) or 1
print(f"{'op':14s} {'inst':>14s} {'%inst':>6s} {'%stall':>6s}")
for op, v in ins.most_common(top):
    print(f"{op:14s} {v:14.0f} {100 * v / ti:6.1f} {100 * stall[op] / ts:6.1f}")
