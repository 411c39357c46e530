"""Summarise an ncu report: key raw metrics + top SASS stall sites."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
hdr, units, vals = r[0], r[1], r[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "launch__grid_size",
        "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct", "lts__t_bytes.sum"]
for h, u, v in zip(hdr, units, vals):
    if any(h == w or h.startswith(w) for w in want) and not h.endswith(("min", "max")):
        print(f"{h:70s} {u:10s} {v}")
for h, u, v in zip(hdr, units, vals):
    if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
        try:
            if float(v) > 0.05:
                print(f"{h:70s} {u:10s} {v}")
        except ValueError:
            pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
data = rows[2:]
i_src, i_s, i_e = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(float(x[i_s] or 0) for x in data)
print("stall samples", tot, "instructions", sum(float(x[i_e] or 0) for x in data))
for x in sorted(data, key=lambda x: -float(x[i_s] or 0))[:top]:
    print(x[0][-5:], f"{100 * float(x[i_s]) / tot:5.1f}%", f"{x[i_e]:>10s}", x[i_src][:80])
