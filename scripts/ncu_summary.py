"""Summarise an ncu report (run here, no GPU): key SOL / memory / scheduler metrics
and the top source lines by stall samples.  usage: ncu_summary.py rep.ncu-rep [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
keys = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Executed Instructions",
        "Eligible Warps Per Scheduler", "No Eligible", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Mem Busy", "Max Bandwidth"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = {n: i for i, n in enumerate(r[0])}
for row in r[1:]:
    if row[h["ID"]] == "0" and row[h["Metric Name"]] in keys:
        print(f"{row[h['Metric Name']]:34s} {row[h['Metric Value']]:>14s} {row[h['Metric Unit']]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh = rr[0]
for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "lts__t_bytes.sum",
             "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
             "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
             "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
             "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
             "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct"):
    if name in hh:
        i = hh.index(name)
        print(f"{name:62s} {rr[2][i]:>14s} {rr[1][i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
s = list(csv.reader(io.StringIO(src)))
hs = {n: i for i, n in enumerate(s[1])}
data = []
for row in s[2:]:
    if len(row) < 5 or row[0].startswith("Kernel") or row[0] == "Address":
        break
    data.append(row)
col = "Warp Stall Sampling (All Samples)"
tot = sum(int(x[hs[col]] or 0) for x in data)
print("stall samples", tot, "sass lines", len(data))
for row in sorted(data, key=lambda x: -int(x[hs[col]] or 0))[:top]:
    print(f"{row[hs[col]]:>6s} {row[hs['Instructions Executed']]:>10s}  {row[hs['Source']][:100]}")
# stall reasons, totals over the kernel
names = [n for n in s[1] if n.startswith("stall_") and "Not Issued" not in n]
tot_r = {n: sum(int(x[hs[n]] or 0) for x in data) for n in names}
print("stall reasons:", ", ".join(f"{k[6:]}={v}" for k, v in sorted(tot_r.items(), key=lambda x: -x[1]) if v))
