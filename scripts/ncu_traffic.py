"""Extract per-launch DRAM traffic of the fused pass from a full ncu report into
profiles/ncu_traffic_config<k>.json (read by bench.py's roofline.traffic).
usage: ncu_traffic.py report.ncu-rep config_index [kernel_regex] [passes_per_launch]
(a persistent k_inner_* launch runs several passes: give their number to get per-pass bytes)"""
import csv
import io
import json
import re
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
pat = re.compile(sys.argv[3] if len(sys.argv) > 3 else "k_pass|k_csr|k_inner")
ppl = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
ki, rd, wr, du = (h.index(x) for x in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                        "gpu__time_duration.sum"))
units = r[1]
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tmult = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}  # -> us
rows = [x for x in r[2:] if pat.search(x[ki])]
tr = [(float(x[rd]) * mult[units[rd]] + float(x[wr]) * mult[units[wr]]) / ppl for x in rows]
res = {"report": rep.split("/")[-1], "kernel": rows[0][ki][:80], "launches": len(rows), "passes_per_launch": ppl,
       "bytes_per_launch": sum(tr) / len(tr), "note": "bytes_per_launch is per PASS (launch bytes / passes_per_launch)",
       "dram_read_bytes": [float(x[rd]) * mult[units[rd]] for x in rows],
       "dram_write_bytes": [float(x[wr]) * mult[units[wr]] for x in rows],
       "duration_us": [float(x[du]) * tmult[units[du]] for x in rows]}
json.dump(res, open(f"profiles/ncu_traffic_config{idx}.json", "w"), indent=1)
print(res)
