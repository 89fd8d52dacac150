"""Run the CPU oracle once on a FULL-size BASELINE config and record its own
statistics, decision trace and wall time (calls only oracle/ and workloads/).
Output: profiles/oracle_full_config<k>.json.  Used by bench.py's cpu_baseline /
--impl reference legs to scale a bounded sample to one call."""
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from workloads import configs as W  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
t0 = time.time()
c = W.make(idx)
t_gen = time.time() - t0
t0 = time.time()
w, st, tr, rc = O.kiops(c["op"], c["u"], c["T"], tol=c["tol"], m_init=c["m_init"], m_min=c["m_min"],
                        m_max=c["m_max"], iop_q=c["iop_q"])
t_call = time.time() - t0
cpu = platform.processor() or platform.machine()
try:
    cpu = next(ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name"))
except (OSError, StopIteration):
    pass
SAMPLE_STRIDE = 257  # element-wise check of the GPU outputs at full size (tests/test_gpu_parity.py)
out = {"config": c["name"], "status": rc, "wall_s": t_call, "gen_s": t_gen, "threads": 1,
       "cpu": cpu, "nproc": os.cpu_count(), "stats": st,
       "trace": tr, "out_norms": [float((x * x).sum() ** 0.5) for x in w],
       "sample_stride": SAMPLE_STRIDE, "sample_file": f"oracle_full_config{idx}_sample.npz"}
os.makedirs("profiles", exist_ok=True)
import numpy as np  # noqa: E402

np.savez_compressed(f"profiles/oracle_full_config{idx}_sample.npz",
                    **{f"w{l}": np.asarray(x)[::SAMPLE_STRIDE] for l, x in enumerate(w)})
json.dump(out, open(f"profiles/oracle_full_config{idx}.json", "w"), indent=1)
print(json.dumps({k: out[k] for k in ("config", "status", "wall_s", "stats")}))
