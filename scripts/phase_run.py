"""Debug helper (not product code): one config-4 call on a KIOPS_PHASE_TIMERS build
(KIOPS_LIB=<that .so>), to print the persistent loop's per-launch phase sums.
  nvcc ... -DKIOPS_PHASE_TIMERS -o mbbin/libkiops_phase.so paper_1804_05126_b200/csrc/kiops.cu
  KIOPS_LIB=mbbin/libkiops_phase.so python scripts/phase_run.py [config] [dims...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1804_05126_b200 import Kiops  # noqa: E402
from workloads import configs as W  # noqa: E402

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dims = [int(x) for x in sys.argv[2:]]
c = getattr(W, f"config{cfgn}")(*dims)
k = Kiops(c["op"], c["p"], device="cuda:0", tol=c["tol"], m_init=c["m_init"], m_min=c["m_min"], m_max=c["m_max"])
u = [torch.as_tensor(x, device="cuda:0") for x in c["u"]]
for rep in range(2):
    w, st = k.apply(u, c["T"])
    torch.cuda.synchronize()
    print("STATS", rep, st, flush=True)
