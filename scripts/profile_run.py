"""One KIOPS call through the host-loop profiling hook (kiops_apply_hostloop), so
Nsight Compute can see every kernel (it cannot profile kernel nodes of graphs with
conditional nodes).  Same kernels and results as kiops_apply (tested bitwise).
  python scripts/profile_run.py [--config 4] [--dims 256 256 256]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1804_05126_b200 import Kiops  # noqa: E402
from workloads import configs as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--dims", type=int, nargs="*", default=[])
ap.add_argument("--graph", action="store_true", help="use the graph path instead of the host loop")
a = ap.parse_args()
c = W.make(a.config, *a.dims)
k = Kiops(c["op"], c["p"], device="cuda:0", tol=c["tol"], m_init=c["m_init"], m_min=c["m_min"], m_max=c["m_max"])
u = [torch.as_tensor(x, device="cuda:0") for x in c["u"]]
w, st = k.apply(u, c["T"], hostloop=not a.graph)
torch.cuda.synchronize()
print(c["name"], {x: st[x] for x in ("krylov_vectors", "passes", "substeps", "rejections", "expm_calls", "pass_ms",
                                     "ctrl_ms", "gemv_ms")})
