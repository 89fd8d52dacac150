"""Small calls of every kernel family for compute-sanitizer (test infrastructure):
  compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_run.py
Reduced grids so the instrumented run stays short: config 1 (1-CTA persistent loop,
single-CTA exponential), config 3 on 200 x 72 (2D persistent loop, cp.async rings),
config 4 on 48^3 and on 24 x 20 x 16 with KIOPS_3D-independent p variants (3D recompute
pass: TMA + mbarrier rings, padded copies, padded GEMV, cluster controller for n > 48),
config 5 on 24^3 (CSR split form + SELL SpMV).  Host loop and graph paths both."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1804_05126_b200 import Kiops  # noqa: E402
from workloads import configs as W  # noqa: E402

cases = [W.config1(), W.config3(200, 72), W.config4(48, 48, 48), W.config5(24, 24, 24)]
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    cases = cases[:1] + [W.config4(24, 20, 16)]
for c in cases:
    k = Kiops(c["op"], c["p"], device="cuda:0", tol=c["tol"], m_init=c["m_init"], m_min=c["m_min"], m_max=c["m_max"])
    u = [torch.as_tensor(x, device="cuda:0") for x in c["u"]]
    for hl in (False, True):
        w, st = k.apply(u, c["T"], hostloop=hl)
        torch.cuda.synchronize()
        print(c["name"], "hostloop" if hl else "graph", {x: st[x] for x in ("krylov_vectors", "passes", "substeps")},
              flush=True)
    k.close()
print("SANITIZE_RUN_DONE")
