"""EPIRK driver measurement: constant-step EPIRK4s3 / EPIRK4s3A /
EPIRK5P1 / EXPRB5s3 on the
periodic Allen-Cahn 2D problem (Sec. 4; reading E4) through kiops_epirk_step,
timed with CUDA events on the ctx stream after warm-up steps; the oracle EPIRK
(oracle/epirk.py, 1 thread) timed on a bounded sample of the same steps.  Prints one
JSON line.
  python scripts/epirk_bench.py [--n 1024] [--scheme epirk4s3] [--h 0.01] [--steps 5] [--warmup 2]
  python scripts/epirk_bench.py --problem adr --n 400 --h 0.0025   (ADR 2D with Neumann boundaries,
      P:601-609 / P:649: N = 400^2; the linear part as a CSR matrix, reading E10)"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1804_05126_b200 import KiopsEpirk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--problem", default="allen_cahn", choices=["allen_cahn", "adr", "allen_cahn_noflow"])
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--scheme", default="epirk4s3", choices=["epirk4s3", "epirk4s3a", "epirk5p1", "exprb5s3"])
ap.add_argument("--h", type=float, default=0.01)
ap.add_argument("--tol", type=float, default=1e-10)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--oracle-steps", type=int, default=1, help="bounded CPU sample (0: skip)")
a = ap.parse_args()

n = a.n
if a.problem == "adr":
    from oracle import epirk as E0  # (the problem generator: CSR of L and the initial condition)

    prob, u0 = E0.adr_neumann(n, n)
    pb = {"nx": n, "ny": n, "c": list(prob.c), "L": {"row_ptr": prob.row_ptr, "col_idx": prob.col_idx, "vals": prob.vals}}
    wname, dname = f"adr_neumann_2d_{n}x{n}", "ADR 2D, homogeneous Neumann (CSR linear part)"
elif a.problem == "allen_cahn_noflow":
    from oracle import epirk as E0

    prob, u0 = E0.allen_cahn_noflow(n, n)
    pb = {"nx": n, "ny": n, "c": list(prob.c), "L": {"row_ptr": prob.row_ptr, "col_idx": prob.col_idx, "vals": prob.vals}}
    wname, dname = f"allen_cahn_noflow_2d_{n}x{n}", "Allen-Cahn 2D, no-flow boundaries (CSR linear part)"
else:
    alpha = 0.1
    dx = 2.0 / n
    wa = alpha / dx ** 2
    pb = {"nx": n, "ny": n, "w": [wa, wa, wa, wa, -4 * wa], "c": [0.0, 1.0, 0.0, -1.0]}
    xs = -1.0 + dx * np.arange(n)
    X, Y = np.meshgrid(xs, xs, indexing="xy")
    u0 = (0.1 + 0.1 * np.cos(2 * np.pi * X) * np.cos(2 * np.pi * Y)).ravel()
    wname, dname = f"allen_cahn_2d_{n}x{n}", "Allen-Cahn 2D periodic"

dev = torch.device("cuda:0")
k = KiopsEpirk(pb, a.scheme, a.h, device=dev, tol=a.tol)
u = torch.as_tensor(u0.copy(), device=dev)
k.step(u, a.warmup)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(k.stream)
st = k.step(u, a.steps)
e1.record(k.stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
line = {"metric": f"{a.scheme} step time, {dname} (EPIRK driver, f1)", "value": ms,
        "unit": "ms/step", "n_gpus": 1, "steps": a.steps, "warmup": a.warmup, "higher_is_better": False,
        "dtype": "f64", "data": "synthetic (the paper's initial condition)",
        "config": {"workload": wname, "N": n * n, "h": a.h, "tol": a.tol, "scheme": a.scheme,
                   "kiops_calls_per_step": 3 if a.scheme in ("epirk5p1", "exprb5s3") else 2,
                   "per_step": {"krylov_vectors": st["krylov_vectors"] / a.steps, "passes": st["passes"] / a.steps,
                                "rejections": st["rejections"] / a.steps,
                                "kiops_device_ms": st["kiops_ms"] / a.steps},
                   "final_m": st["final_m"]},
        "gpu_launches_per_step": None}
if a.oracle_steps > 0:
    from oracle import epirk as E

    if a.problem == "allen_cahn":
        prob = E.ReactionDiffusion2D(n, alpha=alpha)
    y = u0.copy()
    t0 = time.perf_counter()
    five = a.scheme in E.SCHEMES5
    m = (10, 10, 10) if five else (10, 10)
    for _ in range(a.oracle_steps):
        y, m, _ = (E.step5 if five else E.step)(prob, a.scheme, y, a.h, tol=a.tol, m_hint=m)
    cpu_ms = (time.perf_counter() - t0) * 1e3 / a.oracle_steps
    line["cpu_baseline"] = {"value": cpu_ms, "unit": "ms/step", "cores": 1, "kind": "oracle",
                            "sample": f"first {a.oracle_steps} step(s) of the same run from u_0 (oracle EPIRK over the C KIOPS oracle)"}
print(json.dumps(line))
