#!/usr/bin/env python
"""bench.py -- KIOPS call time on one B200 (fp64), BASELINE.json's metric.

A step = one kiops_apply (the whole hot path: setup, every fused IOP pass, every
controller attempt, every GEMV) on the synthetic input of one BASELINE config,
inputs resident in HBM.  Default workload: config 4 (3D variable-kappa 256^3,
p = 2, three output times) -- the largest single-GPU config and the one the
HBM-roofline target is stated on.  Every vector is 134 MB and the basis 17 GB, so
inputs exceed the 126 MB L2 between steps (no explicit flush needed).

  python bench.py [--gpus N --steps K --warmup W --config C --impl kiops|reference]

N > 1 (torchrun): independent replicas, one per GPU, no collective in the data
path ("replicas only"); value = max-over-ranks time / (N K).
--impl reference: the CPU oracle (oracle/) timed on the host cores on a bounded
sample of the same workload, rank 0 only.
Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "KIOPS call time (ms) + fused matvec/IOP HBM GB/s vs B200 peak, fp64, 1 GPU"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def hbm_peak():
    p = peaks()
    if "hbm_gbs" in p:
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def box_copy_gbs(torch, dev):
    """This box's copy bandwidth, measured like MEASURED_PEAKS.json (read + write bytes of a
    1 GiB bf16 copy, best of 5, CUDA events): context for the roofline, since boxes of the
    pool differ (the roofline's peak stays the driver-measured figure)."""
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
    b = torch.empty_like(a)
    b.copy_(a)
    best = None
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3
        best = t if best is None or t < best else best
    del a, b
    torch.cuda.empty_cache()
    return 2 * (1 << 30) * 2 / best / 1e9


def oracle_counts(idx):
    """The oracle's OWN counts for the full config (scripts/oracle_full_run.py)."""
    path = os.path.join(ROOT, "profiles", f"oracle_full_config{idx}.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d["stats"], d.get("wall_s")
    return None, None


def host_cpu():
    """CPU model and core count of the host (reported beside every oracle timing)."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model or (os.uname().machine if hasattr(os, "uname") else "?"), "nproc": os.cpu_count()}


def cpu_sample(cfg, idx, n_kv=4, proj_frac=16):
    """Oracle as it stands on the host cores (1 thread).  If one full oracle call of this
    workload takes < 20 s (profiles/oracle_full_config<k>.json), time the full call
    (median of up to 3).  Otherwise a bounded sample of the same workload, every part
    of a call measured at full size and scaled by the oracle's own full-size counts:
      * Alg. 2: n_kv Krylov vectors from the real start vector;
      * one Pade-13 exponential of a 129^2 H~ (the oracle's Alg. 2 on the same-weights
        48^3 grid);
      * Alg. 3's projection w = beta V f (the oracle's own loop, exported as or_project)
        over 1/proj_frac of the rows of a full-size basis with 129 columns (the same
        column stride N + p), times proj_frac, per projection, scaled by j/129, for every
        accepted substep and every crossed output time of the oracle's trace."""
    from oracle import oracle as O
    from workloads import configs as W

    st, wall = oracle_counts(idx)
    if st is not None and wall is not None and wall < 20.0:
        ts = []
        for _ in range(3 if wall < 2.0 else 1):
            t0 = time.perf_counter()
            O.kiops(cfg["op"], cfg["u"], cfg["T"], tol=cfg["tol"], m_init=cfg["m_init"], m_min=cfg["m_min"],
                    m_max=cfg["m_max"], iop_q=cfg["iop_q"])
            ts.append(time.perf_counter() - t0)
        v = float(np.median(ts)) * 1e3
        return dict({"value": v, "unit": "ms/call", "cores": 1, "kind": "oracle",
                     "sample": f"full oracle call (Alg. 1-4, 1 thread), median of {len(ts)}"}, **host_cpu())
    if st is None:
        return None
    p, N = cfg["p"], cfg["N"]
    nu, mu = O.normalisation(cfg["u"])
    v0 = np.r_[cfg["u"][0], np.zeros(max(p - 1, 0)), [mu] if p else []]
    t0 = time.perf_counter()
    O.iop(cfg["op"], cfg["u"], nu, v0, n_kv, cfg["iop_q"])
    t_kv = (time.perf_counter() - t0) / n_kv
    small = W.make(idx, *([48] * (3 if idx in (4, 5) else 2 if idx in (2, 3) else 1)))
    nu2, mu2 = O.normalisation(small["u"])
    v2 = np.r_[small["u"][0], np.zeros(max(p - 1, 0)), [mu2] if p else []]
    m = min(128, small["m_max"])
    V, H, j, happy = O.iop(small["op"], small["u"], nu2, v2, m, 2)
    Ht = np.zeros((j + 1, j + 1))
    Ht[:j, :j] = H[:j, :j]
    Ht[0, j] = 1.0
    tau = float(cfg["T"][-1]) / 8
    t0 = time.perf_counter()
    O.expm(Ht, tau)
    t_exp = time.perf_counter() - t0
    # projection sample: rows 0 .. N/proj_frac of a (N+p) x 129 column-major basis
    ld, jc, rows = N + p, 129, N // proj_frac
    Vb = np.empty(ld * jc)  # virtual; only the sampled rows are touched
    for c in range(jc):
        Vb[c * ld:c * ld + rows] = 1.0 / (c + 1)
    f = np.linspace(1.0, 2.0, jc)
    O.project(Vb, ld, rows, f)  # warm
    t0 = time.perf_counter()
    O.project(Vb, ld, rows, f)
    t_proj = (time.perf_counter() - t0) * proj_frac
    del Vb
    tr = json.load(open(os.path.join(ROOT, "profiles", f"oracle_full_config{idx}.json"))).get("trace", [])
    acc_j = [r["j"] for r in tr if r["accept"]]
    n_cross = len(cfg["T"]) - 1
    j_proj = acc_j + [max(acc_j) if acc_j else jc] * n_cross
    t_gemv = sum(t_proj * jj / jc for jj in j_proj)
    est_ms = 1e3 * (t_kv * st["krylov_vectors"] + t_exp * st["expm_calls"] + t_gemv)
    return dict({"value": est_ms, "unit": "ms/call", "cores": 1, "kind": "oracle",
                 "sample": f"oracle at full size, 1 thread: {n_kv} Krylov vectors ({t_kv*1e3:.0f} ms/KV), one {j+1}^2 "
                           f"Pade-13 expm ({t_exp*1e3:.1f} ms), the Alg. 3 projection on 1/{proj_frac} of the rows of a "
                           f"129-column basis ({t_proj:.1f} s per full projection); scaled by the oracle's own counts "
                           f"({st['krylov_vectors']} KVs, {st['expm_calls']} expm, {len(j_proj)} projections)"
                           + (f"; one measured full oracle call took {wall:.1f} s on the build host" if wall else ""),
                 "t_kv_ms": t_kv * 1e3, "t_expm_ms": t_exp * 1e3, "t_proj_s": t_proj}, **host_cpu())


class ClockSampler:
    def __init__(self, path):
        self.path = path
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self, dev_index=0):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines()]
        except Exception:
            return None
        rows = [[x.strip() for x in r] for r in rows if len(r) >= 9 and r[0].strip() == str(dev_index)]
        if not rows:
            return None
        sm = sorted(float(r[1]) for r in rows)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][2]), "reasons": sorted(reasons),
                "samples": len(rows)}


def max_over_ranks(x, dist=None, device="cpu"):
    """max of a per-rank float over all ranks (identity without a process group)"""
    if dist is None or not dist.is_available() or not dist.is_initialized():
        return float(x)
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def bytes_per_pass(cfg):
    from workloads import configs as W

    return W.algorithmic_bytes_per_pass(cfg)


def secondary_config3(torch, dev, Kiops, W, peak, box_gbs, steps=10):
    """BASELINE config 3 (2D Allen-Cahn Jacobian, 1024^2, p = 3), the other roofline
    target of north_star, timed in the same process right after config 4: ms/call
    (CUDA events, inputs resident) and the fused-pass roofline fraction (per-pass device
    timer, algorithmic bytes).  Its 75 MB per-pass working set fits the 126 MB L2, so
    the 'hbm' fraction is partly an L2 figure."""
    c = W.make(3)
    u = [torch.as_tensor(x).to(dev) for x in c["u"]]
    k = Kiops(c["op"], c["p"], device=dev, tol=c["tol"], m_init=c["m_init"], m_min=c["m_min"], m_max=c["m_max"],
              iop_q=c["iop_q"])
    w = [torch.empty(c["N"], dtype=torch.float64, device=dev) for _ in c["T"]]
    for _ in range(3):
        k.apply(u, c["T"], w)
    torch.cuda.synchronize()
    tot = {"pass_ms": 0.0, "ctrl_ms": 0.0, "gemv_ms": 0.0, "passes": 0}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(k.stream)
    for _ in range(steps):
        _, st = k.apply(u, c["T"], w)
        for key in tot:
            tot[key] += st[key]
    e1.record(k.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    k.close()
    bpp = bytes_per_pass(c)
    ach = bpp * tot["passes"] / (tot["pass_ms"] * 1e-3) / 1e9
    return {"workload": c["name"], "value": ms, "unit": "ms/call", "steps": steps,
            "passes_per_call": tot["passes"] / steps, "pass_us": 1e3 * tot["pass_ms"] / tot["passes"],
            "device_ms": {"fused_pass": tot["pass_ms"] / steps, "controller": tot["ctrl_ms"] / steps,
                          "gemv": tot["gemv_ms"] / steps},
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "frac_of_box_copy": ach / box_gbs, "kernel": "k_inner_2d_lazy (fused IOP pass, persistent)",
                         "algorithmic_bytes_per_pass": bpp,
                         "note": "75 MB per-pass working set < 126 MB L2: partly an L2 figure (D10)"}}


def run_reference(args):
    from workloads import configs as W

    cfg = W.make(args.config)
    for _ in range(args.warmup):
        cpu_sample(cfg, args.config, n_kv=2)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s = cpu_sample(cfg, args.config, n_kv=2)
        if s is None:
            print(json.dumps({"impl": "reference", "unavailable": "profiles/oracle_full_config*.json missing"}))
            return
        vals.append(s["value"])
    wall = time.perf_counter() - t0
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "ms/call", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "N": cfg["N"], "p": cfg["p"], "T": list(map(float, cfg["T"])),
                       "tol": cfg["tol"], "sample_wall_s": wall},
            "cpu_baseline": dict(s, value=v),
            "e2e": {"value": v, "unit": "ms/call", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="kiops", choices=["kiops", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-secondary", action="store_true", help="skip the config-3 secondary line")
    ap.add_argument("--hostloop", action="store_true",
                    help="profiling only: same kernels, host-driven loop (ncu cannot see kernels in conditional graphs)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_1804_05126_b200 import Kiops
    from workloads import configs as W

    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    cfg = W.make(args.config)
    u = [torch.as_tensor(x).to(dev) for x in cfg["u"]]
    k = Kiops(cfg["op"], cfg["p"], device=dev, tol=cfg["tol"], m_init=cfg["m_init"], m_min=cfg["m_min"],
              m_max=cfg["m_max"], iop_q=cfg["iop_q"], host_staging=1, max_outputs=len(cfg["T"]))
    stream = k.stream
    w = [torch.empty(cfg["N"], dtype=torch.float64, device=dev) for _ in cfg["T"]]
    for _ in range(max(3, args.warmup)):
        k.apply(u, cfg["T"], w, hostloop=args.hostloop)
    torch.cuda.synchronize()

    clk = ClockSampler(os.path.join(ROOT, f"gpurun_out/clocks_rank{rank}.csv"
                                    if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else f"/tmp/clocks_{rank}.csv"))
    totals = {"pass_ms": 0.0, "ctrl_ms": 0.0, "expm_ms": 0.0, "gemv_ms": 0.0, "passes": 0, "krylov_vectors": 0, "expm_calls": 0,
              "substeps": 0, "rejections": 0, "pass_launches": 0}
    with clk:
        time.sleep(0.3)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            _, st = k.apply(u, cfg["T"], w, hostloop=args.hostloop)
            for key in totals:
                totals[key] += st[key]
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms_total = max_over_ranks(ev0.elapsed_time(ev1), dist if world > 1 else None, dev)
    ms_step = ms_total / args.steps

    # end to end: host buffers through kiops_apply_host, copies inside the timed region
    hu = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in cfg["u"]]
    hw = [torch.empty(cfg["N"], dtype=torch.float64).pin_memory() for _ in cfg["T"]]
    k.apply_host(hu, cfg["T"], hw)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e2e_dev = 0.0
    e0.record(stream)
    for _ in range(args.e2e_steps):
        _, st2 = k.apply_host(hu, cfg["T"], hw)
        e2e_dev += st2["pass_ms"] + st2["ctrl_ms"] + st2["gemv_ms"]
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps, dist if world > 1 else None, dev)
    e2e_dev /= args.e2e_steps

    bpp = bytes_per_pass(cfg)
    passes = totals["passes"] / args.steps
    pass_ms = totals["pass_ms"] / args.steps
    achieved = bpp * passes / (pass_ms * 1e-3) / 1e9 if pass_ms > 0 else None
    peak, peak_src = hbm_peak()
    box_gbs = box_copy_gbs(torch, dev)
    per_step = {key: totals[key] / args.steps for key in totals}
    # setup + pass kernels (per pass, or one persistent launch per Alg. 2 run; CSR: form + SpMV per
    # pass) + one controller per attempt + one GEMV per accepted substep
    launches_per_step = 1 + (2 if cfg["op"]["kind"] == "csr" else 1) * per_step["pass_launches"] + \
        (per_step["substeps"] + per_step["rejections"]) + per_step["substeps"]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_config{args.config}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": ms_step / world, "unit": "ms/call", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "N": cfg["N"], "p": cfg["p"], "T": [float(t) for t in cfg["T"]],
                   "tol": cfg["tol"], "m_max": cfg["m_max"], "iop_q": cfg["iop_q"],
                   "parallelism": f"replicas{world}" if world > 1 else "single",
                   "control_flow": "host loop (profiling)" if args.hostloop else "device graph (WHILE/IF conditional nodes)",
                   "l2": "inputs larger than L2 (vector 134 MB, basis 17 GB); no flush needed",
                   "per_call": {"krylov_vectors": per_step["krylov_vectors"], "passes": per_step["passes"],
                                "substeps": per_step["substeps"], "rejections": per_step["rejections"],
                                "expm_calls": per_step["expm_calls"],
                                "device_ms": {"fused_pass": pass_ms, "controller": per_step["ctrl_ms"],
                                              "controller_expm": per_step["expm_ms"], "gemv": per_step["gemv_ms"]},
                                "kv_per_s": per_step["krylov_vectors"] / (ms_step * 1e-3)}},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "kernel": {"stencil3d7": ("k_inner_3d_lazyq (fused IOP pass, persistent inner loop)" if
                                               os.environ.get("KIOPS_3D") == "lazy" else
                                               "k_inner_3d_rc (fused IOP pass, recompute form, TMA-fed, persistent inner loop)"),
                                "stencil2d5": "k_inner_2d_lazy (fused IOP pass, persistent inner loop)",
                                "stencil1d3": "k_inner_2d_lazy (fused IOP pass, ny = 1, persistent inner loop)",
                                "csr": "k_csr_form + k_sell_spmv (fused IOP pass)"}.get(cfg["op"]["kind"], "fused IOP pass"),
                     "algorithmic_bytes_per_pass": bpp, "passes_per_launch": (per_step["passes"] / per_step["pass_launches"]) if per_step["pass_launches"] else None, "peak_source": peak_src,
                     "box_copy_gbs": box_gbs, "frac_of_box_copy": (achieved / box_gbs) if achieved else None,
                     "timing": "device %globaltimer per pass (pass start to the end of its grid reduction and "
                               "finalisation), accumulated inside the graph over the timed steps"},
        "gpu_launches": int(round(launches_per_step * args.steps)),
        "e2e": {"value": e2e_ms / world, "unit": "ms/call",
                "h2d_bytes_per_step": 8 * cfg["N"] * (cfg["p"] + 1),
                "d2h_bytes_per_step": 8 * cfg["N"] * len(cfg["T"]),
                "steps": args.e2e_steps,
                "device_kernel_ms": e2e_dev,
                "note": "kiops_apply_host: H2D of u_0..u_p from pinned memory, then the graph; outputs are pinned "
                        "device-mapped host buffers written by the GEMV over the host link (no staging + D2H). "
                        "device_kernel_ms = the in-graph %globaltimer sums (passes + controller + GEMV) of these "
                        "calls; the rest of the call is the H2D copies, k_setup and the host-link output writes"},
        "clocks": clk.summary(local),
    }
    if rank == 0 and args.config == 4 and not args.no_secondary:
        line["secondary"] = secondary_config3(torch, dev, Kiops, W, peak, box_gbs)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_sample(cfg, args.config)
        except Exception as e:  # report, never fake
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(line))
    k.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
