"""Thin ctypes binding of the KIOPS C ABI (include/kiops.h).

Argument marshalling only: torch tensors provide device memory and the CUDA
stream; every step of the method runs inside libkiops_b200.so (sm_100a kernels).
There is no CPU fallback: if the shared library is missing or no CUDA device is
present, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KIOPS_LIB") or os.path.join(HERE, "libkiops_b200.so")  # KIOPS_LIB: debug builds (scripts/)

MAX_P, MAX_OUT, MAX_M, MAX_FORCED, TRACE_CAP = 8, 64, 128, 256, 16384
KIND = {"stencil1d3": 1, "stencil2d5": 2, "stencil3d7": 3, "csr": 4}
STATUS = {0: "KIOPS_OK", 1: "KIOPS_ERR_INVALID_ARG", 2: "KIOPS_ERR_UNSUPPORTED", 3: "KIOPS_ERR_CUDA",
          4: "KIOPS_ERR_NO_CONVERGENCE", 5: "KIOPS_ERR_NONFINITE", 6: "KIOPS_ERR_WORKSPACE"}

_dp = C.POINTER(C.c_double)


class OperatorDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("periodic", C.c_int32), ("nx", C.c_int64), ("ny", C.c_int64),
                ("nz", C.c_int64), ("w", C.c_double * 5), ("diag", C.c_void_p), ("kappa", C.c_void_p),
                ("inv_h2", C.c_double), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
                ("vals", C.c_void_p), ("nnz", C.c_int64)]


class Options(C.Structure):
    _fields_ = [("tol", C.c_double), ("m_init", C.c_int32), ("m_min", C.c_int32), ("m_max", C.c_int32),
                ("iop_q", C.c_int32), ("task1", C.c_int32), ("max_attempts", C.c_int64),
                ("host_staging", C.c_int32), ("max_outputs", C.c_int32), ("corrected", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("substeps", C.c_int64), ("rejections", C.c_int64), ("krylov_vectors", C.c_int64),
                ("expm_calls", C.c_int64), ("passes", C.c_int64), ("final_m", C.c_int32),
                ("happy_breakdowns", C.c_int32), ("t_reached", C.c_double), ("nu", C.c_double),
                ("mu", C.c_double), ("pass_ms", C.c_double), ("ctrl_ms", C.c_double), ("gemv_ms", C.c_double),
                ("expm_ms", C.c_double), ("pass_launches", C.c_int64)]


class TraceRow(C.Structure):
    _fields_ = [("attempt", C.c_int64), ("j", C.c_int32), ("happy", C.c_int32), ("accept", C.c_int32),
                ("m_new", C.c_int32), ("t_now", C.c_double), ("tau", C.c_double), ("beta", C.c_double),
                ("h_next", C.c_double), ("eps", C.c_double), ("omega", C.c_double),
                ("tau_new", C.c_double)]


SYMBOLS = ["kiops_options_default", "kiops_workspace_bytes", "kiops_create", "kiops_apply",
           "kiops_apply_host", "kiops_apply_hostloop", "kiops_get_trace", "kiops_set_m_init",
           "kiops_set_forced_schedule", "kiops_debug_basis", "kiops_destroy", "kiops_status_string", "kiops_last_error",
           "kiops_epirk_workspace_bytes", "kiops_epirk_create", "kiops_epirk_step", "kiops_epirk_destroy",
           "kiops_epirk_last_error"]


class RDProblem(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("w", C.c_double * 5), ("c", C.c_double * 4),
                ("L_row_ptr", C.c_void_p), ("L_col_idx", C.c_void_p), ("L_vals", C.c_void_p), ("L_nnz", C.c_int64)]


class EpirkStats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("krylov_vectors", C.c_int64), ("passes", C.c_int64),
                ("substeps", C.c_int64), ("rejections", C.c_int64), ("expm_calls", C.c_int64),
                ("final_m", C.c_int32 * 3), ("kiops_ms", C.c_double)]


EPIRK_HIST_ATTEMPTS = 64


class EpirkCallRecord(C.Structure):
    _fields_ = [("step", C.c_int32), ("call", C.c_int32), ("final_m", C.c_int32), ("n_attempts", C.c_int32),
                ("krylov_vectors", C.c_int64), ("substeps", C.c_int64), ("rejections", C.c_int64),
                ("j", C.c_int16 * EPIRK_HIST_ATTEMPTS), ("m_new", C.c_int16 * EPIRK_HIST_ATTEMPTS),
                ("accept", C.c_int8 * EPIRK_HIST_ATTEMPTS), ("omega", C.c_double * EPIRK_HIST_ATTEMPTS)]


EPIRK_SCHEMES = {"epirk4s3": 1, "epirk4s3a": 2, "epirk5p1": 3, "exprb5s3": 4}

_lib = None


def lib():
    """Load libkiops_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.kiops_options_default.argtypes = [C.POINTER(Options)]
        L.kiops_options_default.restype = None
        L.kiops_workspace_bytes.argtypes = [C.POINTER(OperatorDesc), C.c_int, C.POINTER(Options),
                                            C.POINTER(C.c_size_t)]
        L.kiops_create.argtypes = [C.POINTER(OperatorDesc), C.c_int, C.POINTER(Options), C.c_void_p,
                                   C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]
        L.kiops_apply.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), _dp, C.c_int, C.POINTER(C.c_void_p),
                                  C.POINTER(Stats)]
        L.kiops_apply_host.argtypes = L.kiops_apply.argtypes
        L.kiops_apply_hostloop.argtypes = L.kiops_apply.argtypes
        L.kiops_get_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_int64)]
        L.kiops_set_forced_schedule.argtypes = [C.c_void_p, _dp, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                                C.c_int]
        L.kiops_debug_basis.argtypes = [C.c_void_p, _dp, _dp, C.POINTER(C.c_int32)]
        L.kiops_set_m_init.argtypes = [C.c_void_p, C.c_int]
        L.kiops_refresh_operator.argtypes = [C.c_void_p]
        L.kiops_debug_expm.argtypes = [C.c_void_p, C.c_int, _dp, C.c_double, _dp, C.POINTER(C.c_int32)]
        L.kiops_epirk_workspace_bytes.argtypes = [C.POINTER(RDProblem), C.c_int, C.POINTER(Options),
                                                  C.POINTER(C.c_size_t)]
        L.kiops_epirk_create.argtypes = [C.POINTER(RDProblem), C.c_int, C.c_double, C.POINTER(Options), C.c_void_p,
                                         C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]
        L.kiops_epirk_step.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(EpirkStats)]
        L.kiops_epirk_record_history.argtypes = [C.c_void_p, C.c_int]
        L.kiops_epirk_history.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
        L.kiops_epirk_set_forced_schedule.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.POINTER(C.c_int32),
                                                      C.POINTER(C.c_int32), C.c_int]
        L.kiops_epirk_destroy.argtypes = [C.c_void_p]
        L.kiops_epirk_last_error.argtypes = [C.c_void_p]
        L.kiops_epirk_last_error.restype = C.c_char_p
        L.kiops_destroy.argtypes = [C.c_void_p]
        L.kiops_status_string.argtypes = [C.c_int]
        L.kiops_status_string.restype = C.c_char_p
        L.kiops_last_error.argtypes = [C.c_void_p]
        L.kiops_last_error.restype = C.c_char_p
        for name in ("kiops_workspace_bytes", "kiops_create", "kiops_apply", "kiops_apply_host", "kiops_apply_hostloop",
                     "kiops_get_trace", "kiops_set_m_init", "kiops_refresh_operator", "kiops_debug_expm",
                     "kiops_set_forced_schedule",
                     "kiops_debug_basis",
                     "kiops_destroy", "kiops_epirk_workspace_bytes", "kiops_epirk_create", "kiops_epirk_step",
                     "kiops_epirk_record_history", "kiops_epirk_history", "kiops_epirk_set_forced_schedule",
                     "kiops_epirk_destroy"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


class KiopsError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = STATUS.get(status, status)


def default_options(**kw) -> Options:
    o = Options()
    lib().kiops_options_default(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def _ptr(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def operator_desc(op: dict, dev_arrays: dict) -> OperatorDesc:
    """op: workload dict (kind, nx, ny, nz, w, inv_h2, ...); dev_arrays: torch CUDA
    tensors for 'diag', 'kappa', 'row_ptr', 'col_idx', 'vals' (those that apply)."""
    d = OperatorDesc()
    d.kind = KIND[op["kind"]]
    d.periodic = 1
    d.nx, d.ny, d.nz = int(op.get("nx", 1)), int(op.get("ny", 1)), int(op.get("nz", 1))
    w = list(op.get("w", [])) + [0.0] * (5 - len(op.get("w", [])))
    for i in range(5):
        d.w[i] = float(w[i])
    d.inv_h2 = float(op.get("inv_h2", 0.0))
    d.diag = _ptr(dev_arrays.get("diag"))
    d.kappa = _ptr(dev_arrays.get("kappa"))
    d.row_ptr = _ptr(dev_arrays.get("row_ptr"))
    d.col_idx = _ptr(dev_arrays.get("col_idx"))
    d.vals = _ptr(dev_arrays.get("vals"))
    d.nnz = int(dev_arrays["vals"].numel()) if dev_arrays.get("vals") is not None else 0
    return d


class Kiops:
    """One kiops_ctx: operator + p + options, a torch-allocated device workspace and
    the instantiated CUDA graph."""

    def __init__(self, op: dict, p: int, device="cuda:0", stream=None, **options):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("KIOPS B200 path needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.device = torch.device(device)
        self.p = int(p)
        self.op = op
        self.N = int(op.get("nx", 1)) * int(op.get("ny", 1)) * int(op.get("nz", 1))
        self.dev = {}
        for name, dt in (("diag", torch.float64), ("kappa", torch.float64), ("vals", torch.float64),
                         ("row_ptr", torch.int64), ("col_idx", torch.int32)):
            a = op.get(name)
            if a is not None:
                self.dev[name] = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(a), dtype=dt)
                self.dev[name] = self.dev[name].to(self.device, dtype=dt).contiguous()
        self.desc = operator_desc(op, self.dev)
        self.opts = default_options(**options)
        nb = C.c_size_t(0)
        s = lib().kiops_workspace_bytes(C.byref(self.desc), self.p, C.byref(self.opts), C.byref(nb))
        if s != 0:
            raise KiopsError(s, "kiops_workspace_bytes")
        self.ws_bytes = nb.value
        self.workspace = torch.empty(self.ws_bytes + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        aligned = (base + 255) & ~255
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        ctx = C.c_void_p()
        s = lib().kiops_create(C.byref(self.desc), self.p, C.byref(self.opts), C.c_void_p(self.stream.cuda_stream),
                               C.c_void_p(aligned), C.c_size_t(self.ws_bytes), C.byref(ctx))
        if s != 0:
            raise KiopsError(s, "kiops_create")
        self.ctx = ctx
        self.last_stats = None

    def debug_expm(self, M, scale=1.0):
        """TEST HOOK: exp(scale * M) by the controller's projected exponential; M: (n, n) numpy."""
        M = np.asfortranarray(M, dtype=np.float64)
        n = M.shape[0]
        mf = M.ravel(order="F").copy()
        f = np.zeros(n * n)
        nm = C.c_int32(0)
        s = lib().kiops_debug_expm(self.ctx, n, mf.ctypes.data_as(_dp), float(scale), f.ctypes.data_as(_dp), C.byref(nm))
        if s != 0:
            raise KiopsError(s, "kiops_debug_expm")
        return f.reshape((n, n), order="F"), nm.value

    def refresh_operator(self):
        """After rewriting the operator's device value arrays in place (diag, kappa, CSR
        vals): rebuilds the SELL-32 copy of a CSR operator (no-op for the stencil kinds)."""
        s = lib().kiops_refresh_operator(self.ctx)
        if s != 0:
            raise KiopsError(s, "kiops_refresh_operator")

    def close(self):
        if getattr(self, "ctx", None):
            lib().kiops_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _err(self, s, what):
        msg = lib().kiops_last_error(self.ctx)
        raise KiopsError(s, f"{what}: {msg.decode() if msg else ''}")

    def set_forced_schedule(self, sched):
        """sched: list of (tau, m) (all accepted) or (tau, m, accept) (trace replay)."""
        n = len(sched)
        tau = (C.c_double * max(1, n))(*[float(e[0]) for e in sched])
        m = (C.c_int32 * max(1, n))(*[int(e[1]) for e in sched])
        acc = (C.c_int32 * max(1, n))(*[int(e[2]) if len(e) > 2 else 1 for e in sched])
        s = lib().kiops_set_forced_schedule(self.ctx, tau, m, acc, n)
        if s != 0:
            self._err(s, "kiops_set_forced_schedule")

    def apply(self, u, T, w=None, check=True, hostloop=False):
        """u: p+1 CUDA float64 tensors (N,), T: output times, w: optional outputs.
        hostloop: profiling hook (kiops_apply_hostloop).  Returns (outputs, stats)."""
        torch = self.torch
        T = [float(t) for t in T]
        if w is None:
            w = [torch.empty(self.N, dtype=torch.float64, device=self.device) for _ in T]
        if len(u) != self.p + 1:
            raise ValueError(f"need p + 1 = {self.p + 1} input vectors u_0..u_p, got {len(u)}")
        dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        for name, xs in (("u", u), ("w", w)):
            for i, x in enumerate(xs):
                if not isinstance(x, torch.Tensor) or x.dtype != torch.float64 or not x.is_contiguous() \
                        or x.device.type != "cuda" or x.device.index != dev_index or x.numel() != self.N:
                    raise ValueError(f"{name}[{i}] must be a contiguous float64 tensor of {self.N} elements on "
                                     f"{self.device}")
        uarr = (C.c_void_p * (self.p + 1))(*[x.data_ptr() for x in u])
        warr = (C.c_void_p * len(T))(*[x.data_ptr() for x in w])
        Tarr = (C.c_double * len(T))(*T)
        st = Stats()
        fn = lib().kiops_apply_hostloop if hostloop else lib().kiops_apply
        s = fn(self.ctx, uarr, Tarr, len(T), warr, C.byref(st))
        self.last_stats = {k: getattr(st, k) for k, _ in Stats._fields_}
        if s != 0 and check:
            self._err(s, "kiops_apply")
        return w, self.last_stats

    def apply_host(self, u, T, w=None):
        """u: p+1 host float64 arrays (numpy, ideally pinned), w: host outputs."""
        T = [float(t) for t in T]
        if w is None:
            w = [np.empty(self.N) for _ in T]
        keep = [np.ascontiguousarray(x, dtype=np.float64) if isinstance(x, np.ndarray) else x for x in u]
        uarr = (C.c_void_p * (self.p + 1))(*[_host_ptr(x) for x in keep])
        warr = (C.c_void_p * len(T))(*[_host_ptr(x) for x in w])
        Tarr = (C.c_double * len(T))(*T)
        st = Stats()
        s = lib().kiops_apply_host(self.ctx, uarr, Tarr, len(T), warr, C.byref(st))
        self.last_stats = {k: getattr(st, k) for k, _ in Stats._fields_}
        if s != 0:
            self._err(s, "kiops_apply_host")
        return w, self.last_stats

    def trace(self):
        rows = C.c_int64(0)
        buf = (TraceRow * TRACE_CAP)()
        s = lib().kiops_get_trace(self.ctx, buf, C.sizeof(buf), C.byref(rows))
        if s != 0:
            self._err(s, "kiops_get_trace")
        n = min(rows.value, TRACE_CAP)
        return [{k: getattr(buf[i], k) for k, _ in TraceRow._fields_} for i in range(n)]

    def debug_basis(self):
        ld = MAX_M + 2
        h = np.zeros(ld * ld)
        sig = np.zeros(ld)
        npass = C.c_int32(0)
        s = lib().kiops_debug_basis(self.ctx, h.ctypes.data_as(_dp), sig.ctypes.data_as(_dp), C.byref(npass))
        if s != 0:
            self._err(s, "kiops_debug_basis")
        return h.reshape((ld, ld), order="F"), sig, npass.value


def _host_ptr(x):
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()  # pinned torch CPU tensor


class KiopsEpirk:
    """EPIRK4s3 / EPIRK4s3A (Eqs. 50-51) for u' = L u + R(u) on a periodic grid through
    the kiops_epirk_* C ABI: problem {"nx", "ny", "w": 5 stencil weights {W,E,S,N,C},
    "c": 4 cubic reaction coefficients}, constant step h, KIOPS options.  A general
    linear part (e.g. Neumann boundaries, advection) is given instead of "w" as
    "L": {"row_ptr", "col_idx", "vals"} (CSR, numpy or torch; copied to the device)."""

    def __init__(self, problem: dict, scheme: str, h: float, device="cuda:0", stream=None, **options):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("KIOPS B200 path needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.device = torch.device(device)
        self.scheme = scheme
        self.N = int(problem["nx"]) * int(problem["ny"])
        pb = RDProblem()
        pb.nx, pb.ny = int(problem["nx"]), int(problem["ny"])
        for i in range(5):
            pb.w[i] = float(problem["w"][i]) if "w" in problem else 0.0
        for i in range(4):
            pb.c[i] = float(problem["c"][i])
        self._L = None
        if problem.get("L") is not None:
            Lm = problem["L"]
            rp = torch.as_tensor(Lm["row_ptr"]).to(device=self.device, dtype=torch.int64).contiguous()
            ci = torch.as_tensor(Lm["col_idx"]).to(device=self.device, dtype=torch.int32).contiguous()
            lv = torch.as_tensor(Lm["vals"]).to(device=self.device, dtype=torch.float64).contiguous()
            if rp.numel() != self.N + 1 or ci.numel() != lv.numel():
                raise ValueError("L: row_ptr needs N + 1 entries, col_idx and vals nnz each")
            self._L = (rp, ci, lv)  # borrowed by the ctx for its life
            pb.L_row_ptr, pb.L_col_idx, pb.L_vals = rp.data_ptr(), ci.data_ptr(), lv.data_ptr()
            pb.L_nnz = int(lv.numel())
        self.pb = pb
        self.opts = default_options(**options)
        nb = C.c_size_t(0)
        s = lib().kiops_epirk_workspace_bytes(C.byref(pb), EPIRK_SCHEMES[scheme], C.byref(self.opts), C.byref(nb))
        if s != 0:
            raise KiopsError(s, "kiops_epirk_workspace_bytes")
        self.workspace = torch.empty(nb.value + 256, dtype=torch.uint8, device=self.device)
        aligned = (self.workspace.data_ptr() + 255) & ~255
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        ctx = C.c_void_p()
        s = lib().kiops_epirk_create(C.byref(pb), EPIRK_SCHEMES[scheme], float(h), C.byref(self.opts),
                                     C.c_void_p(self.stream.cuda_stream), C.c_void_p(aligned), C.c_size_t(nb.value),
                                     C.byref(ctx))
        if s != 0:
            raise KiopsError(s, "kiops_epirk_create")
        self.ctx = ctx

    def step(self, u, nsteps=1):
        """u: CUDA float64 tensor (N,), advanced in place by nsteps constant steps."""
        st = EpirkStats()
        s = lib().kiops_epirk_step(self.ctx, C.c_void_p(u.data_ptr()), int(nsteps), C.byref(st))
        if s != 0:
            msg = lib().kiops_epirk_last_error(self.ctx)
            raise KiopsError(s, f"kiops_epirk_step: {msg.decode() if msg else ''}")
        out = {k: getattr(st, k) for k, _ in EpirkStats._fields_ if k != "final_m"}
        out["final_m"] = tuple(st.final_m[i] for i in range(3 if self.scheme in ("epirk5p1", "exprb5s3") else 2))
        return out

    def record_history(self, on=True):
        s = lib().kiops_epirk_record_history(self.ctx, 1 if on else 0)
        if s != 0:
            raise KiopsError(s, "kiops_epirk_record_history")

    def set_forced_schedules(self, calls):
        """Test hook (trace replay): calls = iterable of (step, call, [(tau, m, accept), ...])
        for the next step(); an empty iterable clears every schedule."""
        lib().kiops_epirk_set_forced_schedule(self.ctx, -1, 0, None, None, None, 0)
        for step, call, sched in calls:
            n = len(sched)
            tau = (C.c_double * n)(*[float(e[0]) for e in sched])
            m = (C.c_int32 * n)(*[int(e[1]) for e in sched])
            acc = (C.c_int32 * n)(*[int(e[2]) for e in sched])
            s = lib().kiops_epirk_set_forced_schedule(self.ctx, int(step), int(call), tau, m, acc, n)
            if s != 0:
                raise KiopsError(s, "kiops_epirk_set_forced_schedule")

    def history(self):
        """Per-call records of the last step() (record_history(True) first): dicts with
        step, call, final_m, krylov_vectors, substeps, rejections, attempts [(j, accept)]."""
        rows = C.c_int64(0)
        lib().kiops_epirk_history(self.ctx, None, 0, C.byref(rows))
        buf = (EpirkCallRecord * max(1, rows.value))()
        s = lib().kiops_epirk_history(self.ctx, buf, rows.value, C.byref(rows))
        if s != 0:
            raise KiopsError(s, "kiops_epirk_history")
        out = []
        for r in buf[:rows.value]:
            n = min(r.n_attempts, EPIRK_HIST_ATTEMPTS)
            out.append({"step": r.step, "call": r.call, "final_m": r.final_m, "krylov_vectors": r.krylov_vectors,
                        "substeps": r.substeps, "rejections": r.rejections, "n_attempts": r.n_attempts,
                        "attempts": [(r.j[a], r.accept[a]) for a in range(n)],
                        "m_new": [r.m_new[a] for a in range(n)], "omega": [r.omega[a] for a in range(n)]})
        return out

    def close(self):
        if getattr(self, "ctx", None):
            lib().kiops_epirk_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
