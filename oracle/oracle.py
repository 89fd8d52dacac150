"""ctypes binding of the plain-C KIOPS oracle (oracle/kiops_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs import this module.  The product package
(paper_1804_05126_b200/) never imports it.

Operators are plain dicts (the same dicts workloads/configs.py produces):
  {"kind": "stencil1d3"|"stencil2d5"|"stencil3d7"|"csr"|"dense",
   "nx", "ny", "nz", "w": [...], "diag": ndarray|None, "kappa": ndarray|None,
   "inv_h2": float, "row_ptr", "col_idx", "vals", "dense": ndarray (N x N)}
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "kiops_oracle.c")
LIB = os.path.join(HERE, "libkiops_oracle.so")
if os.environ.get("KIOPS_ORACLE_LIB"):  # mutation checks (scripts/oracle_mutations.py) load a scratch build
    LIB = os.environ["KIOPS_ORACLE_LIB"]

KIND = {"stencil1d3": 1, "stencil2d5": 2, "stencil3d7": 3, "csr": 4, "dense": 5}
STATUS = {0: "OK", 1: "INVALID_ARG", 4: "NO_CONVERGENCE", 5: "NONFINITE", 6: "ALLOC"}

_dp = C.POINTER(C.c_double)


class _Op(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
        ("w", C.c_double * 5), ("diag", _dp), ("kappa", _dp), ("inv_h2", C.c_double),
        ("row_ptr", C.POINTER(C.c_int64)), ("col_idx", C.POINTER(C.c_int32)),
        ("vals", _dp), ("dense", _dp),
    ]


class _Opts(C.Structure):
    _fields_ = [
        ("tol", C.c_double), ("m_init", C.c_int), ("m_min", C.c_int), ("m_max", C.c_int),
        ("iop_q", C.c_int), ("task1", C.c_int), ("max_attempts", C.c_int64),
        ("n_forced", C.c_int), ("forced_tau", _dp), ("forced_m", C.POINTER(C.c_int)),
        ("forced_accept", C.POINTER(C.c_int)), ("corrected", C.c_int),
    ]


class _Stats(C.Structure):
    _fields_ = [
        ("substeps", C.c_int64), ("rejections", C.c_int64), ("krylov_vectors", C.c_int64),
        ("expm_calls", C.c_int64), ("final_m", C.c_int), ("happy_breakdowns", C.c_int),
        ("t_reached", C.c_double), ("nu", C.c_double), ("mu", C.c_double),
    ]


class _Trace(C.Structure):
    _fields_ = [
        ("attempt", C.c_int64), ("j", C.c_int), ("happy", C.c_int), ("accept", C.c_int),
        ("m_new", C.c_int), ("t_now", C.c_double), ("tau", C.c_double), ("beta", C.c_double),
        ("h_next", C.c_double), ("eps", C.c_double), ("omega", C.c_double),
        ("tau_new", C.c_double),
    ]


def build(force: bool = False) -> str:
    """Compile the oracle with plain IEEE flags (no fast-math, no contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
               "-fno-fast-math", "-o", LIB + ".tmp", SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.or_expm.argtypes = [C.c_int, _dp, C.c_double, _dp, C.POINTER(C.c_int)]
        L.or_apply.argtypes = [C.POINTER(_Op), _dp, _dp]
        L.or_normalisation.argtypes = [C.c_int64, C.c_int, C.POINTER(_dp), _dp, _dp]
        L.or_augmented_matvec.argtypes = [C.POINTER(_Op), C.c_int64, C.c_int, C.POINTER(_dp),
                                          C.c_double, _dp, _dp]
        L.or_iop.argtypes = [C.POINTER(_Op), C.c_int64, C.c_int, C.POINTER(_dp), C.c_double, _dp,
                             C.c_int, C.c_int, _dp, _dp, C.POINTER(C.c_int)]
        L.or_adapt.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                               C.c_double, C.c_double, C.c_double, C.c_int, C.c_double,
                               C.c_double, C.c_int, _dp]
        L.or_kiops.argtypes = [C.POINTER(_Op), C.c_int, C.POINTER(_dp), C.c_int, _dp,
                               C.POINTER(_dp), C.POINTER(_Opts), C.POINTER(_Stats),
                               C.POINTER(_Trace), C.c_int64, C.POINTER(C.c_int64)]
        L.or_project.argtypes = [C.c_int64, C.c_int64, C.c_int, _dp, _dp, C.c_double, _dp]
        L.or_dense_phi_combination.argtypes = [C.POINTER(_Op), C.c_int, C.POINTER(_dp),
                                               C.c_double, _dp]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


class Operator:
    """Keeps the numpy arrays alive while the C struct points at them."""

    def __init__(self, d: dict):
        self.d = d
        s = _Op()
        s.kind = KIND[d["kind"]]
        self.nx, self.ny, self.nz = int(d.get("nx", 1)), int(d.get("ny", 1)), int(d.get("nz", 1))
        s.nx, s.ny, s.nz = self.nx, self.ny, self.nz
        w = list(d.get("w", [])) + [0.0] * (5 - len(d.get("w", [])))
        for i in range(5):
            s.w[i] = float(w[i])
        self._keep = []
        for name in ("diag", "kappa", "vals", "dense"):
            a = _f64(d.get(name))
            if name == "dense" and a is not None:
                a = np.asfortranarray(a).ravel(order="F").copy()
            self._keep.append(a)
            setattr(s, name, _ptr(a))
        s.inv_h2 = float(d.get("inv_h2", 0.0))
        if d["kind"] == "csr":
            rp = np.ascontiguousarray(d["row_ptr"], dtype=np.int64)
            ci = np.ascontiguousarray(d["col_idx"], dtype=np.int32)
            self._keep += [rp, ci]
            s.row_ptr = rp.ctypes.data_as(C.POINTER(C.c_int64))
            s.col_idx = ci.ctypes.data_as(C.POINTER(C.c_int32))
        self.s = s
        self.N = self.nx * self.ny * self.nz

    @property
    def ref(self):
        return C.byref(self.s)


def _as_op(op):
    return op if isinstance(op, Operator) else Operator(op)


def _vec_array(vs):
    vs = [_f64(v) for v in vs]
    arr = (_dp * max(1, len(vs)))(*[_ptr(v) for v in vs])
    return vs, arr


def expm(M, scale=1.0):
    """F = exp(scale*M) by the oracle's Pade-13 scaling and squaring."""
    M = np.asfortranarray(M, dtype=np.float64)
    n = M.shape[0]
    Mf = M.ravel(order="F").copy()
    F = np.zeros(n * n)
    nm = C.c_int(0)
    rc = lib().or_expm(n, _ptr(Mf), float(scale), _ptr(F), C.byref(nm))
    if rc != 0:
        raise FloatingPointError(f"or_expm rc={rc}")
    return F.reshape((n, n), order="F"), nm.value


def apply(op, x):
    op = _as_op(op)
    x = _f64(x)
    y = np.empty(op.N)
    lib().or_apply(op.ref, _ptr(x), _ptr(y))
    return y


def normalisation(u):
    u, arr = _vec_array(u)
    nu, mu = C.c_double(), C.c_double()
    lib().or_normalisation(len(u[0]), len(u) - 1, arr, C.byref(nu), C.byref(mu))
    return nu.value, mu.value


def augmented_matvec(op, u, nu, v):
    op = _as_op(op)
    u, arr = _vec_array(u)
    v = _f64(v)
    y = np.empty(op.N + len(u) - 1)
    lib().or_augmented_matvec(op.ref, op.N, len(u) - 1, arr, float(nu), _ptr(v), _ptr(y))
    return y


def iop(op, u, nu, v0, m, q=2):
    """Alg. 2 from v0: returns V ((N+p) x (m+1)), H ((m+1) x m), j, happy."""
    op = _as_op(op)
    u, arr = _vec_array(u)
    p = len(u) - 1
    v0 = _f64(v0)
    V = np.zeros((m + 1) * (op.N + p))
    H = np.zeros((m + 1) * m)
    happy = C.c_int(0)
    j = lib().or_iop(op.ref, op.N, p, arr, float(nu), _ptr(v0), int(m), int(q), _ptr(V), _ptr(H),
                     C.byref(happy))
    return V.reshape((op.N + p, m + 1), order="F"), H.reshape((m + 1, m), order="F"), j, happy.value


def project(V, ld, rows, f, beta=1.0):
    """w = beta V(0:rows, 0:j) f on a column-major V (flat, leading dimension ld)."""
    f = _f64(f)
    w = np.empty(rows)
    lib().or_project(int(rows), int(ld), len(f), _ptr(V), _ptr(f), float(beta), _ptr(w))
    return w


def adapt(happy, accept, j, m, m_min, m_max, tau, omega, t_now, t_end, hist_valid=0,
          omega_old=0.0, tau_old=0.0, j_old=0):
    tn = C.c_double()
    mn = lib().or_adapt(int(happy), int(accept), int(j), int(m), int(m_min), int(m_max),
                        float(tau), float(omega), float(t_now), float(t_end), int(hist_valid),
                        float(omega_old), float(tau_old), int(j_old), C.byref(tn))
    return tn.value, mn


def dense_phi_combination(op, u, tau):
    op = _as_op(op)
    u, arr = _vec_array(u)
    out = np.empty(op.N + len(u) - 1)
    rc = lib().or_dense_phi_combination(op.ref, len(u) - 1, arr, float(tau), _ptr(out))
    if rc != 0:
        raise FloatingPointError(f"or_dense_phi_combination rc={rc}")
    return out


def kiops(op, u, T, tol=1e-7, m_init=10, m_min=10, m_max=128, iop_q=2, task1=0,
          max_attempts=10000, forced=None, trace_cap=20000, out=None, corrected=0):
    """Alg. 1: returns (w list, stats dict, trace list of dicts, status string)."""
    op = _as_op(op)
    u, arr = _vec_array(u)
    T = np.ascontiguousarray(T, dtype=np.float64)
    n_out = len(T)
    w = out if out is not None else [np.zeros(op.N) for _ in range(n_out)]
    warr = (_dp * n_out)(*[_ptr(x) for x in w])
    o = _Opts(tol=tol, m_init=m_init, m_min=m_min, m_max=m_max, iop_q=iop_q, task1=task1,
              max_attempts=max_attempts, corrected=int(corrected))
    if forced:
        ft = np.ascontiguousarray([e[0] for e in forced], dtype=np.float64)
        fm = np.ascontiguousarray([e[1] for e in forced], dtype=np.int32)
        fa = np.ascontiguousarray([e[2] if len(e) > 2 else 1 for e in forced], dtype=np.int32)
        o.n_forced, o.forced_tau = len(forced), _ptr(ft)
        o.forced_m = fm.ctypes.data_as(C.POINTER(C.c_int))
        o.forced_accept = fa.ctypes.data_as(C.POINTER(C.c_int))
    st = _Stats()
    tr = (_Trace * trace_cap)()
    tl = C.c_int64(0)
    rc = lib().or_kiops(op.ref, len(u) - 1, arr, n_out, _ptr(T), warr, C.byref(o), C.byref(st),
                        tr, trace_cap, C.byref(tl))
    stats = {k: getattr(st, k) for k, _ in _Stats._fields_}
    trace = [{k: getattr(tr[i], k) for k, _ in _Trace._fields_} for i in range(min(tl.value, trace_cap))]
    return w, stats, trace, STATUS.get(rc, str(rc))
