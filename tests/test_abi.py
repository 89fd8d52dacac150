"""CPU-side checks of the C ABI library (no compute calls without a GPU): it loads,
exports every function include/kiops.h declares, and its host-only entry points
(options, workspace sizing, argument validation, status strings) behave as the
header documents."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__ as g

    g.build_cuda()
    from paper_1804_05126_b200 import kiops

    return kiops.lib()


def header_functions():
    src = open(os.path.join(ROOT, "include", "kiops.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kiops_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = header_functions()
    assert len(names) >= 11
    for n in names:
        assert hasattr(L, n), n


def test_options_default_and_status_strings(L):
    from paper_1804_05126_b200 import kiops as K

    o = K.default_options()
    assert (o.tol, o.m_init, o.m_min, o.m_max, o.iop_q, o.task1, o.max_attempts) == (1e-7, 10, 10, 128, 2, 0, 10000)
    for s, name in K.STATUS.items():
        assert L.kiops_status_string(s).decode() == name


def desc_for(cfg):
    from paper_1804_05126_b200 import kiops as K

    fake = {}
    for nm in ("diag", "kappa", "row_ptr", "col_idx", "vals"):
        if cfg["op"].get(nm) is not None:
            fake[nm] = _Fake(len(cfg["op"][nm]))
    return K.operator_desc(cfg["op"], fake)


class _Fake:
    """stands in for a device tensor when only the pointer value is needed"""

    def __init__(self, n):
        self.n = n

    def data_ptr(self):
        return 4096

    def numel(self):
        return self.n


def test_workspace_bytes_layout(L):
    from paper_1804_05126_b200 import kiops as K
    from workloads import configs as W

    c = W.config4(8, 8, 8)
    d = desc_for(c)
    o = K.default_options(m_max=128)
    nb = C.c_size_t()
    assert L.kiops_workspace_bytes(C.byref(d), 2, C.byref(o), C.byref(nb)) == 0
    small = nb.value
    # full-size config 4 (descriptor only): the basis dominates, (m_max+1) vectors of N doubles
    d.nx = d.ny = d.nz = 256
    assert L.kiops_workspace_bytes(C.byref(d), 2, C.byref(o), C.byref(nb)) == 0
    # padded mode (3D recompute pass): (m_max + 1) basis slots + the p
    # copies of B's columns + the kappa copy, each a ghost-padded 260 x 260 x 256 grid
    # (rounded to 32 doubles), + small state; no r_k buffers
    vec = (260 * 260 * 256 + 31) // 32 * 32 * 8
    assert (129 + 2 + 1) * vec <= nb.value <= (129 + 2 + 1) * vec + 64 * 2 ** 20
    assert small < nb.value


@pytest.mark.parametrize("bad,status", [
    ({"tol": 0.0}, 1), ({"m_min": 0}, 1), ({"m_min": 20, "m_max": 10}, 1), ({"iop_q": 0}, 1),
    ({"iop_q": 129}, 1), ({"m_max": 200}, 2), ({"max_attempts": 0}, 1)])
def test_validation_before_any_launch(L, bad, status):
    from paper_1804_05126_b200 import kiops as K
    from workloads import configs as W

    c = W.config1(16)
    d = desc_for(c)
    o = K.default_options(**bad)
    nb = C.c_size_t()
    assert L.kiops_workspace_bytes(C.byref(d), 3, C.byref(o), C.byref(nb)) == status
    ctx = C.c_void_p()
    assert L.kiops_create(C.byref(d), 3, C.byref(o), None, None, 0, C.byref(ctx)) == status
    assert not ctx.value


def test_bad_operator_and_workspace(L):
    from paper_1804_05126_b200 import kiops as K
    from workloads import configs as W

    c = W.config2(8, 8)
    d = desc_for(c)
    o = K.default_options()
    nb = C.c_size_t()
    d.nz = 2  # 2D stencil with nz != 1
    assert L.kiops_workspace_bytes(C.byref(d), 1, C.byref(o), C.byref(nb)) == 1
    d.nz = 1
    d.periodic = 0
    assert L.kiops_workspace_bytes(C.byref(d), 1, C.byref(o), C.byref(nb)) == 2
    d.periodic = 1
    assert L.kiops_workspace_bytes(C.byref(d), 9, C.byref(o), C.byref(nb)) == 1  # p > KIOPS_MAX_P
    ctx = C.c_void_p()
    # NULL / misaligned / short workspace are rejected before touching the device
    assert L.kiops_create(C.byref(d), 1, C.byref(o), None, None, 0, C.byref(ctx)) == 6
    assert L.kiops_create(C.byref(d), 1, C.byref(o), None, C.c_void_p(4096 + 8), 1 << 40, C.byref(ctx)) == 6
    assert L.kiops_create(C.byref(d), 1, C.byref(o), None, C.c_void_p(4096), 16, C.byref(ctx)) == 6


def test_epirk_workspace_and_validation(L):
    # host-only checks of the EPIRK entry points: sizes grow with the number of
    # KIOPS call shapes per scheme; invalid scheme / h / workspace are rejected before any launch
    from paper_1804_05126_b200 import kiops as K

    pb = K.RDProblem()
    pb.nx, pb.ny = 64, 48
    for i, w in enumerate([1.0, 1.0, 1.0, 1.0, -4.0]):
        pb.w[i] = w
    for i, c in enumerate([0.0, 1.0, 0.0, -1.0]):
        pb.c[i] = c
    o = K.default_options(m_max=64)
    sizes = {}
    for name, sch in K.EPIRK_SCHEMES.items():
        nb = C.c_size_t()
        assert L.kiops_epirk_workspace_bytes(C.byref(pb), sch, C.byref(o), C.byref(nb)) == 0
        sizes[name] = nb.value
    # two call shapes (p = 1, 4) for the fourth-order schemes and EPIRK5P1 (p = 1, 3); three for EXPRB5s3
    assert sizes["epirk4s3"] == sizes["epirk4s3a"]
    assert sizes["exprb5s3"] > sizes["epirk4s3"] and sizes["exprb5s3"] > sizes["epirk5p1"]
    nb = C.c_size_t()
    assert L.kiops_epirk_workspace_bytes(C.byref(pb), 9, C.byref(o), C.byref(nb)) == 1
    ctx = C.c_void_p()
    assert L.kiops_epirk_create(C.byref(pb), 1, C.c_double(-0.1), C.byref(o), None, C.c_void_p(4096),
                                C.c_size_t(1 << 40), C.byref(ctx)) == 1  # h <= 0
    assert L.kiops_epirk_create(C.byref(pb), 1, C.c_double(0.1), C.byref(o), None, None, C.c_size_t(0),
                                C.byref(ctx)) == 6  # no workspace
    assert not ctx.value
    bad = K.default_options(iop_q=0)
    assert L.kiops_epirk_workspace_bytes(C.byref(pb), 1, C.byref(bad), C.byref(nb)) == 1
