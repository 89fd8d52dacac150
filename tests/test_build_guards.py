"""Performance guards on the built sm_100a library (CPU only: reads cuobjdump -res-usage).

The persistent 3D pass runs 640 threads per CTA at the 96-register cap, and its speed
moved with the spill stack that unrelated code in the same kernel produced: 64-72
bytes measured 177-180 ms of passes per config-4 call, 104-136 bytes 189-257 ms
(profiles/r01_kernel_evolution.md, session 3).  The SELL SpMV's schedule likewise
depended on code inlined into it (62 registers: 313 us per launch at config 5, 48: 447 us).
These guards catch such a change at build time instead of at the next GPU benchmark.
"""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1804_05126_b200", "libkiops_b200.so")
CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"


def _res_usage():
    if not os.path.exists(LIB) or not os.path.exists(CUOBJDUMP):
        pytest.skip("library not built or cuobjdump missing")
    out = subprocess.run([CUOBJDUMP, "-res-usage", LIB], capture_output=True, text=True).stdout
    res, fn = {}, None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+)", line)
        if m and fn:
            res[fn] = tuple(int(x) for x in m.groups())
    return res


def _find(res, pattern):
    hits = {k: v for k, v in res.items() if re.search(pattern, k)}
    assert hits, f"no kernel matches {pattern}"
    return hits


def test_persistent_3d_pass_spill_stack_small():
    # k_inner_3d_lazyq<PM = 1..4, 7, 2, DD, NH = 2>: the product kernels of config 4 and its p variants
    for fn, (reg, stack, _) in _find(_res_usage(), r"k_inner_3d_lazyqILi\dELi7ELi2ELi\dELi2E").items():
        assert reg <= 96, (fn, reg)
        assert stack <= 96, f"{fn}: {stack} bytes of stack (config-4 passes slowed by 7-45% at 104-136)"


def test_p2_persistent_3d_pass_stack_in_measured_fast_range():
    (fn, (reg, stack, _)), = _find(_res_usage(), r"k_inner_3d_lazyqILi2ELi7ELi2ELi2ELi2E").items()
    assert stack <= 72, f"{fn}: stack {stack} bytes (measured fast: 56-72)"


def test_sell_spmv_keeps_its_register_schedule():
    (fn, (reg, stack, _)), = _find(_res_usage(), r"k_sell_spmv").items()
    assert reg >= 56, f"{fn}: {reg} registers (the 48-register schedule ran 40% slower at config 5)"


def test_ring_kernels_static_shared_is_128_aligned():
    # the cp.async ring base is extern __align__(128) + a fixed residue: the static part is
    # padded to a multiple of 128 bytes by that alignment
    for fn, (_, _, shared) in _find(_res_usage(), r"k_inner_(2d|3d)_lazy").items():
        assert shared % 128 == 0, (fn, shared)


def test_recompute_3d_pass_no_spills_and_tma():
    # k_inner_3d_rc<PM> (config 4's pass since round 2): 10 warps per CTA, 168-register cap
    # (3 warps on two of the four schedulers); no spill stack, and its loads are TMA
    # tensor-map loads (UTMALDG) with mbarrier completion, no cp.async (LDGSTS)
    for fn, (reg, stack, _) in _find(_res_usage(), r"k_inner_3d_rcILi\dE").items():
        assert reg <= 168, (fn, reg)
        # PM = 2 is config 4's kernel: no stack at all.  The F-form stencil (5477fcc) leaves
        # PM = 3 (p = 3, not a bench config) with one 8-byte spill slot at the register cap.
        assert stack == 0 if "ILi2E" in fn else stack <= 16, (fn, stack)
    out = subprocess.run([CUOBJDUMP, "-sass", "-fun", "_Z13k_inner_3d_rcILi2EEv7KParams", LIB], capture_output=True,
                         text=True).stdout
    assert "UTMALDG" in out and "SYNCS" in out and "LDGSTS" not in out
