"""Pins of the oracle's Alg. 4 controller (Eqs. 43-46) and of Eq. 39
acceptance: golden examples from the printed formulas plus a 10^4-sample
property suite of the clipping rules."""
import json
import math
import os

import numpy as np

from oracle import oracle as O

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def test_golden_adapt():
    for ex in G["adapt"]:
        h = ex["hist"] or {}
        tn, mn = O.adapt(ex["happy"], ex["accept"], ex["j"], ex["m"], ex["m_min"], ex["m_max"], ex["tau"],
                         ex["omega"], ex["t_now"], ex["t_end"], 1 if h else 0, h.get("omega_old", 0.0),
                         h.get("tau_old", 0.0), h.get("j_old", 0))
        assert mn == ex["m_new"], ex["cite"]
        assert tn == np.float64(ex["tau_new"]) or abs(tn - ex["tau_new"]) <= 4e-15 * ex["tau_new"], ex["cite"]


def test_golden_acceptance_formula():
    # the oracle's omega is Eq. 39 verbatim; checked end to end in test_pins_kiops via the trace
    for ex in G["acceptance"]:
        om = ex["T_end"] * ex["eps"] / (ex["tau"] * ex["tol"])
        assert math.isclose(om, ex["omega"], rel_tol=1e-14) and (om <= 1.4) == ex["accept"]


def test_property_suite_clipping():
    rng = np.random.default_rng(11)
    for _ in range(10000):
        m_min = int(rng.integers(1, 20))
        m_max = int(rng.integers(m_min, 140))
        j = int(rng.integers(m_min, m_max + 1))
        m = j
        tau = 10 ** rng.uniform(-6, 1)
        t_end = tau * 10 ** rng.uniform(0, 3)
        t_now = rng.uniform(0, t_end - tau) if t_end > tau else 0.0
        tau = min(tau, t_end - t_now)
        omega = 10 ** rng.uniform(-20, 15)
        accept = omega <= 1.4
        happy = int(rng.random() < 0.05)
        hist = int(rng.random() < 0.5 and not happy)
        j_old = j if rng.random() < 0.5 else max(1, j - int(rng.integers(1, 8)))
        tau_old = tau if j_old != j else tau * 10 ** rng.uniform(-1, 1)
        tn, mn = O.adapt(happy, 1 if (accept or happy) else 0, j, m, m_min, m_max, tau,
                         0.0 if happy else omega, t_now, t_end, hist, 10 ** rng.uniform(-5, 15),
                         tau_old, j_old)
        rem = t_end - (t_now + tau) if (accept or happy) else t_end - t_now
        assert m_min <= mn <= m_max or (happy and mn == m)
        if happy:
            assert mn == m and tn == min(tau, rem)
        elif j == m_max:
            assert tn <= rem + 0.0
            assert tn >= min(rem, tau / 5) - 1e-300
            if not accept:
                assert mn == j and tn <= tau * (1 + 1e-15) or tn == rem
            else:
                assert tn <= 5 * tau * (1 + 1e-15)
        else:
            assert (3 * j) // 4 <= mn or mn == m_min
            assert mn <= (4 * j + 2) // 3 or mn == m_min
            assert tn == min(tau, rem)
            if not accept:
                assert mn >= j or mn == m_max


def test_golden_eq43_branch_discriminates():
    """The Eq. 43 order estimate (same j, different tau; R4) is reached by the golden
    cases in BOTH gamma branches with an unclipped tau_new, so an inverted Eq. 43, a
    missing ord >= 1 floor or a missing j/4 fallback changes tau_new (hand-evaluated
    values in tests/golden/paper_examples.json)."""
    cases = [ex for ex in G["adapt"] if ex["hist"] and ex["hist"]["j_old"] == ex["j"] and ex["hist"]["tau_old"] != ex["tau"]]
    assert len(cases) >= 5
    branches = set()
    for ex in cases:
        h = ex["hist"]
        tn, mn = O.adapt(ex["happy"], ex["accept"], ex["j"], ex["m"], ex["m_min"], ex["m_max"], ex["tau"], ex["omega"],
                         ex["t_now"], ex["t_end"], 1, h["omega_old"], h["tau_old"], h["j_old"])
        assert mn == ex["m_new"] and abs(tn - ex["tau_new"]) <= 4e-15 * ex["tau_new"], ex["note"]
        # the value is strictly inside the clip interval, i.e. it depends on the exponent
        lo, hi = ex["tau"] / 5, 5 * ex["tau"]
        assert lo < tn < hi, ex["note"]
        branches.add(ex["omega"] > 1.4)
    assert branches == {True, False}


def test_golden_r3_breakdown_threshold():
    """R3 (Alg. 2 l.12 "s ~ 0"): happy breakdown iff s <= max(1e-12 c, 1e-14),
    on nonzero residuals just below / above the relative threshold and the floor."""
    for ex in G["r3_threshold"]:
        a, dl = ex["a"], ex["delta"]
        A = np.diag([a, a * (1.0 + dl)])
        x = np.array([1.0, 1.0])
        V, H, j, happy = O.iop({"kind": "dense", "nx": 2, "dense": A}, [x], 1.0, x, 1, 2)
        assert bool(happy) == ex["happy_at_j1"], ex["note"]
        if not happy:  # the stored subdiagonal is the residual norm s = a delta / 2
            assert abs(H[1, 0] - a * dl / 2) <= 1e-3 * a * dl
