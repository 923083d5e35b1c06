"""Pins for the coefficient-fitter oracle (oracle/fit.py)
against things other than itself:

* closed forms of both objectives at k = 1, c = 0 (tests/golden/fit_closed_forms.json,
  derived by hand) -- pin h, h', the ReLU combination and
  the quadrature wiring;
* reductions: k = 2 with a = (0, 0) or (1, 0) is the k = 1 objective at c3 / c1
  (a dropped or mis-indexed last weight 1 - sum(a) fails it);
* mirror symmetry: h - ReLU is even for GELU and SiLU, so for any theta that
  satisfies Eq. 14's constraint J(w, c) = J(w, -c) on the symmetric [A, B]
  (a sign error in h or in the combination breaks it);
* near-optimality of the published constants: a local search started at the
  paper's (a*, c*) (App. I P:L1346-1347 for the
  derivative objective) lowers J by < 0.05 % and moves no parameter by more
  than 0.05 -- a wrong objective moves its minimiser far from the paper's;
* the paper's tail bounds: each side's closed-form
  bound at the oracle's B is eps/2 and the mpmath tails lie below it;
* J at the paper's constants by 40-digit mpmath quadrature.
"""
import json
import math
import os

import mpmath
import numpy as np
import pytest
from scipy import optimize

import oracle
from oracle import fit

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "paper_constants.json")) as f:
    PAPER = json.load(f)

CLOSED = {  # evaluated here from the expressions in golden/fit_closed_forms.json
    ("gelu", fit.OBJ_H): 4.0 / (3.0 * math.sqrt(math.pi)) * (1.0 / math.sqrt(2.0) - 5.0 / 8.0),
    ("silu", fit.OBJ_H): 3.0 * float(mpmath.zeta(3)) - math.pi ** 2 / 3.0,
    ("gelu", fit.OBJ_DH): 1.0 / (4.0 * math.sqrt(math.pi)),
    ("silu", fit.OBJ_DH): (math.pi ** 2 - 6.0) / 18.0,
}


def paper_theta(key):
    return np.array([float(v) for v in PAPER[key]["a"] + PAPER[key]["c"]])


def test_closed_forms_file_matches_expressions():
    with open(os.path.join(GOLD, "fit_closed_forms.json")) as f:
        g = json.load(f)
    for (kind, obj), v in CLOSED.items():
        key = f"{kind}_{'h' if obj == fit.OBJ_H else 'dh'}"
        assert abs(float(g[key]["value"]) - v) < 1e-15


@pytest.mark.parametrize("kind", ["gelu", "silu"])
@pytest.mark.parametrize("obj", [fit.OBJ_H, fit.OBJ_DH])
def test_k1_relu_closed_form(kind, obj):
    J = fit.objective(kind, 1, [0.0], obj)
    assert abs(J - CLOSED[(kind, obj)]) < 1e-8 + 1e-10 * J   # truncation < eps (paper's bound)


@pytest.mark.parametrize("kind", ["gelu", "silu"])
@pytest.mark.parametrize("obj", [fit.OBJ_H, fit.OBJ_DH])
def test_k2_reduces_to_k1(kind, obj):
    rng = np.random.default_rng(3)
    for _ in range(3):
        c = np.sort(rng.uniform(-2, 2, 3))
        assert fit.objective(kind, 2, [0.0, 0.0, *c], obj) == pytest.approx(fit.objective(kind, 1, [c[2]], obj), rel=1e-9)
        assert fit.objective(kind, 2, [1.0, 0.0, *c], obj) == pytest.approx(fit.objective(kind, 1, [c[0]], obj), rel=1e-9)
        assert fit.objective(kind, 2, [0.0, 1.0, *c], obj) == pytest.approx(fit.objective(kind, 1, [c[1]], obj), rel=1e-9)


@pytest.mark.parametrize("kind", ["gelu", "silu"])
def test_mirror_symmetry_under_constraint(kind):
    rng = np.random.default_rng(7)
    for _ in range(3):
        a1, a2 = rng.uniform(-0.3, 0.8, 2)
        c1, c2 = rng.uniform(-3, 3, 2)
        c3 = -(a1 * c1 + a2 * c2) / (1 - a1 - a2)          # Eq. 14 constraint
        th = np.array([a1, a2, c1, c2, c3])
        assert abs(fit.constraint_residual(2, th)) < 1e-12
        mir = np.array([a1, a2, -c1, -c2, -c3])
        assert fit.objective(kind, 2, th) == pytest.approx(fit.objective(kind, 2, mir), rel=1e-9)
    # without the constraint the mirror image differs (the pin has teeth)
    th = np.array([0.2, 0.5, -1.0, 0.5, 1.5])
    assert abs(fit.objective(kind, 2, th) - fit.objective(kind, 2, -th * np.array([-1, -1, 1, 1, 1]))) > 1e-3


@pytest.mark.parametrize("key,kind,obj", [("gelu", "gelu", fit.OBJ_H), ("silu", "silu", fit.OBJ_H),
                                          ("gelu_d", "gelu", fit.OBJ_DH)])
def test_paper_constants_are_near_optimal(key, kind, obj):
    th0 = paper_theta(key)
    J0 = fit.objective(kind, 2, th0, obj)
    r = optimize.minimize(lambda t: fit.objective(kind, 2, t, obj), th0, method="Nelder-Mead",
                          options=dict(xatol=1e-8, fatol=1e-15, maxfev=1500))
    assert r.fun <= J0 * (1 + 1e-12)
    assert (J0 - r.fun) / J0 < 5e-4
    assert np.max(np.abs(r.x - th0)) < 0.05


def test_near_optimality_pin_has_teeth():
    """The same search under a perturbed objective (SiLU's thresholds fitted
    against GELU) ends far from the paper's SiLU constants."""
    th0 = paper_theta("silu")
    r = optimize.minimize(lambda t: fit.objective("gelu", 2, t), th0, method="Nelder-Mead",
                          options=dict(xatol=1e-6, fatol=1e-12, maxfev=600))
    assert np.max(np.abs(r.x - th0)) > 0.5


@pytest.mark.parametrize("kind", ["gelu", "silu"])
def test_paper_tail_bound(kind):
    """int_{-inf}^A h^2 + int_B^inf (h - x)^2 < eps for the paper's A, B."""
    mpmath.mp.dps = 30
    A, B = fit.tail_bounds(kind)
    if kind == "gelu":
        h = lambda x: x * mpmath.ncdf(x)
    else:
        h = lambda x: x / (1 + mpmath.exp(-x))
    left = mpmath.quad(lambda x: h(x) ** 2, [-mpmath.inf, A])
    right = mpmath.quad(lambda x: (h(x) - x) ** 2, [B, mpmath.inf])
    assert 0 < left + right < fit.EPS_TAIL


@pytest.mark.parametrize("key,kind", [("gelu", "gelu"), ("silu", "silu")])
def test_objective_at_paper_constants_vs_mpmath(key, kind):
    mpmath.mp.dps = 40
    th = paper_theta(key)
    w, c = fit.split(2, th)
    A, B = fit.tail_bounds(kind)
    W = [mpmath.mpf(x) for x in w]
    C = [mpmath.mpf(x) for x in c]
    if kind == "gelu":
        h = lambda x: x * mpmath.ncdf(x)
    else:
        h = lambda x: x / (1 + mpmath.exp(-x))
    f = lambda x: (h(x) - sum(wi * max(x - ci, 0) for wi, ci in zip(W, C))) ** 2
    ref = mpmath.quad(f, [A] + sorted(C) + [B])
    assert fit.objective(kind, 2, th) == pytest.approx(float(ref), rel=1e-10)


def test_step_table_from_theta():
    th = paper_theta("gelu")
    c, s = fit.step_table(2, th)
    c_ref, s_ref, _ = oracle.step_table("gelu")
    assert np.array_equal(c, c_ref)
    assert np.allclose(s, s_ref, rtol=0, atol=1e-15)


def test_bad_theta_rejected():
    with pytest.raises(ValueError):
        fit.objective("gelu", 2, [0.0, 1.0, 0.0])


@pytest.mark.parametrize("kind", ["gelu", "silu"])
@pytest.mark.parametrize("eps", [1e-8, 1e-4])
def test_tail_bounds_meet_the_papers_inequalities(kind, eps):
    """App. E bounds each tail by a closed form -- GELU 1/2 exp(-B^2/2)
    (P:L1030), SiLU exp(-B/2) -- and picks B so that the
    two sides add up to eps: each side's bound at the
    oracle's B is eps/2, and the true tails (mpmath) lie below it."""
    mpmath.mp.dps = 30
    A, B = fit.tail_bounds(kind, eps)
    assert A == -B
    if kind == "gelu":
        side = 0.5 * math.exp(-B * B / 2.0)
        h = lambda x: x * mpmath.ncdf(x)
    else:
        side = math.exp(-B / 2.0)
        h = lambda x: x / (1 + mpmath.exp(-x))
    assert side == pytest.approx(eps / 2.0, rel=1e-12)
    left = mpmath.quad(lambda x: h(x) ** 2, [-mpmath.inf, A])
    right = mpmath.quad(lambda x: (h(x) - x) ** 2, [B, mpmath.inf])
    assert left < side and right < side
