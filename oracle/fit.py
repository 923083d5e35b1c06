"""Oracle for the offline coefficient fitter:
the objective App. E minimises to obtain the ReGELU2 / ReSiLU2 constants,
and the derivative objective App. I minimises for ReGELU2-d.

TEST INFRASTRUCTURE ONLY, like the rest of ``oracle/``: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It shares nothing with the CUDA
fitter (``paper_2406_16282_b200/csrc/fit.cu``): the kernel uses a fixed
composite Gauss-Legendre rule; this oracle uses QUADPACK's adaptive
Gauss-Kronrod (``scipy.integrate.quad``), the library the paper cites for the
integral ("piessens1983quadpack, 2020SciPy-NMeth").

Parameter vector ("theta"), the paper's own five scalars for k = 2
(P:L1062-1063): theta = (a_1 .. a_{m-1}, c_1 .. c_m), m = 2^k - 1 ReLUs,
with the last weight a_m = 1 - sum(a) (Eq. 14).

Steps, in the paper's order (App. E, P:L1009-1065 GELU, P:L1086-1142 SiLU):
1. tail truncation: B = -A = sqrt(-2 ln eps) for GELU,
   B = -A = -2 ln(eps/2) for SiLU, eps = 1e-8;
2. J(a, c) = int_A^B (h(x) - h~_{a,c}(x))^2 dx  (P:L1038-1040 / P:L1130),
   evaluated by adaptive quadrature with the kinks c_i as break points;
3. App. I: the same with h', h~' in place of h, h~ on the
   same [A, B] (reading F2).
The search itself (simulated annealing) is stochastic; what is
unique is the optimum, so the GPU fitter is judged by this objective
(DESIGN.md section "Coefficient fitter").

Pinned in tests/test_fit_oracle.py (closed forms at k = 1, mirror symmetry,
near-optimality of the published constants, mpmath, the tail bound).
"""
from __future__ import annotations

import math

import numpy as np
from scipy import integrate

from . import GELU, SILU, _kind, act, act_deriv

EPS_TAIL = 1e-8          # P:L1049 (GELU), P:L1126 (SiLU)
OBJ_H, OBJ_DH = 0, 1     # Eq. 15 / Eq. 17


def n_relus(k: int) -> int:
    """2^k - 1 ReLUs for k bits (Eq. 14)."""
    return (1 << int(k)) - 1


def n_params(k: int) -> int:
    """m - 1 free weights and m thresholds."""
    return 2 * n_relus(k) - 1


def tail_bounds(kind, eps: float = EPS_TAIL):
    """(A, B) with B = -A (App. E).  GELU: sqrt(-2 ln eps);
    SiLU: -2 ln(eps / 2)."""
    if _kind(kind) == GELU:
        B = math.sqrt(-2.0 * math.log(eps))
    else:
        B = -2.0 * math.log(eps / 2.0)
    return -B, B


def split(k: int, theta):
    """theta -> (w[m], c[m]) with w_m = 1 - sum(a) (Eq. 14)."""
    m = n_relus(k)
    theta = np.asarray(theta, dtype=np.float64)
    if theta.shape != (n_params(k),):
        raise ValueError(f"theta must hold {n_params(k)} values for k={k}")
    a = theta[:m - 1]
    w = np.concatenate([a, [1.0 - a.sum()]])
    return w, theta[m - 1:].copy()


def combo(x: float, w, c) -> float:
    """h~_{a,c}(x) = sum_i w_i max(x - c_i, 0) (Eq. 14)."""
    return float(sum(wi * max(x - ci, 0.0) for wi, ci in zip(w, c)))


def combo_deriv(x: float, w, c) -> float:
    """h~'(x) = sum_i w_i [x > c_i] (strict, R1)."""
    return float(sum(wi for wi, ci in zip(w, c) if x > ci))


def objective(kind, k: int, theta, which: int = OBJ_H, eps: float = EPS_TAIL) -> float:
    """J = int_A^B (h - h~)^2 dx (which = OBJ_H, App. E) or
    int_A^B (h' - h~')^2 dx (which = OBJ_DH, App. I)."""
    w, c = split(k, theta)
    A, B = tail_bounds(kind, eps)
    if which == OBJ_H:
        def f(x):
            return (act(kind, x) - combo(x, w, c)) ** 2
    elif which == OBJ_DH:
        def f(x):
            return (act_deriv(kind, x) - combo_deriv(x, w, c)) ** 2
    else:
        raise ValueError(which)
    pts = sorted(float(ci) for ci in c if A < ci < B)
    val, _ = integrate.quad(f, A, B, points=pts or None, epsabs=1e-14, epsrel=1e-12, limit=1000)
    return float(val)


def constraint_residual(k: int, theta) -> float:
    """sum_i w_i c_i -- Eq. 14's constraint, 0 when it holds."""
    w, c = split(k, theta)
    return float(np.dot(w, c))


def step_table(k: int, theta):
    """(thresholds, levels) of the fitted activation for stepact_fwd/bwd:
    the ReLUs sorted by c; level j = derivative of h~ on segment j =
    sum of the weights of the j lowest thresholds (P:L1017 generalised)."""
    w, c = split(k, theta)
    order = np.argsort(c, kind="stable")
    cs, ws = c[order], w[order]
    levels = np.concatenate([[0.0], np.cumsum(ws)])
    return cs, levels
