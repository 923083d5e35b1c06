"""Offline coefficient fitter: re-derive the step
tables of ReGELU2 / ReSiLU2 (App. E), ReGELU2-d
(App. I) or a k-bit variant (Eq. 14 with 2^k - 1 ReLUs,
P:L353-362) by simulated annealing on the GPU (``lmbp_fit_anneal``), and turn
a fitted theta into the (thresholds, levels) table ``stepact_fwd/bwd`` take.

Binding only: the objective and the search run in liblmbp.so's kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import ops


@dataclass
class Fit:
    act: str
    k: int
    objective: str
    a: list          # m - 1 weights of the ReLUs sorted by threshold
    c: list          # m thresholds, increasing
    J: float         # objective at (a, c)

    @property
    def weights(self):
        return list(self.a) + [1.0 - sum(self.a)]

    def table(self):
        """(thresholds, levels) for stepact_fwd / stepact_bwd: level j = h~'
        on segment j = sum of the j lowest ReLUs' weights."""
        lv, acc = [0.0], 0.0
        for w in self.weights:
            acc += w
            lv.append(acc)
        lv[-1] = 1.0   # the weights sum to 1 (Eq. 14); exact, as s3 = 1 in R5
        return list(self.c), lv


def fit(act: str, k: int = 2, objective: str = "h", refine_iters: int = 40, projected: bool = True,
        **anneal_kw) -> Fit:
    """Global search, then local refinement, both in GPU kernels with no host
    round trip: simulated annealing from many random starts (P:L1050-1053,
    "searching multiple times with different initialization"), then every
    chain's best point finished by Levenberg-Marquardt (lmbp_fit_refine) and
    the best refined point taken.  projected (default) anneals only the
    thresholds with least-squares weights (lmbp_fit_anneal_vp): the same k = 2
    optimum 2-3x sooner, and the only variant that converges for k >= 3;
    projected=False anneals all 2m - 1 parameters (lmbp_fit_anneal); it is
    also taken when the projected anneal refuses the interval (a tail
    tolerance so small that [A, B] exceeds its tables: LMBP_ERR_EPS)."""
    from ._lib import LMBP_ERR_EPS, LmbpError
    try:
        best, chain_theta, chain_J = ops.fit_anneal(act, k=k, objective=objective, projected=projected, **anneal_kw)
    except LmbpError as e:
        if not (projected and e.status == LMBP_ERR_EPS and anneal_kw.get("eps", 1e-8) > 0):
            raise
        best, chain_theta, chain_J = ops.fit_anneal(act, k=k, objective=objective, projected=False, **anneal_kw)
    if refine_iters > 0:
        best, _, _ = ops.fit_refine(chain_theta, act, k=k, objective=objective,
                                    eps=anneal_kw.get("eps", 1e-8), iters=refine_iters)
    b = best.double().cpu().tolist()
    m = (1 << k) - 1
    return Fit(act=act, k=k, objective=objective, a=b[:m - 1], c=b[m - 1:2 * m - 1], J=b[-1])


def objective(theta, act: str, k: int = 2, objective: str = "h", eps: float = 1e-8, device="cuda"):
    """J for one theta (sequence) or a batch [n, P]; returns a CUDA tensor."""
    t = torch.as_tensor(theta, dtype=torch.float64, device=device)
    if t.dim() == 1:
        t = t[None]
    return ops.fit_objective(t.contiguous(), act, k=k, objective=objective, eps=eps)
