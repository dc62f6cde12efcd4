"""Oracle solver (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py): Riemannian trust-region Newton
with Steihaug-Toint truncated CG on the Grassmann manifold and p-continuation, written out plainly
in numpy over the oracle's F / EucGrad / EucHessianEta (plp_oracle.c).

Follows PAPER.md:120-121 ("Newton's method on the Grassmann manifold", "truncated conjugate gradient
scheme", "progressively smaller values of p") with the SPEC's statement of the trust-region method
 and DESIGN.md's readings #21-#24:
  * point U (n x k, orthonormal); tangent vectors xi with U^T xi = 0; <x, y> = sum x_il y_il;
  * grad = P(G) = G - U (U^T G), G = EucGrad (oracle.euc_grad);
  * Hess[xi] = P(EucHess[xi]) - xi S, S = (U^T G + G^T U) / 2;
  * retraction: Q of the thin QR of U + xi with R_ii > 0 (oracle.dense.retract, Householder);
  * tCG: Absil-Baker-Gallivan 2007, Algorithm 2 (no preconditioner), stopping at
    ||r|| <= ||r0|| min(||r0||^theta, kappa), negative curvature or the trust boundary;
  * rho = (F(U) - F(R(U, eta))) / (-<grad, eta> - <eta, Hess eta> / 2), accept if rho > 0.1,
    radius halved if rho < 1/4, doubled (up to the maximum) if rho > 3/4 at the boundary;
  * defaults grad_tol = 1e-6 sqrt(n k), Delta_max = sqrt(k), Delta_0 = Delta_max / 8,
    tcg_max_iters = min(2 n k, 1000), max_outer = 200.
Parity: end-to-end labels (up to permutation) and RCut against the GPU solver (tests/).
"""
from __future__ import annotations

import math

import numpy as np

from . import dense


def _state(g, U, p, fns):
    objective, euc_grad = fns["objective"], fns["euc_grad"]
    F, A, B = objective(g, U, p)
    G = euc_grad(g, U, p, A, B)
    M = U.T @ G
    grad = G - U @ M
    S = 0.5 * (M + M.T)
    return {"U": U, "F": F, "A": A, "B": B, "G": G, "grad": grad, "S": S}


def _hess(g, st, p, xi, eps, mode, fns):
    EH = fns["hessvec"](g, st["U"], xi, p, eps, mode, AB=(st["A"], st["B"]))
    U = st["U"]
    PEH = EH - U @ (U.T @ EH)
    return PEH - xi @ st["S"]


def tcg(hess_op, grad, U, delta, cfg):
    """Steihaug-Toint tCG for min <grad, s> + <s, H s> / 2, ||s|| <= delta, on the horizontal space
    at U (U None: plain Euclidean space).  Returns (eta, H eta, iterations, status)."""
    eta = np.zeros_like(grad)
    Heta = np.zeros_like(grad)
    r = grad.copy()
    z_r = float(np.sum(r * r))
    r0 = math.sqrt(z_r)
    if r0 == 0.0:
        return eta, Heta, 0, "interior"
    d = -r
    e_Pe, e_Pd, d_Pd = 0.0, 0.0, z_r
    stop_tol = r0 * min(r0 ** cfg["tcg_theta"], cfg["tcg_kappa"])
    status, j = "maxiter", 0
    for j in range(1, cfg["tcg_max_iters"] + 1):
        Hd = hess_op(d)
        d_Hd = float(np.sum(d * Hd))
        alpha = z_r / d_Hd if d_Hd != 0.0 else math.inf
        e_Pe_new = e_Pe + 2.0 * alpha * e_Pd + alpha * alpha * d_Pd
        if d_Hd <= 0.0 or e_Pe_new >= delta * delta:
            tau = (-e_Pd + math.sqrt(e_Pd * e_Pd + d_Pd * (delta * delta - e_Pe))) / d_Pd
            eta = eta + tau * d
            Heta = Heta + tau * Hd
            status = "negative_curvature" if d_Hd <= 0.0 else "boundary"
            break
        e_Pe = e_Pe_new
        eta = eta + alpha * d
        Heta = Heta + alpha * Hd
        r = r + alpha * Hd
        if U is not None:
            r = r - U @ (U.T @ r)
        z_new = float(np.sum(r * r))
        if math.sqrt(z_new) <= stop_tol:
            status = "converged"
            break
        beta = z_new / z_r
        z_r = z_new
        d = -r + beta * d
        e_Pd = beta * (e_Pd + alpha * d_Pd)
        d_Pd = z_r + beta * beta * d_Pd
    return eta, Heta, j, status


def default_cfg(n, k, **over):
    cfg = {"grad_tol": 1e-6 * math.sqrt(n * k), "max_outer": 200, "delta_max": math.sqrt(k),
           "rho_accept": 0.1, "tcg_kappa": 0.1, "tcg_theta": 1.0, "tcg_max_iters": min(2 * n * k, 1000),
           "mode": "sparse", "eps": 1e-9}
    cfg["delta0"] = cfg["delta_max"] / 8.0
    cfg.update(over)
    return cfg


def trust_region(g, U0, p, cfg, fns, trace):
    st = _state(g, U0, p, fns)
    delta = cfg["delta0"]
    for it in range(cfg["max_outer"]):
        gnorm = math.sqrt(float(np.sum(st["grad"] * st["grad"])))
        if gnorm <= cfg["grad_tol"] or delta < 1e-14:
            trace.append((p, it, st["F"], gnorm, delta, 0, "stop", math.nan, False))
            break
        eta, Heta, nit, status = tcg(lambda xi: _hess(g, st, p, xi, cfg["eps"], cfg["mode"], fns),
                                     st["grad"], st["U"], delta, cfg)
        model_dec = -float(np.sum(st["grad"] * eta)) - 0.5 * float(np.sum(eta * Heta))
        Q, R = dense.retract(st["U"], eta)
        if np.min(np.abs(np.diag(R))) > 0:
            cand = _state(g, Q, p, fns)
            F_new = cand["F"]
        else:
            cand, F_new = None, math.inf
        if model_dec > 0.0:
            rho = (st["F"] - F_new) / model_dec
        else:
            rho = 1.0 if F_new <= st["F"] else -math.inf
        accepted = cand is not None and math.isfinite(F_new) and rho > cfg["rho_accept"]
        if rho < 0.25:
            delta *= 0.5
        elif rho > 0.75 and status in ("boundary", "negative_curvature"):
            delta = min(2.0 * delta, cfg["delta_max"])
        trace.append((p, it, F_new if accepted else st["F"], gnorm, delta, nit, status, rho, accepted))
        if accepted:
            st = cand
    return st["U"]


def oracle_fns():
    from . import objective, euc_grad, hessvec
    return {"objective": objective, "euc_grad": euc_grad, "hessvec": hessvec}


def continuation_solve(g, Z, schedule, fns=None, **over):
    """QR of the seeded Gaussian Z, trust-region solve at each p of the schedule, QR re-orthonormal
    warm starts between stages."""
    fns = oracle_fns() if fns is None else fns
    n, k = Z.shape
    cfg = default_cfg(n, k, **over)
    U, _ = dense.retract(Z, np.zeros_like(Z))
    trace = []
    for j, p in enumerate(schedule):
        if j > 0:
            U, _ = dense.retract(U, np.zeros_like(U))
        U = trust_region(g, U, float(p), cfg, fns, trace)
    return U, trace
