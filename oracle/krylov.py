"""Restarted GMRES(m), right-preconditioned, modified Gram-Schmidt (oracle; test infrastructure only).

P:225 names GMRES (Saad & Schultz 1986) as the Krylov method for the nonsymmetric system; BASELINE.json
fixes GMRES(30) to relative residual 1e-8.  Readings: x0 = 0 unless given, right
preconditioning  A P^{-1} y = b, x = P^{-1} y;  one iteration = one Arnoldi step (one P^{-1} apply and
one A-matvec);  convergence on the implicit residual |g_{j+1}| <= rtol ||b||, confirmed by the true
residual at the top of the next cycle;  never normalise by h_{j+1,j} after convergence is declared.
"""
import math

import numpy as np


def gmres(matvec, b, precond=None, x0=None, m=30, rtol=1e-8, max_iters=1000):
    """Returns (x, report) with report = dict(iters, restarts, converged, rel_res_true, rel_res_implicit, history)."""
    N = b.shape[0]
    Pinv = precond if precond is not None else (lambda v: v.copy())
    x = np.zeros(N) if x0 is None else np.array(x0, dtype=np.float64)
    bnorm = math.sqrt(float(b @ b))
    target = rtol * bnorm
    iters, restarts = 0, 0
    history = []
    rel_implicit = float("nan")
    converged = False
    while True:
        r = b - matvec(x)
        beta = math.sqrt(float(r @ r))
        if beta <= target or bnorm == 0.0:
            converged = True
            break
        if iters >= max_iters:
            break
        V = np.zeros((m + 1, N))
        Hm = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        k = 0
        for j in range(m):
            z = Pinv(V[j])
            w = matvec(z)
            iters += 1
            for i in range(j + 1):                 # modified Gram-Schmidt
                Hm[i, j] = float(w @ V[i])
                w = w - Hm[i, j] * V[i]
            Hm[j + 1, j] = math.sqrt(float(w @ w))
            for i in range(j):                     # apply previous Givens rotations
                t = cs[i] * Hm[i, j] + sn[i] * Hm[i + 1, j]
                Hm[i + 1, j] = -sn[i] * Hm[i, j] + cs[i] * Hm[i + 1, j]
                Hm[i, j] = t
            a, bb = Hm[j, j], Hm[j + 1, j]
            rr = math.hypot(a, bb)
            cs[j], sn[j] = (1.0, 0.0) if rr == 0.0 else (a / rr, bb / rr)
            Hm[j, j] = rr
            Hm[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            rel_implicit = abs(g[j + 1]) / bnorm
            history.append(rel_implicit)
            k = j + 1
            if abs(g[j + 1]) <= target or bb == 0.0 or iters >= max_iters:
                break
            V[j + 1] = w / bb
        # y = R_k^{-1} g_{0..k-1} (back substitution), x += P^{-1}(V_k y)
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - Hm[i, i + 1:k] @ y[i + 1:k]) / Hm[i, i]
        x = x + Pinv(V[:k].T @ y)
        restarts += 1
    rel_true = math.sqrt(float(np.sum((b - matvec(x)) ** 2))) / bnorm if bnorm > 0 else 0.0
    return x, dict(iters=iters, restarts=restarts, converged=converged, rel_res_true=rel_true,
                   rel_res_implicit=rel_implicit, history=history)


def bicgstab(matvec, b, precond=None, x0=None, rtol=1e-8, max_iters=1000):
    """Right-preconditioned BiCGStab (van der Vorst 1992), the paper's solver: every
    iteration is one BiCG step followed by one GMRES(1) step ("each iteration of BiCGStab consists in a
    Biconjugate Gradient (BiCG) step followed by a single iteration of GMRES").  Half-iteration
    accounting (reading 15): convergence after the BiCG half of iteration k (1-based)
    reports k - 0.5, i.e. "(completed iterations) + 0.5"; after the full iteration it reports k.

    Steps, in van der Vorst's order, with r^ = r_0 (shadow residual), x0 = 0 unless given:
        rho_k = r^ . r_{k-1};  p_k = r_{k-1} + beta (p_{k-1} - omega_{k-1} v_{k-1}),
                               beta = (rho_k / rho_{k-1}) (alpha_{k-1} / omega_{k-1})   (p_1 = r_0)
        p^ = P^{-1} p_k;  v_k = A p^;  alpha_k = rho_k / (r^ . v_k)
        s = r_{k-1} - alpha_k v_k;  x <- x + alpha_k p^          (BiCG half step; stop if ||s|| <= rtol ||b||)
        s^ = P^{-1} s;  t = A s^;  omega_k = (t . s) / (t . t)
        x <- x + omega_k s^;  r_k = s - omega_k t                (GMRES(1) half step; stop if ||r_k|| <= rtol ||b||)
    Breakdown (rho = 0, r^.v = 0, t.t = 0 or omega = 0 before convergence) is reported, not converged.
    Returns (x, report) with report = dict(iters (float), converged, breakdown, rel_res_true,
    rel_res_recursive, history) -- history holds the recursive relative residual after every half step.
    """
    N = b.shape[0]
    Pinv = precond if precond is not None else (lambda v: v.copy())
    x = np.zeros(N) if x0 is None else np.array(x0, dtype=np.float64)
    bnorm = math.sqrt(float(b @ b))
    target = rtol * bnorm
    r = b - matvec(x)
    rhat = r.copy()
    history = []
    rel_rec = math.sqrt(float(r @ r)) / bnorm if bnorm > 0 else 0.0
    iters, converged, breakdown = 0.0, bnorm == 0.0 or math.sqrt(float(r @ r)) <= target, False
    rho_prev = alpha = omega = 1.0
    p = np.zeros(N)
    v = np.zeros(N)
    k = 0
    while not converged and k < max_iters:
        k += 1
        rho = float(rhat @ r)
        if rho == 0.0:
            breakdown = True
            break
        if k == 1:
            p = r.copy()
        else:
            beta = (rho / rho_prev) * (alpha / omega)
            p = r + beta * (p - omega * v)
        phat = Pinv(p)
        v = matvec(phat)
        sigma = float(rhat @ v)
        if sigma == 0.0:
            breakdown = True
            break
        alpha = rho / sigma
        s = r - alpha * v
        x = x + alpha * phat
        snorm = math.sqrt(float(s @ s))
        history.append(snorm / bnorm)
        if snorm <= target:
            iters, converged, rel_rec = k - 0.5, True, snorm / bnorm
            break
        shat = Pinv(s)
        t = matvec(shat)
        tt = float(t @ t)
        if tt == 0.0:
            breakdown = True
            break
        omega = float(t @ s) / tt
        x = x + omega * shat
        r = s - omega * t
        rnorm = math.sqrt(float(r @ r))
        history.append(rnorm / bnorm)
        iters, rel_rec = float(k), rnorm / bnorm
        if rnorm <= target:
            converged = True
            break
        if omega == 0.0:
            breakdown = True
            break
        rho_prev = rho
    rel_true = math.sqrt(float(np.sum((b - matvec(x)) ** 2))) / bnorm if bnorm > 0 else 0.0
    return x, dict(iters=iters, converged=converged, breakdown=breakdown, rel_res_true=rel_true,
                   rel_res_recursive=rel_rec, history=history)
