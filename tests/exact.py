"""Exact reference solutions used to pin the oracle (test infrastructure).

These are textbook closed forms independent of the finite-volume method:
* oblique-shock theta-beta-M relation and Rankine-Hugoniot jumps
  (Anderson, Modern Compressible Flow, ch. 4), weak branch;
* exact Riemann solver for the 1D Euler equations (Toro, ch. 4), used for
  the Sod pin of SPEC.md:200.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.optimize import brentq


def theta_from_beta(M, beta, g=1.4):
    """tan(theta) = 2 cot(beta) (M^2 sin^2 b - 1) / (M^2 (g + cos 2b) + 2)."""
    s2 = (M * math.sin(beta)) ** 2
    return math.atan(2.0 / math.tan(beta) * (s2 - 1.0) / (M * M * (g + math.cos(2 * beta)) + 2.0))


def oblique_shock(M, theta_deg, g=1.4):
    """Weak-branch oblique shock: returns dict(beta_deg, p21, rho21, T21, M2)."""
    th = math.radians(theta_deg)
    mu = math.asin(1.0 / M)
    # theta(beta) rises from 0 at the Mach angle to theta_max; weak root first
    bs = np.linspace(mu + 1e-9, math.pi / 2 - 1e-9, 20001)
    ths = np.array([theta_from_beta(M, b, g) for b in bs])
    k = int(np.argmax(ths))
    if th > ths[k]:
        raise ValueError("detached shock: theta > theta_max")
    beta = brentq(lambda b: theta_from_beta(M, b, g) - th, mu + 1e-12, bs[k], xtol=1e-15)
    Mn1 = M * math.sin(beta)
    p21 = 1.0 + 2.0 * g / (g + 1.0) * (Mn1 * Mn1 - 1.0)
    rho21 = (g + 1.0) * Mn1 * Mn1 / ((g - 1.0) * Mn1 * Mn1 + 2.0)
    T21 = p21 / rho21
    Mn2 = math.sqrt((1.0 + 0.5 * (g - 1.0) * Mn1 * Mn1) / (g * Mn1 * Mn1 - 0.5 * (g - 1.0)))
    M2 = Mn2 / math.sin(beta - th)
    return dict(beta_deg=math.degrees(beta), p21=p21, rho21=rho21, T21=T21, M2=M2,
                theta_max_deg=math.degrees(ths[k]))


def normal_shock_states(M1, rho1=1.0, p1=1.0, g=1.4):
    """Stationary normal shock: (rho, u, p) upstream and downstream."""
    a1 = math.sqrt(g * p1 / rho1)
    u1 = M1 * a1
    rho21 = (g + 1.0) * M1 * M1 / ((g - 1.0) * M1 * M1 + 2.0)
    p21 = 1.0 + 2.0 * g / (g + 1.0) * (M1 * M1 - 1.0)
    rho2 = rho1 * rho21
    u2 = rho1 * u1 / rho2
    return (rho1, u1, p1), (rho2, u2, p1 * p21)


# ---------------------------------------------------------------- Riemann
def _fK(p, rhoK, pK, g):
    aK = math.sqrt(g * pK / rhoK)
    if p > pK:  # shock
        A = 2.0 / ((g + 1.0) * rhoK)
        B = (g - 1.0) / (g + 1.0) * pK
        return (p - pK) * math.sqrt(A / (p + B))
    return 2.0 * aK / (g - 1.0) * ((p / pK) ** ((g - 1.0) / (2.0 * g)) - 1.0)


def riemann_star(L, R, g=1.4):
    rL, uL, pL = L
    rR, uR, pR = R
    f = lambda p: _fK(p, rL, pL, g) + _fK(p, rR, pR, g) + (uR - uL)
    ps = brentq(f, 1e-12, 100.0 * max(pL, pR), xtol=1e-15, rtol=1e-15)
    us = 0.5 * (uL + uR) + 0.5 * (_fK(ps, rR, pR, g) - _fK(ps, rL, pL, g))
    return ps, us


def riemann_sample(L, R, x, t, x0=0.5, g=1.4):
    """Exact density at positions x (array) and time t (Toro ch. 4)."""
    rL, uL, pL = L
    rR, uR, pR = R
    ps, us = riemann_star(L, R, g)
    aL = math.sqrt(g * pL / rL); aR = math.sqrt(g * pR / rR)
    out = np.empty_like(np.asarray(x, dtype=float))
    gm = (g - 1.0) / (g + 1.0)
    for n, xx in enumerate(np.asarray(x, dtype=float)):
        S = (xx - x0) / t
        if S <= us:  # left of contact
            if ps > pL:
                SL = uL - aL * math.sqrt((g + 1) / (2 * g) * ps / pL + (g - 1) / (2 * g))
                out[n] = rL if S <= SL else rL * (ps / pL + gm) / (gm * ps / pL + 1.0)
            else:
                SHL = uL - aL
                asL = aL * (ps / pL) ** ((g - 1) / (2 * g))
                STL = us - asL
                if S <= SHL:
                    out[n] = rL
                elif S >= STL:
                    out[n] = rL * (ps / pL) ** (1.0 / g)
                else:
                    out[n] = rL * (2 / (g + 1) + gm / aL * (uL - S)) ** (2 / (g - 1))
        else:
            if ps > pR:
                SR = uR + aR * math.sqrt((g + 1) / (2 * g) * ps / pR + (g - 1) / (2 * g))
                out[n] = rR if S >= SR else rR * (ps / pR + gm) / (gm * ps / pR + 1.0)
            else:
                SHR = uR + aR
                asR = aR * (ps / pR) ** ((g - 1) / (2 * g))
                STR = us + asR
                if S >= SHR:
                    out[n] = rR
                elif S <= STR:
                    out[n] = rR * (ps / pR) ** (1.0 / g)
                else:
                    out[n] = rR * (2 / (g + 1) - gm / aR * (uR - S)) ** (2 / (g - 1))
    return out
