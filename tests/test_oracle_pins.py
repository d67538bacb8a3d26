"""Pins of the CPU oracle against what the paper and mathematics fix
(SURVEY.md §8(c).4).  None of these compare the oracle with itself by
retyping its formulas: each expected value is a printed number (golden
file, cited), a closed form derived independently, an invariant, or a
textbook solution (tests/exact.py)."""
import math
import os

import numpy as np
import pytest

from paper_2305_18057_b200 import inputs as I
import exact


def rel(a, b):
    a = np.asarray(a, float); b = np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


# ------------------------------------------------------------------ metrics
def test_metrics_unit_square(oracle_mod):
    X = np.array([[0.0, 1.0], [0.0, 1.0]]); Y = np.array([[0.0, 0.0], [1.0, 1.0]])
    fi, fj, V = oracle_mod.metrics(X, Y)
    assert V[0, 0] == 1.0
    np.testing.assert_array_equal(fi[0, 0], [1.0, 0.0, 1.0])   # west face, +x normal
    np.testing.assert_array_equal(fi[0, 1], [1.0, 0.0, 1.0])
    np.testing.assert_array_equal(fj[0, 0], [0.0, 1.0, 1.0])   # south face, +y normal
    np.testing.assert_array_equal(fj[1, 0], [0.0, 1.0, 1.0])


def test_metrics_quad_area(oracle_mod, golden):
    g = golden["quad_area"]
    (x0, y0), (x1, y1), (x2, y2), (x3, y3) = g["nodes"]
    X = np.array([[x0, x1], [x3, x2]]); Y = np.array([[y0, y1], [y3, y2]])
    _, _, V = oracle_mod.metrics(X, Y)
    assert abs(V[0, 0] - g["V"]) < 1e-15


@pytest.mark.parametrize("theta", [0.0, 10.0, 15.0, 30.0])
def test_metrics_closed_surface_and_positive(oracle_mod, theta):
    X, Y = I.ramp_nodes(40, 20, theta)
    fi, fj, V = oracle_mod.metrics(X, Y)
    assert np.all(V > 0)
    # outward sum: -W + E - S + N  (normals point +i / +j)
    sx = (-fi[:, :-1, 0] * fi[:, :-1, 2] + fi[:, 1:, 0] * fi[:, 1:, 2]
          - fj[:-1, :, 0] * fj[:-1, :, 2] + fj[1:, :, 0] * fj[1:, :, 2])
    sy = (-fi[:, :-1, 1] * fi[:, :-1, 2] + fi[:, 1:, 1] * fi[:, 1:, 2]
          - fj[:-1, :, 1] * fj[:-1, :, 2] + fj[1:, :, 1] * fj[1:, :, 2])
    perim = fi[:, :-1, 2] + fi[:, 1:, 2] + fj[:-1, :, 2] + fj[1:, :, 2]
    assert np.max(np.abs(sx) / perim) < 1e-12 and np.max(np.abs(sy) / perim) < 1e-12
    # |n| = 1
    assert np.max(np.abs(np.hypot(fi[..., 0], fi[..., 1]) - 1)) < 1e-14
    # shoelace area equals the analytic trapezoid area of the sheared column
    x = X[0]
    yb, yt = Y[0], Y[-1]
    col_area = 0.5 * (x[1:] - x[:-1]) * ((yt[1:] - yb[1:]) + (yt[:-1] - yb[:-1]))
    np.testing.assert_allclose(V.sum(axis=0), col_area, rtol=1e-12)


def test_metrics_refinement_quarter(oracle_mod):
    X1, Y1 = I.cartesian_nodes(4, 2, 2.0, 1.0)
    X2, Y2 = I.cartesian_nodes(8, 4, 2.0, 1.0)
    V1 = oracle_mod.metrics(X1, Y1)[2]; V2 = oracle_mod.metrics(X2, Y2)[2]
    assert np.all(V2 == 0.25 * V1[0, 0]) and np.all(V1 == 0.25)


def test_metrics_rejects_tangled(oracle_mod):
    X = np.array([[0.0, 1.0], [1.0, 0.0]]); Y = np.array([[0.0, 0.0], [1.0, 1.0]])
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.metrics(X, Y)


# ---------------------------------------------------------------------- gas
def test_gas_quiescent(oracle_mod, golden):
    g = golden["quiescent_pressure"]
    np.testing.assert_allclose(oracle_mod.primitive(g["U"]), g["prim"], rtol=0, atol=1e-15)
    for prim, ht in golden["total_enthalpy"]["cases"]:
        U = I.conserved_from_primitive(prim)
        p = oracle_mod.primitive(U)
        assert abs((U[3] + p[3]) / U[0] - ht) < 1e-15


def test_table1_freestream(oracle_mod, golden):
    t1 = golden["table1"]; d = golden["table1_derived"]
    prim = I.freestream_primitive(t1["mach"], t1["p"], t1["T"])
    U = I.freestream_conserved()
    tol = 0.5 * 10.0 ** (-d["digits"])
    assert abs(prim[0] / d["rho"] - 1) < tol
    assert abs(prim[1] / d["u"] - 1) < tol
    assert abs(U[3] / d["E"] - 1) < tol
    back = oracle_mod.primitive(U)
    np.testing.assert_allclose(back, prim, rtol=1e-15, atol=1e-12)
    a = math.sqrt(1.4 * back[3] / back[0])
    assert abs(a / d["a"] - 1) < tol
    assert abs((U[1] * back[1] + back[3]) / d["momentum_flux"] - 1) < tol
    # rho u^2 + p = p (1 + gamma M^2) and h_t = c_p T + u^2/2 (closed forms)
    assert abs((U[1] * back[1] + back[3]) / (t1["p"] * (1 + 1.4 * 16.0)) - 1) < 1e-14
    ht = (U[3] + back[3]) / U[0]
    assert abs(ht / (1.4 * 287 / 0.4 * t1["T"] + 0.5 * back[1] ** 2) - 1) < 1e-14
    assert abs(ht / d["h_t"] - 1) < tol


# ------------------------------------------------------------ limiter/MUSCL
def test_limiter_special_values(oracle_mod):
    L = oracle_mod.limiter
    assert L(0, 0.0, 0.0) == 1.0            # uniform line -> exactly 1
    for d in [1e-3, 0.7, 1.0, 123.0]:
        assert L(0, d, d) == 1.0           # linear data -> exactly 1
    assert L(0, -1.0, 1.0) == 0.0          # extremum -> 0
    assert L(0, 1.0, -1.0) == 0.0
    r = np.linspace(0, 10, 101)
    for x in r:
        v2 = L(1, x, 1.0)
        assert 0.0 <= v2 <= 1.0 + 1e-15    # VA2 bounded in [0, 1]
    # VA1 maximum (1+sqrt2)/2 at r = 1+sqrt2 (documented deviation from S:166)
    rm = 1 + math.sqrt(2)
    assert abs(L(0, rm, 1.0, 0.0) - (1 + math.sqrt(2)) / 2) < 1e-15
    assert L(2, -5.0, 3.0) == 1.0


def test_muscl_pins(oracle_mod):
    M = oracle_mod.muscl
    assert M([2.0, 2.0, 2.0, 2.0]) == (2.0, 2.0)
    assert M([0.0, 1.0, 5.0, -3.0], eps=0.0) == (1.0, 5.0)
    for kappa in [-1.0, 0.0, 1.0 / 3.0, 1.0]:
        assert M([0.0, 1.0, 2.0, 3.0], kappa=kappa) == (1.5, 1.5)
    # extremum -> limiter zero -> first order
    assert M([0.0, 1.0, 0.0, 1.0]) == (1.0, 0.0)


def test_muscl_kappa_independence(oracle_mod):
    """With VA1 and delta = 0, psi(1/r) = psi(r)/r, so the kappa terms of
    Eq. 7 coincide and Q^L, Q^R do not depend on kappa.  A swapped
    Psi^+/Psi^- convention (reading A-R4) breaks this by O(1)."""
    rng = np.random.default_rng(0)
    worst = 0.0
    for _ in range(2000):
        w = np.cumsum(rng.uniform(0.1, 1.0, 4)) * rng.choice([-1, 1])
        ref = np.array(oracle_mod.muscl(w, kappa=-1.0, delta=0.0))
        for kappa in [0.0, 1.0 / 3.0, 1.0]:
            q = np.array(oracle_mod.muscl(w, kappa=kappa, delta=0.0))
            worst = max(worst, float(np.max(np.abs(q - ref) / np.abs(ref))))
    assert worst < 4 * 2.2e-16


# --------------------------------------------------------------------- Roe
def test_roe_consistency_printed(oracle_mod, golden):
    g = golden["consistency_flux"]
    U = I.conserved_from_primitive(g["prim"])
    F = oracle_mod.roe_flux(U, U, *g["n"])
    np.testing.assert_array_equal(F, g["F"])


def test_roe_consistency_table1_30deg(oracle_mod):
    rho, u, v, p = I.freestream_primitive()
    U = I.freestream_conserved()
    c, s = math.cos(math.radians(30)), math.sin(math.radians(30))
    F = oracle_mod.roe_flux(U, U, c, s)
    # analytic normal flux (Eq. 2) with Vn = u cos30 written independently
    Vn = u * c
    want = [rho * Vn, rho * u * Vn + p * c, p * s, (U[3] + p) * Vn]
    assert rel(F, want) < 1e-15


def test_roe_stationary_contact(oracle_mod):
    L = I.conserved_from_primitive([1.0, 0.0, 0.0, 1.0])
    R = I.conserved_from_primitive([0.125, 0.0, 0.0, 1.0])
    np.testing.assert_array_equal(oracle_mod.roe_flux(L, R, 1.0, 0.0), [0.0, 1.0, 0.0, 0.0])


def analytic_flux(U, nx, ny, g=1.4):
    rho, mx, my, E = U
    u, v = mx / rho, my / rho
    p = (g - 1) * (E - 0.5 * rho * (u * u + v * v))
    Vn = u * nx + v * ny
    return np.array([rho * Vn, mx * Vn + p * nx, my * Vn + p * ny, (E + p) * Vn])


def test_roe_supersonic_upwind(oracle_mod):
    """All eigenvalues > delta_H: Roe's A~ dQ = dF gives F = F(Q_L)."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        th = rng.uniform(0, 2 * math.pi); n = (math.cos(th), math.sin(th))
        a = 1.0
        qn = rng.uniform(3.0, 5.0)
        base = np.array([1.0, qn * n[0], qn * n[1], 1.0 / 1.4])
        L = base * (1 + 0.05 * rng.uniform(-1, 1, 4)); R = base * (1 + 0.05 * rng.uniform(-1, 1, 4))
        UL = I.conserved_from_primitive(L); UR = I.conserved_from_primitive(R)
        F = oracle_mod.roe_flux(UL, UR, *n)
        FL = analytic_flux(UL, *n)
        assert rel(F, FL) < 2e-15


def test_roe_stationary_normal_shock(oracle_mod):
    (r1, u1, p1), (r2, u2, p2) = exact.normal_shock_states(2.5)
    UL = I.conserved_from_primitive([r1, u1, 0, p1]); UR = I.conserved_from_primitive([r2, u2, 0, p2])
    F = oracle_mod.roe_flux(UL, UR, 1.0, 0.0, harten_eps=0.0)
    # With harten_eps = 0 the floor delta_H = 1e-12 (reading A-R2) still lifts
    # the sonic eigenvalue lambda_1 ~ 0 to delta_H/2, which perturbs F by
    # at most |alpha_1 r_1| delta_H / 4 ~ 1e-12 absolute.
    assert rel(F, analytic_flux(UL, 1, 0)) < 1e-12
    assert rel(F, analytic_flux(UR, 1, 0)) < 1e-12
    Fh = oracle_mod.roe_flux(UL, UR, 1.0, 0.0, harten_eps=0.1)
    assert rel(Fh, analytic_flux(UL, 1, 0)) > 1e-3   # the Harten fix is active


def test_roe_mirrored_wall(oracle_mod):
    rng = np.random.default_rng(2)
    for _ in range(100):
        prim = [rng.uniform(0.5, 2), rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(0.5, 2)]
        UL = I.conserved_from_primitive(prim)
        UR = UL.copy(); UR[1] = -UR[1]                     # mirror across n = (1, 0)
        F = oracle_mod.roe_flux(UL, UR, 1.0, 0.0)
        assert F[0] == 0.0 and F[2] == 0.0 and F[3] == 0.0


def test_roe_rejects_invalid(oracle_mod):
    U = I.conserved_from_primitive([1.0, 0.0, 0.0, 1.0])
    bad = U.copy(); bad[3] = 0.1 * U[3] - 10
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.roe_flux(U, bad, 1.0, 0.0)


# ------------------------------------------------------------- whole solver
def _solver(oracle_mod, ni, nj, theta=30.0, **kw):
    X, Y = I.ramp_nodes(ni, nj, theta) if theta is not None else I.cartesian_nodes(ni, nj)
    cfg = I.default_config(ni, nj, **kw)
    return oracle_mod.Oracle(cfg, X, Y), cfg, X, Y


@pytest.mark.parametrize("theta", [None, 30.0])
def test_freestream_preservation(oracle_mod, theta):
    """Uniform flow with all-inflow boundaries: residual round-off only
    (acceptance 8)."""
    o, cfg, X, Y = _solver(oracle_mod, 24, 12, theta, bc=(0, 0, 0, 0))
    U = I.uniform_state(24, 12)
    R = o.residual(U)
    fi = oracle_mod.metrics(X, Y)[0]
    scale = np.max(np.abs(analytic_flux(U[0, 0], 1, 0))) * np.max(fi[..., 2])
    assert np.max(np.abs(R)) / scale < 1e-11


def test_ghost_fill_rules(oracle_mod):
    o, cfg, X, Y = _solver(oracle_mod, 6, 5, 30.0)
    U = I.perturbed_state(6, 5, seed=3)
    F = o.ghost_frame(U)
    inflow = I.freestream_conserved()
    # W inflow: both layers = U_in
    np.testing.assert_array_equal(F[2:-2, 0], np.broadcast_to(inflow, (5, 4)))
    np.testing.assert_array_equal(F[2:-2, 1], np.broadcast_to(inflow, (5, 4)))
    # E outflow: zeroth-order extrapolation
    np.testing.assert_array_equal(F[2:-2, -1], U[:, -1]); np.testing.assert_array_equal(F[2:-2, -2], U[:, -1])
    # S slip wall: rho, E copied; normal momentum reversed, tangential kept
    fj = oracle_mod.metrics(X, Y)[1]
    for m in range(2):
        g = F[1 - m, 2:-2]; w = U[m]
        n = fj[0, :, :2]
        np.testing.assert_array_equal(g[:, 0], w[:, 0]); np.testing.assert_array_equal(g[:, 3], w[:, 3])
        mn_w = w[:, 1] * n[:, 0] + w[:, 2] * n[:, 1]; mn_g = g[:, 1] * n[:, 0] + g[:, 2] * n[:, 1]
        mt_w = -w[:, 1] * n[:, 1] + w[:, 2] * n[:, 0]; mt_g = -g[:, 1] * n[:, 1] + g[:, 2] * n[:, 0]
        np.testing.assert_allclose(mn_g, -mn_w, rtol=1e-13, atol=1e-12)
        np.testing.assert_allclose(mt_g, mt_w, rtol=1e-13, atol=1e-12)
    # corner ghosts untouched (NaN)
    assert np.all(np.isnan(F[:2, :2])) and np.all(np.isnan(F[-2:, -2:]))


def test_slip_wall_mirror_printed(oracle_mod):
    """slip wall with n = (0,1): ghost (rho, u, -v, p)."""
    o, cfg, X, Y = _solver(oracle_mod, 4, 4, None)
    U = I.perturbed_state(4, 4, seed=5)
    F = o.ghost_frame(U)
    g = F[1, 2:-2]; w = U[0]
    np.testing.assert_array_equal(g[:, [0, 1, 3]], w[:, [0, 1, 3]])
    np.testing.assert_array_equal(g[:, 2], -w[:, 2])


def test_conservation_closed_box(oracle_mod):
    """All slip walls on flat walls: interior faces telescope and wall mass /
    energy fluxes vanish, so sum R_rho = sum R_E = 0."""
    o, cfg, X, Y = _solver(oracle_mod, 16, 12, None, bc=(2, 2, 2, 2))
    U = I.perturbed_state(16, 12, seed=7, prim0=np.array([0.2, 60.0, 0.0, 12270.0]))
    R = o.residual(U)
    for k in (0, 3):
        assert abs(R[..., k].sum()) <= 1e-10 * np.abs(R[..., k]).sum()
    # x-momentum: net = pressure force on the W/E walls only
    assert abs(R[..., 1].sum()) > 0


def test_j_invariance(oracle_mod):
    # nj a power of two so that every row of the Cartesian grid is bitwise
    # identical (y = j/nj exact)
    ni, nj = 20, 8
    o, cfg, X, Y = _solver(oracle_mod, ni, nj, None, bc=(0, 1, 2, 2))
    row = I.perturbed_state(ni, 1, seed=11)
    row[..., 2] = 0.0
    row[..., 3] = I.conserved_from_primitive(np.stack([row[0, :, 0], row[0, :, 1] / row[0, :, 0],
                                                       np.zeros(ni), np.full(ni, I.TABLE1_P)], -1))[:, 3]
    U = np.repeat(row, nj, axis=0)
    o.set_state(U)
    for _ in range(5):
        o.step(4)
        S = o.get_state()
        assert np.all(S == S[0:1])
    assert np.all(np.isfinite(S))


def test_rk_zero_residual_fixed_point(oracle_mod):
    X, Y = I.cartesian_nodes(3, 2)
    for rk in (0, 1, 2):
        cfg = I.default_config(3, 2, rk=rk, dt_fixed=0.1)
        o = oracle_mod.Oracle(cfg, X, Y, residual_kind=oracle_mod.RES_LINEAR, linear_rate=0.0)
        U = I.perturbed_state(3, 2, seed=1)
        o.set_state(U); o.step(3)
        np.testing.assert_array_equal(o.get_state(), U)


@pytest.mark.parametrize("rk,key", [(0, "rk4"), (1, "heun"), (2, "rk4")])
def test_rk_scalar_decay(oracle_mod, golden, rk, key):
    """u' = -u, u0 = 1, dt = 0.1.  Jameson-4 gives the same
    truncated series on a linear ODE."""
    g = golden["rk_scalar"]
    X, Y = I.cartesian_nodes(2, 2)
    cfg = I.default_config(2, 2, rk=rk, dt_fixed=g["dt"])
    o = oracle_mod.Oracle(cfg, X, Y, residual_kind=oracle_mod.RES_LINEAR, linear_rate=1.0)
    U = np.broadcast_to(np.array([1.0, 0.0, 0.0, 2.5]), (2, 2, 4)).copy()
    o.set_state(U); o.step(1)
    S = o.get_state()
    assert abs(S[0, 0, 0] - g[key]) < 1e-15 + 5e-8   # golden printed to 7-8 digits
    series = sum((-g["dt"]) ** k / math.factorial(k) for k in range(4 if key == "rk4" else 2, -1, -1)
                 if k <= (4 if key == "rk4" else 2))
    assert abs(S[0, 0, 0] - series) < 1e-15


@pytest.mark.parametrize("rk,order", [(0, 4.0), (1, 2.0), (2, 2.0)])
def test_rk_temporal_order(oracle_mod, rk, order):
    """Observed order at t = 1 over dt in {0.1, 0.05, 0.025}.
    Jameson-4 is 4th order on linear problems only; on u' = -u it shows 4."""
    X, Y = I.cartesian_nodes(2, 2)
    errs = []
    for dt in (0.1, 0.05, 0.025):
        cfg = I.default_config(2, 2, rk=rk, dt_fixed=dt)
        o = oracle_mod.Oracle(cfg, X, Y, residual_kind=oracle_mod.RES_LINEAR, linear_rate=1.0)
        U = np.broadcast_to(np.array([1.0, 0.0, 0.0, 2.5]), (2, 2, 4)).copy()
        o.set_state(U); o.step(int(round(1.0 / dt)))
        errs.append(abs(o.get_state()[0, 0, 0] - math.exp(-1.0)))
    p = np.polyfit(np.log([0.1, 0.05, 0.025]), np.log(errs), 1)[0]
    want = 4.0 if rk in (0, 2) else 2.0
    assert abs(p - want) < (0.2 if want == 4.0 else 0.1)


def test_dt_closed_form(oracle_mod, golden):
    X, Y = I.cartesian_nodes(3, 3, 3.0, 3.0)
    cfg = I.default_config(3, 3, cfl=1.0, bc=(2, 2, 2, 2))
    o = oracle_mod.Oracle(cfg, X, Y)
    U = np.broadcast_to(np.array([1.0, 0.0, 0.0, 2.5]), (3, 3, 4)).copy()
    o.set_state(U); o.step(1)
    dt0 = o.dt()[0]
    assert abs(dt0 - 1.0 / (4.0 * math.sqrt(1.4))) < 1e-15
    assert abs(dt0 - golden["quiescent_dt"]["dt"]) < 1e-10
    X2, Y2 = I.cartesian_nodes(6, 6, 3.0, 3.0)
    o2 = oracle_mod.Oracle(I.default_config(6, 6, cfl=1.0, bc=(2, 2, 2, 2)), X2, Y2)
    o2.set_state(np.broadcast_to(np.array([1.0, 0.0, 0.0, 2.5]), (6, 6, 4)).copy()); o2.step(1)
    assert o2.dt()[0] == 0.5 * dt0
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.Oracle(I.default_config(3, 3, cfl=0.0), X, Y)


def test_norm_definition_matches_residual(oracle_mod):
    """Recorded norms of step n are L2 (RMS) and Linf of R(U^n) (A-R20),
    checked against an explicit residual evaluation."""
    o, cfg, X, Y = _solver(oracle_mod, 12, 8, 30.0)
    U = I.perturbed_state(12, 8, seed=2)
    R = o.residual(U)
    o.set_state(U); o.step(1)
    n = o.residual_norms()[0]
    np.testing.assert_allclose(n[:4], np.sqrt((R ** 2).reshape(-1, 4).sum(0) / 96), rtol=1e-14)
    np.testing.assert_array_equal(n[4:], np.abs(R).reshape(-1, 4).max(0))


# ----------------------------------------------------------- partition maps
def test_partition_printed(oracle_mod, golden):
    g = golden["partition"]
    s = oracle_mod.split(g["N"], len(g["weights"]), g["weights"])
    assert list(np.diff(s)) == g["widths"]
    assert list(oracle_mod.split(17, 1)) == [0, 17]
    assert list(np.diff(oracle_mod.split(96, 8))) == [12] * 8
    assert list(np.diff(oracle_mod.split(10, 3))) == [4, 3, 3]   # tie -> lower rank
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.split(7, 4)                                   # width < 2


def test_partition_map_neighbours(oracle_mod):
    o, *_ = _solver(oracle_mod, 16, 8, 30.0)
    o.partition(4, 2)
    m = o.partition_map(5)          # bx=1, by=1
    assert list(m) == [4, 8, 4, 8, 4, 6, 1, -1]


@pytest.mark.parametrize("px,py,wx,wy", [(2, 1, None, None), (5, 1, [8, 1, 1, 1, 1], None),
                                         (8, 1, None, None), (2, 2, None, None), (3, 2, [1, 2, 3], [2, 1])])
def test_decomposition_invariance_bitwise(oracle_mod, px, py, wx, wy):
    """PAPER.md:241 (< 1e-12 between serial and parallel solutions; SPEC
    acceptance 1).  The oracle reaches it bitwise."""
    ni, nj = 120, 40
    o1, cfg, X, Y = _solver(oracle_mod, ni, nj, 30.0)
    U = I.perturbed_state(ni, nj, seed=4)
    o1.set_state(U); o1.step(50)
    o2 = oracle_mod.Oracle(cfg, X, Y); o2.partition(px, py, wx, wy)
    o2.set_state(U); o2.step(50)
    np.testing.assert_array_equal(o1.get_state(), o2.get_state())
    np.testing.assert_array_equal(o1.residual_norms(), o2.residual_norms())
    np.testing.assert_array_equal(o1.dt(), o2.dt())


# ------------------------------------------------------------------ physics
def test_theta_beta_m_helper(golden):
    for th, want in golden["oblique_shock_M4"].items():
        if th == "cite":
            continue
        got = exact.oblique_shock(4.0, float(th))
        for k in ("beta_deg", "p21", "rho21", "T21", "M2"):
            assert abs(got[k] - want[k]) < 1e-4 * max(1, abs(want[k])), (th, k)


def test_sod_exact_helper(golden):
    g = golden["sod_star"]
    ps, us = exact.riemann_star((1.0, 0.0, 1.0), (0.125, 0.0, 0.1))
    assert abs(ps - g["p_star"]) < 1e-6 and abs(us - g["u_star"]) < 1e-6


def test_sod_shock_tube(oracle_mod):
    """Sod on a j-invariant 2D grid, 200 cells, t = 0.2: L1(rho) < 0.02
    (SPEC.md:200)."""
    ni, nj = 200, 2
    X, Y = I.cartesian_nodes(ni, nj, 1.0, 0.01)
    cfg = I.default_config(ni, nj, bc=(1, 1, 2, 2), dt_fixed=0.0008)
    o = oracle_mod.Oracle(cfg, X, Y)
    xc = (np.arange(ni) + 0.5) / ni
    prim = np.where(xc[:, None] < 0.5, [1.0, 0.0, 0.0, 1.0], [0.125, 0.0, 0.0, 0.1])
    U = np.repeat(I.conserved_from_primitive(prim)[None], nj, axis=0)
    o.set_state(U); o.step(250)
    rho = o.get_state()[0, :, 0]
    ex = exact.riemann_sample((1.0, 0.0, 1.0), (0.125, 0.0, 0.1), xc, 0.2)
    assert np.mean(np.abs(rho - ex)) < 0.02


def test_oblique_shock_wedge_C1(oracle_mod, golden):
    """Config C1 (64x32, 15 deg wedge, Table 1 freestream): ramp-wall
    pressure mid-ramp matches theta-beta-M p2/p1 = 3.69726 within 3%."""
    ni, nj = 64, 32
    X, Y = I.ramp_nodes(ni, nj, 15.0)
    cfg = I.default_config(ni, nj)
    o = oracle_mod.Oracle(cfg, X, Y)
    o.set_state(I.uniform_state(ni, nj))
    o.step(2000)
    S = o.get_state()
    xc = 0.25 * (X[0, :-1] + X[0, 1:] + X[1, :-1] + X[1, 1:])
    sel = (xc > 1.6) & (xc < 2.4)
    p = np.array([oracle_mod.primitive(S[0, i])[3] for i in np.nonzero(sel)[0]])
    p21 = p.mean() / I.TABLE1_P
    want = golden["oblique_shock_M4"]["15"]["p21"]
    assert abs(p21 / want - 1) < 0.03, p21


def test_stable_dt_matches_solver_dt(oracle_mod):
    """orc_stable_dt (banded, no solver context; used by the C3 window
    parity test) reproduces the solver's dt_0 bit for bit."""
    for (ni, nj, th) in [(300, 200, 30.0), (64, 130, 15.0)]:
        X, Y = I.ramp_nodes(ni, nj, th)
        U = I.perturbed_state(ni, nj, 1)
        o = oracle_mod.Oracle(I.default_config(ni, nj), X, Y)
        o.set_state(U); o.step(1)
        assert o.dt()[0] == oracle_mod.stable_dt(X, Y, U)


def test_openmp_build_is_bitwise_single_thread(tmp_path):
    """The -fopenmp build of oracle.c (bench.py's all-cores CPU baseline) is
    bitwise the single-threaded oracle: state, norm and dt histories after
    30 RK4 steps of a perturbed 30-degree inlet on 4 threads, incl. 2x2
    blocks (row loops shared; norm sums serial; dt min exact)."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
import oracle
from paper_2305_18057_b200 import inputs as I
ni, nj = 96, 48
X, Y = I.ramp_nodes(ni, nj, 30.0)
cfg = I.default_config(ni, nj)
U0 = I.perturbed_state(ni, nj, 4)
out = []
for omp in (False, True):
    for (px, py) in ((1, 1), (2, 2)):
        o = oracle.Oracle(cfg, X, Y, omp=omp)
        o.partition(px, py)
        o.set_state(U0); o.step(30)
        out.append((o.get_state(), o.residual_norms(), o.dt()))
for a, b in zip(out[:2], out[2:]):
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
print("bitwise")
''' % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       env={**os.environ, "OMP_NUM_THREADS": "4"}, timeout=300)
    assert r.returncode == 0 and "bitwise" in r.stdout, r.stdout + r.stderr
