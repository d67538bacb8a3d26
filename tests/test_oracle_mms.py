"""Order of accuracy of the oracle's spatial operator by the method of
manufactured solutions (PAPER.md:46-51 cites MMS verification of SENSEI;
SPEC.md:228-234 asks for observed order >= 1.8).

For a smooth manufactured field U*(x, y) the source is S = dF/dx + dG/dy of
the exact fluxes (and of the viscous fluxes in Navier-Stokes mode),
evaluated here by complex-step differentiation (exact to rounding, no
hand-derived formula to get wrong).  The truncation error of the discrete
operator, TE = R_h(U*)/V - S at the cell centres, must fall as h^2 on grid
refinement for a second-order finite-volume scheme (Eq. 5 with the MUSCL
extrapolation of Eq. 7): a dropped term, a wrong sign or a transposed
metric leaves an O(1) or O(h) error and fails the order check.  The fields
make every conserved variable (the reconstructed ones, reading A-R8)
monotone in x and y over the domain, so the limiter stays at 1 - O(h^2) and
does not clip extrema (a y-momentum extremum in x measured order 1.5)."""
import numpy as np
import pytest

from paper_2305_18057_b200 import inputs as I

G = I.GAMMA
# primitive fields f0 + f1 sin(kx x + ky y + phi): arguments stay in (-pi/2, pi/2)
FIELDS = {"rho": (1.0, 0.15, 0.9, 0.5, -0.7), "u": (800.0, 60.0, 0.6, -0.4, -0.3),
          "v": (150.0, 40.0, 0.5, 0.8, -0.4), "p": (1.0e5, 1.2e4, 0.7, 0.6, -0.6)}


def prim(x, y):
    return {k: f0 + f1 * np.sin(kx * x + ky * y + ph) for k, (f0, f1, kx, ky, ph) in FIELDS.items()}


def dprim(x, y):
    """analytic first derivatives (complex-safe)"""
    out = {}
    for k, (f0, f1, kx, ky, ph) in FIELDS.items():
        c = f1 * np.cos(kx * x + ky * y + ph)
        out[k] = (c * kx, c * ky)
    return out


def inviscid_fluxes(x, y):
    q = prim(x, y)
    r, u, v, p = q["rho"], q["u"], q["v"], q["p"]
    E = p / (G - 1.0) + 0.5 * r * (u * u + v * v)
    F = np.stack([r * u, r * u * u + p, r * u * v, u * (E + p)])
    Gf = np.stack([r * v, r * u * v, r * v * v + p, v * (E + p)])
    return F, Gf


def viscous_fluxes(x, y, mu, k, R):
    q, d = prim(x, y), dprim(x, y)
    r, u, v, p = q["rho"], q["u"], q["v"], q["p"]
    ux, uy = d["u"]; vx, vy = d["v"]
    # T = p / (rho R): dT = (dp rho - p drho) / (rho^2 R)
    Tx = (d["p"][0] * r - p * d["rho"][0]) / (r * r * R)
    Ty = (d["p"][1] * r - p * d["rho"][1]) / (r * r * R)
    lam = -2.0 * mu / 3.0
    txx = 2 * mu * ux + lam * (ux + vy); tyy = 2 * mu * vy + lam * (ux + vy); txy = mu * (uy + vx)
    zero = np.zeros_like(u)
    Fv = np.stack([zero, txx, txy, u * txx + v * txy + k * Tx])
    Gv = np.stack([zero, txy, tyy, u * txy + v * tyy + k * Ty])
    return Fv, Gv


def source(x, y, viscous=None):
    """S = d(F - Fv)/dx + d(G - Gv)/dy by complex step."""
    h = 1e-30
    Fx, _ = inviscid_fluxes(x + 1j * h, y + 0j)
    _, Gy = inviscid_fluxes(x + 0j, y + 1j * h)
    S = np.imag(Fx) / h + np.imag(Gy) / h
    if viscous is not None:
        Fvx, _ = viscous_fluxes(x + 1j * h, y + 0j, *viscous)
        _, Gvy = viscous_fluxes(x + 0j, y + 1j * h, *viscous)
        S = S - (np.imag(Fvx) / h + np.imag(Gvy) / h)
    return S


def conserved(x, y):
    q = prim(x, y)
    r, u, v, p = q["rho"], q["u"], q["v"], q["p"]
    E = p / (G - 1.0) + 0.5 * r * (u * u + v * v)
    return np.stack([r, r * u, r * v, E], axis=-1)


def grid(n, shear):
    x = np.linspace(0.0, 1.0, n + 1)
    X, Y = np.meshgrid(x, x)
    return X + shear * Y, Y


def truncation_error(oracle_mod, n, shear, viscous=None):
    X, Y = grid(n, shear)
    # centroids of the parallelogram cells
    Xc = 0.25 * (X[:-1, :-1] + X[1:, :-1] + X[:-1, 1:] + X[1:, 1:])
    Yc = 0.25 * (Y[:-1, :-1] + Y[1:, :-1] + Y[:-1, 1:] + Y[1:, 1:])
    kw = dict(bc=(I.BC_OUTFLOW,) * 4)
    if viscous is not None:
        kw.update(viscous=1, mu=viscous[0], prandtl=viscous[0] * G * viscous[2] / ((G - 1.0) * viscous[1]),
                  gas_R=viscous[2])
    cfg = I.default_config(n, n, **kw)
    R = oracle_mod.Oracle(cfg, X, Y).residual(conserved(Xc, Yc))
    V = (1.0 / n) ** 2
    S = np.moveaxis(source(Xc, Yc, viscous), 0, -1)
    TE = R / V - S
    m = n // 8  # away from the boundary ghosts (zeroth-order extrapolation)
    inner = TE[m:-m, m:-m]
    return np.sqrt(np.mean(inner ** 2, axis=(0, 1))) / np.max(np.abs(S), axis=(0, 1))


@pytest.mark.parametrize("shear", [0.0, 0.3])
def test_mms_euler_second_order(oracle_mod, shear):
    errs = [truncation_error(oracle_mod, n, shear) for n in (32, 64, 128)]
    orders = [np.log2(errs[k] / errs[k + 1]) for k in range(2)]
    for o in orders:
        assert np.all(o > 1.8), (orders, errs)
    assert np.all(errs[-1] < 1e-3), errs


def test_mms_navier_stokes_second_order(oracle_mod):
    mu, k, Rg = 50.0, 7.0e4, 287.0   # large enough that the viscous terms matter in S
    errs = [truncation_error(oracle_mod, n, 0.0, (mu, k, Rg)) for n in (32, 64, 128)]
    orders = [np.log2(errs[j] / errs[j + 1]) for j in range(2)]
    for o in orders:
        assert np.all(o[1:] > 1.8), (orders, errs)  # momentum and energy carry the viscous terms


def test_mms_detects_a_wrong_operator(oracle_mod):
    """The same study with the viscous terms left out of S must not converge:
    the check has teeth."""
    mu, k, Rg = 50.0, 7.0e4, 287.0

    def te_without(n):
        Xg, Yg = grid(n, 0.0)
        Xc = 0.25 * (Xg[:-1, :-1] + Xg[1:, :-1] + Xg[:-1, 1:] + Xg[1:, 1:])
        Yc = 0.25 * (Yg[:-1, :-1] + Yg[1:, :-1] + Yg[:-1, 1:] + Yg[1:, 1:])
        cfg = I.default_config(n, n, bc=(I.BC_OUTFLOW,) * 4, viscous=1, mu=mu,
                               prandtl=mu * G * Rg / ((G - 1.0) * k), gas_R=Rg)
        R = oracle_mod.Oracle(cfg, Xg, Yg).residual(conserved(Xc, Yc))
        TE = R * n * n - np.moveaxis(source(Xc, Yc, None), 0, -1)
        m = n // 8
        return np.sqrt(np.mean(TE[m:-m, m:-m] ** 2, axis=(0, 1)))
    e1, e2 = te_without(32), te_without(64)
    assert np.log2(e1[3] / e2[3]) < 0.5
