"""Independent pin of the oracle's Roe dissipation and Harten entropy fix
(reading A-R1/A-R2; "Roe flux with Harten entropy fix", SPEC.md:254;
Eq. 2 normal flux at PAPER.md:64-72).

The reference here shares nothing with `orc_roe_flux`'s eigenvector algebra:
  * the Roe matrix A~ is the Jacobian dF_n/dU of the analytic Eq. 2 normal
    flux, taken by complex-step differentiation at the Roe-averaged state
    (sqrt(rho) weighting); its defining property A~ dU = dF (Roe 1981) is
    asserted, which pins the averaging itself;
  * |A~| = R |Lambda| R^-1 is built from the eigenvalues of that matrix
    (`numpy.linalg.eigvals`) and its spectral projectors (Sylvester's formula;
    `test_spectral_projectors` checks them against `numpy.linalg.eig`);
  * Harten's fix (reading A-R2: delta_H = max(eps_H a~, 1e-12), applied to the
    two acoustic eigenvalues only) replaces |lambda| < delta_H by
    (lambda^2 + delta_H^2) / (2 delta_H);
  * F = (F_L + F_R)/2 - |A~| dU / 2.
The faces are chosen so the fix is active (sonic and transonic faces, and
faces with |V~n| < delta_H where a fix wrongly applied to the convective wave
would show).  `test_pins_discriminate_the_mutations` shows that each of the
plausible mis-readings named in VERDICT r1 (missing factor 2, fix applied to
lambda_2, delta_H = eps (|V~n| + a~)) moves F far outside the tolerance on
these faces, so none of them could pass.
"""
import math

import numpy as np
import pytest

from paper_2305_18057_b200 import inputs as I

GAMMA = 1.4
EPS_H = 0.1


def flux_n(U, nx, ny, gamma=GAMMA):
    """Eq. 2 inviscid flux through a face of unit normal n;
    works on complex U for the complex-step Jacobian."""
    rho, mx, my, E = U
    u, v = mx / rho, my / rho
    p = (gamma - 1.0) * (E - 0.5 * rho * (u * u + v * v))
    Vn = u * nx + v * ny
    return np.array([rho * Vn, mx * Vn + p * nx, my * Vn + p * ny, (E + p) * Vn])


def jacobian(U, nx, ny):
    h = 1e-40
    J = np.empty((4, 4))
    for k in range(4):
        Uc = np.array(U, dtype=complex)
        Uc[k] += 1j * h
        J[:, k] = flux_n(Uc, nx, ny).imag / h
    return J


def roe_state(UL, UR, gamma=GAMMA):
    """Conserved state whose (u, v, H) are the sqrt(rho)-weighted Roe averages."""
    def prim(U):
        rho = U[0]; u = U[1] / rho; v = U[2] / rho
        p = (gamma - 1.0) * (U[3] - 0.5 * rho * (u * u + v * v))
        return rho, u, v, (U[3] + p) / rho
    rL, uL, vL, HL = prim(UL)
    rR, uR, vR, HR = prim(UR)
    sL, sR = math.sqrt(rL), math.sqrt(rR)
    u = (sL * uL + sR * uR) / (sL + sR)
    v = (sL * vL + sR * vR) / (sL + sR)
    H = (sL * HL + sR * HR) / (sL + sR)
    rho = sL * sR
    p = (gamma - 1.0) / gamma * rho * (H - 0.5 * (u * u + v * v))
    return I.conserved_from_primitive([rho, u, v, p])


def reference_flux(UL, UR, nx, ny, eps_h=EPS_H, variant="A-R2"):
    """F = (F_L+F_R)/2 - R|Lambda|R^-1 dU/2 with Harten's fix; `variant` selects
    a deliberate mis-reading (used only to show the pins discriminate)."""
    A = jacobian(roe_state(UL, UR), nx, ny)
    ev = np.sort(np.linalg.eigvals(A).real)
    l1, l4 = ev[0], ev[3]                        # the simple acoustic pair V~n -/+ a~
    l2 = 0.5 * (l1 + l4)                         # the double convective eigenvalue V~n
    a_t = 0.5 * (l4 - l1)
    dH = max(eps_h * a_t, 1e-12)
    if variant == "dH_vn":
        dH = max(eps_h * (abs(l2) + a_t), 1e-12)

    def g(lam, acoustic):
        ab = abs(lam)
        if (acoustic or variant == "all_waves") and ab < dH:
            ab = (ab * ab + dH * dH) / (dH if variant == "no_half" else 2.0 * dH)
        return ab
    # |A~| = R |Lambda| R^-1 as the spectral projectors of the diagonalizable A~
    # (Sylvester: P_i = prod_{j != i} (A - l_j I) / (l_i - l_j) over the distinct
    # eigenvalues), which stays well conditioned where eig's eigenvector basis
    # of the double eigenvalue does not
    Id = np.eye(4)
    lams = (l1, l2, l4)
    P = []
    for i, li in enumerate(lams):
        M = Id.copy()
        for j, lj in enumerate(lams):
            if j != i:
                M = M @ (A - lj * Id) / (li - lj)
        P.append(M)
    absA = g(l1, True) * P[0] + g(l2, False) * P[1] + g(l4, True) * P[2]
    D = absA @ (np.asarray(UR) - np.asarray(UL))
    return 0.5 * (flux_n(UL, nx, ny) + flux_n(UR, nx, ny)) - 0.5 * D, np.array([l1, l2, l2, l4]), dH


def scale(UL, UR, nx, ny):
    return max(np.max(np.abs(flux_n(UL, nx, ny))), np.max(np.abs(flux_n(UR, nx, ny))))


def faces():
    """(U_L, U_R, n) with the entropy fix active on an acoustic wave, or a
    convective eigenvalue below delta_H; deterministic."""
    rng = np.random.default_rng(20230518)
    out = []
    for kind in ("sonic", "transonic", "slow", "subsonic"):
        for _ in range(40):
            th = rng.uniform(0, 2 * math.pi)
            n = (math.cos(th), math.sin(th)); t = (-n[1], n[0])
            rho = rng.uniform(0.5, 2.0); p = rng.uniform(0.5, 2.0)
            a = math.sqrt(GAMMA * p / rho)
            if kind == "sonic":        # V_n = a on both sides up to 1 %: lambda_1 ~ 0
                mL, mR = 1.0 + 0.01 * rng.uniform(-1, 1), 1.0 + 0.01 * rng.uniform(-1, 1)
            elif kind == "transonic":  # expansion through the sonic point
                mL, mR = rng.uniform(0.9, 0.98), rng.uniform(1.02, 1.1)
            elif kind == "slow":       # |V~n| << delta_H: only the convective wave is slow
                mL, mR = 0.02 * rng.uniform(-1, 1), 0.02 * rng.uniform(-1, 1)
            else:
                mL, mR = rng.uniform(-0.8, 0.8), rng.uniform(-0.8, 0.8)
            wt = rng.uniform(-1, 1)
            sgn = 1.0 if rng.uniform() < 0.5 else -1.0   # left- and right-running sonic points
            def st(m, drho, dp):
                r = rho * (1 + drho); pp = p * (1 + dp)
                aa = math.sqrt(GAMMA * pp / r)
                vn = sgn * m * aa; vt = wt * aa
                return I.conserved_from_primitive([r, vn * n[0] + vt * t[0], vn * n[1] + vt * t[1], pp])
            d = 0.03 if kind != "subsonic" else 0.2
            UL = st(mL, d * rng.uniform(-1, 1), d * rng.uniform(-1, 1))
            UR = st(mR, d * rng.uniform(-1, 1), d * rng.uniform(-1, 1))
            out.append((kind, UL, UR, n))
    return out


FACES = faces()


def test_roe_matrix_property():
    """A~ (U_R - U_L) = F_R - F_L: the averaged state really is Roe's."""
    for _, UL, UR, n in FACES:
        A = jacobian(roe_state(UL, UR), *n)
        dF = flux_n(UR, *n) - flux_n(UL, *n)
        assert np.max(np.abs(A @ (UR - UL) - dF)) <= 1e-13 * scale(UL, UR, *n)


def test_spectral_projectors():
    """The projectors reproduce A~ = sum l_i P_i, sum P_i = I, and the
    eigenvalues agree with numpy.linalg.eig (V~n -/+ a~ and a double V~n)."""
    for _, UL, UR, n in FACES[::7]:
        A = jacobian(roe_state(UL, UR), *n)
        lam_eig = np.sort(np.linalg.eig(A)[0].real)
        _, lam, _ = reference_flux(UL, UR, *n)
        assert np.max(np.abs(lam - lam_eig)) < 1e-7 * np.max(np.abs(lam_eig))  # (double root: sqrt(eps))
        Ut = roe_state(UL, UR)
        rho, u, v = Ut[0], Ut[1] / Ut[0], Ut[2] / Ut[0]
        p = (GAMMA - 1) * (Ut[3] - 0.5 * rho * (u * u + v * v))
        a = math.sqrt(GAMMA * p / rho); vn = u * n[0] + v * n[1]
        assert abs(lam[0] - (vn - a)) < 1e-13 * a and abs(lam[3] - (vn + a)) < 1e-13 * a
        # Sylvester projectors: sum P_i = I and sum l_i P_i = A~ (diagonalizable)
        Id = np.eye(4); ls = (lam[0], lam[1], lam[3]); P = []
        for i, li in enumerate(ls):
            M = Id.copy()
            for j, lj in enumerate(ls):
                if j != i:
                    M = M @ (A - lj * Id) / (li - lj)
            P.append(M)
        assert np.max(np.abs(sum(P) - Id)) < 1e-11
        assert np.max(np.abs(sum(l * M for l, M in zip(ls, P)) - A)) < 1e-11 * np.max(np.abs(A))


def test_fix_is_active_on_the_chosen_faces():
    active = {"sonic": 0, "transonic": 0, "slow": 0}
    for kind, UL, UR, n in FACES:
        _, lam, dH = reference_flux(UL, UR, *n)
        ac = (abs(lam.min()) < dH) or (abs(lam.max()) < dH)
        conv = np.sort(np.abs(lam))[:2].max() < dH and not ac
        if kind in ("sonic", "transonic"):
            active[kind] += ac
        if kind == "slow":
            active[kind] += conv
    assert active["sonic"] >= 30 and active["transonic"] >= 20 and active["slow"] >= 30, active


@pytest.mark.parametrize("kind", ["sonic", "transonic", "slow", "subsonic"])
def test_oracle_roe_equals_eigendecomposition(oracle_mod, kind):
    worst = 0.0
    for k, UL, UR, n in FACES:
        if k != kind:
            continue
        F = oracle_mod.roe_flux(UL, UR, *n, gamma=GAMMA, harten_eps=EPS_H)
        Fr, _, _ = reference_flux(UL, UR, *n)
        worst = max(worst, np.max(np.abs(F - Fr)) / scale(UL, UR, *n))
    assert worst < 1e-13, worst


def test_exactly_sonic_lambda1_is_half_delta(oracle_mod):
    """U_L = U_R with V_n = a: dU = 0 so F = F(U) whatever the fix; perturb one
    side along the acoustic eigenvector r_1 only: then D = |lambda_1|~ alpha_1 r_1
    with |lambda_1|~ = delta_H/2 exactly at lambda_1 = 0 (A-R2)."""
    rho, p = 1.3, 0.9
    a = math.sqrt(GAMMA * p / rho)
    n = (0.6, 0.8)
    U = I.conserved_from_primitive([rho, a * n[0], a * n[1], p])
    A = jacobian(U, *n)
    lam, R = np.linalg.eig(A)
    k1 = int(np.argmin(lam.real))
    assert abs(lam.real[k1]) < 1e-13 * a
    r1 = R[:, k1].real
    eps = 1e-7 * rho / max(abs(r1[0]), 1e-300)
    UL, UR = U - 0.5 * eps * r1, U + 0.5 * eps * r1
    F = oracle_mod.roe_flux(UL, UR, *n, gamma=GAMMA, harten_eps=EPS_H)
    Fc = 0.5 * (flux_n(UL, *n) + flux_n(UR, *n))
    D = 2.0 * (Fc - F)                       # = lambda~ alpha_1 r_1 with alpha_1 r_1 = dU
    dH = EPS_H * a
    lam_eff = D @ (UR - UL) / ((UR - UL) @ (UR - UL))
    # Roe average of U -/+ eps r1/2 moves lambda_1 by O(eps): relative 1e-6 is the pin
    assert abs(lam_eff - dH / 2.0) < 1e-6 * dH, (lam_eff, dH / 2)


def test_flux_continuous_across_delta_h(oracle_mod):
    """(lambda^2 + d^2)/(2d) meets |lambda| at lambda = d: F is continuous as
    lambda_1 crosses delta_H (a factor-2 slip would jump by ~d |alpha_1 r_1|)."""
    rho, p = 1.0, 1.0
    a = math.sqrt(GAMMA * p / rho)
    n = (1.0, 0.0)
    def F_at(m):
        UL = I.conserved_from_primitive([rho, m * a, 0.0, p])
        UR = I.conserved_from_primitive([rho * 1.02, m * a * 1.001, 0.0, p * 1.03])
        return oracle_mod.roe_flux(UL, UR, *n, gamma=GAMMA, harten_eps=EPS_H), UL, UR
    # find m with lambda_1 = V~n - a~ crossing +delta_H by bisection on the reference
    lo, hi = 1.0, 1.3
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        _, UL, UR = F_at(mid)
        _, lam, dH = reference_flux(UL, UR, *n)
        if abs(lam.min()) < dH:
            lo = mid
        else:
            hi = mid
    Fa, UL, UR = F_at(lo)
    Fb, _, _ = F_at(hi)
    assert np.max(np.abs(Fa - Fb)) / scale(UL, UR, *n) < 1e-9


def test_pins_discriminate_the_mutations(oracle_mod):
    """Each mis-reading of A-R2 differs from the oracle by >> the 1e-13 gate on
    these faces, so a mutated oracle could not pass the equality test above."""
    for variant in ("no_half", "all_waves", "dH_vn"):
        worst = 0.0
        for kind, UL, UR, n in FACES:
            if kind == "subsonic":
                continue
            F = oracle_mod.roe_flux(UL, UR, *n, gamma=GAMMA, harten_eps=EPS_H)
            Fm, _, _ = reference_flux(UL, UR, *n, variant=variant)
            worst = max(worst, np.max(np.abs(F - Fm)) / scale(UL, UR, *n))
        assert worst > 1e-6, (variant, worst)
