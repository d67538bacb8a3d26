"""Pins of the oracle's Navier-Stokes pieces (PAPER.md:73-79
Eq. 2 viscous flux; readings N-R1..N-R5 in DESIGN.md).

Each check is fixed by mathematics, not by re-typing the oracle's formula:
Newtonian shear and dilatation values, rotation covariance of the stress
vector, Green-Gauss exactness for linear fields on parallelogram cells, the
closed-form residual of a linear shear flow, the no-slip ghost rule and
decomposition invariance."""
import numpy as np
import pytest

from paper_2305_18057_b200 import inputs as I


def test_viscous_flux_zero_and_shear(oracle_mod):
    F = oracle_mod.viscous_flux(np.zeros(6), 3.0, -2.0, 0.6, 0.8, 1.7, 2.5)
    assert np.all(F == 0.0)
    # pure shear du/dy = 1, mu = 1, n = (0, 1): tau_yx = 1 (SPEC.md:206 example);
    # energy: u tau_xy with face u = 2
    F = oracle_mod.viscous_flux([0, 1, 0, 0, 0, 0], 2.0, 0.0, 0.0, 1.0, 1.0, 0.0)
    np.testing.assert_allclose(F, [0.0, 1.0, 0.0, 2.0], rtol=0, atol=1e-15)
    # pure dilatation u_x = v_y = a: Stokes' hypothesis gives tau_xx = tau_yy = 2 mu a / 3
    a, mu = 0.3, 2.0
    F = oracle_mod.viscous_flux([a, 0, 0, a, 0, 0], 0.0, 0.0, 1.0, 0.0, mu, 0.0)
    np.testing.assert_allclose(F, [0.0, 2.0 * mu * a / 3.0, 0.0, 0.0], rtol=1e-15)
    # heat conduction only: k dT/dn
    F = oracle_mod.viscous_flux([0, 0, 0, 0, 4.0, -1.0], 0.0, 0.0, 0.6, 0.8, 1.0, 3.0)
    np.testing.assert_allclose(F, [0.0, 0.0, 0.0, 3.0 * (4.0 * 0.6 - 1.0 * 0.8)], rtol=1e-15)


@pytest.mark.parametrize("theta", [0.3, 1.1, 2.5])
def test_viscous_flux_rotation_covariant(oracle_mod, theta):
    """Rotating the frame rotates the stress vector and leaves the energy flux
    invariant: catches a transposed gradient (u_y vs v_x) or a wrong sign."""
    rng = np.random.default_rng(int(theta * 10))
    L = rng.normal(size=(2, 2))           # [[u_x, u_y], [v_x, v_y]]
    gT = rng.normal(size=2)
    vel = rng.normal(size=2)
    n = np.array([np.cos(0.7), np.sin(0.7)])
    Q = np.array([[np.cos(theta), -np.sin(theta)], [np.sin(theta), np.cos(theta)]])
    mu, k = 1.3, 0.9
    F = oracle_mod.viscous_flux([L[0, 0], L[0, 1], L[1, 0], L[1, 1], gT[0], gT[1]], vel[0], vel[1], n[0], n[1], mu, k)
    L2, g2, v2, n2 = Q @ L @ Q.T, Q @ gT, Q @ vel, Q @ n
    F2 = oracle_mod.viscous_flux([L2[0, 0], L2[0, 1], L2[1, 0], L2[1, 1], g2[0], g2[1]], v2[0], v2[1], n2[0], n2[1],
                                 mu, k)
    np.testing.assert_allclose(F2[1:3], Q @ F[1:3], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(F2[3], F[3], rtol=1e-12)


def _linear_state(Xc, Yc, gas_R=I.R_GAS, gamma=I.GAMMA):
    """rho const, u, v, p linear in (x, y): T = p / (rho R) linear too."""
    rho = 0.8
    u = 100.0 + 30.0 * Xc - 20.0 * Yc
    v = -5.0 + 10.0 * Xc + 40.0 * Yc
    p = 1.0e5 + 2.0e3 * Xc + 5.0e3 * Yc
    E = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v)
    U = np.stack([np.full_like(u, rho), rho * u, rho * v, E], axis=-1)
    return U, np.array([30.0, -20.0, 10.0, 40.0, 2.0e3 / (rho * gas_R), 5.0e3 / (rho * gas_R)])


def _centroids(X, Y):
    return 0.25 * (X[:-1, :-1] + X[1:, :-1] + X[:-1, 1:] + X[1:, 1:]), \
        0.25 * (Y[:-1, :-1] + Y[1:, :-1] + Y[:-1, 1:] + Y[1:, 1:])


@pytest.mark.parametrize("shear", [0.0, 0.35])
def test_green_gauss_exact_for_linear_fields(oracle_mod, shear):
    """Green-Gauss with arithmetic face averaging is exact for linear fields
    when face midpoints are the midpoints of the adjacent cell centres:
    uniform Cartesian cells and uniformly sheared parallelograms."""
    ni, nj = 12, 10
    x = np.linspace(0.0, 1.2, ni + 1)
    y = np.linspace(0.0, 0.8, nj + 1)
    X, Y = np.meshgrid(x, y)
    X = X + shear * Y
    Xc, Yc = _centroids(X, Y)
    U, g = _linear_state(Xc, Yc)
    cfg = I.default_config(ni, nj, viscous=1, mu=1.0, bc=(1, 1, 1, 1))
    G = oracle_mod.Oracle(cfg, X, Y).gradients(U)
    inner = G[1:-1, 1:-1]
    # (u, v, T) are exactly linear in the centroid coordinates here
    np.testing.assert_allclose(inner, np.broadcast_to(g, inner.shape), rtol=1e-9, atol=1e-9)


def test_linear_shear_residual_closed_form(oracle_mod):
    """u = s y, v = 0, rho and p uniform on a uniform Cartesian grid: the
    viscous stress is uniform (its momentum flux telescopes to 0 over a
    closed cell) and the viscous energy flux u tau_xy has divergence
    mu s^2, so R_NS - R_Euler = (0, 0, 0, -mu s^2 V) in every interior cell
    (the inviscid parts are the same computation; conserved-variable MUSCL
    of the quadratic E makes them nonzero, so they are subtracted)."""
    ni, nj, s, mu = 10, 12, 80.0, 0.5
    X, Y = np.meshgrid(np.linspace(0.0, 1.0, ni + 1), np.linspace(0.0, 1.2, nj + 1))
    Xc, Yc = _centroids(X, Y)
    rho, p = 0.5, 4.0e4
    u = s * Yc
    E = p / (I.GAMMA - 1.0) + 0.5 * rho * u * u
    U = np.stack([np.full_like(u, rho), rho * u, np.zeros_like(u), E], axis=-1)
    cfg = I.default_config(ni, nj, viscous=1, mu=mu, bc=(1, 1, 1, 1))
    R = oracle_mod.Oracle(cfg, X, Y).residual(U) - \
        oracle_mod.Oracle(I.default_config(ni, nj, bc=(1, 1, 1, 1)), X, Y).residual(U)
    V = (1.0 / ni) * (1.2 / nj)
    inner = R[2:-2, 2:-2]
    scale = mu * s * s * V
    np.testing.assert_allclose(inner[..., 3], -scale, rtol=1e-9)
    assert np.max(np.abs(inner[..., :3])) < 1e-9 * scale


def test_noslip_ghosts(oracle_mod):
    ni, nj = 8, 6
    X, Y = I.ramp_nodes(ni, nj, 15.0)
    cfg = I.default_config(ni, nj, viscous=1, mu=0.1, bc=(3, 1, 3, 2))
    U = I.perturbed_state(ni, nj, 4)
    F = oracle_mod.Oracle(cfg, X, Y).ghost_frame(U)  # [nj+4, ni+4, 4], index (j+2, i+2)
    for m in range(2):
        w = U[:, m]                         # W wall: ghost layer m mirrors interior layer m
        np.testing.assert_array_equal(F[2:-2, 1 - m], w * np.array([1, -1, -1, 1]))
        s_ = U[m, :]                        # S wall
        np.testing.assert_array_equal(F[1 - m, 2:-2], s_ * np.array([1, -1, -1, 1]))


def test_noslip_requires_viscous(oracle_mod):
    X, Y = I.ramp_nodes(8, 6, 15.0)
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.Oracle(I.default_config(8, 6, bc=(0, 1, 3, 2)), X, Y)


@pytest.mark.parametrize("px,py", [(2, 1), (1, 3), (2, 2)])
def test_ns_decomposition_invariance(oracle_mod, px, py):
    """Ghost gradients at cuts are the neighbour's own cell gradients, so the
    partitioned NS oracle is bitwise the single block."""
    ni, nj = 30, 18
    X, Y = I.ramp_nodes(ni, nj, 20.0)
    cfg = I.default_config(ni, nj, viscous=1, mu=0.5, bc=(0, 1, 3, 2))
    U0 = I.perturbed_state(ni, nj, 6)
    o1 = oracle_mod.Oracle(cfg, X, Y); o1.set_state(U0); o1.step(6)
    op = oracle_mod.Oracle(cfg, X, Y); op.partition(px, py); op.set_state(U0); op.step(6)
    np.testing.assert_array_equal(op.get_state(), o1.get_state())


def test_ns_reduces_to_euler_at_zero_viscosity(oracle_mod):
    ni, nj = 24, 12
    X, Y = I.ramp_nodes(ni, nj, 15.0)
    U0 = I.perturbed_state(ni, nj, 2)
    oe = oracle_mod.Oracle(I.default_config(ni, nj), X, Y); oe.set_state(U0); oe.step(4)
    on = oracle_mod.Oracle(I.default_config(ni, nj, viscous=1, mu=0.0), X, Y); on.set_state(U0); on.step(4)
    np.testing.assert_array_equal(on.get_state(), oe.get_state())


def test_heat_conduction_closed_form(oracle_mod):
    """Fluid at rest, rho uniform, T = T0 + a x^2 on a uniform Cartesian grid:
    central Green-Gauss gradients are exact for the quadratic at cell centres,
    their face averages exact at face midpoints, so the face heat flux is
    k 2 a x_f and R_NS - R_Euler = (0, 0, 0, -2 a k V) with
    k = mu c_p / Pr, c_p = gamma R / (gamma - 1) (reading N-R5)."""
    ni, nj, mu, Pr, a = 12, 8, 0.7, 0.72, 300.0
    X, Y = np.meshgrid(np.linspace(0.0, 1.2, ni + 1), np.linspace(0.0, 0.8, nj + 1))
    Xc, _ = _centroids(X, Y)
    rho = 0.4
    T = 250.0 + a * Xc * Xc
    p = rho * I.R_GAS * T
    U = np.stack([np.full_like(T, rho), np.zeros_like(T), np.zeros_like(T), p / (I.GAMMA - 1.0)], axis=-1)
    cfg = I.default_config(ni, nj, viscous=1, mu=mu, prandtl=Pr, bc=(1, 1, 1, 1))
    R = oracle_mod.Oracle(cfg, X, Y).residual(U) - \
        oracle_mod.Oracle(I.default_config(ni, nj, bc=(1, 1, 1, 1)), X, Y).residual(U)
    k = mu * (I.GAMMA * I.R_GAS / (I.GAMMA - 1.0)) / Pr
    V = 0.1 * 0.1
    inner = R[2:-2, 2:-2]
    np.testing.assert_allclose(inner[..., 3], -2.0 * a * k * V, rtol=1e-9)
    assert np.max(np.abs(inner[..., :3])) < 1e-9 * 2.0 * a * k * V


def test_viscous_time_step_closed_form(oracle_mod):
    """Gas at rest on a uniform square grid of spacing d: the 4 faces give
    sigma_c = 4 a d and the viscous spectral radius (reading N-R6)
    sigma_v = 4 max(4/3, gamma) mu / (rho Pr) (d^2 + d^2) / d^2, so
    dt = CFL d^2 / (sigma_c + sigma_v) exactly (one step records dt_0)."""
    n, d, mu, Pr, rho, p = 10, 0.01, 3.0e-3, 0.72, 0.6, 5.0e4
    X, Y = np.meshgrid(np.arange(n + 1) * d, np.arange(n + 1) * d)
    U = np.zeros((n, n, 4)); U[..., 0] = rho; U[..., 3] = p / (I.GAMMA - 1.0)
    cfg = I.default_config(n, n, viscous=1, mu=mu, prandtl=Pr, bc=(1, 1, 1, 1), cfl=0.8)
    o = oracle_mod.Oracle(cfg, X, Y); o.set_state(U); o.step(1)
    a = np.sqrt(I.GAMMA * p / rho)
    sv = 4.0 * max(4.0 / 3.0, I.GAMMA) * mu / (rho * Pr) * 2.0
    np.testing.assert_allclose(o.dt()[0], 0.8 * d * d / (4.0 * a * d + sv), rtol=1e-14)
    oe = oracle_mod.Oracle(I.default_config(n, n, bc=(1, 1, 1, 1), cfl=0.8), X, Y); oe.set_state(U); oe.step(1)
    np.testing.assert_allclose(oe.dt()[0], 0.8 * d * d / (4.0 * a * d), rtol=1e-14)
