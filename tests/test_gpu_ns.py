"""Navier-Stokes mode on the GPU vs the oracle (Eq. 2
viscous flux; readings N-R1..N-R6).  Same gates as the
Euler path: per conserved variable e_k <= 1e-12 after 1 step; residual-norm
histories 1e-10; dt 1e-13; loopback decompositions bitwise equal to one
block (ghost gradients at cuts are the neighbour's own, N-R1)."""
import numpy as np
import pytest

from paper_2305_18057_b200 import inputs as I
from parity_util import dt_error, norm_error, state_error

pytestmark = pytest.mark.gpu

NOSLIP_S = (I.BC_INFLOW, I.BC_OUTFLOW, I.BC_NOSLIP_WALL, I.BC_SLIP_WALL)


@pytest.fixture(scope="module")
def sfv_mod():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2305_18057_b200 import sfv
    sfv.lib()
    return sfv


def _pair(sfv_mod, oracle_mod, cfg, X, Y, U0, steps, **kw):
    g = sfv_mod.Solver(cfg, X, Y, **kw)
    g.set_state(U0); g.step(steps); g.sync()
    o = oracle_mod.Oracle(cfg, X, Y)
    o.set_state(U0); o.step(steps)
    return g, o


@pytest.mark.parametrize("steps,tol", [(1, 1e-12), (100, 1e-10)])
@pytest.mark.parametrize("mu", [0.02, 0.2])
def test_ns_parity(sfv_mod, oracle_mod, steps, tol, mu):
    ni, nj = 64, 32
    X, Y = I.ramp_nodes(ni, nj, 5.0)  # (the impulsive Mach-4 start over a steeper no-slip ramp is not stable)
    cfg = I.default_config(ni, nj, viscous=1, mu=mu, bc=NOSLIP_S)
    U0 = I.perturbed_state(ni, nj, 21)
    g, o = _pair(sfv_mod, oracle_mod, cfg, X, Y, U0, steps)
    e = state_error(g.get_state(), o.get_state())
    assert np.all(e <= tol), e
    assert norm_error(g.residual_norms(), o.residual_norms()) <= 1e-10
    assert dt_error(g.dt(), o.dt()) <= 1e-13


@pytest.mark.parametrize("mu", [0.02, 0.2])
def test_ns_parity_1000_steps(sfv_mod, oracle_mod, mu):
    """The north star's 1000-step gate (1e-9 per conserved variable) in
    Navier-Stokes mode, no-slip ramp wall, next to the oracle's own 1-ulp
    sensitivity: the gate is max(1e-9, 5 x sensitivity) (DESIGN.md A-R30)."""
    ni, nj = 64, 32
    X, Y = I.ramp_nodes(ni, nj, 5.0)
    cfg = I.default_config(ni, nj, viscous=1, mu=mu, bc=NOSLIP_S)
    U0 = I.perturbed_state(ni, nj, 21)
    g, o = _pair(sfv_mod, oracle_mod, cfg, X, Y, U0, 1000)
    U1 = U0.copy(); U1[..., 0] = np.nextafter(U1[..., 0], np.inf)
    s = oracle_mod.Oracle(cfg, X, Y); s.set_state(U1); s.step(1000)
    Uo = o.get_state()
    sens = state_error(s.get_state(), Uo).max()
    nsens = norm_error(s.residual_norms(), o.residual_norms())
    e = state_error(g.get_state(), Uo).max()
    assert e <= max(1e-9, 5.0 * sens), (e, sens)
    assert norm_error(g.residual_norms(), o.residual_norms()) <= max(1e-10, 5.0 * nsens)
    assert dt_error(g.dt(), o.dt()) <= max(1e-13, 5.0 * dt_error(s.dt(), o.dt()))


@pytest.mark.parametrize("rk", [I.RK2_HEUN, I.RK4_JAMESON])
def test_ns_tableaus(sfv_mod, oracle_mod, rk):
    ni, nj = 48, 40
    X, Y = I.ramp_nodes(ni, nj, 5.0)
    cfg = I.default_config(ni, nj, rk=rk, viscous=1, mu=0.3,
                           bc=(I.BC_INFLOW, I.BC_OUTFLOW, I.BC_NOSLIP_WALL, I.BC_NOSLIP_WALL))
    U0 = I.perturbed_state(ni, nj, 5)
    g, o = _pair(sfv_mod, oracle_mod, cfg, X, Y, U0, 10)
    assert np.all(state_error(g.get_state(), o.get_state()) <= 1e-11)


@pytest.mark.parametrize("px,py", [(2, 1), (1, 3), (2, 2), (3, 2)])
def test_ns_loopback_bitwise(sfv_mod, oracle_mod, px, py):
    ni, nj = 90, 70
    X, Y = I.ramp_nodes(ni, nj, 5.0)
    cfg = I.default_config(ni, nj, viscous=1, mu=0.2, bc=NOSLIP_S)
    U0 = I.perturbed_state(ni, nj, 8)
    g1 = sfv_mod.Solver(cfg, X, Y); g1.set_state(U0); g1.step(20); g1.sync()
    gp = sfv_mod.Solver(cfg, X, Y, px=px, py=py); gp.set_state(U0); gp.step(20); gp.sync()
    np.testing.assert_array_equal(gp.get_state(), g1.get_state())
    np.testing.assert_array_equal(gp.dt(), g1.dt())
    o = oracle_mod.Oracle(cfg, X, Y); o.set_state(U0); o.step(20)
    assert np.all(state_error(gp.get_state(), o.get_state()) <= 1e-11)


@pytest.mark.parametrize("px,py,rk", [(2, 1, 0), (1, 3, 0), (2, 2, 0), (3, 2, 1), (2, 2, 2)])
def test_ns_peer_loopback_bitwise(sfv_mod, oracle_mod, px, py, rk):
    """Navier-Stokes with device-initiated halos (SFV_HALO_PEER): the stage
    kernels store the state edge layers, grad_kernel the edge gradients into
    the neighbour block's frames and signal; visc_kernel's edge CTAs wait.
    Bit copies, so bitwise equal to one block."""
    ni, nj, steps = 90, 70, 20
    X, Y = I.ramp_nodes(ni, nj, 5.0)
    cfg = I.default_config(ni, nj, viscous=1, mu=0.2, bc=NOSLIP_S, rk=rk)
    U0 = I.perturbed_state(ni, nj, 8)
    g1 = sfv_mod.Solver(cfg, X, Y); g1.set_state(U0); g1.step(steps); g1.sync()
    gp = sfv_mod.Solver(cfg, X, Y, px=px, py=py)
    gp.enable_peer_halo()
    gp.set_state(U0); gp.step(steps); gp.sync()
    np.testing.assert_array_equal(gp.get_state(), g1.get_state())
    np.testing.assert_array_equal(gp.dt(), g1.dt())
    o = oracle_mod.Oracle(cfg, X, Y); o.set_state(U0); o.step(steps)
    assert np.all(state_error(gp.get_state(), o.get_state()) <= 1e-11)


def test_ns_peer_then_copy_mode(sfv_mod):
    """Switching the halo mode back and forth keeps the NS results bitwise."""
    ni, nj = 64, 40
    X, Y = I.ramp_nodes(ni, nj, 5.0)
    cfg = I.default_config(ni, nj, viscous=1, mu=0.1, bc=NOSLIP_S)
    U0 = I.perturbed_state(ni, nj, 4)
    g = sfv_mod.Solver(cfg, X, Y, px=2, py=2)
    g.enable_peer_halo(); g.set_state(U0); g.step(10); g.sync()
    Up = g.get_state()
    g.set_halo_mode(sfv_mod.HALO_COPY); g.set_state(U0); g.step(10); g.sync()
    np.testing.assert_array_equal(g.get_state(), Up)


def test_ns_operator_matches_oracle(sfv_mod, oracle_mod):
    """The GPU's Green-Gauss gradients and viscous residual sum_f F_v . n A of
    a stage input (Heun stage 2 input W2, read back through
    sfv_debug_block_buffer) equal the oracle's on the same state:
    gradients to 1e-13, R_v to 1e-11 of its maximum."""
    import os
    ni, nj = 64, 32
    X, Y = I.ramp_nodes(ni, nj, 15.0)
    cfg = I.default_config(ni, nj, viscous=1, mu=0.05, rk=I.RK2_HEUN, dt_fixed=1e-6, bc=NOSLIP_S)
    g = sfv_mod.Solver(cfg, X, Y)
    os.environ["SFV_NS_FUSED"] = "0"  # two-kernel path: the gradients go through global memory (readable)
    try:
        g.set_state(I.perturbed_state(ni, nj, 21)); g.step(1); g.sync()
    finally:
        del os.environ["SFV_NS_FUSED"]
    W2 = np.transpose(g.block_buffer(0, 1)[2:-2, :, 2:-2], (2, 0, 1)).copy()
    rv = np.transpose(g.block_buffer(0, -1)[2:-2, :, 2:-2], (2, 0, 1))
    G = np.transpose(g.block_buffer(0, -2)[1:-1, :, 1:-1], (2, 0, 1))
    o = oracle_mod.Oracle(cfg, X, Y)
    Rv = -(o.residual(W2) - oracle_mod.Oracle(dict(cfg, mu=0.0), X, Y).residual(W2))
    Go = o.gradients(W2)
    assert np.max(np.abs(G - Go)) <= 1e-13 * np.max(np.abs(Go))
    assert np.max(np.abs(rv - Rv)) <= 1e-11 * np.max(np.abs(Rv))


@pytest.mark.parametrize("ni,nj,rows", [(70, 45, "32"), (70, 45, "5"), (131, 61, "32"), (40, 90, "7")])
def test_ns_fused_equals_two_kernel_path(sfv_mod, monkeypatch, ni, nj, rows):
    """The fused kernels for blocks without connected edges -- the row-marching
    one (default; segments of SFV_NS_MROWS rows, strips of 28 columns: ragged
    strips and segments) and the tile one -- and the gradient + viscous kernel
    pair give bitwise the same evolution."""
    X, Y = I.ramp_nodes(ni, nj, 5.0)
    cfg = I.default_config(ni, nj, viscous=1, mu=0.1, bc=NOSLIP_S)
    U0 = I.perturbed_state(ni, nj, 17)
    out = []
    monkeypatch.setenv("SFV_NS_MROWS", rows)
    for fused, march in (("1", "1"), ("1", "0"), ("0", "1")):
        monkeypatch.setenv("SFV_NS_FUSED", fused)
        monkeypatch.setenv("SFV_NS_MARCH", march)
        g = sfv_mod.Solver(cfg, X, Y); g.set_state(U0); g.step(15); g.sync()
        out.append(g.get_state())
    np.testing.assert_array_equal(out[0], out[2])
    np.testing.assert_array_equal(out[1], out[2])
