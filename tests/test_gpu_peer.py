"""Device-initiated halo exchange (SFV_HALO_PEER).

In peer mode the stage kernel's edge tasks store the new state's 2 edge
layers directly into the neighbour block's ghost frame and publish the stage
sequence number to the neighbour's inbound flag; the neighbour's edge tasks
wait on that flag before staging their ghosts.  No copy, NCCL call or extra
launch per stage.  The exchanged layers are bit copies, so every run must be
bitwise equal to the single-block run (same per-face arithmetic), for every
decomposition and tableau, and match the oracle (solutions
across partitionings agree to < 1e-12).

Loopback (one process, several blocks on one device) runs the identical
kernel code with the neighbours' own pointers; the two-process test maps the
neighbour's workspace through CUDA IPC exactly as ranks on different GPUs
do (here both on cuda:0, NCCL told the ranks are on different hosts, see
test_gpu_nccl.py)."""
import numpy as np
import pytest

from paper_2305_18057_b200 import inputs as I
from parity_util import dt_error, norm_error, state_error

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sfv_mod():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2305_18057_b200 import sfv
    sfv.lib()
    return sfv


def _run(sfv_mod, cfg, X, Y, U0, steps, peer, **kw):
    g = sfv_mod.Solver(cfg, X, Y, **kw)
    if peer:
        g.enable_peer_halo()
    g.set_state(U0)
    g.step(steps)
    g.sync()
    return g


@pytest.mark.parametrize("px,py,wx,wy,rk", [
    (2, 1, None, None, I.RK4_CLASSIC),
    (1, 2, None, None, I.RK4_CLASSIC),
    (2, 2, None, None, I.RK4_CLASSIC),
    (3, 2, [1, 2, 3], [2, 1], I.RK4_CLASSIC),
    (4, 1, None, None, I.RK2_HEUN),
    (2, 3, None, None, I.RK4_JAMESON),
])
def test_peer_loopback_bitwise(sfv_mod, oracle_mod, px, py, wx, wy, rk):
    ni, nj, steps = 120, 70, 40
    X, Y = I.ramp_nodes(ni, nj, 30.0)
    cfg = I.default_config(ni, nj, rk=rk)
    U0 = I.perturbed_state(ni, nj, 5)
    g1 = _run(sfv_mod, cfg, X, Y, U0, steps, False)
    gp = _run(sfv_mod, cfg, X, Y, U0, steps, True, px=px, py=py, wx=wx, wy=wy)
    np.testing.assert_array_equal(gp.get_state(), g1.get_state())
    np.testing.assert_array_equal(gp.dt(), g1.dt())
    assert norm_error(gp.residual_norms(), g1.residual_norms()) < 1e-14
    o = oracle_mod.Oracle(cfg, X, Y)
    o.set_state(U0); o.step(steps)
    assert np.all(state_error(gp.get_state(), o.get_state()) <= 1e-10)
    assert norm_error(gp.residual_norms(), o.residual_norms()) <= 1e-10
    assert dt_error(gp.dt(), o.dt()) <= 1e-13


def test_peer_c2_eight_slabs(sfv_mod):
    """C2 in the 8-GPU slab layout, peer mode, 20 steps:
    bitwise equal to one block; a second set_state restarts the flags."""
    X, Y = I.config_nodes("C2")
    c = I.CONFIGS["C2"]
    cfg = I.default_config(c["ni"], c["nj"])
    U0 = I.perturbed_state(c["ni"], c["nj"], 2)
    g1 = _run(sfv_mod, cfg, X, Y, U0, 20, False)
    g8 = _run(sfv_mod, cfg, X, Y, U0, 20, True, px=8)
    np.testing.assert_array_equal(g8.get_state(), g1.get_state())
    g8.set_state(U0); g8.step(20); g8.sync()
    np.testing.assert_array_equal(g8.get_state(), g1.get_state())
    np.testing.assert_array_equal(g8.dt(), g1.dt())


def test_peer_mode_needs_new_state(sfv_mod):
    ni, nj = 64, 32
    X, Y = I.ramp_nodes(ni, nj, 15.0)
    g = sfv_mod.Solver(I.default_config(ni, nj), X, Y, px=2)
    g.set_state(I.uniform_state(ni, nj))
    g.step(2); g.sync()
    g.set_halo_mode(sfv_mod.HALO_PEER)
    with pytest.raises(sfv_mod.SfvError) as ex:
        g.step(1)
    assert ex.value.code == sfv_mod.ERR_SEQUENCE
    with pytest.raises(sfv_mod.SfvError) as ex:
        g.set_halo_mode(7)
    assert ex.value.code == sfv_mod.ERR_ARG


def test_peer_freestream_preserved(sfv_mod):
    """Uniform freestream on a uniform rectangular grid with inflow/outflow
    everywhere is an exact steady state; peer-mode ghosts must keep it
    bitwise (any stale or missing ghost would perturb it)."""
    ni, nj = 90, 64
    X, Y = I.cartesian_nodes(ni, nj, 3.0, 1.5)
    cfg = I.default_config(ni, nj)
    cfg["bc"] = [0, 1, 1, 1]
    U0 = I.uniform_state(ni, nj)
    g = _run(sfv_mod, cfg, X, Y, U0, 30, True, px=3, py=2)
    np.testing.assert_array_equal(g.get_state(), U0)


@pytest.mark.parametrize("px,py,rk", [(2, 3, I.RK2_HEUN), (3, 2, I.RK4_CLASSIC), (1, 4, I.RK4_JAMESON)])
def test_peer_ghost_frames_are_neighbour_edges(sfv_mod, px, py, rk):
    """After a step, every connected ghost layer of stage buffer 1 (the
    first stage's output, written by the neighbour's stage kernel) equals
    the neighbour's 2 edge layers bitwise (halo plan of
    sfv_halo_plan).  Middle blocks (py = 3, 4) touch S and N at once."""
    ni, nj = 120, 70
    X, Y = I.ramp_nodes(ni, nj, 30.0)
    cfg = I.default_config(ni, nj, rk=rk)
    g = _run(sfv_mod, cfg, X, Y, I.perturbed_state(ni, nj, 9), 3, True, px=px, py=py)
    for b in range(px * py):
        m = g.partition_map(b)
        B = g.block_buffer(b, 1)
        for e in range(4):
            nb = int(m[4 + e])
            if nb < 0:
                continue
            N = g.block_buffer(nb, 1)
            mine, theirs = {0: (B[0:2, :, 2:-2], N[-4:-2, :, 2:-2]), 1: (B[-2:, :, 2:-2], N[2:4, :, 2:-2]),
                            2: (B[2:-2, :, 0:2], N[2:-2, :, -4:-2]), 3: (B[2:-2, :, -2:], N[2:-2, :, 2:4])}[e]
            np.testing.assert_array_equal(mine, theirs, err_msg=f"block {b} edge {'WESN'[e]}")


@pytest.mark.parametrize("ni,nj,px,py", [(37, 29, 5, 3), (64, 62, 2, 2), (12, 40, 3, 1), (90, 31, 1, 1),
                                         (48, 93, 2, 3)])
def test_peer_small_and_ragged_blocks(sfv_mod, ni, nj, px, py):
    """Blocks of a single segment (ni_b < 8), a last strip of one column
    (nj_b = 31: two strips touch the N edge), 1-column-wide tail strips and
    odd sizes: peer mode stays bitwise equal to the single block."""
    X, Y = I.ramp_nodes(ni, nj, 30.0)
    cfg = I.default_config(ni, nj)
    U0 = I.perturbed_state(ni, nj, 13)
    g1 = _run(sfv_mod, cfg, X, Y, U0, 25, False)
    gp = _run(sfv_mod, cfg, X, Y, U0, 25, True, px=px, py=py)
    np.testing.assert_array_equal(gp.get_state(), g1.get_state())
    np.testing.assert_array_equal(gp.dt(), g1.dt())
