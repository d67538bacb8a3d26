"""The NCCL path (nranks > 1) on ONE GPU.

Every gpurun box and the round-end tiers have a single B200, so the
multi-rank path is exercised by running `world` processes on cuda:0 that
NCCL believes live on different hosts (a distinct NCCL_HOSTID per rank ->
the socket network transport over loopback; NCCL forbids two ranks of one
communicator on one GPU of one host).  Everything above the transport --
sfv_partition's communicator, the grouped send/recv of the row halos on the
comm stream, the pack/unpack of column halos, the sigma max all-reduce, the
zero-padded sum all-reduces of get_state / get_residual_norms, graph
capture with NCCL calls, the edge/interior overlap split -- is the code a
multi-GPU run executes.  The result must be bitwise equal to the same
decomposition run in loopback mode (which is bitwise equal to one block,
test_gpu_parity.py::test_loopback_decomposition_invariance) and match the
oracle within the 1e-12/50-step gates."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, px, py, ni, nj, steps, overlap, halo, rk, wx, visc, out_q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port),
                       "NCCL_HOSTID": f"sfv-sim-host-{rank}", "NCCL_SOCKET_IFNAME": "lo",
                       "NCCL_IB_DISABLE": "1", "NCCL_NVLS_ENABLE": "0", "SFV_OVERLAP": str(overlap)})
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_18057_b200 import inputs as I
        from paper_2305_18057_b200 import sfv
        X, Y = I.ramp_nodes(ni, nj, 5.0 if visc else 30.0)
        cfg = I.default_config(ni, nj, rk=rk, **visc)
        obj = [sfv.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        s = sfv.Solver(cfg, X, Y, px=px, py=py, wx=wx, rank=rank, nranks=world, nccl_id=obj[0], device=0)
        if halo == "peer":
            s.enable_peer_halo()  # CUDA-IPC mapping of the neighbours' workspaces
        s.set_state(I.perturbed_state(ni, nj, 7))
        s.step(steps)
        s.sync()
        U = s.get_state()
        nrm = s.residual_norms()
        dts = s.dt()
        s.close()
        out_q.put((rank, "ok", U if rank == 0 else None, nrm, dts))
    except Exception as ex:  # surface to the parent
        out_q.put((rank, repr(ex), None, None, None))
    finally:
        dist.destroy_process_group()


def _run(world, px, py, ni, nj, steps, overlap, halo="copy", rk=0, wx=None, visc=None):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, px, py, ni, nj, steps, overlap, halo, rk, wx, visc or {}, q))
          for r in range(world)]
    for p in ps:
        p.start()
    try:
        res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for rank, status, *_ in res:
        assert status == "ok", (rank, status)
    return res


@pytest.mark.parametrize("world,px,py,overlap,halo,rk,wx", [
    (2, 2, 1, 1, "copy", 0, None), (2, 2, 1, 0, "copy", 0, None), (2, 1, 2, 1, "copy", 0, None),
    (4, 2, 2, 1, "copy", 0, None), (2, 2, 1, 1, "peer", 0, None), (2, 1, 2, 1, "peer", 0, None),
    (4, 2, 2, 1, "peer", 0, None), (3, 3, 1, 1, "peer", 2, [1, 2, 3]), (2, 2, 1, 1, "peer", 1, None)])
def test_nccl_ranks_match_loopback_and_oracle(oracle_mod, world, px, py, overlap, halo, rk, wx):
    """halo="peer": the stage kernels store the edge layers into the neighbour
    rank's workspace through its CUDA-IPC mapping and the CFL max travels
    through every rank's sigma table; NCCL only for the
    norms and state gathers.  rk: 0 RK4, 1 Heun, 2 Jameson; wx: slab weights."""
    from paper_2305_18057_b200 import inputs as I
    from paper_2305_18057_b200 import sfv
    from parity_util import dt_error, norm_error, state_error
    ni, nj, steps = 160, 64, 50
    res = _run(world, px, py, ni, nj, steps, overlap, halo, rk, wx)
    U = res[0][2]
    X, Y = I.ramp_nodes(ni, nj, 30.0)
    cfg = I.default_config(ni, nj, rk=rk)
    U0 = I.perturbed_state(ni, nj, 7)
    g = sfv.Solver(cfg, X, Y, px=px, py=py, wx=wx)
    g.set_state(U0); g.step(steps); g.sync()
    np.testing.assert_array_equal(U, g.get_state())
    for rank, _, _, nrm, dts in res:  # every rank holds the global histories
        np.testing.assert_array_equal(dts, g.dt())
        # the per-block partial sums group cells by launch (the overlap split
        # adds edge launches), so the norms agree to rounding, not bitwise
        assert norm_error(nrm, g.residual_norms()) < 1e-14
    o = oracle_mod.Oracle(cfg, X, Y)
    o.set_state(U0); o.step(steps)
    assert np.all(state_error(U, o.get_state()) <= 1e-11)
    assert norm_error(res[0][3], o.residual_norms()) <= 1e-10
    assert dt_error(res[0][4], o.dt()) <= 1e-13


@pytest.mark.parametrize("world,px,py,halo", [(2, 2, 1, "copy"), (2, 1, 2, "copy"), (4, 2, 2, "copy"),
                                               (2, 2, 1, "peer"), (2, 1, 2, "peer"), (4, 2, 2, "peer")])
def test_nccl_navier_stokes_ranks(oracle_mod, world, px, py, halo):
    """Navier-Stokes across NCCL ranks: ghost gradients travel by send/recv
    (rows from the frame, columns packed) or, halo="peer", grad_kernel stores
    them into the neighbour rank's gradient frame through its CUDA-IPC
    mapping; bitwise equal to loopback blocks and within the parity gates of
    the oracle."""
    from paper_2305_18057_b200 import inputs as I
    from paper_2305_18057_b200 import sfv
    from parity_util import state_error
    ni, nj, steps = 96, 48, 30
    visc = dict(viscous=1, mu=0.1, bc=(I.BC_INFLOW, I.BC_OUTFLOW, I.BC_NOSLIP_WALL, I.BC_SLIP_WALL))
    res = _run(world, px, py, ni, nj, steps, 1, halo, 0, None, visc)
    U = res[0][2]
    X, Y = I.ramp_nodes(ni, nj, 5.0)
    cfg = I.default_config(ni, nj, **visc)
    U0 = I.perturbed_state(ni, nj, 7)
    g = sfv.Solver(cfg, X, Y, px=px, py=py)
    g.set_state(U0); g.step(steps); g.sync()
    np.testing.assert_array_equal(U, g.get_state())
    o = oracle_mod.Oracle(cfg, X, Y)
    o.set_state(U0); o.step(steps)
    assert np.all(state_error(U, o.get_state()) <= 1e-11)


def _fault_worker(rank, world, port, mode, out_q):
    """mode 'dead_peer': rank 1 dies after set_state; rank 0 must get
    SFV_ERR_NCCL from sfv_sync within the comm timeout instead of hanging
    (SPEC.md:357).  mode 'bad_cell': an invalid cell in rank 1's slab only;
    every rank must return SFV_ERR_STATE from set_state with the same (global)
    cell, none may block in a collective."""
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port),
                       "NCCL_HOSTID": f"sfv-sim-host-{rank}", "NCCL_SOCKET_IFNAME": "lo",
                       "NCCL_IB_DISABLE": "1", "NCCL_NVLS_ENABLE": "0", "SFV_DEBUG_WAIT": "1"})
    import sys
    import time
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_18057_b200 import inputs as I
        from paper_2305_18057_b200 import sfv
        ni, nj = 160, 64
        X, Y = I.ramp_nodes(ni, nj, 30.0)
        cfg = I.default_config(ni, nj)
        obj = [sfv.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        s = sfv.Solver(cfg, X, Y, px=world, py=1, rank=rank, nranks=world, nccl_id=obj[0], device=0)
        s.set_comm_timeout(5.0)
        U0 = I.perturbed_state(ni, nj, 7)
        if mode == "bad_cell":
            U0[10, 150, 0] = -1.0            # rho < 0 in the last slab only (i = 150)
            try:
                s.set_state(U0)
                out_q.put((rank, "no error", None, None))
            except sfv.SfvError as ex:
                out_q.put((rank, ex.code, ex.info, str(ex)))
            return
        s.set_state(U0)
        s.step(5); s.sync()
        dist.barrier()
        if rank == 1:
            os._exit(0)                      # the neighbour disappears
        import faulthandler
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        logf = open(os.path.join(ROOT, "gpurun_out", "dead_peer_rank0.log"), "w")
        os.dup2(logf.fileno(), 2)  # the library's SFV_DEBUG_WAIT trace goes to the same file
        faulthandler.dump_traceback_later(90, exit=False, file=logf)
        def note(m):
            logf.write(f"{time.time():.3f} {m}\n"); logf.flush()
        time.sleep(1.0)
        t0 = time.time()
        try:
            note("step")
            s.step(50)
            note("sync")
            s.sync()
            out_q.put((rank, "no error", None, time.time() - t0))
        except sfv.SfvError as ex:
            note("error " + str(ex))
            out_q.put((rank, ex.code, str(ex), time.time() - t0))
        out_q.close(); out_q.join_thread()   # flush the queue's feeder thread before the hard exit
        os._exit(0)                          # (the communicator is aborted; skip teardown)
    except Exception as ex:
        out_q.put((rank, repr(ex), None, None))


def _run_fault(mode, world=2, expect=2):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_fault_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in ps:
        p.start()
    try:
        res = sorted((q.get(timeout=240) for _ in range(expect)), key=lambda r: r[0])
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    return res


def test_nccl_dead_peer_is_an_error_not_a_hang():
    from paper_2305_18057_b200 import sfv
    (rank, code, msg, secs), = _run_fault("dead_peer", expect=1)
    assert rank == 0 and code == sfv.ERR_NCCL, (code, msg)
    assert "rank 1" in msg and ("deadlock" in msg or "async error" in msg), msg   # names the edge
    assert secs < 60, secs


def test_nccl_invalid_cell_on_one_rank_every_rank_errors():
    from paper_2305_18057_b200 import sfv
    res = _run_fault("bad_cell", expect=2)
    codes = [r[1] for r in res]
    assert codes == [sfv.ERR_STATE, sfv.ERR_STATE], res
    assert res[0][2] == res[1][2] and res[0][2][2:] == (150, 10), res   # same global cell (i, j)
