"""N > 1 host logic on CPU with world_size-2 `gloo` process groups.

Each rank builds its libsfv ctx in planning mode (nranks = 2, no NCCL id,
no device), takes its partition map and halo plan from the C ABI, and
executes the plan with torch.distributed send/recv on a field whose value
encodes the global cell index.  After the exchange every ghost cell must
hold, bit for bit, the neighbour's interior value at that global index
(ghost fidelity) and corner ghosts must be untouched
(reading A-R18); the maps must equal the oracle's."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def field(I, J, k):
    return np.sin(1.0 + 0.37 * I + 1.91 * J + 0.13 * k) * 1e3 + I * 7.0 + J * 0.001


def _worker(rank, world, port, px, py, wx, wy, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        from paper_2305_18057_b200 import inputs as I
        from paper_2305_18057_b200 import sfv
        import oracle
        ni, nj = 37, 23
        X, Y = I.ramp_nodes(ni, nj, 30.0)
        cfg = I.default_config(ni, nj)
        s = sfv.Solver(cfg, X, Y, px=px, py=py, wx=wx, wy=wy, rank=rank, nranks=world, bind=False)
        m = s.partition_map(rank)
        plan = s.halo_plan(rank)
        o = oracle.Oracle(cfg, X, Y)
        o.partition(px, py, wx, wy)
        assert np.array_equal(m, o.partition_map(rank)), (m, o.partition_map(rank))
        i0, i1, j0, j1 = (int(v) for v in m[:4])
        # local frame with 2 ghost layers, NaN everywhere outside the interior
        F = np.full((j1 - j0 + 4, i1 - i0 + 4, 4), np.nan)
        gi = np.arange(i0, i1)[None, :, None]
        gj = np.arange(j0, j1)[:, None, None]
        kk = np.arange(4)[None, None, :]
        F[2:-2, 2:-2] = field(gi, gj, kk)
        reqs, recvbufs = [], []
        for e in range(4):
            nbr, si0, si1, sj0, sj1, ri0, ri1, rj0, rj1 = (int(v) for v in plan[e])
            if nbr < 0:
                continue
            send = np.ascontiguousarray(F[sj0 - j0 + 2:sj1 - j0 + 2, si0 - i0 + 2:si1 - i0 + 2])
            rbuf = torch.empty((rj1 - rj0, ri1 - ri0, 4), dtype=torch.float64)
            reqs.append(dist.isend(torch.from_numpy(send), nbr))
            reqs.append(dist.irecv(rbuf, nbr))
            recvbufs.append((rbuf, ri0, ri1, rj0, rj1))
        for r in reqs:
            r.wait()
        for rbuf, ri0, ri1, rj0, rj1 in recvbufs:
            F[rj0 - j0 + 2:rj1 - j0 + 2, ri0 - i0 + 2:ri1 - i0 + 2] = rbuf.numpy()
        # ghost fidelity: every received ghost equals the field at its global index
        nrecv = 0
        for rbuf, ri0, ri1, rj0, rj1 in recvbufs:
            GI = np.arange(ri0, ri1)[None, :, None]
            GJ = np.arange(rj0, rj1)[:, None, None]
            want = field(GI, GJ, kk)
            assert np.array_equal(F[rj0 - j0 + 2:rj1 - j0 + 2, ri0 - i0 + 2:ri1 - i0 + 2], want)
            nrecv += want.size
        corners = [F[:2, :2], F[:2, -2:], F[-2:, :2], F[-2:, -2:]]
        assert all(np.all(np.isnan(c)) for c in corners)
        out_q.put((rank, "ok", nrecv))
    except Exception as ex:  # surface to the parent
        out_q.put((rank, repr(ex), 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("px,py,wx,wy", [(2, 1, None, None), (1, 2, None, None), (2, 1, [3, 1], None),
                                         (1, 2, None, [1, 4])])
def test_halo_plan_ghost_fidelity_gloo(px, py, wx, wy):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, px, py, wx, wy, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=180) for _ in range(2)]
    for p in ps:
        p.join(timeout=60)
    for rank, status, n in res:
        assert status == "ok", (rank, status)
        assert n > 0
