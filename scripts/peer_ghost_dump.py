"""Ghost-frame fidelity after 1 step in peer mode (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2305_18057_b200 import inputs as I
from paper_2305_18057_b200 import sfv

px, py = 2, 3
ni, nj = 120, 70
X, Y = I.ramp_nodes(ni, nj, 30.0)
U0 = I.perturbed_state(ni, nj, 5)
cfg = I.default_config(ni, nj, rk=I.RK2_HEUN, dt_fixed=1e-7)
g = sfv.Solver(cfg, X, Y, px=px, py=py)
g.enable_peer_halo()
g.set_state(U0)
g.step(1)
try:
    g.sync()
except sfv.SfvError as ex:
    print("error", ex)
for b in range(px * py):
    m = g.partition_map(b)
    B = g.block_buffer(b, 1)
    for e, name in enumerate("WESN"):
        nb = m[4 + e]
        if nb < 0:
            continue
        N = g.block_buffer(nb, 1)
        if e == 0: mine, theirs = B[0:2, :, 2:-2], N[-4:-2, :, 2:-2]
        if e == 1: mine, theirs = B[-2:, :, 2:-2], N[2:4, :, 2:-2]
        if e == 2: mine, theirs = B[2:-2, :, 0:2], N[2:-2, :, -4:-2]
        if e == 3: mine, theirs = B[2:-2, :, -2:], N[2:-2, :, 2:4]
        bad = np.argwhere(mine != theirs)
        print(b, name, "nbr", nb, "mismatches", len(bad), bad[:6].tolist(), flush=True)
