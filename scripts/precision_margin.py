"""Parity margins (state error vs the oracle) of the current library on the
standard gates: C1 wedge 1 / 100 / 1000 steps, perturbed inlet 1000 steps."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle
from paper_2305_18057_b200 import inputs as I, sfv
from parity_util import state_error, norm_error
cases = [("wedge", 64, 32, 15.0, None), ("inlet", 128, 64, 30.0, 3)]
for name, ni, nj, th, seed in cases:
    X, Y = I.ramp_nodes(ni, nj, th)
    cfg = I.default_config(ni, nj)
    U0 = I.uniform_state(ni, nj) if seed is None else I.perturbed_state(ni, nj, seed)
    g = sfv.Solver(cfg, X, Y); g.set_state(U0)
    o = oracle.Oracle(cfg, X, Y); o.set_state(U0)
    done = 0
    for n in (1, 100, 1000):
        g.step(n - done); g.sync(); o.step(n - done); done = n
        print(os.environ.get("SFV_LIB", "default"), name, n, "state", state_error(g.get_state(), o.get_state()).max(),
              "norms", norm_error(g.residual_norms(), o.residual_norms()), flush=True)
