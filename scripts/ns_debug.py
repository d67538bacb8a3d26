"""Isolate NS-mode GPU differences (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2305_18057_b200 import inputs as I, sfv
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from parity_util import state_error
ni, nj = 64, 32
X, Y = I.ramp_nodes(ni, nj, 15.0)
U0 = I.perturbed_state(ni, nj, 21)
def run_g(cfg, steps=1):
    g = sfv.Solver(cfg, X, Y); g.set_state(U0); g.step(steps); g.sync(); return g.get_state()
def run_o(cfg, steps=1):
    o = oracle.Oracle(cfg, X, Y); o.set_state(U0); o.step(steps); return o.get_state()
cases = {
  "euler_slip": I.default_config(ni, nj),
  "ns_mu0_slip": I.default_config(ni, nj, viscous=1, mu=0.0),
  "ns_mu0_noslip": I.default_config(ni, nj, viscous=1, mu=0.0, bc=(0, 1, 3, 2)),
  "ns_mu_slip": I.default_config(ni, nj, viscous=1, mu=0.05),
  "ns_mu_noslip": I.default_config(ni, nj, viscous=1, mu=0.05, bc=(0, 1, 3, 2)),
  "ns_mu_noslip_fixed": I.default_config(ni, nj, viscous=1, mu=0.05, bc=(0, 1, 3, 2), dt_fixed=1e-6),
}
for name, cfg in cases.items():
    Ug, Uo = run_g(cfg), run_o(cfg)
    e = state_error(Ug, Uo)
    d = np.abs(Ug - Uo).max(axis=-1)
    jj, ii = np.unravel_index(np.argmax(d), d.shape)
    print(name, e, "worst cell (i,j)", ii, jj, flush=True)
