"""VA1 limiter (reading A-R3): GPU-vs-oracle state error after 1 / 100 / 1000 steps next to the
oracle's own 1-ulp sensitivity (diagnostic; tests/test_gpu_parity.py gates it)."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2305_18057_b200 import inputs as I, sfv
import oracle
from parity_util import state_error, norm_error, dt_error
ni, nj = 80, 40
X, Y = I.ramp_nodes(ni, nj, 30.0)
cfg = I.default_config(ni, nj, limiter=I.LIM_VAN_ALBADA)
U0 = I.perturbed_state(ni, nj, 9)
U1 = U0.copy(); U1[..., 0] = np.nextafter(U1[..., 0], np.inf)
g = sfv.Solver(cfg, X, Y); g.set_state(U0)
o = oracle.Oracle(cfg, X, Y); o.set_state(U0)
s = oracle.Oracle(cfg, X, Y); s.set_state(U1)
done = 0
print("| steps | GPU vs oracle (state) | oracle 1-ulp sensitivity | ratio | dt err | dt sensitivity |")
print("|---|---|---|---|---|---|")
for n in (1, 100, 1000):
    k = n - done; done = n
    g.step(k); g.sync(); o.step(k); s.step(k)
    e = state_error(g.get_state(), o.get_state()).max(); se = state_error(s.get_state(), o.get_state()).max()
    print(f"| {n} | {e:.2e} | {se:.2e} | {e/max(se,1e-300):.2f} | {dt_error(g.dt(), o.dt()):.1e} | {dt_error(s.dt(), o.dt()):.1e} |")
