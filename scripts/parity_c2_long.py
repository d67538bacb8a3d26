"""C2 at full size (1440 x 720), perturbed inlet: GPU vs oracle after 1, 10 and 100 RK4 steps,
and the oracle's own 1-ulp sensitivity at 100 steps (evidence run, ~4 min of oracle time)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle
from paper_2305_18057_b200 import inputs as I, sfv
from parity_util import state_error, norm_error, dt_error
X, Y = I.config_nodes("C2"); c = I.CONFIGS["C2"]
cfg = I.default_config(c["ni"], c["nj"])
U0 = I.perturbed_state(c["ni"], c["nj"], 2)
g = sfv.Solver(cfg, X, Y); g.set_state(U0)
o = oracle.Oracle(cfg, X, Y); o.set_state(U0)
done = 0
for n in (1, 10, 100):
    t0 = time.time()
    g.step(n - done); g.sync(); o.step(n - done); done = n
    print(f"C2 steps {n}: state {state_error(g.get_state(), o.get_state()).max():.3e} "
          f"norms {norm_error(g.residual_norms(), o.residual_norms()):.3e} dt {dt_error(g.dt(), o.dt()):.3e} "
          f"({time.time() - t0:.0f} s)", flush=True)
U1 = U0.copy(); U1[..., 0] = np.nextafter(U1[..., 0], np.inf)
o2 = oracle.Oracle(cfg, X, Y); o2.set_state(U1); o2.step(100)
print(f"oracle 1-ulp sensitivity at 100 steps: {state_error(o2.get_state(), o.get_state()).max():.3e}")
