"""C2 at full size (1440 x 720) in the launch configuration bench.py times: GPU vs the
oracle (the -fopenmp build, bitwise the single-threaded one) after 1, 100 and 1000 RK4 steps,
for the bench's uniform Table 1 start (the north-star gate: 1e-12 after 1 step, 1e-9 after
1000, norms 1e-10) and for a +-2 % perturbed start next to the oracle's own 1-ulp sensitivity
(reading A-R30).  Evidence run (~5 min of oracle time on 16 cores)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle
from paper_2305_18057_b200 import inputs as I, sfv
from parity_util import state_error, norm_error, dt_error
X, Y = I.config_nodes("C2"); c = I.CONFIGS["C2"]
cfg = I.default_config(c["ni"], c["nj"])
for name, U0 in (("uniform Table 1 start (bench)", I.uniform_state(c["ni"], c["nj"])),
                 ("perturbed +-2 %, seed 4", I.perturbed_state(c["ni"], c["nj"], 4))):
    g = sfv.Solver(cfg, X, Y); g.set_state(U0)
    o = oracle.Oracle(cfg, X, Y, omp=True); o.set_state(U0)
    done = 0
    for n in (1, 100, 1000):
        t0 = time.time()
        g.step(n - done); g.sync(); o.step(n - done); done = n
        print(f"C2 {name}, {n} steps: state {state_error(g.get_state(), o.get_state()).max():.3e} "
              f"norms {norm_error(g.residual_norms(), o.residual_norms()):.3e} dt {dt_error(g.dt(), o.dt()):.3e} "
              f"({time.time() - t0:.0f} s)", flush=True)
    U1 = U0.copy(); U1[..., 0] = np.nextafter(U1[..., 0], np.inf)
    o2 = oracle.Oracle(cfg, X, Y, omp=True); o2.set_state(U1); o2.step(1000)
    print(f"C2 {name}: oracle 1-ulp sensitivity at 1000 steps: state {state_error(o2.get_state(), o.get_state()).max():.3e} "
          f"norms {norm_error(o2.residual_norms(), o.residual_norms()):.3e} dt {dt_error(o2.dt(), o.dt()):.3e}", flush=True)
