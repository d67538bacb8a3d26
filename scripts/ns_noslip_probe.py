"""Which C2 Navier-Stokes settings survive an impulsive Mach-4 start over a no-slip ramp (probe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_18057_b200 import inputs as I, sfv
ni, nj = 1440, 720
for theta, mu, cfl, bcE in [(30, 1e-3, 0.8, 1), (30, 1e-3, 0.4, 1), (30, 1e-2, 0.8, 1), (30, 1e-1, 0.8, 1),
                            (5, 1e-3, 0.8, 1), (30, 1e-3, 0.2, 1), (15, 1e-3, 0.8, 1)]:
    X, Y = I.ramp_nodes(ni, nj, theta)
    cfg = I.default_config(ni, nj, viscous=1, mu=mu, cfl=cfl, bc=(0, bcE, 3, 2))
    g = sfv.Solver(cfg, X, Y)
    g.set_state(I.uniform_state(ni, nj))
    res = "ok"
    for k in range(10):
        try:
            g.step(50); g.sync()
        except sfv.SfvError as ex:
            res = f"failed after ~{50 * k} steps: {str(ex)[:70]}"
            break
    print(theta, mu, cfl, bcE, res, flush=True)
    g.close()
