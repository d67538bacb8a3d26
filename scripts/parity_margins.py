#!/usr/bin/env python
"""1000-step parity margins against the oracle's own sensitivity (VERDICT r1
item 2; SURVEY §8(c).5 gates): for the C1 wedge and the 256 x 128 perturbed
inlet (seeds 0, 1, 2) the GPU-vs-oracle state error e_k (reading A-R22) and
norm-history error after 1 / 100 / 1000 steps, next to the oracle's own
sensitivity: the oracle started from the same state with every density
moved by one ulp (np.nextafter), compared with the unperturbed oracle.
Prints one JSON line per case (library = $SFV_LIB or the default build)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2305_18057_b200 import inputs as I, sfv  # noqa: E402
from parity_util import norm_error, state_error  # noqa: E402

CASES = [("C1_wedge", 64, 32, 15.0, None), ("inlet256_seed0", 256, 128, 30.0, 0),
         ("inlet256_seed1", 256, 128, 30.0, 1), ("inlet256_seed2", 256, 128, 30.0, 2),
         ("C2_full_freestream", 1440, 720, 30.0, None)]  # the bench workload itself (oracle: -fopenmp build)


def ulp_nudge(U):
    V = U.copy()
    V[..., 0] = np.nextafter(V[..., 0], np.inf)
    return V


def main():
    only = sys.argv[1:]
    os.environ.setdefault("OMP_NUM_THREADS", str(len(os.sched_getaffinity(0))))
    for name, ni, nj, th, seed in CASES:
        if only and name not in only:
            continue
        X, Y = I.ramp_nodes(ni, nj, th)
        cfg = I.default_config(ni, nj)
        U0 = I.uniform_state(ni, nj) if seed is None else I.perturbed_state(ni, nj, seed)
        big = ni * nj > 100000  # the bitwise-equal OpenMP oracle build on every host core
        g = sfv.Solver(cfg, X, Y); g.set_state(U0)
        o = oracle.Oracle(cfg, X, Y, omp=big); o.set_state(U0)
        s = oracle.Oracle(cfg, X, Y, omp=big); s.set_state(ulp_nudge(U0))
        done, rec = 0, {"case": name, "lib": os.path.basename(os.environ.get("SFV_LIB", "libsfv.so"))}
        for n in (1, 100, 1000):
            g.step(n - done); g.sync(); o.step(n - done); s.step(n - done); done = n
            Uo = o.get_state()
            rec[str(n)] = {"gpu_vs_oracle": float(state_error(g.get_state(), Uo).max()),
                           "oracle_1ulp_sensitivity": float(state_error(s.get_state(), Uo).max()),
                           "norms_gpu_vs_oracle": float(norm_error(g.residual_norms(), o.residual_norms()))}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
