"""GPU viscous residual / gradients vs the oracle on the stage-2 input of a Heun step (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2305_18057_b200 import inputs as I, sfv
ni, nj = 64, 32
X, Y = I.ramp_nodes(ni, nj, 15.0)
U0 = I.perturbed_state(ni, nj, 21)
cfg = I.default_config(ni, nj, viscous=1, mu=0.05, rk=I.RK2_HEUN, dt_fixed=1e-6)
g = sfv.Solver(cfg, X, Y); g.set_state(U0); g.step(1); g.sync()
W2 = g.block_buffer(0, 1)                    # [ni+4, 4, nj+4]
W2i = np.transpose(W2[2:-2, :, 2:-2], (2, 0, 1)).copy()   # [nj, ni, 4]
rv = g.block_buffer(0, -1)[2:-2, :, 2:-2]      # [ni, 4, nj]
G = g.block_buffer(0, -2)                      # [ni+2, 6, nj+2]
o = oracle.Oracle(cfg, X, Y)
o0 = oracle.Oracle(dict(cfg, mu=0.0), X, Y)
Rv_o = -(o.residual(W2i) - o0.residual(W2i))   # [nj, ni, 4]
Go = o.gradients(W2i)                            # [nj, ni, 6]
Gg = np.transpose(G[1:-1, :, 1:-1], (2, 0, 1))
Rg = np.transpose(rv, (2, 0, 1))
dg = np.abs(Gg - Go).max(axis=-1) / np.abs(Go).max()
dr = np.abs(Rg - Rv_o).max(axis=-1) / np.abs(Rv_o).max()
print("grad max rel", dg.max(), "at (j,i)", np.unravel_index(np.argmax(dg), dg.shape))
print("rv max rel", dr.max(), "at (j,i)", np.unravel_index(np.argmax(dr), dr.shape))
bad = np.argwhere(dr > 1e-9)
print("rv bad cells (j,i):", bad[:20].tolist(), len(bad))
badg = np.argwhere(dg > 1e-9)
print("grad bad cells (j,i):", badg[:20].tolist(), len(badg))
print("sample grad gpu (j=5,i=10):", Gg[5, 10], "\noracle:", Go[5, 10])
print("sample rv gpu:", Rg[5, 10], "\noracle:", Rv_o[5, 10])
print("raw G rows:", G[11, :, 6], G[0, :, 6])
