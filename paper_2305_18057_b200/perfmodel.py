"""The paper's workload performance model (Eqs. 8-13) and
ssspnt (Eq. 14), calibrated on B200.

Host-side analysis only (no part of the hot path).  The paper models one
iteration of a block of N_l x N_w cells as interior work N_l N_w t_I plus
boundary work (2 N_w + 2 N_l) t_B (Eq. 8 with N_d = 1), folds transfers and
synchronisation into t_f = alpha T_b (Eq. 12) and writes t_B = beta t_I
(Eq. 13).  For 1D slabs on G equal GPUs (Eq. 10) every rank holds
N_l/G x N_w cells.

Generalisation used here: unequal ranks / 2D blocks take
the max over ranks of their own Eq. 12 time (the paper's equations assume
equal shares), and a per-launch term t_L is added: on a GPU each stage of
each block is one kernel launch whose fill / drain costs a fixed time
independent of the block's cells (the paper's CPU-era model has no such
term; on one device it is what the paper's t_f absorbs).

Measured on B200 the paper's linear form (interior + boundary cells) does
not describe a stage kernel well: a block's cost is set by its launch
geometry (warp tasks of 30 columns x a segment of rows, in waves of 148 x 12
resident warps), so `GeometryModel` models a stage as
t_L + t_row * waves * (rows per task + 1.5) with the library's own segment
choice (sfv_host.cu choose_launch), and is what the multi-GPU predictions use.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def ssspnt(size, steps, np_units, time_s, s=1e-6):
    """Eq. 14: s * size * steps / (np * time)."""
    return s * size * steps / (np_units * time_s)


def time_seq(Nl, Nw, Nd, tI, tB, t_transfer=0.0):
    """Eq. 8, literally: N_l N_w N_d t_I + (2 N_l N_w + 2 N_l
    N_d + 2 N_w N_d) t_B + t_DH + t_HH + t_HD + 5 t_S (t_transfer)."""
    return Nl * Nw * Nd * tI + (2 * Nl * Nw + 2 * Nl * Nd + 2 * Nw * Nd) * tB + t_transfer


def time_cpu(Nl, Nw, C, tI, tB, t_transfer=0.0):
    """Eq. 9, the 2D slab form on C CPUs:
    N_l N_w / C t_I + (2 N_w + 2 N_l / C) t_B + transfers."""
    return Nl * Nw / C * tI + (2 * Nw + 2 * Nl / C) * tB + t_transfer


def time_hete(Nl, Nw, tI, beta, alpha, G=1, rgc=1.0, C=0):
    """Eq. 13: [N_l N_w / (G r_gc + C) + (2 N_w + 2 N_l /
    (G r_gc + C)) (1 + alpha) beta] t_I.  With G = 1, r_gc = 1, C = 0,
    alpha = 0 this is Eq. 8 with N_d = 1 and t_B = beta t_I."""
    share = G * rgc + C
    return (Nl * Nw / share + (2 * Nw + 2 * Nl / share) * (1.0 + alpha) * beta) * tI


@dataclass
class Block:
    ni: int
    nj: int

    @property
    def cells(self):
        return self.ni * self.nj

    @property
    def perimeter(self):
        # the paper's boundary-cell count of a block, 2 N_w + 2 N_l
        return 2 * self.ni + 2 * self.nj


def split(n, parts, weights=None):
    """Largest-remainder split (the library's sfv_split; reading A-R24),
    reimplemented for planning without a device."""
    w = np.ones(parts, np.int64) if weights is None else np.asarray(weights, np.int64)
    sw = int(w.sum())
    base = [n * int(x) // sw for x in w]
    rem = [n * int(x) % sw for x in w]
    order = sorted(range(parts), key=lambda r: -rem[r])  # stable: ties to the lower index
    for k in range(n - sum(base)):
        base[order[k]] += 1
    return base


def blocks_of(ni, nj, px, py, wx=None, wy=None):
    xs, ys = split(ni, px, wx), split(nj, py, wy)
    return [Block(a, b) for b in ys for a in xs]


@dataclass
class GpuModel:
    """Per stage of one block on one B200: t = cells t_I + perimeter t_B + t_L."""
    tI: float   # s per interior cell-stage
    tB: float   # s per boundary cell-stage
    tL: float   # s per stage launch (fill / drain)
    stages: int = 4

    @property
    def beta(self):
        return self.tB / self.tI

    def block_stage(self, b: Block):
        return b.cells * self.tI + b.perimeter * self.tB + self.tL

    def loopback_step(self, blocks):
        """All blocks on one device, launched one after another: the sum."""
        return self.stages * sum(self.block_stage(b) for b in blocks)

    def multi_gpu_step(self, blocks, t_dt=0.0, alpha=0.0):
        """One block per GPU: the slowest rank, with its boundary work scaled
        by (1 + alpha) for exchange overhead (Eq. 12), plus the per-step dt
        all-reduce t_dt."""
        worst = max(b.cells * self.tI + b.perimeter * self.tB * (1.0 + alpha) + self.tL for b in blocks)
        return self.stages * worst + t_dt


def fit(samples, stages=4):
    """Least squares for (t_I, t_B, t_L) from loopback samples: each sample is
    (blocks, seconds per step).  Rows are scaled by 1/time so the fit
    minimises relative error."""
    A, y = [], []
    for blocks, t in samples:
        row = [stages * sum(b.cells for b in blocks), stages * sum(b.perimeter for b in blocks),
               stages * len(blocks)]
        A.append([v / t for v in row])
        y.append(1.0)
    coef, *_ = np.linalg.lstsq(np.asarray(A), np.asarray(y), rcond=None)
    return GpuModel(float(coef[0]), float(coef[1]), float(coef[2]), stages)


# ---------------------------------------------------------------- GPU-native
NT_OUT = 30          # output columns per warp task (WOUT, CPL = 1)
NSEG_MAX = 256


def launch_geometry(ni, nj, slots=148 * 12):
    """(strips, segments, rows per task, waves) as sfv_host.cu choose_launch
    picks them: minimise (ceil(ni/s) + 1.5) * waves, ties to more segments."""
    strips = -(-nj // NT_OUT)
    cap = min(NSEG_MAX, max(1, ni // 4))
    best, best_cost = 1, float("inf")
    for sgs in range(1, cap + 1):
        rows = -(-ni // sgs)
        waves = -(-(strips * sgs) // slots)
        cost = (rows + 1.5) * waves
        if cost <= best_cost + 1e-9:
            best, best_cost = sgs, cost
    sgs = min(best, ni)
    return strips, sgs, -(-ni // sgs), -(-(strips * sgs) // slots)


@dataclass
class GeometryModel:
    """Per stage of one block: t_L + t_row * waves * (rows per task + 1.5)."""
    t_row: float
    tL: float
    stages: int = 4
    slots: int = 148 * 12

    def block_stage(self, b: Block):
        _, _, rows, waves = launch_geometry(b.ni, b.nj, self.slots)
        return self.tL + self.t_row * waves * (rows + 1.5)

    def loopback_step(self, blocks):
        return self.stages * sum(self.block_stage(b) for b in blocks)

    def multi_gpu_step(self, blocks, t_dt=0.0):
        return self.stages * max(self.block_stage(b) for b in blocks) + t_dt


def fit_geometry(samples, stages=4, slots=148 * 12):
    """Least squares (relative error) for (t_row, t_L) from loopback samples."""
    A = []
    for blocks, t in samples:
        w = sum(launch_geometry(b.ni, b.nj, slots)[3] * (launch_geometry(b.ni, b.nj, slots)[2] + 1.5)
                for b in blocks)
        A.append([stages * w / t, stages * len(blocks) / t])
    coef, *_ = np.linalg.lstsq(np.asarray(A), np.ones(len(A)), rcond=None)
    return GeometryModel(float(coef[0]), float(coef[1]), stages, slots)
