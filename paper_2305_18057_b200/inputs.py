"""Seeded synthetic input generators shared by the CUDA path and the oracle.

This module holds NONE of the method's arithmetic (no metrics, limiter,
flux, residual or time update).  It only produces the inputs both sides
consume, so a parity comparison is always made on identical bits:

* grid node coordinates for the paper's "simplified 2D 30-degree inlet"
   and the 15-degree wedge of BASELINE config C1, built per
  DESIGN.md reading A-R17 (flat inlet section, then a compression ramp, flat
  top wall, vertical grid lines sheared linearly);
* the Table 1 supersonic freestream as a conserved vector
  (reading A-R15, A-R27: the ABI takes conserved values);
* seeded primitive-variable perturbations from a splitmix64 counter hash
   for parity tests;
* the configuration dictionary both sides are built from.

Array conventions (match include/sfv.h): nodes are (nj+1, ni+1) arrays,
index [j, i]; states are (nj, ni, 4) arrays of (rho, rho*u, rho*v, rho*E).
"""
from __future__ import annotations

import math

import numpy as np

# Gas constants fixed by reading A-R14 (SI units, calorically perfect air;
# SPEC.md:139).
GAMMA = 1.4
R_GAS = 287.0

# Table 1 of the paper: supersonic inflow.
TABLE1_MACH = 4.0
TABLE1_P = 12270.0
TABLE1_T = 217.0

# Boundary kinds, limiter kinds and RK tableaus (numeric codes shared by the
# two independent C headers include/sfv.h and oracle/oracle.h by convention;
# each header defines its own constants).
BC_INFLOW, BC_OUTFLOW, BC_SLIP_WALL, BC_NOSLIP_WALL = 0, 1, 2, 3
LIM_VAN_ALBADA, LIM_VAN_ALBADA2, LIM_NONE = 0, 1, 2
RK4_CLASSIC, RK2_HEUN, RK4_JAMESON = 0, 1, 2
RK_STAGES = {RK4_CLASSIC: 4, RK2_HEUN: 2, RK4_JAMESON: 4}

# The four BASELINE.json configurations.
CONFIGS = {
    "C1": dict(ni=64, nj=32, theta_deg=15.0),
    "C2": dict(ni=1440, nj=720, theta_deg=30.0),
    "C3": dict(ni=11520, nj=5760, theta_deg=30.0),
    "C4": dict(ni=5760, nj=2880, theta_deg=30.0),
}


def freestream_primitive(mach=TABLE1_MACH, p=TABLE1_P, T=TABLE1_T,
                         gamma=GAMMA, R=R_GAS):
    """Table 1 inflow as (rho, u, v, p), ideal gas."""
    rho = p / (R * T)
    a = math.sqrt(gamma * R * T)
    return np.array([rho, mach * a, 0.0, p], dtype=np.float64)


def conserved_from_primitive(prim, gamma=GAMMA):
    """(rho, u, v, p) -> (rho, rho u, rho v, rho E); E = p/((g-1) rho) + q^2/2.

    Input preparation only (the state both sides start from).  Works on
    arrays whose last axis is 4.
    """
    prim = np.asarray(prim, dtype=np.float64)
    rho, u, v, p = prim[..., 0], prim[..., 1], prim[..., 2], prim[..., 3]
    out = np.empty_like(prim)
    out[..., 0] = rho
    out[..., 1] = rho * u
    out[..., 2] = rho * v
    out[..., 3] = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v)
    return out


def freestream_conserved(**kw):
    return conserved_from_primitive(freestream_primitive(**kw))


def ramp_nodes(ni, nj, theta_deg, inlet_length=1.0, ramp_length=2.0,
               height=1.5):
    """Node coordinates of the inlet/wedge grid (reading A-R17).

    ni_in = round(ni*L_in/(L_in+L_r)) uniform cells on [0, L_in], the rest
    uniform on [L_in, L_in+L_r].  Lower wall y_w = 0 up to L_in, then
    (x-L_in)*tan(theta); upper wall flat at `height`; y(i,j) =
    y_w(x_i) + (j/nj)*(height - y_w(x_i)).  Returns (X, Y), each (nj+1, ni+1).
    """
    if ni < 1 or nj < 1:
        raise ValueError("ni, nj must be >= 1")
    if not (0.0 <= theta_deg < 45.0):
        raise ValueError("ramp angle must be in [0, 45)")
    L = inlet_length + ramp_length
    ni_in = int(round(ni * inlet_length / L))
    ni_in = min(max(ni_in, 0), ni)
    x = np.empty(ni + 1, dtype=np.float64)
    if ni_in > 0:
        x[: ni_in + 1] = inlet_length * (np.arange(ni_in + 1) / ni_in)
    else:
        x[0] = 0.0
    nr = ni - ni_in
    if nr > 0:
        x[ni_in:] = inlet_length + ramp_length * (np.arange(nr + 1) / nr)
    t = math.tan(math.radians(theta_deg))
    yw = np.where(x > inlet_length, (x - inlet_length) * t, 0.0)
    frac = np.arange(nj + 1, dtype=np.float64) / nj
    X = np.broadcast_to(x[None, :], (nj + 1, ni + 1)).copy()
    Y = yw[None, :] + frac[:, None] * (height - yw[None, :])
    return X, np.ascontiguousarray(Y)


def cartesian_nodes(ni, nj, x_extent=1.0, y_extent=1.0):
    """Uniform Cartesian nodes, (nj+1, ni+1) each."""
    x = x_extent * (np.arange(ni + 1, dtype=np.float64) / ni)
    y = y_extent * (np.arange(nj + 1, dtype=np.float64) / nj)
    X = np.broadcast_to(x[None, :], (nj + 1, ni + 1)).copy()
    Y = np.broadcast_to(y[:, None], (nj + 1, ni + 1)).copy()
    return X, Y


def config_nodes(name):
    c = CONFIGS[name]
    return ramp_nodes(c["ni"], c["nj"], c["theta_deg"])


# --------------------------------------------------------------------------
# splitmix64 counter hash: r = hash(seed, cell, var).
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x):
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def uniform_pm1(seed, n_cells, n_var=4):
    """Counter-based uniforms in [-1, 1), shape (n_cells, n_var)."""
    cell = np.arange(n_cells, dtype=np.uint64)[:, None]
    var = np.arange(n_var, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        ctr = (np.uint64(seed) * np.uint64(0x100000000)
               + cell * np.uint64(n_var) + var) & _M64
    h = _splitmix64(_splitmix64(ctr))
    u = (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return 2.0 * u - 1.0


def perturbed_state(ni, nj, seed, amplitude=0.02, prim0=None):
    """Freestream with +-amplitude relative perturbations on (rho, u, v, p).

    v is perturbed relative to |u| (the freestream v is 0).  Returns the
    conserved state, shape (nj, ni, 4), index [j, i, k].  The default +-2%
    (SURVEY.md §8(c).5 proposed +-5%) keeps every MUSCL face state of the
    Mach-4 inlet valid with the bounded van Albada limiter.
    """
    if prim0 is None:
        prim0 = freestream_primitive()
    r = uniform_pm1(seed, ni * nj).reshape(nj, ni, 4)
    prim = np.empty((nj, ni, 4), dtype=np.float64)
    prim[..., 0] = prim0[0] * (1.0 + amplitude * r[..., 0])
    prim[..., 1] = prim0[1] * (1.0 + amplitude * r[..., 1])
    prim[..., 2] = prim0[2] + amplitude * abs(prim0[1]) * r[..., 2]
    prim[..., 3] = prim0[3] * (1.0 + amplitude * r[..., 3])
    return conserved_from_primitive(prim)


def uniform_state(ni, nj, U0=None):
    if U0 is None:
        U0 = freestream_conserved()
    return np.ascontiguousarray(
        np.broadcast_to(np.asarray(U0, np.float64), (nj, ni, 4)).copy())


def default_config(ni, nj, rk=RK4_CLASSIC, cfl=None, bc=None,
                   inflow=None, dt_fixed=0.0, harten_eps=0.1,
                   limiter=LIM_VAN_ALBADA2, lim_delta=1e-12, eps=1.0,
                   kappa=-1.0, gamma=GAMMA, max_history=4096, viscous=0, mu=0.0, prandtl=0.72,
                   gas_R=None):
    """The scheme settings of SURVEY.md §8(d) "common settings", except the
    limiter: van Albada in its bounded form psi = max(0, (2ab+d)/(a^2+b^2+d))
    (reading A-R3, revised).  It satisfies SPEC.md:166 (0 <= Psi
    <= 1), :177 and :180-182, and is Lipschitz; the VA1 form
    (a^2+ab+d)/(a^2+b^2+d) with the ab<0 switch is discontinuous for
    |b| << sqrt(d), which makes the discrete evolution amplify 1-ulp input
    noise to ~1e-9 (measured on the oracle itself), so it stays an option.

    Returns a plain dict consumed by both the oracle wrapper and the sfv
    binding.  bc order is (W, E, S, N).
    """
    if cfl is None:
        cfl = 0.5 if rk == RK2_HEUN else 0.8
    if bc is None:
        bc = (BC_INFLOW, BC_OUTFLOW, BC_SLIP_WALL, BC_SLIP_WALL)
    if inflow is None:
        inflow = freestream_conserved()
    inflow = np.asarray(inflow, np.float64)
    if inflow.shape == (4,):
        inflow = np.broadcast_to(inflow, (4, 4)).copy()
    return dict(ni=int(ni), nj=int(nj), gamma=float(gamma),
                muscl_eps=float(eps), muscl_kappa=float(kappa),
                limiter=int(limiter), lim_delta=float(lim_delta),
                harten_eps=float(harten_eps), rk=int(rk), cfl=float(cfl),
                dt_fixed=float(dt_fixed), bc=tuple(int(b) for b in bc),
                inflow_U=inflow, max_history=int(max_history),
                viscous=int(viscous), mu=float(mu), prandtl=float(prandtl),
                gas_R=float(R_GAS if gas_R is None else gas_R))
