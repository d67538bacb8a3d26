"""ctypes wrapper of the plain C oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product path
(paper_2305_18057_b200) never imports this package, and this package never
imports the product's CUDA binding.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
LIB_OMP_PATH = os.path.join(HERE, "liboracle_omp.so")  # same source, -fopenmp (bench.py all-cores baseline)
SRC = os.path.join(HERE, "oracle.c")

ORC_OK, ORC_ERR_ARG, ORC_ERR_GEOMETRY, ORC_ERR_STATE, ORC_ERR_SEQUENCE = range(5)
RES_EULER, RES_LINEAR = 0, 1


class OracleError(RuntimeError):
    def __init__(self, code, msg, info=None):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code
        self.info = info


def build(force=False, omp=False):
    """Compile liboracle.so: -O2 -ffp-contract=off (no FMA contraction);
    omp=True: liboracle_omp.so, the same source with -fopenmp (row loops
    shared among threads, bitwise equal to the single-threaded build)."""
    path = LIB_OMP_PATH if omp else LIB_PATH
    if (not force and os.path.exists(path)
            and os.path.getmtime(path) >= max(os.path.getmtime(SRC),
                                              os.path.getmtime(os.path.join(HERE, "oracle.h")))):
        return path
    cmd = ["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math",
           *(["-fopenmp"] if omp else []), "-fPIC", "-shared", "-o", path + ".tmp", SRC, "-lm"]
    subprocess.check_call(cmd)
    os.replace(path + ".tmp", path)
    return path


class orc_config(C.Structure):
    _fields_ = [("ni", C.c_int32), ("nj", C.c_int32), ("gamma", C.c_double),
                ("muscl_eps", C.c_double), ("muscl_kappa", C.c_double),
                ("limiter", C.c_int32), ("lim_delta", C.c_double),
                ("harten_eps", C.c_double), ("rk", C.c_int32),
                ("cfl", C.c_double), ("dt_fixed", C.c_double),
                ("bc", C.c_int32 * 4), ("inflow_U", (C.c_double * 4) * 4),
                ("max_history", C.c_int64), ("residual_kind", C.c_int32),
                ("linear_rate", C.c_double), ("viscous", C.c_int32), ("mu", C.c_double),
                ("prandtl", C.c_double), ("gas_R", C.c_double)]


_lib = None
_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)


_lib_omp = None


def lib(omp=False):
    global _lib, _lib_omp
    if omp:
        if _lib_omp is None:
            build(omp=True)
            _lib_omp = _declare(C.CDLL(LIB_OMP_PATH))
        return _lib_omp
    if _lib is None:
        build()
        _lib = _declare(C.CDLL(LIB_PATH))
    return _lib


def _declare(L):
    if True:
        L.orc_metrics.argtypes = [C.c_int32, C.c_int32, _D, _D, _D, _D, _D, _I64]
        L.orc_primitive.argtypes = [_D, C.c_double, _D]
        L.orc_limiter.argtypes = [C.c_int32, C.c_double, C.c_double, C.c_double]
        L.orc_limiter.restype = C.c_double
        L.orc_muscl.argtypes = [_D, C.c_double, C.c_double, C.c_int32, C.c_double, _D, _D]
        L.orc_muscl.restype = None
        L.orc_roe_flux.argtypes = [_D, _D, C.c_double, C.c_double, C.c_double, C.c_double, _D]
        L.orc_split.argtypes = [C.c_int32, C.c_int32, _I32, _I32]
        L.orc_stable_dt.argtypes = [C.c_int32, C.c_int32, _D, _D, _D, C.c_double, C.c_double, _D]
        L.orc_create.argtypes = [C.POINTER(orc_config), _D, _D, C.POINTER(C.c_void_p)]
        L.orc_partition.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _I32, _I32]
        L.orc_partition_map.argtypes = [C.c_void_p, C.c_int32, _I32]
        L.orc_set_state.argtypes = [C.c_void_p, _D]
        L.orc_step.argtypes = [C.c_void_p, C.c_int32]
        L.orc_get_state.argtypes = [C.c_void_p, _D]
        L.orc_get_residual_norms.argtypes = [C.c_void_p, C.c_int64, C.c_int64, _D]
        L.orc_get_dt.argtypes = [C.c_void_p, C.c_int64, C.c_int64, _D]
        L.orc_residual.argtypes = [C.c_void_p, _D, _D]
        L.orc_ghost_frame.argtypes = [C.c_void_p, _D, _D]
        L.orc_gradients.argtypes = [C.c_void_p, _D, _D]
        L.orc_viscous_flux.argtypes = [_D, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                       C.c_double, _D]
        L.orc_viscous_flux.restype = None
        L.orc_steps_done.argtypes = [C.c_void_p]
        L.orc_steps_done.restype = C.c_int64
        L.orc_error_info.argtypes = [C.c_void_p, _I64]
        L.orc_error_info.restype = None
        L.orc_last_error.argtypes = [C.c_void_p]
        L.orc_last_error.restype = C.c_char_p
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_destroy.restype = None
    return L


def _dp(a):
    return a.ctypes.data_as(_D)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


# ---------------------------------------------------------------- pointwise
def metrics(X, Y):
    X = _f64(X); Y = _f64(Y)
    nj, ni = X.shape[0] - 1, X.shape[1] - 1
    iface = np.empty((nj, ni + 1, 3)); jface = np.empty((nj + 1, ni, 3))
    vol = np.empty((nj, ni)); bad = C.c_int64(-1)
    st = lib().orc_metrics(ni, nj, _dp(X), _dp(Y), _dp(iface), _dp(jface), _dp(vol), C.byref(bad))
    if st:
        raise OracleError(st, f"non-positive volume at cell {bad.value}", bad.value)
    return iface, jface, vol


def primitive(U, gamma=1.4):
    U = _f64(U, (4,)); out = np.empty(4)
    st = lib().orc_primitive(_dp(U), gamma, _dp(out))
    if st:
        raise OracleError(st, "invalid state")
    return out


def limiter(kind, a, b, delta=1e-12):
    return lib().orc_limiter(kind, a, b, delta)


def muscl(w, eps=1.0, kappa=-1.0, kind=0, delta=1e-12):
    w = _f64(w, (4,)); qL = C.c_double(); qR = C.c_double()
    lib().orc_muscl(_dp(w), eps, kappa, kind, delta, C.byref(qL), C.byref(qR))
    return qL.value, qR.value


def roe_flux(QL, QR, nx, ny, gamma=1.4, harten_eps=0.1):
    QL = _f64(QL, (4,)); QR = _f64(QR, (4,)); F = np.empty(4)
    st = lib().orc_roe_flux(_dp(QL), _dp(QR), nx, ny, gamma, harten_eps, _dp(F))
    if st:
        raise OracleError(st, "invalid face state")
    return F


def viscous_flux(grad, u, v, nx, ny, mu, k):
    """F_v . n (Eq. 2 viscous flux) from face gradients (u_x, u_y, v_x, v_y, T_x, T_y)."""
    g = _f64(grad, (6,)); F = np.empty(4)
    lib().orc_viscous_flux(_dp(g), u, v, nx, ny, mu, k, _dp(F))
    return F


def split(n, parts, weights=None):
    starts = np.zeros(parts + 1, dtype=np.int32)
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.int32)
    st = lib().orc_split(n, parts, None if w is None else w.ctypes.data_as(_I32),
                         starts.ctypes.data_as(_I32))
    if st:
        raise OracleError(st, "bad split")
    return starts


def stable_dt(X, Y, U, gamma=1.4, cfl=0.8):
    """CFL dt of a whole grid (same arithmetic as the solver's dt), banded."""
    X = _f64(X); Y = _f64(Y); U = _f64(U)
    nj, ni = X.shape[0] - 1, X.shape[1] - 1
    out = C.c_double()
    st = lib().orc_stable_dt(ni, nj, _dp(X), _dp(Y), _dp(U), gamma, cfl, C.byref(out))
    if st:
        raise OracleError(st, "stable_dt")
    return out.value


# ------------------------------------------------------------------- solver
def make_config(d, residual_kind=RES_EULER, linear_rate=0.0):
    c = orc_config()
    c.ni, c.nj = d["ni"], d["nj"]
    c.gamma = d["gamma"]; c.muscl_eps = d["muscl_eps"]; c.muscl_kappa = d["muscl_kappa"]
    c.limiter = d["limiter"]; c.lim_delta = d["lim_delta"]; c.harten_eps = d["harten_eps"]
    c.rk = d["rk"]; c.cfl = d["cfl"]; c.dt_fixed = d["dt_fixed"]
    for e in range(4):
        c.bc[e] = d["bc"][e]
        for k in range(4):
            c.inflow_U[e][k] = float(d["inflow_U"][e][k])
    c.max_history = d["max_history"]
    c.residual_kind = residual_kind; c.linear_rate = linear_rate
    c.viscous = int(d.get("viscous", 0)); c.mu = float(d.get("mu", 0.0))
    c.prandtl = float(d.get("prandtl", 0.72)); c.gas_R = float(d.get("gas_R", 287.0))
    return c


class Oracle:
    """Mirror of the sfv C ABI on the CPU (SURVEY.md §8(b) 'oracle mirror')."""

    def __init__(self, cfg, X, Y, residual_kind=RES_EULER, linear_rate=0.0, omp=False):
        """omp=True: the -fopenmp build (thread count from OMP_NUM_THREADS)."""
        self._L = lib(omp)
        self.cfg = dict(cfg)
        self._c = make_config(cfg, residual_kind, linear_rate)
        self._X = _f64(X); self._Y = _f64(Y)
        h = C.c_void_p()
        self._h = None
        st = self._L.orc_create(C.byref(self._c), _dp(self._X), _dp(self._Y), C.byref(h))
        if st:
            raise OracleError(st, "orc_create failed")
        self._h = h
        self.ni, self.nj = cfg["ni"], cfg["nj"]

    def _check(self, st):
        if st:
            info = np.zeros(4, np.int64)
            self._L.orc_error_info(self._h, info.ctypes.data_as(_I64))
            raise OracleError(st, self._L.orc_last_error(self._h).decode(), tuple(int(v) for v in info))

    def partition(self, px, py, wx=None, wy=None):
        wxa = None if wx is None else np.ascontiguousarray(wx, np.int32)
        wya = None if wy is None else np.ascontiguousarray(wy, np.int32)
        self._check(self._L.orc_partition(self._h, px, py,
                                        None if wxa is None else wxa.ctypes.data_as(_I32),
                                        None if wya is None else wya.ctypes.data_as(_I32)))
        self.nblocks = px * py

    def partition_map(self, block):
        out = np.zeros(8, np.int32)
        self._check(self._L.orc_partition_map(self._h, block, out.ctypes.data_as(_I32)))
        return out

    def set_state(self, U):
        U = _f64(U, (self.nj, self.ni, 4))
        self._check(self._L.orc_set_state(self._h, _dp(U)))

    def step(self, n=1):
        self._check(self._L.orc_step(self._h, n))

    def get_state(self):
        U = np.empty((self.nj, self.ni, 4))
        self._check(self._L.orc_get_state(self._h, _dp(U)))
        return U

    @property
    def steps_done(self):
        return self._L.orc_steps_done(self._h)

    def residual_norms(self, first=0, count=None):
        if count is None:
            count = self.steps_done - first
        out = np.empty((count, 8))
        self._check(self._L.orc_get_residual_norms(self._h, first, count, _dp(out)))
        return out

    def dt(self, first=0, count=None):
        if count is None:
            count = self.steps_done - first
        out = np.empty(count)
        self._check(self._L.orc_get_dt(self._h, first, count, _dp(out)))
        return out

    def residual(self, U):
        U = _f64(U, (self.nj, self.ni, 4)); R = np.empty_like(U)
        self._check(self._L.orc_residual(self._h, _dp(U), _dp(R)))
        return R

    def gradients(self, U):
        """Green-Gauss cell gradients (u_x, u_y, v_x, v_y, T_x, T_y), [nj, ni, 6]."""
        U = _f64(U, (self.nj, self.ni, 4)); G = np.empty((self.nj, self.ni, 6))
        self._check(self._L.orc_gradients(self._h, _dp(U), _dp(G)))
        return G

    def ghost_frame(self, U):
        U = _f64(U, (self.nj, self.ni, 4))
        F = np.empty((self.nj + 4, self.ni + 4, 4))
        self._check(self._L.orc_ghost_frame(self._h, _dp(U), _dp(F)))
        return F

    def close(self):
        if self._h is not None:
            self._L.orc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
