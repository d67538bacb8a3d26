"""Thin ctypes binding of libsfv.so (include/sfv.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this
module never computes any part of the method, and there is no CPU fallback:
if libsfv.so is missing or no device is present the calls raise.  PyTorch is
used only for device memory (the workspace) and the CUDA stream.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import inputs as _inputs

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SFV_LIB") or os.path.join(HERE, "libsfv.so")  # SFV_LIB: A/B builds only

OK, ERR_ARG, ERR_GEOMETRY, ERR_STATE, ERR_SEQUENCE, ERR_CUDA, ERR_NCCL, ERR_OOM, ERR_UNSUPPORTED, ERR_HALO = range(10)
_NAMES = ["OK", "ARG", "GEOMETRY", "STATE", "SEQUENCE", "CUDA", "NCCL", "OOM", "UNSUPPORTED", "HALO"]
HALO_COPY, HALO_PEER = 0, 1

# every entry point declared in include/sfv.h
ABI_SYMBOLS = ["sfv_create", "sfv_partition", "sfv_nccl_unique_id", "sfv_partition_map", "sfv_halo_plan",
               "sfv_split",
               "sfv_workspace_size", "sfv_bind", "sfv_set_state", "sfv_step", "sfv_sync", "sfv_steps_done",
               "sfv_get_residual_norms", "sfv_get_dt", "sfv_get_state", "sfv_error_info", "sfv_launch_info",
               "sfv_debug_math", "sfv_set_halo_mode", "sfv_peer_handle", "sfv_peer_connect",
               "sfv_debug_block_buffer", "sfv_residual", "sfv_set_profiling", "sfv_get_stage_timings",
               "sfv_set_comm_timeout", "sfv_get_block_state", "sfv_last_error", "sfv_destroy"]


class SfvError(RuntimeError):
    def __init__(self, code, msg, info=None):
        super().__init__(f"sfv error {_NAMES[code] if 0 <= code < len(_NAMES) else code}: {msg}")
        self.code = code
        self.info = info


class sfv_config(C.Structure):
    _fields_ = [("ni", C.c_int32), ("nj", C.c_int32), ("gamma", C.c_double),
                ("muscl_eps", C.c_double), ("muscl_kappa", C.c_double),
                ("limiter", C.c_int32), ("lim_delta", C.c_double),
                ("harten_eps", C.c_double), ("rk", C.c_int32),
                ("cfl", C.c_double), ("dt_fixed", C.c_double),
                ("bc", C.c_int32 * 4), ("inflow_U", (C.c_double * 4) * 4),
                ("max_history", C.c_int64), ("viscous", C.c_int32), ("mu", C.c_double),
                ("prandtl", C.c_double), ("gas_R", C.c_double)]


_lib = None
_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)
_VP = C.c_void_p


def lib():
    """Load libsfv.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.sfv_create.argtypes = [C.POINTER(sfv_config), _D, _D, C.POINTER(_VP)]
        L.sfv_partition.argtypes = [_VP, C.c_int32, C.c_int32, _I32, _I32, C.c_int32, C.c_int32, _VP, C.c_int32]
        L.sfv_nccl_unique_id.argtypes = [_VP]
        L.sfv_partition_map.argtypes = [_VP, C.c_int32, _I32]
        L.sfv_halo_plan.argtypes = [_VP, C.c_int32, _I32]
        L.sfv_split.argtypes = [C.c_int32, C.c_int32, _I32, _I32]
        L.sfv_workspace_size.argtypes = [_VP, C.POINTER(C.c_size_t)]
        L.sfv_bind.argtypes = [_VP, _VP, C.c_size_t, _VP]
        L.sfv_set_state.argtypes = [_VP, _D]
        L.sfv_step.argtypes = [_VP, C.c_int32]
        L.sfv_sync.argtypes = [_VP, _D]
        L.sfv_steps_done.argtypes = [_VP, _I64]
        L.sfv_get_residual_norms.argtypes = [_VP, C.c_int64, C.c_int64, _D]
        L.sfv_get_dt.argtypes = [_VP, C.c_int64, C.c_int64, _D]
        L.sfv_get_state.argtypes = [_VP, _D]
        L.sfv_error_info.argtypes = [_VP, _I64]
        L.sfv_launch_info.argtypes = [_VP, _I32]
        L.sfv_debug_math.argtypes = [_VP, C.c_int32, _VP, _VP, C.c_int64]
        L.sfv_set_halo_mode.argtypes = [_VP, C.c_int32]
        L.sfv_peer_handle.argtypes = [_VP, _VP]
        L.sfv_peer_connect.argtypes = [_VP, _VP]
        L.sfv_debug_block_buffer.argtypes = [_VP, C.c_int32, C.c_int32, _D]
        L.sfv_residual.argtypes = [_VP, _D, _D]
        # (round-2 entry points; an older library build -- A/B experiments
        # via SFV_LIB -- may lack them, every other call still works)
        for name, at in (("sfv_set_profiling", [_VP, C.c_int32]), ("sfv_get_stage_timings", [_VP, _D]),
                         ("sfv_set_comm_timeout", [_VP, C.c_double]),
                         ("sfv_get_block_state", [_VP, C.c_int32, _D])):
            if hasattr(L, name):
                getattr(L, name).argtypes = at
        L.sfv_last_error.argtypes = [_VP]
        L.sfv_last_error.restype = C.c_char_p
        L.sfv_destroy.argtypes = [_VP]
        L.sfv_destroy.restype = None
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(_D)


def make_config(d):
    c = sfv_config()
    c.ni, c.nj = d["ni"], d["nj"]
    c.gamma = d["gamma"]; c.muscl_eps = d["muscl_eps"]; c.muscl_kappa = d["muscl_kappa"]
    c.limiter = d["limiter"]; c.lim_delta = d["lim_delta"]; c.harten_eps = d["harten_eps"]
    c.rk = d["rk"]; c.cfl = d["cfl"]; c.dt_fixed = d["dt_fixed"]
    for e in range(4):
        c.bc[e] = d["bc"][e]
        for k in range(4):
            c.inflow_U[e][k] = float(d["inflow_U"][e][k])
    c.max_history = d["max_history"]
    c.viscous = int(d.get("viscous", 0)); c.mu = float(d.get("mu", 0.0))
    c.prandtl = float(d.get("prandtl", 0.72)); c.gas_R = float(d.get("gas_R", 287.0))
    return c


def split(n, parts, weights=None):
    """Host-only largest-remainder split through the C ABI."""
    starts = np.zeros(parts + 1, np.int32)
    w = None if weights is None else np.ascontiguousarray(weights, np.int32)
    st = lib().sfv_split(n, parts, None if w is None else w.ctypes.data_as(_I32), starts.ctypes.data_as(_I32))
    if st:
        raise SfvError(st, "sfv_split")
    return starts


def nccl_unique_id():
    buf = (C.c_char * 128)()
    st = lib().sfv_nccl_unique_id(C.cast(buf, _VP))
    if st:
        raise SfvError(st, "sfv_nccl_unique_id")
    return bytes(buf)


class Solver:
    """One ctx of the C ABI.  `bind=False` keeps it host-only (partition maps)."""

    def __init__(self, cfg, X, Y, px=1, py=1, wx=None, wy=None, rank=0, nranks=1, nccl_id=None,
                 device=None, stream=None, bind=True):
        self.cfg = dict(cfg)
        self.ni, self.nj = cfg["ni"], cfg["nj"]
        self._c = make_config(cfg)
        X = np.ascontiguousarray(X, np.float64); Y = np.ascontiguousarray(Y, np.float64)
        h = _VP()
        self._h = None
        st = lib().sfv_create(C.byref(self._c), _dp(X), _dp(Y), C.byref(h))
        if st:
            info = None
            if h.value:
                info = self._info(h)
                msg = lib().sfv_last_error(h).decode()
                lib().sfv_destroy(h)
            else:
                msg = "sfv_create rejected the configuration"
            raise SfvError(st, msg, info)
        self._h = h
        self.px, self.py = px, py
        self.rank, self.nranks = rank, nranks
        wxa = None if wx is None else np.ascontiguousarray(wx, np.int32)
        wya = None if wy is None else np.ascontiguousarray(wy, np.int32)
        idbuf = None
        if nccl_id is not None:
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        if device is None:
            device = 0
        self.device = device
        self._check(lib().sfv_partition(h, px, py, None if wxa is None else wxa.ctypes.data_as(_I32),
                                        None if wya is None else wya.ctypes.data_as(_I32), rank, nranks,
                                        None if idbuf is None else C.cast(idbuf, _VP), device))
        self.ws = None
        if bind:
            self.bind(stream)

    @staticmethod
    def _info(h):
        info = np.zeros(4, np.int64)
        lib().sfv_error_info(h, info.ctypes.data_as(_I64))
        return tuple(int(v) for v in info)

    def _check(self, st):
        if st:
            raise SfvError(st, lib().sfv_last_error(self._h).decode(), self._info(self._h))

    def bind(self, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise SfvError(ERR_CUDA, "no CUDA device: the sfv hot path has no CPU fallback")
        dev = torch.device("cuda", self.device)
        n = C.c_size_t()
        self._check(lib().sfv_workspace_size(self._h, C.byref(n)))
        if stream is None:
            stream = torch.cuda.current_stream(dev)
        # allocated on the stream the kernels run on, so the caching allocator
        # cannot hand the memory out again while this stream still uses it
        with torch.cuda.stream(stream):
            self.ws = torch.empty(n.value, dtype=torch.uint8, device=dev)
        self.stream = stream
        self._check(lib().sfv_bind(self._h, C.c_void_p(self.ws.data_ptr()), n.value,
                                   C.c_void_p(stream.cuda_stream)))
        return n.value

    def set_halo_mode(self, mode):
        """sfv_set_halo_mode; call set_state afterwards."""
        self._check(lib().sfv_set_halo_mode(self._h, int(mode)))

    def peer_handle(self):
        buf = (C.c_char * 128)()
        self._check(lib().sfv_peer_handle(self._h, C.cast(buf, _VP)))
        return bytes(buf)

    def peer_connect(self, handles):
        """handles: list of nranks 128-byte descriptors (rank order)."""
        blob = C.create_string_buffer(b"".join(bytes(h) for h in handles), 128 * len(handles))
        self._check(lib().sfv_peer_connect(self._h, C.cast(blob, _VP)))

    def enable_peer_halo(self, group=None):
        """Device-initiated halo exchange (SFV_HALO_PEER).  With nranks > 1 the
        128-byte descriptors are all-gathered over torch.distributed first."""
        if self.nranks > 1:
            import torch.distributed as dist
            hs = [None] * self.nranks
            dist.all_gather_object(hs, self.peer_handle(), group=group)
            self.peer_connect(hs)
        self.set_halo_mode(HALO_PEER)

    def partition_map(self, block):
        out = np.zeros(8, np.int32)
        self._check(lib().sfv_partition_map(self._h, block, out.ctypes.data_as(_I32)))
        return out

    def halo_plan(self, block):
        """(4, 9) int32: per edge W, E, S, N: nbr, send i0,i1,j0,j1, recv i0,i1,j0,j1."""
        out = np.zeros(36, np.int32)
        self._check(lib().sfv_halo_plan(self._h, block, out.ctypes.data_as(_I32)))
        return out.reshape(4, 9)

    def set_state(self, U):
        U = np.ascontiguousarray(U, np.float64)
        assert U.size == self.ni * self.nj * 4
        self._check(lib().sfv_set_state(self._h, _dp(U)))

    def set_state_ptr(self, ptr):
        """Host pointer variant (e.g. a pinned torch tensor's data_ptr())."""
        self._check(lib().sfv_set_state(self._h, C.cast(C.c_void_p(ptr), _D)))

    def step(self, n=1):
        self._check(lib().sfv_step(self._h, n))

    def sync(self):
        ms = C.c_double()
        self._check(lib().sfv_sync(self._h, C.byref(ms)))
        return ms.value

    @property
    def steps_done(self):
        n = C.c_int64()
        self._check(lib().sfv_steps_done(self._h, C.byref(n)))
        return n.value

    def get_state(self, out=None):
        if out is None:
            out = np.empty((self.nj, self.ni, 4))
        self._check(lib().sfv_get_state(self._h, _dp(out)))
        return out

    def get_block_state(self, block=None, out=None):
        """sfv_get_block_state: this rank's block (default: block `rank`), [nj_b, ni_b, 4]."""
        b = self.rank if block is None else block
        m = self.partition_map(b)
        if out is None:
            out = np.empty((int(m[3] - m[2]), int(m[1] - m[0]), 4))
        self._check(lib().sfv_get_block_state(self._h, b, _dp(out)))
        return out

    def get_block_state_ptr(self, block, ptr):
        self._check(lib().sfv_get_block_state(self._h, block, C.cast(C.c_void_p(ptr), _D)))

    def get_state_ptr(self, ptr):
        self._check(lib().sfv_get_state(self._h, C.cast(C.c_void_p(ptr), _D)))

    def residual(self, U):
        """R_h(U) of Eq. 5 on the device (sfv_residual), [nj, ni, 4]."""
        U = np.ascontiguousarray(U, np.float64)
        out = np.empty((self.nj, self.ni, 4))
        self._check(lib().sfv_residual(self._h, _dp(U), _dp(out)))
        return out

    def residual_norms(self, first=0, count=None):
        if count is None:
            count = self.steps_done - first
        out = np.empty((count, 8))
        self._check(lib().sfv_get_residual_norms(self._h, first, count, _dp(out)))
        return out

    def dt(self, first=0, count=None):
        if count is None:
            count = self.steps_done - first
        out = np.empty(count)
        self._check(lib().sfv_get_dt(self._h, first, count, _dp(out)))
        return out

    def launch_info(self):
        out = np.zeros(4, np.int32)
        self._check(lib().sfv_launch_info(self._h, out.ctypes.data_as(_I32)))
        return dict(strips=int(out[0]), segments=int(out[1]), threads=int(out[2]), ctas_per_sm=int(out[3]))

    def debug_math(self, which, x_dev, out_dev):
        self._check(lib().sfv_debug_math(self._h, which, C.c_void_p(x_dev.data_ptr()),
                                         C.c_void_p(out_dev.data_ptr()), x_dev.numel()))

    def block_buffer(self, block, k):
        """Diagnostic: state buffer k of local block `block` with its ghost
        frame, as an array [ni_b+4, 4, nj_b+4] (index i+2, c, j+2)."""
        m = self.partition_map(block)
        nib, njb = int(m[1] - m[0]), int(m[3] - m[2])
        out = np.empty((nib + 2, 6, njb + 2)) if k == -2 else np.empty((nib + 4, 4, njb + 4))
        self._check(lib().sfv_debug_block_buffer(self._h, block, k, _dp(out)))
        return out

    def set_profiling(self, on=True):
        """sfv_set_profiling: per-class CUDA-event timers (no CUDA graph)."""
        self._check(lib().sfv_set_profiling(self._h, 1 if on else 0))

    PROFILE_CLASSES = ("edge", "interior", "row_exchange", "col_exchange", "exposed_wait", "dt_allreduce",
                       "viscous", "norms")

    def stage_timings(self):
        """sfv_get_stage_timings -> dict of accumulated ms per class + 'steps'."""
        out = np.zeros(9)
        self._check(lib().sfv_get_stage_timings(self._h, _dp(out)))
        d = {k: float(v) for k, v in zip(self.PROFILE_CLASSES, out[:8])}
        d["steps"] = int(out[8])
        return d

    def set_comm_timeout(self, seconds):
        """sfv_set_comm_timeout: NCCL deadlock detection."""
        self._check(lib().sfv_set_comm_timeout(self._h, float(seconds)))

    @property
    def error_info(self):
        return self._info(self._h)

    def close(self):
        if self._h is not None:
            lib().sfv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def inlet_solver(name="C2", rk=_inputs.RK4_CLASSIC, **kw):
    """Solver on one of the BASELINE configurations (inputs.CONFIGS)."""
    X, Y = _inputs.config_nodes(name)
    c = _inputs.CONFIGS[name]
    cfg = _inputs.default_config(c["ni"], c["nj"], rk=rk)
    return Solver(cfg, X, Y, **kw), cfg
