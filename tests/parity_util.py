"""Comparison helpers for GPU-vs-oracle parity."""
import numpy as np


def state_error(U_gpu, U_orc):
    """e_k = max_c |dU_k| / s_k (reading A-R22): s_rho = max rho,
    s_mx = s_my = max |m|, s_E = max E over the oracle interior."""
    U_gpu = np.asarray(U_gpu).reshape(-1, 4)
    U_orc = np.asarray(U_orc).reshape(-1, 4)
    s = np.array([np.max(np.abs(U_orc[:, 0])),
                  np.max(np.hypot(U_orc[:, 1], U_orc[:, 2])),
                  np.max(np.hypot(U_orc[:, 1], U_orc[:, 2])),
                  np.max(np.abs(U_orc[:, 3]))])
    return np.max(np.abs(U_gpu - U_orc), axis=0) / s


def norm_error(n_gpu, n_orc):
    """|n_gpu - n_orc| / max(n_orc(step), n_orc(step 0)) per component."""
    n_gpu = np.asarray(n_gpu); n_orc = np.asarray(n_orc)
    scale = np.maximum(np.abs(n_orc), np.abs(n_orc[0:1]))
    scale = np.where(scale > 0, scale, 1.0)
    return np.max(np.abs(n_gpu - n_orc) / scale)


def dt_error(d_gpu, d_orc):
    return float(np.max(np.abs(np.asarray(d_gpu) - np.asarray(d_orc)) / np.abs(np.asarray(d_orc))))
