"""Host-side tests of libsfv (no GPU): the C-ABI library loads, exports every
symbol include/sfv.h declares, validates its inputs, and its integer
partition / ghost maps are bit-exact with the oracle's."""
import os
import re

import numpy as np
import pytest

from paper_2305_18057_b200 import inputs as I
from paper_2305_18057_b200 import sfv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "sfv.h")).read()
    return sorted(set(re.findall(r"^\s*(?:sfv_status|void|const char \*)\s*(sfv_[a-z0-9_]+)\s*\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    L = sfv.lib()
    declared = header_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(sfv.ABI_SYMBOLS) == declared


def test_config_validation():
    X, Y = I.ramp_nodes(8, 4, 30.0)
    good = I.default_config(8, 4)
    for bad in [dict(ni=1), dict(gamma=1.0), dict(muscl_kappa=1.5), dict(muscl_eps=0.5), dict(cfl=0.0),
                dict(rk=7), dict(limiter=9), dict(max_history=0)]:
        cfg = dict(good, **bad)
        if "ni" in bad:
            Xb, Yb = I.ramp_nodes(1, 4, 30.0)
        else:
            Xb, Yb = X, Y
        with pytest.raises(sfv.SfvError) as ei:
            sfv.Solver(cfg, Xb, Yb, bind=False)
        assert ei.value.code == sfv.ERR_ARG, bad


def test_geometry_error_names_cell(oracle_mod):
    X, Y = I.cartesian_nodes(4, 3)
    X = X.copy(); X[1, 2] = 5.0   # node (2, 1) moved past node (3, 1): cell (2, 0) inverts
    with pytest.raises(sfv.SfvError) as ei:
        sfv.Solver(I.default_config(4, 3), X, Y, bind=False)
    assert ei.value.code == sfv.ERR_GEOMETRY
    assert ei.value.info[2:] == (2, 0)
    with pytest.raises(oracle_mod.OracleError) as eo:
        oracle_mod.metrics(X, Y)
    assert eo.value.info == 0 * 4 + 2


def test_split_bit_exact_with_oracle(oracle_mod):
    rng = np.random.default_rng(0)
    for _ in range(300):
        parts = int(rng.integers(1, 10))
        n = int(rng.integers(2 * parts, 5000))
        w = rng.integers(1, 50, parts)
        try:
            want = oracle_mod.split(n, parts, w)
        except oracle_mod.OracleError:
            with pytest.raises(sfv.SfvError):
                sfv.split(n, parts, w)
            continue
        np.testing.assert_array_equal(sfv.split(n, parts, w), want)
    np.testing.assert_array_equal(np.diff(sfv.split(96, 9, [40] + [1] * 8)), [80] + [2] * 8)


@pytest.mark.parametrize("px,py,wx,wy", [(1, 1, None, None), (2, 1, None, None), (4, 1, None, None),
                                         (8, 1, None, None), (4, 2, None, None), (2, 4, None, None),
                                         (1, 8, None, None), (8, 1, [4, 1, 1, 1, 1, 1, 1, 1], None),
                                         (8, 1, [1, 2, 3, 4, 5, 6, 7, 8], None), (3, 2, [1, 2, 3], [2, 1])])
def test_partition_maps_bit_exact(oracle_mod, px, py, wx, wy):
    ni, nj = 11520 // 8, 5760 // 8
    X, Y = I.ramp_nodes(ni, nj, 30.0)
    cfg = I.default_config(ni, nj)
    s = sfv.Solver(cfg, X, Y, px=px, py=py, wx=wx, wy=wy, bind=False)
    o = oracle_mod.Oracle(cfg, X, Y)
    o.partition(px, py, wx, wy)
    for b in range(px * py):
        np.testing.assert_array_equal(s.partition_map(b), o.partition_map(b))


def test_partition_rejects_narrow_blocks():
    X, Y = I.ramp_nodes(6, 4, 30.0)
    with pytest.raises(sfv.SfvError) as ei:
        sfv.Solver(I.default_config(6, 4), X, Y, px=4, bind=False)
    assert ei.value.code == sfv.ERR_ARG
    with pytest.raises(sfv.SfvError):
        sfv.Solver(I.default_config(6, 4), X, Y, px=2, py=1, rank=0, nranks=4, bind=False)


def test_bind_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    X, Y = I.ramp_nodes(8, 4, 30.0)
    s = sfv.Solver(I.default_config(8, 4), X, Y, bind=False)
    with pytest.raises(sfv.SfvError) as ei:
        s.bind()
    assert ei.value.code == sfv.ERR_CUDA


def test_halo_mode_calls_need_bind():
    """sfv_set_halo_mode / sfv_peer_handle / sfv_peer_connect before sfv_bind
    are sequence errors (host-side checks, no device needed)."""
    import ctypes as C
    X, Y = I.ramp_nodes(8, 4, 30.0)
    s = sfv.Solver(I.default_config(8, 4), X, Y, px=2, bind=False)
    L = sfv.lib()
    assert L.sfv_set_halo_mode(s._h, sfv.HALO_PEER) == sfv.ERR_SEQUENCE
    buf = (C.c_char * 128)()
    assert L.sfv_peer_handle(s._h, C.cast(buf, C.c_void_p)) == sfv.ERR_SEQUENCE
    assert L.sfv_peer_connect(s._h, C.cast(buf, C.c_void_p)) == sfv.ERR_SEQUENCE
    assert L.sfv_peer_handle(None, C.cast(buf, C.c_void_p)) == sfv.ERR_ARG


def test_noslip_and_viscous_validation():
    X, Y = I.ramp_nodes(8, 4, 30.0)
    with pytest.raises(sfv.SfvError) as ei:  # no-slip wall needs the viscous mode
        sfv.Solver(I.default_config(8, 4, bc=(0, 1, 3, 2)), X, Y, bind=False)
    assert ei.value.code == sfv.ERR_ARG
    with pytest.raises(sfv.SfvError) as ei:
        sfv.Solver(I.default_config(8, 4, viscous=1, mu=-1.0), X, Y, bind=False)
    assert ei.value.code == sfv.ERR_ARG
    s = sfv.Solver(I.default_config(8, 4, viscous=1, mu=0.1, bc=(0, 1, 3, 3)), X, Y, bind=False)
    s.close()
