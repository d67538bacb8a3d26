"""Host checks of the paper's performance model (Eqs. 8-14)
as implemented in paper_2305_18057_b200/perfmodel.py."""
import numpy as np
import pytest

from paper_2305_18057_b200 import perfmodel as M


def test_ssspnt_definition():
    # Eq. 14 with s = 1e-6: 1e6 cells x 100 steps on 1 unit in 10 s -> 10
    assert M.ssspnt(1_000_000, 100, 1, 10.0) == pytest.approx(10.0)
    assert M.ssspnt(1_000_000, 100, 4, 10.0) == pytest.approx(2.5)


def test_eq13_special_cases():
    Nl, Nw, tI, beta = 1000, 200, 2e-9, 0.3
    # G = 1, r_gc = 1, C = 0, alpha = 0: Eq. 9 with C = 1 and t_B = beta t_I
    assert M.time_hete(Nl, Nw, tI, beta, 0.0) == pytest.approx(M.time_cpu(Nl, Nw, 1, tI, beta * tI))
    # C CPUs only (G = 0): Eq. 9
    assert M.time_hete(Nl, Nw, tI, beta, 0.0, G=0, C=8) == pytest.approx(M.time_cpu(Nl, Nw, 8, tI, beta * tI))
    # Eq. 8 with N_d = 1 counts 2 N_l N_w + 2 N_l + 2 N_w boundary cells
    assert M.time_seq(Nl, Nw, 1, tI, beta * tI) == pytest.approx((Nl * Nw + (2 * Nl * Nw + 2 * Nl + 2 * Nw) * beta) * tI)
    # alpha scales only the boundary term
    d = M.time_hete(Nl, Nw, tI, beta, 1.0) - M.time_hete(Nl, Nw, tI, beta, 0.0)
    assert d == pytest.approx((2 * Nw + 2 * Nl) * beta * tI)


def test_heterogeneous_ratio_example():
    """SPEC-style check: (G, C, r_gc) = (1, 8, 40) speeds the interior term up
    by (40 + 8) / 40 = 1.2 over the GPU alone."""
    Nl, Nw = 10**6, 10
    g = M.time_hete(Nl, Nw, 1.0, 0.0, 0.0, G=1, rgc=40.0, C=0)
    h = M.time_hete(Nl, Nw, 1.0, 0.0, 0.0, G=1, rgc=40.0, C=8)
    assert g / h == pytest.approx(1.2)


@pytest.mark.parametrize("n,parts,w", [(10, 3, None), (11520, 8, [4, 1, 1, 1, 1, 1, 1, 1]),
                                       (11520, 8, [1, 2, 3, 4, 5, 6, 7, 8]), (5760, 7, None), (70, 3, None)])
def test_split_matches_library(n, parts, w):
    """The planner's split equals the C library's sfv_split (host-only call)."""
    from paper_2305_18057_b200 import sfv
    starts = sfv.split(n, parts, w)
    assert M.split(n, parts, w) == list(np.diff(starts))


def test_fit_recovers_synthetic_parameters():
    true = M.GpuModel(tI=1.5e-11, tB=4e-10, tL=5e-6)
    rng = np.random.default_rng(0)
    samples = []
    for px, py in [(1, 1), (2, 1), (8, 1), (4, 2), (2, 4), (1, 8)]:
        for ni, nj in [(1440, 720), (11520, 5760), (5760, 2880)]:
            bl = M.blocks_of(ni, nj, px, py)
            samples.append((bl, true.loopback_step(bl) * (1 + 1e-4 * rng.standard_normal())))
    fit = M.fit(samples)
    assert fit.tI == pytest.approx(true.tI, rel=1e-3)
    assert fit.tB == pytest.approx(true.tB, rel=5e-2)
    assert fit.tL == pytest.approx(true.tL, rel=5e-2)


def test_multi_gpu_is_max_over_ranks():
    m = M.GpuModel(tI=1e-11, tB=1e-10, tL=1e-6)
    even = M.blocks_of(11520, 5760, 8, 1)
    skew = M.blocks_of(11520, 5760, 8, 1, wx=[4, 1, 1, 1, 1, 1, 1, 1])
    assert m.multi_gpu_step(skew) > m.multi_gpu_step(even)
    assert m.multi_gpu_step(even) == pytest.approx(m.stages * m.block_stage(even[0]))


def test_closure_script_predicts_and_calibrates_alpha(tmp_path):
    """scripts/perfmodel_closure.py (SURVEY §8(f) f3 closure): every bench line
    in a file gets the launch-geometry model's prediction for its slab
    decomposition; alpha (Eq. 12) comes from the line's measured halo time
    (config.halo_measured: slab alone vs in the N-rank run)."""
    import json
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "scripts"))
    import perfmodel_closure as PC
    line = {"metric": "m", "value": 1.0, "n_gpus": 4, "ms_per_step": 3.0,
            "config": {"workload": "C3 strong scaling, 11520x5760 = 66,355,200 cells", "global_cells": 66355200,
                       "rk_stages": 4, "halo_measured": {"slab_alone_ms_per_step_max": 2.5}}}
    f = tmp_path / "scale.json"
    f.write_text(json.dumps({"runs": [{"stdout_tail": "== bench\n" + json.dumps(line) + "\n"}]}))
    sys.argv = ["perfmodel_closure.py", str(f)]
    rows = PC.main()
    assert len(rows) == 1 and rows[0]["n"] == 4 and rows[0]["grid"] == "11520x5760"
    assert abs(rows[0]["alpha"] - (3.0 / 2.5 - 1.0)) < 1e-12
    assert rows[0]["predicted_ms"] > 0 and rows[0]["predicted_alpha_ms"] > rows[0]["predicted_ms"]
