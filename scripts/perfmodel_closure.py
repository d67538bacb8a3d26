#!/usr/bin/env python
"""Close the performance-model loop (Eqs. 12-13):
predicted vs measured multi-GPU step times.

    python scripts/perfmodel_closure.py FILE [FILE ...] [--model profiles/r1_perfmodel.json]

FILE may be a bench.py JSON line file, a driver BENCH_r*.json / SCALE_r*.json
(any JSON object with a "metric" key is taken, including ones embedded in
stdout tails).  For every bench line with n_gpus >= 1 the script rebuilds the
slab decomposition (px = n_gpus, the library's largest-remainder split),
predicts the step time with the GPU-native launch-geometry model calibrated
on one B200 (perfmodel.GeometryModel: per stage t_L + t_row waves (rows+1.5),
max over ranks), and prints measured vs predicted.

alpha (Eq. 12, t_f = alpha T_b: exchange and synchronisation charged to the
block) is calibrated from the line's own measurement when bench.py recorded
one (config.halo_measured: each rank's slab timed alone vs inside the N-rank run):
alpha = t_multi / t_alone - 1 for the slowest rank; the prediction with
alpha is then t_model (1 + alpha).  Lines whose ranks shared one GPU
(config.simulated_ranks_on_one_gpu) are flagged: their times are
time-sliced, not a multi-GPU measurement.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2305_18057_b200 import perfmodel as PM  # noqa: E402


def bench_lines(path):
    txt = open(path).read()
    out = []

    def visit(o):
        if isinstance(o, dict):
            if "metric" in o and "ms_per_step" in o:
                out.append(o)
            for v in o.values():
                visit(v)
        elif isinstance(o, list):
            for v in o:
                visit(v)
        elif isinstance(o, str) and '"metric"' in o:
            for m in re.finditer(r"\{\"metric\".*?\}(?=\s*$|\n)", o, re.M):
                try:
                    visit(json.loads(m.group(0)))
                except ValueError:
                    pass
    try:
        visit(json.loads(txt))
    except ValueError:
        for line in txt.splitlines():
            line = line.strip()
            if line.startswith("{"):
                try:
                    visit(json.loads(line))
                except ValueError:
                    pass
    return out


def grid_of(line):
    cfg = line.get("config", {})
    w = cfg.get("workload", "")
    m = re.search(r"global (\d+)x(\d+)", w) or re.search(r"(\d+)x(\d+) =", w)
    if m:
        return int(m.group(1)), int(m.group(2))
    cells = cfg.get("global_cells")
    if cells == 66355200:
        return 11520, 5760
    if cells == 1036800:
        return 1440, 720
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("files", nargs="+")
    ap.add_argument("--model", default=os.path.join(ROOT, "profiles", "r1_perfmodel.json"))
    args = ap.parse_args()
    mp = json.load(open(args.model))["model"]
    gm = PM.GeometryModel(mp["t_row_s"], mp["tL_s_per_launch"])
    rows = []
    seen = set()
    for f in args.files:
        for line in bench_lines(f):
            key = (f, line.get("n_gpus"), line.get("ms_per_step"), line.get("value"))
            if key in seen:
                continue
            seen.add(key)
            if line.get("impl") == "reference":
                continue
            g = grid_of(line)
            if g is None:
                continue
            n = int(line.get("n_gpus", 1))
            ni, nj = g
            blocks = PM.blocks_of(ni, nj, n, 1)
            stages = int(line.get("config", {}).get("rk_stages", 4))
            gm.stages = stages
            pred = gm.multi_gpu_step(blocks) if n > 1 else gm.loopback_step(blocks)
            meas = float(line["ms_per_step"]) * 1e-3
            halo = line.get("config", {}).get("halo_measured", {})
            alpha = None
            if isinstance(halo, dict) and halo.get("slab_alone_ms_per_step_max"):
                t_alone = halo["slab_alone_ms_per_step_max"] * 1e-3
                alpha = meas / t_alone - 1.0
            rows.append(dict(file=os.path.basename(f), n=n, grid=f"{ni}x{nj}", measured_ms=meas * 1e3,
                             predicted_ms=pred * 1e3, rel_err=(pred - meas) / meas, alpha=alpha,
                             predicted_alpha_ms=None if alpha is None else pred * (1 + alpha) * 1e3,
                             simulated=bool(line.get("config", {}).get("simulated_ranks_on_one_gpu"))))
    print(f"{'file':32s} {'N':>2s} {'grid':>11s} {'meas ms':>9s} {'model ms':>9s} {'rel err':>8s} "
          f"{'alpha':>7s} {'model(1+a)':>10s}  note")
    for r in rows:
        a = "" if r["alpha"] is None else f"{r['alpha']:7.3f}"
        pa = "" if r["predicted_alpha_ms"] is None else f"{r['predicted_alpha_ms']:10.3f}"
        note = "ranks time-sliced on one GPU (functional run)" if r["simulated"] else ""
        print(f"{r['file'][:32]:32s} {r['n']:2d} {r['grid']:>11s} {r['measured_ms']:9.3f} {r['predicted_ms']:9.3f} "
              f"{100 * r['rel_err']:7.1f}% {a:>7s} {pa:>10s}  {note}")
    if not rows:
        print("(no bench lines found)")
    return rows


if __name__ == "__main__":
    main()
