"""Per-stage time vs grid length (nj fixed): separates per-stage fixed cost
from per-row cost of the stage kernel (diagnostic)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2305_18057_b200 import inputs as I
from paper_2305_18057_b200 import sfv

nj = int(os.environ.get("NJ", 720))
for ni in [int(x) for x in os.environ.get("NIS", "360,720,1440,2880,5760,11520").split(",")]:
    X, Y = I.ramp_nodes(ni, nj, 30.0)
    cfg = I.default_config(ni, nj, max_history=4096)
    s = sfv.Solver(cfg, X, Y)
    s.set_state(I.uniform_state(ni, nj))
    steps = max(20, int(2000 * 1440 / ni))
    s.step(20); s.sync()
    s.step(steps); ms = s.sync()
    us_stage = ms * 1e3 / steps / 4
    li = s.launch_info()
    print(json.dumps({"ni": ni, "nj": nj, "us_per_stage": round(us_stage, 2),
                      "gcell_stage_s": round(ni * nj / us_stage / 1e3, 2), "launch": li,
                      "env_waves": os.environ.get("SFV_WAVES")}), flush=True)
    s.close()
