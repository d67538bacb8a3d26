"""Diagnostic (not product code): per-CTA globaltimer timeline of the stage
kernel on a workload, from a SFV_TIMELINE=1 build (libsfv_tl.so):
  python paper_2305_18057_b200/build.py --variant tl SFV_TIMELINE=1
  SFV_LIB=paper_2305_18057_b200/libsfv_tl.so python scripts/timeline.py [C2|C3] [steps]
For each stage launch of the last step: launch span, time from the previous
launch's last exit to this launch's first/median post-wait stamp, fill time
(post-wait -> first flux data), compute span and the spread of task ends."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_18057_b200 import inputs as I  # noqa: E402
from paper_2305_18057_b200 import sfv  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ni, nj = {"C2": (1440, 720), "C3": (11520, 5760), "C4": (5760, 2880)}[wl]
X, Y = I.ramp_nodes(ni, nj, 30.0)
cfg = I.default_config(ni, nj)
g = sfv.Solver(cfg, X, Y, device=0)
g.set_state(I.uniform_state(ni, nj))
g.step(steps)
g.sync()
L = sfv.lib()
buf = np.zeros((8, 8192, 10), np.uint64)
L.sfv_debug_timeline.argtypes = [C.c_void_p, C.c_ulonglong]
assert L.sfv_debug_timeline(buf.ctypes.data, buf.nbytes) == 0
prev_end = None
out = []
for s in range(4):
    T = buf[s]
    n = int((T[:, 0] > 0).sum())
    T = T[:n].astype(np.int64)
    t0 = T[:, 0].min()
    e, r, f, x = (T[:, k] - t0 for k in range(4))
    rows = T[:, 5] & 0xffffffff
    nsegs = T[:, 5] >> 32
    line = (f"stage {s+1}: tasks {n} rows {rows.min()}-{rows.max()} segs/task max {nsegs.max()} "
            f"(steals {int((nsegs - 1).clip(0).sum())}) | entry span {e.max()/1e3:.2f} us | "
            f"ready min/med/max {r.min()/1e3:.2f}/{np.median(r)/1e3:.2f}/{r.max()/1e3:.2f} | "
            f"fill (ready->first) med {np.median(f-r)/1e3:.2f} max {(f-r).max()/1e3:.2f} | "
            f"end min/med/max {x.min()/1e3:.2f}/{np.median(x)/1e3:.2f}/{x.max()/1e3:.2f} us")
    if prev_end is not None:
        line += f" | prev last end -> first ready {(T[:, 1].min() - prev_end)/1e3:.2f} us"
    prev_end = T[:, 3].max()
    out.append(line)
    # per-SM end spread
    sm = T[:, 4] & 0xffff
    ends = np.array([x[sm == k].max() for k in np.unique(sm)])
    out.append(f"   per-SM last end: min {ends.min()/1e3:.2f} med {np.median(ends)/1e3:.2f} max {ends.max()/1e3:.2f} us;"
               f" compute (first->end) med {np.median(x-f)/1e3:.2f} us; per-row {np.median((x-f)/rows)/1e3:.3f} us")
print("\n".join(out))
np.save(f"gpurun_out/timeline_{wl}.npy", buf)
