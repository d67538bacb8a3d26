"""Diagnostic (not product code): per-strip view of a stage-kernel timeline
saved by scripts/timeline.py (gpurun_out/timeline_C2.npy): for each stage,
the per-row time and end time of boundary strips (0 and the last) against
interior strips, and which tasks end last (strip, rows, SM, warp slot).
Task tt of a launch is strip tt % nstrips, segment tt // nstrips (argument 3 =
nseg: the SFV_WALL_FIRST mapping, edge strips' main tasks first)."""
import sys

import numpy as np

f = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline_C2.npy"
nstrips = int(sys.argv[2]) if len(sys.argv) > 2 else 24
wall_first = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # nseg of the main tasks if the build maps the edge strips first
buf = np.load(f)
for s in range(4):
    T = buf[s]
    n = int((T[:, 0] > 0).sum())
    T = T[:n].astype(np.int64)
    t0 = T[:, 0].min()
    r, fst, x = T[:, 1] - t0, T[:, 2] - t0, T[:, 3] - t0
    rows = T[:, 5] & 0xffffffff
    sm, warp = T[:, 4] & 0xffff, T[:, 4] >> 16
    tt = np.arange(n)
    strip = tt % nstrips
    if wall_first:
        nb = 2 * wall_first
        m = tt < nstrips * wall_first
        strip = np.where(m & (tt < nb), np.where(tt & 1, nstrips - 1, 0),
                         np.where(m, 1 + (tt - nb) % (nstrips - 2), strip))
    main = rows >= np.median(rows) * 0.75
    per_row = (x - fst) / np.maximum(rows, 1) / 1e3
    bnd = (strip == 0) | (strip == nstrips - 1)
    print(f"stage {s+1}: {n} tasks ({int(main.sum())} main), end max {x.max()/1e3:.2f} us")
    for name, m in (("strip 0", strip == 0), (f"strip {nstrips-1}", strip == nstrips - 1), ("interior", ~bnd)):
        mm = m & main
        print(f"   {name:>9}: per-row med {np.median(per_row[mm]):.3f} us, end med {np.median(x[mm])/1e3:.2f} "
              f"max {x[mm].max()/1e3:.2f} us (main tasks {int(mm.sum())})")
    last = np.argsort(x)[-12:][::-1]
    print("   last to end: " + ", ".join(f"{x[k]/1e3:.1f}us s{strip[k]} r{rows[k]} sm{sm[k]} w{warp[k]}" for k in last))
    # end time by warp slot class (slots 0-3 / 4-7 / 8-11 on the SM)
    cls = np.minimum(warp // 4, 2)
    print("   end med by slot class: " + ", ".join(f"{k}: {np.median(x[main & (cls == k)])/1e3:.2f}" for k in range(3)))
