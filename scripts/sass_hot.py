#!/usr/bin/env python
"""Per-opcode view of one kernel from `ncu --page source --csv --print-source sass`:
executed warp instructions per unit of work and warp-stall samples, grouped by
opcode (measurement tool, not product code).

    ncu -i REP --page source --csv --print-source sass > src.csv
    python scripts/sass_hot.py src.csv KERNEL_INDEX UNITS_PER_LAUNCH
"""
import csv
import sys
from collections import defaultdict


def kernels(path):
    cur, rows, hdr = None, [], None
    for r in csv.reader(open(path)):
        if r and r[0] == "Kernel Name":
            if cur is not None:
                yield cur, hdr, rows
            cur, rows, hdr = r[1], [], None
        elif hdr is None:
            hdr = r
        else:
            rows.append(r)
    if cur is not None:
        yield cur, hdr, rows


def main():
    path, kidx, units = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
    for i, (name, hdr, rows) in enumerate(kernels(path)):
        if i != kidx:
            continue
        H = {h: k for k, h in enumerate(hdr)}
        ex = defaultdict(float); smp = defaultdict(float); stall = defaultdict(lambda: defaultdict(float))
        cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        tot_s = 0.0
        for r in rows:
            src = r[H["Source"]].strip()
            op = src.split()[0] if src else "?"
            if op.startswith("@"):
                op = src.split()[1]
            op = op.split(".")[0]
            n = float(r[H["Instructions Executed"]] or 0)
            s = float(r[H["Warp Stall Sampling (All Samples)"]] or 0)
            ex[op] += n; smp[op] += s; tot_s += s
            for c in cols:
                stall[op][c] += float(r[H[c]] or 0)
        tot = sum(ex.values())
        print(name)
        print(f"warp instructions per unit: {tot * 32 / units:.1f}   stall samples: {tot_s:.0f}")
        print(f"{'opcode':10s} {'inst/unit':>9s} {'%samples':>8s}  top stalls")
        for op in sorted(ex, key=lambda o: -smp[o])[:30]:
            top = sorted(stall[op].items(), key=lambda kv: -kv[1])[:3]
            ts = ", ".join(f"{k[6:]} {100 * v / max(tot_s, 1):.1f}" for k, v in top if v > 0)
            print(f"{op:10s} {ex[op] * 32 / units:9.1f} {100 * smp[op] / max(tot_s, 1):8.1f}  {ts}")


if __name__ == "__main__":
    main()
