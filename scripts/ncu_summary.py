#!/usr/bin/env python
"""Summarise an ncu --set full capture of the stage kernels into profiles/.

    python scripts/ncu_summary.py REP.ncu-rep --cells N --tag NAME [--launches launches.csv]

Writes profiles/NAME.md (human summary) and, with --bench-json, the
profiles/ncu_stage_kernel.json that bench.py reads for `traffic` and the FP64
instruction count per cell-stage.
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def f(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def summarise(rep, cells):
    h, units, rows = raw_rows(rep)
    ix = {k: i for i, k in enumerate(h)}
    res = []
    for r in rows:
        g = lambda k: f(r[ix[k]]) if k in ix else float("nan")
        dur_ns = g("gpu__time_duration.sum") * (1e3 if units[ix["gpu__time_duration.sum"]] == "us" else 1.0)
        if units[ix["gpu__time_duration.sum"]] == "ms":
            dur_ns = g("gpu__time_duration.sum") * 1e6
        clk = g("sm__cycles_elapsed.avg.per_second")  # GHz
        cyc = dur_ns * clk
        mb = lambda k: g(k) * {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0}.get(units[ix[k]], 1.0)
        fp = {op: g(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed") * cyc
              for op in ("dadd", "dfma", "dmul")}
        stalls = {k.split("stalled_")[1].replace("_per_issue_active.ratio", ""): g(k) for k in h
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
        res.append(dict(
            kernel=r[ix["Kernel Name"]], duration_us=dur_ns / 1e3, sm_ghz=clk,
            dram_read_bytes=mb("dram__bytes_read.sum"), dram_write_bytes=mb("dram__bytes_write.sum"),
            dram_bytes_per_cell_stage=(mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")) / cells,
            fp64_inst=fp, fp64_inst_per_cell_stage=sum(fp.values()) / cells,
            fp64_pipe_pct=g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            issue_active_pct=g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            warps_active_pct=g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            dram_pct=g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            regs=g("launch__registers_per_thread"),
            smem_kb=g("launch__shared_mem_per_block_dynamic"),
            occ_limit_regs=g("launch__occupancy_limit_registers"),
            occ_limit_smem=g("launch__occupancy_limit_shared_mem"),
            thread_inst_per_cell_stage=g("thread_inst_executed") / cells,
            stalls_per_issue=dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])))
    return res


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0][:70]].append(f(r[vi]))
    tot = sum(sum(v) for v in agg.values())
    return [(k, len(v), sum(v) / len(v), sum(v) / tot) for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--cells", type=int, required=True)
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--bench-json", action="store_true")
    ap.add_argument("--ns-json", action="store_true",
                    help="Navier-Stokes capture (stage + gradient/viscous kernels): per-stage sums -> profiles/ncu_ns.json")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    res = summarise(a.rep, a.cells)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# ncu summary: {a.tag}", "", a.note, "",
             f"Capture: `{os.path.basename(a.rep)}` (ncu --set full --clock-control none), {a.cells} cells per launch.", "",
             "| kernel | us | SM GHz | DRAM B/cell-stage | FP64 inst/cell-stage | FP64 pipe % | issue % | warps % | DRAM % | regs | smem KB |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in res:
        lines.append(f"| `{r['kernel']}` | {r['duration_us']:.1f} | {r['sm_ghz']:.3f} | {r['dram_bytes_per_cell_stage']:.1f} | "
                     f"{r['fp64_inst_per_cell_stage']:.1f} | {r['fp64_pipe_pct']:.1f} | {r['issue_active_pct']:.1f} | "
                     f"{r['warps_active_pct']:.1f} | {r['dram_pct']:.1f} | {r['regs']:.0f} | {r['smem_kb']:.1f} |")
    lines += ["", "Top stall reasons (warps stalled per issued instruction), first launch:", ""]
    for k, v in res[0]["stalls_per_issue"].items():
        lines.append(f"- {k}: {v:.2f}")
    if a.launches:
        lines += ["", f"Launch list (`{os.path.basename(a.launches)}`, gpu__time_duration.sum, cold and serialised):", "",
                  "| kernel | launches | mean us | share |", "|---|---|---|---|"]
        for k, nl, mean, share in launch_shares(a.launches):
            lines.append(f"| `{k}` | {nl} | {mean / 1e3:.2f} | {100 * share:.1f}% |")
    with open(os.path.join(ROOT, "profiles", f"{a.tag}.md"), "w") as fo:
        fo.write("\n".join(lines) + "\n")
    with open(os.path.join(ROOT, "profiles", f"{a.tag}.json"), "w") as fo:
        json.dump(res, fo, indent=1)
    if a.bench_json:
        # launch-weighted averages over the 4 stage launches of one RK4 step
        n = len(res)
        agg = dict(source=f"profiles/{a.tag}.json", cells=a.cells,
                   dram_bytes_per_cell_stage=sum(r["dram_bytes_per_cell_stage"] for r in res) / n,
                   fp64_inst_per_cell_stage=sum(r["fp64_inst_per_cell_stage"] for r in res) / n,
                   fp64_pipe_pct=sum(r["fp64_pipe_pct"] for r in res) / n)
        with open(os.path.join(ROOT, "profiles", "ncu_stage_kernel.json"), "w") as fo:
            json.dump(agg, fo, indent=1)
    if a.ns_json:
        # all kernels of the captured stages, summed per stage launch
        nst = max(1, sum(1 for r in res if "stage_kernel" in r["kernel"]))
        agg = dict(source=f"profiles/{a.tag}.json", cells=a.cells, stage_launches=nst,
                   kernels=sorted({r["kernel"] for r in res}),
                   dram_bytes_per_cell_stage=sum(r["dram_bytes_per_cell_stage"] for r in res) / nst,
                   fp64_inst_per_cell_stage=sum(r["fp64_inst_per_cell_stage"] for r in res) / nst,
                   fp64_pipe_pct=sum(r["fp64_pipe_pct"] for r in res) / len(res))
        with open(os.path.join(ROOT, "profiles", "ncu_ns.json"), "w") as fo:
            json.dump(agg, fo, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
