#!/usr/bin/env python
"""Benchmark of the SENSEI finite-volume hot path on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C2|C3|C4]

One bench "step" = one full classical-RK4 time step (4 fused stage kernels:
limiter + MUSCL + Roe/Harten + residual + update + ghosts, CFL dt and
residual norms) over the whole grid.  Metric: Mcell-updates/s = cells x
RK stages x steps / device time (reading A-R21: a cell-update is one cell
through one RK stage, so Mcell-updates/s = np x ssspnt of Eq. 14).

N = 1 runs BASELINE config C2 (1440 x 720 = 1,036,800 cells, 30-degree
inlet).  N > 1 (torchrun, one process per GPU, NCCL) runs BASELINE config C3
by default: the 11520 x 5760 = 66.4 M-cell inlet in N slabs along i
(PAPER.md:174), strong scaling -- the north star's >= 80 % efficiency target
at 8 GPUs on >= 64 M cells.  Rank 0 also times the same C3 grid on its one
GPU first ("strong_scaling_base"), each rank times its own slab alone (the
measured halo time fraction), and a short copy-mode run with the per-class
CUDA-event timers gives the edge / interior / exchange / exposed-wait / dt
breakdown.  --workload C2 / C4 select weak scaling (1440 N x 720, 5760 N x
2880) instead.

Timing: W warm-up steps, then R repeats of exactly K steps, each bracketed by
a barrier + device sync and timed with CUDA events on the solver's stream
(max over ranks); `value` / `ms_per_step` come from the median repeat.  R is
chosen so the repeats span >= 0.5 s, so nvidia-smi samples the clocks
during the timed region.

--impl reference times the plain CPU oracle (oracle/, test infrastructure)
as it stands on the host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2305_18057_b200 import inputs as I  # noqa: E402

METRIC = "Mcell-updates/s (fp64, device-timed) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "Mcell-updates/s"
ALG_BYTES_PER_CELL_STAGE = 120.0  # classical RK4, minimal data flow, node geometry
# Measured FP64 (DFMA) issue peak on this pool's B200 at 1965 MHz: ILP 8, 32 warps/SM
# (scripts/microbench_fp64.cu -> profiles/r1_fp64_microbench.txt); nominal 148 x 64 x 1.965e9 = 1.861e13.
FP64_PEAK_INST_S = 1.708e13
L2_BYTES = 126e6


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def workload(name, n_gpus):
    """(ni, nj, theta, description, scaling, px) of the global grid."""
    if name == "C2":
        ni, nj = 1440 * n_gpus, 720
        desc = (f"C2 2D supersonic inlet, 30-deg ramp, {1440}x{720} cells per GPU "
                f"(global {ni}x{nj}), Table 1 freestream, RK4 CFL 0.8, bounded van Albada MUSCL, Roe+Harten")
        return ni, nj, 30.0, desc, "weak", n_gpus
    if name == "C4":
        ni, nj = 5760 * n_gpus, 2880
        return ni, nj, 30.0, f"C4 weak scaling, 5760x2880 per GPU (global {ni}x{nj})", "weak", n_gpus
    if name == "C3":
        return 11520, 5760, 30.0, "C3 strong scaling, 11520x5760 = 66,355,200 cells", "strong", n_gpus
    raise SystemExit(f"unknown workload {name}")


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.05)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()
                self.out = ""

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                rows.append((float(f[0]), float(f[1]), f[4], f[5], f[6], f[7]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def load_profile_traffic(ns=False):
    p = os.path.join(ROOT, "profiles", "ncu_ns.json" if ns else "ncu_stage_kernel.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_cell_stage"), d
    except (OSError, ValueError):
        return None, None


def operand_roofline(args, clocks, avg_launch_s, nj, ni, world, nblk):
    """The stage kernel against the sub-partition's register-operand bandwidth
    (profiles/r2b_tail_analysis.md section 2): the executed instruction mix of
    the same workload (ncu source page, scripts/opcost.py ->
    profiles/opcost_stage_kernel[_c3].json) charged with the microbenchmarked
    costs gives the cycles a warp-row needs at that bound; achieved = the
    average stage-kernel time x the sampled SM clock / warp-rows per
    sub-partition.  C2 and C3 on one GPU only (where a capture exists)."""
    name = {"C2": "opcost_stage_kernel.json", "C3": "opcost_stage_kernel_c3.json"}.get(args.workload)
    if not name or world != 1 or nblk != 1 or args.ns or not clocks.get("sm_mhz"):
        return None
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    import torch
    nsmsp = torch.cuda.get_device_properties(0).multi_processor_count * 4
    warp_rows = ((nj + 29) // 30) * ni / nsmsp  # per sub-partition and stage
    achieved = avg_launch_s * clocks["sm_mhz"] * 1e6 / warp_rows
    model = d["model_cycles_per_warp_row_mean"]
    return {"bound": "operand", "unit": "sub-partition cycles per warp-row", "achieved": achieved, "peak": model,
            "frac": model / achieved, "profile": "profiles/" + name,
            "note": "peak = cycles the executed mix needs at the register-operand bound (lower is faster), "
                    "frac = peak / achieved"}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# --ns: constant viscosity (Re ~ 2e5 on the unit-length inlet).
NS_MU = 1.0e-3
# Navier-Stokes workload: the C2 grid with a 5-degree ramp and a no-slip adiabatic
# ramp wall (an impulsive Mach-4 start against a no-slip 30-degree
# ramp gives invalid MUSCL face states within ~20 steps at mu <= 1e-2,
# profiles/r1_ns_noslip_probe.txt; the 5-degree ramp runs)
NS_THETA = 5.0


def ns_kwargs():
    return dict(viscous=1, mu=NS_MU, bc=(I.BC_INFLOW, I.BC_OUTFLOW, I.BC_NOSLIP_WALL, I.BC_SLIP_WALL))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _time_oracle(omp, budget_s, ni, rows, ns, threads=None):
    import oracle
    X, Y = I.ramp_nodes(ni, rows, NS_THETA if ns else 30.0)
    cfg = I.default_config(ni, rows, **(ns_kwargs() if ns else {}))
    o = oracle.Oracle(cfg, X, Y, omp=omp)
    o.set_state(I.uniform_state(ni, rows))
    o.step(1)  # warm
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < budget_s:
        o.step(1)
        n += 1
    dt = time.perf_counter() - t0
    return ni * rows * 4 * n / dt / 1e6, n, dt, o


def cpu_baseline_oracle(budget_s=12.0, ns=False):
    """The oracle, as it stands, on a bounded sample (the bottom rows of the
    C2 grid, ramp included, for as many RK4 steps as fit the budget):
    single-threaded pinned to one host core (taskset-equivalent
    sched_setaffinity), then the same source built with -fopenmp on every
    core of this process's affinity mask (bitwise equal to one thread:
    tests/test_oracle_pins.py::test_openmp_build_is_bitwise_single_thread,
    re-checked here on the sample)."""
    import numpy as _np
    import oracle
    oracle.build()
    ni, rows = 1440, 16
    cores = sorted(os.sched_getaffinity(0))
    pinned = cores[-1]
    try:
        os.sched_setaffinity(0, {pinned})
        v1, n1, dt1, o1 = _time_oracle(False, budget_s, ni, rows, ns)
    finally:
        os.sched_setaffinity(0, set(cores))
    out = {"value": v1, "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": f"C2 grid bottom {rows} rows ({ni}x{rows} cells incl. ramp), {n1} RK4 steps"
                     f"{' (Navier-Stokes)' if ns else ''}, {dt1:.1f} s single-threaded -O2 -ffp-contract=off, "
                     f"pinned to core {pinned}",
           "cpu_model": cpu_model(), "affinity_cores": len(cores)}
    try:
        oracle.build(omp=True)
        os.environ["OMP_NUM_THREADS"] = str(len(cores))
        vN, nN, dtN, oN = _time_oracle(True, budget_s / 2, ni, rows, ns)
        # bitwise check against the single-threaded run over the common steps
        same = None
        k = min(n1, nN) + 1
        if k >= 2:
            a = oracle.Oracle(dict(o1.cfg), *I.ramp_nodes(ni, rows, 30.0))
            a.set_state(I.uniform_state(ni, rows)); a.step(k)
            b = oracle.Oracle(dict(oN.cfg), *I.ramp_nodes(ni, rows, 30.0), omp=True)
            b.set_state(I.uniform_state(ni, rows)); b.step(k)
            same = bool(_np.array_equal(a.get_state(), b.get_state()) and _np.array_equal(a.dt(), b.dt()))
        out["all_cores"] = {"value": vN, "unit": UNIT, "cores": len(cores), "kind": "oracle (-fopenmp build)",
                            "bitwise_equal_to_single_thread": same,
                            "sample": f"same sample, {nN} RK4 steps, {dtN:.1f} s, OMP_NUM_THREADS={len(cores)}"}
    except Exception as ex:  # the all-cores leg is context; never lose the line for it
        out["all_cores"] = {"unavailable": repr(ex)[:200]}
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle
    oracle.build()
    ni, nj, theta, desc, scaling, px = workload(args.workload, args.gpus)
    ni1 = 1440 if args.workload == "C2" else (5760 if args.workload == "C4" else 11520)
    # bounded sample: the bottom `rows` rows of one GPU's share, sized so the
    # whole run stays around a minute of CPU time
    rows = max(2, min(nj, int(round(60.0 * 2.0e6 / (4.0 * ni1 * (args.steps + args.warmup))))))
    X, Y = I.ramp_nodes(ni1, rows, theta)
    cfg = I.default_config(ni1, rows)
    o = oracle.Oracle(cfg, X, Y)
    o.set_state(I.uniform_state(ni1, rows))
    o.step(args.warmup)
    t0 = time.perf_counter()
    o.step(args.steps)
    dt = time.perf_counter() - t0
    cells = ni1 * rows
    v = cells * 4 * args.steps / dt / 1e6
    sample = (f"{ni1}x{rows} bottom rows of the {args.workload} grid per step "
              f"({cells} cells, ramp included), oracle single-threaded")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / max(args.steps, 1),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded inputs)",
            "config": {"workload": desc, "sample_cells": cells, "rk_stages": 4},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model(), "affinity_cores": len(os.sched_getaffinity(0))},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


# The JSON line goes to the process's original stdout; everything else that
# writes to fd 1 while the run is in flight (NCCL's "NCCL version" banner when
# NCCL_DEBUG is set, library diagnostics) is sent to stderr, so stdout holds
# exactly one line per run.
_JSON_FD = None


def quiet_stdout():
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line):
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def main():
    quiet_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="K steps per timed repeat (default: C2 2000, C3 100, C4 200)")
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto", "C2", "C3", "C4"],
                    help="auto: C2 at N = 1, C3 strong scaling at N > 1")
    ap.add_argument("--min-timed-s", type=float, default=0.5,
                    help="repeat the K-step timed region until it spans this long (clock sampling)")
    ap.add_argument("--rk", default="rk4", choices=["rk4", "heun", "jst4"],
                    help="RK tableau (reading A-R5; SURVEY §8(f) f1: per-substep cost RK2 vs RK4, PAPER.md:276)")
    ap.add_argument("--halo", default="peer", choices=["copy", "peer"],
                    help="halo exchange: peer = device-initiated stores into the neighbour's ghost frame from "
                         "the stage kernel (DESIGN.md §5.2); copy = NCCL send/recv / device copies on a comm stream")
    ap.add_argument("--blocks", type=int, default=1,
                    help="N = 1 only: decompose the grid into this many slabs on the one GPU (loopback "
                         "partition-overhead experiment; not the headline configuration)")
    ap.add_argument("--ns", action="store_true",
                    help="Navier-Stokes mode (SURVEY §8(f) f4): viscous flux with mu = 1e-3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="N > 1: skip the strong-scaling base, halo and breakdown runs")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = env_int("WORLD_SIZE", 1)
    if args.workload == "auto":
        args.workload = "C2" if world == 1 else "C3"
    if args.steps is None:
        args.steps = {"C2": 2000, "C3": 100, "C4": 200}[args.workload]
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2305_18057_b200 import sfv

    assert torch.cuda.is_available(), "bench.py needs a GPU (no CPU fallback)"
    ndev = torch.cuda.device_count()
    sim = world > ndev
    if sim:
        # more ranks than GPUs: only as a functional check of the N > 1 path
        # (SFV_SIM_HOSTS=1 gives each rank its own NCCL host id, as in
        # tests/test_gpu_nccl.py); the numbers of such a run are not a bench value
        assert os.environ.get("SFV_SIM_HOSTS") == "1", f"WORLD_SIZE {world} > {ndev} GPUs"
        os.environ["NCCL_HOSTID"] = f"sfv-sim-host-{rank}"
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
        os.environ.setdefault("NCCL_IB_DISABLE", "1")
        os.environ.setdefault("NCCL_NVLS_ENABLE", "0")
    local_rank = local_rank % ndev
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n_gpus = world
    if args.gpus != n_gpus and rank == 0:
        print(f"# note: --gpus {args.gpus} but WORLD_SIZE {world}; using {world}", file=sys.stderr)

    ni, nj, theta, desc, scaling, px = workload(args.workload, n_gpus)
    if world == 1 and args.blocks > 1:
        px = args.blocks
        desc += f"; {px} loopback slabs on one GPU"
    if args.ns:
        theta = NS_THETA
        desc = (f"Navier-Stokes terms (mu = 1e-3, Green-Gauss gradients, no-slip adiabatic ramp wall, "
                f"{NS_THETA:g}-deg ramp) on " + desc.replace("30-deg ramp", f"{NS_THETA:g}-deg ramp"))
    X, Y = I.ramp_nodes(ni, nj, theta)
    rk = {"rk4": I.RK4_CLASSIC, "heun": I.RK2_HEUN, "jst4": I.RK4_JAMESON}[args.rk]
    cfg = I.default_config(ni, nj, rk=rk, max_history=max(args.steps + args.warmup + 16, 64),
                           **(ns_kwargs() if args.ns else {}))
    U0 = I.uniform_state(ni, nj)
    nccl_id = None
    if world > 1:
        obj = [sfv.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    stream = torch.cuda.Stream(device=dev)
    solver = sfv.Solver(cfg, X, Y, px=px, py=1, rank=rank, nranks=world, nccl_id=nccl_id,
                        device=local_rank, stream=stream)
    nblk = px if world == 1 else 1
    halo_note = args.halo
    if args.halo == "peer" and px > 1:
        if world == 1:
            solver.enable_peer_halo()
        else:
            # collective: peer mode only if every rank could map its neighbours
            hs = [None] * world
            dist.all_gather_object(hs, solver.peer_handle())
            ok, why = 1, ""
            try:
                solver.peer_connect(hs)
            except sfv.SfvError as ex:
                ok, why = 0, str(ex)
            flag = torch.tensor([ok], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 1:
                solver.set_halo_mode(sfv.HALO_PEER)
            else:
                args.halo = "copy"
                halo_note = f"copy (peer mapping unavailable on some rank: {why or 'other rank'})"
    def warm():
        solver.set_state(U0)
        solver.step(args.warmup)
        solver.sync()

    if world > 1 and args.halo == "peer":
        # a peer-mode failure on a real multi-GPU node (a neighbour's signal never
        # arriving -> SFV_ERR_HALO after the device-side timeout) falls back,
        # collectively, to NCCL copy-mode halos instead of losing the run
        ok, why = 1, ""
        try:
            warm()
            if os.environ.get("SFV_BENCH_FAKE_PEER_FAILURE") == str(rank):  # exercises the fallback (tests only)
                raise sfv.SfvError(sfv.ERR_HALO, "injected peer-mode failure")
        except sfv.SfvError as ex:
            ok, why = 0, str(ex)
        flag = torch.tensor([ok], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            solver.set_halo_mode(sfv.HALO_COPY)
            args.halo = "copy"
            halo_note = f"copy (peer-mode warm-up failed on some rank: {why or 'other rank'})"
            warm()
    else:
        warm()

    # host-side barrier (gloo): a rank waiting in it leaves no NCCL kernel spinning on
    # its GPU (with simulated ranks sharing one GPU such a kernel would time-slice
    # against the rank that is measuring)
    cpu_group = dist.new_group(backend="gloo") if world > 1 else None

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier(group=cpu_group)

    # ---- device-timed region (inputs resident in HBM) ----
    # R repeats of exactly K steps (each bracketed by barrier + sync, CUDA
    # events on the solver's stream, max over ranks); median repeat reported
    def timed_once():
        barrier()
        solver.step(args.steps)
        ms_ = solver.sync()
        barrier()
        return ms_

    probe = timed_once()  # (also a last warm-up; not reported)
    tp = torch.tensor([probe], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tp, op=dist.ReduceOp.MAX)
    reps = int(min(2000, max(5, np.ceil(args.min_timed_s * 1e3 / max(float(tp.item()), 1e-3)))))
    rep_ms = []
    with Clocks(local_rank) as clk:
        for _ in range(reps):
            rep_ms.append(timed_once())
    t = torch.tensor(rep_ms, dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    rep_max = [float(x) for x in t.cpu().numpy()]
    ms_max = float(statistics.median(rep_max))
    cells_total = ni * nj
    stages = I.RK_STAGES[rk]
    value = cells_total * stages * args.steps / (ms_max * 1e-3) / 1e6
    cells_rank = cells_total // world
    cells_launch = cells_rank // nblk
    # our kernels per step: the stage kernels (plus 1-2 two-row edge launches per
    # stage on a rank with neighbours, overlap split); one norms-reduction kernel
    # per block after every 32nd step since set_state (history >= 32)
    # (peer mode: one launch per stage and block, the edge tasks store the halos)
    if world > 1:
        edges = (rank > 0) + (rank < world - 1)
    else:
        edges = 0 if nblk == 1 else 2 * (nblk - 1) / nblk  # average per loopback block
    if args.halo == "peer":
        edges = 0
    launches = int(round(nblk * (stages * (1 + edges + (2 if args.ns else 0)) * args.steps + args.steps / 32.0)))
    stage_launches = stages * args.steps * nblk

    # ---- roofline of the dominant kernel (the fused stage kernel) ----
    # At N = 1 a step is the stage kernels (plus a tiny norms kernel every 32
    # steps), so the timed region / stage launches is a (slightly conservative)
    # average stage-kernel duration.
    avg_launch_s = ms_max * 1e-3 / stage_launches
    alg_bytes = ALG_BYTES_PER_CELL_STAGE * cells_launch
    hbm_achieved = alg_bytes / avg_launch_s / 1e9
    peak, peak_src = measured_peak()
    traffic_pc, prof = load_profile_traffic(ns=args.ns)
    hbm = {"bound": "hbm", "achieved": hbm_achieved, "peak": peak, "unit": "GB/s", "frac": hbm_achieved / peak,
           "traffic": (traffic_pc * cells_launch) if traffic_pc else None,
           "alg_bytes_per_cell_stage": ALG_BYTES_PER_CELL_STAGE, "peak_source": peak_src}
    roof = dict(hbm, kernel=("sfv::stage_kernel + NS gradient/viscous kernels (per stage, averaged)" if args.ns
                                  else "sfv::stage_kernel (4 launches per step, averaged)"))
    if prof and prof.get("fp64_inst_per_cell_stage"):
        # FP64 pipe is the nearer roof: report it as the bound, HBM alongside
        fp64_rate = prof["fp64_inst_per_cell_stage"] * cells_launch / avg_launch_s
        roof = {"bound": "alu", "achieved": fp64_rate / 1e12, "peak": FP64_PEAK_INST_S / 1e12,
                "unit": "T FP64-inst/s", "frac": fp64_rate / FP64_PEAK_INST_S,
                "traffic": hbm["traffic"], "fp64_inst_per_cell_stage": prof["fp64_inst_per_cell_stage"],
                "peak_source": "measured DFMA issue rate (profiles/r1_fp64_microbench.txt)",
                "profile": prof.get("source"), "kernel": ("sfv::stage_kernel + NS gradient/viscous kernels (per stage, averaged)" if args.ns
                           else "sfv::stage_kernel (4 launches per step, averaged)"),
                "hbm": hbm,
                **({"note": "NS: FP64 instructions and DRAM bytes per cell-stage summed over the stage kernel and "
                            "the fused gradient / viscous-flux kernel of each stage (ncu, profiles/ncu_ns.json); "
                            "achieved = that count x cell-stages / the average stage time"} if args.ns else {})}

    # ---- end to end through the public API with host buffers ----
    # set_state(pinned host U) + K steps + residual norms of the K steps
    # (64 B/step) + the solution back to pinned host memory (N = 1: the full
    # grid; N > 1: every rank its own slab, sfv_get_block_state)
    e2e = None
    if not args.no_e2e:
        Uh = torch.from_numpy(np.ascontiguousarray(U0)).pin_memory()
        if world == 1:
            Uout = torch.empty(Uh.shape, dtype=torch.float64, pin_memory=True)
        else:
            m = solver.partition_map(rank)
            Uout = torch.empty((int(m[3] - m[2]), int(m[1] - m[0]), 4), dtype=torch.float64, pin_memory=True)
        K = args.steps
        # one untimed pass over the same pinned buffers (first DMA touch of the
        # pages; like the warm-up steps of the device-timed region)
        solver.set_state_ptr(Uh.data_ptr())
        if world == 1:
            solver.get_state_ptr(Uout.data_ptr())
        else:
            solver.get_block_state_ptr(rank, Uout.data_ptr())
        barrier()
        t0 = time.perf_counter()
        solver.set_state_ptr(Uh.data_ptr())
        t1 = time.perf_counter()
        solver.step(K)
        norms = solver.residual_norms(0, K)
        t2 = time.perf_counter()
        if world == 1:
            solver.get_state_ptr(Uout.data_ptr())
        else:
            solver.get_block_state_ptr(rank, Uout.data_ptr())
        barrier()
        t3 = time.perf_counter()
        tw = torch.tensor([t3 - t0, t1 - t0, t2 - t1, t3 - t2], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        wall, w_set, w_step, w_get = (float(x) for x in tw.cpu().numpy())
        rank_bytes = Uout.numel() * 8
        e2e = {"value": cells_total * stages * K / wall / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": rank_bytes * world / K, "d2h_bytes_per_step": (rank_bytes * world + 64.0 * K) / K,
               "phases_ms": {"set_state": 1e3 * w_set, "steps_and_norms": 1e3 * w_step, "get_state": 1e3 * w_get},
               "fixed_overhead_ms": 1e3 * wall - ms_max,
               "note": "set_state(pinned host U) + K steps + residual norms (64 B/step) + solution to pinned host "
                       "memory (" + ("full grid" if world == 1 else "each rank its slab") + "), wall clock, max over ranks; "
                       "fixed_overhead_ms = wall - device time of K steps"}
        assert np.all(np.isfinite(norms))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_oracle(ns=args.ns)

    li = solver.launch_info()
    halo_info = None
    extras = {}
    if px > 1:
        # halo traffic per step of the busiest rank (2 edge rows x 4 components per
        # connected cut, every stage) and the time it would take at NVLink 5's
        # 900 GB/s per direction (a bandwidth model, next to the measured fraction below)
        cuts = 2 if px > 2 or world == 1 else 1
        hb = cuts * 2 * 4 * 8 * nj * stages
        halo_info = {"bytes_per_step_per_rank": hb, "nvlink_gbs": 900.0,
                     "nvlink_time_fraction_model": hb / 900e9 / (ms_max * 1e-3 / args.steps)}
    if world > 1 and not args.no_extras:
        extras = multi_gpu_extras(args, solver, dev, rank, world, ni, nj, theta, cfg, U0, ms_max, barrier, sfv,
                                  torch, dist, local_rank)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded inputs)",
                "config": {"workload": desc, "global_cells": cells_total, "cells_per_gpu": cells_rank,
                           "rk_stages": stages, "rk": args.rk, "parallelism": f"slab{px}x1",
                           "halo": halo_note if px > 1 else "none",
                           **({"halo_traffic": halo_info} if halo_info else {}),
                           **({"simulated_ranks_on_one_gpu": True} if sim else {}),
                           "l2": f"no flush: working set {solver.ws.numel() / 1e6:.0f} MB per GPU vs 126 MB L2",
                           "launch": li,
                           "timing": {"repeats": reps, "steps_per_repeat": args.steps,
                                      "ms_per_repeat_median": ms_max, "ms_per_repeat_min": min(rep_max),
                                      "ms_per_repeat_max": max(rep_max)},
                           "mcell_steps_per_s": value / stages,
                           "pct_hbm_roofline_8TBs": 100.0 * value * 1e6 * ALG_BYTES_PER_CELL_STAGE / n_gpus / 8e12,
                           **extras},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches * reps,
                "clocks": clk.summary()}
        opr = operand_roofline(args, line["clocks"], avg_launch_s, nj, ni, world, nblk)
        if opr and isinstance(roof, dict) and roof.get("bound") == "alu":
            roof["operand"] = opr
        emit(line)
    if world > 1:
        dist.destroy_process_group()


def multi_gpu_extras(args, solver, dev, rank, world, ni, nj, theta, cfg, U0, ms_multi, barrier, sfv, torch, dist,
                     local_rank):
    """N > 1 context measured in the same job (BASELINE configs[2]/[3]):
    * strong_scaling_base (C3): rank 0 times the whole grid on its one GPU;
    * halo: each rank times its own slab as an isolated single-block run; the
      measured halo time fraction is 1 - t_alone / t_multi (PAPER.md:157,
      :172 -- exchange cost as the paper's model separates it);
    * breakdown_copy_mode: a short run with copy-mode (NCCL send/recv) halos
      and the per-class CUDA-event timers (sfv_get_stage_timings), ms per step,
      max over ranks.
    Each measurement runs one rank at a time where it would otherwise share a
    GPU with other ranks' work."""
    K = max(args.steps, 10)
    out = {}
    stages = I.RK_STAGES[cfg["rk"]]

    def single(ni_, nj_, steps):
        X_, Y_ = I.ramp_nodes(ni_, nj_, theta)
        c_ = dict(cfg, ni=ni_, nj=nj_)
        s_ = sfv.Solver(c_, X_, Y_, device=local_rank)
        s_.set_state(I.uniform_state(ni_, nj_))
        s_.step(args.warmup); s_.sync()
        s_.step(steps)
        ms_ = s_.sync()
        s_.close()
        return ms_

    if args.workload == "C3":
        barrier()
        base = None
        if rank == 0:
            base = single(ni, nj, K)
            out["strong_scaling_base"] = {"n_gpus": 1, "ms_per_step": base / K,
                                          "value": ni * nj * stages * K / (base * 1e-3) / 1e6, "unit": UNIT,
                                          "note": "the same C3 grid on rank 0's one GPU, timed in this job"}
        barrier()
    m = solver.partition_map(rank)
    nib, njb = int(m[1] - m[0]), int(m[3] - m[2])
    alone = 0.0
    for r in range(world):  # one rank at a time
        barrier()
        if r == rank:
            alone = single(nib, njb, K)
        barrier()
    frac = 1.0 - (alone / K) / (ms_multi / args.steps)
    ft = torch.tensor([frac, alone / K], dtype=torch.float64, device=dev)
    lst = [torch.zeros_like(ft) for _ in range(world)]
    dist.all_gather(lst, ft)
    fr = [float(x[0]) for x in lst]
    out["halo_measured"] = {"time_fraction_measured_max": max(fr), "time_fraction_measured_mean": sum(fr) / len(fr),
                   "slab_alone_ms_per_step_max": max(float(x[1]) for x in lst),
                   "multi_ms_per_step": ms_multi / args.steps, "mode": args.halo}
    # copy-mode breakdown with the per-class timers
    try:
        solver.set_halo_mode(sfv.HALO_COPY)
        solver.set_state(U0)
        solver.step(args.warmup); solver.sync()
        solver.set_profiling(True)
        barrier()
        solver.step(10)
        solver.sync()
        tm = solver.stage_timings()
        solver.set_profiling(False)
        keys = list(sfv.Solver.PROFILE_CLASSES)
        v = torch.tensor([tm[k] / max(tm["steps"], 1) for k in keys], dtype=torch.float64, device=dev)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        out["breakdown_copy_mode_ms_per_step_max_over_ranks"] = {k: float(x) for k, x in zip(keys, v.cpu().numpy())}
    except sfv.SfvError as ex:
        out["breakdown_copy_mode_ms_per_step_max_over_ranks"] = {"unavailable": str(ex)[:200]}
    return out


if __name__ == "__main__":
    main()
