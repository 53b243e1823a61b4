"""bench.py — distributed 3D FFT throughput on 1/2/4/8 B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (driver launch for N > 1)

A step is one forward + inverse 3D FFT (the whole hot path: x/y/z stages and both
exchanges, each direction) of the workload below.  Default workload: BASELINE configs[3],
1024^3 complex64 c2c, pencil decomposition (N=1: 1x1, 2: 1x2, 4: 2x2, 8: 2x4) — strong
scaling of one global problem.  Rank 0 prints one JSON line (contract in the task statement);
`value` is GFLOP/s with the 5·N·log2(N) convention, fwd+inv counted (2x), over all GPUs.

--impl reference times the CPU oracle (oracle/, plain C + OpenMP, fp64) on the host cores on
a bounded sample of the same workload (there is no installable reference implementation:
/root/reference holds only the paper).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "3D FFT ms and GFLOP/s (5N·log2N) at 1/2/4/8 B200; % of HBM/NVLink roofline"
NVLINK_GBS = 900.0  # per direction per GPU, nominal (north star)
NVLINK_MEASURED_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md): the NVLink roofline peak
GRIDS = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--grid", default="1024,1024,1024", help="global nx,ny,nz")
    p.add_argument("--precision", default="f32", choices=["f32", "f64"])
    p.add_argument("--strategy", default="pencil", choices=["pencil", "slab"])
    p.add_argument("--grid-p", default="", help="process grid P1,P2 (default by N)")
    p.add_argument("--kind", default="c2c", choices=["c2c", "r2c", "r2r"],
                   help="r2c: real input, R2C forward + C2R inverse; r2r: DCT-II forward + DCT-III inverse per axis")
    p.add_argument("--poisson", action="store_true",
                   help="periodic Poisson solve: R2C/C2C forward with the fused 1/λ(k) multiplier, then the inverse "
                        "(SURVEY §8(f) f3, P:606-620)")
    p.add_argument("--chunks", type=int, default=0)
    p.add_argument("--no-overlap", action="store_true")
    p.add_argument("--exchange", default="auto", choices=["auto", "ce", "p2p", "hybrid", "nccl"],
                   help="p2p: FFT epilogues store into peers' IPC windows over NVLink; ce: copy engines move "
                        "packed blocks into the windows; hybrid: p2p for the x-FFT, ce elsewhere; nccl: grouped "
                        "send/recv; auto: p2p")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay timing")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--seed", type=int, default=260112209 + 4)
    return p.parse_args()


def flops_fwd_inv(shape, kind="c2c"):
    """5·N·log2N per c2c transform; R2C/C2R with the real-data convention 2.5·N·log2N (reading Z9)."""
    N = shape[0] * shape[1] * shape[2]
    return 2 * (2.5 if kind in ("r2c", "r2r") else 5.0) * N * math.log2(N)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.lines, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------ CPU oracle timing
def oracle_sample(shape_full, seconds_budget=20.0):
    """Time the oracle (fp64 C, OpenMP on the host cores) on a bounded sample of the workload:
    fwd+inv of the largest cube edge <= the workload's that fits the budget (512^3 by default)."""
    import oracle

    oracle.build()
    oracle.set_threads(len(os.sched_getaffinity(0)))  # every host core (torchrun sets OMP_NUM_THREADS=1)
    edge = min(512, min(shape_full))
    shp = (edge, edge, edge)
    a = oracle.gen_complex(1, shp)
    t0 = time.perf_counter()
    reps = 0
    while True:
        oracle.fft3d_inplace(a, -1)
        oracle.fft3d_inplace(a, +1)
        reps += 1
        el = time.perf_counter() - t0
        if el > seconds_budget / 2 or reps >= 3:
            break
    per = el / reps
    return {"value": flops_fwd_inv(shp) / per / 1e9, "unit": "GFLOP/s", "cores": oracle.num_threads(),
            "kind": "oracle",
            "sample": f"{edge}^3 complex128 c2c fwd+inv, fp64 oracle, {reps} rep(s), {per * 1e3:.0f} ms each"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    shape = tuple(int(v) for v in args.grid.split(","))
    import oracle

    oracle.build()
    oracle.set_threads(len(os.sched_getaffinity(0)))  # every host core (torchrun sets OMP_NUM_THREADS=1)
    edge = 512 if (args.steps + args.warmup) <= 20 else 256
    edge = min(edge, min(shape))
    shp = (edge, edge, edge)
    a = oracle.gen_complex(1, shp)
    for _ in range(args.warmup):
        oracle.fft3d_inplace(a, -1)
        oracle.fft3d_inplace(a, +1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.fft3d_inplace(a, -1)
        oracle.fft3d_inplace(a, +1)
    el = (time.perf_counter() - t0) / max(args.steps, 1)
    val = flops_fwd_inv(shp) / el / 1e9
    grid = GRIDS.get(args.gpus, (1, args.gpus))
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{shape[0]}x{shape[1]}x{shape[2]} complex64 c2c {args.strategy} "
                                  f"{grid[0]}x{grid[1]} fwd+inv (oracle sample {edge}^3 complex128)"},
           "cpu_baseline": {"kind": "oracle", "cores": oracle.num_threads(), "value": val, "unit": "GFLOP/s",
                            "sample": f"{edge}^3 complex128 c2c fwd+inv per step (fp64 oracle)"},
           "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------------------ GPU arm
def _union(iv):
    """Total length of a union of intervals [(t0, t1), ...]."""
    tot, end = 0.0, -1e30
    for t0, t1 in sorted(iv):
        if t1 <= end:
            continue
        tot += t1 - max(t0, end)
        end = t1
    return tot


def _intersect_len(a, b):
    """Length of (union of a) ∩ (union of b)."""
    return _union(a) + _union(b) - _union(a + b)


def breakdown_from_timeline(spans, remote_phases):
    """Fig. 9 analog per execute: wall, FFT busy (any stage kernel running), the part of
    the NVLink-bound (fused-exchange) stages that ran with no local stage beside it (exposed
    exchange, Eq. 2's non-overlapped part), the part overlapped with a local stage, and
    idle (no kernel of ours running: flag waits, pipeline fill/drain, launch gaps)."""
    by_exec = {}
    for sp in spans:
        by_exec.setdefault(sp["exec"], []).append(sp)
    rows = []
    for ex, ss in by_exec.items():
        allv = [(s["t0_ms"], s["t1_ms"]) for s in ss]
        nvl = [(s["t0_ms"], s["t1_ms"]) for s in ss if s["phase"] in remote_phases]
        loc = [(s["t0_ms"], s["t1_ms"]) for s in ss if s["phase"] not in remote_phases]
        wall = max(t1 for _, t1 in allv)
        busy = _union(allv)
        ov = _intersect_len(nvl, loc) if nvl and loc else 0.0
        rows.append({"wall": wall, "busy": busy, "idle": wall - busy, "exchange_exposed": _union(nvl) - ov,
                     "exchange_overlapped": ov, "local_fft": _union(loc)})
    if not rows:
        return None
    return {k: statistics.mean(r[k] for r in rows) for k in rows[0]}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import inputs
    import paper_2601_12209_b200 as dfft

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    N = args.gpus
    if world != N:
        raise SystemExit(f"--gpus {N} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    shape = tuple(int(v) for v in args.grid.split(","))
    if args.grid_p:
        grid = tuple(int(v) for v in args.grid_p.split(","))
    else:
        grid = (N, 1) if args.strategy == "slab" else GRIDS.get(N, (1, N))
    dt = args.kind + "_" + args.precision
    es = 8 if args.precision == "f32" else 16
    comm = dfft.Comm.create(nranks=world, rank=rank, device=local)
    fwd = dfft.Plan(comm, shape, args.strategy, grid, dt, dfft.FORWARD, chunks=args.chunks,
                    overlap=not args.no_overlap, exchange=args.exchange)
    inv = dfft.Plan(comm, shape, args.strategy, grid, dt, dfft.INVERSE, chunks=args.chunks,
                    overlap=not args.no_overlap, exchange=args.exchange)
    if args.poisson:
        fwd.set_poisson((1.0, 1.0, 1.0))
    lo, n = fwd.box(0)
    x = fwd.alloc_in()
    inputs.fill_box_cuda(x, args.seed, shape, lo, n, args.kind == "c2c")
    y = fwd.alloc_out()
    z = inv.alloc_out()
    stream = torch.cuda.current_stream()

    def step():
        fwd.execute(x, y)
        inv.execute(y, z)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    host_ms = {}

    def timed(fn, iters, tag=None):
        """back-to-back: `iters` calls between one pair of events, barrier + sync on both sides."""
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h0 = time.perf_counter()
        for _ in range(iters):
            fn()
        if tag:  # host time to enqueue the calls (the GPU may still be running them)
            host_ms[tag] = (time.perf_counter() - h0) * 1e3 / max(iters, 1)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return e0.elapsed_time(e1)

    def per_iteration(fn, iters):
        """§8(d) ("average execution time over multiple iterations"): every iteration
        barrier-separated and timed alone; per-iteration max over ranks."""
        out = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(iters):
            barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1))
        return max_over_ranks(out)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    # --- headline timed region: K back-to-back fwd+inv steps (no profiling events inside)
    n_launch0 = dfft.kernel_launches()
    ms_local = timed(step, args.steps, "headline")
    n_launch = dfft.kernel_launches() - n_launch0
    ms_total = max_over_ranks([ms_local])[0]
    ms_step = ms_total / max(args.steps, 1)
    gflops = flops_fwd_inv(shape, args.kind) / (ms_step * 1e-3) / 1e9
    # --- §8(d) timing procedure: per-iteration statistics, forward only, CUDA graph
    it_ms = per_iteration(step, max(args.steps, 3))
    fwd_ms = per_iteration(lambda: fwd.execute(x, y), max(args.steps, 3))
    step()  # y is the forward of x again (the inverse reads it)
    graph_ms = None
    if not args.no_graph:
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            fwd.execute(x, y, stream=gs)
            inv.execute(y, z, stream=gs)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        graph_ms = max_over_ranks([timed(g.replay, args.steps)])[0] / max(args.steps, 1)
        del g
    timing = {
        "procedure": "P:558 / SURVEY §8(d): back-to-back mean (headline, the contract's timed region); "
                     "per-iteration barrier-separated fwd+inv and forward-only, max over ranks per iteration",
        "back_to_back_ms": ms_step,
        "per_iteration_ms": {"median": statistics.median(it_ms), "min": min(it_ms), "mean": statistics.mean(it_ms),
                             "sd": statistics.pstdev(it_ms), "n": len(it_ms)},
        "forward_only_ms": {"median": statistics.median(fwd_ms), "min": min(fwd_ms), "mean": statistics.mean(fwd_ms),
                            "sd": statistics.pstdev(fwd_ms), "n": len(fwd_ms)},
        "cuda_graph_ms": graph_ms,
        "host_enqueue_ms_per_step": host_ms.get("headline"),
    }
    # --- profiled pass (separate from the headline): per-phase times, timeline, roofline
    R = max(3, min(args.steps, 10))
    fwd.set_profiling(True)
    inv.set_profiling(True)
    fwd.phase_times(reset=True)
    inv.phase_times(reset=True)
    prof_ms = timed(step, R) / R
    pf, pi = fwd.phase_times(reset=False), inv.phase_times(reset=False)
    tf, ti = fwd.timeline(), inv.timeline()
    fwd.set_profiling(False)
    inv.set_profiling(False)
    clk = clocks.stop()
    timing["profiled_pass_ms"] = max_over_ranks([prof_ms])[0]

    # --- roofline: every FFT stage against its binding resource; the dominant one is `roofline`
    hbm_peak, peak_kind = load_peaks()
    bf, bi = fwd.stage_bytes(), inv.stage_bytes()
    P = grid[0] * grid[1]
    fused = world > 1 and args.exchange in ("auto", "p2p")
    # with fused stores stage A carries exchange 1 and stage B exchange 2 inside their epilogues
    carries = {"stage_A": "exchange_1", "stage_B": "exchange_2"}
    traffic_tab = {}
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic_tab = json.load(f).get(f"{shape[0]}x{shape[1]}x{shape[2]}_{args.precision}_{grid[0]}x{grid[1]}", {})
    except Exception:
        pass
    if P == 1 and any(d["family"] == "xz8" for d in fwd.describe()):
        # single GPU, nz = 8·M: the x pass carries one radix-8 z step; the z stage is M points long
        stage_names = {"fwd": {"stage_A": "x-FFT + radix-8 z step (xz8, whole lines to [q][z1][y][x])",
                               "stage_B": "z-FFT, M = nz/8 points (strided TMA, 256 B rows)",
                               "stage_C": "y-FFT (strided TMA)"},
                       "inv": {"stage_A": "y-IFFT (strided TMA)",
                               "stage_B": "z-IFFT, M = nz/8 points (strided TMA, 256 B rows)",
                               "stage_C": "inverse radix-8 z step + x-IFFT (xz8, 1/N)"}}
    elif P == 1:  # single GPU: forward x, z, y; inverse y, z, x
        stage_names = {"fwd": {"stage_A": "x-FFT (contig)", "stage_B": "z-FFT (strided TMA, reads [y][z][x])",
                               "stage_C": "y-FFT (strided TMA)"},
                       "inv": {"stage_A": "y-IFFT (strided TMA)", "stage_B": "z-IFFT (strided TMA, writes [y][z][x])",
                               "stage_C": "x-IFFT (contig, 1/N)"}}
    else:  # fused stores: the epilogue writes the peers' windows; NCCL / CE: it packs local send blocks
        pk = "fused T{} pack/store" if fused else "T{} pack into send blocks"
        stage_names = {"fwd": {"stage_A": f"x-FFT (contig, {pk.format(1)})",
                               "stage_B": f"y-FFT (strided, {pk.format(2)})", "stage_C": "z-FFT (strided)"},
                       "inv": {"stage_A": f"z-IFFT (strided, {pk.format(2)})",
                               "stage_B": f"y-IFFT (strided, {pk.format(1)})",
                               "stage_C": "x-IFFT (contig, fused unpack, 1/N)"}}
    stages = []
    for tag, pt, bt in (("fwd", pf, bf), ("inv", pi, bi)):
        for ph in ("stage_A", "stage_B", "stage_C"):
            ms, cnt = pt[ph]
            if not cnt:
                continue
            launches = cnt / R
            avg = ms / cnt
            xb = bt.get(carries.get(ph, ""), 0.0) if fused else 0.0
            if xb > 0:  # NVLink-bound: off-rank bytes of the exchange this stage stores
                ach = xb / launches / (avg * 1e-3) / 1e9
                ent = {"bound": "nvlink", "achieved": ach, "peak": NVLINK_MEASURED_GBS, "unit": "GB/s",
                       "frac": ach / NVLINK_MEASURED_GBS, "frac_of_nominal_900": ach / NVLINK_GBS,
                       "bytes_per_launch": xb / launches, "peak_kind": "measured peer copy (B200_PROFILING.md)"}
            else:
                ach = bt[ph] / launches / (avg * 1e-3) / 1e9
                ent = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                       "bytes_per_launch": bt[ph] / launches, "peak_kind": peak_kind}
            tr = traffic_tab.get(f"{tag}_{ph}")
            ent.update({"kernel": f"{tag} {stage_names[tag][ph]}", "avg_launch_ms": avg, "ms_per_step": ms / R,
                        "traffic": tr / launches if tr is not None and ent["bound"] == "hbm" else None})
            # pipelined plans run a stage beside another (on an SM cap): the share of its time it
            # shared the GPU, from the timeline of the profiled pass
            spans = tf if tag == "fwd" else ti
            mine = [(x["t0_ms"] + 1e3 * x["exec"], x["t1_ms"] + 1e3 * x["exec"]) for x in spans if x["phase"] == ph]
            other = [(x["t0_ms"] + 1e3 * x["exec"], x["t1_ms"] + 1e3 * x["exec"]) for x in spans if x["phase"] != ph]
            if mine and other:
                ent["concurrent_frac"] = _intersect_len(mine, other) / max(_union(mine), 1e-12)
            stages.append(ent)
    dom = max(stages, key=lambda e: e["ms_per_step"])
    roofline = {k: dom[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "kernel", "peak_kind",
                                    "bytes_per_launch", "avg_launch_ms")}
    roofline["stages"] = stages

    # --- north-star roofline: T_roof = max(T_HBM, T_NVL) per GPU for fwd+inv
    Nloc = shape[0] * shape[1] * shape[2] / P
    # complex elements per rank after stage 1 (R2C: nx/2+1 bins along x) and stage-1 bytes
    Ncl = Nloc * ((shape[0] // 2 + 1) / shape[0] if args.kind == "r2c" else 0.5 if args.kind == "r2r" else 1.0)
    a_bytes = (Nloc * es / 2 if args.kind in ("r2c", "r2r") else Nloc * es) + Ncl * es
    t_hbm = 2 * (a_bytes + 4 * Ncl * es) / (hbm_peak * 1e9)
    p1, p2 = (1, P) if args.strategy == "slab" else grid
    nvl_bytes = Ncl * es * ((p1 - 1) / p1 + (p2 - 1) / p2)
    t_nvl = 2 * nvl_bytes / (NVLINK_GBS * 1e9)
    t_roof = max(t_hbm, t_nvl)
    breakdown = {f"fwd_{k}": v[0] / R for k, v in pf.items() if v[1]}
    breakdown.update({f"inv_{k}": v[0] / R for k, v in pi.items() if v[1]})
    # Fig. 9 analog: FFT / exchange (exposed vs overlapped) / idle per direction, and each
    # exchange's NVLink rate (off-rank bytes over the time of the stage that carries them)
    fig9 = None
    if world > 1:
        remote = {"stage_A", "stage_B"} if fused else {"exchange_1", "exchange_2"}
        fig9 = {"fwd": breakdown_from_timeline(tf, {p for p in remote if bf.get(carries.get(p, p), 1) > 0}),
                "inv": breakdown_from_timeline(ti, {p for p in remote if bi.get(carries.get(p, p), 1) > 0}),
                "exchange_gbs": {}}
        for tag, pt, bt in (("fwd", pf, bf), ("inv", pi, bi)):
            for ex, carrier in (("exchange_1", "stage_A"), ("exchange_2", "stage_B")):
                ph = carrier if fused else ex
                if bt[ex] > 0 and pt[ph][1]:
                    gbs = bt[ex] * R / (pt[ph][0] * 1e-3) / 1e9
                    fig9["exchange_gbs"][f"{tag}_{ex}"] = {"gbs": gbs, "frac_of_770": gbs / NVLINK_MEASURED_GBS,
                                                           "frac_of_900": gbs / NVLINK_GBS, "timed_on": ph}
    gpu_launches = n_launch  # our kernels (FFT stages + flag kernels) in the headline region, counted by libdfft

    # --- e2e: pinned host input -> device -> fwd -> inv -> pinned host, through the C ABI
    # (dfft_execute_host_chain: double-buffered staging, H2D / D2H on their own streams)
    e2e = None
    if not args.no_e2e:
        xh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        xh.copy_(x)
        zh = torch.empty(z.shape, dtype=z.dtype, pin_memory=True)
        # all K steps: the chain pipelines across calls (H2D of call i+1 under compute + D2H of
        # call i), so the first H2D and the last D2H, each alone on PCIe, amortise over the K steps
        ke = max(2, args.steps)
        chain = lambda: dfft.execute_host_chain([fwd, inv], xh, zh, async_=True)  # noqa: E731
        chain()
        torch.cuda.synchronize()
        el = max_over_ranks([timed(chain, ke) / ke])[0]
        e2e = {"value": flops_fwd_inv(shape, args.kind) / (el * 1e-3) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(x.numel() * x.element_size()),
               "d2h_bytes_per_step": int(z.numel() * z.element_size()), "ms_per_step": el,
               "path": "dfft_execute_host_chain([fwd, inv]): pinned host -> device -> fwd -> inv -> pinned host, "
                       "asynchronous, H2D/D2H on their own copy streams (double-buffered staging)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(shape)

    if rank == 0:
        out = {
            "metric": METRIC, "value": gflops * 1.0, "unit": "GFLOP/s", "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
            "config": {"workload": f"{shape[0]}x{shape[1]}x{shape[2]} "
                                   + (f"complex{'64' if es == 8 else '128'} c2c" if args.kind == "c2c" else
                                      f"{'f32' if es == 8 else 'f64'} {args.kind}")
                                   + f" {args.strategy} {grid[0]}x{grid[1]} "
                                   + ("Poisson solve (fwd + 1/λ fused + inv)" if args.poisson else "fwd+inv"),
                       "flop_convention": "2.5·N·log2N per real transform" if args.kind != "c2c" else "5·N·log2N per c2c",
                       "grid": list(shape), "proc_grid": list(grid), "chunks": fwd.chunks(),
                       "exchange": ("fused stores into peer IPC windows (auto)" if args.exchange == "auto" else
                                    args.exchange) if world > 1 else "none",
                       "overlap": not args.no_overlap,
                       "l2": f"inputs larger than L2 ({Nloc * es / 2**30:.2f} GiB per GPU)"
                             if Nloc * es > 2 * 126e6 else "inputs L2-resident (flagged)",
                       "seed": args.seed},
            "roofline": roofline,
            "north_star_roofline": {"t_roof_ms": t_roof * 1e3, "t_hbm_ms": t_hbm * 1e3, "t_nvl_ms": t_nvl * 1e3,
                                    "frac": t_roof / (ms_step * 1e-3), "hbm_peak_gbs": hbm_peak,
                                    "nvlink_gbs": NVLINK_GBS},
            "timing": timing,
            "phase_ms_per_step": breakdown,
            "fig9_breakdown_ms": fig9,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": int(gpu_launches),
            "clocks": clk,
        }
        print(json.dumps(out), flush=True)
    fwd.destroy()
    inv.destroy()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
