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
NVLINK_GBS = 900.0  # per direction per GPU, nominal (north star); measured peer copy ~770 (B200_PROFILING.md)
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

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    # --- timed region: K fwd+inv steps, barrier + sync on both sides, events on the stream
    fwd.set_profiling(True)
    inv.set_profiling(True)
    fwd.phase_times(reset=True)
    inv.phase_times(reset=True)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_launch0 = dfft.kernel_launches()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    n_launch = dfft.kernel_launches() - n_launch0
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms_local = ev0.elapsed_time(ev1)
    pf, pi = fwd.phase_times(), inv.phase_times()
    fwd.set_profiling(False)
    inv.set_profiling(False)
    t = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = t.item()
    ms_step = ms_total / max(args.steps, 1)
    gflops = flops_fwd_inv(shape, args.kind) / (ms_step * 1e-3) / 1e9

    # --- roofline of the dominant kernel (largest total time among the FFT stages)
    hbm_peak, peak_kind = load_peaks()
    bf, bi = fwd.stage_bytes(), inv.stage_bytes()
    kernels = []
    for tag, pt, bt in (("fwd", pf, bf), ("inv", pi, bi)):
        for ph in ("stage_A", "stage_B", "stage_C"):
            ms, cnt = pt[ph]
            if cnt:
                per_launch_bytes = bt[ph] / (cnt / args.steps)
                kernels.append((ms, tag, ph, cnt, per_launch_bytes))
    kernels.sort(reverse=True)
    ms_k, tag_k, ph_k, cnt_k, bytes_k = kernels[0]
    avg_ms = ms_k / cnt_k
    achieved = bytes_k / (avg_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f)
        traffic = tr.get(f"{shape[0]}x{shape[1]}x{shape[2]}_{args.precision}_{grid[0]}x{grid[1]}", {}).get(
            f"{tag_k}_{ph_k}")
        if traffic is not None:
            traffic = traffic / (cnt_k / args.steps)  # per launch
    except Exception:
        pass
    if grid[0] * grid[1] == 1:  # single GPU: forward x, z, y; inverse y, z, x
        stage_names = {"fwd": {"stage_A": "x-FFT (contig)", "stage_B": "z-FFT (strided TMA, writes [y][z][x])",
                               "stage_C": "y-FFT (strided TMA)"},
                       "inv": {"stage_A": "y-IFFT (strided TMA)", "stage_B": "z-IFFT (strided TMA)",
                               "stage_C": "x-IFFT (contig, 1/N)"}}
    else:
        stage_names = {"fwd": {"stage_A": "x-FFT (contig, fused T1 pack)", "stage_B": "y-FFT (strided, fused T2 pack)",
                               "stage_C": "z-FFT (strided)"},
                       "inv": {"stage_A": "z-IFFT (strided, fused T2 pack)", "stage_B": "y-IFFT (strided, fused pack)",
                               "stage_C": "x-IFFT (contig, fused unpack, 1/N)"}}
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic,
                "kernel": f"{tag_k} {stage_names[tag_k][ph_k]}", "peak_kind": peak_kind,
                "bytes_per_launch": bytes_k, "avg_launch_ms": avg_ms}

    # --- north-star roofline: T_roof = max(T_HBM, T_NVL) per GPU for fwd+inv
    P = grid[0] * grid[1]
    Nloc = shape[0] * shape[1] * shape[2] / P
    # complex elements per rank after stage 1 (R2C: nx/2+1 bins along x) and stage-1 bytes
    Ncl = Nloc * ((shape[0] // 2 + 1) / shape[0] if args.kind == "r2c" else 0.5 if args.kind == "r2r" else 1.0)
    a_bytes = (Nloc * es / 2 if args.kind in ("r2c", "r2r") else Nloc * es) + Ncl * es
    t_hbm = 2 * (a_bytes + 4 * Ncl * es) / (hbm_peak * 1e9)
    p1, p2 = (1, P) if args.strategy == "slab" else grid
    nvl_bytes = Ncl * es * ((p1 - 1) / p1 + (p2 - 1) / p2)
    t_nvl = 2 * nvl_bytes / (NVLINK_GBS * 1e9)
    t_roof = max(t_hbm, t_nvl)
    breakdown = {f"fwd_{k}": v[0] / args.steps for k, v in pf.items() if v[1]}
    breakdown.update({f"inv_{k}": v[0] / args.steps for k, v in pi.items() if v[1]})
    launches_per_step = sum(v[1] for v in pf.values() if v[1]) + sum(v[1] for v in pi.values() if v[1])
    exch = sum(pf[k][1] + pi[k][1] for k in ("exchange_1", "exchange_2"))
    gpu_launches = n_launch  # our kernels (FFT stages + flag signals) in the timed region, counted by libdfft

    # --- e2e: host pinned input -> device -> fwd+inv -> host, through the public API
    e2e = None
    if not args.no_e2e:
        xh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        xh.copy_(x)
        zh = torch.empty(z.shape, dtype=z.dtype, pin_memory=True)
        ke = max(2, min(args.steps, 5))
        for it in range(ke + 1):
            if it == 1:
                barrier()
                torch.cuda.synchronize()
                e0 = time.perf_counter()
                s0 = torch.cuda.Event(enable_timing=True)
                s1 = torch.cuda.Event(enable_timing=True)
                s0.record(stream)
            x.copy_(xh, non_blocking=True)
            step()
            zh.copy_(z, non_blocking=True)
        s1.record(stream)
        torch.cuda.synchronize()
        el = s0.elapsed_time(s1) / ke
        te = torch.tensor([el], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        el = te.item()
        e2e = {"value": flops_fwd_inv(shape, args.kind) / (el * 1e-3) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(x.numel() * x.element_size()),
               "d2h_bytes_per_step": int(z.numel() * z.element_size()), "ms_per_step": el,
               "path": "pinned host -> Plan.execute(fwd) -> Plan.execute(inv) -> pinned host"}

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
            "phase_ms_per_step": breakdown,
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
