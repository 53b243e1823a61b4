"""Per-stage DRAM traffic of the multi-GPU plans, on simulated ranks (design aid / evidence).

    python tools/sim_stage_traffic.py P1 P2 [n] [prec]
Runs fwd+inv twice on simulated ranks (the product schedule, fused-store layouts); under
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:"fft_(strided|contig|generic)" \
        -s <launches per fwd+inv> -c <launches per fwd+inv> --csv
the second fwd+inv's stage kernels are captured.  Prints the launch count per fwd+inv and the
algorithmic bytes of every stage launch (read + write of the local array chunk) in issue order.
On simulated ranks the peers' windows are on the same GPU, so the "remote" stores show up as local
DRAM writes — the traffic of a stage is its reads plus all its stores.
"""
import sys

import torch

sys.path.insert(0, ".")
import inputs  # noqa: E402
import paper_2601_12209_b200 as dfft  # noqa: E402

p1, p2 = int(sys.argv[1]), int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
prec = sys.argv[4] if len(sys.argv) > 4 else "f32"
shape = (n, n, n)
P = p1 * p2
comm = dfft.Comm.simulated(P, 0)
fwd = dfft.Plan(comm, shape, "pencil", (p1, p2), "c2c_" + prec, dfft.FORWARD, exchange="p2p")
inv = dfft.Plan(comm, shape, "pencil", (p1, p2), "c2c_" + prec, dfft.INVERSE, exchange="p2p")
xs, ys, zs = [], [], []
for r in range(P):
    lo, nn = fwd.box(0, r)
    x = fwd.alloc_in(r)
    inputs.fill_box_cuda(x, 1, shape, lo, nn, True)
    xs.append(x)
    ys.append(fwd.alloc_out(r))
    zs.append(inv.alloc_out(r))
k0 = dfft.kernel_launches()
fwd.execute_sim(xs, ys)
inv.execute_sim(ys, zs)
torch.cuda.synchronize()
per = dfft.kernel_launches() - k0
fwd.set_profiling(True)
inv.set_profiling(True)
fwd.phase_times(reset=True)
inv.phase_times(reset=True)
fwd.execute_sim(xs, ys)
inv.execute_sim(ys, zs)
torch.cuda.synchronize()
sf, si = fwd.timeline(), inv.timeline()
nstage = len(sf) + len(si)
print(f"grid {p1}x{p2} {n}^3 {prec}: {per} library launches per fwd+inv (incl. flag kernels), {nstage} stage launches, "
      f"K = {fwd.chunks()}")
bf, bi = fwd.stage_bytes(), inv.stage_bytes()
for tag, spans, b in (("fwd", sf, bf), ("inv", si, bi)):
    counts = {}
    for s in spans:
        counts[s["phase"]] = counts.get(s["phase"], 0) + 1
    for ph, c in counts.items():
        # per rank, per launch: the plan's stage bytes are per rank (rank 0's plan geometry)
        print(f"  {tag} {ph}: {c // P} launches per rank, algorithmic {b[ph] / (c // P) / 1e9:.4f} GB per launch")
