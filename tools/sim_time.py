"""Simulated-rank timing / ncu target (development aid): every rank's kernels of a P-rank plan
run in one process on cuda:0, so ncu can profile the multi-GPU layouts' kernels one by one.
    python tools/sim_time.py 1024,1024,1024 2,2 p2p f32 [iters]"""
import sys

import torch

sys.path.insert(0, ".")
import inputs
import paper_2601_12209_b200 as dfft

shape = tuple(int(v) for v in sys.argv[1].split(","))
grid = tuple(int(v) for v in sys.argv[2].split(","))
exch = sys.argv[3] if len(sys.argv) > 3 else "p2p"
prec = sys.argv[4] if len(sys.argv) > 4 else "f32"
n = int(sys.argv[5]) if len(sys.argv) > 5 else 3
torch.cuda.set_device(0)
P = grid[0] * grid[1]
comm = dfft.Comm.simulated(P, 0)
fwd = dfft.Plan(comm, shape, "pencil", grid, "c2c_" + prec, dfft.FORWARD, exchange=exch)
inv = dfft.Plan(comm, shape, "pencil", grid, "c2c_" + prec, dfft.INVERSE, exchange=exch)
xs, ys, zs = [], [], []
for r in range(P):
    lo, nn = fwd.box(0, r)
    x = fwd.alloc_in(r)
    inputs.fill_box_cuda(x, 1, shape, lo, nn, True)
    xs.append(x)
    ys.append(fwd.alloc_out(r))
    zs.append(inv.alloc_out(r))
for _ in range(n):
    fwd.execute_sim(xs, ys)
    inv.execute_sim(ys, zs)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(n):
    fwd.execute_sim(xs, ys)
    inv.execute_sim(ys, zs)
e.record()
torch.cuda.synchronize()
err = (sum((z - x).abs().pow(2).sum().item() for z, x in zip(zs, xs)) /
       sum(x.abs().pow(2).sum().item() for x in xs)) ** 0.5
print(f"sim {shape} grid {grid} {exch} {prec}: fwd+inv of all {P} ranks {s.elapsed_time(e) / n:.3f} ms, roundtrip {err:.2e}")
