"""Quick per-stage timing of the single-GPU path (development aid)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import inputs
import paper_2601_12209_b200 as dfft

torch.cuda.set_device(0)
shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1024,1024,1024").split(","))
prec = sys.argv[2] if len(sys.argv) > 2 else "f32"
comm = dfft.Comm.create(nranks=1, rank=0, device=0)
fwd = dfft.Plan(comm, shape, "pencil", (1, 1), "c2c_" + prec, dfft.FORWARD)
inv = dfft.Plan(comm, shape, "pencil", (1, 1), "c2c_" + prec, dfft.INVERSE)
n = int(sys.argv[3]) if len(sys.argv) > 3 else 10
x = fwd.alloc_in()
inputs.fill_box_cuda(x, 1, shape, (0, 0, 0), shape, True)
y = fwd.alloc_out()
z = inv.alloc_out()
for _ in range(3 if n > 1 else 1):
    fwd.execute(x, y)
    inv.execute(y, z)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(n):
    fwd.execute(x, y)
e.record()
torch.cuda.synchronize()
tf = s.elapsed_time(e) / n
s.record()
for _ in range(n):
    fwd.execute(x, y)
    inv.execute(y, z)
e.record()
torch.cuda.synchronize()
tfi = s.elapsed_time(e) / n
N = shape[0] * shape[1] * shape[2]
es = 8 if prec == "f32" else 16
hbm = 6 * N * es
print(f"{shape} {prec}: fwd {tf:.3f} ms ({hbm / tf / 1e6:.0f} GB/s eff), fwd+inv {tfi:.3f} ms, "
      f"roundtrip err {((z - x).abs().pow(2).sum() / x.abs().pow(2).sum()).sqrt().item():.2e}")
fwd.set_profiling(True)
inv.set_profiling(True)
fwd.phase_times()
inv.phase_times()
for _ in range(3):
    fwd.execute(x, y)
    inv.execute(y, z)
pf, pi = fwd.phase_times(), inv.phase_times()
print("  fwd " + " ".join(f"{k}={v[0] / 3:.3f}" for k, v in pf.items() if v[1]) +
      " | inv " + " ".join(f"{k}={v[0] / 3:.3f}" for k, v in pi.items() if v[1]))
