import sys, torch
sys.path.insert(0, ".")
import inputs, paper_2601_12209_b200 as dfft
torch.cuda.set_device(0)
shape = tuple(int(v) for v in sys.argv[1].split(","))
comm = dfft.Comm.create(nranks=1, rank=0, device=0)
fwd = dfft.Plan(comm, shape, "pencil", (1, 1), "c2c_f32", dfft.FORWARD)
x = fwd.alloc_in(); inputs.fill_box_cuda(x, 1, shape, (0, 0, 0), shape, True)
y = fwd.alloc_out()
fwd.execute(x, y); torch.cuda.synchronize(); print("ok", shape)
