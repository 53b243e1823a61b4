import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import inputs, oracle
import paper_2601_12209_b200 as dfft
oracle.build()
torch.cuda.set_device(0)
comm = dfft.Comm.create(nranks=1, rank=0, device=0)
for shape in [(4, 4, 16), (4, 16, 4), (16, 4, 4), (16, 12, 8)]:
    nx, ny, nz = shape
    inv = dfft.Plan(comm, shape, "pencil", (1, 1), "r2r_f64", dfft.INVERSE)
    H = inputs.gen_real_np(5, shape)
    h = torch.from_numpy(H).cuda()
    z = inv.alloc_out()
    inv.execute(h, z)
    torch.cuda.synchronize()
    ref = oracle.dct3d(H, inverse=True)
    Z = z.cpu().numpy()
    print(shape, "rel", oracle.rel_l2(Z, ref))
    if oracle.rel_l2(Z, ref) > 1e-10:
        # which axis: apply oracle forward to Z and compare with H per axis
        import scipy.fft as sf
        for ax, name in ((2, "x"), (1, "y"), (0, "z")):
            part = sf.idct(H, type=2, axis=ax)
            print("   after only", name, "inverse: rel to GPU", oracle.rel_l2(Z, part))
        print("   GPU[0,0,:8]", Z[0, 0, :8])
        print("   ref[0,0,:8]", ref[0, 0, :8])
