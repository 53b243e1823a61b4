"""GPU parity of the per-axis transform kinds ("C2C, R2C and R2R", "DCT and
DST", P:620 the (Periodic, Periodic, Bounded) topology; reading R22) against the oracle's
written-out per-axis transforms (oracle.transform_kinds), and of the mixed-boundary Poisson solve
(readings R20 + R22) against oracle.poisson_kinds — one GPU, and simulated ranks in the
fused-store (IPC-window) and NCCL layouts."""
import numpy as np
import pytest

from helpers import GATE, QUALITY, box_slice

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import inputs  # noqa: E402
import paper_2601_12209_b200 as dfft  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    torch.cuda.set_device(0)


def _plans(shape, grid, dtype, kinds, exchange, decomp="pencil"):
    P = grid[0] * grid[1]
    comm = dfft.Comm.simulated(P, 0) if P > 1 else dfft.Comm.create(nranks=1, rank=0, device=0)
    fwd = dfft.Plan(comm, shape, decomp, grid, dtype, dfft.FORWARD, exchange=exchange, kinds=kinds)
    inv = dfft.Plan(comm, shape, decomp, grid, dtype, dfft.INVERSE, exchange=exchange, kinds=kinds)
    return comm, fwd, inv


def _run(plan, xs, ys):
    if plan.comm.nranks > 1:
        plan.execute_sim(xs, ys)
    else:
        plan.execute(xs[0], ys[0])


def _case(oracle_mod, shape, grid, prec, kinds, exchange="auto", decomp="pencil", seed=29, poisson=None):
    nx, ny, nz = shape
    r2r = kinds[0] != "dft"
    dtype = ("r2r_" if r2r else "r2c_") + prec
    comm, fwd, inv = _plans(shape, grid, dtype, kinds, exchange, decomp)
    if poisson:
        fwd.set_poisson(poisson)
    P = comm.nranks
    f32 = prec == "f32"
    xs, ys, zs = [], [], []
    for r in range(P):
        lo, n = fwd.box(0, r)
        x = fwd.alloc_in(r)
        inputs.fill_box_cuda(x, seed, shape, lo, n, False)
        xs.append(x)
        ys.append(fwd.alloc_out(r))
        zs.append(inv.alloc_out(r))
    _run(fwd, xs, ys)
    _run(inv, ys, zs)
    torch.cuda.synchronize()
    f = oracle_mod.gen_real(seed, shape, f32=f32)
    Z = np.zeros((nz, ny, nx))
    for r in range(P):
        lo, n = inv.box(1, r)
        box_slice(Z, lo, n)[...] = zs[r].cpu().numpy()
    if poisson:
        return oracle_mod.rel_l2(Z, oracle_mod.poisson_kinds(f, kinds, poisson)), None, None
    X = oracle_mod.transform_kinds(f if not r2r else f + 0j, kinds, real_x=not r2r)
    if r2r:
        X = X.real.copy()
    Y = np.zeros_like(X)
    for r in range(P):
        lo, n = fwd.box(1, r)
        box_slice(Y, lo, n)[...] = ys[r].cpu().numpy()
    # the inverse alone on an arbitrary spectrum (not the forward's output)
    H = (inputs.gen_real_np(seed + 1, shape, f32=f32) if r2r
         else inputs.gen_complex_np(seed + 1, (nx // 2 + 1, ny, nz), f32=f32).astype(np.complex128))
    hs, ws = [], []
    for r in range(P):
        lo, n = inv.box(0, r)
        t = torch.from_numpy(np.ascontiguousarray(box_slice(H, lo, n)))
        hs.append(t.to(torch.float32 if f32 else torch.float64).cuda() if r2r else
                  t.to(torch.complex64 if f32 else torch.complex128).cuda())
        ws.append(inv.alloc_out(r))
    _run(inv, hs, ws)
    torch.cuda.synchronize()
    W = np.zeros((nz, ny, nx))
    for r in range(P):
        lo, n = inv.box(1, r)
        box_slice(W, lo, n)[...] = ws[r].cpu().numpy()
    Wref = oracle_mod.transform_kinds(H if not r2r else H + 0j, kinds, inverse=True, real_x=not r2r, nx=nx)
    Wref = np.real(Wref)
    return oracle_mod.rel_l2(Y, X), oracle_mod.rel_l2(W, Wref), oracle_mod.rel_l2(Z, f)


KIND_CASES = [("dft", "dft", "dct"), ("dft", "dft", "dst"), ("dft", "dct", "dst"), ("dft", "dst", "dft"),
              ("dst", "dst", "dst"), ("dct", "dst", "dct")]


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("kinds", KIND_CASES)
@pytest.mark.parametrize("shape", [(16, 12, 8), (64, 48, 32)])
def test_kinds_single_gpu(oracle_mod, shape, kinds, prec):
    ef, ei, er = _case(oracle_mod, shape, (1, 1), prec, kinds)
    assert ef <= GATE[prec] and ei <= GATE[prec] and er <= GATE[prec], (ef, ei, er)
    assert ef <= QUALITY[prec] and ei <= QUALITY[prec], (ef, ei, er)


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("kinds", [("dft", "dft", "dct"), ("dft", "dft", "dst"), ("dst", "dct", "dst")])
@pytest.mark.parametrize("grid,exchange,decomp", [((2, 4), "p2p", "pencil"), ((2, 2), "nccl", "pencil"),
                                                  ((4, 1), "p2p", "slab")])
def test_kinds_simulated_ranks(oracle_mod, kinds, grid, exchange, decomp, prec):
    ef, ei, er = _case(oracle_mod, (48, 24, 16), grid, prec, kinds, exchange, decomp)
    assert ef <= GATE[prec] and ei <= GATE[prec] and er <= GATE[prec], (ef, ei, er)
    assert ef <= QUALITY[prec] and ei <= QUALITY[prec], (ef, ei, er)


@pytest.mark.parametrize("kinds", [("dft", "dft", "dct"), ("dft", "dft", "dst")])
def test_cfg5_box_ppb_f64(oracle_mod, kinds):
    # BASELINE configs[4]'s Oceananigans-shaped box (768x768x384 f64) in P:620's (Periodic, Periodic,
    # Bounded) form: R2C along x, DFT along y, DCT (Neumann) or DST (Dirichlet) along z
    ef, ei, er = _case(oracle_mod, (768, 768, 384), (1, 1), "f64", kinds, seed=260112209 + 5)
    assert ef <= 1e-12 and ei <= 1e-12 and er <= 1e-12, (ef, ei, er)


def test_cfg5_box_ppb_2x4_fused_store_f64(oracle_mod):
    ef, ei, er = _case(oracle_mod, (768, 768, 384), (2, 4), "f64", ("dft", "dft", "dct"), "p2p", seed=260112209 + 5)
    assert ef <= 1e-12 and ei <= 1e-12 and er <= 1e-12, (ef, ei, er)


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("kinds,grid,exchange,h", [
    (("dft", "dft", "dct"), (1, 1), "auto", (1.0, 0.5, 2.0)),
    (("dft", "dft", "dst"), (1, 1), "auto", (1.0, 1.0, 1.0)),
    (("dct", "dct", "dct"), (1, 1), "auto", (1.0, 2.0, 0.5)),
    (("dst", "dct", "dst"), (1, 1), "auto", (0.5, 1.0, 1.0)),
    (("dft", "dst", "dct"), (1, 1), "auto", (2.0, 1.0, 0.25)),
    (("dft", "dft", "dct"), (2, 4), "p2p", (1.0, 0.5, 2.0)),   # fused-store layouts, last stage = z DCT
    (("dst", "dct", "dst"), (2, 2), "p2p", (0.5, 1.0, 1.0)),
])
def test_poisson_mixed_boundaries(oracle_mod, kinds, grid, exchange, h, prec):
    e, _, _ = _case(oracle_mod, (48, 24, 16), grid, prec, kinds, exchange, poisson=h)
    assert e <= GATE[prec], e


def test_poisson_cfg5_box_ppb_f64(oracle_mod):
    # the paper's application on P:620's (Periodic, Periodic, Bounded) box, Neumann along z
    e, _, _ = _case(oracle_mod, (768, 768, 384), (1, 1), "f64", ("dft", "dft", "dct"), poisson=(1.0, 1.0, 1.0),
                    seed=260112209 + 5)
    assert e <= 1e-12, e


def test_kinds_rejected_combinations():
    comm = dfft.Comm.create(nranks=1, rank=0, device=0)
    for dtype, kinds in (("c2c_f64", ("dct", "dft", "dft")), ("r2r_f64", ("dct", "dft", "dct")),
                         ("r2c_f64", ("dst", "dft", "dft"))):
        with pytest.raises(dfft.DfftError):
            dfft.Plan(comm, (16, 12, 8), "pencil", (1, 1), dtype, dfft.FORWARD, kinds=kinds)
    with pytest.raises(dfft.DfftError):  # odd extent on a DCT axis
        dfft.Plan(comm, (16, 12, 7), "pencil", (1, 1), "r2c_f64", dfft.FORWARD, kinds=("dft", "dft", "dct"))
