"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Gates (BASELINE.json north_star): rel-L2 <= 2e-5 (fp32), <= 1e-12 (fp64) vs the fp64 oracle
fed bit-identical inputs (fp32 plans: inputs rounded to float on both sides).  Tighter
QUALITY bounds catch precision bugs the gate is blind to.
"""
import numpy as np
import pytest

from helpers import GATE, LENGTHS, QUALITY, box_slice, rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import inputs  # noqa: E402
import paper_2601_12209_b200 as dfft  # noqa: E402

CDT = {"f32": torch.complex64, "f64": torch.complex128}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    torch.cuda.set_device(0)


def _t(a, prec):
    return torch.from_numpy(np.ascontiguousarray(a)).to(CDT[prec]).cuda()


# ------------------------------------------------------------------------------ generator bits
def test_cuda_generator_matches_numpy_bits():
    g, lo, n = (24, 20, 12), (3, 5, 2), (17, 9, 7)
    for f32 in (False, True):
        t = torch.empty((n[2], n[1], n[0]), dtype=torch.complex64 if f32 else torch.complex128, device="cuda")
        inputs.fill_box_cuda(t, 99, g, lo, n, True)
        ref = inputs.gen_complex_np(99, g, lo, n, f32=f32)
        assert np.array_equal(t.cpu().numpy().view(np.uint8), ref.view(np.uint8))
        r = torch.empty((n[2], n[1], n[0]), dtype=torch.float32 if f32 else torch.float64, device="cuda")
        inputs.fill_box_cuda(r, 99, g, lo, n, False)
        assert np.array_equal(r.cpu().numpy(), inputs.gen_real_np(99, g, lo, n, f32=f32))


# ------------------------------------------------------------------------------ 1D kernels
@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("n", LENGTHS)
def test_fft1d_every_length(oracle_mod, n, prec):
    batch = 37  # ragged against lines-per-CTA
    x = inputs.gen_complex_np(7, (n, batch, 1), f32=(prec == "f32"))[0]  # (batch, n)
    xt = _t(x, prec)
    for sign in (-1, 1):
        y = torch.empty_like(xt)
        dfft.fft1d(xt, y, sign)
        torch.cuda.synchronize()
        ref = np.stack([oracle_mod.fft1d(row.astype(np.complex128), sign) for row in x])
        e = rel_l2(y.cpu().numpy(), ref)
        assert e <= GATE[prec], (n, sign, e)
        assert e <= QUALITY[prec], (n, sign, e)


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("n", [8, 64, 384, 480, 720, 768, 840, 1024, 4096])
def test_fft1d_plane_waves_exact_bins(n, prec):
    # exp(+2πi m t/n) -> n at k = m only: a misplaced bin is an O(1) error (pin independent of the oracle)
    ms = [0, 1, n // 3, n // 2, n - 1]
    t = np.arange(n)
    x = np.stack([np.exp(2j * np.pi * ((m * t) % n) / n) for m in ms])
    y = torch.empty((len(ms), n), dtype=CDT[prec], device="cuda")
    dfft.fft1d(_t(x, prec), y, -1)
    torch.cuda.synchronize()
    e = np.zeros((len(ms), n), complex)
    e[np.arange(len(ms)), ms] = n
    tol = (2e-4 if prec == "f32" else 1e-11) * n
    assert np.abs(y.cpu().numpy() - e).max() < tol


# ------------------------------------------------------------------------------ 3D, one GPU
def _run_single(oracle_mod, shape, decomp, prec, seed=3):
    comm = dfft.Comm.create(nranks=1, rank=0, device=0)
    dt = "c2c_" + prec
    fwd = dfft.Plan(comm, shape, decomp, (1, 1), dt, dfft.FORWARD)
    inv = dfft.Plan(comm, shape, decomp, (1, 1), dt, dfft.INVERSE)
    x = fwd.alloc_in()
    inputs.fill_box_cuda(x, seed, shape, (0, 0, 0), shape, True)
    y = fwd.alloc_out()
    z = inv.alloc_out()
    fwd.execute(x, y)
    inv.execute(y, z)
    torch.cuda.synchronize()
    a = oracle_mod.gen_complex(seed, shape, f32=(prec == "f32"))
    A = oracle_mod.fft3d(a, -1)
    ef = oracle_mod.rel_l2(y.cpu().numpy(), A)
    er = oracle_mod.rel_l2(z.cpu().numpy(), a)
    # inverse alone against the oracle's inverse of the same (GPU-produced) spectrum
    B = oracle_mod.fft3d(y.cpu().numpy().astype(np.complex128), +1)
    ei = oracle_mod.rel_l2(z.cpu().numpy(), B)
    return ef, er, ei


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape", [(64, 64, 64), (8, 8, 8), (16, 12, 8), (6, 24, 48), (480, 3, 7), (2, 4, 4096),
                                   (1024, 8, 6), (5, 768, 2), (840, 4, 2), (4, 720, 3)])
def test_3d_single_gpu(oracle_mod, shape, prec):
    ef, er, ei = _run_single(oracle_mod, shape, "pencil", prec)
    assert ef <= GATE[prec] and er <= GATE[prec] and ei <= GATE[prec], (ef, er, ei)
    assert ef <= QUALITY[prec] and ei <= QUALITY[prec], (ef, er, ei)


def test_cfg1_64cubed_c128_slab(oracle_mod):
    # BASELINE.json configs[0]: 64^3 complex128 c2c forward+inverse, single GPU, slab
    ef, er, ei = _run_single(oracle_mod, (64, 64, 64), "slab", "f64", seed=260112209 + 1)
    assert ef <= 1e-12 and er <= 1e-12 and ei <= 1e-12


def test_closed_forms_3d_gpu():
    shape = (64, 48, 32)
    comm = dfft.Comm.create(nranks=1, rank=0, device=0)
    fwd = dfft.Plan(comm, shape, "pencil", (1, 1), "c2c_f64", dfft.FORWARD)
    x = fwd.alloc_in().zero_()
    x[0, 0, 0] = 1
    y = fwd.alloc_out()
    fwd.execute(x, y)
    assert (y - 1).abs().max().item() < 1e-14  # delta -> all ones
    c = 0.25 - 0.5j
    x.fill_(c)
    fwd.execute(x, y)
    yy = y.cpu().numpy()
    assert abs(yy[0, 0, 0] - c * x.numel()) < 1e-9
    yy[0, 0, 0] = 0
    assert np.abs(yy).max() < 1e-9  # constant -> DC spike only


# ------------------------------------------------------------------------------ simulated ranks
def _run_sim(oracle_mod, shape, decomp, grid, prec, chunks, seed=5, exchange="auto"):
    P = grid[0] * grid[1]
    comm = dfft.Comm.simulated(P, 0)
    dt = "c2c_" + prec
    fwd = dfft.Plan(comm, shape, decomp, grid, dt, dfft.FORWARD, chunks=chunks, exchange=exchange)
    inv = dfft.Plan(comm, shape, decomp, grid, dt, dfft.INVERSE, chunks=chunks, exchange=exchange)
    xs, ys, zs = [], [], []
    for r in range(P):
        lo, n = fwd.box(0, r)
        x = fwd.alloc_in(r)
        inputs.fill_box_cuda(x, seed, shape, lo, n, True)
        xs.append(x)
        ys.append(fwd.alloc_out(r))
        zs.append(inv.alloc_out(r))
    fwd.execute_sim(xs, ys)
    inv.execute_sim(ys, zs)
    torch.cuda.synchronize()
    a = oracle_mod.gen_complex(seed, shape, f32=(prec == "f32"))
    A = oracle_mod.fft3d(a, -1)
    Y = np.zeros_like(A)
    Z = np.zeros_like(a)
    for r in range(P):
        lo, n = fwd.box(1, r)
        box_slice(Y, lo, n)[...] = ys[r].cpu().numpy()
        lo, n = inv.box(1, r)
        box_slice(Z, lo, n)[...] = zs[r].cpu().numpy()
    return oracle_mod.rel_l2(Y, A), oracle_mod.rel_l2(Z, a), Y


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape,decomp,grid,chunks", [
    ((32, 24, 16), "pencil", (2, 4), 1),
    ((32, 24, 16), "pencil", (2, 4), 2),
    ((32, 24, 16), "pencil", (2, 4), 3),
    ((16, 16, 12), "slab", (4, 1), 2),
    ((48, 12, 6), "pencil", (5, 2), 3),      # uneven splits on every axis
    ((24, 96, 64), "pencil", (4, 2), 4),
    ((64, 64, 64), "slab", (8, 1), 4),
    ((12, 6, 8), "pencil", (3, 2), 2),
])
def test_simulated_ranks(oracle_mod, shape, decomp, grid, chunks, prec):
    ef, er, _ = _run_sim(oracle_mod, shape, decomp, grid, prec, chunks)
    assert ef <= GATE[prec] and er <= GATE[prec], (ef, er)
    assert ef <= QUALITY[prec], ef


# fused-store ("p2p") layouts on simulated ranks: the column-blocked receive windows and the
# peer-window side maps the multi-GPU default uses, at grids gpurun cannot run (2x4, 4x2, 5x2)
@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape,decomp,grid", [
    ((32, 24, 16), "pencil", (2, 4)),
    ((64, 64, 64), "pencil", (4, 2)),
    ((48, 12, 6), "pencil", (5, 2)),       # uneven splits on every axis
    ((96, 48, 24), "pencil", (2, 4)),      # blocks not multiples of the 64 B column tile
    ((64, 64, 64), "slab", (8, 1)),
    ((256, 128, 64), "pencil", (2, 2)),
])
def test_simulated_ranks_fused_store(oracle_mod, shape, decomp, grid, prec):
    ef, er, _ = _run_sim(oracle_mod, shape, decomp, grid, prec, 0, exchange="p2p")
    assert ef <= GATE[prec] and er <= GATE[prec], (ef, er)
    assert ef <= QUALITY[prec], ef


# chunked fused-store plans (two-stream pipeline on real ranks): z-chunks forward, x-chunks on
# column-block bounds inverse, incl. chunks that come out empty
@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape,decomp,grid,chunks", [
    ((64, 64, 64), "pencil", (1, 4), 4),
    ((64, 64, 64), "pencil", (2, 4), 3),
    ((96, 48, 24), "pencil", (2, 2), 2),
    ((48, 12, 6), "pencil", (5, 2), 3),
    ((128, 64, 32), "slab", (2, 1), 8),
])
def test_simulated_ranks_fused_store_chunked(oracle_mod, shape, decomp, grid, chunks, prec):
    ef, er, _ = _run_sim(oracle_mod, shape, decomp, grid, prec, chunks, exchange="p2p")
    assert ef <= GATE[prec] and er <= GATE[prec], (ef, er)
    assert ef <= QUALITY[prec], ef


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape,grid", [((480, 96, 48), (2, 2)), ((96, 720, 48), (1, 2)), ((48, 96, 840), (2, 4))])
def test_simulated_ranks_fused_store_radix57(oracle_mod, shape, grid, prec):
    # the paper's GPU shapes' lengths (radix 5/7, f1) through the multi-GPU default layouts
    ef, er, _ = _run_sim(oracle_mod, shape, "pencil", grid, prec, 0, exchange="p2p")
    assert ef <= GATE[prec] and er <= GATE[prec], (ef, er)
    assert ef <= QUALITY[prec], ef


def test_fused_store_bitwise_equals_nccl_layouts(oracle_mod):
    # same kernels and radix schedules, different exchange layouts => identical bits
    shape = (32, 24, 16)
    _, _, Y1 = _run_sim(oracle_mod, shape, "pencil", (2, 4), "f64", 1)
    _, _, Y2 = _run_sim(oracle_mod, shape, "pencil", (2, 4), "f64", 0, exchange="p2p")
    assert np.array_equal(Y1, Y2)


def test_simulated_rank_invariance(oracle_mod):
    # same kernels on every decomposition: identical arithmetic per line => identical bits
    shape = (32, 24, 16)
    _, _, Y1 = _run_sim(oracle_mod, shape, "pencil", (2, 4), "f64", 1)
    _, _, Y2 = _run_sim(oracle_mod, shape, "pencil", (2, 4), "f64", 3)
    _, _, Y3 = _run_sim(oracle_mod, shape, "pencil", (4, 2), "f64", 2)
    _, _, Y4 = _run_sim(oracle_mod, shape, "slab", (8, 1), "f64", 2)
    assert np.array_equal(Y1, Y2) and np.array_equal(Y1, Y3) and np.array_equal(Y1, Y4)


# ------------------------------------------------------------------------------ full size
def test_headline_1024cubed_c64_single_gpu(oracle_mod):
    """BASELINE configs[3] at N=1 (the bench workload): sampled bins vs the oracle's direct sums,
    round trip vs the regenerated input, Parseval — in the launch configuration bench.py times."""
    shape = (1024, 1024, 1024)
    seed = 260112209 + 4
    comm = dfft.Comm.create(nranks=1, rank=0, device=0)
    fwd = dfft.Plan(comm, shape, "pencil", (1, 1), "c2c_f32", dfft.FORWARD)
    inv = dfft.Plan(comm, shape, "pencil", (1, 1), "c2c_f32", dfft.INVERSE)
    x = fwd.alloc_in()
    inputs.fill_box_cuda(x, seed, shape, (0, 0, 0), shape, True)
    y = fwd.alloc_out()
    fwd.execute(x, y)
    rng = np.random.default_rng(0)
    ks = [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (1023, 1023, 1023), (512, 512, 512)]
    ks += [tuple(int(v) for v in rng.integers(0, 1024, 3)) for _ in range(6)]
    got = [complex(y[kz, ky, kx].item()) for kx, ky, kz in ks]
    N = float(np.prod(shape))
    err2 = 0.0
    for (kx, ky, kz), g in zip(ks, got):
        ref = oracle_mod.dft3d_bin_seeded(seed, shape, (kx, ky, kz), f32=True)
        err2 += abs(g - ref) ** 2
    # normalise by the expected bin magnitude sqrt(N * E|x|^2) = sqrt(2N/3) for uniform[-1,1) re/im
    rms_rel = np.sqrt(err2 / len(ks)) / np.sqrt(2 * N / 3)
    assert rms_rel <= GATE["f32"], rms_rel
    # Parseval: sum|X|^2 = N sum|x|^2
    sx = torch.sum(x.abs().double() ** 2).item()
    sX = torch.sum(y.abs().double() ** 2).item()
    assert abs(sX / (N * sx) - 1) < 1e-5
    z = inv.alloc_out()
    inv.execute(y, z)
    del y
    d = (z - x).abs().double().pow(2).sum().item()
    assert np.sqrt(d / sx) <= GATE["f32"]


def test_headline_1024cubed_c64_2x4_fused_store_simulated(oracle_mod):
    """BASELINE configs[3] in the 8-GPU headline's decomposition (pencil 2x4, fused-store layouts,
    the multi-GPU default) on one GPU with simulated ranks: sampled bins vs the oracle's direct
    sums and the round trip.  Same kernels and addresses as 8 processes, stream order for flags."""
    shape = (1024, 1024, 1024)
    seed = 260112209 + 4
    grid = (2, 4)
    P = 8
    comm = dfft.Comm.simulated(P, 0)
    fwd = dfft.Plan(comm, shape, "pencil", grid, "c2c_f32", dfft.FORWARD, exchange="p2p")
    inv = dfft.Plan(comm, shape, "pencil", grid, "c2c_f32", dfft.INVERSE, exchange="p2p")
    xs, ys, zs = [], [], []
    for r in range(P):
        lo, n = fwd.box(0, r)
        x = fwd.alloc_in(r)
        inputs.fill_box_cuda(x, seed, shape, lo, n, True)
        xs.append(x)
        ys.append(fwd.alloc_out(r))
    fwd.execute_sim(xs, ys)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    ks = [(0, 0, 0), (511, 255, 1023), (512, 256, 0), (1023, 1023, 1023)]
    ks += [tuple(int(v) for v in rng.integers(0, 1024, 3)) for _ in range(8)]
    N = float(np.prod(shape))
    err2 = 0.0
    for kx, ky, kz in ks:
        for r in range(P):
            lo, n = fwd.box(1, r)
            if all(lo[d] <= k < lo[d] + n[d] for d, k in enumerate((kx, ky, kz))):
                g = complex(ys[r][kz - lo[2], ky - lo[1], kx - lo[0]].item())
        ref = oracle_mod.dft3d_bin_seeded(seed, shape, (kx, ky, kz), f32=True)
        err2 += abs(g - ref) ** 2
    rms_rel = np.sqrt(err2 / len(ks)) / np.sqrt(2 * N / 3)
    assert rms_rel <= GATE["f32"], rms_rel
    zs = [inv.alloc_out(r) for r in range(P)]
    inv.execute_sim(ys, zs)
    torch.cuda.synchronize()
    d = sum((z - x).abs().double().pow(2).sum().item() for z, x in zip(zs, xs))
    sx = sum(x.abs().double().pow(2).sum().item() for x in xs)
    assert np.sqrt(d / sx) <= GATE["f32"]


# ------------------------------------------------------------------------------ R2C / C2R
def _r2c_case(oracle_mod, shape, decomp, grid, prec, chunks=0, seed=9, exchange="auto"):
    """Forward R2C vs oracle rfft3d; C2R of an arbitrary (non-Hermitian) half spectrum vs the
    oracle's Hermitian-extension C2R (reading R8); C2R(R2C(x)) round trip."""
    nx, ny, nz = shape
    P = grid[0] * grid[1]
    comm = dfft.Comm.simulated(P, 0) if P > 1 else dfft.Comm.create(nranks=1, rank=0, device=0)
    dt = "r2c_" + prec
    fwd = dfft.Plan(comm, shape, decomp, grid, dt, dfft.FORWARD, chunks=chunks, exchange=exchange)
    inv = dfft.Plan(comm, shape, decomp, grid, dt, dfft.INVERSE, chunks=chunks, exchange=exchange)
    f32 = prec == "f32"
    xs, ys = [], []
    for r in range(P):
        lo, n = fwd.box(0, r)
        x = fwd.alloc_in(r)
        inputs.fill_box_cuda(x, seed, shape, lo, n, False)
        xs.append(x)
        ys.append(fwd.alloc_out(r))
    # arbitrary complex half spectrum for the C2R check
    H = inputs.gen_complex_np(seed + 1, (nx // 2 + 1, ny, nz), f32=f32).astype(np.complex128)
    hs = []
    for r in range(P):
        lo, n = inv.box(0, r)
        hs.append(_t(box_slice(H, lo, n), prec))
    zs = [inv.alloc_out(r) for r in range(P)]
    ws = [inv.alloc_out(r) for r in range(P)]
    if P > 1:
        fwd.execute_sim(xs, ys)
        inv.execute_sim(hs, zs)
        inv.execute_sim(ys, ws)
    else:
        fwd.execute(xs[0], ys[0])
        inv.execute(hs[0], zs[0])
        inv.execute(ys[0], ws[0])
    torch.cuda.synchronize()
    a = oracle_mod.gen_real(seed, shape, f32=f32)
    A = oracle_mod.rfft3d(a)
    Y = np.zeros_like(A)
    Zc = np.zeros((nz, ny, nx))
    Wr = np.zeros((nz, ny, nx))
    for r in range(P):
        lo, n = fwd.box(1, r)
        box_slice(Y, lo, n)[...] = ys[r].cpu().numpy()
        lo, n = inv.box(1, r)
        box_slice(Zc, lo, n)[...] = zs[r].cpu().numpy()
        box_slice(Wr, lo, n)[...] = ws[r].cpu().numpy()
    ef = oracle_mod.rel_l2(Y, A)
    ec = oracle_mod.rel_l2(Zc, oracle_mod.irfft3d(H, nx))
    er = oracle_mod.rel_l2(Wr, a)
    return ef, ec, er


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape,decomp,grid,chunks", [
    ((16, 12, 8), "pencil", (1, 1), 0),
    ((768, 48, 24), "pencil", (1, 1), 0),
    ((24, 16, 12), "pencil", (2, 4), 0),    # nx/2+1 = 13 bins split 7/6 (uneven, like cfg5's 193/192)
    ((24, 16, 12), "pencil", (2, 4), 3),
    ((48, 24, 12), "slab", (4, 1), 2),
    ((96, 48, 24), "pencil", (2, 2), 2),
])
def test_r2c_c2r(oracle_mod, shape, decomp, grid, chunks, prec):
    ef, ec, er = _r2c_case(oracle_mod, shape, decomp, grid, prec, chunks)
    assert ef <= GATE[prec] and ec <= GATE[prec] and er <= GATE[prec], (ef, ec, er)
    assert ef <= QUALITY[prec] and ec <= QUALITY[prec], (ef, ec, er)


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape,grid", [((24, 16, 12), (2, 4)), ((96, 48, 24), (2, 2)), ((48, 24, 12), (4, 1))])
def test_r2c_c2r_fused_store_simulated(oracle_mod, shape, grid, prec):
    ef, ec, er = _r2c_case(oracle_mod, shape, "pencil", grid, prec, exchange="p2p")
    assert ef <= GATE[prec] and ec <= GATE[prec] and er <= GATE[prec], (ef, ec, er)
    assert ef <= QUALITY[prec] and ec <= QUALITY[prec], (ef, ec, er)


def test_cfg5_r2c_2x4_fused_store_simulated(oracle_mod):
    # BASELINE configs[4] (768x768x384 r2c f64, pencil 2x4, uneven 193/192 bins) in the 8-GPU
    # default layouts, simulated on one GPU
    ef, ec, er = _r2c_case(oracle_mod, (768, 768, 384), "pencil", (2, 4), "f64", seed=260112209 + 5, exchange="p2p")
    assert ef <= 1e-12 and ec <= 1e-12 and er <= 1e-12, (ef, ec, er)


def test_cfg5_r2c_768x768x384_f64_single_gpu(oracle_mod):
    # BASELINE configs[4] shape (fp64, mixed radix 3·2^k) on one GPU: forward vs oracle, round trip
    ef, ec, er = _r2c_case(oracle_mod, (768, 768, 384), "pencil", (1, 1), "f64", seed=260112209 + 5)
    assert ef <= 1e-12 and ec <= 1e-12 and er <= 1e-12, (ef, ec, er)


# ------------------------------------------------------------------------------ Poisson (f3)
def _poisson_case(oracle_mod, shape, decomp, grid, prec, spacing, kind="r2c", exchange="auto", seed=21):
    """Forward plan with the fused 1/λ(k) multiplier, then the inverse plan: φ vs the oracle's
    poisson3d (reading R20) on the same seeded f."""
    nx, ny, nz = shape
    P = grid[0] * grid[1]
    comm = dfft.Comm.simulated(P, 0) if P > 1 else dfft.Comm.create(nranks=1, rank=0, device=0)
    dt = kind + "_" + prec
    fwd = dfft.Plan(comm, shape, decomp, grid, dt, dfft.FORWARD, exchange=exchange).set_poisson(spacing)
    inv = dfft.Plan(comm, shape, decomp, grid, dt, dfft.INVERSE, exchange=exchange)
    f32 = prec == "f32"
    xs, ys, zs = [], [], []
    for r in range(P):
        lo, n = fwd.box(0, r)
        x = fwd.alloc_in(r)
        inputs.fill_box_cuda(x, seed, shape, lo, n, kind == "c2c")
        xs.append(x)
        ys.append(fwd.alloc_out(r))
        zs.append(inv.alloc_out(r))
    if P > 1:
        fwd.execute_sim(xs, ys)
        inv.execute_sim(ys, zs)
    else:
        fwd.execute(xs[0], ys[0])
        inv.execute(ys[0], zs[0])
    torch.cuda.synchronize()
    if kind == "r2c":
        f = oracle_mod.gen_real(seed, shape, f32=f32)
        ref = oracle_mod.poisson3d(f, spacing)
        Z = np.zeros((nz, ny, nx))
    else:  # complex f: the solve is linear, so re and im parts separately
        a = oracle_mod.gen_complex(seed, shape, f32=f32)
        ref = oracle_mod.poisson3d(a.real.copy(), spacing) + 1j * oracle_mod.poisson3d(a.imag.copy(), spacing)
        Z = np.zeros((nz, ny, nx), dtype=complex)
    for r in range(P):
        lo, n = inv.box(1, r)
        box_slice(Z, lo, n)[...] = zs[r].cpu().numpy()
    return oracle_mod.rel_l2(Z, ref)


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape,decomp,grid,spacing,kind", [
    ((16, 12, 8), "pencil", (1, 1), (1.0, 1.0, 1.0), "r2c"),
    ((64, 48, 24), "pencil", (1, 1), (0.5, 2.0, 1.5), "r2c"),
    ((32, 24, 16), "pencil", (1, 1), (1.0, 0.25, 3.0), "c2c"),
    ((128, 12, 256), "pencil", (1, 1), (1.0, 0.5, 2.0), "c2c"),  # the xz8 plan: multiplier in its y pass
    ((48, 24, 12), "pencil", (2, 4), (1.0, 2.0, 0.5), "r2c"),   # fused-store layouts, B->C chunks
    ((96, 48, 24), "pencil", (2, 2), (1.0, 1.0, 1.0), "c2c"),
    ((64, 32, 16), "slab", (4, 1), (2.0, 1.0, 1.0), "r2c"),
])
def test_poisson_fused(oracle_mod, shape, decomp, grid, spacing, kind, prec):
    e = _poisson_case(oracle_mod, shape, decomp, grid, prec, spacing, kind, exchange="p2p" if grid != (1, 1) else "auto")
    assert e <= GATE[prec], e


def test_poisson_nccl_layouts_simulated(oracle_mod):
    e = _poisson_case(oracle_mod, (48, 24, 12), "pencil", (2, 4), "f64", (1.0, 1.0, 1.0), "r2c", exchange="nccl")
    assert e <= GATE["f64"], e


def test_poisson_cfg5_box_f64(oracle_mod):
    # the paper's application shape class (Oceananigans periodic box, BASELINE configs[4])
    e = _poisson_case(oracle_mod, (768, 768, 384), "pencil", (1, 1), "f64", (1.0, 1.0, 1.0), "r2c", seed=260112209 + 5)
    assert e <= 1e-12, e


# ------------------------------------------------------------------------------ R2R (f4)
def _r2r_case(oracle_mod, shape, decomp, grid, prec, exchange="auto", chunks=0, seed=23):
    """R2R forward (DCT-II per axis) vs oracle.dct3d, inverse of the oracle's spectrum (DCT-III /
    2N per axis) vs oracle.dct3d(inverse=True), round trip (reading R21)."""
    nx, ny, nz = shape
    P = grid[0] * grid[1]
    comm = dfft.Comm.simulated(P, 0) if P > 1 else dfft.Comm.create(nranks=1, rank=0, device=0)
    dt = "r2r_" + prec
    fwd = dfft.Plan(comm, shape, decomp, grid, dt, dfft.FORWARD, chunks=chunks, exchange=exchange)
    inv = dfft.Plan(comm, shape, decomp, grid, dt, dfft.INVERSE, chunks=chunks, exchange=exchange)
    f32 = prec == "f32"
    a = oracle_mod.gen_real(seed, shape, f32=f32)
    X = oracle_mod.dct3d(a)
    H = inputs.gen_real_np(seed + 1, shape, f32=f32)
    xs, ys, hs, zs, ws = [], [], [], [], []
    for r in range(P):
        lo, n = fwd.box(0, r)
        x = fwd.alloc_in(r)
        inputs.fill_box_cuda(x, seed, shape, lo, n, False)
        xs.append(x)
        ys.append(fwd.alloc_out(r))
        lo, n = inv.box(0, r)
        hs.append(torch.from_numpy(np.ascontiguousarray(box_slice(H, lo, n))).to(
            torch.float32 if f32 else torch.float64).cuda())
        zs.append(inv.alloc_out(r))
        ws.append(inv.alloc_out(r))
    if P > 1:
        fwd.execute_sim(xs, ys)
        inv.execute_sim(hs, zs)
        inv.execute_sim(ys, ws)
    else:
        fwd.execute(xs[0], ys[0])
        inv.execute(hs[0], zs[0])
        inv.execute(ys[0], ws[0])
    torch.cuda.synchronize()
    Y, Z, Wr = np.zeros_like(X), np.zeros_like(X), np.zeros_like(X)
    for r in range(P):
        lo, n = fwd.box(1, r)
        box_slice(Y, lo, n)[...] = ys[r].cpu().numpy()
        lo, n = inv.box(1, r)
        box_slice(Z, lo, n)[...] = zs[r].cpu().numpy()
        box_slice(Wr, lo, n)[...] = ws[r].cpu().numpy()
    return (oracle_mod.rel_l2(Y, X), oracle_mod.rel_l2(Z, oracle_mod.dct3d(H, inverse=True)),
            oracle_mod.rel_l2(Wr, a))


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape,decomp,grid,exchange", [
    ((16, 12, 8), "pencil", (1, 1), "auto"),
    ((64, 48, 32), "pencil", (1, 1), "auto"),
    ((24, 16, 12), "pencil", (2, 4), "nccl"),
    ((24, 16, 12), "pencil", (2, 4), "p2p"),   # fused-store layouts, B->C chunks
    ((48, 24, 12), "slab", (4, 1), "p2p"),
    ((48, 24, 12), "pencil", (5, 2), "nccl"),  # uneven pair splits
])
def test_r2r_dct(oracle_mod, shape, decomp, grid, exchange, prec):
    ef, ei, er = _r2r_case(oracle_mod, shape, decomp, grid, prec, exchange)
    assert ef <= GATE[prec] and ei <= GATE[prec] and er <= GATE[prec], (ef, ei, er)
    assert ef <= QUALITY[prec] and ei <= QUALITY[prec], (ef, ei, er)


def test_r2r_dct_256_f64_single_gpu(oracle_mod):
    ef, ei, er = _r2r_case(oracle_mod, (256, 128, 64), "pencil", (1, 1), "f64")
    assert ef <= 1e-12 and ei <= 1e-12 and er <= 1e-12, (ef, ei, er)


def test_cuda_graph_capture_single_gpu(oracle_mod):
    """dfft_execute is stream-ordered and capturable for single-rank plans: capture fwd+inv once,
    replay on new input, compare with the oracle (launch-bound small configs use this)."""
    shape = (64, 64, 64)
    comm = dfft.Comm.create(nranks=1, rank=0, device=0)
    fwd = dfft.Plan(comm, shape, "slab", (1, 1), "c2c_f64", dfft.FORWARD)
    inv = dfft.Plan(comm, shape, "slab", (1, 1), "c2c_f64", dfft.INVERSE)
    x, y, z = fwd.alloc_in(), fwd.alloc_out(), inv.alloc_out()
    inputs.fill_box_cuda(x, 3, shape, (0, 0, 0), shape, True)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up outside the capture (lazy init)
        fwd.execute(x, y, stream=s)
        inv.execute(y, z, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fwd.execute(x, y, stream=s)
        inv.execute(y, z, stream=s)
    inputs.fill_box_cuda(x, 7, shape, (0, 0, 0), shape, True)
    g.replay()
    torch.cuda.synchronize()
    a = oracle_mod.gen_complex(7, shape)
    assert oracle_mod.rel_l2(y.cpu().numpy(), oracle_mod.fft3d(a, -1)) <= 1e-12
    assert oracle_mod.rel_l2(z.cpu().numpy(), a) <= 1e-12


# ------------------------------------------------------------------------------ generic lengths
GENERIC = [10, 14, 45, 49, 60, 100, 343, 600, 960, 1000, 2187, 4000]


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("n", GENERIC)
def test_fft1d_generic_lengths(oracle_mod, n, prec):
    """2^a 3^b 5^c 7^d lengths without a specialised kernel run the generic runtime-schedule kernel
    (csrc/fft_kernels.cuh fft_generic_kernel): the DFT definition vs the oracle."""
    batch = 11
    x = inputs.gen_complex_np(3, (n, batch, 1), f32=(prec == "f32"))[0]
    xt = _t(x, prec)
    for sign in (-1, 1):
        y = torch.empty_like(xt)
        dfft.fft1d(xt, y, sign)
        torch.cuda.synchronize()
        ref = np.stack([oracle_mod.fft1d(row.astype(np.complex128), sign) for row in x])
        e = rel_l2(y.cpu().numpy(), ref)
        assert e <= QUALITY[prec], (n, sign, e)


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape", [(60, 50, 42), (100, 14, 96), (600, 10, 8)])
def test_3d_generic_lengths_single_gpu(oracle_mod, shape, prec):
    ef, er, ei = _run_single(oracle_mod, shape, "pencil", prec)
    assert ef <= QUALITY[prec] and ei <= QUALITY[prec] and er <= GATE[prec], (ef, er, ei)


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape,grid,exchange", [((60, 50, 42), (2, 2), "p2p"), ((100, 14, 96), (2, 4), "p2p"),
                                                 ((60, 50, 42), (2, 2), "nccl")])
def test_generic_lengths_simulated_ranks(oracle_mod, shape, grid, exchange, prec):
    ef, er, _ = _run_sim(oracle_mod, shape, "pencil", grid, prec, 0, exchange=exchange)
    assert ef <= QUALITY[prec] and er <= GATE[prec], (ef, er)


def test_generic_length_poisson(oracle_mod):
    # the strided generic kernel carries the Poisson multiplier too (last forward stage)
    e = _poisson_case(oracle_mod, (60, 50, 42), "pencil", (1, 1), "f64", (1.0, 2.0, 0.5), "c2c")
    assert e <= GATE["f64"], e


# ------------------------------------------------------------------ single-GPU radix-8 z split (xz8)
# nz = 8·M with M specialised: the single-GPU c2c plan splits the z-FFT by one radix-8 DIF step fused
# into the x pass (fft_xz8_kernel).  The oracle's plain 3D DFT is the reference; the
# DFFT_NO_XZ8 plan (three whole-axis passes) is a second, independent check of the same transform.
XZ8_SHAPES = [(128, 16, 256), (256, 6, 512), (480, 5, 384), (840, 3, 256), (720, 4, 512), (1024, 4, 256),
              (128, 9, 1024), (768, 3, 192), (2048, 2, 256), (480, 5, 96)]
# the fused kernel needs two CTAs an SM: f32 radix-32 lines (512 | N, N >= 512) and
# radix-16 lines of <= 512 threads (f32); nx = 2048 (f32) / 1024 (f64) hold 135-139 KB of lines, and
# 840 (f32/f64), 720 / 768 (f64) need more registers than two CTAs leave: whole-axis plan
XZ8_FUSED = {"f32": [(128, 16, 256), (256, 6, 512), (480, 5, 384), (720, 4, 512), (1024, 4, 256), (128, 9, 1024),
                     (768, 3, 192), (480, 5, 96)],
             "f64": [(128, 16, 256), (256, 6, 512), (480, 5, 384), (128, 9, 1024), (480, 5, 96)]}
# nx without the fused kernel (64: fewer than 64 threads; 60: generic; 4096: over 1024 threads) or
# nz/8 without a TMA strided kernel (8, 16: one pass; 21: not specialised): the whole-axis plan
XZ8_FALLBACK = [(64, 16, 256), (64, 16, 64), (256, 6, 128), (96, 7, 168), (60, 5, 64), (4096, 2, 256)]


def _families(shape, prec):
    comm = dfft.Comm.create(nranks=1, rank=0, device=0)
    return [d["family"] for d in dfft.Plan(comm, shape, "pencil", (1, 1), "c2c_" + prec, dfft.FORWARD).describe()]


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape", XZ8_SHAPES + XZ8_FALLBACK)
def test_3d_single_gpu_xz8(oracle_mod, shape, prec):
    fused = shape in XZ8_FUSED[prec]
    assert ("xz8" in _families(shape, prec)) == fused, (_families(shape, prec), shape, prec)
    ef, er, ei = _run_single(oracle_mod, shape, "pencil", prec, seed=31)
    assert ef <= GATE[prec] and er <= GATE[prec] and ei <= GATE[prec], (ef, er, ei)
    assert ef <= QUALITY[prec] and ei <= QUALITY[prec], (ef, er, ei)


@pytest.mark.parametrize("shape", [(256, 6, 512), (128, 9, 1024)])
def test_xz8_matches_whole_axis_plan(shape, monkeypatch):
    comm = dfft.Comm.create(nranks=1, rank=0, device=0)
    x = None
    outs = []
    for off in (False, True):
        if off:
            monkeypatch.setenv("DFFT_NO_XZ8", "1")
        fwd = dfft.Plan(comm, shape, "pencil", (1, 1), "c2c_f64", dfft.FORWARD)
        fams = [d["family"] for d in fwd.describe()]
        assert ("xz8" in fams) == (not off) and fams[1] == "strided", fams
        if x is None:
            x = fwd.alloc_in()
            inputs.fill_box_cuda(x, 17, shape, (0, 0, 0), shape, True)
        y = fwd.alloc_out()
        fwd.execute(x, y)
        torch.cuda.synchronize()
        outs.append(y.cpu().numpy())
    assert rel_l2(outs[0], outs[1]) < 1e-14


def _sweep_shapes(count=16, seed=2601):
    """Seeded 3D shapes over the specialised lengths, <= 2^21 points: the plan picks xz8 or the
    whole-axis passes, radix 16 or 32, by the rules of DESIGN.md §5 — none chosen by hand."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        s = tuple(int(v) for v in rng.choice(LENGTHS, 3))
        if 8 <= s[0] * s[1] * s[2] <= (1 << 21) and (s[0], s[1], s[2]) not in out:
            out.append(s)
    return out


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape", _sweep_shapes())
def test_3d_single_gpu_seeded_sweep(oracle_mod, shape, prec):
    ef, er, ei = _run_single(oracle_mod, shape, "pencil", prec, seed=47)
    assert ef <= GATE[prec] and er <= GATE[prec] and ei <= GATE[prec], (shape, ef, er, ei)
