"""GPU: the product's multi-rank executor on simulated ranks, and element-wise parity of the
full-size kernel configurations the 1024^3 bench runs.

Simulated ranks with an IPC-window transport (exchange p2p / ce / hybrid) run every rank's own
execute schedule exactly as a real rank does (include/dfft.h dfft_execute_sim): its stream pair,
the READY/DONE flag words in its workspace (standing in for its IPC window), cuStreamWaitValue32
waits, the B->C / K-chunk pipeline and the SM caps.  That is Alg. 2's progressive exchange
 and Fig. 1's per-chunk pipeline; the results must equal the
oracle's 3D DFT and, bit for bit, the serial NCCL-layout simulation (same kernels, same
arithmetic per line).
"""
import time

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


def _sim_plans(shape, decomp, grid, dtype, exchange, chunks=0, overlap=True):
    P = grid[0] * grid[1]
    comm = dfft.Comm.simulated(P, 0)
    fwd = dfft.Plan(comm, shape, decomp, grid, dtype, dfft.FORWARD, chunks=chunks, exchange=exchange, overlap=overlap)
    inv = dfft.Plan(comm, shape, decomp, grid, dtype, dfft.INVERSE, chunks=chunks, exchange=exchange, overlap=overlap)
    return comm, fwd, inv


def _fill(plan, shape, seed, cplx=True):
    xs = []
    for r in range(plan.comm.nranks):
        lo, n = plan.box(0, r)
        x = plan.alloc_in(r)
        inputs.fill_box_cuda(x, seed, shape, lo, n, cplx)
        xs.append(x)
    return xs


def _gather(plan, ts, which, like):
    G = np.zeros_like(like)
    for r, t in enumerate(ts):
        lo, n = plan.box(which, r)
        box_slice(G, lo, n)[...] = t.cpu().numpy()
    return G


def _run(shape, decomp, grid, prec, exchange, chunks=0, overlap=True, seed=5, repeats=2):
    """fwd+inv `repeats` times (the second execute runs the flag-reset / buffer-reuse path)."""
    comm, fwd, inv = _sim_plans(shape, decomp, grid, "c2c_" + prec, exchange, chunks, overlap)
    P = comm.nranks
    xs = _fill(fwd, shape, seed)
    ys = [fwd.alloc_out(r) for r in range(P)]
    zs = [inv.alloc_out(r) for r in range(P)]
    for it in range(repeats):
        for y in ys:
            y.fill_(float("nan"))  # a missed store must show
        fwd.execute_sim(xs, ys)
        inv.execute_sim(ys, zs)
        torch.cuda.synchronize()
    assert fwd.status() == 0 and inv.status() == 0
    return fwd, inv, xs, ys, zs


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape,decomp,grid,exchange,chunks", [
    ((32, 24, 16), "pencil", (2, 4), "p2p", 0),      # 8-GPU headline grid, B->C pipeline, K = 1
    ((64, 64, 64), "pencil", (2, 4), "p2p", 4),      # B->C with 4 chunks (SM caps, two streams)
    ((64, 64, 64), "pencil", (2, 2), "p2p", 3),
    ((64, 64, 64), "pencil", (1, 4), "p2p", 4),      # 1xP2: forward B->C, inverse A||B chunks
    ((48, 12, 6), "pencil", (5, 2), "p2p", 2),       # uneven splits
    ((128, 64, 32), "slab", (2, 1), "p2p", 8),
    ((64, 64, 64), "pencil", (2, 2), "ce", 4),       # copy-engine transport, K-chunk pipeline
    ((48, 12, 6), "pencil", (5, 2), "ce", 3),
    ((64, 32, 16), "pencil", (2, 4), "hybrid", 2),   # fused forward x-FFT, CE elsewhere
])
def test_sim_product_executor(oracle_mod, shape, decomp, grid, exchange, chunks, prec):
    fwd, inv, xs, ys, zs = _run(shape, decomp, grid, prec, exchange, chunks)
    a = oracle_mod.gen_complex(5, shape, f32=(prec == "f32"))
    A = oracle_mod.fft3d(a, -1)
    Y = _gather(fwd, ys, 1, A)
    Z = _gather(inv, zs, 1, a)
    ef, er = oracle_mod.rel_l2(Y, A), oracle_mod.rel_l2(Z, a)
    assert ef <= GATE[prec] and er <= GATE[prec], (ef, er)
    assert ef <= QUALITY[prec], ef
    # bitwise equal to the serial NCCL-layout simulation: same kernels, same per-line arithmetic
    _, fwd_n, _ = _sim_plans(shape, decomp, grid, "c2c_" + prec, "nccl", chunks)
    ys_n = [fwd_n.alloc_out(r) for r in range(len(xs))]
    fwd_n.execute_sim(xs, ys_n)
    torch.cuda.synchronize()
    assert np.array_equal(Y, _gather(fwd_n, ys_n, 1, A))


@pytest.mark.parametrize("shape,grid,chunks", [
    ((128, 384, 256), (1, 2), 4),   # wy = 10, wz = 16 (f32 TMA tile widths): chunk bounds at lcm = 80
    ((128, 384, 256), (2, 2), 4),
    ((384, 384, 256), (1, 2), 4),   # 5 blocks of 80 columns over 4 chunks, partial last block
])
def test_sim_chunk_bounds_unequal_tile_widths(oracle_mod, shape, grid, chunks):
    fwd, inv, xs, ys, zs = _run(shape, "pencil", grid, "f32", "p2p", chunks, seed=11)
    a = oracle_mod.gen_complex(11, shape, f32=True)
    A = oracle_mod.fft3d(a, -1)
    ef = oracle_mod.rel_l2(_gather(fwd, ys, 1, A), A)
    er = oracle_mod.rel_l2(_gather(inv, zs, 1, a), a)
    assert ef <= QUALITY["f32"] and er <= GATE["f32"], (ef, er)


@pytest.mark.parametrize("exchange", ["p2p", "ce"])
def test_sim_no_overlap_bitwise(exchange):
    # DFFT_FLAG_NO_OVERLAP on the IPC transports: one stream, whole-GPU stages, identical bits
    shape, grid = (64, 64, 64), (2, 2)
    _, _, _, y1, z1 = _run(shape, "pencil", grid, "f64", exchange, 4, overlap=True, repeats=1)
    _, _, _, y2, z2 = _run(shape, "pencil", grid, "f64", exchange, 4, overlap=False, repeats=1)
    for a, b in zip(y1 + z1, y2 + z2):
        assert torch.equal(a, b)


def test_sim_graph_capture_replay(oracle_mod):
    """The multi-rank schedule (flag waits for constant values) captured in one CUDA graph and
    replayed on fresh inputs, twice — §8(b): dfft_execute is capturable for every plan."""
    shape, grid, prec = (64, 48, 32), (2, 2), "f64"
    comm, fwd, inv = _sim_plans(shape, "pencil", grid, "c2c_" + prec, "p2p", 2)
    P = comm.nranks
    xs = _fill(fwd, shape, 1)
    ys = [fwd.alloc_out(r) for r in range(P)]
    zs = [inv.alloc_out(r) for r in range(P)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fwd.execute_sim(xs, ys, stream=s)
        inv.execute_sim(ys, zs, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fwd.execute_sim(xs, ys, stream=s)
        inv.execute_sim(ys, zs, stream=s)
    for seed in (7, 8):
        for r, x in enumerate(xs):
            lo, n = fwd.box(0, r)
            inputs.fill_box_cuda(x, seed, shape, lo, n, True)
        for y in ys:
            y.zero_()
        g.replay()
        torch.cuda.synchronize()
        a = oracle_mod.gen_complex(seed, shape)
        A = oracle_mod.fft3d(a, -1)
        assert oracle_mod.rel_l2(_gather(fwd, ys, 1, A), A) <= QUALITY[prec]
        assert oracle_mod.rel_l2(_gather(inv, zs, 1, a), a) <= GATE[prec]


def test_watchdog_releases_a_dead_peer():
    """Rank 1 never executes: rank 0 waits on its flags until the watchdog times out, releases
    the waits (the stream drains, nothing hangs) and fails the plan (DFFT_ERR_PEER)."""
    shape, grid = (32, 24, 16), (1, 2)
    comm, fwd, _ = _sim_plans(shape, "pencil", grid, "c2c_f32", "p2p")
    xs = _fill(fwd, shape, 3)
    ys = [fwd.alloc_out(r) for r in range(2)]
    dfft.set_timeout_ms(1500)
    try:
        t0 = time.time()
        fwd.execute_sim([xs[0], None], [ys[0], None])
        torch.cuda.synchronize()  # returns once the watchdog has released the waits
        assert time.time() - t0 < 60
        deadline = time.time() + 10
        while fwd.status() == 0 and time.time() < deadline:
            time.sleep(0.05)
        assert fwd.status() == 8
        with pytest.raises(dfft.DfftError) as ei:
            fwd.execute_sim(xs, ys)
        assert ei.value.status == 8
    finally:
        dfft.set_timeout_ms(120000)
    fwd.destroy()  # bounded: the released flags let the teardown poll finish


def test_timeline_spans_cover_every_stage():
    # f2 instrumentation: one span per stage launch per rank, inside its execute, on its stream
    shape, grid = (256, 64, 64), (2, 2)  # 128 local x columns = 2 column blocks of 64 -> 2 chunks
    comm, fwd, _ = _sim_plans(shape, "pencil", grid, "c2c_f32", "p2p", 2)
    xs = _fill(fwd, shape, 2)
    ys = [fwd.alloc_out(r) for r in range(4)]
    fwd.execute_sim(xs, ys)
    fwd.set_profiling(True)
    fwd.phase_times(reset=True)
    fwd.execute_sim(xs, ys)
    spans = fwd.timeline()
    assert spans and all(0 <= s["t0_ms"] <= s["t1_ms"] for s in spans)
    per_rank = {}
    for s in spans:
        per_rank.setdefault(s["rank"], []).append(s)
    assert sorted(per_rank) == [0, 1, 2, 3]
    for r, ss in per_rank.items():
        phases = sorted({s["phase"] for s in ss})
        assert phases == ["stage_A", "stage_B", "stage_C"], phases
        assert sum(s["phase"] == "stage_B" for s in ss) == 2  # two chunks of B (B->C pipeline)


# ------------------------------------------------------------------------------ full-size kernels
def _single(oracle_mod, shape, prec, seed):
    comm = dfft.Comm.create(nranks=1, rank=0, device=0)
    fwd = dfft.Plan(comm, shape, "pencil", (1, 1), "c2c_" + prec, dfft.FORWARD)
    inv = dfft.Plan(comm, shape, "pencil", (1, 1), "c2c_" + prec, dfft.INVERSE)
    x = fwd.alloc_in()
    inputs.fill_box_cuda(x, seed, shape, (0, 0, 0), shape, True)
    y, z = fwd.alloc_out(), inv.alloc_out()
    fwd.execute(x, y)
    torch.cuda.synchronize()
    a = oracle_mod.gen_complex(seed, shape, f32=(prec == "f32"))
    A = oracle_mod.fft3d(a, -1)
    ef = oracle_mod.rel_l2(y.cpu().numpy(), A)
    # the inverse alone, on the oracle's spectrum (rounded to the plan precision)
    yt = torch.from_numpy(A.astype(np.complex64 if prec == "f32" else np.complex128)).cuda()
    inv.execute(yt, z)
    torch.cuda.synchronize()
    ei = oracle_mod.rel_l2(z.cpu().numpy(), oracle_mod.fft3d(yt.cpu().numpy().astype(np.complex128), +1))
    return ef, ei


@pytest.mark.parametrize("shape,prec", [
    ((16, 1024, 1024), "f32"),   # the bench's radix-32 TMA strided kernel at n = 1024, both 1-GPU orders
    ((16, 512, 768), "f32"),     # n = 768 (3·256) along y, 512 along z
    ((16, 768, 512), "f32"),
    ((8, 1024, 1024), "f64"),    # fp64 strided n = 1024 (radix 16)
])
def test_full_length_strided_kernels_elementwise(oracle_mod, shape, prec):
    ef, ei = _single(oracle_mod, shape, prec, seed=31)
    assert ef <= GATE[prec] and ei <= GATE[prec], (ef, ei)
    assert ef <= QUALITY[prec] and ei <= QUALITY[prec], (ef, ei)


def test_full_length_2x4_fused_store_elementwise(oracle_mod):
    """The 8-GPU headline's 2x4 fused-store layouts at full axis length 1024 (bulk-copy epilogue
    into the column-blocked windows, 4D TMA loads), element-wise vs the oracle, 4 B->C chunks."""
    shape, grid = (64, 1024, 1024), (2, 4)
    fwd, inv, xs, ys, zs = _run(shape, "pencil", grid, "f32", "p2p", chunks=4, seed=41, repeats=1)
    a = oracle_mod.gen_complex(41, shape, f32=True)
    A = oracle_mod.fft3d(a, -1)
    ef = oracle_mod.rel_l2(_gather(fwd, ys, 1, A), A)
    er = oracle_mod.rel_l2(_gather(inv, zs, 1, a), a)
    assert ef <= QUALITY["f32"] and er <= GATE["f32"], (ef, er)


# ------------------------------------------------------------------------------ host-buffer entry points
def test_execute_host_and_chain(oracle_mod):
    """dfft_execute_host (pageable numpy in/out) and dfft_execute_host_chain (fwd -> inv, pinned,
    asynchronous, several calls in flight on the double-buffered staging) vs the oracle."""
    shape, seed = (64, 48, 32), 17
    comm = dfft.Comm.create(nranks=1, rank=0, device=0)
    fwd = dfft.Plan(comm, shape, "pencil", (1, 1), "c2c_f64", dfft.FORWARD)
    inv = dfft.Plan(comm, shape, "pencil", (1, 1), "c2c_f64", dfft.INVERSE)
    a = oracle_mod.gen_complex(seed, shape)
    y = np.empty_like(a)
    fwd.execute_host(np.ascontiguousarray(a), y)
    assert oracle_mod.rel_l2(y, oracle_mod.fft3d(a, -1)) <= QUALITY["f64"]
    xs = [torch.from_numpy(oracle_mod.gen_complex(seed + q, shape)).pin_memory() for q in range(3)]
    zs = [torch.empty_like(x).pin_memory() for x in xs]
    for x, z in zip(xs, zs):
        dfft.execute_host_chain([fwd, inv], x, z, async_=True)
    torch.cuda.synchronize()
    for x, z in zip(xs, zs):
        assert oracle_mod.rel_l2(z.numpy(), x.numpy()) <= GATE["f64"]
    with pytest.raises(dfft.DfftError):  # asynchronous calls need pinned host memory
        dfft.execute_host_chain([fwd, inv], np.ascontiguousarray(a), np.empty_like(a), async_=True)


def test_kernel_launch_counter_counts_graph_replays():
    # dfft_kernel_launches credits each replay of a plan's internal graph with the kernels it holds
    comm = dfft.Comm.create(nranks=1, rank=0, device=0)
    shape = (64, 48, 64)
    fwd = dfft.Plan(comm, shape, "pencil", (1, 1), "c2c_f32", dfft.FORWARD)
    x = fwd.alloc_in()
    y = fwd.alloc_out()
    x.normal_()
    deltas = []
    for _ in range(4):
        n0 = dfft.kernel_launches()
        fwd.execute(x, y)
        deltas.append(dfft.kernel_launches() - n0)
    torch.cuda.synchronize()
    assert deltas == [3] * 4, deltas  # three FFT stages per execute, captured or replayed


@pytest.mark.parametrize("grid,x_maxr", [((1, 2), 32), ((2, 2), 16)])
def test_x_radix_by_plan(oracle_mod, grid, x_maxr):
    # fp32 x-lines of 512: radix-32 passes unless the plan's T1 exchange has remote peers (P1 > 1),
    # whose x-FFTs keep radix 16; both are checked against the oracle
    shape = (512, 16, 8)
    fwd, inv, xs, ys, zs = _run(shape, "pencil", grid, "f32", "p2p", 2)
    fx = [d for d in fwd.describe() if d["phase"] == "stage_A"]
    ix = [d for d in inv.describe() if d["phase"] == "stage_C"]
    assert all(d["family"] == "contig" and d["n"] == 512 and d["maxr"] == x_maxr for d in fx + ix), (fx, ix)
    a = oracle_mod.gen_complex(5, shape, f32=True)
    A = oracle_mod.fft3d(a, -1)
    ef = oracle_mod.rel_l2(_gather(fwd, ys, 1, A), A)
    er = oracle_mod.rel_l2(_gather(inv, zs, 1, a), a)
    assert ef <= QUALITY["f32"] and er <= GATE["f32"], (ef, er)


def _sim_sweep_cases(count=12, seed=2602):
    """Seeded (shape, grid, chunks, transport) cases for the simulated product executor: lengths
    from the specialised set, 2-8 ranks, 1-4 chunks; a grid that does not fit the shape is skipped
    by plan creation (DFFT_ERR_INVALID_VALUE / UNSUPPORTED)."""
    from helpers import LENGTHS
    rng = np.random.default_rng(seed)
    grids = [(1, 2), (2, 1), (2, 2), (1, 4), (4, 1), (2, 4), (4, 2), (1, 8)]
    lens = [n for n in LENGTHS if n >= 8]
    out = []
    while len(out) < count:
        s = tuple(int(v) for v in rng.choice(lens, 3))
        if not (1 << 12) <= s[0] * s[1] * s[2] <= (1 << 20):
            continue
        g = grids[int(rng.integers(len(grids)))]
        out.append((s, g, int(rng.integers(1, 5)), ["p2p", "ce"][int(rng.integers(2))]))
    return out


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("shape,grid,chunks,exchange", _sim_sweep_cases())
def test_sim_product_executor_seeded_sweep(oracle_mod, shape, grid, chunks, exchange, prec):
    try:
        fwd, inv, xs, ys, zs = _run(shape, "pencil", grid, prec, exchange, chunks)
    except dfft.DfftError as e:
        if e.status in (1, 3):  # the grid does not divide / fit this shape
            pytest.skip(str(e))
        raise
    a = oracle_mod.gen_complex(5, shape, f32=(prec == "f32"))
    A = oracle_mod.fft3d(a, -1)
    Y = _gather(fwd, ys, 1, A)
    ef, er = oracle_mod.rel_l2(Y, A), oracle_mod.rel_l2(_gather(inv, zs, 1, a), a)
    assert ef <= GATE[prec] and er <= GATE[prec], (ef, er)
    _, fwd_n, _ = _sim_plans(shape, "pencil", grid, "c2c_" + prec, "nccl", chunks)
    ys_n = [fwd_n.alloc_out(r) for r in range(len(xs))]
    fwd_n.execute_sim(xs, ys_n)
    torch.cuda.synchronize()
    assert np.array_equal(Y, _gather(fwd_n, ys_n, 1, A))
