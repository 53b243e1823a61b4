"""Pins for the CPU oracle (``oracle/``) — things other than the oracle itself fix its values.

PAPER.md prints no worked numeric example, so the pins are: closed forms
(tests/golden/), brute-force O(N^2) sums on tiny inputs, an independent library (numpy's
pocketfft), and invariants (Parseval, round trip, linearity, Hermitian symmetry).  Each is
chosen so that a plausible oracle bug (dropped term, wrong sign, transposed axis, wrong
twiddle index, missing 1/N) fails at least one of them.
"""
import os

import numpy as np
import scipy.fft as sf
import pytest

import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _parse_vec(s):
    out = []
    for pair in s.split(";"):
        re, im = pair.split(",")
        out.append(complex(float(re), float(im)))
    return np.array(out)


def _golden_1d():
    rows = []
    with open(os.path.join(GOLDEN, "closed_forms_1d.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            name, x, X = [t.strip() for t in line.split("|")]
            rows.append((name, _parse_vec(x), _parse_vec(X)))
    return rows


# --------------------------------------------------------------------- generator

def test_splitmix64_known_value():
    # splitmix64 (Steele, Lea, Flood 2014) seeded with 0 emits 0xE220A8397B1DCDAF first;
    # our mixer applied to state 0 is exactly that first output.
    z = inputs._splitmix64(np.array([0], dtype=np.uint64))[0]
    assert int(z) == 0xE220A8397B1DCDAF


def test_generator_oracle_matches_numpy_bits(oracle_mod):
    g = (12, 10, 6)
    lo, n = (3, 2, 1), (7, 5, 4)
    for f32 in (False, True):
        a = oracle_mod.gen_complex(77, g, lo, n, f32=f32)
        b = inputs.gen_complex_np(77, g, lo, n, f32=f32).astype(np.complex128)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
        r1 = oracle_mod.gen_real(77, g, lo, n, f32=f32)
        r2 = inputs.gen_real_np(77, g, lo, n, f32=f32).astype(np.float64)
        assert np.array_equal(r1, r2)
    a = oracle_mod.gen_complex(5, (64, 64, 64))
    assert a.real.min() >= -1 and a.real.max() < 1
    assert abs(a.real.mean()) < 0.01 and abs(a.imag.var() - 1 / 3) < 0.01


# --------------------------------------------------------------------- 1D

@pytest.mark.parametrize("row", _golden_1d(), ids=lambda r: r[0])
def test_1d_closed_forms(oracle_mod, row):
    _, x, X = row
    np.testing.assert_allclose(oracle_mod.dft1d_naive(x), X, atol=1e-14)
    np.testing.assert_allclose(oracle_mod.fft1d(x), X, atol=1e-14)
    # inverse kernel (sign +1, unscaled) maps X back to n*x
    np.testing.assert_allclose(oracle_mod.fft1d(X, +1), len(x) * x, atol=1e-13)


LENGTHS = list(range(1, 33)) + [48, 64, 96, 97, 128, 192, 256, 384, 512, 768, 1024]


@pytest.mark.parametrize("n", LENGTHS)
def test_1d_fast_vs_bruteforce_and_numpy(oracle_mod, n):
    rng = np.random.default_rng(n)
    x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    naive = oracle_mod.dft1d_naive(x)
    fast = oracle_mod.fft1d(x)
    ref = np.fft.fft(x)  # independent library (pocketfft)
    scale = np.sqrt(n)
    assert np.abs(naive - ref).max() < 1e-13 * scale * max(1, np.log2(n))
    assert np.abs(fast - naive).max() < 1e-13 * scale * max(1, np.log2(n))
    inv = oracle_mod.fft1d(fast, +1) / n
    assert np.abs(inv - x).max() < 1e-14 * max(1, np.log2(n))


@pytest.mark.parametrize("n", [5, 16, 24, 1024])
def test_1d_plane_wave_every_bin(oracle_mod, n):
    # exp(+2 pi i m t / n) -> n at k = m, 0 elsewhere: a misplaced bin is an O(1) error
    t = np.arange(n)
    for m in sorted({0, 1, n // 3, n - 1}):
        x = np.exp(2j * np.pi * ((m * t) % n) / n)  # exact phase reduction
        X = oracle_mod.fft1d(x)
        e = np.zeros(n, complex)
        e[m] = n
        assert np.abs(X - e).max() < 1e-11


# --------------------------------------------------------------------- 3D vs brute force

@pytest.mark.parametrize("shape", [(2, 2, 2), (4, 4, 4), (8, 8, 8), (16, 8, 4), (4, 6, 12), (8, 5, 3), (7, 3, 2)])
def test_3d_fast_vs_triple_sum(oracle_mod, shape):
    nx, ny, nz = shape
    a = oracle_mod.gen_complex(11, shape)
    naive = oracle_mod.dft3d_naive(a)
    fast = oracle_mod.fft3d(a, -1)
    assert oracle_mod.rel_l2(fast, naive) < 1e-14
    inv_naive = oracle_mod.dft3d_naive(naive, +1) / a.size
    inv_fast = oracle_mod.fft3d(fast, +1)
    assert oracle_mod.rel_l2(inv_fast, inv_naive) < 1e-14
    assert oracle_mod.rel_l2(inv_fast, a) < 1e-14


def test_3d_axis_order_non_cubic(oracle_mod):
    # a transposed-axis bug passes on cubes; a plane wave with distinct (mx,my,mz) on a
    # non-cubic grid lands on exactly one bin
    nx, ny, nz = 12, 8, 6
    mx, my, mz = 5, 3, 1
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    a = np.exp(2j * np.pi * ((mx * x) % nx / nx + (my * y) % ny / ny + (mz * z) % nz / nz))
    X = oracle_mod.fft3d(a, -1)
    e = np.zeros_like(X)
    e[mz, my, mx] = a.size
    assert np.abs(X - e).max() < 1e-10


# --------------------------------------------------------------------- closed forms at config sizes

@pytest.mark.parametrize("shape", [(64, 64, 64), (96, 64, 48)])
def test_3d_closed_forms(oracle_mod, shape):
    nx, ny, nz = shape
    N = nx * ny * nz
    # delta at origin -> all ones
    a = np.zeros((nz, ny, nx), complex)
    a[0, 0, 0] = 1
    assert np.abs(oracle_mod.fft3d(a) - 1).max() < 1e-13
    # delta at (ax, ay, az) -> pure phase exp(-2 pi i (kx ax/nx + ky ay/ny + kz az/nz))
    ax, ay, az = 3, 5, 7
    a = np.zeros((nz, ny, nx), complex)
    a[az, ay, ax] = 1
    kz, ky, kx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ph = np.exp(-2j * np.pi * ((kx * ax) % nx / nx + (ky * ay) % ny / ny + (kz * az) % nz / nz))
    assert np.abs(oracle_mod.fft3d(a) - ph).max() < 1e-12
    # constant c -> c*N at DC only
    c = 0.25 - 0.5j
    X = oracle_mod.fft3d(np.full((nz, ny, nx), c))
    assert abs(X[0, 0, 0] - c * N) < 1e-9
    X[0, 0, 0] = 0
    assert np.abs(X).max() < 1e-9
    # inverse of all-ones -> delta (the 1/N is applied)
    d = oracle_mod.fft3d(np.ones((nz, ny, nx), complex), +1)
    e = np.zeros_like(d)
    e[0, 0, 0] = 1
    assert np.abs(d - e).max() < 1e-14


def test_3d_invariants_and_numpy(oracle_mod):
    shape = (64, 32, 48)
    a = oracle_mod.gen_complex(3, shape)
    b = oracle_mod.gen_complex(4, shape)
    A = oracle_mod.fft3d(a)
    B = oracle_mod.fft3d(b)
    N = a.size
    # Parseval: sum |X|^2 = N sum |x|^2
    assert abs(np.vdot(A, A).real / (N * np.vdot(a, a).real) - 1) < 1e-13
    # linearity
    alpha, beta = 0.7 - 0.2j, -1.3 + 0.4j
    assert oracle_mod.rel_l2(oracle_mod.fft3d(alpha * a + beta * b), alpha * A + beta * B) < 1e-14
    # round trip
    assert oracle_mod.rel_l2(oracle_mod.fft3d(A, +1), a) < 1e-15
    # independent library: numpy axes (z, y, x) == our (nz, ny, nx) storage
    assert oracle_mod.rel_l2(A, np.fft.fftn(a)) < 1e-14
    assert oracle_mod.rel_l2(oracle_mod.fft3d(a, +1), np.fft.ifftn(a)) < 1e-14


# --------------------------------------------------------------------- R2C / C2R

def test_r2c_relations(oracle_mod):
    nx, ny, nz = 12, 8, 6
    r = oracle_mod.gen_real(9, (nx, ny, nz))
    H = oracle_mod.rfft3d(r)
    assert H.shape == (nz, ny, nx // 2 + 1)
    full = oracle_mod.fft3d(r.astype(complex))
    assert oracle_mod.rel_l2(H, full[:, :, : nx // 2 + 1]) < 1e-15
    # Hermitian symmetry of the spectrum of a real input
    sym = np.conj(full[(-np.arange(nz)) % nz][:, (-np.arange(ny)) % ny][:, :, (-np.arange(nx)) % nx])
    assert oracle_mod.rel_l2(full, sym) < 1e-14
    assert oracle_mod.rel_l2(H, np.fft.rfftn(r)) < 1e-14
    assert oracle_mod.rel_l2(oracle_mod.irfft3d(H, nx), r) < 1e-15


def test_c2r_arbitrary_input_matches_numpy(oracle_mod):
    # reading R8: C2R on arbitrary (non-Hermitian) input = numpy irfftn convention
    nx, ny, nz = 10, 8, 6
    rng = np.random.default_rng(0)
    h = rng.standard_normal((nz, ny, nx // 2 + 1)) + 1j * rng.standard_normal((nz, ny, nx // 2 + 1))
    ref = np.fft.irfftn(h, s=(nz, ny, nx), axes=(0, 1, 2))
    assert np.abs(oracle_mod.irfft3d(h, nx) - ref).max() < 1e-15


# --------------------------------------------------------------------- sampled bins

def test_sampled_bins_match_full_transform(oracle_mod):
    for shape, real in (((16, 12, 8), False), ((64, 64, 64), False), ((24, 16, 12), True)):
        a = oracle_mod.gen_real(21, shape) if real else oracle_mod.gen_complex(21, shape)
        X = oracle_mod.rfft3d(a) if real else oracle_mod.fft3d(a)
        rng = np.random.default_rng(1)
        for _ in range(6):
            kx = int(rng.integers(0, X.shape[2]))
            ky, kz = int(rng.integers(0, shape[1])), int(rng.integers(0, shape[2]))
            v = oracle_mod.dft3d_bin_seeded(21, shape, (kx, ky, kz), real_input=real)
            assert abs(v - X[kz, ky, kx]) < 1e-10 * np.sqrt(a.size)


def test_err_sums(oracle_mod):
    y = np.array([1 + 1j, 2, 3j])
    ref = np.array([1, 2 + 1j, 3j])
    e, r = oracle_mod.err_sums(y, ref)
    assert e == pytest.approx(2.0) and r == pytest.approx(1 + 5 + 9)


# ------------------------------------------------------------------ periodic Poisson solve (f3)
def _lap_np(phi, h):
    """The 7-point periodic Laplacian written with numpy rolls (independent of the oracle's C)."""
    hx, hy, hz = h
    out = (np.roll(phi, 1, 2) - 2 * phi + np.roll(phi, -1, 2)) / hx**2
    out += (np.roll(phi, 1, 1) - 2 * phi + np.roll(phi, -1, 1)) / hy**2
    out += (np.roll(phi, 1, 0) - 2 * phi + np.roll(phi, -1, 0)) / hz**2
    return out


@pytest.mark.parametrize("shape,h", [((8, 6, 4), (1.0, 1.0, 1.0)), ((16, 12, 10), (0.5, 2.0, 1.5)),
                                     ((48, 24, 12), (1.0, 0.25, 3.0))])
def test_poisson_inverts_the_discrete_laplacian(oracle_mod, shape, h):
    # P:606-620 (§VI-B) solves the pressure Poisson equation; reading R20: 7-point Laplacian,
    # zero-mean solution.  Pin: applying the operator (numpy, not the oracle) gives back f - mean(f).
    nx, ny, nz = shape
    f = oracle_mod.gen_real(31, shape)
    phi = oracle_mod.poisson3d(f, h)
    assert abs(phi.mean()) < 1e-12
    r = _lap_np(phi, h) - (f - f.mean())
    assert np.abs(r).max() <= 1e-11 * np.abs(f).max() * max(1.0, max(1 / v**2 for v in h))
    assert np.allclose(oracle_mod.laplacian7(phi, h), _lap_np(phi, h), rtol=0, atol=1e-12)


def test_poisson_single_mode_closed_form(oracle_mod):
    # f = cos(2π(mx x/nx + my y/ny + mz z/nz)) is an eigenfunction of the 7-point Laplacian with
    # eigenvalue -Σ (2 sin(π m_d/n_d)/h_d)² (textbook), so φ = f / λ exactly.
    nx, ny, nz, h = 24, 16, 12, (1.0, 0.5, 2.0)
    m = (5, 3, 7)
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    f = np.cos(2 * np.pi * (m[0] * x / nx + m[1] * y / ny + m[2] * z / nz))
    lam = -sum((2 * np.sin(np.pi * md / nd) / hd) ** 2 for md, nd, hd in zip(m, (nx, ny, nz), h))
    phi = oracle_mod.poisson3d(f, h)
    assert np.abs(phi - f / lam).max() < 1e-13
    lx = oracle_mod.poisson_eigen(nx, 0.5)
    assert lx[0] == 0.0 and abs(lx[nx // 2] + 16.0) < 1e-13  # -(2/h)^2 at the Nyquist mode


# ------------------------------------------------------------------ R2R: DCT-II / DCT-III (f4)
@pytest.mark.parametrize("shape", [(8, 6, 4), (16, 12, 10), (32, 8, 24)])
def test_dct3d_vs_scipy(oracle_mod, shape):
    # P:403 (R2R), reading R21: DCT-II per axis = scipy.fft.dctn(type=2) (pocketfft, an
    # independent library), inverse = DCT-III/(2N) per axis = scipy.fft.idctn(type=2)
    import scipy.fft as sf
    a = oracle_mod.gen_real(41, shape)
    X = oracle_mod.dct3d(a)
    assert np.allclose(X, sf.dctn(a, type=2), rtol=0, atol=1e-12 * np.abs(X).max())
    assert np.allclose(oracle_mod.dct3d(X, inverse=True), a, rtol=0, atol=1e-13)
    assert np.allclose(oracle_mod.dct3d(X, inverse=True), sf.idctn(X, type=2), rtol=0, atol=1e-13)


def test_dct3d_closed_forms(oracle_mod):
    # cos(π m (2n+1) / (2N)) along each axis is a DCT-II basis vector: X = 8·Nx·Ny·Nz/8 at (mx,my,mz)
    # for m > 0 (orthogonality, textbook); a constant c gives 8·N·c at DC only
    nx, ny, nz = 12, 8, 6
    m = (5, 3, 1)
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    f = (np.cos(np.pi * m[0] * (2 * x + 1) / (2 * nx)) * np.cos(np.pi * m[1] * (2 * y + 1) / (2 * ny))
         * np.cos(np.pi * m[2] * (2 * z + 1) / (2 * nz)))
    X = oracle_mod.dct3d(f)
    ref = np.zeros_like(X)
    ref[m[2], m[1], m[0]] = nx * ny * nz
    assert np.abs(X - ref).max() < 1e-11
    C = oracle_mod.dct3d(np.full((nz, ny, nx), 0.5))
    ref = np.zeros_like(C)
    ref[0, 0, 0] = 8 * nx * ny * nz * 0.5
    assert np.abs(C - ref).max() < 1e-11


# ------------------------------------------------------------------ per-axis kinds: DST, mixed topologies (f4)
@pytest.mark.parametrize("kind,fwd,inv", [
    ("dct", lambda a, ax: sf.dct(a, 2, axis=ax), lambda a, ax: sf.idct(a, 2, axis=ax)),
    ("dst", lambda a, ax: sf.dst(a, 2, axis=ax), lambda a, ax: sf.idst(a, 2, axis=ax)),
    ("dft", lambda a, ax: sf.fft(a, axis=ax), lambda a, ax: sf.ifft(a, axis=ax)),
])
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_axis_transform_vs_scipy(oracle_mod, kind, fwd, inv, axis):
    # P:409 "DCT and DST" (reading R22: FFTW REDFT10/RODFT10 forward, REDFT01/RODFT01 ÷ 2N inverse)
    # = scipy.fft dct/dst type 2 with norm=None and their idct/idst (pocketfft, independent code);
    # on complex data the real and imaginary parts are transformed alike
    rng = np.random.default_rng(axis)
    a = rng.standard_normal((6, 10, 8)) + 1j * rng.standard_normal((6, 10, 8))
    ax = 2 - axis  # numpy axis of x / y / z in a (nz, ny, nx) array
    Y = oracle_mod.axis_transform(a, axis, kind)
    ref = fwd(a, ax) if kind == "dft" else fwd(a.real, ax) + 1j * fwd(a.imag, ax)
    assert np.abs(Y - ref).max() <= 1e-13 * np.abs(ref).max()
    back = oracle_mod.axis_transform(Y, axis, kind, inverse=True)
    ref_b = inv(Y, ax) if kind == "dft" else inv(Y.real, ax) + 1j * inv(Y.imag, ax)
    assert np.abs(back - ref_b).max() <= 1e-13 and np.abs(back - a).max() <= 1e-13


def test_dst_closed_forms(oracle_mod):
    # textbook: the DST-II basis vector sin(π(m+1)(2n+1)/(2N)) maps to N at k = m only (orthogonality;
    # 2N for m = N-1, whose vector is (-1)^n), and RODFT01 of a spike 2N at k = N-1 is (-1)^n
    N = 12
    n = np.arange(N)
    for m in (0, 3, N - 1):
        v = np.sin(np.pi * (m + 1) * (2 * n + 1) / (2 * N)).reshape(1, 1, N)
        Y = oracle_mod.axis_transform(v, 0, "dst").real.ravel()
        e = np.zeros(N)
        e[m] = N if m < N - 1 else 2 * N
        assert np.abs(Y - e).max() < 1e-12
    s = np.zeros((1, 1, N))
    s[0, 0, N - 1] = 2 * N
    assert np.abs(oracle_mod.axis_transform(s, 0, "dst", inverse=True).real.ravel() - (-1.0) ** n).max() < 1e-13


def test_rfft_irfft_x_vs_numpy(oracle_mod):
    rng = np.random.default_rng(5)
    f = rng.standard_normal((4, 6, 10))
    H = oracle_mod.rfft_x(f)
    assert np.abs(H - np.fft.rfft(f, axis=2)).max() < 1e-13
    G = rng.standard_normal(H.shape) + 1j * rng.standard_normal(H.shape)  # arbitrary (non-Hermitian)
    assert np.abs(oracle_mod.irfft_x(G, 10) - np.fft.irfft(G, 10, axis=2)).max() < 1e-13


@pytest.mark.parametrize("kinds", [("dft", "dft", "dct"), ("dft", "dst", "dft"), ("dft", "dct", "dst"),
                                   ("dct", "dst", "dct"), ("dst", "dst", "dst")])
def test_mixed_kinds_vs_scipy_axis_by_axis(oracle_mod, kinds):
    # P:620's (Periodic, Periodic, Bounded) topology and its relatives: the separable transform is
    # each axis's 1D transform in turn, composed here with scipy along each axis
    nx, ny, nz = 12, 8, 6
    f = oracle_mod.gen_real(7, (nx, ny, nz))
    real_x = kinds[0] == "dft"
    ref = np.fft.rfft(f, axis=2) if real_x else (sf.dct if kinds[0] == "dct" else sf.dst)(f, 2, axis=2) + 0j
    for k, ax in ((kinds[1], 1), (kinds[2], 0)):
        if k == "dft":
            ref = np.fft.fft(ref, axis=ax)
        else:
            t = sf.dct if k == "dct" else sf.dst
            ref = t(ref.real, 2, axis=ax) + 1j * t(ref.imag, 2, axis=ax)
    X = oracle_mod.transform_kinds(f if real_x else f + 0j, kinds, real_x=real_x)
    assert np.abs(X - ref).max() <= 1e-12 * np.abs(ref).max()
    back = oracle_mod.transform_kinds(X, kinds, inverse=True, real_x=real_x, nx=nx)
    assert np.abs(np.real(back) - f).max() <= 1e-13


def _lap_bc(phi, h, kinds):
    """3-point second differences per axis with the boundary each kind encodes (numpy, independent
    of the oracle): periodic wrap (DFT), cell-centred mirror ghost φ_{-1} = φ_0 (Neumann, DCT-II),
    antimirror ghost φ_{-1} = -φ_0 (Dirichlet, DST-II)."""
    out = np.zeros_like(phi)
    for d, (k, hd) in enumerate(zip(kinds, h)):
        ax = 2 - d
        if k == "dft":
            lo, hi = np.roll(phi, 1, ax), np.roll(phi, -1, ax)
        else:
            s = 1.0 if k == "dct" else -1.0
            first = np.take(phi, [0], axis=ax)
            last = np.take(phi, [phi.shape[ax] - 1], axis=ax)
            lo = np.concatenate([s * first, np.take(phi, range(phi.shape[ax] - 1), axis=ax)], axis=ax)
            hi = np.concatenate([np.take(phi, range(1, phi.shape[ax]), axis=ax), s * last], axis=ax)
        out += (lo - 2 * phi + hi) / hd**2
    return out


@pytest.mark.parametrize("kinds,h", [(("dft", "dft", "dct"), (1.0, 0.5, 2.0)), (("dft", "dft", "dst"), (1.0, 1.0, 1.0)),
                                     (("dct", "dct", "dct"), (1.0, 2.0, 0.5)), (("dst", "dct", "dst"), (0.5, 1.0, 1.0)),
                                     (("dft", "dst", "dct"), (2.0, 1.0, 0.25))])
def test_poisson_kinds_inverts_the_bounded_laplacian(oracle_mod, kinds, h):
    # P:606-620 with P:620's bounded directions (readings R20, R22): applying the 7-point operator
    # with each axis's boundary (numpy) to φ gives back f, minus its mean when no axis is Dirichlet
    # (the operator is then singular on constants and the solver returns the zero-mean solution)
    shape = (12, 8, 10)
    f = oracle_mod.gen_real(13, shape)
    phi = oracle_mod.poisson_kinds(f, kinds, h)
    target = f - f.mean() if "dst" not in kinds else f
    r = _lap_bc(phi, h, kinds) - target
    assert np.abs(r).max() <= 1e-11 * np.abs(f).max() * max(1.0, max(1 / v**2 for v in h))
    if kinds == ("dft", "dft", "dft"):
        assert np.abs(phi - oracle_mod.poisson3d(f, h)).max() < 1e-12
