"""CPU oracle for the distributed 3D FFT — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2601_12209_b200``) never imports it and shares no code with it.

Thin ctypes wrapper over ``oracle/dfft_oracle.c`` (plain C + OpenMP, fp64).  Every function
cites the PAPER.md passage it follows in the C source; see also DESIGN.md §3.
Arrays are numpy, x fastest: a complex box of extents (nx, ny, nz) is ``shape (nz, ny, nx)``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dfft_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_int = ctypes.c_int
_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -fopenmp, no -ffast-math, no SIMD intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.or_gen_complex_box.argtypes = [_u64, _i64, _i64, _i64, _i64p, _i64p, _int, _dp]
        lib.or_gen_real_box.argtypes = [_u64, _i64, _i64, _i64, _i64p, _i64p, _int, _dp]
        lib.or_dft1d_naive.argtypes = [_dp, _i64, _int, _dp]
        lib.or_fft1d.argtypes = [_dp, _i64, _int]
        lib.or_fft3d.argtypes = [_dp, _i64, _i64, _i64, _int]
        lib.or_dft3d_naive.argtypes = [_dp, _i64, _i64, _i64, _int, _dp]
        lib.or_rfft3d.argtypes = [_dp, _i64, _i64, _i64, _dp]
        lib.or_irfft3d.argtypes = [_dp, _i64, _i64, _i64, _dp]
        _d = ctypes.c_double
        lib.or_poisson_eigen.argtypes = [_i64, _d, _dp]
        lib.or_poisson3d.argtypes = [_dp, _i64, _i64, _i64, _d, _d, _d, _dp]
        lib.or_laplacian7.argtypes = [_dp, _i64, _i64, _i64, _d, _d, _d, _dp]
        lib.or_dct3d.argtypes = [_dp, _i64, _i64, _i64, _int]
        lib.or_axis_transform.argtypes = [_dp, _i64, _i64, _i64, _int, _int, _int]
        lib.or_rfft_x.argtypes = [_dp, _i64, _i64, _i64, _dp]
        lib.or_irfft_x.argtypes = [_dp, _i64, _i64, _i64, _dp]
        lib.or_poisson_eigen_kind.argtypes = [_i64, ctypes.c_double, _int, _dp]
        lib.or_set_threads.argtypes = [_int]
        lib.or_dft3d_bin_seeded.argtypes = [_u64, _i64, _i64, _i64, _int, _int, _i64, _i64, _i64, _dp]
        lib.or_err_sums.argtypes = [_dp, _dp, _i64, _dp]
        lib.or_num_threads.restype = _int
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _i3(v):
    return (ctypes.c_int64 * 3)(*[int(t) for t in v])


def num_threads() -> int:
    return int(_load().or_num_threads())


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle (timing legs use every host core; torchrun sets 1 per rank)."""
    _load().or_set_threads(int(n))


# ----------------------------------------------------------------- generator

def gen_complex(seed: int, gshape, lo=(0, 0, 0), n=None, f32: bool = False) -> np.ndarray:
    """Box [lo, lo+n) of the seeded global complex input (x,y,z order), as complex128 (nz,ny,nx)."""
    gnx, gny, gnz = gshape
    n = n or (gnx, gny, gnz)
    out = np.empty((n[2], n[1], n[0]), dtype=np.complex128)
    _load().or_gen_complex_box(seed, gnx, gny, gnz, _i3(lo), _i3(n), int(f32), _p(out.view(np.float64)))
    return out


def gen_real(seed: int, gshape, lo=(0, 0, 0), n=None, f32: bool = False) -> np.ndarray:
    gnx, gny, gnz = gshape
    n = n or (gnx, gny, gnz)
    out = np.empty((n[2], n[1], n[0]), dtype=np.float64)
    _load().or_gen_real_box(seed, gnx, gny, gnz, _i3(lo), _i3(n), int(f32), _p(out))
    return out


# ----------------------------------------------------------------- transforms

def dft1d_naive(x: np.ndarray, sign: int = -1) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.complex128)
    X = np.empty_like(x)
    _load().or_dft1d_naive(_p(x.view(np.float64)), x.size, sign, _p(X.view(np.float64)))
    return X


def fft1d(x: np.ndarray, sign: int = -1) -> np.ndarray:
    a = np.array(x, dtype=np.complex128, copy=True, order="C")
    _load().or_fft1d(_p(a.view(np.float64)), a.size, sign)
    return a


def fft3d(a: np.ndarray, sign: int = -1) -> np.ndarray:
    """Forward (sign -1, unscaled) or inverse (sign +1, ×1/N) 3D FFT of a (nz,ny,nx) array."""
    a = np.array(a, dtype=np.complex128, copy=True, order="C")
    nz, ny, nx = a.shape
    _load().or_fft3d(_p(a.view(np.float64)), nx, ny, nz, sign)
    return a


def fft3d_inplace(a: np.ndarray, sign: int = -1) -> np.ndarray:
    assert a.dtype == np.complex128 and a.flags.c_contiguous
    nz, ny, nx = a.shape
    _load().or_fft3d(_p(a.view(np.float64)), nx, ny, nz, sign)
    return a


def dft3d_naive(a: np.ndarray, sign: int = -1) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.complex128)
    nz, ny, nx = a.shape
    if a.size > 4096:
        raise ValueError("dft3d_naive is O(N^2); refusing N > 4096 (16^3)")
    out = np.empty_like(a)
    _load().or_dft3d_naive(_p(a.view(np.float64)), nx, ny, nz, sign, _p(out.view(np.float64)))
    return out


def rfft3d(real: np.ndarray) -> np.ndarray:
    real = np.ascontiguousarray(real, dtype=np.float64)
    nz, ny, nx = real.shape
    out = np.empty((nz, ny, nx // 2 + 1), dtype=np.complex128)
    _load().or_rfft3d(_p(real), nx, ny, nz, _p(out.view(np.float64)))
    return out


def irfft3d(half: np.ndarray, nx: int) -> np.ndarray:
    half = np.ascontiguousarray(half, dtype=np.complex128)
    nz, ny, nxc = half.shape
    assert nxc == nx // 2 + 1 and nx % 2 == 0
    out = np.empty((nz, ny, nx), dtype=np.float64)
    _load().or_irfft3d(_p(half.view(np.float64)), nx, ny, nz, _p(out))
    return out


def dct3d(a: np.ndarray, inverse: bool = False) -> np.ndarray:
    """R2R (reading R21): DCT-II along every axis (FFTW REDFT10), or DCT-III / (2N) per axis."""
    out = np.array(a, dtype=np.float64, order="C", copy=True)
    nz, ny, nx = out.shape
    _load().or_dct3d(_p(out), nx, ny, nz, int(bool(inverse)))
    return out


KINDS = {"dft": 0, "dct": 1, "dst": 2}


def axis_transform(a: np.ndarray, axis: int, kind: str, inverse: bool = False) -> np.ndarray:
    """One axis (0 x, 1 y, 2 z) of a complex (nz,ny,nx) array: DFT (inverse ×1/n), DCT-II /
    DCT-III/(2n), DST-II / DST-III/(2n) of the real and imaginary parts (reading R22)."""
    out = np.array(a, dtype=np.complex128, order="C", copy=True)
    nz, ny, nx = out.shape
    _load().or_axis_transform(_p(out.view(np.float64)), nx, ny, nz, int(axis), KINDS[kind], int(bool(inverse)))
    return out


def rfft_x(f: np.ndarray) -> np.ndarray:
    """R2C along x only: (nz,ny,nx) real -> (nz,ny,nx/2+1) complex."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    nz, ny, nx = f.shape
    out = np.empty((nz, ny, nx // 2 + 1), dtype=np.complex128)
    _load().or_rfft_x(_p(f), nx, ny, nz, _p(out.view(np.float64)))
    return out


def irfft_x(h: np.ndarray, nx: int) -> np.ndarray:
    """C2R along x only (Hermitian extension per line, reading R8)."""
    h = np.ascontiguousarray(h, dtype=np.complex128)
    nz, ny, _ = h.shape
    out = np.empty((nz, ny, nx), dtype=np.float64)
    _load().or_irfft_x(_p(h.view(np.float64)), nx, ny, nz, _p(out))
    return out


def transform_kinds(a: np.ndarray, kinds, inverse: bool = False, real_x: bool = False, nx: int = 0) -> np.ndarray:
    """The 3D transform with per-axis kinds (x, y, z), in the paper's axis order: forward x, y, z;
    inverse z, y, x.  real_x: x is the R2C axis (forward: real input, half
    spectrum out; inverse: half spectrum in, real output of length nx).  R2R plans: real data
    with DCT/DST on every axis (the complex view is only the carrier)."""
    kinds = list(kinds)
    if not inverse:
        if real_x:
            out = rfft_x(a)
        elif kinds[0] == "dft":
            out = axis_transform(a, 0, "dft")
        else:
            out = axis_transform(a, 0, kinds[0])
        for ax in (1, 2):
            out = axis_transform(out, ax, kinds[ax])
        return out
    out = np.asarray(a, dtype=np.complex128)
    for ax in (2, 1):
        out = axis_transform(out, ax, kinds[ax], inverse=True)
    if real_x:
        return irfft_x(out, nx)
    return axis_transform(out, 0, kinds[0], inverse=True)


def poisson_eigen_kind(n: int, h: float, kind: str) -> np.ndarray:
    """λ_k of the 3-point second difference on the basis of the axis's transform kind (R22)."""
    out = np.empty(n)
    _load().or_poisson_eigen_kind(n, float(h), KINDS[kind], _p(out))
    return out


def poisson_kinds(f: np.ndarray, kinds, spacing=(1.0, 1.0, 1.0)) -> np.ndarray:
    """∇²φ = f with per-axis boundary kinds (periodic DFT, Neumann DCT, Dirichlet DST), step by step
    as the solver does it: forward transform (R2C along x if x is periodic), Φ = F/λ(k) with
    λ = Σ_d λ_d(k_d) and Φ = 0 where λ = 0 (the zero-mean solution when no axis is Dirichlet),
    inverse transform (readings R20, R22)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    nz, ny, nx = f.shape
    real_x = kinds[0] == "dft"
    F = transform_kinds(f if real_x else f.astype(np.complex128), kinds, real_x=real_x)
    lam = (poisson_eigen_kind(nx, spacing[0], kinds[0])[: F.shape[2]][None, None, :]
           + poisson_eigen_kind(ny, spacing[1], kinds[1])[None, :, None]
           + poisson_eigen_kind(nz, spacing[2], kinds[2])[:, None, None])
    with np.errstate(divide="ignore", invalid="ignore"):
        Phi = np.where(lam != 0, F / np.where(lam != 0, lam, 1.0), 0)
    out = transform_kinds(Phi, kinds, inverse=True, real_x=real_x, nx=nx)
    return np.real(out).copy() if not real_x else out


def poisson_eigen(n: int, h: float = 1.0) -> np.ndarray:
    """λ_k = -(2 sin(πk/n)/h)², k < n: eigenvalues of the 3-point second difference (reading R20)."""
    out = np.empty(n)
    _load().or_poisson_eigen(n, float(h), _p(out))
    return out


def poisson3d(f: np.ndarray, spacing=(1.0, 1.0, 1.0)) -> np.ndarray:
    """Zero-mean periodic solution of the 7-point discrete Poisson equation (R20)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    nz, ny, nx = f.shape
    out = np.empty_like(f)
    _load().or_poisson3d(_p(f), nx, ny, nz, *[float(h) for h in spacing], _p(out))
    return out


def laplacian7(phi: np.ndarray, spacing=(1.0, 1.0, 1.0)) -> np.ndarray:
    """7-point periodic discrete Laplacian (pins the Poisson solve)."""
    phi = np.ascontiguousarray(phi, dtype=np.float64)
    nz, ny, nx = phi.shape
    out = np.empty_like(phi)
    _load().or_laplacian7(_p(phi), nx, ny, nz, *[float(h) for h in spacing], _p(out))
    return out


def dft3d_bin_seeded(seed: int, gshape, k, f32: bool = False, real_input: bool = False) -> complex:
    """X(kx,ky,kz) of the seeded input by the direct O(N) sum (input regenerated on the fly)."""
    out = np.zeros(2, dtype=np.float64)
    nx, ny, nz = gshape
    _load().or_dft3d_bin_seeded(seed, nx, ny, nz, int(f32), int(real_input), int(k[0]), int(k[1]), int(k[2]), _p(out))
    return complex(out[0], out[1])


def err_sums(y: np.ndarray, ref: np.ndarray):
    """(Σ|y-ref|², Σ|ref|²), Kahan-compensated, over the same-shape arrays."""
    y = np.ascontiguousarray(y)
    ref = np.ascontiguousarray(ref)
    if np.iscomplexobj(y) or np.iscomplexobj(ref):
        y = y.astype(np.complex128).view(np.float64)
        ref = ref.astype(np.complex128).view(np.float64)
    else:
        y = y.astype(np.float64)
        ref = ref.astype(np.float64)
    out = np.zeros(2, dtype=np.float64)
    _load().or_err_sums(_p(y.reshape(-1)), _p(ref.reshape(-1)), y.size, _p(out))
    return float(out[0]), float(out[1])


def rel_l2(y: np.ndarray, ref: np.ndarray) -> float:
    e, r = err_sums(y, ref)
    return (e / r) ** 0.5 if r > 0 else e ** 0.5
