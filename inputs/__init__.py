"""Seeded synthetic inputs shared by tests and bench (holds none of the FFT's arithmetic).

Counter-based generator (DESIGN.md §4 "input recipe"), identical bits on every implementation:
  value(part p, global index g) = U(splitmix64((seed << 32) ^ (2g + p))),
  U(u) = (u >> 11) * 2^-52 - 1  in [-1, 1)  (exact in fp64),  g = x + nx*(y + ny*z),
  p = 0 for the real part, 1 for the imaginary part; fp32 plans round with RN to float.
Implementations: ``gen_complex_np`` / ``gen_real_np`` (numpy, here) and the CUDA kernels
in ``inputs/gen.cu`` (``libdfft_inputs.so``, device-side fill of a rank's box).  The
oracle carries its own C implementation; tests check all three agree bit for bit.

Seeds: config c in BASELINE.json uses seed 260112209 + c (c = 1..5).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

SEED_BASE = 260112209
_HERE = os.path.dirname(os.path.abspath(__file__))

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def _splitmix64(state: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = state + _M1
        z = (z ^ (z >> np.uint64(30))) * _M2
        z = (z ^ (z >> np.uint64(27))) * _M3
        return z ^ (z >> np.uint64(31))


def _uniform(seed: int, g: np.ndarray, part: int) -> np.ndarray:
    state = (np.uint64(seed) << np.uint64(32)) ^ (np.uint64(2) * g.astype(np.uint64) + np.uint64(part))
    return (_splitmix64(state) >> np.uint64(11)).astype(np.float64) * 2.0 ** -52 - 1.0


def _gidx(gshape, lo, n) -> np.ndarray:
    gnx, gny, _ = gshape
    z = np.arange(lo[2], lo[2] + n[2], dtype=np.int64)[:, None, None]
    y = np.arange(lo[1], lo[1] + n[1], dtype=np.int64)[None, :, None]
    x = np.arange(lo[0], lo[0] + n[0], dtype=np.int64)[None, None, :]
    return x + gnx * (y + gny * z)


def gen_complex_np(seed: int, gshape, lo=(0, 0, 0), n=None, f32: bool = False) -> np.ndarray:
    """Box of the seeded complex input, shape (nz, ny, nx); complex64 if f32 else complex128."""
    n = tuple(n or gshape)
    g = _gidx(gshape, lo, n)
    re, im = _uniform(seed, g, 0), _uniform(seed, g, 1)
    if f32:
        out = np.empty(g.shape, dtype=np.complex64)
        out.real, out.imag = re.astype(np.float32), im.astype(np.float32)
        return out
    return re + 1j * im


def gen_real_np(seed: int, gshape, lo=(0, 0, 0), n=None, f32: bool = False) -> np.ndarray:
    n = tuple(n or gshape)
    re = _uniform(seed, _gidx(gshape, lo, n), 0)
    return re.astype(np.float32) if f32 else re


# ---------------------------------------------------------------- device fill (CUDA)

_lib = None


def _load_cuda():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libdfft_inputs.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        lib.dfft_inputs_fill_box.argtypes = [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
            ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        lib.dfft_inputs_fill_box.restype = ctypes.c_int
        _lib = lib
    return _lib


def fill_box_cuda(t, seed: int, gshape, lo, n, complex_: bool, stream=None) -> None:
    """Fill the CUDA torch tensor ``t`` (shape (nz,ny,nx), complex64/128 or float32/64) in place."""
    import torch

    f32 = t.dtype in (torch.complex64, torch.float32)
    assert t.is_cuda and t.is_contiguous() and t.numel() == n[0] * n[1] * n[2]
    s = stream if stream is not None else torch.cuda.current_stream(t.device)
    rc = _load_cuda().dfft_inputs_fill_box(
        ctypes.c_void_p(t.data_ptr()), int(f32), int(complex_), seed,
        gshape[0], gshape[1], gshape[2], lo[0], lo[1], lo[2], n[0], n[1], n[2],
        ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"dfft_inputs_fill_box failed: cuda error {rc}")
