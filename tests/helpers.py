"""Shared test helpers: box slicing of global arrays (numpy, (nz, ny, nx) order) and tolerances."""
import numpy as np

# BASELINE.json north_star gates (relative L2 vs the fp64 oracle)
GATE = {"f32": 2e-5, "f64": 1e-12}
# tighter diagnostic bounds (a well-implemented FFT sits near 2e-7 / 3e-16)
QUALITY = {"f32": 1e-6, "f64": 1e-14}

# lengths instantiated in libdfft.so (csrc/registry.h DFFT_LENGTHS)
LENGTHS = [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096,
           3, 6, 12, 24, 48, 96, 192, 384, 768, 1536, 3072, 5, 7, 480, 720, 840]


def box_slice(arr, lo, n):
    """View of the (nz, ny, nx)-ordered global array for box (lo, n) given in x,y,z order."""
    return arr[lo[2]:lo[2] + n[2], lo[1]:lo[1] + n[1], lo[0]:lo[0] + n[0]]


def rel_l2(y, ref):
    y = np.asarray(y, dtype=np.complex128)
    ref = np.asarray(ref, dtype=np.complex128)
    return float(np.sqrt(np.sum(np.abs(y - ref) ** 2) / np.sum(np.abs(ref) ** 2)))
