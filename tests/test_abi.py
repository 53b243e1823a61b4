"""CPU checks of the C ABI: the library loads, exports every symbol include/dfft.h declares, and
its host-side logic (validation, geometry) behaves — no GPU needed."""
import ctypes
import os
import re

import pytest

import paper_2601_12209_b200 as dfft

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "dfft.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dfft_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(dfft.LIB_PATH)
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), f"{n} declared in dfft.h but not exported"
    assert sorted(dfft.EXPORTS) == names


def test_inputs_library_exports():
    L = ctypes.CDLL(os.path.join(ROOT, "inputs", "libdfft_inputs.so"))
    assert hasattr(L, "dfft_inputs_fill_box")


def test_version_and_status_strings():
    assert dfft.version() == 100
    L = dfft.lib()
    assert L.dfft_status_string(0) == b"success"
    assert L.dfft_status_string(2) == b"infeasible decomposition"


def test_no_oracle_in_product_path():
    # the product package never imports the test oracle
    for root, _, files in os.walk(os.path.join(ROOT, "paper_2601_12209_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(root, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "dfft_oracle" not in txt, f


@pytest.mark.parametrize("shape,decomp,grid", [((8, 8, 8), "pencil", (2, 2)), ((8, 8, 8), "slab", (4, 1)),
                                               ((8, 8, 8), "pencil", (1, 1)), ((48, 12, 6), "pencil", (5, 2)),
                                               ((768, 768, 384), "pencil", (2, 4))])
def test_boxes_tile_the_grid(shape, decomp, grid):
    import numpy as np

    P = grid[0] * grid[1]
    for direction in (dfft.FORWARD, dfft.INVERSE):
        for which in (0, 1):
            cover = np.zeros(shape[::-1], dtype=np.int32) if np.prod(shape) < 1e7 else None
            total = 0
            for r in range(P):
                lo, n = dfft.decomp_box(shape, decomp, grid, "c2c_f32", direction, r, which)
                assert all(v > 0 for v in n)
                total += n[0] * n[1] * n[2]
                if cover is not None:
                    cover[lo[2]:lo[2] + n[2], lo[1]:lo[1] + n[1], lo[0]:lo[0] + n[0]] += 1
            assert total == shape[0] * shape[1] * shape[2]
            if cover is not None:
                assert (cover == 1).all()


def test_spec_decomposition_examples():
    # SPEC.md S:55-66 (TRIVIAL/DERIVED examples), recomputed by the library
    for r in range(4):
        lo, n = dfft.decomp_box((8, 8, 8), "pencil", (2, 2), "c2c_f32", -1, r, 0)
        assert n == (8, 4, 4) and lo[0] == 0 and lo[1] in (0, 4) and lo[2] in (0, 4)
    for r in range(4):
        lo, n = dfft.decomp_box((8, 8, 8), "slab", (4, 1), "c2c_f32", -1, r, 0)
        assert n == (8, 8, 2) and lo == (0, 0, 2 * r)
    lo, n = dfft.decomp_box((8, 8, 8), "pencil", (2, 2), "c2c_f32", -1, 3, 1)
    assert lo == (4, 4, 0) and n == (4, 4, 8)
    # uneven balanced blocks: remainder to the lowest parts (reading R5)
    # cfg5: r2c 768x768x384 -> 385 bins split 193/192 over P1 = 2
    xs = [dfft.decomp_box((768, 768, 384), "pencil", (2, 4), "r2c_f64", -1, r, 1)[1][0] for r in (0, 4)]
    assert xs == [193, 192]
    ys = [dfft.decomp_box((48, 12, 6), "pencil", (5, 2), "c2c_f32", -1, 2 * i, 0)[1][1] for i in range(5)]
    assert ys == [3, 3, 2, 2, 2]


@pytest.mark.parametrize("args,code", [
    (((0, 8, 8), "pencil", (1, 1)), 1),          # empty grid
    (((8, 8, 8), "slab", (2, 2)), 1),            # slab needs (P, 1)
    (((8, 8, 8), "pencil", (16, 1)), 2),         # P1 > ny
    (((8, 8, 8), "pencil", (1, 16)), 2),         # P2 > nz
    (((11, 8, 8), "pencil", (1, 1)), 3),         # prime 11 unsupported
    (((8192, 8, 8), "pencil", (1, 1)), 3),       # > 4096
])
def test_validation_errors(args, code):
    shape, decomp, grid = args
    with pytest.raises(dfft.DfftError) as ei:
        dfft.decomp_box(shape, decomp, grid, "c2c_f32", -1, 0, 0)
    assert f"({code})" in str(ei.value)
    assert dfft.lib().dfft_last_error().decode()


def test_r2c_odd_nx_unsupported():
    with pytest.raises(dfft.DfftError) as ei:
        dfft.decomp_box((9, 8, 8), "pencil", (1, 1), "r2c_f64", -1, 0, 0)
    assert "(3)" in str(ei.value)


@pytest.mark.parametrize("shape,decomp,grid", [((16, 12, 8), "pencil", (1, 1)), ((24, 16, 12), "pencil", (2, 4)),
                                               ((48, 24, 12), "pencil", (5, 2)), ((48, 24, 12), "slab", (4, 1))])
def test_r2r_boxes_are_real_and_split_in_pairs(shape, decomp, grid):
    # R2R (reading R21): real boxes on both sides; the x split of D2/D3 is in pairs of reals
    import numpy as np

    P = grid[0] * grid[1]
    for direction in (dfft.FORWARD, dfft.INVERSE):
        for which in (0, 1):
            cover = np.zeros(shape[::-1], dtype=np.int32)
            for r in range(P):
                lo, n = dfft.decomp_box(shape, decomp, grid, "r2r_f64", direction, r, which)
                assert lo[0] % 2 == 0 and n[0] % 2 == 0
                cover[lo[2]:lo[2] + n[2], lo[1]:lo[1] + n[1], lo[0]:lo[0] + n[0]] += 1
            assert (cover == 1).all()


@pytest.mark.parametrize("shape", [(9, 8, 8), (8, 9, 8), (8, 8, 6 + 1)])
def test_r2r_odd_extents_unsupported(shape):
    with pytest.raises(dfft.DfftError) as ei:
        dfft.decomp_box(shape, "pencil", (1, 1), "r2r_f32", -1, 0, 0)
    assert "(3)" in str(ei.value)


def test_kernel_launch_counter_exported():
    assert dfft.kernel_launches() >= 0
