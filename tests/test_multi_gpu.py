"""N>1 paths.  CPU (gloo, world_size 2): the host-side multi-rank logic — unique-id style
broadcast, per-rank boxes tiling the grid, scatter/gather of boxes, max-over-ranks timing
reduction.  GPU (>= 2 devices): tests/mp_check.py under torchrun — NCCL parity vs the oracle."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import inputs
    import paper_2601_12209_b200 as dfft

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1. 128-byte unique-id broadcast over the process group (as Comm.create does)
        buf = torch.arange(128, dtype=torch.uint8) if rank == 0 else torch.zeros(128, dtype=torch.uint8)
        dist.broadcast(buf, src=0)
        assert bytes(buf.tolist()) == bytes(range(128))
        # 2. each rank's boxes of 2-rank pencils and slab; gather and tile the global input
        shape = (12, 12, 6)
        for decomp, grid in (("pencil", (1, 2)), ("pencil", (2, 1)), ("slab", (2, 1))):
            for direction, which in ((dfft.FORWARD, 0), (dfft.FORWARD, 1), (dfft.INVERSE, 1)):
                lo, n = dfft.decomp_box(shape, decomp, grid, "c2c_f64", direction, rank, which)
                part = inputs.gen_complex_np(3, shape, lo, n)
                parts = [None] * world
                dist.all_gather_object(parts, (lo, n, part))
                if rank == 0:
                    full = np.full(shape[::-1], np.nan + 0j)
                    for lo_, n_, arr in parts:
                        full[lo_[2]:lo_[2] + n_[2], lo_[1]:lo_[1] + n_[1], lo_[0]:lo_[0] + n_[0]] = arr
                    assert np.array_equal(full, inputs.gen_complex_np(3, shape))
        # 3. bench.py's timing reduction: max over ranks
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == float(world)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, "ok"), (1, "ok")], res


@pytest.mark.gpu
def test_nccl_multi_gpu():
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (run under gpurun --gpus 2|4)")
    n = 4 if n >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "mp_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0 and "MP_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
