"""paper_2601_12209_b200 — B200-native distributed 3D FFT (DaggerFFT's hot path, arXiv 2601.12209).

Thin ctypes binding over ``libdfft.so`` (include/dfft.h): argument marshalling only — every
step of the transform runs in the library's CUDA kernels and NCCL calls.  PyTorch is used for
device memory, streams and (for the 128-byte NCCL unique id) process groups.  There is no CPU
fallback: if the native library is missing, importing the binding's functions raises.

    comm = Comm.create()                       # 1 process per GPU; uses torch.distributed if initialised
    fwd = Plan(comm, (nx, ny, nz), "pencil", (p1, p2), "c2c_f32", FORWARD)
    x = fwd.alloc_in(); y = fwd.alloc_out()    # this rank's D1 / D3 boxes (torch, x fastest)
    fwd.execute(x, y)                          # stream-ordered on torch's current stream
"""
from __future__ import annotations

import ctypes
import os
from typing import Sequence

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DFFT_LIB", os.path.join(PKG, "libdfft.so"))  # DFFT_LIB: dev A/B builds only

FORWARD, INVERSE = -1, 1
SLAB, PENCIL = 1, 2
TYPES = {"c2c_f32": 1, "c2c_f64": 2, "r2c_f32": 3, "r2c_f64": 4, "r2r_f32": 5, "r2r_f64": 6}
FLAG_NO_OVERLAP = 1 << 8
FLAG_NCCL = 1 << 9
FLAG_FUSED_STORE = 1 << 10
FLAG_CE = 1 << 11
FLAG_HYBRID = 1 << 12

# symbols include/dfft.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "dfft_version", "dfft_status_string", "dfft_last_error", "dfft_get_unique_id", "dfft_comm_init",
    "dfft_comm_init_sim", "dfft_comm_destroy", "dfft_plan_create", "dfft_plan_box", "dfft_plan_box_rank",
    "dfft_plan_bytes", "dfft_decomp_box", "dfft_plan_chunks", "dfft_execute", "dfft_execute_host", "dfft_execute_sim",
    "dfft_destroy", "dfft_fft1d", "dfft_plan_set_profiling", "dfft_plan_phase_times", "dfft_plan_stage_bytes",
    "dfft_plan_describe",
    "dfft_plan_set_poisson", "dfft_kernel_launches", "dfft_plan_timeline", "dfft_set_timeout_ms", "dfft_plan_status",
    "dfft_execute_host_chain", "dfft_plan_create_kinds",
]
KINDS = {"dft": 0, "dct": 1, "dst": 2}  # DFFT_KIND_*: periodic, Neumann (DCT-II), Dirichlet (DST-II)
PHASES = ["stage_A", "exchange_1", "stage_B", "exchange_2", "stage_C"]

_lib = None
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int


class DfftError(RuntimeError):
    def __init__(self, msg, status=None):
        super().__init__(msg)
        self.status = status


class Span(ctypes.Structure):
    """dfft_span_t: one stage launch / exchange step of a profiled execute (times in ms relative
    to its execute's origin event)."""
    _fields_ = [("phase", ctypes.c_int), ("stream", ctypes.c_int), ("chunk", ctypes.c_int), ("rank", ctypes.c_int),
                ("exec", ctypes.c_int), ("t0_ms", ctypes.c_double), ("t1_ms", ctypes.c_double)]


def flag_chunks(k: int) -> int:
    return k & 0xFF


def lib():
    """Load libdfft.so (raises if it was not built — no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DfftError(f"{LIB_PATH} not built; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        L.dfft_version.restype = _int
        if hasattr(L, "dfft_kernel_launches"):
            L.dfft_kernel_launches.restype = ctypes.c_longlong
        L.dfft_status_string.restype = ctypes.c_char_p
        L.dfft_status_string.argtypes = [_int]
        L.dfft_last_error.restype = ctypes.c_char_p
        L.dfft_get_unique_id.argtypes = [ctypes.c_char_p]
        L.dfft_comm_init.argtypes = [ctypes.POINTER(_vp), _int, _int, ctypes.c_char_p, _int]
        L.dfft_comm_init_sim.argtypes = [ctypes.POINTER(_vp), _int, _int]
        L.dfft_comm_destroy.argtypes = [_vp]
        L.dfft_plan_create.argtypes = [ctypes.POINTER(_vp), _vp, _i64, _i64, _i64, _int, _int, _int, _int, _int,
                                       ctypes.c_uint64]
        L.dfft_plan_create_kinds.argtypes = [ctypes.POINTER(_vp), _vp, _i64, _i64, _i64, _int, _int, _int, _int,
                                             ctypes.POINTER(_int), _int, ctypes.c_uint64]
        L.dfft_plan_box.argtypes = [_vp, _int, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
        L.dfft_plan_box_rank.argtypes = [_vp, _int, _int, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
        L.dfft_plan_bytes.argtypes = [_vp, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t),
                                      ctypes.POINTER(ctypes.c_size_t)]
        L.dfft_decomp_box.argtypes = [_i64, _i64, _i64, _int, _int, _int, _int, _int, _int, _int,
                                      ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
        L.dfft_plan_chunks.argtypes = [_vp, ctypes.POINTER(_int)]
        L.dfft_execute.argtypes = [_vp, _vp, _vp, _vp]
        L.dfft_execute_host.argtypes = [_vp, _vp, _vp, _vp]
        L.dfft_execute_host_chain.argtypes = [ctypes.POINTER(_vp), _int, _vp, _vp, _vp, _int]
        L.dfft_execute_sim.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp]
        L.dfft_destroy.argtypes = [_vp]
        L.dfft_fft1d.argtypes = [_vp, _vp, _i64, _i64, _int, _int, _vp]
        L.dfft_plan_set_profiling.argtypes = [_vp, _int]
        if hasattr(L, "dfft_plan_set_poisson"):  # (absent from older dev A/B builds)
            L.dfft_plan_set_poisson.argtypes = [_vp, ctypes.c_double, ctypes.c_double, ctypes.c_double]
        L.dfft_plan_phase_times.argtypes = [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_longlong), _int]
        L.dfft_plan_stage_bytes.argtypes = [_vp, ctypes.POINTER(ctypes.c_double)]
        L.dfft_plan_describe.argtypes = [_vp, ctypes.c_char_p, ctypes.c_size_t]
        L.dfft_plan_timeline.argtypes = [_vp, ctypes.POINTER(Span), _int, ctypes.POINTER(_int)]
        L.dfft_set_timeout_ms.argtypes = [ctypes.c_longlong]
        L.dfft_plan_status.argtypes = [_vp]
        for name in EXPORTS:
            if name not in ("dfft_version", "dfft_status_string", "dfft_last_error", "dfft_kernel_launches") and hasattr(L, name):
                getattr(L, name).restype = _int  # (every symbol exists in the in-tree build: test_abi)
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        L = lib()
        raise DfftError(f"{what}: {L.dfft_status_string(rc).decode()} ({rc}): {L.dfft_last_error().decode()}", rc)


def _stream_ptr(stream, device):
    import torch

    if stream is None:
        stream = torch.cuda.current_stream(device)
    return _vp(stream.cuda_stream)


def version() -> int:
    return lib().dfft_version()


def decomp_box(shape, decomp: str, grid, dtype: str, direction: int, rank: int, which: int):
    """Pure geometry query (no GPU): (lo, n) of `rank`'s input (0) / output (1) box."""
    lo, n = (_i64 * 3)(), (_i64 * 3)()
    d = SLAB if decomp == "slab" else PENCIL
    _check(lib().dfft_decomp_box(*[int(s) for s in shape], d, int(grid[0]), int(grid[1]), TYPES[dtype], direction,
                                 rank, which, lo, n), "dfft_decomp_box")
    return tuple(lo), tuple(n)


# ---------------------------------------------------------------------------------- comm
class Comm:
    """One rank's communicator (NCCL), or a simulated all-ranks-in-one-process comm."""

    def __init__(self, handle, nranks: int, rank: int, device: int, sim: bool):
        self.h, self.nranks, self.rank, self.device, self.sim = handle, nranks, rank, device, sim

    @classmethod
    def create(cls, nranks: int | None = None, rank: int | None = None, device: int | None = None, group=None):
        """NCCL comm over the torch.distributed world (unique id broadcast over `group`)."""
        import torch

        dist = torch.distributed
        if nranks is None:
            nranks = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank(group) if nranks > 1 else 0
        if device is None:
            device = torch.cuda.current_device()
        uid = None
        if nranks > 1:
            buf = ctypes.create_string_buffer(128)
            if rank == 0:
                _check(lib().dfft_get_unique_id(buf), "dfft_get_unique_id")
            backend = dist.get_backend(group)
            dev = torch.device("cuda", device) if backend == "nccl" else torch.device("cpu")
            t = torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8).to(dev)
            dist.broadcast(t, src=0, group=group)
            uid = bytes(t.cpu().tolist())
        h = _vp()
        _check(lib().dfft_comm_init(ctypes.byref(h), nranks, rank, uid, device), "dfft_comm_init")
        return cls(h, nranks, rank, device, False)

    @classmethod
    def simulated(cls, nranks: int, device: int = 0):
        h = _vp()
        _check(lib().dfft_comm_init_sim(ctypes.byref(h), nranks, device), "dfft_comm_init_sim")
        return cls(h, nranks, 0, device, True)

    def destroy(self):
        if self.h:
            lib().dfft_comm_destroy(self.h)
            self.h = None


# ---------------------------------------------------------------------------------- plan
class Plan:
    """A distributed 3D FFT plan (dfft_plan_create).  dtype: c2c_f32 | c2c_f64 | r2c_f32 | r2c_f64 |
    r2r_f32 | r2r_f64 (DCT-II forward / DCT-III/(2N) inverse per axis, real boxes).  kinds: per-axis
    transform kinds ("dft" | "dct" | "dst" for x, y, z; dfft_plan_create_kinds), e.g. the paper's
    (Periodic, Periodic, Bounded) box = r2c with ("dft", "dft", "dct")."""

    def __init__(self, comm: Comm, shape: Sequence[int], decomp: str = "pencil", grid: Sequence[int] = (1, 1),
                 dtype: str = "c2c_f32", direction: int = FORWARD, chunks: int = 0, overlap: bool = True,
                 exchange: str = "auto", kinds=None):
        self.comm, self.shape, self.dtype, self.direction = comm, tuple(int(s) for s in shape), dtype, direction
        self.decomp = decomp
        flags = flag_chunks(chunks) | (0 if overlap else FLAG_NO_OVERLAP) | {"nccl": FLAG_NCCL, "p2p": FLAG_FUSED_STORE, "ce": FLAG_CE, "hybrid": FLAG_HYBRID, "auto": 0}[exchange]
        h = _vp()
        d = SLAB if decomp == "slab" else PENCIL
        self.kinds = tuple(kinds) if kinds is not None else None
        if kinds is None:
            _check(lib().dfft_plan_create(ctypes.byref(h), comm.h, *self.shape, d, int(grid[0]), int(grid[1]),
                                          TYPES[dtype], direction, flags), "dfft_plan_create")
        else:
            ks = (_int * 3)(*[KINDS[k] for k in kinds])
            _check(lib().dfft_plan_create_kinds(ctypes.byref(h), comm.h, *self.shape, d, int(grid[0]), int(grid[1]),
                                                TYPES[dtype], ks, direction, flags), "dfft_plan_create_kinds")
        self.h = h

    # boxes ------------------------------------------------------------------------
    def box(self, which: int, rank: int | None = None):
        """(lo, n) in x,y,z order of the input (0) or output (1) box."""
        lo, n = (_i64 * 3)(), (_i64 * 3)()
        if rank is None:
            _check(lib().dfft_plan_box(self.h, which, lo, n), "dfft_plan_box")
        else:
            _check(lib().dfft_plan_box_rank(self.h, rank, which, lo, n), "dfft_plan_box_rank")
        return tuple(lo), tuple(n)

    def chunks(self) -> int:
        k = _int()
        _check(lib().dfft_plan_chunks(self.h, ctypes.byref(k)), "dfft_plan_chunks")
        return k.value

    def nbytes(self):
        a, b, c = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        _check(lib().dfft_plan_bytes(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), "dfft_plan_bytes")
        return a.value, b.value, c.value

    def _torch_dtype(self, which: int):
        import torch

        f64 = self.dtype.endswith("f64")
        real = self.dtype.startswith("r2r") or (self.dtype.startswith("r2c") and ((which == 0) == (self.direction == FORWARD)))
        if real:
            return torch.float64 if f64 else torch.float32
        return torch.complex128 if f64 else torch.complex64

    def alloc(self, which: int, rank: int | None = None):
        import torch

        _, n = self.box(which, rank)
        return torch.empty((n[2], n[1], n[0]), dtype=self._torch_dtype(which),
                           device=torch.device("cuda", self.comm.device))

    def alloc_in(self, rank=None):
        return self.alloc(0, rank)

    def alloc_out(self, rank=None):
        return self.alloc(1, rank)

    # execution --------------------------------------------------------------------
    def _check_tensor(self, t, which, rank=None):
        _, n = self.box(which, rank)
        assert t.is_cuda and t.is_contiguous(), "tensors must be contiguous CUDA tensors"
        assert t.dtype == self._torch_dtype(which), f"dtype {t.dtype} != {self._torch_dtype(which)}"
        assert t.numel() == n[0] * n[1] * n[2], f"box has {n} elements, tensor {tuple(t.shape)}"

    def execute(self, x, y, stream=None):
        """Enqueue the transform x -> y on `stream` (default: torch's current stream)."""
        self._check_tensor(x, 0)
        self._check_tensor(y, 1)
        _check(lib().dfft_execute(self.h, _vp(x.data_ptr()), _vp(y.data_ptr()), _stream_ptr(stream, x.device)),
               "dfft_execute")
        return y

    def execute_host(self, x_host, y_host, stream=None):
        """End-to-end: host buffers (numpy arrays or pinned CPU tensors) in and out; synchronises."""
        import torch

        dev = torch.device("cuda", self.comm.device)
        _check(lib().dfft_execute_host(self.h, _vp(_host_ptr(x_host)), _vp(_host_ptr(y_host)), _stream_ptr(stream, dev)),
               "dfft_execute_host")
        return y_host

    def execute_sim(self, xs, ys, stream=None):
        """Simulated comm: xs[r], ys[r] are rank r's boxes (xs[r] None: rank r does not take part —
        a failed peer, IPC-window plans only)."""
        P = self.comm.nranks
        for r in range(P):
            if xs[r] is not None:
                self._check_tensor(xs[r], 0, r)
                self._check_tensor(ys[r], 1, r)
        ins = (_vp * P)(*[None if x is None else x.data_ptr() for x in xs])
        outs = (_vp * P)(*[None if y is None else y.data_ptr() for y in ys])
        dev = next(x for x in xs if x is not None).device
        _check(lib().dfft_execute_sim(self.h, ins, outs, _stream_ptr(stream, dev)), "dfft_execute_sim")
        return ys

    def status(self) -> int:
        """0 while usable; DFFT_ERR_PEER (8) once the plan failed (dfft_plan_status)."""
        return int(lib().dfft_plan_status(self.h))

    # periodic Poisson solve (fused spectral divide; forward plans) ------------------
    def set_poisson(self, spacing=(1.0, 1.0, 1.0)):
        """Forward plan: multiply the spectrum by 1/λ(k) of the 7-point Laplacian (0 at k = 0) in
        the last stage's epilogue; spacing None switches it off (dfft_plan_set_poisson)."""
        dx, dy, dz = (0.0, 0.0, 0.0) if spacing is None else (float(v) for v in spacing)
        _check(lib().dfft_plan_set_poisson(self.h, dx, dy, dz), "dfft_plan_set_poisson")
        return self

    # profiling ----------------------------------------------------------------------
    def set_profiling(self, on: bool = True):
        _check(lib().dfft_plan_set_profiling(self.h, int(on)), "dfft_plan_set_profiling")

    def phase_times(self, reset: bool = True):
        """{phase: (total ms, launches)} accumulated since the last reset (synchronises)."""
        ms, n = (ctypes.c_double * 5)(), (ctypes.c_longlong * 5)()
        _check(lib().dfft_plan_phase_times(self.h, ms, n, int(reset)), "dfft_plan_phase_times")
        return {PHASES[q]: (ms[q], n[q]) for q in range(5)}

    def timeline(self):
        """Spans of the profiled executes since the last read: list of dicts (dfft_plan_timeline)."""
        n = _int()
        _check(lib().dfft_plan_timeline(self.h, None, 0, ctypes.byref(n)), "dfft_plan_timeline")
        if n.value == 0:
            return []
        buf = (Span * n.value)()
        _check(lib().dfft_plan_timeline(self.h, buf, n.value, ctypes.byref(n)), "dfft_plan_timeline")
        return [{"phase": PHASES[s.phase], "stream": s.stream, "chunk": s.chunk, "rank": s.rank, "exec": s.exec,
                 "t0_ms": s.t0_ms, "t1_ms": s.t1_ms} for s in buf[:n.value]]

    def stage_bytes(self):
        b = (ctypes.c_double * 5)()
        _check(lib().dfft_plan_stage_bytes(self.h, b), "dfft_plan_stage_bytes")
        return {PHASES[q]: b[q] for q in range(5)}

    def describe(self):
        """Rank 0's stages: [{"phase", "family", "n", "L0", "L1", "in_tstride", "out_tstride", "tma", "maxr"}]."""
        buf = ctypes.create_string_buffer(8192)
        _check(lib().dfft_plan_describe(self.h, buf, len(buf)), "dfft_plan_describe")
        out = []
        for line in buf.value.decode().splitlines():
            ph, fam, *kv = line.split()
            d = {"phase": ph, "family": fam}
            d.update({k: int(v) for k, v in (t.split("=") for t in kv)})
            out.append(d)
        return out

    def destroy(self):
        if getattr(self, "h", None):
            lib().dfft_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def fft1d(x, y, sign: int = FORWARD, stream=None):
    """Batched 1D c2c of the rows of x (…, n) into y with the stage-1 kernel (diagnostic)."""
    import torch

    n = x.shape[-1]
    assert x.is_contiguous() and y.is_contiguous() and x.dtype == y.dtype and x.numel() == y.numel()
    f64 = x.dtype == torch.complex128
    _check(lib().dfft_fft1d(_vp(x.data_ptr()), _vp(y.data_ptr()), n, x.numel() // n, int(f64), sign,
                            _stream_ptr(stream, x.device)), "dfft_fft1d")
    return y


def _host_ptr(a):
    import torch

    return a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data


def execute_host_chain(plans, x_host, y_host, stream=None, async_: bool = False):
    """Host x -> plans[0] -> ... -> plans[-1] -> host y (dfft_execute_host_chain).  async_: return
    after enqueueing (pinned host buffers; the stream completes when y holds the result)."""
    import torch

    hs = (_vp * len(plans))(*[p.h.value for p in plans])
    dev = torch.device("cuda", plans[0].comm.device)
    _check(lib().dfft_execute_host_chain(hs, len(plans), _vp(_host_ptr(x_host)), _vp(_host_ptr(y_host)),
                                         _stream_ptr(stream, dev), int(bool(async_))), "dfft_execute_host_chain")
    return y_host


def set_timeout_ms(ms: int) -> None:
    """Watchdog timeout of multi-rank executes (process-wide, dfft_set_timeout_ms)."""
    _check(lib().dfft_set_timeout_ms(int(ms)), "dfft_set_timeout_ms")


def kernel_launches() -> int:
    """Kernels libdfft has launched in this process so far (dfft_kernel_launches)."""
    return int(lib().dfft_kernel_launches())
