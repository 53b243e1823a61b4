/*
 * dfft.h — C ABI of libdfft.so, the B200-native distributed 3D FFT (DaggerFFT's hot path).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (arXiv 2601.12209), with its section.
 * No C++ or torch types cross this boundary: plain pointers (device or host, as stated),
 * int64 sizes, enums.  All functions return a dfft_status_t; none aborts or throws.  On
 * failure dfft_last_error() returns a thread-local human-readable detail.
 *
 * The operation (§III-A): the unnormalised forward 3D DFT
 *     X(kx,ky,kz) = Σ_x Σ_y Σ_z A(x,y,z) · exp(-2πi (kx x/Nx + ky y/Ny + kz z/Nz))
 * evaluated as three stages of batched 1D FFTs along x, y, z, each on its own
 * stage-owned decomposition D1/D2/D3 (Alg. 1), with a pack → exchange →
 * unpack redistribution between stages.  The inverse applies the same sequence
 * mirrored, z then y then x (§IV-A), with the conjugate kernel and a 1/(Nx·Ny·Nz)
 * scale (reading R1).  R2C/C2R halve the x axis: Nx/2+1 bins.
 *
 * Decompositions (readings R4-R6), rank r = i·P2 + j (row-major process grid):
 *   PENCIL P1×P2:  D1 = x whole, y split by i over P1, z split by j over P2   (input, forward)
 *                  D2 = x split by i, y whole, z split by j                    (internal)
 *                  D3 = x split by i, y split by j, z whole                    (output, forward)
 *   SLAB (p1 = P, p2 = 1):  D1 = z-slabs (x, y whole), D3 = y-slabs (x, z whole): "the first
 *                  two transforms are performed locally on each slab before a single global
 *                  transpose".  Internally identical to PENCIL with grid 1×P.
 *   Splits are balanced blocks: part q of n over p has n/p + (q < n%p) elements, lowest
 *   indices first.  For R2C the split x extent is Nx/2+1.
 *   Every user-visible box is stored dense, x fastest: element (x,y,z) of a box with origin lo
 *   and extents n is at ((z-lo_z)·n_y + (y-lo_y))·n_x + (x-lo_x).  Complex = interleaved
 *   (re, im) = torch.complex64 / complex128.
 */
#ifndef DFFT_H_
#define DFFT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFFT_VERSION 100 /* 1.0.0 */

typedef struct dfft_comm_s* dfft_comm_t;
typedef struct dfft_plan_s* dfft_plan_t;

typedef enum {
  DFFT_SUCCESS = 0,
  DFFT_ERR_INVALID_VALUE = 1,     /* bad argument: sizes <= 0, p1*p2 != nranks, null/misaligned ptr, in == out */
  DFFT_ERR_INFEASIBLE_DECOMP = 2, /* some rank would own an empty block in some layout */
  DFFT_ERR_UNSUPPORTED = 3,       /* an FFT axis length the library has no kernel for (not one of the
                                     lengths listed at dfft_plan_create), odd Nx for R2C, odd extents for R2R */
  DFFT_ERR_ALLOC = 4,             /* cudaMalloc failed */
  DFFT_ERR_CUDA = 5,              /* a CUDA runtime call failed (detail in dfft_last_error) */
  DFFT_ERR_NCCL = 6,              /* an NCCL call failed or the communicator reported an async error
                                     (ncclCommGetAsyncError, checked at every execute of an NCCL plan) */
  DFFT_ERR_INTERNAL = 7,
  DFFT_ERR_PEER = 8               /* the plan has failed: an execute made no progress within the watchdog
                                     timeout (a peer never signalled; its waits were released and the
                                     results are invalid) or an enqueue failed part-way.  Destroy it. */
} dfft_status_t;

typedef enum { DFFT_SLAB = 1, DFFT_PENCIL = 2 } dfft_decomp_t;

/* Transform type and precision.  R2C with direction INVERSE is the C2R transform.
 * R2R (reading R21 in DESIGN.md): by default FORWARD = the DCT-II along every axis (FFTW
 * REDFT10, X_k = 2 Σ x_n cos(πk(2n+1)/(2N))), INVERSE = the DCT-III along every axis divided by 2N
 * per axis, so INVERSE(FORWARD(x)) = x; dfft_plan_create_kinds picks DCT or DST per axis.  Both
 * boxes are real (float/double), x-fastest; every extent must be even and nx/2, ny, nz supported
 * lengths; the x split of the D2/D3 layouts is in pairs of reals. */
typedef enum {
  DFFT_C2C_F32 = 1, DFFT_C2C_F64 = 2, DFFT_R2C_F32 = 3, DFFT_R2C_F64 = 4, DFFT_R2R_F32 = 5, DFFT_R2R_F64 = 6
} dfft_type_t;

/* Per-axis transform kinds (dfft_plan_create_kinds; "C2C, R2C and R2R", "DCT and DST",
 * P:620 the (Periodic, Periodic, Bounded) topology; reading R22).  Forward / inverse:
 *   DFFT_KIND_DFT  (Periodic):            the DFT / the conjugate DFT ÷ n
 *   DFFT_KIND_DCT2 (Bounded, Neumann):    DCT-II  X_k = 2 Σ x_n cos(πk(2n+1)/(2n_))  / DCT-III ÷ 2n_
 *   DFFT_KIND_DST2 (Bounded, Dirichlet):  DST-II  X_k = 2 Σ x_n sin(π(k+1)(2n+1)/(2n_)) / DST-III ÷ 2n_
 * (FFTW REDFT10 / RODFT10 and their inverses REDFT01 / RODFT01 ÷ 2n_.)  A DCT / DST along y or z of
 * complex data transforms the real and imaginary parts alike. */
enum { DFFT_KIND_DFT = 0, DFFT_KIND_DCT2 = 1, DFFT_KIND_DST2 = 2 };

/* Sign of the exponent: FORWARD = -1, INVERSE = +1 with the 1/N scale. */
typedef enum { DFFT_FORWARD = -1, DFFT_INVERSE = 1 } dfft_direction_t;

/*
 * flags (bit field, 0 = defaults):
 *   bits 0-7  DFFT_FLAG_CHUNKS(k): pipeline chunk count K (0 = automatic).  The work and the
 *             exchanges are split into K chunks and run as a two-stream pipeline (P:115-126,
 *             Fig. 1 "progressive per-chunk pipelining"; Alg. 2 phases 3/5): NCCL / CE plans chunk
 *             stages A, B and both exchanges along the axis no exchange touches (z forward, x
 *             inverse); fused-store plans with both exchanges remote (p1 > 1 and p2 > 1, and the
 *             1×P2 forward) run stage A whole and chunk stages B and C (x forward, z inverse) so
 *             the local C(k) overlaps the NVLink-bound B(k+1).  Automatic K: NCCL 4, CE 8, fused
 *             stores 4 from 1 GiB per rank, 2 from 256 MiB, else 1.
 *   DFFT_FLAG_NO_OVERLAP: the same steps on the caller's stream alone, each exchange completing
 *             before the next stage starts and every stage on the whole GPU (the "SimpleMPIFFT"
 *             static-barrier ablation of P:438), for every transport.  Results are bitwise
 *             identical to the pipelined schedule.
 *   Exchange transport for P > 1 (same kernels and bitwise-identical results in every mode).
 *   Every rank's workspace is a CUDA IPC window exchanged at plan creation; flag words in the
 *   windows order producer and consumer per chunk (READY) and consumer -> producer for buffer
 *   reuse across executes (DONE): a flag kernel resets the words this rank waited on and then
 *   publishes its own with system-scope release stores; waits are cuStreamWaitValue32 for the
 *   constant value 1, so every schedule can be captured in a CUDA graph and replayed.
 *     DFFT_FLAG_FUSED_STORE (the default for P > 1): each FFT epilogue stores its off-rank
 *               elements straight into the peers' windows over NVLink (pack + send + unpack
 *               fused into the FFT's stores; bulk copies per tile from the strided stages).
 *     DFFT_FLAG_CE: the FFT epilogue packs each off-rank block into a local send block and the
 *               comm stream's copy engine moves it into the receiver's window, K chunks
 *               pipelined against the FFTs (no SM time on transfers).
 *     DFFT_FLAG_HYBRID: fused stores for the forward x-FFT (long x-runs), CE elsewhere.
 *     DFFT_FLAG_NCCL: grouped ncclSend/ncclRecv of the send blocks (baseline/ablation).
 *   Env overrides (read at plan creation, real communicators only; every rank must resolve the
 *   same plan, which plan creation checks): DFFT_EXCHANGE=p2p|ce|hybrid|nccl, DFFT_NO_BC=1 (no
 *   B→C pipeline), DFFT_NO_BC_1XP=1 (no B→C pipeline on 1×P2 forwards), DFFT_NVL_SMS=n (SMs of
 *   the NVLink-bound stage of a pipelined pair, default 80).
 *   Layout overrides (local to a rank, any communicator): DFFT_NO_XZ8=1 (single GPU: the
 *   whole-axis x, z, y passes instead of the x-FFT fused with a radix-8 z step),
 *   DFFT_NO_NAT1=1 (1×P2 fused stores: the inverse y-IFFT writes wy-column blocks instead of
 *   natural x-lines).  dfft_plan_describe reports the plan each resolves to.
 */
#define DFFT_FLAG_CHUNKS(k) ((uint64_t)((k) & 0xff))
#define DFFT_FLAG_NO_OVERLAP ((uint64_t)1 << 8)
#define DFFT_FLAG_NCCL ((uint64_t)1 << 9)
#define DFFT_FLAG_FUSED_STORE ((uint64_t)1 << 10)
#define DFFT_FLAG_CE ((uint64_t)1 << 11)
#define DFFT_FLAG_HYBRID ((uint64_t)1 << 12)

int dfft_version(void);
const char* dfft_status_string(dfft_status_t status);
/* Thread-local detail of the last failure on this thread ("" if none).  Valid until the next call. */
const char* dfft_last_error(void);

/* ------------------------------------------------------------------ communicators
 * One process per GPU.  Rank 0 calls dfft_get_unique_id and the caller broadcasts the
 * 128 bytes (e.g. over a torch.distributed process group); every rank then calls
 * dfft_comm_init collectively.  nranks == 1 needs no id (pass NULL) and creates no NCCL
 * communicator.  The comm must outlive its plans.
 */
dfft_status_t dfft_get_unique_id(unsigned char id[128]);
dfft_status_t dfft_comm_init(dfft_comm_t* comm, int nranks, int rank, const unsigned char id[128],
                             int cuda_device);
/*
 * Simulated communicator (test/diagnostic): all `nranks` ranks live in this process on one
 * GPU.  Plans created on it hold every rank's buffers; dfft_execute_sim runs every rank's
 * stage kernels and performs the exchange with device-to-device copies of exactly the
 * blocks NCCL would move.  Used to validate P = 8 layouts when fewer GPUs are available.
 */
dfft_status_t dfft_comm_init_sim(dfft_comm_t* comm, int nranks, int cuda_device);
dfft_status_t dfft_comm_destroy(dfft_comm_t comm);

/* ------------------------------------------------------------------ plans
 * Supported FFT axis lengths: every n = 2^a 3^b 5^c 7^d <= 4096.  Specialised kernels (persistent
 * TMA strided kernel, fused pack epilogues, R2C / C2R / DCT / DST variants) exist for 2^a (2..4096),
 * 3·2^a (3..3072), 5, 7 and the paper's GPU shapes 480, 720, 840; other lengths run a
 * generic kernel with the radix schedule at run time (c2c axes only: an R2C / R2R x axis — nx/2 —
 * and DCT / DST axes need a specialised length).  Anything else returns DFFT_ERR_UNSUPPORTED.
 * Collective over comm (every rank calls it with the same arguments).  Builds the stage
 * geometry, twiddle tables, per-stage address tables, work buffers, sub-communicators
 * (row = ranks with the same j, column = same i), streams and events once; execution
 * reuses them ("plan creation is performed only once per distinct transform
 * configuration", §V-B; "persistent workspaces and buffer reuse").
 * proc grid: PENCIL takes p1 × p2; SLAB requires p2 == 1 and p1 == nranks.
 */
dfft_status_t dfft_plan_create(dfft_plan_t* plan, dfft_comm_t comm, int64_t nx, int64_t ny, int64_t nz,
                               dfft_decomp_t decomp, int p1, int p2, dfft_type_t type,
                               dfft_direction_t direction, uint64_t flags);
/*
 * Same, with a transform kind per axis (x, y, z): kinds[d] ∈ DFFT_KIND_*.  dfft_plan_create is this
 * with all-DFT kinds for C2C / R2C types and all-DCT2 for R2R.  Allowed combinations:
 *   C2C and R2C: kinds[0] = DFT (x periodic; R2C halves it), kinds[1], kinds[2] any — e.g. the
 *                paper's (Periodic, Periodic, Bounded) box is R2C with {DFT, DFT, DCT2} (Neumann)
 *                or {DFT, DFT, DST2} (Dirichlet);
 *   R2R:         DCT2 or DST2 on every axis (real boxes both ways, x split in pairs of reals).
 * Every DCT / DST axis needs an even extent.  Boxes, layouts, transports and the other arguments
 * are as for dfft_plan_create; errors: INVALID_VALUE for a bad kind, UNSUPPORTED for a combination
 * outside the list.
 */
dfft_status_t dfft_plan_create_kinds(dfft_plan_t* plan, dfft_comm_t comm, int64_t nx, int64_t ny, int64_t nz,
                                     dfft_decomp_t decomp, int p1, int p2, dfft_type_t type, const int kinds[3],
                                     dfft_direction_t direction, uint64_t flags);

/* This rank's input (which = 0) or output (which = 1) box, x,y,z order.  For a simulated
 * comm use dfft_plan_box_rank. */
dfft_status_t dfft_plan_box(dfft_plan_t plan, int which, int64_t lo[3], int64_t n[3]);
dfft_status_t dfft_plan_box_rank(dfft_plan_t plan, int rank, int which, int64_t lo[3], int64_t n[3]);

/* Bytes of this rank's input box, output box, and plan-owned device workspace. */
dfft_status_t dfft_plan_bytes(dfft_plan_t plan, size_t* in_bytes, size_t* out_bytes, size_t* workspace_bytes);

/* Pure geometry (no GPU needed): the input (which = 0) or output (which = 1) box of `rank`
 * for these plan arguments, with the same validation as dfft_plan_create. */
dfft_status_t dfft_decomp_box(int64_t nx, int64_t ny, int64_t nz, dfft_decomp_t decomp, int p1, int p2,
                              dfft_type_t type, dfft_direction_t direction, int rank, int which, int64_t lo[3],
                              int64_t n[3]);

/* Chunk count K actually used. */
dfft_status_t dfft_plan_chunks(dfft_plan_t plan, int* chunks);

/*
 * Execute on device buffers.  `in` is this rank's input box (forward: D1; inverse: D3),
 * `out` its output box (forward: D3; inverse: D1), both device pointers on the plan's
 * GPU, 16-byte aligned, dense as described above, non-overlapping; `in` is never written.
 * Stream-ordered and asynchronous: work is enqueued after everything already on `stream`
 * and `stream` waits for its completion; no host synchronisation.  Capturable in a CUDA graph
 * for every transport (the IPC-window flag protocol waits for constant values; NCCL plans follow
 * NCCL's own capture rules).
 * Collective: all ranks execute matching plans in the same order.  A multi-rank execute that
 * makes no progress for the watchdog timeout (dfft_set_timeout_ms, env DFFT_TIMEOUT_MS, default
 * 120 s) is reported on stderr, its waits are released so the streams drain, and the plan fails:
 * this and later calls return DFFT_ERR_PEER.  If an enqueue fails part-way, the remaining flag
 * waits and signals are still issued (peers stay in step), the error is returned and the plan
 * fails likewise.
 * `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 */
dfft_status_t dfft_execute(dfft_plan_t plan, const void* in, void* out, void* stream);

/*
 * Same, with host pointers (pageable or pinned): copies `in` to a plan-owned device staging
 * buffer, executes, copies the result back to `out`, and synchronises `stream` before
 * returning.  This is the end-to-end entry point (host → device → host).
 */
dfft_status_t dfft_execute_host(dfft_plan_t plan, const void* in_host, void* out_host, void* stream);

/*
 * End to end through a chain of plans (e.g. forward then inverse, or the Poisson solve's forward
 * with the 1/λ multiplier then the C2R inverse): host `in` → device → plans[0] → … →
 * plans[nplans-1] → host `out`, with the intermediate results kept on the device.  Plan q's output
 * box must be plan q+1's input box (same bytes).  The host→device copy runs on a plan-owned copy
 * stream and the device→host copy on another, with double-buffered device staging (owned by
 * plans[0], reused while the chain stays the same), so with async != 0 the host→device copy of the
 * next call overlaps this call's transforms and device→host copy.  `stream` completes when `out`
 * holds the result.  async == 0: returns after synchronising `stream` (any host memory); async != 0:
 * returns after enqueueing — both host buffers must then be page-locked (else INVALID_VALUE) and
 * stay untouched until `stream` completes.  Collective like dfft_execute.
 */
dfft_status_t dfft_execute_host_chain(const dfft_plan_t* plans, int nplans, const void* in_host, void* out_host,
                                      void* stream, int async);

/* Simulated comm only: ins[r] / outs[r] are rank r's device boxes, r < nranks.
 * Plans with an IPC-window transport (DFFT_FLAG_FUSED_STORE / _CE / _HYBRID on a simulated comm)
 * run every rank's own execute schedule as a real rank does — its stream pair, the flag words in
 * its workspace (which stands in for its IPC window), chunks, the B→C pipeline and SM caps —
 * issued interleaved, so all ranks run concurrently on the one GPU; ins[r] == NULL means rank r
 * does not take part (a failed peer: the others wait until the watchdog releases them).
 * Otherwise (NCCL layouts) every rank's stages run in stream order with device copies of the
 * blocks NCCL would move. */
dfft_status_t dfft_execute_sim(dfft_plan_t plan, const void* const* ins, void* const* outs, void* stream);

/*
 * Poisson solve, fused (the paper's application, §VI-B: the
 * Oceananigans pressure Poisson solver on a (Periodic, Periodic, Periodic) box, and P:620's
 * (Periodic, Periodic, Bounded) box).  Turns a FORWARD plan into  F(k) -> F(k) / λ(k),
 * λ(k) = Σ_d λ_d(k_d) with λ_d(k) = -(2 sin(θ_k) / h_d)² and θ_k = πk/n_d on a DFT axis
 * (periodic), πk/(2n_d) on a DCT2 axis (Neumann: cell-centred mirror boundary), π(k+1)/(2n_d) on
 * a DST2 axis (Dirichlet: antimirror boundary) — the eigenvalues of the 7-point discrete Laplacian
 * with spacings h = (dx, dy, dz) and those boundaries (readings R20, R22) — and F(k) -> 0
 * where λ(k) = 0 (the zero-mean solution; only k = 0 without a Dirichlet axis).  The multiply is
 * fused into the epilogue of the plan's last stage (no extra pass over HBM).  Executing the
 * forward plan and then the matching INVERSE plan solves ∇²φ = f.  dx = dy = dz = 0 switches the
 * multiplier off again.  Synchronises the device (plan setup, not for the hot path).  Errors:
 * INVALID_VALUE for an inverse plan or non-positive spacings.
 */
dfft_status_t dfft_plan_set_poisson(dfft_plan_t plan, double dx, double dy, double dz);

/* ------------------------------------------------------------------ per-phase profiling
 * Phases (Fig. 9 breakdown analog): 0 stage-A FFT, 1 first exchange, 2 stage-B FFT,
 * 3 second exchange, 4 stage-C FFT.  When enabled, every stage launch and exchange of
 * dfft_execute is bracketed by CUDA timing events on the stream that runs it.
 * dfft_plan_phase_times synchronises those events and returns the accumulated milliseconds
 * and launch counts per phase (reset != 0 zeroes the accumulators afterwards).
 * dfft_plan_stage_bytes returns the algorithmic bytes per execute of each phase: FFT stages
 * read + write their local array once (2·elements·element size); exchanges count the bytes
 * this rank sends to other ranks.
 */
dfft_status_t dfft_plan_set_profiling(dfft_plan_t plan, int on);
dfft_status_t dfft_plan_phase_times(dfft_plan_t plan, double ms[5], long long launches[5], int reset);
dfft_status_t dfft_plan_stage_bytes(dfft_plan_t plan, double bytes[5]);
/* Plan description (rank 0's stages): one text line per stage launch unit, "<phase> <kernel
 * family> n=<length> L0=.. L1=.. in_tstride=.. out_tstride=.. tma=0|1 maxr=<largest radix of the
 * kernel's passes>", NUL-terminated in buf
 * (caller-owned, len bytes).  DFFT_ERR_INVALID_VALUE when it does not fit (buf holds a truncated
 * copy).  Families: contig, strided, contig_r2c, contig_c2r, contig_dct, strided_dct, contig_dst,
 * strided_dst, xz8 (the single-GPU x-FFT fused with a radix-8 z step). */
dfft_status_t dfft_plan_describe(dfft_plan_t plan, char* buf, size_t len);
/* Timeline of the profiled executes (Fig. 9 per-chunk analog): one span per stage launch or
 * exchange step, on stream 0 (compute X) or 1 (Y), with its chunk and rank, in milliseconds
 * relative to the origin event its execute recorded on the caller's stream (exec numbers count
 * the executes since the last read).  Synchronises.  cap = 0 returns the count in *n; otherwise up
 * to cap spans are copied and removed (dfft_plan_phase_times with reset != 0 discards them). */
typedef struct {
  int phase, stream, chunk, rank, exec;
  double t0_ms, t1_ms;
} dfft_span_t;
dfft_status_t dfft_plan_timeline(dfft_plan_t plan, dfft_span_t* spans, int cap, int* n);

/* Watchdog timeout for multi-rank executes, process-wide (ms > 0). */
dfft_status_t dfft_set_timeout_ms(long long ms);
/* DFFT_SUCCESS while the plan is usable; DFFT_ERR_PEER once it failed; DFFT_ERR_NCCL if its NCCL
 * communicator reports an asynchronous error. */
dfft_status_t dfft_plan_status(dfft_plan_t plan);

/* Number of kernels this library has launched in the process so far (FFT stages and flag
 * signals; NCCL's own kernels and copy-engine transfers are not kernels of ours).  Monotonic;
 * the bench reads it around its timed region. */
long long dfft_kernel_launches(void);

/* Synchronises the plan's internal streams, then frees everything the plan owns. */
dfft_status_t dfft_destroy(dfft_plan_t plan);

/* ------------------------------------------------------------------ diagnostics
 * Batched 1D transform of `howmany` contiguous lines of length n (device pointers), in the
 * same kernels the 3D path uses (stage-1 contiguous kernel, c2c only).  Used by parity tests
 * of the per-length radix schedules.  sign = -1 forward, +1 inverse (unscaled).
 */
dfft_status_t dfft_fft1d(const void* in, void* out, int64_t n, int64_t howmany, int f64, int sign,
                         void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DFFT_H_ */
