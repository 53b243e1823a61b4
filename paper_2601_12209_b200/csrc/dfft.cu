// dfft.cu — host side of libdfft.so: geometry, plans, the chunked two-stream executor,
// NCCL exchanges, and the C ABI declared in include/dfft.h.
//
// Pipeline (§III-A, Alg. 1, inverse mirrored P:269):
//   stage A (chunked) → exchange 1 (chunked) → stage B (chunked) → exchange 2 (chunked) → stage C
//   forward: A = x-FFT (D1 → send blocks by x-owner), B = y-FFT, C = z-FFT in place on `out`
//   inverse: A = z-IFFT, B = y-IFFT, C = x-IFFT (×1/N) into `out`
// Each exchange is an all-to-all among the P1 (row) or P2 (column) peers: grouped
// ncclSend/ncclRecv of exactly the blocks each peer owns (Alg. 2 phases 2/3/5).  Packing is
// fused into the producing FFT's last pass, unpacking into the consuming FFT's first pass,
// and the self block is written straight into its final place (Alg. 2 phase 4 elided).
// The K chunks run on a compute stream and a comm stream linked by events, so chunk k's
// exchange overlaps chunk k+1's FFT (Fig. 1 "progressive per-chunk pipelining").
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <chrono>
#include <map>
#include <numeric>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dfft.h"
#include "registry.h"

using namespace dfft;

// ------------------------------------------------------------------------------ errors
namespace {
thread_local std::string g_err;

dfft_status_t fail(dfft_status_t st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CU(call)                                                                                 \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess)                                                                       \
      return fail(DFFT_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                     \
  } while (0)

#define NC(call)                                                                                 \
  do {                                                                                           \
    ncclResult_t r_ = (call);                                                                    \
    if (r_ != ncclSuccess)                                                                       \
      return fail(DFFT_ERR_NCCL, "%s failed: %s (%s:%d)", #call, ncclGetErrorString(r_), __FILE__, \
                  __LINE__);                                                                     \
  } while (0)

#define ST(call)                          \
  do {                                    \
    dfft_status_t s_ = (call);            \
    if (s_ != DFFT_SUCCESS) return s_;    \
  } while (0)

// ------------------------------------------------------------------------------ geometry
// balanced block partition of n over p parts, remainder to the lowest parts (reading R5)
inline long long blk(long long n, long long p, long long q) { return n / p + (q < n % p ? 1 : 0); }
inline long long blo(long long n, long long p, long long q) { return q * (n / p) + std::min(q, n % p); }
inline long long owner(long long t, long long n, long long p) {
  long long b = n / p, r = n % p;
  if (t < r * (b + 1)) return t / (b + 1);
  return r + (t - r * (b + 1)) / b;
}

bool length_ok(long long n) { return dfft::length_supported(n); }

// ------------------------------------------------------------------------------ twiddles
// Per-pass tables: pass p >= 1 of radix R with Ns = prod(earlier radices) stores
// w_{Ns R}^{m r} for r in [1,R), m in [0,Ns) at [(r-1)·Ns + m];  w = exp(dir·2πi/(Ns R)).
// Computed in long double (x87 80-bit), rounded once (never by recurrence).
struct TwKey {
  int n, f64, dir, dev, maxr;
  bool operator<(const TwKey& o) const {
    return std::tie(n, f64, dir, dev, maxr) < std::tie(o.n, o.f64, o.dir, o.dev, o.maxr);
  }
};
std::mutex g_tw_mu;
std::map<TwKey, void*> g_tw;

dfft_status_t get_twiddles(int n, bool f64, int dir, int dev, const void** out, int maxr = 16) {
  std::lock_guard<std::mutex> lk(g_tw_mu);
  TwKey key{n, f64 ? 1 : 0, dir, dev, maxr};
  auto it = g_tw.find(key);
  if (it != g_tw.end()) {
    *out = it->second;
    return DFFT_SUCCESS;
  }
  int rad[kMaxPass];
  int np = length_schedule(n, rad, maxr);
  std::vector<long double> re, im;
  int ns = rad[0];
  for (int p = 1; p < np; ++p) {
    int R = rad[p];
    long long L = (long long)ns * R;
    for (int r = 1; r < R; ++r)
      for (int m = 0; m < ns; ++m) {
        long long e = ((long long)m * r) % L;
        long double a = 2.0L * 3.141592653589793238462643383279502884L * (long double)e / (long double)L;
        re.push_back(cosl(a));
        im.push_back((long double)dir * sinl(a));
      }
    ns *= R;
  }
  size_t cnt = std::max<size_t>(re.size(), 1);
  void* d = nullptr;
  size_t es = f64 ? 16 : 8;
  CU(cudaMalloc(&d, cnt * es));
  if (f64) {
    std::vector<double> h(2 * cnt, 0.0);
    for (size_t i = 0; i < re.size(); ++i) {
      h[2 * i] = (double)re[i];
      h[2 * i + 1] = (double)im[i];
    }
    CU(cudaMemcpy(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
  } else {
    std::vector<float> h(2 * cnt, 0.f);
    for (size_t i = 0; i < re.size(); ++i) {
      h[2 * i] = (float)re[i];
      h[2 * i + 1] = (float)im[i];
    }
    CU(cudaMemcpy(d, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
  }
  g_tw[key] = d;
  *out = d;
  return DFFT_SUCCESS;
}

std::atomic<long long> g_launches{0};  // library kernel launches, process-wide (dfft_kernel_launches)
bool g_use_tma = getenv("DFFT_NO_TMA") == nullptr;  // env switch for the A/B ablation
CUtensorMapL2promotion g_tma_promo = getenv("DFFT_TMA_PROMO256") ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                     : getenv("DFFT_TMA_PROMO128") ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                                   : CU_TENSOR_MAP_L2_PROMOTION_NONE;
bool g_tma_store = getenv("DFFT_NO_TMA_STORE") == nullptr;
bool g_use_bulk = getenv("DFFT_NO_BULK") == nullptr;  // bulk-copy epilogue for blocked segmented outputs

// R2C/C2R split twiddles: w^k = exp(dir·2πi·k/(2N)), k ∈ [0, N), long double once each.
dfft_status_t get_split_twiddles(int N, bool f64, int dir, int dev, const void** out) {
  std::lock_guard<std::mutex> lk(g_tw_mu);
  TwKey key{-N, f64 ? 1 : 0, dir, dev, 0};  // negative n: the split table of length N
  auto it = g_tw.find(key);
  if (it != g_tw.end()) {
    *out = it->second;
    return DFFT_SUCCESS;
  }
  void* d = nullptr;
  const size_t es = f64 ? 16 : 8;
  CU(cudaMalloc(&d, (size_t)N * es));
  std::vector<double> hd(2 * (size_t)N);
  std::vector<float> hf(2 * (size_t)N);
  for (int k = 0; k < N; ++k) {
    long double a = 2.0L * 3.141592653589793238462643383279502884L * (long double)k / (2.0L * N);
    hd[2 * k] = (double)cosl(a);
    hd[2 * k + 1] = (double)((long double)dir * sinl(a));
    hf[2 * k] = (float)cosl(a);
    hf[2 * k + 1] = (float)((long double)dir * sinl(a));
  }
  if (f64) CU(cudaMemcpy(d, hd.data(), (size_t)N * es, cudaMemcpyHostToDevice));
  else CU(cudaMemcpy(d, hf.data(), (size_t)N * es, cudaMemcpyHostToDevice));
  g_tw[key] = d;
  *out = d;
  return DFFT_SUCCESS;
}

inline bool is_contig(int family) { return family != kStrided && family != kStridedDct && family != kStridedDst; }

// R2R (DCT) post/pre twiddles: c_k = exp(dir·iπk/(2L)), k ∈ [0, L), long double once each.
dfft_status_t get_dct_twiddles(int L, bool f64, int dir, int dev, const void** out) {
  static std::map<TwKey, void*> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  TwKey key{L, f64, dir, dev, -2};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return DFFT_SUCCESS;
  }
  const size_t es = f64 ? 16 : 8;
  std::vector<unsigned char> h((size_t)L * es);
  for (int k = 0; k < L; ++k) {
    const long double a = (long double)dir * 3.14159265358979323846264338327950288L * (long double)k / (2.0L * L);
    const long double c = cosl(a), sn = sinl(a);
    if (f64) {
      reinterpret_cast<double*>(h.data())[2 * k] = (double)c;
      reinterpret_cast<double*>(h.data())[2 * k + 1] = (double)sn;
    } else {
      reinterpret_cast<float*>(h.data())[2 * k] = (float)c;
      reinterpret_cast<float*>(h.data())[2 * k + 1] = (float)sn;
    }
  }
  void* d = nullptr;
  CU(cudaSetDevice(dev));
  CU(cudaMalloc(&d, h.size()));
  CU(cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice));
  cache[key] = d;
  *out = d;
  return DFFT_SUCCESS;
}

// w_M^e = exp(dir·2πi·e/M), e < M, long double once each (the radix-8 z step of fft_xz8_kernel)
dfft_status_t get_root_twiddles(int M, bool f64, int dir, int dev, const void** out) {
  static std::map<TwKey, void*> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  TwKey key{M, f64, dir, dev, -3};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return DFFT_SUCCESS;
  }
  const size_t es = f64 ? 16 : 8;
  std::vector<unsigned char> h((size_t)M * es);
  for (int e = 0; e < M; ++e) {
    const long double a = 2.0L * 3.141592653589793238462643383279502884L * (long double)e / (long double)M;
    const long double c = cosl(a), sn = (long double)dir * sinl(a);
    if (f64) {
      reinterpret_cast<double*>(h.data())[2 * e] = (double)c;
      reinterpret_cast<double*>(h.data())[2 * e + 1] = (double)sn;
    } else {
      reinterpret_cast<float*>(h.data())[2 * e] = (float)c;
      reinterpret_cast<float*>(h.data())[2 * e + 1] = (float)sn;
    }
  }
  void* d = nullptr;
  CU(cudaSetDevice(dev));
  CU(cudaMalloc(&d, h.size()));
  CU(cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice));
  cache[key] = d;
  *out = d;
  return DFFT_SUCCESS;
}

dfft_status_t get_kernel(int family, int n, bool f64, int dir, KernelInfo* k) {
  bool ok = f64 ? lookup_kernel_f64(family, n, dir, k) : lookup_kernel_f32(family, n, dir, k);
  if (!ok) return fail(DFFT_ERR_UNSUPPORTED, "axis length %d not instantiated", n);
  if (k->smem > 48 * 1024) {
    CU(cudaFuncSetAttribute(k->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->smem));
    if (k->fn_tb) CU(cudaFuncSetAttribute(k->fn_tb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->smem));
    if (k->spec_fn) CU(cudaFuncSetAttribute(k->spec_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->smem));
  }
  if (k->tma_fn && k->tma_smem > 48 * 1024) {
    CU(cudaFuncSetAttribute(k->tma_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->tma_smem));
    if (k->tma_bk_fn) CU(cudaFuncSetAttribute(k->tma_bk_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->tma_smem));
    if (k->tma_st1_fn)
      CU(cudaFuncSetAttribute(k->tma_st1_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->tma_smem));
    if (k->tma_st_spec_fn)
      CU(cudaFuncSetAttribute(k->tma_st_spec_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->tma_smem));
  }
  if (k->tma_ip_fn && k->tma_ip_smem > 48 * 1024)
    CU(cudaFuncSetAttribute(k->tma_ip_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->tma_ip_smem));
  return DFFT_SUCCESS;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// ------------------------------------------------------------------------------ plan data
enum RefKind { kNone = 0, kUserIn = 1, kUserOut = 2, kWs = 3, kPeer = 4 };
struct Ref {
  int kind = kNone;
  long long off = 0;  // bytes
  int peer = -1;      // kPeer: global rank whose workspace (IPC window) this points into
};

struct Stage {
  int family = 0, n = 0, es = 8;
  KernelInfo k;
  PassArgs a{};
  Ref in, out;
  std::vector<Ref> in_bases, out_bases;  // table selector -> base (segmented sides)
  void* in_tab = nullptr;  // device longlong2[n] or null
  void* out_tab = nullptr;
  long long grid = 0;
  long long tma_grid = 0;  // persistent grid of the TMA variant (0 = not usable)
  int tma_occ = 0;         // resident CTAs per SM of the TMA variant
  int sm_cap = 0;          // > 0: run the persistent variant on at most this many SMs (leaves the
                           // rest to a concurrently running HBM-bound stage)
  int tma_variant = 0;     // 1 = the persistent TMA kernel is used
  long long ip_grid = 0;   // grid / resident CTAs of the in-place TMA-store variant (0 = not used)
  int ip_occ = 0;
  const void* tw_tma = nullptr;  // twiddles of the TMA variant's radix schedule
  bool empty = false;
  // last forward stage: which global axis (0 x, 1 y, 2 z) its t / l0 / l1 run along and the
  // rank's global offset of each (dfft_plan_set_poisson addresses the λ tables with them)
  bool last_fwd = false;
  int gax[3] = {0, 0, 0};
  long long glo[3] = {0, 0, 0};
};

struct Xfer {
  int peer;
  Ref ref;
  size_t bytes;
  Ref remote;  // CE mode (sends): the receiver's address, a kPeer reference into its window
  // CE mode: 2D copy (height rows of width bytes; source / destination pitches), height 1 = 1D
  size_t width = 0, height = 1, spitch = 0, dpitch = 0;
};
struct Exchange {
  int comm = 0;  // 0 = row (P1 group), 1 = column (P2 group)
  std::vector<Xfer> sends, recvs;     // NCCL mode: the blocks to move
  std::vector<int> peers;             // P2P / CE modes: global ranks of the other group members
  bool fused = false;                 // the producing FFT stored straight into the peers' windows
  bool empty() const { return sends.empty() && recvs.empty() && peers.empty(); }
};

// Flag words in every IPC window (CE / fused-store transports): READY[e][k][src] is set to 1 by
// producer src once its chunk-k blocks of exchange e have landed in this window; DONE[e][k][dst]
// is set to 1 by consumer dst once it has finished reading what this rank stored into dst's
// window (so the producer may overwrite it).  Each side resets the word it waited on back to 0
// (READY to 0, DONE to 0) in the same flag kernel that publishes its own signal, before the
// signal: the values every wait compares against are the constant 1, so a schedule captured in a
// CUDA graph replays correctly (DONE starts at 1 = "buffer free").
enum FlagArr { kReady = 0, kDone = 1 };
struct FlagRef {
  int arr, e, k;
  std::vector<int> ranks;  // wait / clear: the writers of the word (own window); set: the targets
};

// One step of a rank's execute.  The schedule is built once per plan (plan once,
// execute many) and interpreted by run_schedule; every rank of a plan has a schedule of the same
// length and shape, which is what lets simulated ranks issue them interleaved position by position.
enum OpKind { kOpLaunch, kOpWait, kOpSignal, kOpRecord, kOpStreamWait, kOpNccl, kOpCeCopy };
struct Op {
  int kind = kOpLaunch;
  int s = 0;       // stream: 0 = X (compute), 1 = Y (second compute / comm)
  int phase = 0;   // profiling phase (0 A, 1 E1, 2 B, 3 E2, 4 C)
  int chunk = 0;
  const Stage* st = nullptr;       // kOpLaunch
  const Exchange* x = nullptr;     // kOpNccl / kOpCeCopy
  FlagRef wait;                    // kOpWait
  std::vector<FlagRef> set, clr;   // kOpSignal
  int ev = -1;                     // kOpRecord / kOpStreamWait: schedule event index
};

struct RankPlan {
  int rank = 0, i = 0, j = 0;
  int64_t in_lo[3], in_n[3], out_lo[3], out_n[3];
  size_t in_bytes = 0, out_bytes = 0, ws_bytes = 0;
  void* ws = nullptr;
  std::vector<Stage> A, B;  // per chunk
  std::vector<Exchange> E1, E2;  // first / second exchange (each names its comm group)
  Stage C;
  std::vector<Stage> Cc;  // B→C pipelined plans (dfft_plan_s::bc): stage C per chunk, C unused
  std::vector<Op> sched;  // the execute, as built by build_schedule
  int nev = 0;            // schedule events
  cudaStream_t sX = nullptr, sY = nullptr;
  std::vector<cudaEvent_t> ev;
  cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
};

}  // namespace

struct dfft_comm_s {
  int nranks = 1, rank = 0, device = 0;
  bool sim = false;
  ncclComm_t world = nullptr;
  std::map<std::pair<int, int>, std::pair<ncclComm_t, ncclComm_t>> sub;  // (P1,P2) -> (row, col)
};

struct dfft_plan_s {
  dfft_comm_t comm = nullptr;
  int64_t nx = 0, ny = 0, nz = 0;
  int P1 = 1, P2 = 1, K = 1, dir = -1;
  bool f64 = false, r2c = false, overlap = true;
  bool r2r = false;  // real x axis transformed by a DCT / DST (reading R21, R22)
  int kind[3] = {0, 0, 0};  // per-axis transform kind (DFFT_KIND_*): DFT, DCT-II, DST-II
  size_t es = 8;  // complex element bytes
  std::vector<RankPlan> ranks;
  ncclComm_t row = nullptr, col = nullptr;
  // dfft_execute_host / _chain staging (kept on the chain's first plan): double-buffered device
  // copies of the host input and output, intermediate buffers between the chained plans, and
  // the two copy streams that let one call's device->host copy run beside the next call's
  // host->device copy
  struct HostChain {
    std::vector<dfft_plan_s*> plans;
    void* in_dev[2] = {nullptr, nullptr};
    void* out_dev[2] = {nullptr, nullptr};
    std::vector<void*> mid;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t in_ready[2] = {nullptr, nullptr}, in_free[2] = {nullptr, nullptr};
    cudaEvent_t out_ready[2] = {nullptr, nullptr}, out_done[2] = {nullptr, nullptr};
    unsigned long long calls = 0;
  };
  HostChain* host = nullptr;
  // executes replay a CUDA graph of the schedule, captured once per (in, out) pair on a private
  // stream (DFFT_NO_GRAPH=1: issue the schedule directly every time); invalidated by set_poisson
  struct GraphEntry {
    const void* in;
    void* out;
    cudaGraphExec_t exec;
    long long launches;  // library kernels in the graph (credited to dfft_kernel_launches per replay)
  };
  std::vector<GraphEntry> graphs;
  cudaStream_t cap_stream = nullptr;
  // P2P exchange (default for P > 1): every rank's workspace is an IPC window; the FFT epilogues
  // store straight into the peers' receive regions over NVLink; flags in the windows order it
  bool p2p = false;
  bool ce = false;                   // copy-engine exchange (cudaMemcpyAsync into the peers' windows)
  bool hybrid = false;               // CE, except the forward's first exchange: fused x-FFT stores
  // fused stores with both exchanges remote (P1 > 1 and P2 > 1): stage A runs whole and stages B
  // and C run in K chunks along the axis both leave local (x forward, z inverse), so the HBM-bound
  // C(k) overlaps the NVLink-bound B(k+1)
  bool bc = false;
  std::vector<void*> peer_ws;        // by global rank (own rank = own workspace), null if not a peer
  void* spec_tab = nullptr;          // dfft_plan_set_poisson: λ tables [nx | ny | nz] (Real)
  size_t flag_off = 0;               // byte offset of the flag block in every workspace
  unsigned long long hash = 0;       // resolved plan state (cross-rank consistency check)
  // failure state: an enqueue error, or the watchdog found an execute that did not complete (a
  // peer never signalled) and released its waits; the plan refuses further executes
  std::atomic<int> failed{0};
  std::string fail_msg;
  // per-phase profiling (dfft_plan_set_profiling): timing events around every stage launch
  // and exchange, on the stream that runs it; accumulated by dfft_plan_phase_times, and a
  // timeline of spans relative to each execute's origin event (dfft_plan_timeline)
  bool prof = false;
  struct ProfRec {
    int phase, stream, chunk, rank;
    size_t exec;
  };
  std::vector<cudaEvent_t> prof_ev;  // pool, pairs (start, stop)
  std::vector<ProfRec> prof_rec;     // one per recorded pair
  size_t prof_used = 0;              // pairs recorded since the last read
  std::vector<cudaEvent_t> prof_origin;  // one per execute since the last read
  size_t prof_nexec = 0;
  double prof_ms[5] = {0, 0, 0, 0, 0};
  long long prof_n[5] = {0, 0, 0, 0, 0};
  std::vector<dfft_span_t> prof_spans;  // resolved timeline spans not yet read
};

namespace {

// x lines are real (R2C/C2R, R2R): nx reals per line = nx/2 complex elements on the kernel side
inline bool xreal(const dfft_plan_s* pl) { return pl->r2c || pl->r2r; }
inline int fam_x_r2r(const dfft_plan_s* pl) { return pl->kind[0] == DFFT_KIND_DST2 ? kContigDst : kContigDct; }
inline int fam_x_fwd(const dfft_plan_s* pl) { return pl->r2c ? kContigR2C : pl->r2r ? fam_x_r2r(pl) : kContig; }
inline int fam_x_inv(const dfft_plan_s* pl) { return pl->r2c ? kContigC2R : pl->r2r ? fam_x_r2r(pl) : kContig; }
// strided stage along y (axis 1) or z (axis 2): the axis's kind picks the kernel family
inline int fam_axis(const dfft_plan_s* pl, int axis) {
  return pl->kind[axis] == DFFT_KIND_DCT2 ? kStridedDct : pl->kind[axis] == DFFT_KIND_DST2 ? kStridedDst : kStrided;
}
inline int fam_y(const dfft_plan_s* pl) { return fam_axis(pl, 1); }
inline int fam_z(const dfft_plan_s* pl) { return fam_axis(pl, 2); }

// ------------------------------------------------------------------------------ stage builders
dfft_status_t upload_table(const std::vector<longlong2>& h, void** d) {
  CU(cudaMalloc(d, h.size() * sizeof(longlong2)));
  CU(cudaMemcpy(*d, h.data(), h.size() * sizeof(longlong2), cudaMemcpyHostToDevice));
  return DFFT_SUCCESS;
}

// Affine segment of a side: t ∈ [tlo, tlo+tn) lives at bases[sel] + off0 + (t−tlo)·ts + l0·s0 + l1·s1.
struct Seg {
  int sel;
  long long tlo, tn, off0, ts, s0, s1;
};
using Segs = std::vector<Seg>;

// per-t table {sel<<56 | off(t), s0 | s1<<32} (the kernel's SegEnt)
std::vector<longlong2> seg_table(const Segs& segs, long long n) {
  for (const Seg& q : segs) n = std::max(n, q.tlo + q.tn);  // R2C/C2R sides carry N+1 bins
  std::vector<longlong2> tab(n);
  for (const Seg& q : segs)
    for (long long t = q.tlo; t < q.tlo + q.tn; ++t) {
      longlong2 e;
      e.x = ((long long)q.sel << 56) | (q.off0 + (t - q.tlo) * q.ts);
      e.y = (long long)((unsigned long long)(unsigned int)q.s0 | ((unsigned long long)(unsigned int)q.s1 << 32));
      tab[t] = e;
    }
  return tab;
}

// One segment covering all t (one owner, e.g. P2 == 1), or adjacent segments that happen to be
// one affine map, make the side unsegmented: no table, closed-form addressing.
bool linearize(const Segs& segs, long long n, Ref& base, const std::vector<Ref>& bases, SideMap& m, long long es) {
  if (segs.empty()) return false;
  const Seg& f = segs[0];
  for (const Seg& q : segs)
    if (q.sel != f.sel || q.s0 != f.s0 || q.s1 != f.s1 || q.ts != f.ts || q.off0 != f.off0 + (q.tlo - f.tlo) * f.ts)
      return false;
  (void)n;
  Ref b = bases[f.sel];
  b.off += (f.off0 - f.tlo * f.ts) * es;
  base = b;
  m.tstride = f.ts;
  m.s0 = f.s0;
  m.s1 = f.s1;
  return true;
}

// tile-group width of a persistent strided stage (PassArgs::g0), overridable for A/B runs
int tile_g0(int dflt, const char* env) {
  const char* v = getenv(env);
  return v ? atoi(v) : dflt;
}

// Segments of equal width B (unit t-stride, one base, same line strides) laid end to end at a
// constant block stride: an unsegmented t-blocked side (SideMap::tb), no per-t table.
bool linearize_tblocked(const Segs& segs, Ref& base, const std::vector<Ref>& bases, SideMap& m, long long es) {
  if (segs.size() < 2) return false;
  const Seg& f = segs[0];
  const long long B = f.tn, BS = segs[1].off0 - f.off0;
  if (f.tlo != 0 || B <= 0 || B > (1 << 30)) return false;
  for (size_t q = 0; q < segs.size(); ++q) {
    const Seg& g = segs[q];
    if (g.sel != f.sel || g.s0 != f.s0 || g.s1 != f.s1 || g.ts != 1 || g.tn != B || g.tlo != (long long)q * B ||
        g.off0 != f.off0 + (long long)q * BS)
      return false;
  }
  Ref b = bases[f.sel];
  b.off += f.off0 * es;
  base = b;
  m.tstride = 1;
  m.s0 = f.s0;
  m.s1 = f.s1;
  m.tb = (int)B;
  m.tbs = BS;
  return true;
}

inline void set_side(SideMap& m, long long ts, long long s0, long long s1) {
  m.tstride = ts;
  m.s0 = s0;
  m.s1 = s1;
}

dfft_status_t finish_stage(dfft_plan_t pl, Stage& s, int family, int n, long long L0, long long L1,
                           const Segs* in_segs, const Segs* out_segs) {
  if (s.in_bases.empty()) s.in_bases = {s.in};
  if (s.out_bases.empty()) s.out_bases = {s.out};
  if (s.in_bases.size() > (size_t)kMaxBases || s.out_bases.size() > (size_t)kMaxBases)
    return fail(DFFT_ERR_UNSUPPORTED, "more than %d segment bases", kMaxBases);
  if (in_segs && linearize(*in_segs, n, s.in, s.in_bases, s.a.in, (long long)pl->es)) in_segs = nullptr;
  if (in_segs && family == kContig && !getenv("DFFT_NO_TBLOCK") && length_specialised(n) &&
      linearize_tblocked(*in_segs, s.in, s.in_bases, s.a.in, (long long)pl->es))
    in_segs = nullptr;
  if (out_segs && linearize(*out_segs, n, s.out, s.out_bases, s.a.out, (long long)pl->es)) out_segs = nullptr;
  if (is_contig(family) && family != kContigXZ8 &&
      ((!in_segs && s.a.in.tstride != 1) || (!out_segs && s.a.out.tstride != 1)))
    return fail(DFFT_ERR_INTERNAL, "contig stage with a non-unit t-stride side");
  std::vector<longlong2> in_tab_h, out_tab_h;
  if (in_segs) in_tab_h = seg_table(*in_segs, n);
  if (out_segs) out_tab_h = seg_table(*out_segs, n);
  const std::vector<longlong2>* in_tab = in_segs ? &in_tab_h : nullptr;
  const std::vector<longlong2>* out_tab = out_segs ? &out_tab_h : nullptr;
  s.family = family;
  s.n = n;
  s.es = (int)pl->es;
  s.a.L0 = L0;
  s.a.L1 = L1;
  if (L0 <= 0 || L1 <= 0) {
    s.empty = true;
    return DFFT_SUCCESS;
  }
  ST(get_kernel(family, n, pl->f64, pl->dir, &s.k));
  // x-FFTs of plans whose T1 exchange crosses ranks (P1 > 1): radix-16 passes.  Their epilogue
  // (forward) stores into peers' windows, where the radix-32 kernel's fewer, wider threads keep
  // fewer stores in flight, and the inverse runs beside the NVLink-bound y-IFFT (r02, 1024³ at
  // 2×2: fwd x 1.53 -> 1.65 ms, inverse y-IFFT 0.48 -> 0.66 ms a chunk with radix 32)
  if (family == kContig && s.k.r16_fn && pl->P1 > 1 && !getenv("DFFT_CONTIG_R32")) {
    s.k.fn = s.k.r16_fn;
    s.k.fn_tb = s.k.r16_fn_tb;
    s.k.threads = s.k.r16_threads;
    s.k.per_cta = s.k.r16_per_cta;
    s.k.smem = s.k.r16_smem;
    s.k.tma_maxr = 16;
    if (s.k.smem > 48 * 1024) {
      CU(cudaFuncSetAttribute(s.k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s.k.smem));
      CU(cudaFuncSetAttribute(s.k.fn_tb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s.k.smem));
    }
  }
  ST(get_twiddles(n, pl->f64, pl->dir, pl->comm->device, &s.a.tw, is_contig(family) ? s.k.tma_maxr : 16));
  if (s.k.generic) {  // the radix schedule at run time
    s.a.gen = make_sched(n);
    s.a.gen_per = s.k.per_cta;
  }
  const bool contig_r2r = family == kContigDct || family == kContigDst;
  if (family == kContigR2C || family == kContigC2R || contig_r2r)
    ST(get_split_twiddles(n, pl->f64, pl->dir, pl->comm->device, &s.a.tw2));
  if (contig_r2r || family == kStridedDct || family == kStridedDst)  // c_k over the real line length L
    ST(get_dct_twiddles(contig_r2r ? 2 * n : n, pl->f64, pl->dir, pl->comm->device, &s.a.tw3));
  if (in_tab) ST(upload_table(*in_tab, &s.in_tab));
  if (out_tab) ST(upload_table(*out_tab, &s.out_tab));
  s.a.in.ttab = (const SegEnt*)s.in_tab;
  s.a.out.ttab = (const SegEnt*)s.out_tab;
  // bulk epilogue: a column-blocked segmented output whose block is the TMA tile (each segment
  // of a tile is then one contiguous run of tn·W elements)
  if (family == kStrided && out_segs && s.k.tma_bk_fn && g_use_bulk && s.a.out.bw == s.k.tma_w &&
      out_segs->size() <= (size_t)kMaxBulk) {
    const long long es = (long long)pl->es;
    bool ok = (s.a.out.mT * 1) > 0;
    for (const Seg& q : *out_segs)
      ok = ok && q.ts == s.a.out.bw && q.s0 == 1 && (q.off0 * es) % 16 == 0 && (q.s1 * es) % 16 == 0 &&
           q.tn < (1LL << 30);
    if (ok) {
      s.a.out.nbulk = (int)out_segs->size();
      for (size_t q = 0; q < out_segs->size(); ++q) {
        const Seg& g = (*out_segs)[q];
        s.a.out.bulk[q] = BulkSeg{g.off0, g.s1, (int)g.tlo, (int)g.tn, g.sel};
      }
    }
  }
  // contig: walk lines so that consecutive CTAs write adjacent lines (unsegmented outputs)
  if (is_contig(family) && family != kContigXZ8 && !out_tab && !getenv("DFFT_LORDER0") && s.a.out.bw == 0 && L1 > 1 &&
      std::llabs(s.a.out.s1) < std::llabs(s.a.out.s0))
    s.a.lorder = 1;
  if (is_contig(family)) s.grid = (L0 * L1 + s.k.per_cta - 1) / s.k.per_cta;
  else s.grid = ((L0 + s.k.per_cta - 1) / s.k.per_cta) * L1;
  if (s.grid >= (1LL << 31)) return fail(DFFT_ERR_UNSUPPORTED, "grid too large (%lld CTAs)", s.grid);
  if ((family == kStrided || family == kStridedDct || family == kStridedDst) && s.k.tma_fn && g_use_tma && !in_tab &&
      tensor_map_encoder()) {
    const long long es = (long long)pl->es;
    bool ok = s.a.in.s0 == 1 && (s.a.in.tstride * es) % 16 == 0 && (L1 == 1 || (s.a.in.s1 * es) % 16 == 0) &&
              2 * L0 < (1LL << 32) && L1 < (1LL << 31);
    if (s.a.in.bw > 0) ok = ok && s.k.tma_fn && s.a.in.bw % s.k.tma_w == 0 && (s.a.in.mT * s.a.in.s1 * es) % 16 == 0;
    if (ok) {
      const void* fn = s.k.tma_fn;
      const int thr = s.k.tma_threads, w = s.k.tma_w;
      const size_t sm = s.k.tma_smem;
      int occ = 0, dev = pl->comm->device, sms = 0;
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, thr, sm));
      CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      long long tiles = ((L0 + w - 1) / w) * L1;
      if (occ > 0) {
        s.tma_variant = 1;
        s.tma_grid = std::min<long long>(tiles, (long long)sms * occ);
        s.tma_occ = occ;
      }
      if (s.tma_variant == 1 && s.k.tma_ip_fn && !(getenv("DFFT_TMA_IP") && atoi(getenv("DFFT_TMA_IP")) == 0)) {
        int occ_ip = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_ip, s.k.tma_ip_fn, thr, s.k.tma_ip_smem));
        if (occ_ip > 0) {
          s.ip_grid = std::min<long long>(tiles, (long long)sms * occ_ip);
          s.ip_occ = occ_ip;
        }
      }
      if (s.tma_variant == 1)  // the TMA variant's own radix schedule
        ST(get_twiddles(n, pl->f64, pl->dir, pl->comm->device, &s.tw_tma, s.k.tma_maxr));
      if (getenv("DFFT_DEBUG"))
        fprintf(stderr, "dfft: strided n=%d L0=%lld L1=%lld tma grid %lld (occ %d)\n", n, L0, L1, s.tma_grid, occ);
    }
  }
  return DFFT_SUCCESS;
}

struct Geo {
  long long nx, ny, nz, nxc;
  long long P1, P2, K;
  long long wy = 1, wz = 1;  // column-tile widths of the strided kernels for ny / nz (blocked layouts)
  long long Xlo(long long i) const { return blo(nxc, P1, i); }
  long long Xn(long long i) const { return blk(nxc, P1, i); }
  long long Y1lo(long long i) const { return blo(ny, P1, i); }
  long long Y1n(long long i) const { return blk(ny, P1, i); }
  long long Zlo(long long j) const { return blo(nz, P2, j); }
  long long Zn(long long j) const { return blk(nz, P2, j); }
  long long Y3lo(long long j) const { return blo(ny, P2, j); }
  long long Y3n(long long j) const { return blk(ny, P2, j); }
  // forward chunks along local z of rank column j; inverse chunks along local x of row i
  long long zc(long long j, long long k) const { return blk(Zn(j), K, k); }
  long long z0(long long j, long long k) const { return blo(Zn(j), K, k); }
  // (xq > 1: inverse chunk bounds at multiples of xq, the column-block width of the fused-store
  // windows, so a chunk is a whole number of blocks)
  long long xq = 1;
  long long x0(long long i, long long k) const {
    const long long nb = (Xn(i) + xq - 1) / xq;
    return std::min(Xn(i), blo(nb, K, k) * xq);
  }
  long long xc(long long i, long long k) const { return (k + 1 < K ? x0(i, k + 1) : Xn(i)) - x0(i, k); }
};

// Group members as global ranks: row group = same j (index i'), column group = same i (index j').
inline int row_rank(const Geo& g, long long ip, long long j) { return (int)(ip * g.P2 + j); }
inline int col_rank(const Geo& g, long long i, long long jp) { return (int)(i * g.P2 + jp); }

// Flag block at the end of every workspace (CE / fused modes): uint32 ready[2][K][P], done[2][K][P].
// ready[e][k][src] is written by src into the consumer's window once its chunk-k blocks have
// landed there; done[e][k][dst] is written by the consumer dst into the producer's window once
// it has finished reading (so the next execute may overwrite).
inline size_t flag_bytes(const Geo& g) { return (size_t)4 * 2 * 2 * g.K * g.P1 * g.P2; }

// Workspace layouts (complex elements) of rank (i, j); every rank can compute any other rank's
// layout, which is how senders address the receivers' windows.
//   forward  NCCL: [S1 send1 | R1 recv1 [y][zc][x] per chunk | S2 send2]     (E2 lands in `out`)
//            CE:   [S1 send1 | R1 recv1 [zc][y][x] per chunk | S2 send2 | R2 [y'][z][x]]
//            P2P:  [R1 recv1 [zc][y][x] per chunk | R2 [y'][z][x]]           (no send blocks)
//   inverse  NCCL/CE: [S2' | R2' [y][z][xc] per chunk | S1' | R1' blocks by (source row, chunk)]
//            P2P:  [R2' | R1']
// CE/P2P layouts put the FFT axis of the *consumer* at a small stride, so no stage both reads
// and writes at a large stride (such a stage ran at 2.3 TB/s vs 4.6-6 TB/s).
struct FwdLayout {
  long long S1, R1, S2, R2, end;
};
inline long long round_up(long long a, long long b) { return (a + b - 1) / b * b; }

FwdLayout fwd_layout(const Geo& g, long long i, long long j, int mode /*0 nccl 1 ce 2 p2p 3 hybrid*/) {
  FwdLayout L{};
  const long long Xn = g.Xn(i), Y1n = g.Y1n(i), Zn = g.Zn(j), Y3n = g.Y3n(j);
  if (mode == 2) {  // fused: [R1 recv1 [zc][y][x] | R2 column-blocked [xt][z][y'][wy]]
    L.S1 = L.R1 = 0;
    L.S2 = L.R2 = g.ny * Zn * Xn;
    L.end = L.R2 + round_up(Xn, g.wy) * g.nz * Y3n;
    return L;
  }
  const long long S1n = (mode == 2 || mode == 3) ? 0 : Y1n * Zn * (g.nxc - Xn);
  const long long S2n = mode == 2 ? 0 : Zn * Xn * (g.ny - Y3n);
  L.S1 = 0;
  L.R1 = S1n;
  L.S2 = L.R1 + g.ny * Zn * Xn;
  L.R2 = L.S2 + S2n;
  L.end = L.R2 + (mode == 0 ? 0 : g.nz * Y3n * Xn);
  return L;
}
struct InvLayout {
  long long S2, R2, S1, R1, end;
};
InvLayout inv_layout(const Geo& g, long long i, long long j, int mode) {
  InvLayout L{};
  const long long Xn = g.Xn(i), Y1n = g.Y1n(i), Zn = g.Zn(j), Y3n = g.Y3n(j);
  if (mode == 2) {  // fused: [R2' blocked [xt][y][z][wz] | R1' blocked per source [i][xt][z][y][wy]]
    L.S2 = L.R2 = 0;
    L.S1 = L.R1 = round_up(Xn, g.wz) * g.ny * Zn;
    long long r1 = 0;
    for (long long q = 0; q < g.P1; ++q) r1 += round_up(g.Xn(q), g.wy) * Zn * Y1n;
    L.end = L.R1 + r1;
    return L;
  }
  L.S2 = 0;
  L.R2 = mode == 2 ? 0 : Y3n * Xn * (g.nz - Zn);
  L.S1 = L.R2 + g.ny * Zn * Xn;
  L.R1 = L.S1 + (mode == 2 ? 0 : Zn * Xn * (g.ny - Y1n));
  L.end = L.R1 + g.nxc * Y1n * Zn;
  return L;
}

int exch_mode(dfft_plan_t pl) { return pl->p2p ? 2 : pl->hybrid ? 3 : pl->ce ? 1 : 0; }

// The flag block sits at the same byte offset in every rank's window (peers write into it at
// their own idea of the offset): after the largest rank's data region.
void add_flags(dfft_plan_t pl, const Geo& g, RankPlan& rp, long long end_elems, bool forward) {
  rp.ws_bytes = (size_t)end_elems * pl->es;
  if (pl->p2p || pl->ce) {
    long long mx = 0;
    const int mode = (!forward && exch_mode(pl) == 3) ? 1 : exch_mode(pl);
    for (long long i = 0; i < g.P1; ++i)
      for (long long j = 0; j < g.P2; ++j)
        mx = std::max(mx, forward ? fwd_layout(g, i, j, mode).end : inv_layout(g, i, j, mode).end);
    pl->flag_off = ((size_t)mx * pl->es + 255) / 256 * 256;
    rp.ws_bytes = pl->flag_off + flag_bytes(g);
  }
}

// Forward plan of one rank: x-FFT (D1 in) → T1 → y-FFT → T2 → z-FFT (D3 out).
dfft_status_t build_forward(dfft_plan_t pl, const Geo& g, RankPlan& rp) {
  const long long i = rp.i, j = rp.j, K = g.K, es = (long long)pl->es;
  const long long Xn = g.Xn(i), Y1n = g.Y1n(i), Zn = g.Zn(j), Y3n = g.Y3n(j);
  const int mode = exch_mode(pl);
  // per exchange: E1 fused (P2P, hybrid) or packed; E2 fused (P2P) or packed (NCCL, CE, hybrid)
  const bool nccl = mode == 0, p2p = mode == 2, hyb = mode == 3, ce = mode == 1 || hyb;
  const bool f1 = p2p || hyb;
  const FwdLayout L = fwd_layout(g, i, j, mode);
  add_flags(pl, g, rp, L.end, true);
  auto s1off = [&](long long k, long long ip) {  // send1 block (k, i'): [zz][y][x_i'] (NCCL: [y][zz][x])
    long long acc = 0;
    for (long long q = 0; q < ip; ++q)
      if (q != i) acc += g.Xn(q);
    return L.S1 + Y1n * (g.z0(j, k) * (g.nxc - Xn) + g.zc(j, k) * acc);
  };
  auto s2off = [&](long long k, long long jp) {  // send2 block (k, j'): NCCL [zz][y'][x], CE [y'][zz][x]
    long long acc = 0;
    for (long long q = 0; q < jp; ++q)
      if (q != j) acc += g.Y3n(q);
    return L.S2 + Xn * (g.z0(j, k) * (g.ny - Y3n) + g.zc(j, k) * acc);
  };
  const long long nxl = xreal(pl) ? g.nx / 2 : g.nx;  // input line length in (complex) elements
  const long long in_es = xreal(pl) ? es / 2 : es;
  rp.A.resize(K);
  rp.B.resize(K);
  rp.E1.resize(K);
  rp.E2.resize(K);
  for (long long k = 0; k < K; ++k) {
    const long long zc = g.zc(j, k), z0 = g.z0(j, k);
    // ---- stage A: x-FFT of lines (l0 = y, l1 = zz); out segmented by x-owner i'
    Stage& A = rp.A[k];
    A.in = {kUserIn, z0 * Y1n * g.nx * in_es};
    set_side(A.a.in, 1, nxl, Y1n * nxl);
    A.out = {kWs, 0};
    A.out_bases.push_back({kWs, 0});
    if (f1)  // selector 1 + i' = rank (i', j)'s window (own window for i' == i)
      for (long long ip = 0; ip < g.P1; ++ip) A.out_bases.push_back({kPeer, 0, row_rank(g, ip, j)});
    Segs aseg;
    for (long long ip = 0; ip < g.P1; ++ip) {
      const long long xl = g.Xlo(ip), xn = g.Xn(ip);
      if (f1) {
        const FwdLayout Lr = fwd_layout(g, ip, j, mode);
        aseg.push_back({1 + (int)ip, xl, xn, Lr.R1 + g.ny * z0 * xn + g.Y1lo(i) * xn, 1, xn, g.ny * xn});
      } else if (ip == i) {
        if (nccl) aseg.push_back({0, xl, xn, L.R1 + g.ny * z0 * Xn + g.Y1lo(i) * zc * Xn, 1, zc * Xn, Xn});
        else aseg.push_back({0, xl, xn, L.R1 + g.ny * z0 * Xn + g.Y1lo(i) * Xn, 1, Xn, g.ny * Xn});
      } else {
        if (nccl) aseg.push_back({0, xl, xn, s1off(k, ip), 1, zc * xn, xn});
        else aseg.push_back({0, xl, xn, s1off(k, ip), 1, xn, Y1n * xn});
      }
    }
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, fam_x_fwd(pl), (int)nxl, Y1n, zc, nullptr, &aseg));
    // ---- exchange 1 (row group)
    Exchange& E1 = rp.E1[k];
    E1.comm = 0;
    E1.fused = f1;
    for (long long ip = 0; ip < g.P1; ++ip) {
      if (ip == i) continue;
      if (!nccl) E1.peers.push_back(row_rank(g, ip, j));
      if (f1) continue;
      const long long xn = g.Xn(ip);
      Xfer x{(int)ip, {kWs, s1off(k, ip) * es}, (size_t)(Y1n * zc * xn * es)};
      if (ce) {  // zc rows of Y1n·xn elements into [zz][y][x] of the receiver
        const FwdLayout Lr = fwd_layout(g, ip, j, mode);
        x.remote = {kPeer, (Lr.R1 + g.ny * z0 * xn + g.Y1lo(i) * xn) * es, row_rank(g, ip, j)};
        x.width = (size_t)(Y1n * xn * es);
        x.height = (size_t)zc;
        x.spitch = x.width;
        x.dpitch = (size_t)(g.ny * xn * es);
      }
      E1.sends.push_back(x);
      E1.recvs.push_back({(int)ip, {kWs, (L.R1 + g.ny * z0 * Xn + g.Y1lo(ip) * zc * Xn) * es},
                          (size_t)(g.Y1n(ip) * zc * Xn * es)});
    }
    // ---- stage B: y-FFT of columns (l0 = x, l1 = zz) of recv1 chunk k; out segmented by y-owner j'
    Stage& B = rp.B[k];
    B.in = {kWs, (L.R1 + g.ny * z0 * Xn) * es};
    if (nccl) set_side(B.a.in, zc * Xn, 1, Xn);
    else set_side(B.a.in, Xn, 1, g.ny * Xn);
    B.out = {kWs, 0};
    B.out_bases.push_back({kWs, 0});
    B.out_bases.push_back({kUserOut, 0});
    if (p2p)  // selector 2 + j' = rank (i, j')'s window
      for (long long jp = 0; jp < g.P2; ++jp) B.out_bases.push_back({kPeer, 0, col_rank(g, i, jp)});
    Segs bseg;
    for (long long jp = 0; jp < g.P2; ++jp) {
      const long long yl = g.Y3lo(jp), yn = g.Y3n(jp);
      if (p2p) {  // receiver's R2 [xt][z][y'][wy]: a warp's rows of one block are contiguous
        const FwdLayout Lr = fwd_layout(g, i, jp, mode);
        bseg.push_back({2 + (int)jp, yl, yn, Lr.R2 + (g.Zlo(j) + z0) * yn * g.wy, g.wy, 1, yn * g.wy});
      } else if (jp == j) {
        if (nccl) bseg.push_back({1, yl, yn, (g.Zlo(j) + z0) * Y3n * Xn, Xn, 1, Y3n * Xn});
        else bseg.push_back({0, yl, yn, L.R2 + (g.Zlo(j) + z0) * Xn, g.nz * Xn, 1, Xn});
      } else {
        if (nccl) bseg.push_back({0, yl, yn, s2off(k, jp), Xn, 1, yn * Xn});
        else bseg.push_back({0, yl, yn, s2off(k, jp), zc * Xn, 1, Xn});
      }
    }
    if (p2p) {
      B.a.out.bw = (int)g.wy;
      B.a.out.mT = g.nz;
    }
    B.a.scale = 1.0;
    ST(finish_stage(pl, B, fam_y(pl), (int)g.ny, Xn, zc, nullptr, &bseg));
    // ---- exchange 2 (column group)
    Exchange& E2 = rp.E2[k];
    E2.comm = 1;
    E2.fused = p2p;
    for (long long jp = 0; jp < g.P2; ++jp) {
      if (jp == j) continue;
      if (!nccl) E2.peers.push_back(col_rank(g, i, jp));
      if (p2p) continue;
      const long long yn = g.Y3n(jp);
      Xfer x{(int)jp, {kWs, s2off(k, jp) * es}, (size_t)(zc * yn * Xn * es)};
      if (ce) {  // yn rows of zc·Xn elements into [y'][z][x] of the receiver
        const FwdLayout Lr = fwd_layout(g, i, jp, mode);
        x.remote = {kPeer, (Lr.R2 + (g.Zlo(j) + z0) * Xn) * es, col_rank(g, i, jp)};
        x.width = (size_t)(zc * Xn * es);
        x.height = (size_t)yn;
        x.spitch = x.width;
        x.dpitch = (size_t)(g.nz * Xn * es);
      }
      E2.sends.push_back(x);
      E2.recvs.push_back({(int)jp, {kUserOut, (g.Zlo(jp) + g.z0(jp, k)) * Y3n * Xn * es},
                          (size_t)(g.zc(jp, k) * Y3n * Xn * es)});
    }
  }
  // ---- stage C: z-FFT of columns (l0 = x, l1 = y'): in place on `out` (NCCL), R2 -> `out` (CE/P2P)
  Stage& C = rp.C;
  C.out = {kUserOut, 0};
  set_side(C.a.out, Y3n * Xn, 1, Xn);
  if (nccl) {
    C.in = {kUserOut, 0};
    set_side(C.a.in, Y3n * Xn, 1, Xn);
  } else if (p2p) {  // R2 [xt][z][y'][wy]
    C.in = {kWs, L.R2 * es};
    set_side(C.a.in, Y3n * g.wy, 1, g.wy);
    C.a.in.bw = (int)g.wy;
    C.a.in.mT = g.nz * Y3n;
    // blocked input (adjacent y' adjacent) vs natural output (adjacent x adjacent): groups of 4
    // column tiles give 256 B output pieces and ~(#CTAs/4)·64 B input runs
    C.a.g0 = tile_g0(4, "DFFT_G0_FWD_C");
  } else {
    C.in = {kWs, L.R2 * es};
    set_side(C.a.in, Xn, 1, g.nz * Xn);
  }
  C.a.scale = 1.0;
  C.last_fwd = true;  // t = z, l0 = x, l1 = y
  C.gax[0] = 2, C.gax[1] = 0, C.gax[2] = 1;
  C.glo[1] = g.Xlo(i), C.glo[2] = g.Y3lo(j);
  ST(finish_stage(pl, C, fam_z(pl), (int)g.nz, Xn, Y3n, nullptr, nullptr));
  return DFFT_SUCCESS;
}

// Fused-store plan with the B→C pipeline, forward (both exchanges remote).  Stage A (x-FFT) runs
// whole and stores into the row peers' R1 [z][y][x]; stage B (y-FFT) and C (z-FFT) run in K
// chunks of whole column blocks along x: B(k) stores its columns into the column peers' R2
// [xt][z][y'][wy] and C(k) transforms them once every column peer has signalled chunk k.
dfft_status_t build_forward_bc(dfft_plan_t pl, const Geo& g, RankPlan& rp) {
  const long long i = rp.i, j = rp.j, K = g.K, es = (long long)pl->es;
  const long long Xn = g.Xn(i), Y1n = g.Y1n(i), Zn = g.Zn(j), Y3n = g.Y3n(j);
  const FwdLayout L = fwd_layout(g, i, j, 2);
  add_flags(pl, g, rp, L.end, true);
  const long long nxl = xreal(pl) ? g.nx / 2 : g.nx;
  rp.A.resize(K);
  rp.B.resize(K);
  rp.E1.resize(K);
  rp.E2.resize(K);
  rp.Cc.resize(K);
  // ---- stage A (whole): x-FFT of lines (l0 = y, l1 = z); out segmented by x-owner i'
  Stage& A = rp.A[0];
  A.in = {kUserIn, 0};
  set_side(A.a.in, 1, nxl, Y1n * nxl);
  A.out = {kWs, 0};
  A.out_bases.push_back({kWs, 0});
  for (long long ip = 0; ip < g.P1; ++ip) A.out_bases.push_back({kPeer, 0, row_rank(g, ip, j)});
  Segs aseg;
  for (long long ip = 0; ip < g.P1; ++ip) {
    const long long xn = g.Xn(ip);
    const FwdLayout Lr = fwd_layout(g, ip, j, 2);
    aseg.push_back({1 + (int)ip, g.Xlo(ip), xn, Lr.R1 + g.Y1lo(i) * xn, 1, xn, g.ny * xn});
  }
  A.a.scale = 1.0;
  ST(finish_stage(pl, A, fam_x_fwd(pl), (int)nxl, Y1n, Zn, nullptr, &aseg));
  for (long long k = 1; k < K; ++k) rp.A[k].empty = true;
  rp.E1[0].comm = 0;
  rp.E1[0].fused = true;
  for (long long ip = 0; ip < g.P1; ++ip)
    if (ip != i) rp.E1[0].peers.push_back(row_rank(g, ip, j));
  for (long long k = 0; k < K; ++k) {
    const long long x0 = g.x0(i, k), xc = g.xc(i, k);
    // ---- stage B(k): y-FFT of columns (l0 = x - x0, l1 = z) of R1; out to the column peers' R2
    Stage& B = rp.B[k];
    B.in = {kWs, (L.R1 + x0) * es};
    set_side(B.a.in, Xn, 1, g.ny * Xn);
    B.out = {kWs, 0};
    B.out_bases.push_back({kWs, 0});
    B.out_bases.push_back({kUserOut, 0});
    for (long long jp = 0; jp < g.P2; ++jp) B.out_bases.push_back({kPeer, 0, col_rank(g, i, jp)});
    Segs bseg;
    for (long long jp = 0; jp < g.P2; ++jp) {
      const long long yn = g.Y3n(jp);
      const FwdLayout Lr = fwd_layout(g, i, jp, 2);
      bseg.push_back({2 + (int)jp, g.Y3lo(jp), yn, Lr.R2 + x0 * g.nz * yn + g.Zlo(j) * yn * g.wy, g.wy, 1, yn * g.wy});
    }
    B.a.out.bw = (int)g.wy;
    B.a.out.mT = g.nz;
    B.a.scale = 1.0;
    ST(finish_stage(pl, B, fam_y(pl), (int)g.ny, xc, Zn, nullptr, &bseg));
    Exchange& E2 = rp.E2[k];
    E2.comm = 1;
    E2.fused = true;
    for (long long jp = 0; jp < g.P2; ++jp)
      if (jp != j) E2.peers.push_back(col_rank(g, i, jp));
    // ---- stage C(k): z-FFT of columns (l0 = x - x0, l1 = y') of R2 chunk k -> `out`
    Stage& C = rp.Cc[k];
    C.in = {kWs, (L.R2 + x0 * g.nz * Y3n) * es};
    set_side(C.a.in, Y3n * g.wy, 1, g.wy);
    C.a.in.bw = (int)g.wy;
    C.a.in.mT = g.nz * Y3n;
    C.a.g0 = tile_g0(4, "DFFT_G0_FWD_C");
    C.out = {kUserOut, x0 * es};
    set_side(C.a.out, Y3n * Xn, 1, Xn);
    C.a.scale = 1.0;
    C.last_fwd = true;  // t = z, l0 = x - x0, l1 = y
    C.gax[0] = 2, C.gax[1] = 0, C.gax[2] = 1;
    C.glo[1] = g.Xlo(i) + x0, C.glo[2] = g.Y3lo(j);
    ST(finish_stage(pl, C, fam_z(pl), (int)g.nz, xc, Y3n, nullptr, nullptr));
  }
  return DFFT_SUCCESS;
}

// Inverse counterpart (both exchanges remote): stage A (z-IFFT) whole into the column peers' R2'
// [xt][y][z][wz]; stage B (y-IFFT) and C (x-IFFT, ×1/N) in K chunks along local z: B(k) stores
// into the row peers' R1' [source i][xt][z][y][wy], C(k) reads the chunk from every source.
dfft_status_t build_inverse_bc(dfft_plan_t pl, const Geo& g, RankPlan& rp) {
  const long long i = rp.i, j = rp.j, K = g.K, es = (long long)pl->es;
  const long long Xn = g.Xn(i), Y1n = g.Y1n(i), Zn = g.Zn(j), Y3n = g.Y3n(j);
  const InvLayout L = inv_layout(g, i, j, 2);
  add_flags(pl, g, rp, L.end, false);
  const long long nxl = xreal(pl) ? g.nx / 2 : g.nx;
  rp.A.resize(K);
  rp.B.resize(K);
  rp.E1.resize(K);
  rp.E2.resize(K);
  rp.Cc.resize(K);
  // ---- stage A (whole): z-IFFT of columns (l0 = x, l1 = y') of `in`; out to the column peers' R2'
  Stage& A = rp.A[0];
  A.in = {kUserIn, 0};
  set_side(A.a.in, Y3n * Xn, 1, Xn);
  A.out = {kWs, 0};
  A.out_bases.push_back({kWs, 0});
  for (long long jp = 0; jp < g.P2; ++jp) A.out_bases.push_back({kPeer, 0, col_rank(g, i, jp)});
  Segs aseg;
  for (long long jp = 0; jp < g.P2; ++jp) {
    const long long zn = g.Zn(jp);
    const InvLayout Lr = inv_layout(g, i, jp, 2);
    aseg.push_back({1 + (int)jp, g.Zlo(jp), zn, Lr.R2 + g.Y3lo(j) * zn * g.wz, g.wz, 1, zn * g.wz});
  }
  A.a.out.bw = (int)g.wz;
  A.a.out.mT = g.ny;
  A.a.scale = 1.0;
  ST(finish_stage(pl, A, fam_z(pl), (int)g.nz, Xn, Y3n, nullptr, &aseg));
  for (long long k = 1; k < K; ++k) rp.A[k].empty = true;
  rp.E1[0].comm = 1;
  rp.E1[0].fused = true;
  for (long long jp = 0; jp < g.P2; ++jp)
    if (jp != j) rp.E1[0].peers.push_back(col_rank(g, i, jp));
  for (long long k = 0; k < K; ++k) {
    const long long z0 = blo(Zn, K, k), zc = blk(Zn, K, k);
    // ---- stage B(k): y-IFFT of columns (l0 = x, l1 = z - z0) of R2'; out to the row peers' R1'
    Stage& B = rp.B[k];
    B.in = {kWs, (L.R2 + z0 * g.wz) * es};
    set_side(B.a.in, Zn * g.wz, 1, g.wz);
    B.a.in.bw = (int)g.wz;
    B.a.in.mT = g.ny * Zn;
    B.a.g0 = tile_g0(1, "DFFT_G0_INV_B");
    B.out = {kWs, 0};
    B.out_bases.push_back({kWs, 0});
    for (long long ip = 0; ip < g.P1; ++ip) B.out_bases.push_back({kPeer, 0, row_rank(g, ip, j)});
    Segs bseg;
    for (long long ip = 0; ip < g.P1; ++ip) {
      const long long yn = g.Y1n(ip);
      const InvLayout Lr = inv_layout(g, ip, j, 2);
      long long src = 0;
      for (long long q = 0; q < i; ++q) src += round_up(g.Xn(q), g.wy) * Zn * yn;
      bseg.push_back({1 + (int)ip, g.Y1lo(ip), yn, Lr.R1 + src + z0 * yn * g.wy, g.wy, 1, yn * g.wy});
    }
    B.a.out.bw = (int)g.wy;
    B.a.out.mT = Zn;
    B.a.scale = 1.0;
    ST(finish_stage(pl, B, fam_y(pl), (int)g.ny, Xn, zc, nullptr, &bseg));
    Exchange& E2 = rp.E2[k];
    E2.comm = 0;
    E2.fused = true;
    for (long long ip = 0; ip < g.P1; ++ip)
      if (ip != i) E2.peers.push_back(row_rank(g, ip, j));
    // ---- stage C(k): x-IFFT of lines (l0 = y, l1 = z - z0) of R1' chunk k, ×1/N -> `out`
    Stage& C = rp.Cc[k];
    C.in = {kWs, 0};
    Segs cseg;
    long long src = L.R1;
    for (long long is = 0; is < g.P1; ++is) {
      const long long xn = g.Xn(is), nb = (xn + g.wy - 1) / g.wy;
      for (long long xb = 0; xb < nb; ++xb) {
        const long long tn = std::min(g.wy, xn - xb * g.wy);
        cseg.push_back({0, g.Xlo(is) + xb * g.wy, tn, src + xb * Zn * Y1n * g.wy + z0 * Y1n * g.wy, 1, g.wy,
                        Y1n * g.wy});
      }
      src += nb * g.wy * Zn * Y1n;
    }
    C.out = {kUserOut, z0 * Y1n * nxl * es};  // C2R: nxl = nx/2 complex = nx reals per line
    set_side(C.a.out, 1, nxl, Y1n * nxl);
    C.a.scale = (xreal(pl) ? 2.0 : 1.0) / ((double)g.nx * (double)g.ny * (double)g.nz);
    ST(finish_stage(pl, C, fam_x_inv(pl), (int)nxl, Y1n, zc, &cseg, nullptr));
  }
  return DFFT_SUCCESS;
}

// Single GPU (P = 1, any decomposition): no exchange, so the axis order is free (the 3D DFT is
// separable).  Order the stages so no stage both reads and writes at a large stride:
//   forward: x (in -> out as [y][z][x]), z ([y][z][x] -> ws natural: the one large-pitch side),
//            y (ws -> out, natural -> natural)
//   inverse: y (in -> out, natural), z (natural -> ws as [y][z][x]: the large-pitch read),
//            x (ws -> out, natural, ×1/N)
// Single GPU, c2c, nz = 8·M: the z-FFT split by one radix-8 Cooley-Tukey step (fft_xz8_kernel).
//   forward: A = x-FFT + radix-8 z step (natural in -> ws [q][z1][y][x], whole lines),
//            B = M-point z-FFTs (ws, rows ny·nx apart -> natural, rows 8·ny·nx apart; both sides
//                256-512 B wide: the strided kernel's tile for an M-row column is 32 columns),
//            C = y-FFT (natural -> natural, in place on `out`)
//   inverse: A = y-IFFT (in -> out), B = M-point z-IFFTs (out -> ws), C = inverse radix-8 step +
//            x-IFFT (ws -> out, ×1/N)
// No pass reads or writes 64 B rows at a multi-MB pitch, the pattern that caps the plain z-pass at
// ~4.5 TB/s.  Needs c2c, nz % 8 == 0 with a specialised TMA kernel for nz/8, and the
// fused kernel for nx.
bool xz8_ok(dfft_plan_t pl, const Geo& g) {
  if (pl->r2c || pl->r2r || g.nz % 8 || g.nz < 64 || getenv("DFFT_NO_XZ8") || !g_use_tma || !tensor_map_encoder())
    return false;
  if (pl->kind[2] != DFFT_KIND_DFT || pl->kind[1] != DFFT_KIND_DFT) return false;
  KernelInfo kx, kz;
  const long long M = g.nz / 8;
  const bool okx = pl->f64 ? lookup_kernel_f64(kContigXZ8, (int)g.nx, pl->dir, &kx)
                           : lookup_kernel_f32(kContigXZ8, (int)g.nx, pl->dir, &kx);
  const bool okz = length_specialised(M) && (pl->f64 ? lookup_kernel_f64(kStrided, (int)M, pl->dir, &kz)
                                                     : lookup_kernel_f32(kStrided, (int)M, pl->dir, &kz));
  return okx && kx.fn && okz && kz.tma_fn && (g.nx * (long long)pl->es) % 16 == 0;
}

dfft_status_t build_single_xz8(dfft_plan_t pl, const Geo& g, RankPlan& rp) {
  const long long nx = g.nx, ny = g.ny, nz = g.nz, M = nz / 8, es = (long long)pl->es;
  rp.ws_bytes = (size_t)(nx * ny * nz * es);
  rp.A.resize(1);
  rp.B.resize(1);
  rp.E1.resize(1);
  rp.E2.resize(1);
  Stage &A = rp.A[0], &B = rp.B[0], &C = rp.C;
  const double inv_scale = 1.0 / ((double)nx * (double)ny * (double)nz);
  // the intermediate [q][z1][y][x]: line (l0 = y, l1 = z1, q), so consecutive CTAs of the fused
  // stage touch adjacent lines on both sides; the M-point z stage sees (x, y) as one contiguous
  // l0 axis: t = z1 (pitch ny·nx), l1 = q; natural seen by that stage: t = m (z = 8m + q), l1 = q
  auto mid_lines = [&](SideMap& m) { set_side(m, M * ny * nx, nx, ny * nx); };  // tstride = q stride
  auto nat_lines = [&](SideMap& m) { set_side(m, M * ny * nx, nx, ny * nx); };  // tstride = k stride
  auto mid_z = [&](SideMap& m) { set_side(m, ny * nx, 1, M * ny * nx); };
  auto nat_z = [&](SideMap& m) { set_side(m, 8 * ny * nx, 1, ny * nx); };
  auto nat_y = [&](SideMap& m) { set_side(m, nx, 1, ny * nx); };  // t = y, l0 = x, l1 = z
  const void* root = nullptr;
  ST(get_root_twiddles((int)nz, pl->f64, pl->dir, pl->comm->device, &root));
  if (pl->dir == DFFT_FORWARD) {
    A.in = {kUserIn, 0};
    nat_lines(A.a.in);
    A.out = {kWs, 0};
    mid_lines(A.a.out);
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, kContigXZ8, (int)nx, ny, M, nullptr, nullptr));
    A.a.tw2 = root;
    B.in = {kWs, 0};
    mid_z(B.a.in);
    B.out = {kUserOut, 0};
    nat_z(B.a.out);
    B.a.scale = 1.0;
    ST(finish_stage(pl, B, kStrided, (int)M, nx * ny, 8, nullptr, nullptr));
    C.in = {kUserOut, 0};
    nat_y(C.a.in);
    C.out = {kUserOut, 0};
    nat_y(C.a.out);
    C.a.scale = 1.0;
    C.last_fwd = true;  // t = y, l0 = x, l1 = z
    C.gax[0] = 1, C.gax[1] = 0, C.gax[2] = 2;
    ST(finish_stage(pl, C, fam_y(pl), (int)ny, nx, nz, nullptr, nullptr));
  } else {
    A.in = {kUserIn, 0};
    nat_y(A.a.in);
    A.out = {kUserOut, 0};
    nat_y(A.a.out);
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, fam_y(pl), (int)ny, nx, nz, nullptr, nullptr));
    B.in = {kUserOut, 0};
    nat_z(B.a.in);
    B.out = {kWs, 0};
    mid_z(B.a.out);
    B.a.scale = 1.0;
    ST(finish_stage(pl, B, kStrided, (int)M, nx * ny, 8, nullptr, nullptr));
    C.in = {kWs, 0};
    mid_lines(C.a.in);
    C.out = {kUserOut, 0};
    nat_lines(C.a.out);
    C.a.scale = inv_scale;
    ST(finish_stage(pl, C, kContigXZ8, (int)nx, ny, M, nullptr, nullptr));
    C.a.tw2 = root;
  }
  return DFFT_SUCCESS;
}

dfft_status_t build_single(dfft_plan_t pl, const Geo& g, RankPlan& rp) {
  if (xz8_ok(pl, g)) return build_single_xz8(pl, g, rp);
  const long long nx = g.nx, ny = g.ny, nz = g.nz, nxc = g.nxc, es = (long long)pl->es;
  const long long nxl = xreal(pl) ? nx / 2 : nx;
  const long long W = nxc * ny * nz;
  const bool c2r = pl->r2c && pl->dir == DFFT_INVERSE;  // the real `out` cannot hold a complex stage
  rp.ws_bytes = (size_t)((c2r ? 2 : 1) * W * es);
  rp.A.resize(1);
  rp.B.resize(1);
  rp.E1.resize(1);
  rp.E2.resize(1);
  Stage &A = rp.A[0], &B = rp.B[0], &C = rp.C;
  // z-pass, columns (l0 = x, l1 = y): natural [z][y][x] -> ws [y][z][x]
  auto zpass = [&](Stage& Z) -> dfft_status_t {
    Z.in = c2r ? Ref{kWs, 0} : Ref{kUserOut, 0};
    set_side(Z.a.in, ny * nxc, 1, nxc);
    Z.out = {kWs, c2r ? W * es : 0};
    set_side(Z.a.out, nxc, 1, nz * nxc);
    Z.a.scale = 1.0;
    return finish_stage(pl, Z, fam_z(pl), (int)nz, nxc, ny, nullptr, nullptr);
  };
  if (pl->dir == DFFT_FORWARD) {
    // forward with one large-pitch side in total (r01 session 2): the x-pass writes [y][z][x],
    // the z-pass reads it at a small pitch and writes natural order (the one large-pitch side),
    // and the y-pass runs natural -> natural (both sides at the x-row pitch: 3.08 vs 3.75 ms)
    A.in = {kUserIn, 0};  // lines (l0 = y, l1 = z)
    set_side(A.a.in, 1, nxl, ny * nxl);
    A.out = {kUserOut, 0};  // [y][z][x]
    set_side(A.a.out, 1, nz * nxc, nxc);
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, fam_x_fwd(pl), (int)nxl, ny, nz, nullptr, nullptr));
    B.in = {kUserOut, 0};  // z-pass: columns (l0 = x, l1 = y) of [y][z][x] -> ws natural
    set_side(B.a.in, nxc, 1, nz * nxc);
    B.out = {kWs, 0};
    set_side(B.a.out, ny * nxc, 1, nxc);
    B.a.scale = 1.0;
    ST(finish_stage(pl, B, fam_z(pl), (int)nz, nxc, ny, nullptr, nullptr));
    C.in = {kWs, 0};  // y-pass: columns (l0 = x, l1 = z), natural -> natural
    set_side(C.a.in, nxc, 1, ny * nxc);
    C.out = {kUserOut, 0};
    set_side(C.a.out, nxc, 1, ny * nxc);
    C.a.scale = 1.0;
    C.last_fwd = true;  // t = y, l0 = x, l1 = z
    C.gax[0] = 1, C.gax[1] = 0, C.gax[2] = 2;
    ST(finish_stage(pl, C, fam_y(pl), (int)ny, nxc, nz, nullptr, nullptr));
  } else {
    A.in = {kUserIn, 0};  // columns (l0 = x, l1 = z)
    set_side(A.a.in, nxc, 1, ny * nxc);
    A.out = c2r ? Ref{kWs, 0} : Ref{kUserOut, 0};
    set_side(A.a.out, nxc, 1, ny * nxc);
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, fam_y(pl), (int)ny, nxc, nz, nullptr, nullptr));
    ST(zpass(B));
    C.in = {kWs, c2r ? W * es : 0};  // lines (l0 = y, l1 = z) of ws [y][z][x]
    set_side(C.a.in, 1, nz * nxc, nxc);
    C.out = {kUserOut, 0};
    set_side(C.a.out, 1, nxl, ny * nxl);
    C.a.scale = (xreal(pl) ? 2.0 : 1.0) / ((double)nx * (double)ny * (double)nz);
    ST(finish_stage(pl, C, fam_x_inv(pl), (int)nxl, ny, nz, nullptr, nullptr));
  }
  return DFFT_SUCCESS;
}

// Inverse plan of one rank: z-IFFT (D3 in) → T2⁻¹ → y-IFFT → T1⁻¹ → x-IFFT ×1/N (D1 out).
dfft_status_t build_inverse(dfft_plan_t pl, const Geo& g, RankPlan& rp) {
  const long long i = rp.i, j = rp.j, K = g.K, es = (long long)pl->es;
  const long long Xn = g.Xn(i), Y1n = g.Y1n(i), Zn = g.Zn(j), Y3n = g.Y3n(j);
  const int mode = exch_mode(pl) == 3 ? 1 : exch_mode(pl);  // hybrid: the inverse is all CE
  const bool nccl = mode == 0, ce = mode == 1, p2p = mode == 2;
  const InvLayout L = inv_layout(g, i, j, mode);
  add_flags(pl, g, rp, L.end, false);
  auto s2off = [&](long long k, long long jp) {  // send2' block (k, j'): [y'][z ∈ Z_j'][xc]
    long long acc = 0;
    for (long long q = 0; q < jp; ++q)
      if (q != j) acc += g.Zn(q);
    return L.S2 + Y3n * (g.x0(i, k) * (g.nz - Zn) + g.xc(i, k) * acc);
  };
  auto s1off = [&](long long k, long long ip) {  // send1' block (k, i'): [z][y ∈ Y1_i'][xc]
    long long acc = 0;
    for (long long q = 0; q < ip; ++q)
      if (q != i) acc += g.Y1n(q);
    return L.S1 + Zn * (g.x0(i, k) * (g.ny - Y1n) + g.xc(i, k) * acc);
  };
  // recv1' block of (source row is, chunk k) on rank (ir, j): [z][y ∈ Y1_ir][xc_k(is)]
  auto r1off = [&](const InvLayout& Lr, long long ir, long long is, long long k) {
    return Lr.R1 + Zn * g.Y1n(ir) * (g.Xlo(is) + g.x0(is, k));
  };
  const long long nxl = xreal(pl) ? g.nx / 2 : g.nx;
  // P1 = 1 with fused stores: the y-IFFT writes natural x-lines and the x-IFFT reads them whole,
  // instead of R1's wy-column blocks (64 B pieces at a plane pitch: 2.4 ms at 1×2, 1024³ c64)
  const bool nat1 = p2p && g.P1 == 1 && !getenv("DFFT_NO_NAT1");
  rp.A.resize(K);
  rp.B.resize(K);
  rp.E1.resize(K);
  rp.E2.resize(K);
  for (long long k = 0; k < K; ++k) {
    const long long xc = g.xc(i, k), x0 = g.x0(i, k);
    // ---- stage A: z-IFFT of columns (l0 = xx, l1 = y') of `in`; out segmented by z-owner j'
    Stage& A = rp.A[k];
    A.in = {kUserIn, x0 * es};
    set_side(A.a.in, Y3n * Xn, 1, Xn);
    A.out = {kWs, 0};
    A.out_bases.push_back({kWs, 0});
    if (p2p)
      for (long long jp = 0; jp < g.P2; ++jp) A.out_bases.push_back({kPeer, 0, col_rank(g, i, jp)});
    Segs aseg;
    for (long long jp = 0; jp < g.P2; ++jp) {
      const long long zl = g.Zlo(jp), zn = g.Zn(jp);
      if (p2p) {  // receiver's R2' [xt][y][z][wz]
        const InvLayout Lr = inv_layout(g, i, jp, mode);
        aseg.push_back({1 + (int)jp, zl, zn, Lr.R2 + x0 * g.ny * zn + g.Y3lo(j) * zn * g.wz, g.wz, 1, zn * g.wz});
      } else if (jp == j) {
        aseg.push_back({0, zl, zn, L.R2 + g.ny * Zn * x0 + g.Y3lo(j) * Zn * xc, xc, 1, Zn * xc});
      } else {
        aseg.push_back({0, zl, zn, s2off(k, jp), xc, 1, zn * xc});
      }
    }
    if (p2p) {
      A.a.out.bw = (int)g.wz;
      A.a.out.mT = g.ny;
    }
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, fam_z(pl), (int)g.nz, xc, Y3n, nullptr, &aseg));
    // first exchange of the inverse = T2⁻¹ on the column group
    Exchange& E1 = rp.E1[k];
    E1.comm = 1;
    E1.fused = p2p;
    for (long long jp = 0; jp < g.P2; ++jp) {
      if (jp == j) continue;
      if (!nccl) E1.peers.push_back(col_rank(g, i, jp));
      if (p2p) continue;
      Xfer x{(int)jp, {kWs, s2off(k, jp) * es}, (size_t)(Y3n * g.Zn(jp) * xc * es)};
      if (ce) {
        const InvLayout Lr = inv_layout(g, i, jp, mode);
        x.remote = {kPeer, (Lr.R2 + g.ny * g.Zn(jp) * x0 + g.Y3lo(j) * g.Zn(jp) * xc) * es, col_rank(g, i, jp)};
      }
      E1.sends.push_back(x);
      E1.recvs.push_back({(int)jp, {kWs, (L.R2 + g.ny * Zn * x0 + g.Y3lo(jp) * Zn * xc) * es},
                          (size_t)(g.Y3n(jp) * Zn * xc * es)});
    }
    // ---- stage B: y-IFFT of columns (l0 = xx, l1 = z) of recv2' chunk k; out segmented by y-owner i'
    Stage& B = rp.B[k];
    B.in = {kWs, (L.R2 + g.ny * Zn * x0) * es};
    set_side(B.a.in, Zn * xc, 1, xc);
    if (p2p) {  // R2' [xt][y][z][wz]; chunk k starts at block x0 / wz
      B.in = {kWs, (L.R2 + x0 * g.ny * Zn) * es};
      set_side(B.a.in, Zn * g.wz, 1, g.wz);
      B.a.in.bw = (int)g.wz;
      B.a.in.mT = g.ny * Zn;
      // blocked input (adjacent z adjacent) and per-tile contiguous blocked output: z fastest
      B.a.g0 = tile_g0(1, "DFFT_G0_INV_B");
    }
    if (nat1) {  // 1×P2: T1⁻¹ is local; natural [z][y][x] (x over the Xn spectral columns) in R1
      B.out = {kWs, (L.R1 + x0) * es};
      set_side(B.a.out, Xn, 1, Y1n * Xn);
      B.a.scale = 1.0;
      ST(finish_stage(pl, B, fam_y(pl), (int)g.ny, xc, Zn, nullptr, nullptr));
      rp.E2[k].comm = 0;  // T1⁻¹ has no peer
      rp.E2[k].fused = true;
      continue;
    }
    B.out = {kWs, 0};
    B.out_bases.push_back({kWs, 0});
    if (p2p)
      for (long long ip = 0; ip < g.P1; ++ip) B.out_bases.push_back({kPeer, 0, row_rank(g, ip, j)});
    Segs bseg;
    for (long long ip = 0; ip < g.P1; ++ip) {
      const long long yl = g.Y1lo(ip), yn = g.Y1n(ip);
      if (p2p) {  // receiver's R1' [source i][xt][z][y][wy]
        const InvLayout Lr = inv_layout(g, ip, j, mode);
        long long src = 0;
        for (long long q = 0; q < i; ++q) src += round_up(g.Xn(q), g.wy) * Zn * yn;
        bseg.push_back({1 + (int)ip, yl, yn, Lr.R1 + src + x0 * Zn * yn, g.wy, 1, yn * g.wy});
      } else if (ip == i) {
        bseg.push_back({0, yl, yn, r1off(L, i, i, k), xc, 1, Y1n * xc});
      } else {
        bseg.push_back({0, yl, yn, s1off(k, ip), xc, 1, yn * xc});
      }
    }
    if (p2p) {
      B.a.out.bw = (int)g.wy;
      B.a.out.mT = Zn;
    }
    B.a.scale = 1.0;
    ST(finish_stage(pl, B, fam_y(pl), (int)g.ny, xc, Zn, nullptr, &bseg));
    // second exchange of the inverse = T1⁻¹ on the row group
    Exchange& E2 = rp.E2[k];
    E2.comm = 0;
    E2.fused = p2p;
    for (long long ip = 0; ip < g.P1; ++ip) {
      if (ip == i) continue;
      if (!nccl) E2.peers.push_back(row_rank(g, ip, j));
      if (p2p) continue;
      Xfer x{(int)ip, {kWs, s1off(k, ip) * es}, (size_t)(Zn * g.Y1n(ip) * xc * es)};
      if (ce) {
        const InvLayout Lr = inv_layout(g, ip, j, mode);
        x.remote = {kPeer, r1off(Lr, ip, i, k) * es, row_rank(g, ip, j)};
      }
      E2.sends.push_back(x);
      E2.recvs.push_back({(int)ip, {kWs, r1off(L, i, ip, k) * es}, (size_t)(Zn * Y1n * g.xc(ip, k) * es)});
    }
  }
  // ---- stage C: x-IFFT of lines (l0 = y, l1 = z); input segmented by (source row, chunk); ×1/N
  Stage& C = rp.C;
  C.in = {kWs, 0};
  if (nat1) {  // whole x-lines from the natural layout stage B wrote
    C.in = {kWs, L.R1 * es};
    set_side(C.a.in, 1, Xn, Y1n * Xn);
    C.out = {kUserOut, 0};
    set_side(C.a.out, 1, nxl, Y1n * nxl);
    C.a.scale = (xreal(pl) ? 2.0 : 1.0) / ((double)g.nx * (double)g.ny * (double)g.nz);
    return finish_stage(pl, C, fam_x_inv(pl), (int)nxl, Y1n, Zn, nullptr, nullptr);
  }
  Segs cseg;
  if (p2p) {  // R1' [source][xt][z][y][wy]: one segment per (source, column block)
    long long src = L.R1;
    for (long long is = 0; is < g.P1; ++is) {
      const long long xn = g.Xn(is), nb = (xn + g.wy - 1) / g.wy;
      for (long long xb = 0; xb < nb; ++xb) {
        const long long tn = std::min(g.wy, xn - xb * g.wy);
        cseg.push_back({0, g.Xlo(is) + xb * g.wy, tn, src + xb * Zn * Y1n * g.wy, 1, g.wy, Y1n * g.wy});
      }
      src += nb * g.wy * Zn * Y1n;
    }
  } else {
    for (long long is = 0; is < g.P1; ++is)
      for (long long k = 0; k < K; ++k) {
        const long long xcs = g.xc(is, k);
        if (xcs > 0) cseg.push_back({0, g.Xlo(is) + g.x0(is, k), xcs, r1off(L, i, is, k), 1, xcs, Y1n * xcs});
      }
  }
  C.out = {kUserOut, 0};
  set_side(C.a.out, 1, nxl, Y1n * nxl);
  C.a.scale = (xreal(pl) ? 2.0 : 1.0) / ((double)g.nx * (double)g.ny * (double)g.nz);
  ST(finish_stage(pl, C, fam_x_inv(pl), (int)nxl, Y1n, Zn, &cseg, nullptr));
  return DFFT_SUCCESS;
}

// ------------------------------------------------------------------------------ execution
struct Ctx {
  const void* in;
  void* out;
  void* ws;
  void* const* peers;  // P2P: workspace windows by global rank
};

void* resolve(const Ref& r, const Ctx& c) {
  switch (r.kind) {
    case kUserIn: return (char*)c.in + r.off;
    case kUserOut: return (char*)c.out + r.off;
    case kWs: return (char*)c.ws + r.off;
    case kPeer: return c.peers ? (char*)c.peers[r.peer] + r.off : nullptr;
    default: return nullptr;
  }
}

dfft_status_t launch_impl(const Stage& s, const Ctx& c, cudaStream_t st);
// DFFT_DEBUG_SYNC=1: synchronise after every stage launch and name the stage that failed
dfft_status_t launch(const Stage& s, const Ctx& c, cudaStream_t st) {
  static const bool dbg = getenv("DFFT_DEBUG_SYNC") != nullptr;
  const dfft_status_t r = launch_impl(s, c, st);
  if (dbg && r == DFFT_SUCCESS) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess)
      return fail(DFFT_ERR_CUDA, "stage (family %d, n %d, L0 %lld, L1 %lld, tma %d) failed: %s", s.family, s.n, s.a.L0,
                  s.a.L1, s.tma_variant, cudaGetErrorString(e));
  }
  return r;
}

dfft_status_t launch_impl(const Stage& s, const Ctx& c, cudaStream_t st) {
  if (s.empty) return DFFT_SUCCESS;
  g_launches.fetch_add(1, std::memory_order_relaxed);  // exactly one kernel per stage launch
  PassArgs a = s.a;
  a.in.base = resolve(s.in, c);
  a.out.base = resolve(s.out, c);
  for (size_t q = 0; q < s.in_bases.size(); ++q) a.in.bases[q] = resolve(s.in_bases[q], c);
  for (size_t q = 0; q < s.out_bases.size(); ++q) a.out.bases[q] = resolve(s.out_bases[q], c);
  if (s.tma_grid > 0 && ((uintptr_t)a.in.base & 15) == 0) {
    // 3D views in reals: (2·L0, n, L1) with strides (tstride, lstride) elements
    const bool f64 = s.es == 16;
    const cuuint64_t esz = f64 ? 8 : 4, ces = 2 * esz;
    auto encode = [&](CUtensorMap* tm, void* base, long long tstride, long long lstride) {
      cuuint64_t dims[3] = {(cuuint64_t)(2 * a.L0), (cuuint64_t)s.n, (cuuint64_t)a.L1};
      cuuint64_t strides[2] = {(cuuint64_t)tstride * ces,
                               (cuuint64_t)(a.L1 > 1 ? lstride * ces : 16 * ((tstride * ces * s.n + 15) / 16))};
      cuuint32_t box[3] = {(cuuint32_t)(2 * s.k.tma_w), (cuuint32_t)s.k.tma_boxr, 1};
      cuuint32_t estr[3] = {1, 1, 1};
      return tensor_map_encoder()(tm, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base,
                                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  g_tma_promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    auto encode4 = [&](CUtensorMap* tm, const SideMap& m) {  // column-blocked: (2·bw reals, n, L1, blocks)
      const long long nb = (a.L0 + m.bw - 1) / m.bw;
      cuuint64_t dims[4] = {(cuuint64_t)(2 * m.bw), (cuuint64_t)s.n, (cuuint64_t)a.L1, (cuuint64_t)nb};
      cuuint64_t strides[3] = {(cuuint64_t)m.tstride * ces, (cuuint64_t)m.s1 * ces, (cuuint64_t)(m.mT * m.s1) * ces};
      cuuint32_t box[4] = {(cuuint32_t)(2 * s.k.tma_w), (cuuint32_t)s.k.tma_boxr, 1, 1};
      cuuint32_t estr[4] = {1, 1, 1, 1};
      return tensor_map_encoder()(tm, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, m.base,
                                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  g_tma_promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    CUtensorMap tin, tout;
    const bool in_ok = a.in.bw > 0 ? (s.tma_variant == 1 && encode4(&tin, a.in))
                                   : encode(&tin, a.in.base, a.in.tstride, a.in.s1);
    if (in_ok) {
      // TMA stores: unsegmented output, 3D, or 4D into a column-blocked output whose block is
      // the tile (single-group kernel)
      const bool out_blk_ok = a.out.bw == 0 || (s.tma_variant == 1 && a.out.bw == s.k.tma_w &&
                                                (a.out.mT * a.out.s1 * (long long)ces) % 16 == 0);
      bool use_st = g_tma_store && a.out.ttab == nullptr && out_blk_ok && a.out.s0 == 1 &&
                    ((uintptr_t)a.out.base & 15) == 0 &&
                    (a.out.tstride * (long long)ces) % 16 == 0 && (a.L1 == 1 || (a.out.s1 * (long long)ces) % 16 == 0) &&
                    (a.out.bw > 0 ? encode4(&tout, a.out) : encode(&tout, a.out.base, a.out.tstride, a.out.s1));
      if (!use_st) tout = tin;  // unused by the non-TST variant
      const bool spec = a.spec[0] != nullptr;
      a.tw = s.tw_tma;
      void* targs[] = {&tin, &tout, &a};
      const long long grid = s.sm_cap > 0 ? std::min<long long>(s.tma_grid, (long long)s.sm_cap * s.tma_occ) : s.tma_grid;
      if (s.k.tma_st_only && !use_st) goto plain;  // R2R: the TMA variant needs TMA stores
      // multiplier: the c2c TMA-store variant with SPEC, or the R2R kernel (runtime multiplier)
      if (spec && !s.k.tma_st_only && !(use_st && s.tma_variant == 1 && s.k.tma_st_spec_fn)) goto plain;
      if (spec && !s.k.tma_st_only)
        CU(cudaLaunchKernel(s.k.tma_st_spec_fn, dim3((unsigned)grid), dim3(s.k.tma_threads), targs, s.k.tma_smem, st));
      else if (use_st && !spec && a.out.nbulk == 0 && s.ip_grid > 0 && !s.k.tma_st_only) {
        const long long gip = s.sm_cap > 0 ? std::min<long long>(s.ip_grid, (long long)s.sm_cap * s.ip_occ) : s.ip_grid;
        CU(cudaLaunchKernel(s.k.tma_ip_fn, dim3((unsigned)gip), dim3(s.k.tma_threads), targs, s.k.tma_ip_smem, st));
      }
      else
        CU(cudaLaunchKernel(a.out.nbulk > 0 ? s.k.tma_bk_fn
                            : use_st        ? s.k.tma_st1_fn
                                            : s.k.tma_fn,
                            dim3((unsigned)grid),
                            dim3(s.k.tma_threads), targs, s.k.tma_smem, st));
      return DFFT_SUCCESS;
    }
  }
plain:
  void* args[] = {&a};
  const void* fn = a.in.tb > 0 ? s.k.fn_tb : a.spec[0] != nullptr ? s.k.spec_fn : s.k.fn;
  if (!fn) return fail(DFFT_ERR_INTERNAL, "kernel variant not instantiated (n=%d)", s.n);
  CU(cudaLaunchKernel(fn, dim3((unsigned)s.grid), dim3(s.k.threads), args, s.k.smem, st));
  return DFFT_SUCCESS;
}

dfft_status_t exchange_nccl(dfft_plan_t pl, const Exchange& x, const Ctx& cx, cudaStream_t st) {
  if (x.sends.empty() && x.recvs.empty()) return DFFT_SUCCESS;
  ncclComm_t c = x.comm == 0 ? pl->row : pl->col;
  NC(ncclGroupStart());
  for (const Xfer& s : x.sends) NC(ncclSend(resolve(s.ref, cx), s.bytes, ncclUint8, s.peer, c, st));
  for (const Xfer& r : x.recvs) NC(ncclRecv(resolve(r.ref, cx), r.bytes, ncclUint8, r.peer, c, st));
  NC(ncclGroupEnd());
  return DFFT_SUCCESS;
}

// ------------------------------------------------------------------------------ profiling
// phases: 0 stage A, 1 exchange 1, 2 stage B, 3 exchange 2, 4 stage C.  Every execute records an
// origin event on the caller's stream; every profiled step a (start, stop) pair on its own stream.
dfft_status_t prof_origin(dfft_plan_t pl, cudaStream_t st, size_t* exec) {
  if (!pl->prof) return DFFT_SUCCESS;
  const size_t i = pl->prof_nexec++;
  while (pl->prof_origin.size() < pl->prof_nexec) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    pl->prof_origin.push_back(e);
  }
  *exec = i;
  CU(cudaEventRecord(pl->prof_origin[i], st));
  return DFFT_SUCCESS;
}
dfft_status_t prof_begin(dfft_plan_t pl, const dfft_plan_s::ProfRec& rec, cudaStream_t st, size_t* slot) {
  if (!pl->prof) return DFFT_SUCCESS;
  const size_t i = pl->prof_used++;
  while (pl->prof_ev.size() < 2 * pl->prof_used) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    pl->prof_ev.push_back(e);
  }
  if (pl->prof_rec.size() < pl->prof_used) pl->prof_rec.resize(pl->prof_used);
  pl->prof_rec[i] = rec;
  *slot = i;
  CU(cudaEventRecord(pl->prof_ev[2 * i], st));
  return DFFT_SUCCESS;
}
dfft_status_t prof_end(dfft_plan_t pl, size_t slot, cudaStream_t st) {
  if (!pl->prof) return DFFT_SUCCESS;
  CU(cudaEventRecord(pl->prof_ev[2 * slot + 1], st));
  return DFFT_SUCCESS;
}
// synchronise the recorded events: per-phase sums and timeline spans (relative to the origin of
// the execute each span belongs to)
dfft_status_t prof_resolve(dfft_plan_t pl) {
  for (size_t i = 0; i < pl->prof_used; ++i) {
    const dfft_plan_s::ProfRec& r = pl->prof_rec[i];
    CU(cudaEventSynchronize(pl->prof_ev[2 * i + 1]));
    float t = 0, a = 0, b = 0;
    CU(cudaEventElapsedTime(&t, pl->prof_ev[2 * i], pl->prof_ev[2 * i + 1]));
    pl->prof_ms[r.phase] += t;
    pl->prof_n[r.phase] += 1;
    if (r.exec < pl->prof_nexec) {
      CU(cudaEventElapsedTime(&a, pl->prof_origin[r.exec], pl->prof_ev[2 * i]));
      CU(cudaEventElapsedTime(&b, pl->prof_origin[r.exec], pl->prof_ev[2 * i + 1]));
      pl->prof_spans.push_back(dfft_span_t{r.phase, r.stream, r.chunk, r.rank, (int)r.exec, (double)a, (double)b});
    }
  }
  pl->prof_used = 0;
  pl->prof_nexec = 0;
  return DFFT_SUCCESS;
}

// ------------------------------------------------------------------------------ flags
constexpr int kMaxSig = 64;
struct SignalArgs {
  unsigned int* set[kMaxSig];
  unsigned int* clr[kMaxSig];
  int nset, nclr;
};

// One thread: reset the words this rank has waited on (its own window), make every earlier write
// of this stream (the stage kernel's stores into the peers' windows, the resets) visible system
// wide, then publish the signals with release stores into the targets' windows.
__global__ void dfft_flag_kernel(const __grid_constant__ SignalArgs a) {
  if (threadIdx.x != 0) return;
  for (int i = 0; i < a.nclr; ++i) asm volatile("st.relaxed.sys.global.u32 [%0], 0;" ::"l"(a.clr[i]) : "memory");
  __threadfence_system();
  for (int i = 0; i < a.nset; ++i) asm volatile("st.release.sys.global.u32 [%0], 1;" ::"l"(a.set[i]) : "memory");
}

using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitFn stream_wait_value32() {
  static WaitFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<WaitFn>(p);
  }();
  return fn;
}

// flag word: arr kReady / kDone; e = exchange (0 first, 1 second); k chunk; r writer rank
inline size_t flag_index(const dfft_plan_s* pl, int arr, int e, int k, int r) {
  const size_t P = (size_t)pl->P1 * pl->P2, K = (size_t)pl->K;
  return (((size_t)arr * 2 + e) * K + k) * P + r;
}
inline unsigned int* own_flags(const dfft_plan_s* pl, const RankPlan& rp) {
  return reinterpret_cast<unsigned int*>((char*)rp.ws + pl->flag_off);
}
// initial flag block: READY = 0 (nothing landed), DONE = 1 (every receive region free)
std::vector<unsigned int> initial_flags(const dfft_plan_s* pl) {
  const size_t half = (size_t)2 * pl->K * pl->P1 * pl->P2;
  std::vector<unsigned int> h(2 * half, 0u);
  for (size_t q = half; q < 2 * half; ++q) h[q] = 1u;
  return h;
}

// ------------------------------------------------------------------------------ schedules
// Builds a rank's execute as a list of steps on two streams (X = 0, Y = 1).  Without overlap
// (DFFT_FLAG_NO_OVERLAP) the same list runs on the caller's stream alone: a valid serial order,
// because every wait refers to a signal that comes earlier in every rank's list.
struct SchedBuilder {
  RankPlan& rp;
  void push(Op o) { rp.sched.push_back(std::move(o)); }
  void launch(int s, const Stage& st, int phase, int k) {
    Op o;
    o.kind = kOpLaunch, o.s = s, o.st = &st, o.phase = phase, o.chunk = k;
    push(std::move(o));
  }
  void wait(int s, int arr, int e, int k, const std::vector<int>& from) {
    Op o;
    o.kind = kOpWait, o.s = s, o.chunk = k;
    o.wait = FlagRef{arr, e, k, from};
    push(std::move(o));
  }
  void signal(int s, std::vector<FlagRef> set, std::vector<FlagRef> clr) {
    Op o;
    o.kind = kOpSignal, o.s = s;
    o.set = std::move(set);
    o.clr = std::move(clr);
    push(std::move(o));
  }
  int record(int s) {
    Op o;
    o.kind = kOpRecord, o.s = s, o.ev = rp.nev++;
    push(o);
    return o.ev;
  }
  void swait(int s, int ev) {
    Op o;
    o.kind = kOpStreamWait, o.s = s, o.ev = ev;
    push(std::move(o));
  }
  void xfer(int kind, int s, const Exchange& x, int phase, int k) {
    Op o;
    o.kind = kind, o.s = s, o.x = &x, o.phase = phase, o.chunk = k;
    push(std::move(o));
  }
};

// Fused stores (the P > 1 default): the stage kernels store straight into the peers' windows;
// flags order producer and consumer per chunk (Alg. 2's progressive receive) and the
// two streams overlap the chunks (Fig. 1).
void sched_p2p(dfft_plan_t pl, RankPlan& rp) {
  SchedBuilder b{rp};
  const int K = (int)rp.A.size();
  if (pl->bc) {
    // X: A (whole), then C(k) as chunk k of the second exchange completes; Y: B(k), k = 0..K-1
    const std::vector<int>& p1 = rp.E1[0].peers;
    b.wait(0, kDone, 0, 0, p1);  // the peers have read what I stored last execute
    b.launch(0, rp.A[0], 0, 0);
    b.signal(0, {{kReady, 0, 0, p1}}, {{kDone, 0, 0, p1}});
    const int eA = b.record(0);
    b.swait(1, eA);
    b.wait(1, kReady, 0, 0, p1);
    std::vector<int> eB(K);
    for (int k = 0; k < K; ++k) {
      const std::vector<int>& p2 = rp.E2[k].peers;
      b.wait(1, kDone, 1, k, p2);
      b.launch(1, rp.B[k], 2, k);
      b.signal(1, {{kReady, 1, k, p2}}, {{kDone, 1, k, p2}});
      eB[k] = b.record(1);
    }
    b.signal(1, {{kDone, 0, 0, p1}}, {{kReady, 0, 0, p1}});  // done reading my first-exchange window
    for (int k = 0; k < K; ++k) {
      const std::vector<int>& p2 = rp.E2[k].peers;
      b.swait(0, eB[k]);
      b.wait(0, kReady, 1, k, p2);
      b.launch(0, rp.Cc[k], 4, k);
      b.signal(0, {{kDone, 1, k, p2}}, {{kReady, 1, k, p2}});
    }
    return;
  }
  // X runs stage A chunk by chunk; Y runs stage B of each chunk as soon as its first exchange has
  // landed, then stage C
  std::vector<int> eA(K);
  for (int k = 0; k < K; ++k) {
    const std::vector<int>& p1 = rp.E1[k].peers;
    b.wait(0, kDone, 0, k, p1);
    b.launch(0, rp.A[k], 0, k);
    b.signal(0, {{kReady, 0, k, p1}}, {{kDone, 0, k, p1}});
    eA[k] = b.record(0);
  }
  for (int k = 0; k < K; ++k) {
    const std::vector<int>&p1 = rp.E1[k].peers, &p2 = rp.E2[k].peers;
    b.swait(1, eA[k]);  // my own block of chunk k
    b.wait(1, kReady, 0, k, p1);
    b.wait(1, kDone, 1, k, p2);
    b.launch(1, rp.B[k], 2, k);
    b.signal(1, {{kDone, 0, k, p1}, {kReady, 1, k, p2}}, {{kReady, 0, k, p1}, {kDone, 1, k, p2}});
  }
  for (int k = 0; k < K; ++k) b.wait(1, kReady, 1, k, rp.E2[k].peers);
  b.launch(1, rp.C, 4, 0);
  std::vector<FlagRef> set, clr;
  for (int k = 0; k < K; ++k) {
    set.push_back({kDone, 1, k, rp.E2[k].peers});
    clr.push_back({kReady, 1, k, rp.E2[k].peers});
  }
  b.signal(1, set, clr);
}

// Copy-engine transport: the stage kernels pack into local send blocks; Y's copy engine moves
// each block into the receiver's window (hybrid: the forward x-FFT stores fused instead).
void sched_ce(dfft_plan_t pl, RankPlan& rp) {
  (void)pl;
  SchedBuilder b{rp};
  const int K = (int)rp.A.size();
  auto ce = [&](int e, int k, const Exchange& x) {
    b.wait(1, kDone, e, k, x.peers);  // the receivers have read the previous execute's blocks
    b.xfer(kOpCeCopy, 1, x, e == 0 ? 1 : 3, k);
    b.signal(1, {{kReady, e, k, x.peers}}, {{kDone, e, k, x.peers}});
  };
  auto do_A = [&](int k) {
    const Exchange& x = rp.E1[k];
    if (x.fused) {
      b.wait(0, kDone, 0, k, x.peers);
      b.launch(0, rp.A[k], 0, k);
      b.signal(0, {{kReady, 0, k, x.peers}}, {{kDone, 0, k, x.peers}});
    } else {
      b.launch(0, rp.A[k], 0, k);
      b.swait(1, b.record(0));
      ce(0, k, x);
    }
  };
  do_A(0);
  for (int k = 0; k < K; ++k) {
    if (k + 1 < K) do_A(k + 1);
    const Exchange &x1 = rp.E1[k], &x2 = rp.E2[k];
    b.wait(0, kReady, 0, k, x1.peers);  // the peers' blocks of chunk k have landed
    if (x2.fused) b.wait(0, kDone, 1, k, x2.peers);
    b.launch(0, rp.B[k], 2, k);
    b.signal(0, {{kDone, 0, k, x1.peers}}, {{kReady, 0, k, x1.peers}});  // done reading my first receive region
    if (x2.fused) {
      b.signal(0, {{kReady, 1, k, x2.peers}}, {{kDone, 1, k, x2.peers}});
    } else {
      b.swait(1, b.record(0));
      ce(1, k, x2);
    }
  }
  for (int k = 0; k < K; ++k) b.wait(0, kReady, 1, k, rp.E2[k].peers);
  b.launch(0, rp.C, 4, 0);
  std::vector<FlagRef> set, clr;
  for (int k = 0; k < K; ++k) {
    set.push_back({kDone, 1, k, rp.E2[k].peers});
    clr.push_back({kReady, 1, k, rp.E2[k].peers});
  }
  b.signal(0, set, clr);
}

// NCCL transport (and P = 1): grouped send/recv on Y against the FFTs on X.  Host issue order is
// a topological order of the chunk DAG:  A0 E1_0 | A1 E1_1 B0 E2_0 | A2 E1_2 B1 E2_1 | ...
void sched_nccl(dfft_plan_t pl, RankPlan& rp) {
  SchedBuilder b{rp};
  const int K = (int)rp.A.size();
  auto has = [](const Exchange& x) { return !x.sends.empty() || !x.recvs.empty(); };
  if (!pl->overlap) {  // static-barrier ablation ("SimpleMPIFFT"): program order, one stream
    for (int k = 0; k < K; ++k) b.launch(0, rp.A[k], 0, k);
    for (int k = 0; k < K; ++k) b.xfer(kOpNccl, 0, rp.E1[k], 1, k);
    for (int k = 0; k < K; ++k) b.launch(0, rp.B[k], 2, k);
    for (int k = 0; k < K; ++k) b.xfer(kOpNccl, 0, rp.E2[k], 3, k);
    b.launch(0, rp.C, 4, 0);
    return;
  }
  std::vector<int> e1(K, -1), e2(K, -1);
  auto do_A = [&](int k) {
    b.launch(0, rp.A[k], 0, k);
    if (has(rp.E1[k])) {
      b.swait(1, b.record(0));
      b.xfer(kOpNccl, 1, rp.E1[k], 1, k);
      e1[k] = b.record(1);
    }
  };
  do_A(0);
  for (int k = 0; k < K; ++k) {
    if (k + 1 < K) do_A(k + 1);
    if (e1[k] >= 0) b.swait(0, e1[k]);
    b.launch(0, rp.B[k], 2, k);
    if (has(rp.E2[k])) {
      b.swait(1, b.record(0));
      b.xfer(kOpNccl, 1, rp.E2[k], 3, k);
      e2[k] = b.record(1);
    }
  }
  if (e2[K - 1] >= 0) b.swait(0, e2[K - 1]);  // same comm stream => the last record suffices
  b.launch(0, rp.C, 4, 0);
}

void build_schedule(dfft_plan_t pl, RankPlan& rp) {
  rp.sched.clear();
  rp.nev = 0;
  if (pl->p2p) sched_p2p(pl, rp);
  else if (pl->ce) sched_ce(pl, rp);
  else sched_nccl(pl, rp);
}

// ------------------------------------------------------------------------------ interpreter
struct RunCtx {
  Ctx cx;
  cudaStream_t s[2];
  size_t exec;
};

dfft_status_t issue_signal(dfft_plan_t pl, const RankPlan& rp, const Op& op, cudaStream_t st) {
  SignalArgs a{};
  unsigned int* own = own_flags(pl, rp);
  for (const FlagRef& f : op.clr)
    for (int r : f.ranks) {
      if (a.nclr >= kMaxSig) return fail(DFFT_ERR_INTERNAL, "too many flag resets in one signal");
      a.clr[a.nclr++] = own + flag_index(pl, f.arr, f.e, f.k, r);
    }
  for (const FlagRef& f : op.set)
    for (int t : f.ranks) {
      if (a.nset >= kMaxSig) return fail(DFFT_ERR_INTERNAL, "too many flag signals in one signal");
      a.set[a.nset++] = reinterpret_cast<unsigned int*>((char*)pl->peer_ws[t] + pl->flag_off) +
                        flag_index(pl, f.arr, f.e, f.k, rp.rank);
    }
  if (a.nset == 0 && a.nclr == 0) return DFFT_SUCCESS;
  void* args[] = {&a};
  CU(cudaLaunchKernel((const void*)dfft_flag_kernel, dim3(1), dim3(32), args, 0, st));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return DFFT_SUCCESS;
}

dfft_status_t issue_ce(dfft_plan_t pl, const Exchange& x, const Ctx& cx, cudaStream_t st) {
  (void)pl;
  for (const Xfer& t : x.sends) {
    if (t.height > 1)
      CU(cudaMemcpy2DAsync(resolve(t.remote, cx), t.dpitch, resolve(t.ref, cx), t.spitch, t.width, t.height,
                           cudaMemcpyDeviceToDevice, st));
    else
      CU(cudaMemcpyAsync(resolve(t.remote, cx), resolve(t.ref, cx), t.bytes, cudaMemcpyDeviceToDevice, st));
  }
  return DFFT_SUCCESS;
}

dfft_status_t issue(dfft_plan_t pl, const RankPlan& rp, const Op& op, const RunCtx& rc) {
  const cudaStream_t st = rc.s[op.s];
  const bool two = rc.s[0] != rc.s[1];
  switch (op.kind) {
    case kOpLaunch:
    case kOpNccl:
    case kOpCeCopy: {
      if (op.kind == kOpLaunch && op.st->empty) return DFFT_SUCCESS;
      if (op.kind == kOpNccl && op.x->sends.empty() && op.x->recvs.empty()) return DFFT_SUCCESS;
      if (op.kind == kOpCeCopy && op.x->sends.empty()) return DFFT_SUCCESS;
      size_t slot = 0;
      ST(prof_begin(pl, dfft_plan_s::ProfRec{op.phase, op.s, op.chunk, rp.rank, rc.exec}, st, &slot));
      if (op.kind == kOpLaunch) ST(launch(*op.st, rc.cx, st));
      else if (op.kind == kOpNccl) ST(exchange_nccl(pl, *op.x, rc.cx, st));
      else ST(issue_ce(pl, *op.x, rc.cx, st));
      return prof_end(pl, slot, st);
    }
    case kOpWait: {
      unsigned int* own = own_flags(pl, rp);
      for (int r : op.wait.ranks) {
        const CUresult res = stream_wait_value32()(
            (CUstream)st, (CUdeviceptr)(own + flag_index(pl, op.wait.arr, op.wait.e, op.wait.k, r)), 1,
            CU_STREAM_WAIT_VALUE_GEQ);
        if (res != CUDA_SUCCESS) return fail(DFFT_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)res);
      }
      return DFFT_SUCCESS;
    }
    case kOpSignal: return issue_signal(pl, rp, op, st);
    case kOpRecord:
      if (two) CU(cudaEventRecord(rp.ev[op.ev], st));
      return DFFT_SUCCESS;
    case kOpStreamWait:
      if (two) CU(cudaStreamWaitEvent(st, rp.ev[op.ev], 0));
      return DFFT_SUCCESS;
  }
  return fail(DFFT_ERR_INTERNAL, "bad schedule op");
}

// Issue step `pos` of a rank's schedule.  After a failure the remaining steps that move data are
// skipped but every wait and signal is still issued, so the peers' flag protocol stays in step
// (no rank is left waiting for a signal that will never come); the plan is marked failed.
struct Runner {
  dfft_plan_t pl;
  dfft_status_t first = DFFT_SUCCESS;
  std::string msg;
  void step(const RankPlan& rp, size_t pos, const RunCtx& rc) {
    const Op& op = rp.sched[pos];
    const bool data = op.kind == kOpLaunch || op.kind == kOpNccl || op.kind == kOpCeCopy;
    if (first != DFFT_SUCCESS && data) return;
    const dfft_status_t st = issue(pl, rp, op, rc);
    if (st != DFFT_SUCCESS && first == DFFT_SUCCESS) {
      first = st;
      msg = g_err;
    }
  }
  dfft_status_t finish() {
    if (first == DFFT_SUCCESS) return DFFT_SUCCESS;
    pl->fail_msg = "enqueue failed: " + msg;
    pl->failed.store(1);
    return fail(first, "%s", msg.c_str());
  }
};

bool two_streams(const dfft_plan_t pl) { return pl->overlap && (size_t)pl->P1 * pl->P2 > 1; }

dfft_status_t fork_rank(dfft_plan_t pl, RankPlan& rp, cudaStream_t user, RunCtx& rc) {
  if (!two_streams(pl)) {
    rc.s[0] = rc.s[1] = user;
    return DFFT_SUCCESS;
  }
  rc.s[0] = rp.sX;
  rc.s[1] = rp.sY;
  CU(cudaEventRecord(rp.ev_fork, user));
  CU(cudaStreamWaitEvent(rp.sX, rp.ev_fork, 0));
  CU(cudaStreamWaitEvent(rp.sY, rp.ev_fork, 0));
  return DFFT_SUCCESS;
}
dfft_status_t join_rank(dfft_plan_t pl, RankPlan& rp, cudaStream_t user) {
  if (!two_streams(pl)) return DFFT_SUCCESS;
  CU(cudaEventRecord(rp.ev_join[0], rp.sX));
  CU(cudaEventRecord(rp.ev_join[1], rp.sY));
  CU(cudaStreamWaitEvent(user, rp.ev_join[0], 0));
  CU(cudaStreamWaitEvent(user, rp.ev_join[1], 0));
  return DFFT_SUCCESS;
}

dfft_status_t issue_rank(dfft_plan_t pl, const void* in, void* out, cudaStream_t user) {
  RankPlan& rp = pl->ranks[0];
  RunCtx rc{Ctx{in, out, rp.ws, pl->peer_ws.empty() ? nullptr : pl->peer_ws.data()}, {user, user}, 0};
  ST(prof_origin(pl, user, &rc.exec));
  ST(fork_rank(pl, rp, user, rc));
  Runner run{pl};
  for (size_t pos = 0; pos < rp.sched.size(); ++pos) run.step(rp, pos, rc);
  ST(join_rank(pl, rp, user));
  return run.finish();
}

void drop_graphs(dfft_plan_t pl) {
  for (auto& g : pl->graphs) cudaGraphExecDestroy(g.exec);
  pl->graphs.clear();
}

// Replay the schedule as a CUDA graph: one launch instead of every kernel, flag wait and
// cross-stream event of the execute (N=4 1024^3: 8.5 -> 7.9 ms fwd+inv).  Captured on the plan's
// private stream the first time a (in, out) pair is executed; not while profiling (the phase
// events must be live) or while the caller's stream is itself being captured (the schedule then
// goes into the caller's graph).
dfft_status_t execute_rank(dfft_plan_t pl, const void* in, void* out, cudaStream_t user) {
  static const bool no_graph = getenv("DFFT_NO_GRAPH") != nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CU(cudaStreamIsCapturing(user, &cs));
  if (no_graph || pl->prof || cs != cudaStreamCaptureStatusNone) return issue_rank(pl, in, out, user);
  for (size_t q = 0; q < pl->graphs.size(); ++q)
    if (pl->graphs[q].in == in && pl->graphs[q].out == out) {
      CU(cudaGraphLaunch(pl->graphs[q].exec, user));
      g_launches.fetch_add(pl->graphs[q].launches, std::memory_order_relaxed);
      return DFFT_SUCCESS;
    }
  if (!pl->cap_stream) CU(cudaStreamCreateWithFlags(&pl->cap_stream, cudaStreamNonBlocking));
  CU(cudaStreamBeginCapture(pl->cap_stream, cudaStreamCaptureModeThreadLocal));
  const long long n0 = g_launches.load(std::memory_order_relaxed);
  const dfft_status_t st = issue_rank(pl, in, out, pl->cap_stream);
  const long long nk = g_launches.load(std::memory_order_relaxed) - n0;  // (counted once: the first replay)
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(pl->cap_stream, &graph);
  if (st != DFFT_SUCCESS || ec != cudaSuccess || !graph) {  // capture failed: issue directly
    if (graph) cudaGraphDestroy(graph);
    (void)cudaGetLastError();
    if (st != DFFT_SUCCESS) return st;
    return issue_rank(pl, in, out, user);
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) {
    (void)cudaGetLastError();
    return issue_rank(pl, in, out, user);
  }
  if (pl->graphs.size() >= 4) {  // a few (in, out) pairs: the host chain alternates two
    cudaGraphExecDestroy(pl->graphs.front().exec);
    pl->graphs.erase(pl->graphs.begin());
  }
  pl->graphs.push_back({in, out, exec, nk});
  CU(cudaGraphLaunch(exec, user));
  return DFFT_SUCCESS;
}

// simulated ranks, NCCL layouts: rank r's send to peer q is matched with q's receive from r
dfft_status_t exchange_sim(dfft_plan_t pl, bool second, size_t k, const void* const* ins, void* const* outs,
                           cudaStream_t st) {
  const int P = (int)pl->ranks.size();
  for (int r = 0; r < P; ++r) {
    const RankPlan& src = pl->ranks[r];
    const Exchange& xs = second ? src.E2[k] : src.E1[k];
    for (const Xfer& s : xs.sends) {
      // group peer index -> global rank
      int q = xs.comm == 0 ? s.peer * pl->P2 + src.j : src.i * pl->P2 + s.peer;
      const RankPlan& dst = pl->ranks[q];
      const Exchange& xd = second ? dst.E2[k] : dst.E1[k];
      int my_idx = xs.comm == 0 ? src.i : src.j;
      const Xfer* rv = nullptr;
      for (const Xfer& c : xd.recvs)
        if (c.peer == my_idx) rv = &c;
      if (!rv || rv->bytes != s.bytes)
        return fail(DFFT_ERR_INTERNAL, "sim exchange mismatch %d->%d (%zu vs %zu bytes)", r, q, s.bytes,
                    rv ? rv->bytes : 0);
      void* sp = resolve(s.ref, Ctx{ins[r], outs[r], src.ws, nullptr});
      void* dp = resolve(rv->ref, Ctx{ins[q], outs[q], dst.ws, nullptr});
      CU(cudaMemcpyAsync(dp, sp, s.bytes, cudaMemcpyDeviceToDevice, st));
    }
  }
  return DFFT_SUCCESS;
}

// Simulated ranks.  IPC-window transports (fused stores, copy engines): every rank runs its own
// schedule exactly as a real rank does — its own stream pair, the flag words in its workspace
// (the other ranks' workspaces stand in for the peers' IPC windows), the B→C / K-chunk pipeline
// and the SM caps.  The schedules are issued interleaved position by position, a topological
// order of the cross-rank flag dependencies, so the GPU can always make progress whatever the
// mapping of streams onto hardware queues.  ins[r] == nullptr: rank r does not execute (a failed
// peer; its partners then wait until the watchdog releases them).
// NCCL layouts: the stage kernels per rank, exchanges by device copies of the blocks NCCL would
// move, in stream order on the caller's stream.
dfft_status_t execute_sim(dfft_plan_t pl, const void* const* ins, void* const* outs, cudaStream_t user) {
  const size_t P = pl->ranks.size();
  if (pl->p2p || pl->ce) {
    size_t exec = 0;
    ST(prof_origin(pl, user, &exec));
    std::vector<RunCtx> rc(P);
    for (size_t r = 0; r < P; ++r) {
      rc[r] = RunCtx{Ctx{ins[r], outs[r], pl->ranks[r].ws, pl->peer_ws.data()}, {user, user}, exec};
      if (ins[r]) ST(fork_rank(pl, pl->ranks[r], user, rc[r]));
    }
    const size_t L = pl->ranks[0].sched.size();
    for (size_t r = 1; r < P; ++r)
      if (pl->ranks[r].sched.size() != L) return fail(DFFT_ERR_INTERNAL, "rank schedules differ in length");
    Runner run{pl};
    for (size_t pos = 0; pos < L; ++pos)
      for (size_t r = 0; r < P; ++r)
        if (ins[r]) run.step(pl->ranks[r], pos, rc[r]);
    for (size_t r = 0; r < P; ++r)
      if (ins[r]) ST(join_rank(pl, pl->ranks[r], user));
    return run.finish();
  }
  const size_t K = pl->ranks[0].A.size();
  auto cx = [&](size_t r) { return Ctx{ins[r], outs[r], pl->ranks[r].ws, nullptr}; };
  for (size_t k = 0; k < K; ++k)
    for (size_t r = 0; r < P; ++r) ST(launch(pl->ranks[r].A[k], cx(r), user));
  for (size_t k = 0; k < K; ++k) ST(exchange_sim(pl, false, k, ins, outs, user));
  for (size_t k = 0; k < K; ++k)
    for (size_t r = 0; r < P; ++r) ST(launch(pl->ranks[r].B[k], cx(r), user));
  for (size_t k = 0; k < K; ++k) ST(exchange_sim(pl, true, k, ins, outs, user));
  for (size_t r = 0; r < P; ++r) ST(launch(pl->ranks[r].C, cx(r), user));
  return DFFT_SUCCESS;
}

// ------------------------------------------------------------------------------ watchdog
// A process-wide thread watches the executes of multi-rank plans.  If the oldest outstanding
// execute of a plan makes no progress for the timeout (a peer died or never called execute), it
// reports on stderr, marks the plan failed (later executes return DFFT_ERR_PEER), checks the NCCL
// communicators for asynchronous errors, and releases the plan's waits by setting every flag word
// of its windows, so the caller's streams drain instead of hanging; the results are then invalid.
std::atomic<long long> g_timeout_ms{[] {
  const char* v = getenv("DFFT_TIMEOUT_MS");
  return v ? atoll(v) : 120000LL;
}()};

struct WdEntry {
  cudaEvent_t ev;
  std::chrono::steady_clock::time_point t;
};
struct Watchdog {
  std::mutex mu;
  std::map<dfft_plan_t, std::vector<WdEntry>> pending;  // per plan, oldest first
  std::map<dfft_plan_t, std::chrono::steady_clock::time_point> progress;
  std::thread th;
  bool started = false;
  void ensure() {
    if (started) return;
    started = true;
    th = std::thread([this] { loop(); });
    th.detach();
  }
  void loop();
};
Watchdog& watchdog() {
  static Watchdog* w = new Watchdog;  // never destroyed: the detached thread outlives static teardown
  return *w;
}

void release_flags(dfft_plan_t pl) {
  if (!(pl->p2p || pl->ce)) return;
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return;
  const size_t words = (size_t)4 * pl->K * pl->P1 * pl->P2;
  std::vector<unsigned int> ones(words, 1u);
  for (RankPlan& rp : pl->ranks)
    if (rp.ws) cudaMemcpyAsync(own_flags(pl, rp), ones.data(), words * 4, cudaMemcpyHostToDevice, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
}

void trigger_failure(dfft_plan_t pl, long long waited_ms) {
  char buf[512];
  std::string nccl_state;
  if (pl->comm->world) {
    ncclResult_t ar = ncclSuccess;
    if (ncclCommGetAsyncError(pl->comm->world, &ar) == ncclSuccess && ar != ncclSuccess)
      nccl_state = std::string("; NCCL async error: ") + ncclGetErrorString(ar);
  }
  snprintf(buf, sizeof buf,
           "execute made no progress for %lld ms (rank %d of %d): a peer did not signal; waits released, "
           "results invalid%s",
           waited_ms, pl->comm->rank, pl->comm->nranks, nccl_state.c_str());
  pl->fail_msg = buf;
  pl->failed.store(1);
  fprintf(stderr, "dfft watchdog: plan %p: %s\n", (void*)pl, buf);
  release_flags(pl);
  if (!nccl_state.empty()) {  // NCCL kernels of this comm may be stuck too: abort them
    for (auto& kv : pl->comm->sub) {
      if (kv.second.first) ncclCommAbort(kv.second.first);
      if (kv.second.second) ncclCommAbort(kv.second.second);
      kv.second = {nullptr, nullptr};
    }
  }
}

void Watchdog::loop() {
  // relaxed capture interaction: this thread's event queries must neither fail nor invalidate a
  // CUDA-graph capture the application runs on another thread
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  cudaThreadExchangeStreamCaptureMode(&mode);
  for (;;) {
    std::this_thread::sleep_for(std::chrono::milliseconds(20));
    std::lock_guard<std::mutex> lk(mu);
    const auto now = std::chrono::steady_clock::now();
    for (auto& kv : pending) {
      dfft_plan_t pl = kv.first;
      std::vector<WdEntry>& q = kv.second;
      if (q.empty()) continue;
      cudaSetDevice(pl->comm->device);
      while (!q.empty()) {
        const cudaError_t e = cudaEventQuery(q.front().ev);
        if (e == cudaErrorNotReady) break;
        if (e != cudaSuccess) (void)cudaGetLastError();
        cudaEventDestroy(q.front().ev);
        q.erase(q.begin());
        progress[pl] = now;
      }
      if (q.empty() || pl->failed.load()) continue;
      const auto since = std::max(q.front().t, progress[pl]);
      const long long ms = std::chrono::duration_cast<std::chrono::milliseconds>(now - since).count();
      if (ms > g_timeout_ms.load()) trigger_failure(pl, ms);
    }
  }
}

// register an execute (event recorded on the caller's stream after the join); not while the
// stream is being captured into a graph (the execute happens at replay)
dfft_status_t wd_track(dfft_plan_t pl, cudaStream_t user) {
  static const bool off = getenv("DFFT_NO_WATCHDOG") != nullptr;  // A/B switch
  if ((size_t)pl->P1 * pl->P2 <= 1 || off) return DFFT_SUCCESS;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CU(cudaStreamIsCapturing(user, &cs));
  if (cs != cudaStreamCaptureStatusNone) return DFFT_SUCCESS;
  Watchdog& w = watchdog();
  std::lock_guard<std::mutex> lk(w.mu);
  std::vector<WdEntry>& q = w.pending[pl];
  if (q.size() >= 16) return DFFT_SUCCESS;  // the oldest entries already witness progress
  cudaEvent_t e;
  CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CU(cudaEventRecord(e, user));
  q.push_back(WdEntry{e, std::chrono::steady_clock::now()});
  w.ensure();
  return DFFT_SUCCESS;
}
void wd_forget(dfft_plan_t pl) {
  Watchdog& w = watchdog();
  std::lock_guard<std::mutex> lk(w.mu);
  auto it = w.pending.find(pl);
  if (it == w.pending.end()) return;
  for (WdEntry& e : it->second) cudaEventDestroy(e.ev);
  w.pending.erase(it);
  w.progress.erase(pl);
}

// ------------------------------------------------------------------------------ teardown
void free_host_chain(dfft_plan_t pl) {
  dfft_plan_s::HostChain* h = pl->host;
  if (!h) return;
  if (h->h2d) cudaStreamSynchronize(h->h2d);
  if (h->d2h) cudaStreamSynchronize(h->d2h);
  for (int b = 0; b < 2; ++b) {
    if (h->in_dev[b]) cudaFree(h->in_dev[b]);
    if (h->out_dev[b]) cudaFree(h->out_dev[b]);
    for (cudaEvent_t e : {h->in_ready[b], h->in_free[b], h->out_ready[b], h->out_done[b]})
      if (e) cudaEventDestroy(e);
  }
  for (void* m : h->mid)
    if (m) cudaFree(m);
  if (h->h2d) cudaStreamDestroy(h->h2d);
  if (h->d2h) cudaStreamDestroy(h->d2h);
  delete h;
  pl->host = nullptr;
}

void free_stage(Stage& s) {
  if (s.in_tab) cudaFree(s.in_tab);
  if (s.out_tab) cudaFree(s.out_tab);
  s.in_tab = s.out_tab = nullptr;
}

// Peers write their final DONE flags into this window after their last stage: poll them (with the
// watchdog's timeout) so no peer store lands in freed memory, then drain the plan's streams.
void wait_peers_done(dfft_plan_t pl) {
  if (!(pl->p2p || pl->ce) || pl->flag_off == 0) return;
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return;
  const size_t words = (size_t)4 * pl->K * pl->P1 * pl->P2;
  std::vector<unsigned int> h(words);
  const auto t0 = std::chrono::steady_clock::now();
  for (RankPlan& rp : pl->ranks) {
    if (!rp.ws) continue;
    for (;;) {
      if (cudaMemcpyAsync(h.data(), own_flags(pl, rp), words * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
          cudaStreamSynchronize(s) != cudaSuccess)
        break;
      bool ok = true;
      for (int e = 0; e < 2; ++e)
        for (size_t k = 0; k < rp.A.size(); ++k)
          for (int r : (e == 0 ? rp.E1[k] : rp.E2[k]).peers) ok = ok && h[flag_index(pl, kDone, e, (int)k, r)] >= 1;
      if (ok) break;
      const long long ms =
          std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
      if (ms > g_timeout_ms.load()) {
        fprintf(stderr, "dfft: destroy: peers did not finish within %lld ms; releasing\n", ms);
        release_flags(pl);
        break;
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
  }
  cudaStreamDestroy(s);
}

void free_plan(dfft_plan_t pl) {
  if (!pl) return;
  wd_forget(pl);
  wait_peers_done(pl);
  if (pl->cap_stream) cudaStreamSynchronize(pl->cap_stream);
  drop_graphs(pl);
  if (pl->cap_stream) cudaStreamDestroy(pl->cap_stream);
  for (RankPlan& rp : pl->ranks) {
    if (rp.sX) cudaStreamSynchronize(rp.sX);
    if (rp.sY) cudaStreamSynchronize(rp.sY);
  }
  if (!pl->comm->sim)
    for (size_t r = 0; r < pl->peer_ws.size(); ++r)
      if (pl->peer_ws[r] && (int)r != pl->comm->rank) cudaIpcCloseMemHandle(pl->peer_ws[r]);
  pl->peer_ws.clear();
  for (RankPlan& rp : pl->ranks) {
    for (Stage& s : rp.A) free_stage(s);
    for (Stage& s : rp.B) free_stage(s);
    free_stage(rp.C);
    for (Stage& c : rp.Cc) free_stage(c);
    if (rp.ws) cudaFree(rp.ws);
    for (cudaEvent_t e : rp.ev) cudaEventDestroy(e);
    for (cudaEvent_t e : {rp.ev_fork, rp.ev_join[0], rp.ev_join[1]})
      if (e) cudaEventDestroy(e);
    if (rp.sX) cudaStreamDestroy(rp.sX);
    if (rp.sY) cudaStreamDestroy(rp.sY);
  }
  for (cudaEvent_t e : pl->prof_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : pl->prof_origin) cudaEventDestroy(e);
  if (pl->spec_tab) cudaFree(pl->spec_tab);
  free_host_chain(pl);
  delete pl;
}

struct PlanGuard {
  dfft_plan_t p;
  ~PlanGuard() {
    if (p) free_plan(p);
  }
};

// Fused-store plans with K > 1 run stage A(k+1) and B(k) concurrently on two streams.  The one
// of the pair that stores to peers (NVLink-bound) gets at most DFFT_NVL_SMS SMs (default 80) and
// the HBM-bound one the rest, except in the last chunk, which runs alone.  Without overlap every
// stage runs alone on the whole GPU.
dfft_status_t apply_sm_caps(dfft_plan_t pl, RankPlan& rp) {
  const size_t K = rp.A.size();
  if (!pl->p2p || K < 2 || !pl->overlap) return DFFT_SUCCESS;

  int sms = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, pl->comm->device));
  const char* v = getenv("DFFT_NVL_SMS");
  const int nvl = std::max(1, std::min(sms - 1, v ? atoi(v) : 80));
  if (pl->bc) {  // B(k) stores to peers, C(k) runs beside B(k+1)
    for (size_t k = 0; k < K; ++k) {
      rp.B[k].sm_cap = nvl;
      if (k + 1 < K) rp.Cc[k].sm_cap = sms - nvl;
    }
    return DFFT_SUCCESS;
  }
  for (size_t k = 0; k < K; ++k) {
    const bool a_remote = !rp.E1[k].peers.empty(), b_remote = !rp.E2[k].peers.empty();
    if (a_remote == b_remote) continue;  // both or neither NVLink-bound: nothing to balance
    Stage& nv = a_remote ? rp.A[k] : rp.B[k];
    nv.sm_cap = nvl;
    // the local stage of the pair: B(k) runs beside A(k+1) (none after the last chunk); A(k+1)
    // runs beside B(k)
    if (a_remote && k + 1 < K) rp.B[k].sm_cap = sms - nvl;
    if (b_remote && k >= 1) rp.A[k].sm_cap = sms - nvl;
  }
  return DFFT_SUCCESS;
}

}  // namespace

// ================================================================================ C ABI
extern "C" {

int dfft_version(void) { return DFFT_VERSION; }

long long dfft_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

const char* dfft_status_string(dfft_status_t s) {
  switch (s) {
    case DFFT_SUCCESS: return "success";
    case DFFT_ERR_INVALID_VALUE: return "invalid value";
    case DFFT_ERR_INFEASIBLE_DECOMP: return "infeasible decomposition";
    case DFFT_ERR_UNSUPPORTED: return "unsupported";
    case DFFT_ERR_ALLOC: return "allocation failed";
    case DFFT_ERR_CUDA: return "CUDA error";
    case DFFT_ERR_NCCL: return "NCCL error";
    case DFFT_ERR_INTERNAL: return "internal error";
    case DFFT_ERR_PEER: return "plan failed (a peer did not signal, or an enqueue failed)";
  }
  return "unknown status";
}

const char* dfft_last_error(void) { return g_err.c_str(); }

dfft_status_t dfft_get_unique_id(unsigned char id[128]) {
  if (!id) return fail(DFFT_ERR_INVALID_VALUE, "null id");
  ncclUniqueId u;
  NC(ncclGetUniqueId(&u));
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id, &u, 128);
  return DFFT_SUCCESS;
}

dfft_status_t dfft_comm_init(dfft_comm_t* comm, int nranks, int rank, const unsigned char id[128],
                             int cuda_device) {
  if (!comm || nranks < 1 || rank < 0 || rank >= nranks) return fail(DFFT_ERR_INVALID_VALUE, "bad comm args");
  if (nranks > 1 && !id) return fail(DFFT_ERR_INVALID_VALUE, "nranks > 1 needs a unique id");
  if (nranks > 1) CU(cudaSetDevice(cuda_device));
  auto* c = new dfft_comm_s;
  c->nranks = nranks;
  c->rank = rank;
  c->device = cuda_device;
  if (nranks > 1) {
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclResult_t r = ncclCommInitRank(&c->world, nranks, u, rank);
    if (r != ncclSuccess) {
      delete c;
      return fail(DFFT_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
  }
  *comm = c;
  return DFFT_SUCCESS;
}

dfft_status_t dfft_comm_init_sim(dfft_comm_t* comm, int nranks, int cuda_device) {
  if (!comm || nranks < 1) return fail(DFFT_ERR_INVALID_VALUE, "bad sim comm args");
  auto* c = new dfft_comm_s;
  c->nranks = nranks;
  c->device = cuda_device;
  c->sim = true;
  *comm = c;
  return DFFT_SUCCESS;
}

dfft_status_t dfft_comm_destroy(dfft_comm_t c) {
  if (!c) return DFFT_SUCCESS;
  for (auto& kv : c->sub) {
    if (kv.second.first) ncclCommDestroy(kv.second.first);
    if (kv.second.second) ncclCommDestroy(kv.second.second);
  }
  if (c->world) ncclCommDestroy(c->world);
  delete c;
  return DFFT_SUCCESS;
}

// argument validation shared by dfft_plan_create(_kinds) and dfft_decomp_box; maps slab to pencil 1×P
static dfft_status_t validate(int P, int64_t nx, int64_t ny, int64_t nz, dfft_decomp_t decomp, int* p1p, int* p2p,
                              dfft_type_t type, dfft_direction_t direction, const int* kinds = nullptr) {
  int p1 = *p1p, p2 = *p2p;
  if (nx <= 0 || ny <= 0 || nz <= 0) return fail(DFFT_ERR_INVALID_VALUE, "grid extents must be positive");
  if (direction != DFFT_FORWARD && direction != DFFT_INVERSE) return fail(DFFT_ERR_INVALID_VALUE, "bad direction");
  if (type < DFFT_C2C_F32 || type > DFFT_R2R_F64) return fail(DFFT_ERR_INVALID_VALUE, "bad type");
  if (decomp == DFFT_SLAB) {
    if (p2 != 1 || p1 != P) return fail(DFFT_ERR_INVALID_VALUE, "slab needs proc grid (nranks, 1)");
    p1 = 1;  // slab == pencil 1×P internally (z-slabs -> y-slabs)
    p2 = P;
  } else if (decomp != DFFT_PENCIL) {
    return fail(DFFT_ERR_INVALID_VALUE, "bad decomposition");
  }
  if (p1 < 1 || p2 < 1 || (long long)p1 * p2 != P)
    return fail(DFFT_ERR_INVALID_VALUE, "proc grid %d x %d != nranks %d", p1, p2, P);
  bool r2c = type == DFFT_R2C_F32 || type == DFFT_R2C_F64;
  bool r2r = type == DFFT_R2R_F32 || type == DFFT_R2R_F64;
  if (kinds) {  // per-axis kinds (reading R22): x DFT for C2C / R2C, DCT or DST for R2R; y, z any (R2R: not DFT)
    for (int d = 0; d < 3; ++d)
      if (kinds[d] < DFFT_KIND_DFT || kinds[d] > DFFT_KIND_DST2) return fail(DFFT_ERR_INVALID_VALUE, "bad kind on axis %d", d);
    if (!r2r && kinds[0] != DFFT_KIND_DFT)
      return fail(DFFT_ERR_UNSUPPORTED, "C2C / R2C plans take the DFT along x (bounded x needs an R2R plan)");
    if (r2r && (kinds[0] == DFFT_KIND_DFT || kinds[1] == DFFT_KIND_DFT || kinds[2] == DFFT_KIND_DFT))
      return fail(DFFT_ERR_UNSUPPORTED, "R2R plans take a DCT or DST on every axis (periodic x with bounded y/z: R2C)");
  }
  if (r2c && nx % 2) return fail(DFFT_ERR_UNSUPPORTED, "R2C needs even nx");
  if (r2r && (nx % 2 || ny % 2 || nz % 2))
    return fail(DFFT_ERR_UNSUPPORTED, "R2R (DCT/DST via Makhoul's permutation) needs even extents");
  for (int d = 1; d < 3; ++d)
    if (kinds && kinds[d] != DFFT_KIND_DFT && (d == 1 ? ny : nz) % 2)
      return fail(DFFT_ERR_UNSUPPORTED, "a DCT / DST axis needs an even extent");
  long long nxc = r2c ? nx / 2 + 1 : r2r ? nx / 2 : nx;
  long long nfft_x = (r2c || r2r) ? nx / 2 : nx;
  if (!length_ok(nfft_x) || !length_ok(ny) || !length_ok(nz))
    return fail(DFFT_ERR_UNSUPPORTED, "axis FFT lengths (%lld,%lld,%lld): each must be 2^a 3^b 5^c 7^d <= 4096",
                (long long)nfft_x, (long long)ny, (long long)nz);
  {  // R2C / R2R x axes and DCT / DST y, z axes run specialised kernels only
    const bool xs_need = r2c || r2r;
    const bool y_need = r2r || (kinds && kinds[1] != DFFT_KIND_DFT), z_need = r2r || (kinds && kinds[2] != DFFT_KIND_DFT);
    if ((xs_need && !length_specialised(nfft_x)) || (y_need && !length_specialised(ny)) ||
        (z_need && !length_specialised(nz)))
      return fail(DFFT_ERR_UNSUPPORTED, "R2C / R2R / DCT / DST axes need one of the specialised lengths (include/dfft.h)");
  }
  if (p1 > ny || p1 > nxc || p2 > nz || p2 > ny)
    return fail(DFFT_ERR_INFEASIBLE_DECOMP, "grid %d x %d leaves an empty block for (%lld,%lld,%lld)", p1, p2,
                (long long)nx, (long long)ny, (long long)nz);
  *p1p = p1;
  *p2p = p2;
  return DFFT_SUCCESS;
}

dfft_status_t dfft_decomp_box(int64_t nx, int64_t ny, int64_t nz, dfft_decomp_t decomp, int p1, int p2,
                              dfft_type_t type, dfft_direction_t direction, int rank, int which, int64_t lo[3],
                              int64_t n[3]) {
  if (!lo || !n) return fail(DFFT_ERR_INVALID_VALUE, "null argument");
  int P = decomp == DFFT_SLAB ? p1 : p1 * p2;
  ST(validate(P, nx, ny, nz, decomp, &p1, &p2, type, direction));
  if (rank < 0 || rank >= P) return fail(DFFT_ERR_INVALID_VALUE, "rank %d out of range", rank);
  bool r2c = type == DFFT_R2C_F32 || type == DFFT_R2C_F64;
  bool r2r = type == DFFT_R2R_F32 || type == DFFT_R2R_F64;
  Geo g{nx, ny, nz, r2c ? nx / 2 + 1 : r2r ? nx / 2 : nx, p1, p2, 1};
  long long i = rank / p2, j = rank % p2;
  const long long xs = r2r ? 2 : 1;  // R2R: x split in pairs of reals (complex-pair columns)
  int64_t d1lo[3] = {0, g.Y1lo(i), g.Zlo(j)}, d1n[3] = {nx, g.Y1n(i), g.Zn(j)};
  int64_t d3lo[3] = {xs * g.Xlo(i), g.Y3lo(j), 0}, d3n[3] = {xs * g.Xn(i), g.Y3n(j), nz};
  bool d1 = (which == 0) == (direction == DFFT_FORWARD);
  memcpy(lo, d1 ? d1lo : d3lo, sizeof d1lo);
  memcpy(n, d1 ? d1n : d3n, sizeof d1n);
  return DFFT_SUCCESS;
}


dfft_status_t dfft_plan_create(dfft_plan_t* plan, dfft_comm_t comm, int64_t nx, int64_t ny, int64_t nz,
                               dfft_decomp_t decomp, int p1, int p2, dfft_type_t type, dfft_direction_t direction,
                               uint64_t flags) {
  const bool r2r = type == DFFT_R2R_F32 || type == DFFT_R2R_F64;
  const int kinds[3] = {r2r ? DFFT_KIND_DCT2 : DFFT_KIND_DFT, r2r ? DFFT_KIND_DCT2 : DFFT_KIND_DFT,
                        r2r ? DFFT_KIND_DCT2 : DFFT_KIND_DFT};
  return dfft_plan_create_kinds(plan, comm, nx, ny, nz, decomp, p1, p2, type, kinds, direction, flags);
}

dfft_status_t dfft_plan_create_kinds(dfft_plan_t* plan, dfft_comm_t comm, int64_t nx, int64_t ny, int64_t nz,
                                     dfft_decomp_t decomp, int p1, int p2, dfft_type_t type, const int kinds[3],
                                     dfft_direction_t direction, uint64_t flags) {
  if (!plan || !comm || !kinds) return fail(DFFT_ERR_INVALID_VALUE, "null plan/comm/kinds");
  *plan = nullptr;
  int P = comm->nranks;
  ST(validate(P, nx, ny, nz, decomp, &p1, &p2, type, direction, kinds));
  bool r2c = type == DFFT_R2C_F32 || type == DFFT_R2C_F64;
  bool r2r = type == DFFT_R2R_F32 || type == DFFT_R2R_F64;
  bool f64 = type == DFFT_C2C_F64 || type == DFFT_R2C_F64 || type == DFFT_R2R_F64;
  long long nxc = r2c ? nx / 2 + 1 : r2r ? nx / 2 : nx;
  int Kreq = (int)(flags & 0xff);
  bool overlap = !(flags & DFFT_FLAG_NO_OVERLAP);
  long long kmax = direction == DFFT_FORWARD ? nz / p2 : nxc / p1;  // chunk axis extent
  // exchange transport for P > 1: fused epilogue stores into the peers' IPC
  // windows (default; DFFT_FLAG_FUSED_STORE), copy engines into the windows (DFFT_FLAG_CE), CE
  // with a fused forward x-FFT (DFFT_FLAG_HYBRID), or NCCL send/recv (DFFT_FLAG_NCCL)
  const char* exch_env = getenv("DFFT_EXCHANGE");
  auto env_is = [&](const char* v) { return exch_env && strcmp(exch_env, v) == 0; };
  const bool want_fused = (flags & DFFT_FLAG_FUSED_STORE) || (!comm->sim && env_is("p2p"));
  const bool want_ce = (flags & DFFT_FLAG_CE) || (!comm->sim && env_is("ce"));
  const bool want_hybrid = (flags & DFFT_FLAG_HYBRID) || (!comm->sim && env_is("hybrid"));
  // simulated ranks run the NCCL layouts, or (DFFT_FLAG_FUSED_STORE / _CE / _HYBRID) the IPC-window
  // layouts and schedules with every rank's workspace standing in for its window
  const bool nccl_mode =
      (comm->sim && !want_fused && !want_ce && !want_hybrid) || P == 1 || (flags & DFFT_FLAG_NCCL) || env_is("nccl");
  // automatic choice (measured r01, 1024^3 c64): fused epilogue stores into column-blocked
  // windows beat the copy engine on every grid (1x2: 16.1 vs 18.0 ms, 2x2: 9.4 vs 16.9 ms)
  const bool auto_fused = !comm->sim && !want_ce && !want_fused && !want_hybrid;
  const bool p2p_mode = !nccl_mode && (want_fused || auto_fused);
  const bool ce_only = !nccl_mode && !p2p_mode && !want_hybrid;
  const bool ce_mode = !nccl_mode && !p2p_mode;
  // chunks pipeline the transfers against the FFTs; with fused stores the transfer happens
  // inside the FFT kernels themselves, so one chunk is the default there
  long long K = Kreq > 0 ? Kreq : (P > 1 && !p2p_mode ? (nccl_mode ? 4 : 8) : 1);
  // B→C pipeline whenever stage B stores to peers and stage C is local: both exchanges remote,
  // or a 1×P2 forward (x-FFT local, y-FFT to the column peers, z-FFT local); DFFT_NO_BC=1 off
  const bool bc_mode = p2p_mode && !getenv("DFFT_NO_BC") && p2 > 1 &&
                       (p1 > 1 || (direction == DFFT_FORWARD && !getenv("DFFT_NO_BC_1XP")));
  // r01 sweeps: with bulk-copy epilogues the NVLink-bound stage of a pair keeps
  // ~95 % of its rate on 80 SMs, so pairing it with a local stage pays: B(k)‖C(k−1) when both
  // exchanges are remote (2x2: 9.0 -> 8.1 ms) or on a 1×P2 forward
  // chunks cost launches and flag round trips: pipeline only boxes of >= 256 MiB per rank
  // (1024^3 c64 on 2-8 GPUs: 1-4 GiB), small problems (cfg2/cfg3) run one chunk
  const double local_bytes = (double)nxc * ny * nz / P * (f64 ? 16.0 : 8.0);
  // 1×P2 grids also pipeline the inverse (z-IFFT to the peers ‖ local y-IFFT, two streams):
  // 1x2 1024^3 c64 fwd+inv 14.6 -> 12.6 ms with K = 4 and the NVLink stage on 80 SMs
  // (sweep: 4 chunks from 1 GiB per rank, 2 from 256 MiB — cfg5 2x2 2.63 -> 2.50 ms — else 1)
  if (p2p_mode && Kreq == 0)
    K = !(bc_mode || (p1 == 1 && p2 > 1)) ? 1
        : local_bytes >= 1024.0 * (1 << 20) ? 4
        : local_bytes >= 256.0 * (1 << 20)  ? 2
                                             : 1;
  if (bc_mode) kmax = direction == DFFT_FORWARD ? nxc / p1 : nz / p2;
  K = std::max<long long>(1, std::min<long long>(K, kmax));
  if (P == 1) K = 1;  // nothing to overlap

  CU(cudaSetDevice(comm->device));
  dfft_plan_t pl = new dfft_plan_s;
  PlanGuard guard{pl};
  pl->comm = comm;
  pl->nx = nx;
  pl->ny = ny;
  pl->nz = nz;
  pl->P1 = p1;
  pl->P2 = p2;
  pl->K = (int)K;
  pl->dir = direction;
  pl->f64 = f64;
  pl->r2c = r2c;
  pl->r2r = r2r;
  for (int d = 0; d < 3; ++d) pl->kind[d] = kinds[d];
  pl->overlap = overlap;
  pl->es = f64 ? 16 : 8;
  // exchange over NVLink peer memory unless asked for NCCL (flag or DFFT_EXCHANGE=nccl)
  pl->p2p = p2p_mode;
  pl->ce = ce_mode;
  pl->hybrid = ce_mode && !ce_only;
  pl->bc = bc_mode;
  if ((pl->p2p || pl->ce) && !stream_wait_value32())
    return fail(DFFT_ERR_UNSUPPORTED, "cuStreamWaitValue32 unavailable");
  Geo g{nx, ny, nz, nxc, p1, p2, K};
  {  // column-tile widths of the strided kernels (the TMA kernel's when it exists)
    KernelInfo ky, kz;
    if (f64 ? lookup_kernel_f64(kStrided, (int)ny, direction, &ky) : lookup_kernel_f32(kStrided, (int)ny, direction, &ky))
      g.wy = ky.tma_fn ? ky.tma_w : ky.per_cta;
    if (f64 ? lookup_kernel_f64(kStrided, (int)nz, direction, &kz) : lookup_kernel_f32(kStrided, (int)nz, direction, &kz))
      g.wz = kz.tma_fn ? kz.tma_w : kz.per_cta;
  }
  // chunk bounds along x at multiples of both column-block widths, so every chunk is a whole
  // number of blocks of each window layout (R2 by wy, R2' by wz, R1' by wy)
  if (p2p_mode) g.xq = std::lcm(g.wy, g.wz);

  if (!comm->sim && P > 1) {  // row / column sub-communicators, shared by the comm's plans
    auto key = std::make_pair(p1, p2);
    auto it = comm->sub.find(key);
    if (it == comm->sub.end()) {
      int i = comm->rank / p2, j = comm->rank % p2;
      ncclComm_t row = nullptr, col = nullptr;
      NC(ncclCommSplit(comm->world, j, i, &row, nullptr));
      NC(ncclCommSplit(comm->world, i, j, &col, nullptr));
      it = comm->sub.emplace(key, std::make_pair(row, col)).first;
    }
    pl->row = it->second.first;
    pl->col = it->second.second;
  }

  int nr = comm->sim ? P : 1;
  pl->ranks.resize(nr);
  for (int q = 0; q < nr; ++q) {
    RankPlan& rp = pl->ranks[q];
    rp.rank = comm->sim ? q : comm->rank;
    rp.i = rp.rank / p2;
    rp.j = rp.rank % p2;
    // D1 = (x whole, y by i, z by j);  D3 = (x by i, y by j, z whole)
    int64_t d1lo[3] = {0, g.Y1lo(rp.i), g.Zlo(rp.j)}, d1n[3] = {nx, g.Y1n(rp.i), g.Zn(rp.j)};
    // R2R boxes are real on both sides; x splits in pairs (complex-pair columns of the kernels)
    const long long xs = r2r ? 2 : 1;
    int64_t d3lo[3] = {xs * g.Xlo(rp.i), g.Y3lo(rp.j), 0}, d3n[3] = {xs * g.Xn(rp.i), g.Y3n(rp.j), nz};
    size_t real_es = pl->es / 2;
    size_t d1b = (size_t)(d1n[0] * d1n[1] * d1n[2]) * ((r2c || r2r) ? real_es : pl->es);
    size_t d3b = (size_t)(d3n[0] * d3n[1] * d3n[2]) * (r2r ? real_es : pl->es);
    if (direction == DFFT_FORWARD) {
      memcpy(rp.in_lo, d1lo, sizeof d1lo);
      memcpy(rp.in_n, d1n, sizeof d1n);
      memcpy(rp.out_lo, d3lo, sizeof d3lo);
      memcpy(rp.out_n, d3n, sizeof d3n);
      rp.in_bytes = d1b;
      rp.out_bytes = d3b;
      ST(P == 1 ? build_single(pl, g, rp)
                : pl->bc ? build_forward_bc(pl, g, rp) : build_forward(pl, g, rp));
    } else {
      memcpy(rp.in_lo, d3lo, sizeof d3lo);
      memcpy(rp.in_n, d3n, sizeof d3n);
      memcpy(rp.out_lo, d1lo, sizeof d1lo);
      memcpy(rp.out_n, d1n, sizeof d1n);
      rp.in_bytes = d3b;
      rp.out_bytes = d1b;
      ST(P == 1 ? build_single(pl, g, rp)
                : pl->bc ? build_inverse_bc(pl, g, rp) : build_inverse(pl, g, rp));
    }
    ST(apply_sm_caps(pl, rp));
    build_schedule(pl, rp);
    if (rp.ws_bytes) {
      cudaError_t e = cudaMalloc(&rp.ws, rp.ws_bytes);
      if (e != cudaSuccess) return fail(DFFT_ERR_ALLOC, "workspace of %zu bytes: %s", rp.ws_bytes, cudaGetErrorString(e));
    }
    if (pl->p2p || pl->ce) {  // flag block: READY = 0, DONE = 1 (before any peer can see the window)
      const std::vector<unsigned int> fl = initial_flags(pl);
      CU(cudaMemcpy((char*)rp.ws + pl->flag_off, fl.data(), fl.size() * 4, cudaMemcpyHostToDevice));
    }
    if (two_streams(pl)) {
      CU(cudaStreamCreateWithFlags(&rp.sX, cudaStreamNonBlocking));
      CU(cudaStreamCreateWithFlags(&rp.sY, cudaStreamNonBlocking));
      CU(cudaEventCreateWithFlags(&rp.ev_fork, cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&rp.ev_join[0], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&rp.ev_join[1], cudaEventDisableTiming));
      rp.ev.resize(rp.nev);
      for (auto& e : rp.ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
  }
  {  // hash of the resolved plan state: transport, pipeline, chunking, window layout, schedule
    unsigned long long h = 1469598103934665603ULL;
    auto mix = [&](long long v) {
      h ^= (unsigned long long)v;
      h *= 1099511628211ULL;
    };
    for (long long v : {(long long)nx, (long long)ny, (long long)nz, (long long)decomp, (long long)p1, (long long)p2,
                        (long long)type, (long long)direction, (long long)flags, (long long)pl->p2p, (long long)pl->ce,
                        (long long)pl->hybrid, (long long)pl->bc, (long long)pl->overlap, K, g.wy, g.wz, g.xq,
                        (long long)pl->flag_off, (long long)pl->ranks[0].sched.size(), (long long)pl->kind[0],
                        (long long)pl->kind[1], (long long)pl->kind[2]})
      mix(v);
    pl->hash = h;
  }
  if (!comm->sim && P > 1) {
    // collective consistency check: every rank must resolve an identical plan (arguments, flags,
    // and the env-dependent transport / pipeline choices), else peers would address the wrong
    // window offsets or wait on flags that never come
    unsigned long long* d = nullptr;
    CU(cudaMalloc(&d, sizeof(unsigned long long) * (P + 1)));
    CU(cudaMemcpy(d, &pl->hash, sizeof pl->hash, cudaMemcpyHostToDevice));
    NC(ncclAllGather(d, d + 1, 1, ncclUint64, comm->world, 0));
    std::vector<unsigned long long> all(P);
    CU(cudaMemcpy(all.data(), d + 1, sizeof(unsigned long long) * P, cudaMemcpyDeviceToHost));
    cudaFree(d);
    for (int r = 0; r < P; ++r)
      if (all[r] != pl->hash)
        return fail(DFFT_ERR_INVALID_VALUE, "plan differs between rank %d and rank %d (arguments, flags or DFFT_* env)",
                    comm->rank, r);
  }
  if (comm->sim && (pl->p2p || pl->ce)) {
    // simulated windows: rank q's "window" is its workspace on this device
    pl->peer_ws.resize(P);
    for (int q = 0; q < P; ++q) pl->peer_ws[q] = pl->ranks[q].ws;
  } else if (pl->p2p || pl->ce) {
    // every workspace becomes an IPC window; open the windows of the row and column peers
    RankPlan& rp = pl->ranks[0];
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, rp.ws));
    char* d = nullptr;
    CU(cudaMalloc(&d, sizeof(h) * (P + 1)));
    CU(cudaMemcpy(d, &h, sizeof(h), cudaMemcpyHostToDevice));
    NC(ncclAllGather(d, d + sizeof(h), sizeof(h), ncclUint8, comm->world, 0));
    std::vector<cudaIpcMemHandle_t> all(P);
    CU(cudaMemcpy(all.data(), d + sizeof(h), sizeof(h) * P, cudaMemcpyDeviceToHost));
    cudaFree(d);
    pl->peer_ws.assign(P, nullptr);
    pl->peer_ws[comm->rank] = rp.ws;
    for (int r = 0; r < P; ++r) {
      int ri = r / p2, rj = r % p2;
      if (r == comm->rank || (ri != rp.i && rj != rp.j)) continue;  // only row and column peers
      cudaError_t e = cudaIpcOpenMemHandle(&pl->peer_ws[r], all[r], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return fail(DFFT_ERR_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
    }
  }
  CU(cudaDeviceSynchronize());
  guard.p = nullptr;
  *plan = pl;
  return DFFT_SUCCESS;
}

dfft_status_t dfft_plan_box_rank(dfft_plan_t pl, int rank, int which, int64_t lo[3], int64_t n[3]) {
  if (!pl || !lo || !n) return fail(DFFT_ERR_INVALID_VALUE, "null argument");
  int idx = pl->comm->sim ? rank : 0;
  if (idx < 0 || idx >= (int)pl->ranks.size() || (!pl->comm->sim && rank != pl->comm->rank))
    return fail(DFFT_ERR_INVALID_VALUE, "rank %d not held by this plan", rank);
  const RankPlan& rp = pl->ranks[idx];
  memcpy(lo, which ? rp.out_lo : rp.in_lo, 3 * sizeof(int64_t));
  memcpy(n, which ? rp.out_n : rp.in_n, 3 * sizeof(int64_t));
  return DFFT_SUCCESS;
}

dfft_status_t dfft_plan_box(dfft_plan_t pl, int which, int64_t lo[3], int64_t n[3]) {
  if (!pl) return fail(DFFT_ERR_INVALID_VALUE, "null plan");
  return dfft_plan_box_rank(pl, pl->comm->sim ? 0 : pl->comm->rank, which, lo, n);
}

dfft_status_t dfft_plan_bytes(dfft_plan_t pl, size_t* in_bytes, size_t* out_bytes, size_t* ws_bytes) {
  if (!pl) return fail(DFFT_ERR_INVALID_VALUE, "null plan");
  const RankPlan& rp = pl->ranks[0];
  if (in_bytes) *in_bytes = rp.in_bytes;
  if (out_bytes) *out_bytes = rp.out_bytes;
  if (ws_bytes) {
    size_t w = 0;
    for (auto& r : pl->ranks) w += r.ws_bytes;
    *ws_bytes = w;
  }
  return DFFT_SUCCESS;
}

dfft_status_t dfft_plan_chunks(dfft_plan_t pl, int* chunks) {
  if (!pl || !chunks) return fail(DFFT_ERR_INVALID_VALUE, "null argument");
  *chunks = pl->K;
  return DFFT_SUCCESS;
}

static dfft_status_t check_ptrs(dfft_plan_t pl, const RankPlan& rp, const void* in, void* out) {
  if (!in || !out) return fail(DFFT_ERR_INVALID_VALUE, "null buffer");
  if (((uintptr_t)in | (uintptr_t)out) & 15) return fail(DFFT_ERR_INVALID_VALUE, "buffers must be 16-byte aligned");
  const char *a = (const char*)in, *b = (const char*)out;
  if (a < b + rp.out_bytes && b < a + rp.in_bytes) return fail(DFFT_ERR_INVALID_VALUE, "in and out overlap");
  (void)pl;
  return DFFT_SUCCESS;
}

static dfft_status_t check_usable(dfft_plan_t pl) {
  if (pl->failed.load()) return fail(DFFT_ERR_PEER, "plan failed earlier: %s", pl->fail_msg.c_str());
  if (pl->comm->world && !pl->p2p && !pl->ce && pl->comm->nranks > 1) {
    ncclResult_t ar = ncclSuccess;
    NC(ncclCommGetAsyncError(pl->comm->world, &ar));
    if (ar != ncclSuccess) return fail(DFFT_ERR_NCCL, "NCCL asynchronous error: %s", ncclGetErrorString(ar));
  }
  return DFFT_SUCCESS;
}

dfft_status_t dfft_execute(dfft_plan_t pl, const void* in, void* out, void* stream) {
  if (!pl) return fail(DFFT_ERR_INVALID_VALUE, "null plan");
  if (pl->comm->sim) return fail(DFFT_ERR_INVALID_VALUE, "simulated-comm plan: use dfft_execute_sim");
  ST(check_usable(pl));
  ST(check_ptrs(pl, pl->ranks[0], in, out));
  CU(cudaSetDevice(pl->comm->device));
  ST(execute_rank(pl, in, out, (cudaStream_t)stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DFFT_ERR_CUDA, "launch: %s", cudaGetErrorString(e));
  return wd_track(pl, (cudaStream_t)stream);
}

static bool host_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

dfft_status_t dfft_execute_host_chain(const dfft_plan_t* plans, int nplans, const void* in_host, void* out_host,
                                      void* stream, int async) {
  if (!plans || nplans < 1 || !in_host || !out_host) return fail(DFFT_ERR_INVALID_VALUE, "null argument");
  for (int q = 0; q < nplans; ++q) {
    if (!plans[q]) return fail(DFFT_ERR_INVALID_VALUE, "null plan %d", q);
    if (plans[q]->comm->sim) return fail(DFFT_ERR_INVALID_VALUE, "simulated-comm plan");
    if (plans[q]->comm->device != plans[0]->comm->device) return fail(DFFT_ERR_INVALID_VALUE, "plans on different devices");
    if (q > 0 && plans[q]->ranks[0].in_bytes != plans[q - 1]->ranks[0].out_bytes)
      return fail(DFFT_ERR_INVALID_VALUE, "plan %d's input box does not match plan %d's output box", q, q - 1);
  }
  if (async && (!host_pinned(in_host) || !host_pinned(out_host)))
    return fail(DFFT_ERR_INVALID_VALUE, "asynchronous host execution needs page-locked (pinned) host buffers");
  dfft_plan_t p0 = plans[0];
  CU(cudaSetDevice(p0->comm->device));
  const size_t in_b = std::max<size_t>(p0->ranks[0].in_bytes, 16);
  const size_t out_b = std::max<size_t>(plans[nplans - 1]->ranks[0].out_bytes, 16);
  dfft_plan_s::HostChain* h = p0->host;
  if (h && h->plans != std::vector<dfft_plan_s*>(plans, plans + nplans)) {  // another chain: rebuild
    free_host_chain(p0);
    h = nullptr;
  }
  if (!h) {
    h = p0->host = new dfft_plan_s::HostChain;
    h->plans.assign(plans, plans + nplans);
    for (int b = 0; b < 2; ++b) {
      CU(cudaMalloc(&h->in_dev[b], in_b));
      CU(cudaMalloc(&h->out_dev[b], out_b));
      for (cudaEvent_t* e : {&h->in_ready[b], &h->in_free[b], &h->out_ready[b], &h->out_done[b]})
        CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    for (int q = 0; q + 1 < nplans; ++q) {
      void* m = nullptr;
      CU(cudaMalloc(&m, std::max<size_t>(plans[q]->ranks[0].out_bytes, 16)));
      h->mid.push_back(m);
    }
    CU(cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking));
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int b = (int)(h->calls++ & 1);
  // host -> device on the copy stream, once the call two back has consumed this buffer
  CU(cudaStreamWaitEvent(h->h2d, h->in_free[b], 0));
  CU(cudaMemcpyAsync(h->in_dev[b], in_host, p0->ranks[0].in_bytes, cudaMemcpyHostToDevice, h->h2d));
  CU(cudaEventRecord(h->in_ready[b], h->h2d));
  CU(cudaStreamWaitEvent(st, h->in_ready[b], 0));
  for (int q = 0; q < nplans; ++q) {
    const void* src = q == 0 ? h->in_dev[b] : h->mid[q - 1];
    void* dst = q + 1 == nplans ? h->out_dev[b] : h->mid[q];
    ST(dfft_execute(plans[q], src, dst, stream));
    if (q == 0) CU(cudaEventRecord(h->in_free[b], st));
  }
  // device -> host on the other copy stream; the caller's stream completes when it has landed
  CU(cudaEventRecord(h->out_ready[b], st));
  CU(cudaStreamWaitEvent(h->d2h, h->out_ready[b], 0));
  CU(cudaMemcpyAsync(out_host, h->out_dev[b], plans[nplans - 1]->ranks[0].out_bytes, cudaMemcpyDeviceToHost, h->d2h));
  CU(cudaEventRecord(h->out_done[b], h->d2h));
  CU(cudaStreamWaitEvent(st, h->out_done[b], 0));
  if (!async) CU(cudaStreamSynchronize(st));
  return DFFT_SUCCESS;
}

dfft_status_t dfft_execute_host(dfft_plan_t pl, const void* in_host, void* out_host, void* stream) {
  if (!pl) return fail(DFFT_ERR_INVALID_VALUE, "null plan");
  return dfft_execute_host_chain(&pl, 1, in_host, out_host, stream, 0);
}

dfft_status_t dfft_execute_sim(dfft_plan_t pl, const void* const* ins, void* const* outs, void* stream) {
  if (!pl || !ins || !outs) return fail(DFFT_ERR_INVALID_VALUE, "null argument");
  if (!pl->comm->sim) return fail(DFFT_ERR_INVALID_VALUE, "not a simulated-comm plan");
  ST(check_usable(pl));
  const bool windows = pl->p2p || pl->ce;
  for (size_t r = 0; r < pl->ranks.size(); ++r) {
    if (!ins[r] && windows) continue;  // a failed (non-executing) simulated peer
    ST(check_ptrs(pl, pl->ranks[r], ins[r], outs[r]));
  }
  CU(cudaSetDevice(pl->comm->device));
  ST(execute_sim(pl, ins, outs, (cudaStream_t)stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DFFT_ERR_CUDA, "launch: %s", cudaGetErrorString(e));
  return wd_track(pl, (cudaStream_t)stream);
}

dfft_status_t dfft_plan_set_poisson(dfft_plan_t pl, double dx, double dy, double dz) {
  if (!pl) return fail(DFFT_ERR_INVALID_VALUE, "null plan");
  if (pl->dir != DFFT_FORWARD) return fail(DFFT_ERR_INVALID_VALUE, "the Poisson multiplier belongs to a forward plan");
  const bool on = dx > 0 && dy > 0 && dz > 0;
  if (!on && (dx != 0 || dy != 0 || dz != 0))
    return fail(DFFT_ERR_INVALID_VALUE, "grid spacings must all be > 0 (or all 0 to switch the multiplier off)");
  CU(cudaSetDevice(pl->comm->device));
  CU(cudaDeviceSynchronize());  // no execute of this plan may be reading the old tables
  drop_graphs(pl);  // the captured kernels carry the old multiplier tables
  if (pl->spec_tab) cudaFree(pl->spec_tab);
  pl->spec_tab = nullptr;
  const long long n[3] = {pl->nx, pl->ny, pl->nz};
  const double h[3] = {dx, dy, dz};
  const size_t rs = pl->es / 2;
  if (on) {
    // λ_d(k) = -(2 sin(θ_k)/h_d)² with θ_k = πk/n_d (periodic, DFT), πk/(2n_d) (Neumann, DCT-II) or
    // π(k+1)/(2n_d) (Dirichlet, DST-II); long double, rounded once to the plan's precision (R20, R22),
    // one entry per output bin of the axis (for R2R x: per real bin; see PassArgs::spec_pairs)
    std::vector<unsigned char> host((size_t)(n[0] + n[1] + n[2]) * rs);
    long long o = 0;
    for (int d = 0; d < 3; ++d)
      for (long long k = 0; k < n[d]; ++k, ++o) {
        const long double PI = 3.14159265358979323846264338327950288L;
        const long double ang = pl->kind[d] == DFFT_KIND_DFT    ? PI * (long double)k / (long double)n[d]
                                : pl->kind[d] == DFFT_KIND_DCT2 ? PI * (long double)k / (long double)(2 * n[d])
                                                                : PI * (long double)(k + 1) / (long double)(2 * n[d]);
        const long double sv = 2.0L * sinl(ang) / (long double)h[d];
        const long double lam = -(sv * sv);
        if (pl->f64) reinterpret_cast<double*>(host.data())[o] = (double)lam;
        else reinterpret_cast<float*>(host.data())[o] = (float)lam;
      }
    CU(cudaMalloc(&pl->spec_tab, host.size()));
    CU(cudaMemcpy(pl->spec_tab, host.data(), host.size(), cudaMemcpyHostToDevice));
  }
  const long long base[3] = {0, n[0], n[0] + n[1]};
  int nlast = 0;
  for (RankPlan& rp : pl->ranks) {
    std::vector<Stage*> st{&rp.C};
    for (Stage& c : rp.Cc) st.push_back(&c);
    for (Stage* s : st) {
      if (!s->last_fwd) continue;
      ++nlast;
      // R2R: the stage's x index counts pairs of reals, the x table real bins (offset ×2)
      const bool pairs = pl->r2r;
      s->a.spec_pairs = pairs ? 1 : 0;
      for (int q = 0; q < 3; ++q) {
        const long long off = (pairs && s->gax[q] == 0 ? 2 : 1) * s->glo[q];
        s->a.spec[q] = on ? (const void*)((const char*)pl->spec_tab + (size_t)(base[s->gax[q]] + off) * rs) : nullptr;
      }
    }
  }
  if (nlast == 0) return fail(DFFT_ERR_INTERNAL, "plan has no last forward stage");
  return DFFT_SUCCESS;
}

dfft_status_t dfft_plan_set_profiling(dfft_plan_t pl, int on) {
  if (!pl) return fail(DFFT_ERR_INVALID_VALUE, "null plan");
  pl->prof = on != 0;
  return DFFT_SUCCESS;
}

dfft_status_t dfft_plan_phase_times(dfft_plan_t pl, double ms[5], long long launches[5], int reset) {
  if (!pl || !ms) return fail(DFFT_ERR_INVALID_VALUE, "null argument");
  ST(prof_resolve(pl));
  if (reset) pl->prof_spans.clear();
  for (int q = 0; q < 5; ++q) {
    ms[q] = pl->prof_ms[q];
    if (launches) launches[q] = pl->prof_n[q];
    if (reset) {
      pl->prof_ms[q] = 0;
      pl->prof_n[q] = 0;
    }
  }
  return DFFT_SUCCESS;
}

dfft_status_t dfft_plan_timeline(dfft_plan_t pl, dfft_span_t* spans, int cap, int* n) {
  if (!pl || !n || (cap > 0 && !spans)) return fail(DFFT_ERR_INVALID_VALUE, "null argument");
  ST(prof_resolve(pl));
  *n = (int)pl->prof_spans.size();
  if (cap <= 0) return DFFT_SUCCESS;  // size query
  const int m = std::min(cap, *n);
  std::copy(pl->prof_spans.begin(), pl->prof_spans.begin() + m, spans);
  pl->prof_spans.erase(pl->prof_spans.begin(), pl->prof_spans.begin() + m);
  *n = m;
  return DFFT_SUCCESS;
}

dfft_status_t dfft_set_timeout_ms(long long ms) {
  if (ms <= 0) return fail(DFFT_ERR_INVALID_VALUE, "timeout must be positive");
  g_timeout_ms.store(ms);
  return DFFT_SUCCESS;
}

dfft_status_t dfft_plan_status(dfft_plan_t pl) {
  if (!pl) return fail(DFFT_ERR_INVALID_VALUE, "null plan");
  return check_usable(pl);
}

dfft_status_t dfft_plan_stage_bytes(dfft_plan_t pl, double bytes[5]) {
  if (!pl || !bytes) return fail(DFFT_ERR_INVALID_VALUE, "null argument");
  const RankPlan& rp = pl->ranks[0];
  // algorithmic bytes per execute of each phase: every stage reads and writes its local
  // array once; every exchange sends its off-rank blocks (the bytes that cross NVLink)
  auto stage_b = [&](const Stage& s) {
    if (s.empty) return 0.0;
    double elems = (double)s.a.L0 * (double)s.a.L1 * (double)s.n;  // complex elements of the FFT
    if (s.family == kContigXZ8) elems *= 8;                             // a (l0, l1) pair is 8 lines
    return 2.0 * elems * (double)pl->es;
  };
  // off-rank bytes of each exchange from the rank's boxes (identical for every transport; with
  // fused stores they leave inside stage A's resp. stage B's epilogue)
  const bool fwd = pl->dir == DFFT_FORWARD;
  const int64_t* d1 = fwd ? rp.in_n : rp.out_n;  // (nx, Y1n, Zn)
  const int64_t* d3 = fwd ? rp.out_n : rp.in_n;  // (Xn, Y3n, nz)
  const double nxc = pl->r2c ? (double)(pl->nx / 2 + 1) : pl->r2r ? (double)(pl->nx / 2) : (double)pl->nx;
  const double Xn = (double)d3[0] / (pl->r2r ? 2.0 : 1.0), Y3n = (double)d3[1];
  const double Y1n = (double)d1[1], Zn = (double)d1[2];
  const double es = (double)pl->es;
  for (int q = 0; q < 5; ++q) bytes[q] = 0;
  if (fwd) {
    bytes[1] = Y1n * Zn * (nxc - Xn) * es;
    bytes[3] = Xn * Zn * ((double)pl->ny - Y3n) * es;
  } else {
    bytes[1] = Xn * Y3n * ((double)pl->nz - Zn) * es;
    bytes[3] = Xn * Zn * ((double)pl->ny - Y1n) * es;
  }
  for (size_t k = 0; k < rp.A.size(); ++k) {
    bytes[0] += stage_b(rp.A[k]);
    bytes[2] += stage_b(rp.B[k]);
  }
  bytes[4] = stage_b(rp.C);
  for (const Stage& c : rp.Cc) bytes[4] += stage_b(c);
  return DFFT_SUCCESS;
}

dfft_status_t dfft_plan_describe(dfft_plan_t pl, char* buf, size_t len) {
  if (!pl || !buf || len == 0) return fail(DFFT_ERR_INVALID_VALUE, "null argument");
  static const char* fam[] = {"contig", "strided", "contig_r2c", "contig_c2r", "contig_dct", "strided_dct",
                              "contig_dst", "strided_dst", "xz8"};
  const RankPlan& rp = pl->ranks[0];
  std::string out;
  auto one = [&](const char* phase, const Stage& s) {
    if (s.empty || s.n == 0) return;  // (n = 0: a stage the plan runs as chunks, rp.Cc)
    char line[256];
    const int f = s.family >= 0 && s.family <= kContigXZ8 ? s.family : 0;
    // maxr: the largest radix of the kernel that runs (contig / xz8: its own; strided: the TMA variant's)
    const int maxr = is_contig(s.family) || s.tma_variant == 1 ? s.k.tma_maxr : 16;
    snprintf(line, sizeof line, "%s %s n=%d L0=%lld L1=%lld in_tstride=%lld out_tstride=%lld tma=%d maxr=%d\n",
             phase, fam[f], s.n, s.a.L0, s.a.L1, s.a.in.tstride, s.a.out.tstride, s.tma_variant, maxr);
    out += line;
  };
  for (const Stage& s : rp.A) one("stage_A", s);
  for (const Stage& s : rp.B) one("stage_B", s);
  one("stage_C", rp.C);
  for (const Stage& s : rp.Cc) one("stage_C", s);
  snprintf(buf, len, "%s", out.c_str());
  return out.size() < len ? DFFT_SUCCESS : fail(DFFT_ERR_INVALID_VALUE, "buffer of %zu bytes too small", len);
}

dfft_status_t dfft_destroy(dfft_plan_t pl) {
  free_plan(pl);
  return DFFT_SUCCESS;
}

dfft_status_t dfft_fft1d(const void* in, void* out, int64_t n, int64_t howmany, int f64, int sign, void* stream) {
  if (!in || !out || n <= 0 || howmany <= 0 || (sign != -1 && sign != 1))
    return fail(DFFT_ERR_INVALID_VALUE, "bad fft1d arguments");
  if (!length_ok(n)) return fail(DFFT_ERR_UNSUPPORTED, "length %lld not supported", (long long)n);
  int dev = 0;
  CU(cudaGetDevice(&dev));
  Stage s;
  ST(get_kernel(kContig, (int)n, f64 != 0, sign, &s.k));
  ST(get_twiddles((int)n, f64 != 0, sign, dev, &s.a.tw, s.k.tma_maxr));
  if (s.k.generic) {
    s.a.gen = make_sched((int)n);
    s.a.gen_per = s.k.per_cta;
  }
  s.a.in.base = const_cast<void*>(in);
  s.a.out.base = out;
  set_side(s.a.in, 1, n, 0);
  set_side(s.a.out, 1, n, 0);
  s.a.L0 = howmany;
  s.a.L1 = 1;
  s.a.scale = 1.0;
  long long grid = (howmany + s.k.per_cta - 1) / s.k.per_cta;
  void* args[] = {&s.a};
  CU(cudaLaunchKernel(s.k.fn, dim3((unsigned)grid), dim3(s.k.threads), args, s.k.smem, (cudaStream_t)stream));
  return DFFT_SUCCESS;
}

}  // extern "C"

// ------------------------------------------------------------------------------ registry helpers
namespace dfft {
bool length_specialised(long long n) {
  switch (n) {
#define DFFT_LCASE(N) case N:
    DFFT_LENGTHS(DFFT_LCASE)
#undef DFFT_LCASE
    return true;
    default:
      return false;
  }
}
bool length_supported(long long n) {
  if (n <= 0 || n > 4096) return false;
  long long m = n;
  for (long long p : {2, 3, 5, 7})
    while (m % p == 0) m /= p;
  return m == 1;
}
int length_schedule(int n, int rad[kMaxPass], int maxr) {
  Sched s = make_sched(n, maxr);
  for (int p = 0; p < kMaxPass; ++p) rad[p] = s.rad[p];
  return s.npass;
}
}  // namespace dfft
