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
#include <map>
#include <mutex>
#include <string>
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
bool g_use_tma2 = getenv("DFFT_TMA2") != nullptr;  // two-group variant: correct, not faster
bool g_use_bulk = getenv("DFFT_NO_BULK") == nullptr;  // bulk-copy epilogue for blocked segmented outputs
// TMA-store kernels: the work-buffer flow (OM 1) is the default; the stage-as-output flow (OM 3,
// two barriers per tile but a one-tile prefetch distance) measured 3-10 % slower
bool g_tst_work = getenv("DFFT_TST_STAGEOUT") == nullptr;

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

inline bool is_contig(int family) { return family != kStrided && family != kStridedDct; }

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
    CU(cudaFuncSetAttribute(k->tma_st_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->tma_smem));
    if (k->tma_bk_fn) CU(cudaFuncSetAttribute(k->tma_bk_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->tma_smem));
    if (k->tma_st1_fn)
      CU(cudaFuncSetAttribute(k->tma_st1_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->tma_smem));
    if (k->tma_st_spec_fn)
      CU(cudaFuncSetAttribute(k->tma_st_spec_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->tma_smem));
  }
  if (k->tma2_fn && k->tma2_smem > 48 * 1024) {
    CU(cudaFuncSetAttribute(k->tma2_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->tma2_smem));
    CU(cudaFuncSetAttribute(k->tma2_st_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->tma2_smem));
  }
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
  int tma_variant = 0;     // 1 = single-group TMA kernel, 2 = two-group in-place kernel
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

struct RankPlan {
  int rank = 0, i = 0, j = 0;
  int64_t in_lo[3], in_n[3], out_lo[3], out_n[3];
  size_t in_bytes = 0, out_bytes = 0, ws_bytes = 0;
  void* ws = nullptr;
  std::vector<Stage> A, B;  // per chunk
  std::vector<Exchange> E1, E2;  // first / second exchange (each names its comm group)
  Stage C;
  std::vector<Stage> Cc;  // B→C pipelined plans (dfft_plan_s::bc): stage C per chunk, C unused
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
  bool r2r = false;  // DCT-II forward / DCT-III inverse along every axis (reading R21)
  size_t es = 8;  // complex element bytes
  std::vector<RankPlan> ranks;
  ncclComm_t row = nullptr, col = nullptr;
  cudaStream_t s_comp = nullptr, s_comm = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join_comp = nullptr, ev_join_comm = nullptr;
  std::vector<cudaEvent_t> evA, evE1, evB, evE2;
  void* stage_in = nullptr;  // dfft_execute_host staging buffers
  void* stage_out = nullptr;
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
  unsigned int epoch = 0;            // executes so far (flag values)
  // per-phase profiling (dfft_plan_set_profiling): timing events around every stage launch
  // and exchange, on the stream that runs it; accumulated by dfft_plan_phase_times
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;                 // pool, pairs (start, stop)
  std::vector<int> prof_phase;                      // phase id per recorded pair
  size_t prof_used = 0;                             // pairs recorded since the last read
  double prof_ms[5] = {0, 0, 0, 0, 0};
  long long prof_n[5] = {0, 0, 0, 0, 0};
};

namespace {

// x lines are real (R2C/C2R, R2R): nx reals per line = nx/2 complex elements on the kernel side
inline bool xreal(const dfft_plan_s* pl) { return pl->r2c || pl->r2r; }
inline int fam_x_fwd(const dfft_plan_s* pl) { return pl->r2c ? kContigR2C : pl->r2r ? kContigDct : kContig; }
inline int fam_x_inv(const dfft_plan_s* pl) { return pl->r2c ? kContigC2R : pl->r2r ? kContigDct : kContig; }
inline int fam_s(const dfft_plan_s* pl) { return pl->r2r ? kStridedDct : kStrided; }

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
  if (in_segs && family == kContig && !getenv("DFFT_NO_TBLOCK") &&
      linearize_tblocked(*in_segs, s.in, s.in_bases, s.a.in, (long long)pl->es))
    in_segs = nullptr;
  if (out_segs && linearize(*out_segs, n, s.out, s.out_bases, s.a.out, (long long)pl->es)) out_segs = nullptr;
  if (is_contig(family) && ((!in_segs && s.a.in.tstride != 1) || (!out_segs && s.a.out.tstride != 1)))
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
  ST(get_twiddles(n, pl->f64, pl->dir, pl->comm->device, &s.a.tw));
  if (family == kContigR2C || family == kContigC2R || family == kContigDct)
    ST(get_split_twiddles(n, pl->f64, pl->dir, pl->comm->device, &s.a.tw2));
  if (family == kContigDct || family == kStridedDct)  // c_k over the real line length L
    ST(get_dct_twiddles(family == kContigDct ? 2 * n : n, pl->f64, pl->dir, pl->comm->device, &s.a.tw3));
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
  if (is_contig(family)) s.grid = (L0 * L1 + s.k.per_cta - 1) / s.k.per_cta;
  else s.grid = ((L0 + s.k.per_cta - 1) / s.k.per_cta) * L1;
  if (s.grid >= (1LL << 31)) return fail(DFFT_ERR_UNSUPPORTED, "grid too large (%lld CTAs)", s.grid);
  if ((family == kStrided || family == kStridedDct) && (s.k.tma_fn || s.k.tma2_fn) && g_use_tma && !in_tab &&
      tensor_map_encoder()) {
    const long long es = (long long)pl->es;
    bool ok = s.a.in.s0 == 1 && (s.a.in.tstride * es) % 16 == 0 && (L1 == 1 || (s.a.in.s1 * es) % 16 == 0) &&
              2 * L0 < (1LL << 32) && L1 < (1LL << 31);
    if (s.a.in.bw > 0) ok = ok && s.k.tma_fn && s.a.in.bw % s.k.tma_w == 0 && (s.a.in.mT * s.a.in.s1 * es) % 16 == 0;
    if (ok) {
      const bool v2 = g_use_tma2 && s.k.tma2_fn;
      const void* fn = v2 ? s.k.tma2_fn : s.k.tma_fn;
      const int thr = v2 ? s.k.tma2_threads : s.k.tma_threads, w = v2 ? s.k.tma2_w : s.k.tma_w;
      const size_t sm = v2 ? s.k.tma2_smem : s.k.tma_smem;
      int occ = 0, dev = pl->comm->device, sms = 0;
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, thr, sm));
      CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      long long tiles = ((L0 + w - 1) / w) * L1;
      if (occ > 0) {
        s.tma_variant = v2 ? 2 : 1;
        s.tma_grid = std::min<long long>(tiles, (long long)sms * occ);
        s.tma_occ = occ;
        ST(get_twiddles(n, pl->f64, pl->dir, pl->comm->device, &s.tw_tma, v2 ? s.k.tma2_maxr : s.k.tma_maxr));
      }
      if (getenv("DFFT_DEBUG"))
        fprintf(stderr, "dfft: strided n=%d L0=%lld L1=%lld tma variant %d grid %lld (occ %d, tma2_fn %p)\n", n, L0, L1,
                s.tma_variant, s.tma_grid, occ, s.k.tma2_fn);
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
    ST(finish_stage(pl, B, fam_s(pl), (int)g.ny, Xn, zc, nullptr, &bseg));
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
  ST(finish_stage(pl, C, fam_s(pl), (int)g.nz, Xn, Y3n, nullptr, nullptr));
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
    ST(finish_stage(pl, B, fam_s(pl), (int)g.ny, xc, Zn, nullptr, &bseg));
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
    ST(finish_stage(pl, C, fam_s(pl), (int)g.nz, xc, Y3n, nullptr, nullptr));
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
  ST(finish_stage(pl, A, fam_s(pl), (int)g.nz, Xn, Y3n, nullptr, &aseg));
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
    ST(finish_stage(pl, B, fam_s(pl), (int)g.ny, Xn, zc, nullptr, &bseg));
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
//   forward: x (in -> out, natural), z (out -> ws as [y][z][x]), y (ws -> out, natural)
//   inverse: y (in -> out, natural), z (out -> ws as [y][z][x]), x (ws -> out, natural, ×1/N)
// Single GPU, blocked middle layout (r01 session 2): every pass keeps both sides at a small
// pitch, so a 1024-row column spans a few 2 MB pages instead of one page per row.
//   forward: x (in -> L1 = [y][z][x] in `out`), z (L1 -> L2 = [xb][z][y][w] in ws),
//            y (L2 -> `out`, natural)
//   inverse: y (in -> L2), z (L2 -> L1), x (L1 -> `out`, natural, ×1/N)
// L2 is column-blocked with the strided TMA tile width w (a y-pass tile = one contiguous
// 64 KB block; the z-pass writes it with 4D TMA stores).  Needs the TMA kernel for ny and nz
// with equal tile widths; otherwise build_single (the natural-layout order) is used.
bool single_blocked_ok(dfft_plan_t pl, const Geo& g) {
  // opt-in (measured slower): the z-pass's 4D TMA stores at a 64 KB pitch ran at
  // 3.3 TB/s and the blocked y-pass reads did not beat the 8 MB-pitch ones (1024^3 c64:
  // fwd+inv 25.1 vs 22.8 ms on the same B200)
  if (!getenv("DFFT_SINGLE_BLOCKED") || !g_use_tma || !g_tma_store) return false;
  KernelInfo ky, kz;
  const int dir = pl->dir;
  const bool oky = pl->f64 ? lookup_kernel_f64(kStrided, (int)g.ny, dir, &ky) : lookup_kernel_f32(kStrided, (int)g.ny, dir, &ky);
  const bool okz = pl->f64 ? lookup_kernel_f64(kStrided, (int)g.nz, dir, &kz) : lookup_kernel_f32(kStrided, (int)g.nz, dir, &kz);
  if (!oky || !okz || !ky.tma_fn || !kz.tma_fn || ky.tma_w != kz.tma_w) return false;
  const long long w = ky.tma_w;
  // the inverse c2c uses `out` as the L2 scratch: no padding room there
  if (pl->dir == DFFT_INVERSE && !pl->r2c && g.nxc % w != 0) return false;
  if (pl->r2r) return false;
  return g.ny * (long long)pl->es % 16 == 0 && g.nxc * (long long)pl->es % 16 == 0;
}

dfft_status_t build_single_blocked(dfft_plan_t pl, const Geo& g, RankPlan& rp) {
  const long long nx = g.nx, ny = g.ny, nz = g.nz, nxc = g.nxc, es = (long long)pl->es;
  const long long nxl = xreal(pl) ? nx / 2 : nx;
  KernelInfo ky;
  if (!(pl->f64 ? lookup_kernel_f64(kStrided, (int)ny, pl->dir, &ky) : lookup_kernel_f32(kStrided, (int)ny, pl->dir, &ky)))
    return fail(DFFT_ERR_INTERNAL, "no strided kernel for ny");
  const long long w = ky.tma_w;
  const long long W = nxc * ny * nz, Wb = round_up(nxc, w) * ny * nz;
  const bool c2r = pl->r2c && pl->dir == DFFT_INVERSE;
  rp.A.resize(1);
  rp.B.resize(1);
  rp.E1.resize(1);
  rp.E2.resize(1);
  Stage &A = rp.A[0], &B = rp.B[0], &C = rp.C;
  // L1 [y][z][x]: (x, y, z) at x + nxc·(z + nz·y);  L2 [xb][z][y][w]: blocked, block stride ny·nz·w
  auto set_l1_lines = [&](SideMap& m) { set_side(m, 1, nz * nxc, nxc); };  // contig: l0 = y, l1 = z
  auto set_l2_zpass = [&](SideMap& m) {  // t = z, l0 = x, l1 = y
    set_side(m, ny * w, 1, w);
    m.bw = (int)w;
    m.mT = nz * ny;
  };
  auto set_l2_ypass = [&](SideMap& m) {  // t = y, l0 = x, l1 = z
    set_side(m, w, 1, ny * w);
    m.bw = (int)w;
    m.mT = nz;
  };
  if (pl->dir == DFFT_FORWARD) {
    rp.ws_bytes = (size_t)(Wb * es);
    A.in = {kUserIn, 0};  // x-pass: lines (l0 = y, l1 = z), natural in
    set_side(A.a.in, 1, nxl, ny * nxl);
    A.out = {kUserOut, 0};
    set_l1_lines(A.a.out);
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, fam_x_fwd(pl), (int)nxl, ny, nz, nullptr, nullptr));
    B.in = {kUserOut, 0};  // z-pass: columns (l0 = x, l1 = y) of L1 -> L2
    set_side(B.a.in, nxc, 1, nz * nxc);
    B.out = {kWs, 0};
    set_l2_zpass(B.a.out);
    B.a.scale = 1.0;
    ST(finish_stage(pl, B, fam_s(pl), (int)nz, nxc, ny, nullptr, nullptr));
    C.in = {kWs, 0};  // y-pass: columns (l0 = x, l1 = z) of L2 -> natural `out`
    set_l2_ypass(C.a.in);
    C.out = {kUserOut, 0};
    set_side(C.a.out, nxc, 1, ny * nxc);
    C.a.scale = 1.0;
    C.last_fwd = true;  // t = y, l0 = x, l1 = z
    C.gax[0] = 1, C.gax[1] = 0, C.gax[2] = 2;
    ST(finish_stage(pl, C, fam_s(pl), (int)ny, nxc, nz, nullptr, nullptr));
  } else {
    // scratch: c2c: L2 in `out` (nxc % w == 0 checked), L1 in ws;  c2r: both in ws
    rp.ws_bytes = (size_t)((c2r ? Wb + W : W) * es);
    const Ref l2 = c2r ? Ref{kWs, 0} : Ref{kUserOut, 0};
    const Ref l1 = c2r ? Ref{kWs, Wb * es} : Ref{kWs, 0};
    A.in = {kUserIn, 0};  // y-pass: columns (l0 = x, l1 = z), natural in -> L2
    set_side(A.a.in, nxc, 1, ny * nxc);
    A.out = l2;
    set_l2_ypass(A.a.out);
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, fam_s(pl), (int)ny, nxc, nz, nullptr, nullptr));
    B.in = l2;  // z-pass: columns (l0 = x, l1 = y) of L2 -> L1
    set_l2_zpass(B.a.in);
    B.out = l1;
    set_side(B.a.out, nxc, 1, nz * nxc);
    B.a.scale = 1.0;
    ST(finish_stage(pl, B, fam_s(pl), (int)nz, nxc, ny, nullptr, nullptr));
    C.in = l1;  // x-pass: lines (l0 = y, l1 = z) of L1 -> natural `out`, ×1/N
    set_l1_lines(C.a.in);
    C.out = {kUserOut, 0};
    set_side(C.a.out, 1, nxl, ny * nxl);
    C.a.scale = (xreal(pl) ? 2.0 : 1.0) / ((double)nx * (double)ny * (double)nz);
    ST(finish_stage(pl, C, fam_x_inv(pl), (int)nxl, ny, nz, nullptr, nullptr));
  }
  return DFFT_SUCCESS;
}

dfft_status_t build_single(dfft_plan_t pl, const Geo& g, RankPlan& rp) {
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
    return finish_stage(pl, Z, fam_s(pl), (int)nz, nxc, ny, nullptr, nullptr);
  };
  if (pl->dir == DFFT_FORWARD && !getenv("DFFT_SINGLE_FWD_ZREAD")) {
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
    ST(finish_stage(pl, B, fam_s(pl), (int)nz, nxc, ny, nullptr, nullptr));
    C.in = {kWs, 0};  // y-pass: columns (l0 = x, l1 = z), natural -> natural
    set_side(C.a.in, nxc, 1, ny * nxc);
    C.out = {kUserOut, 0};
    set_side(C.a.out, nxc, 1, ny * nxc);
    C.a.scale = 1.0;
    C.last_fwd = true;  // t = y, l0 = x, l1 = z
    C.gax[0] = 1, C.gax[1] = 0, C.gax[2] = 2;
    ST(finish_stage(pl, C, fam_s(pl), (int)ny, nxc, nz, nullptr, nullptr));
  } else if (pl->dir == DFFT_FORWARD) {
    A.in = {kUserIn, 0};  // lines (l0 = y, l1 = z)
    set_side(A.a.in, 1, nxl, ny * nxl);
    A.out = {kUserOut, 0};
    set_side(A.a.out, 1, nxc, ny * nxc);
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, fam_x_fwd(pl), (int)nxl, ny, nz, nullptr, nullptr));
    ST(zpass(B));
    C.in = {kWs, 0};  // columns (l0 = x, l1 = z)
    set_side(C.a.in, nz * nxc, 1, nxc);
    C.out = {kUserOut, 0};
    set_side(C.a.out, nxc, 1, ny * nxc);
    C.a.scale = 1.0;
    C.last_fwd = true;  // t = y, l0 = x, l1 = z
    C.gax[0] = 1, C.gax[1] = 0, C.gax[2] = 2;
    ST(finish_stage(pl, C, fam_s(pl), (int)ny, nxc, nz, nullptr, nullptr));
  } else if (!c2r && getenv("DFFT_SINGLE_INV_YWRITE")) {
    // inverse with the large-pitch side on a store: y-pass natural -> [y][z][x] (in `out`),
    // z-pass [y][z][x] -> ws [y][z][x] (both small), x-pass ws -> natural (A/B option)
    A.in = {kUserIn, 0};  // y-pass: columns (l0 = x, l1 = z)
    set_side(A.a.in, nxc, 1, ny * nxc);
    A.out = {kUserOut, 0};
    set_side(A.a.out, nz * nxc, 1, nxc);
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, fam_s(pl), (int)ny, nxc, nz, nullptr, nullptr));
    B.in = {kUserOut, 0};  // z-pass: columns (l0 = x, l1 = y)
    set_side(B.a.in, nxc, 1, nz * nxc);
    B.out = {kWs, 0};
    set_side(B.a.out, nxc, 1, nz * nxc);
    B.a.scale = 1.0;
    ST(finish_stage(pl, B, fam_s(pl), (int)nz, nxc, ny, nullptr, nullptr));
    C.in = {kWs, 0};  // x-pass: lines (l0 = y, l1 = z) of [y][z][x]
    set_side(C.a.in, 1, nz * nxc, nxc);
    C.out = {kUserOut, 0};
    set_side(C.a.out, 1, nxl, ny * nxl);
    C.a.scale = (xreal(pl) ? 2.0 : 1.0) / ((double)nx * (double)ny * (double)nz);
    ST(finish_stage(pl, C, fam_x_inv(pl), (int)nxl, ny, nz, nullptr, nullptr));
  } else {
    A.in = {kUserIn, 0};  // columns (l0 = x, l1 = z)
    set_side(A.a.in, nxc, 1, ny * nxc);
    A.out = c2r ? Ref{kWs, 0} : Ref{kUserOut, 0};
    set_side(A.a.out, nxc, 1, ny * nxc);
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, fam_s(pl), (int)ny, nxc, nz, nullptr, nullptr));
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
    ST(finish_stage(pl, A, fam_s(pl), (int)g.nz, xc, Y3n, nullptr, &aseg));
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
    ST(finish_stage(pl, B, fam_s(pl), (int)g.ny, xc, Zn, nullptr, &bseg));
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

dfft_status_t launch(const Stage& s, const Ctx& c, cudaStream_t st) {
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
      const bool v2 = s.tma_variant == 2;
      cuuint32_t box[3] = {(cuuint32_t)(2 * (v2 ? s.k.tma2_w : s.k.tma_w)), (cuuint32_t)(v2 ? s.k.tma2_r0 : s.k.tma_boxr),
                           1};
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
      if (spec && !(use_st && s.tma_variant == 1 && s.k.tma_st_spec_fn)) goto plain;  // multiplier: TST or plain
      if (s.k.tma_st_only && !use_st) goto plain;  // R2R: the TMA variant needs TMA stores
      if (spec)
        CU(cudaLaunchKernel(s.k.tma_st_spec_fn, dim3((unsigned)grid), dim3(s.k.tma_threads), targs, s.k.tma_smem, st));
      else if (s.tma_variant == 2)
        CU(cudaLaunchKernel(use_st ? s.k.tma2_st_fn : s.k.tma2_fn, dim3((unsigned)grid), dim3(s.k.tma2_threads),
                            targs, s.k.tma2_smem, st));
      else
        CU(cudaLaunchKernel(a.out.nbulk > 0 ? s.k.tma_bk_fn
                            : use_st        ? (g_tst_work ? s.k.tma_st1_fn : s.k.tma_st_fn)
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

// simulated ranks: rank r's send to peer q is matched with q's receive from r, in order
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

// phases: 0 stage A, 1 exchange 1, 2 stage B, 3 exchange 2, 4 stage C
dfft_status_t prof_begin(dfft_plan_t pl, int phase, cudaStream_t st, size_t* slot) {
  if (!pl->prof) return DFFT_SUCCESS;
  size_t i = pl->prof_used++;
  while (pl->prof_ev.size() < 2 * pl->prof_used) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    pl->prof_ev.push_back(e);
  }
  if (pl->prof_phase.size() < pl->prof_used) pl->prof_phase.resize(pl->prof_used);
  pl->prof_phase[i] = phase;
  *slot = i;
  CU(cudaEventRecord(pl->prof_ev[2 * i], st));
  return DFFT_SUCCESS;
}
dfft_status_t prof_end(dfft_plan_t pl, size_t slot, cudaStream_t st) {
  if (!pl->prof) return DFFT_SUCCESS;
  CU(cudaEventRecord(pl->prof_ev[2 * slot + 1], st));
  return DFFT_SUCCESS;
}
dfft_status_t launch_p(dfft_plan_t pl, int phase, const Stage& s, const Ctx& c, cudaStream_t st) {
  if (s.empty) return DFFT_SUCCESS;
  size_t slot = 0;
  ST(prof_begin(pl, phase, st, &slot));
  ST(launch(s, c, st));
  return prof_end(pl, slot, st);
}
dfft_status_t exchange_p(dfft_plan_t pl, int phase, const Exchange& x, const Ctx& c, cudaStream_t st) {
  if (x.sends.empty() && x.recvs.empty()) return DFFT_SUCCESS;
  size_t slot = 0;
  ST(prof_begin(pl, phase, st, &slot));
  ST(exchange_nccl(pl, x, c, st));
  return prof_end(pl, slot, st);
}

// ---- P2P exchange: stage kernels store into the peers' windows; flags order the stages.
struct SignalArgs {
  unsigned int* ptr[2 * kMaxBases];
  int n;
  unsigned int value;
};

__global__ void dfft_signal_kernel(const __grid_constant__ SignalArgs a) {
  // stream order puts this after the stage kernel whose stores it publishes; the system-scope
  // fence + release store make them visible to the peer that acquires the flag
  if ((int)threadIdx.x < a.n) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.ptr[threadIdx.x]), "r"(a.value) : "memory");
  }
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

// flag word: arr 0 = ready, 1 = done; e = exchange (0 first, 1 second); k chunk; r writer/reader rank
inline size_t flag_index(const dfft_plan_s* pl, int arr, int e, int k, int r) {
  const size_t P = (size_t)pl->P1 * pl->P2, K = (size_t)pl->K;
  return (((size_t)arr * 2 + e) * K + k) * P + r;
}

dfft_status_t p2p_signal(dfft_plan_t pl, int arr, int e, int k, const std::vector<int>& targets, unsigned value,
                         cudaStream_t st) {
  if (targets.empty()) return DFFT_SUCCESS;
  SignalArgs a{};
  a.n = (int)targets.size();
  a.value = value;
  const int me = pl->comm->rank;
  for (size_t q = 0; q < targets.size(); ++q)
    a.ptr[q] = reinterpret_cast<unsigned int*>((char*)pl->peer_ws[targets[q]] + pl->flag_off) +
               flag_index(pl, arr, e, k, me);
  void* args[] = {&a};
  CU(cudaLaunchKernel((const void*)dfft_signal_kernel, dim3(1), dim3(32), args, 0, st));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return DFFT_SUCCESS;
}

dfft_status_t p2p_wait(dfft_plan_t pl, int arr, int e, int k, const std::vector<int>& from, unsigned value,
                       cudaStream_t st) {
  unsigned int* flags = reinterpret_cast<unsigned int*>((char*)pl->ranks[0].ws + pl->flag_off);
  for (int r : from) {
    CUresult res = stream_wait_value32()((CUstream)st, (CUdeviceptr)(flags + flag_index(pl, arr, e, k, r)), value,
                                         CU_STREAM_WAIT_VALUE_GEQ);
    if (res != CUDA_SUCCESS) return fail(DFFT_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)res);
  }
  return DFFT_SUCCESS;
}

// Two compute streams: X runs stage A chunk by chunk, Y runs stage B of each chunk as soon as
// its first exchange has landed, then stage C.  So A(k+1) overlaps B(k) (Fig. 1, the
// progressive per-chunk pipelining); when one of the two is NVLink-bound (fused remote stores)
// it runs on at most sm_cap SMs so the HBM-bound one can co-reside (Stage::sm_cap).
dfft_status_t execute_p2p(dfft_plan_t pl, const Ctx& cx, cudaStream_t user) {
  RankPlan& rp = pl->ranks[0];
  const int K = (int)rp.A.size();
  const unsigned ep = ++pl->epoch;
  cudaStream_t X = pl->s_comp, Y = pl->s_comm;
  CU(cudaEventRecord(pl->ev_fork, user));
  CU(cudaStreamWaitEvent(X, pl->ev_fork, 0));
  CU(cudaStreamWaitEvent(Y, pl->ev_fork, 0));
  if (pl->bc) {
    // X: A (whole), then C(k) as chunk k of the second exchange completes; Y: B(k), k = 0..K-1
    const std::vector<int>& p1 = rp.E1[0].peers;
    if (ep > 1) ST(p2p_wait(pl, 1, 0, 0, p1, ep - 1, X));
    ST(launch_p(pl, 0, rp.A[0], cx, X));
    ST(p2p_signal(pl, 0, 0, 0, p1, ep, X));
    CU(cudaEventRecord(pl->evA[0], X));
    CU(cudaStreamWaitEvent(Y, pl->evA[0], 0));
    ST(p2p_wait(pl, 0, 0, 0, p1, ep, Y));
    for (int k = 0; k < K; ++k) {
      if (ep > 1) ST(p2p_wait(pl, 1, 1, k, rp.E2[k].peers, ep - 1, Y));
      ST(launch_p(pl, 2, rp.B[k], cx, Y));
      ST(p2p_signal(pl, 0, 1, k, rp.E2[k].peers, ep, Y));
      CU(cudaEventRecord(pl->evB[k], Y));
    }
    ST(p2p_signal(pl, 1, 0, 0, p1, ep, Y));  // done reading my first-exchange window
    for (int k = 0; k < K; ++k) {
      CU(cudaStreamWaitEvent(X, pl->evB[k], 0));
      ST(p2p_wait(pl, 0, 1, k, rp.E2[k].peers, ep, X));
      ST(launch_p(pl, 4, rp.Cc[k], cx, X));
      ST(p2p_signal(pl, 1, 1, k, rp.E2[k].peers, ep, X));
    }
  } else {
  for (int k = 0; k < K; ++k) {
    // my epoch-1 stores into the first-exchange peers were consumed
    if (ep > 1) ST(p2p_wait(pl, 1, 0, k, rp.E1[k].peers, ep - 1, X));
    ST(launch_p(pl, 0, rp.A[k], cx, X));
    ST(p2p_signal(pl, 0, 0, k, rp.E1[k].peers, ep, X));
    CU(cudaEventRecord(pl->evA[k], X));
  }
  for (int k = 0; k < K; ++k) {
    CU(cudaStreamWaitEvent(Y, pl->evA[k], 0));  // my own block of chunk k
    ST(p2p_wait(pl, 0, 0, k, rp.E1[k].peers, ep, Y));
    if (ep > 1) ST(p2p_wait(pl, 1, 1, k, rp.E2[k].peers, ep - 1, Y));
    ST(launch_p(pl, 2, rp.B[k], cx, Y));
    ST(p2p_signal(pl, 1, 0, k, rp.E1[k].peers, ep, Y));  // done reading my first-exchange window
    ST(p2p_signal(pl, 0, 1, k, rp.E2[k].peers, ep, Y));  // ready: stored into the peers' second windows
  }
  for (int k = 0; k < K; ++k) ST(p2p_wait(pl, 0, 1, k, rp.E2[k].peers, ep, Y));
  ST(launch_p(pl, 4, rp.C, cx, Y));
  for (int k = 0; k < K; ++k) ST(p2p_signal(pl, 1, 1, k, rp.E2[k].peers, ep, Y));
  }
  CU(cudaEventRecord(pl->ev_join_comp, X));
  CU(cudaEventRecord(pl->ev_join_comm, Y));
  CU(cudaStreamWaitEvent(user, pl->ev_join_comp, 0));
  CU(cudaStreamWaitEvent(user, pl->ev_join_comm, 0));
  return DFFT_SUCCESS;
}

// ---- CE exchange: stage kernels pack into local send blocks (as for NCCL); the copy engine of
// the comm stream moves each block into the receiver's window; flags order producer/consumer.
dfft_status_t exchange_ce(dfft_plan_t pl, int e, int k, const Exchange& x, const Ctx& cx, unsigned ep,
                          cudaStream_t st) {
  if (x.peers.empty()) return DFFT_SUCCESS;
  if (ep > 1) ST(p2p_wait(pl, 1, e, k, x.peers, ep - 1, st));  // receivers consumed epoch ep-1
  for (const Xfer& t : x.sends) {
    if (t.height > 1)
      CU(cudaMemcpy2DAsync(resolve(t.remote, cx), t.dpitch, resolve(t.ref, cx), t.spitch, t.width, t.height,
                           cudaMemcpyDeviceToDevice, st));
    else
      CU(cudaMemcpyAsync(resolve(t.remote, cx), resolve(t.ref, cx), t.bytes, cudaMemcpyDeviceToDevice, st));
  }
  return p2p_signal(pl, 0, e, k, x.peers, ep, st);
}

dfft_status_t execute_ce(dfft_plan_t pl, const Ctx& cx, cudaStream_t user) {
  RankPlan& rp = pl->ranks[0];
  const size_t K = rp.A.size();
  const unsigned ep = ++pl->epoch;
  cudaStream_t sc = pl->s_comp, sm = pl->s_comm;
  CU(cudaEventRecord(pl->ev_fork, user));
  CU(cudaStreamWaitEvent(sc, pl->ev_fork, 0));
  CU(cudaStreamWaitEvent(sm, pl->ev_fork, 0));
  // a fused exchange is produced inside the FFT kernel: WAR wait before it, ready signal after it,
  // both on the compute stream; a CE exchange is a copy on the comm stream after the kernel
  auto do_A = [&](size_t k) -> dfft_status_t {
    const Exchange& x = rp.E1[k];
    if (x.fused && ep > 1) ST(p2p_wait(pl, 1, 0, (int)k, x.peers, ep - 1, sc));
    ST(launch_p(pl, 0, rp.A[k], cx, sc));
    if (x.fused) return p2p_signal(pl, 0, 0, (int)k, x.peers, ep, sc);
    CU(cudaEventRecord(pl->evA[k], sc));
    CU(cudaStreamWaitEvent(sm, pl->evA[k], 0));
    size_t slot = 0;
    ST(prof_begin(pl, 1, sm, &slot));
    ST(exchange_ce(pl, 0, (int)k, x, cx, ep, sm));
    return prof_end(pl, slot, sm);
  };
  ST(do_A(0));
  for (size_t k = 0; k < K; ++k) {
    if (k + 1 < K) ST(do_A(k + 1));
    const Exchange& x2 = rp.E2[k];
    ST(p2p_wait(pl, 0, 0, (int)k, rp.E1[k].peers, ep, sc));  // peers' blocks of chunk k have landed
    if (x2.fused && ep > 1) ST(p2p_wait(pl, 1, 1, (int)k, x2.peers, ep - 1, sc));
    ST(launch_p(pl, 2, rp.B[k], cx, sc));
    ST(p2p_signal(pl, 1, 0, (int)k, rp.E1[k].peers, ep, sc));  // done reading my first receive region
    if (x2.fused) {
      ST(p2p_signal(pl, 0, 1, (int)k, x2.peers, ep, sc));
    } else {
      CU(cudaEventRecord(pl->evB[k], sc));
      CU(cudaStreamWaitEvent(sm, pl->evB[k], 0));
      size_t slot = 0;
      ST(prof_begin(pl, 3, sm, &slot));
      ST(exchange_ce(pl, 1, (int)k, x2, cx, ep, sm));
      ST(prof_end(pl, slot, sm));
    }
  }
  for (size_t k = 0; k < K; ++k) ST(p2p_wait(pl, 0, 1, (int)k, rp.E2[k].peers, ep, sc));
  ST(launch_p(pl, 4, rp.C, cx, sc));
  for (size_t k = 0; k < K; ++k) ST(p2p_signal(pl, 1, 1, (int)k, rp.E2[k].peers, ep, sc));
  CU(cudaEventRecord(pl->ev_join_comp, sc));
  CU(cudaEventRecord(pl->ev_join_comm, sm));
  CU(cudaStreamWaitEvent(user, pl->ev_join_comp, 0));
  CU(cudaStreamWaitEvent(user, pl->ev_join_comm, 0));
  return DFFT_SUCCESS;
}

dfft_status_t execute_rank(dfft_plan_t pl, const void* in, void* out, cudaStream_t user) {
  RankPlan& rp = pl->ranks[0];
  const size_t K = rp.A.size();
  const Ctx cx{in, out, rp.ws, pl->peer_ws.empty() ? nullptr : pl->peer_ws.data()};
  if (pl->p2p) return execute_p2p(pl, cx, user);
  if (pl->ce) return execute_ce(pl, cx, user);
  if (!pl->overlap) {
    // static-barrier ablation: every step in program order on the user's stream
    for (size_t k = 0; k < K; ++k) ST(launch_p(pl, 0, rp.A[k], cx, user));
    for (size_t k = 0; k < K; ++k) ST(exchange_p(pl, 1, rp.E1[k], cx, user));
    for (size_t k = 0; k < K; ++k) ST(launch_p(pl, 2, rp.B[k], cx, user));
    for (size_t k = 0; k < K; ++k) ST(exchange_p(pl, 3, rp.E2[k], cx, user));
    return launch_p(pl, 4, rp.C, cx, user);
  }
  cudaStream_t sc = pl->s_comp, sm = pl->s_comm;
  CU(cudaEventRecord(pl->ev_fork, user));
  CU(cudaStreamWaitEvent(sc, pl->ev_fork, 0));
  CU(cudaStreamWaitEvent(sm, pl->ev_fork, 0));
  // host issue order is a topological order of the chunk DAG, so every wait refers to the
  // record issued in this execute:  A0 E1_0 | A1 E1_1 B0 E2_0 | A2 E1_2 B1 E2_1 | ...
  auto do_A = [&](size_t k) -> dfft_status_t {
    ST(launch_p(pl, 0, rp.A[k], cx, sc));
    if (!rp.E1[k].sends.empty() || !rp.E1[k].recvs.empty()) {
      CU(cudaEventRecord(pl->evA[k], sc));
      CU(cudaStreamWaitEvent(sm, pl->evA[k], 0));
      ST(exchange_p(pl, 1, rp.E1[k], cx, sm));
      CU(cudaEventRecord(pl->evE1[k], sm));
    }
    return DFFT_SUCCESS;
  };
  ST(do_A(0));
  for (size_t k = 0; k < K; ++k) {
    if (k + 1 < K) ST(do_A(k + 1));
    if (!rp.E1[k].sends.empty() || !rp.E1[k].recvs.empty()) CU(cudaStreamWaitEvent(sc, pl->evE1[k], 0));
    ST(launch_p(pl, 2, rp.B[k], cx, sc));
    if (!rp.E2[k].sends.empty() || !rp.E2[k].recvs.empty()) {
      CU(cudaEventRecord(pl->evB[k], sc));
      CU(cudaStreamWaitEvent(sm, pl->evB[k], 0));
      ST(exchange_p(pl, 3, rp.E2[k], cx, sm));
      CU(cudaEventRecord(pl->evE2[k], sm));
    }
  }
  // stage C needs every chunk of exchange 2 (same comm stream => the last record suffices)
  if (!rp.E2[K - 1].sends.empty() || !rp.E2[K - 1].recvs.empty()) CU(cudaStreamWaitEvent(sc, pl->evE2[K - 1], 0));
  ST(launch_p(pl, 4, rp.C, cx, sc));
  CU(cudaEventRecord(pl->ev_join_comp, sc));
  CU(cudaEventRecord(pl->ev_join_comm, sm));
  CU(cudaStreamWaitEvent(user, pl->ev_join_comp, 0));
  CU(cudaStreamWaitEvent(user, pl->ev_join_comm, 0));
  return DFFT_SUCCESS;
}

dfft_status_t execute_sim(dfft_plan_t pl, const void* const* ins, void* const* outs, cudaStream_t st) {
  const size_t P = pl->ranks.size(), K = pl->ranks[0].A.size();
  if (pl->p2p) {
    // fused-store layouts: every stage of every rank stores straight into the other ranks'
    // workspaces; stream order replaces the ready/done flags
    void* const* peers = pl->peer_ws.data();
    auto cx = [&](size_t r) { return Ctx{ins[r], outs[r], pl->ranks[r].ws, peers}; };
    for (size_t k = 0; k < K; ++k)
      for (size_t r = 0; r < P; ++r) ST(launch(pl->ranks[r].A[k], cx(r), st));
    for (size_t k = 0; k < K; ++k)
      for (size_t r = 0; r < P; ++r) ST(launch(pl->ranks[r].B[k], cx(r), st));
    for (size_t r = 0; r < P; ++r) {
      if (pl->bc)
        for (size_t k = 0; k < K; ++k) ST(launch(pl->ranks[r].Cc[k], cx(r), st));
      else
        ST(launch(pl->ranks[r].C, cx(r), st));
    }
    return DFFT_SUCCESS;
  }
  for (size_t k = 0; k < K; ++k)
    for (size_t r = 0; r < P; ++r) ST(launch(pl->ranks[r].A[k], Ctx{ins[r], outs[r], pl->ranks[r].ws, nullptr}, st));
  for (size_t k = 0; k < K; ++k) ST(exchange_sim(pl, false, k, ins, outs, st));
  for (size_t k = 0; k < K; ++k)
    for (size_t r = 0; r < P; ++r) ST(launch(pl->ranks[r].B[k], Ctx{ins[r], outs[r], pl->ranks[r].ws, nullptr}, st));
  for (size_t k = 0; k < K; ++k) ST(exchange_sim(pl, true, k, ins, outs, st));
  for (size_t r = 0; r < P; ++r) ST(launch(pl->ranks[r].C, Ctx{ins[r], outs[r], pl->ranks[r].ws, nullptr}, st));
  return DFFT_SUCCESS;
}

void free_stage(Stage& s) {
  if (s.in_tab) cudaFree(s.in_tab);
  if (s.out_tab) cudaFree(s.out_tab);
  s.in_tab = s.out_tab = nullptr;
}

void free_plan(dfft_plan_t pl) {
  if (!pl) return;
  if ((pl->p2p || pl->ce) && pl->epoch > 0 && pl->s_comp) {
    // peers write their final `done` flags into this window after their last stage: wait for
    // them so no peer store lands in freed memory
    RankPlan& rp = pl->ranks[0];
    for (int k = 0; k < (int)rp.A.size(); ++k) {
      p2p_wait(pl, 1, 0, k, rp.E1[k].peers, pl->epoch, pl->s_comp);
      p2p_wait(pl, 1, 1, k, rp.E2[k].peers, pl->epoch, pl->s_comp);
    }
  }
  if (pl->s_comp) cudaStreamSynchronize(pl->s_comp);
  if (pl->s_comm) cudaStreamSynchronize(pl->s_comm);
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
  }
  for (auto* v : {&pl->evA, &pl->evE1, &pl->evB, &pl->evE2})
    for (cudaEvent_t e : *v) cudaEventDestroy(e);
  for (cudaEvent_t e : pl->prof_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : {pl->ev_fork, pl->ev_join_comp, pl->ev_join_comm})
    if (e) cudaEventDestroy(e);
  if (pl->s_comp) cudaStreamDestroy(pl->s_comp);
  if (pl->s_comm) cudaStreamDestroy(pl->s_comm);
  if (pl->spec_tab) cudaFree(pl->spec_tab);
  if (pl->stage_in) cudaFree(pl->stage_in);
  if (pl->stage_out) cudaFree(pl->stage_out);
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
// the HBM-bound one the rest, except in the last chunk, which runs alone.
dfft_status_t apply_sm_caps(dfft_plan_t pl, RankPlan& rp) {
  const size_t K = rp.A.size();
  if (!pl->p2p || K < 2) return DFFT_SUCCESS;
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

// argument validation shared by dfft_plan_create and dfft_decomp_box; maps slab to pencil 1×P
static dfft_status_t validate(int P, int64_t nx, int64_t ny, int64_t nz, dfft_decomp_t decomp, int* p1p, int* p2p,
                              dfft_type_t type, dfft_direction_t direction) {
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
  if (r2c && nx % 2) return fail(DFFT_ERR_UNSUPPORTED, "R2C needs even nx");
  if (r2r && (nx % 2 || ny % 2 || nz % 2))
    return fail(DFFT_ERR_UNSUPPORTED, "R2R (DCT via Makhoul's permutation) needs even extents");
  long long nxc = r2c ? nx / 2 + 1 : r2r ? nx / 2 : nx;
  long long nfft_x = (r2c || r2r) ? nx / 2 : nx;
  if (!length_ok(nfft_x) || !length_ok(ny) || !length_ok(nz))
    return fail(DFFT_ERR_UNSUPPORTED, "axis lengths (%lld,%lld,%lld): need 2^a 3^b 5^c 7^d from the instantiated set",
                (long long)nfft_x, (long long)ny, (long long)nz);
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
  if (!plan || !comm) return fail(DFFT_ERR_INVALID_VALUE, "null plan/comm");
  *plan = nullptr;
  int P = comm->nranks;
  ST(validate(P, nx, ny, nz, decomp, &p1, &p2, type, direction));
  bool r2c = type == DFFT_R2C_F32 || type == DFFT_R2C_F64;
  bool r2r = type == DFFT_R2R_F32 || type == DFFT_R2R_F64;
  bool f64 = type == DFFT_C2C_F64 || type == DFFT_R2C_F64 || type == DFFT_R2R_F64;
  long long nxc = r2c ? nx / 2 + 1 : r2r ? nx / 2 : nx;
  int Kreq = (int)(flags & 0xff);
  bool overlap = !(flags & DFFT_FLAG_NO_OVERLAP);
  long long kmax = direction == DFFT_FORWARD ? nz / p2 : nxc / p1;  // chunk axis extent
  // exchange transport for P > 1: copy engines into IPC windows (default),
  // fused epilogue stores into the windows (DFFT_FLAG_FUSED_STORE), or NCCL (DFFT_FLAG_NCCL)
  const char* exch_env = getenv("DFFT_EXCHANGE");
  auto env_is = [&](const char* v) { return exch_env && strcmp(exch_env, v) == 0; };
  const bool want_fused = (flags & DFFT_FLAG_FUSED_STORE) || (!comm->sim && env_is("p2p"));
  // simulated ranks run the NCCL layouts, or (DFFT_FLAG_FUSED_STORE) the fused-store layouts with
  // every rank's workspace standing in for its IPC window (same kernels, same addresses)
  const bool nccl_mode = (comm->sim && !want_fused) || P == 1 || (flags & DFFT_FLAG_NCCL) || env_is("nccl");
  const bool want_ce = !comm->sim && ((flags & DFFT_FLAG_CE) || env_is("ce"));
  const bool want_hybrid = !comm->sim && ((flags & DFFT_FLAG_HYBRID) || env_is("hybrid"));
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
  if (p2p_mode) g.xq = std::max(g.wy, g.wz);

  if (!comm->sim && P > 1) {
    // collective consistency check: every rank must pass identical arguments
    unsigned long long h = 1469598103934665603ULL;
    for (long long v : {(long long)nx, (long long)ny, (long long)nz, (long long)decomp, (long long)p1,
                        (long long)p2, (long long)type, (long long)direction, (long long)flags}) {
      h ^= (unsigned long long)v;
      h *= 1099511628211ULL;
    }
    unsigned long long* d = nullptr;
    CU(cudaMalloc(&d, sizeof(unsigned long long) * (P + 1)));
    CU(cudaMemcpy(d, &h, sizeof h, cudaMemcpyHostToDevice));
    NC(ncclAllGather(d, d + 1, 1, ncclUint64, comm->world, 0));
    std::vector<unsigned long long> all(P);
    CU(cudaMemcpy(all.data(), d + 1, sizeof(unsigned long long) * P, cudaMemcpyDeviceToHost));
    cudaFree(d);
    for (int r = 0; r < P; ++r)
      if (all[r] != h) return fail(DFFT_ERR_INVALID_VALUE, "plan arguments differ between rank %d and rank %d", comm->rank, r);
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
      ST(P == 1 ? (single_blocked_ok(pl, g) ? build_single_blocked(pl, g, rp) : build_single(pl, g, rp))
                : pl->bc ? build_forward_bc(pl, g, rp) : build_forward(pl, g, rp));
    } else {
      memcpy(rp.in_lo, d3lo, sizeof d3lo);
      memcpy(rp.in_n, d3n, sizeof d3n);
      memcpy(rp.out_lo, d1lo, sizeof d1lo);
      memcpy(rp.out_n, d1n, sizeof d1n);
      rp.in_bytes = d3b;
      rp.out_bytes = d1b;
      ST(P == 1 ? (single_blocked_ok(pl, g) ? build_single_blocked(pl, g, rp) : build_single(pl, g, rp))
                : pl->bc ? build_inverse_bc(pl, g, rp) : build_inverse(pl, g, rp));
    }
    ST(apply_sm_caps(pl, rp));
    if (rp.ws_bytes) {
      cudaError_t e = cudaMalloc(&rp.ws, rp.ws_bytes);
      if (e != cudaSuccess) return fail(DFFT_ERR_ALLOC, "workspace of %zu bytes: %s", rp.ws_bytes, cudaGetErrorString(e));
    }
  }
  if (comm->sim && pl->p2p) {
    // simulated fused stores: rank q's "window" is its workspace on this device
    pl->peer_ws.resize(P);
    for (int q = 0; q < P; ++q) pl->peer_ws[q] = pl->ranks[q].ws;
  } else if (pl->p2p || pl->ce) {
    // every workspace becomes an IPC window; open the windows of the row and column peers
    RankPlan& rp = pl->ranks[0];
    CU(cudaMemset((char*)rp.ws + pl->flag_off, 0, flag_bytes(g)));
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
  CU(cudaStreamCreateWithFlags(&pl->s_comp, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&pl->s_comm, cudaStreamNonBlocking));
  for (auto* v : {&pl->evA, &pl->evE1, &pl->evB, &pl->evE2}) {
    v->resize(K);
    for (auto& e : *v) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  CU(cudaEventCreateWithFlags(&pl->ev_fork, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&pl->ev_join_comp, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&pl->ev_join_comm, cudaEventDisableTiming));
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

dfft_status_t dfft_execute(dfft_plan_t pl, const void* in, void* out, void* stream) {
  if (!pl) return fail(DFFT_ERR_INVALID_VALUE, "null plan");
  if (pl->comm->sim) return fail(DFFT_ERR_INVALID_VALUE, "simulated-comm plan: use dfft_execute_sim");
  ST(check_ptrs(pl, pl->ranks[0], in, out));
  ST(execute_rank(pl, in, out, (cudaStream_t)stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DFFT_ERR_CUDA, "launch: %s", cudaGetErrorString(e));
  return DFFT_SUCCESS;
}

dfft_status_t dfft_execute_host(dfft_plan_t pl, const void* in_host, void* out_host, void* stream) {
  if (!pl || !in_host || !out_host) return fail(DFFT_ERR_INVALID_VALUE, "null argument");
  if (pl->comm->sim) return fail(DFFT_ERR_INVALID_VALUE, "simulated-comm plan");
  const RankPlan& rp = pl->ranks[0];
  if (!pl->stage_in) CU(cudaMalloc(&pl->stage_in, std::max<size_t>(rp.in_bytes, 16)));
  if (!pl->stage_out) CU(cudaMalloc(&pl->stage_out, std::max<size_t>(rp.out_bytes, 16)));
  cudaStream_t st = (cudaStream_t)stream;
  CU(cudaMemcpyAsync(pl->stage_in, in_host, rp.in_bytes, cudaMemcpyHostToDevice, st));
  ST(dfft_execute(pl, pl->stage_in, pl->stage_out, stream));
  CU(cudaMemcpyAsync(out_host, pl->stage_out, rp.out_bytes, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return DFFT_SUCCESS;
}

dfft_status_t dfft_execute_sim(dfft_plan_t pl, const void* const* ins, void* const* outs, void* stream) {
  if (!pl || !ins || !outs) return fail(DFFT_ERR_INVALID_VALUE, "null argument");
  if (!pl->comm->sim) return fail(DFFT_ERR_INVALID_VALUE, "not a simulated-comm plan");
  for (size_t r = 0; r < pl->ranks.size(); ++r) ST(check_ptrs(pl, pl->ranks[r], ins[r], outs[r]));
  ST(execute_sim(pl, ins, outs, (cudaStream_t)stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DFFT_ERR_CUDA, "launch: %s", cudaGetErrorString(e));
  return DFFT_SUCCESS;
}

dfft_status_t dfft_plan_set_poisson(dfft_plan_t pl, double dx, double dy, double dz) {
  if (!pl) return fail(DFFT_ERR_INVALID_VALUE, "null plan");
  if (pl->dir != DFFT_FORWARD) return fail(DFFT_ERR_INVALID_VALUE, "the Poisson multiplier belongs to a forward plan");
  if (pl->r2r) return fail(DFFT_ERR_UNSUPPORTED, "the periodic Poisson multiplier applies to C2C/R2C plans");
  const bool on = dx > 0 && dy > 0 && dz > 0;
  if (!on && (dx != 0 || dy != 0 || dz != 0))
    return fail(DFFT_ERR_INVALID_VALUE, "grid spacings must all be > 0 (or all 0 to switch the multiplier off)");
  CU(cudaSetDevice(pl->comm->device));
  CU(cudaDeviceSynchronize());  // no execute of this plan may be reading the old tables
  if (pl->spec_tab) cudaFree(pl->spec_tab);
  pl->spec_tab = nullptr;
  const long long n[3] = {pl->nx, pl->ny, pl->nz};
  const double h[3] = {dx, dy, dz};
  const size_t rs = pl->es / 2;
  if (on) {
    // λ_d(k) = -(2 sin(πk/n_d)/h_d)², long double, rounded once to the plan's precision (reading R20)
    std::vector<unsigned char> host((size_t)(n[0] + n[1] + n[2]) * rs);
    long long o = 0;
    for (int d = 0; d < 3; ++d)
      for (long long k = 0; k < n[d]; ++k, ++o) {
        const long double sv = 2.0L * sinl(3.14159265358979323846264338327950288L * (long double)k / (long double)n[d]) /
                               (long double)h[d];
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
      for (int q = 0; q < 3; ++q)
        s->a.spec[q] = on ? (const void*)((const char*)pl->spec_tab + (size_t)(base[s->gax[q]] + s->glo[q]) * rs)
                          : nullptr;
      if (on && s->tma_variant == 2) s->tma_grid = 0;  // the two-group kernel has no multiplier
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
  for (size_t i = 0; i < pl->prof_used; ++i) {
    CU(cudaEventSynchronize(pl->prof_ev[2 * i + 1]));
    float t = 0;
    CU(cudaEventElapsedTime(&t, pl->prof_ev[2 * i], pl->prof_ev[2 * i + 1]));
    pl->prof_ms[pl->prof_phase[i]] += t;
    pl->prof_n[pl->prof_phase[i]] += 1;
  }
  pl->prof_used = 0;
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

dfft_status_t dfft_plan_stage_bytes(dfft_plan_t pl, double bytes[5]) {
  if (!pl || !bytes) return fail(DFFT_ERR_INVALID_VALUE, "null argument");
  const RankPlan& rp = pl->ranks[0];
  // algorithmic bytes per execute of each phase: every stage reads and writes its local
  // array once; every exchange sends its off-rank blocks (the bytes that cross NVLink)
  auto stage_b = [&](const Stage& s) {
    if (s.empty) return 0.0;
    double elems = (double)s.a.L0 * (double)s.a.L1 * (double)s.n;  // complex elements of the FFT
    return 2.0 * elems * (double)pl->es;
  };
  auto xch_b = [&](const Exchange& x) {
    double b = 0;
    for (const Xfer& t : x.sends) b += (double)t.bytes;
    return b;
  };
  for (int q = 0; q < 5; ++q) bytes[q] = 0;
  for (size_t k = 0; k < rp.A.size(); ++k) {
    bytes[0] += stage_b(rp.A[k]);
    bytes[1] += xch_b(rp.E1[k]);
    bytes[2] += stage_b(rp.B[k]);
    bytes[3] += xch_b(rp.E2[k]);
  }
  bytes[4] = stage_b(rp.C);
  for (const Stage& c : rp.Cc) bytes[4] += stage_b(c);
  return DFFT_SUCCESS;
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
  ST(get_twiddles((int)n, f64 != 0, sign, dev, &s.a.tw));
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
bool length_supported(long long n) {
  KernelInfo k;
  return n > 0 && n <= 4096 && lookup_kernel_f32(kContig, (int)n, -1, &k);
}
int length_schedule(int n, int rad[kMaxPass], int maxr) {
  Sched s = make_sched(n, maxr);
  for (int p = 0; p < kMaxPass; ++p) rad[p] = s.rad[p];
  return s.npass;
}
}  // namespace dfft
