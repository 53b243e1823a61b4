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
  int n, f64, dir, dev;
  bool operator<(const TwKey& o) const {
    return std::tie(n, f64, dir, dev) < std::tie(o.n, o.f64, o.dir, o.dev);
  }
};
std::mutex g_tw_mu;
std::map<TwKey, void*> g_tw;

dfft_status_t get_twiddles(int n, bool f64, int dir, int dev, const void** out) {
  std::lock_guard<std::mutex> lk(g_tw_mu);
  TwKey key{n, f64 ? 1 : 0, dir, dev};
  auto it = g_tw.find(key);
  if (it != g_tw.end()) {
    *out = it->second;
    return DFFT_SUCCESS;
  }
  int rad[kMaxPass];
  int np = length_schedule(n, rad);
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

bool g_use_tma = getenv("DFFT_NO_TMA") == nullptr;  // env switch for the A/B ablation
CUtensorMapL2promotion g_tma_promo = getenv("DFFT_TMA_PROMO256") ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                     : getenv("DFFT_TMA_PROMO128") ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                                   : CU_TENSOR_MAP_L2_PROMOTION_NONE;
bool g_oop_z = getenv("DFFT_OOP_Z") != nullptr;  // dev: P=1 forward z-stage out of place
bool g_tma_store = getenv("DFFT_NO_TMA_STORE") == nullptr;

dfft_status_t get_kernel(int family, int n, bool f64, int dir, KernelInfo* k) {
  bool ok = f64 ? lookup_kernel_f64(family, n, dir, k) : lookup_kernel_f32(family, n, dir, k);
  if (!ok) return fail(DFFT_ERR_UNSUPPORTED, "axis length %d not instantiated", n);
  if (k->smem > 48 * 1024) CU(cudaFuncSetAttribute(k->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->smem));
  if (k->tma_fn && k->tma_smem > 48 * 1024) {
    CU(cudaFuncSetAttribute(k->tma_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->tma_smem));
    CU(cudaFuncSetAttribute(k->tma_st_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k->tma_smem));
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
enum RefKind { kNone = 0, kUserIn = 1, kUserOut = 2, kWs = 3 };
struct Ref {
  int kind = kNone;
  long long off = 0;  // bytes
};

struct Stage {
  int family = 0, n = 0, es = 8;
  KernelInfo k;
  PassArgs a{};
  Ref in, in1, out, out1;
  void* in_tab = nullptr;  // device longlong2[n] or null
  void* out_tab = nullptr;
  long long grid = 0;
  long long tma_grid = 0;  // persistent grid of the TMA variant (0 = not usable)
  bool empty = false;
};

struct Xfer {
  int peer;
  Ref ref;
  size_t bytes;
};
struct Exchange {
  int comm = 0;  // 0 = row (P1 group), 1 = column (P2 group)
  std::vector<Xfer> sends, recvs;
  bool empty() const { return sends.empty() && recvs.empty(); }
};

struct RankPlan {
  int rank = 0, i = 0, j = 0;
  int64_t in_lo[3], in_n[3], out_lo[3], out_n[3];
  size_t in_bytes = 0, out_bytes = 0, ws_bytes = 0;
  void* ws = nullptr;
  std::vector<Stage> A, B;  // per chunk
  std::vector<Exchange> E1, E2;  // first / second exchange (each names its comm group)
  Stage C;
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
  size_t es = 8;  // complex element bytes
  std::vector<RankPlan> ranks;
  ncclComm_t row = nullptr, col = nullptr;
  cudaStream_t s_comp = nullptr, s_comm = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join_comp = nullptr, ev_join_comm = nullptr;
  std::vector<cudaEvent_t> evA, evE1, evB, evE2;
  void* stage_in = nullptr;  // dfft_execute_host staging buffers
  void* stage_out = nullptr;
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

// ------------------------------------------------------------------------------ stage builders
dfft_status_t upload_table(const std::vector<longlong2>& h, void** d) {
  CU(cudaMalloc(d, h.size() * sizeof(longlong2)));
  CU(cudaMemcpy(*d, h.data(), h.size() * sizeof(longlong2), cudaMemcpyHostToDevice));
  return DFFT_SUCCESS;
}

// table entry: {sel<<62 | element offset, line stride}
inline longlong2 tent(int sel, long long off, long long lstr) {
  longlong2 e;
  e.x = ((long long)sel << 62) | off;
  e.y = lstr;
  return e;
}

// A segmented side whose table is a single affine segment (one owner, e.g. P2 == 1) becomes an
// unsegmented side: base += toff(0), tstride = toff(1) - toff(0), lstride = lstr.
bool linearize(const std::vector<longlong2>& tab, Ref& base, const Ref& base1, SideMap& m, long long es, bool unit_t) {
  const long long mask = (1LL << 62) - 1;
  const long long sel = tab[0].x >> 62, off0 = tab[0].x & mask, lstr = tab[0].y;
  const long long ts = tab.size() > 1 ? (tab[1].x & mask) - off0 : 1;
  if (unit_t && ts != 1) return false;
  for (size_t t = 0; t < tab.size(); ++t)
    if ((tab[t].x >> 62) != sel || (tab[t].x & mask) != off0 + (long long)t * ts || tab[t].y != lstr) return false;
  Ref b = sel ? base1 : base;
  b.off += off0 * es;
  base = b;
  m.tstride = ts;
  m.lstride = lstr;
  return true;
}

dfft_status_t finish_stage(dfft_plan_t pl, Stage& s, int family, int n, long long L0, long long L1,
                           const std::vector<longlong2>* in_tab, const std::vector<longlong2>* out_tab) {
  if (in_tab && linearize(*in_tab, s.in, s.in1, s.a.in, (long long)pl->es, family == kContig)) in_tab = nullptr;
  if (out_tab && linearize(*out_tab, s.out, s.out1, s.a.out, (long long)pl->es, family == kContig)) out_tab = nullptr;
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
  if (in_tab) ST(upload_table(*in_tab, &s.in_tab));
  if (out_tab) ST(upload_table(*out_tab, &s.out_tab));
  s.a.in.ttab = (const longlong2*)s.in_tab;
  s.a.out.ttab = (const longlong2*)s.out_tab;
  if (family == kContig) s.grid = (L0 * L1 + s.k.per_cta - 1) / s.k.per_cta;
  else s.grid = ((L0 + s.k.per_cta - 1) / s.k.per_cta) * L1;
  if (s.grid >= (1LL << 31)) return fail(DFFT_ERR_UNSUPPORTED, "grid too large (%lld CTAs)", s.grid);
  if (family == kStrided && s.k.tma_fn && g_use_tma && !in_tab && tensor_map_encoder()) {
    const long long es = (long long)pl->es;
    bool ok = (s.a.in.tstride * es) % 16 == 0 && (L1 == 1 || (s.a.in.lstride * es) % 16 == 0) &&
              2 * L0 < (1LL << 32) && L1 < (1LL << 31);
    if (ok) {
      int occ = 0, dev = pl->comm->device, sms = 0;
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, s.k.tma_fn, s.k.tma_threads, s.k.tma_smem));
      CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      long long tiles = ((L0 + s.k.tma_w - 1) / s.k.tma_w) * L1;
      if (occ > 0) s.tma_grid = std::min<long long>(tiles, (long long)sms * occ);
    }
  }
  return DFFT_SUCCESS;
}

struct Geo {
  long long nx, ny, nz, nxc;
  long long P1, P2, K;
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
  long long xc(long long i, long long k) const { return blk(Xn(i), K, k); }
  long long x0(long long i, long long k) const { return blo(Xn(i), K, k); }
};

// Forward plan of one rank (all offsets in complex elements unless named *_b).
dfft_status_t build_forward(dfft_plan_t pl, const Geo& g, RankPlan& rp) {
  const long long i = rp.i, j = rp.j, K = g.K, es = (long long)pl->es;
  const long long Xn = g.Xn(i), Y1n = g.Y1n(i), Zn = g.Zn(j), Y3n = g.Y3n(j);
  // workspace: [S1 send1][R1 recv1][S2 send2]
  const long long S1 = 0, S1n = Y1n * Zn * (g.nxc - Xn);
  const long long R1 = S1 + S1n, R1n = g.ny * Zn * Xn;
  const long long S2 = R1 + R1n, S2n = Zn * Xn * (g.ny - Y3n);
  rp.ws_bytes = (size_t)(S2 + S2n) * es;
  if (g_oop_z && g.P1 == 1 && g.P2 == 1) rp.ws_bytes = std::max<size_t>(rp.ws_bytes, (size_t)(g.nxc * g.ny * g.nz * es));
  auto s1off = [&](long long k, long long ip) {
    long long acc = 0;
    for (long long q = 0; q < ip; ++q)
      if (q != i) acc += g.Xn(q);
    return S1 + Y1n * (g.z0(j, k) * (g.nxc - Xn) + g.zc(j, k) * acc);
  };
  auto s2off = [&](long long k, long long jp) {
    long long acc = 0;
    for (long long q = 0; q < jp; ++q)
      if (q != j) acc += g.Y3n(q);
    return S2 + Xn * (g.z0(j, k) * (g.ny - Y3n) + g.zc(j, k) * acc);
  };
  const long long in_es = pl->r2c ? es / 2 : es;  // bytes of one input element
  // P = 1 variant: A writes the transposed buffer into `out`, B writes natural order into the
  // workspace, C runs out of place workspace -> `out` (dev switch DFFT_OOP_Z)
  const bool oop = g_oop_z && g.P1 == 1 && g.P2 == 1;
  rp.A.resize(K);
  rp.B.resize(K);
  rp.E1.resize(K);
  rp.E2.resize(K);
  for (long long k = 0; k < K; ++k) {
    const long long zc = g.zc(j, k), z0 = g.z0(j, k);
    // ---- stage A: x-FFT of lines (y, zz); out segmented by x-owner i'
    Stage& A = rp.A[k];
    A.in = {kUserIn, z0 * Y1n * g.nx * in_es};
    A.a.in.tstride = 1;
    A.a.in.lstride = pl->r2c ? g.nx / 2 : g.nx;
    A.a.in_l0s = 1;
    A.a.in_l1s = Y1n;
    A.out = {oop ? kUserOut : kWs, 0};
    A.a.out_l0s = zc;  // Lidx = y·zc + zz
    A.a.out_l1s = 1;
    std::vector<longlong2> ot(g.nxc);
    for (long long t = 0; t < g.nxc; ++t) {
      long long ip = owner(t, g.nxc, g.P1), tl = t - g.Xlo(ip);
      if (ip == i) ot[t] = tent(0, R1 + g.ny * z0 * Xn + g.Y1lo(i) * zc * Xn + tl, Xn);
      else ot[t] = tent(0, s1off(k, ip) + tl, g.Xn(ip));
    }
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, kContig, (int)(pl->r2c ? g.nx / 2 : g.nx), Y1n, zc, nullptr, &ot));
    // ---- exchange 1 (row group)
    Exchange& E1 = rp.E1[k];
    E1.comm = 0;
    for (long long ip = 0; ip < g.P1; ++ip) {
      if (ip == i) continue;
      E1.sends.push_back({(int)ip, {kWs, s1off(k, ip) * es}, (size_t)(Y1n * zc * g.Xn(ip) * es)});
      E1.recvs.push_back({(int)ip, {kWs, (R1 + g.ny * z0 * Xn + g.Y1lo(ip) * zc * Xn) * es},
                          (size_t)(g.Y1n(ip) * zc * Xn * es)});
    }
    // ---- stage B: y-FFT of columns (x, zz) of recv1 chunk k; out segmented by y-owner j'
    Stage& B = rp.B[k];
    B.in = {oop ? kUserOut : kWs, (R1 + g.ny * z0 * Xn) * es};
    B.a.in.tstride = zc * Xn;
    B.a.in.lstride = Xn;
    B.out = {kWs, 0};
    B.out1 = {oop ? kWs : kUserOut, 0};
    std::vector<longlong2> bt(g.ny);
    for (long long t = 0; t < g.ny; ++t) {
      long long jp = owner(t, g.ny, g.P2), tl = t - g.Y3lo(jp);
      if (jp == j) bt[t] = tent(1, (g.Zlo(j) + z0) * Y3n * Xn + tl * Xn, Y3n * Xn);
      else bt[t] = tent(0, s2off(k, jp) + tl * Xn, g.Y3n(jp) * Xn);
    }
    B.a.scale = 1.0;
    ST(finish_stage(pl, B, kStrided, (int)g.ny, Xn, zc, nullptr, &bt));
    // ---- exchange 2 (column group): peers' chunk k lands in `out` at its z offset
    Exchange& E2 = rp.E2[k];
    E2.comm = 1;
    for (long long jp = 0; jp < g.P2; ++jp) {
      if (jp == j) continue;
      E2.sends.push_back({(int)jp, {kWs, s2off(k, jp) * es}, (size_t)(zc * g.Y3n(jp) * Xn * es)});
      E2.recvs.push_back({(int)jp, {kUserOut, (g.Zlo(jp) + g.z0(jp, k)) * Y3n * Xn * es},
                          (size_t)(g.zc(jp, k) * Y3n * Xn * es)});
    }
  }
  // ---- stage C: z-FFT in place on `out`
  Stage& C = rp.C;
  C.in = {oop ? kWs : kUserOut, 0};
  C.out = {kUserOut, 0};
  C.a.in.tstride = C.a.out.tstride = Y3n * Xn;
  C.a.in.lstride = C.a.out.lstride = Xn;
  C.a.scale = 1.0;
  ST(finish_stage(pl, C, kStrided, (int)g.nz, Xn, Y3n, nullptr, nullptr));
  return DFFT_SUCCESS;
}

// Single GPU (P = 1, any decomposition): no exchange, so the axis order is free (the 3D DFT is
// separable).  Order the stages so every stage writes at a small stride (large-stride stores
// throttle a pass; large-stride loads do not — r01 measurements):
//   forward: x (in -> out, natural), z (out -> ws as [y][z][x]), y (ws -> out, natural)
//   inverse: y (in -> out, natural), z (out -> ws as [y][z][x]), x (ws -> out, natural, ×1/N)
dfft_status_t build_single(dfft_plan_t pl, const Geo& g, RankPlan& rp) {
  const long long nx = g.nx, ny = g.ny, nz = g.nz, nxc = g.nxc, es = (long long)pl->es;
  rp.ws_bytes = (size_t)(nxc * ny * nz * es);
  rp.A.resize(1);
  rp.B.resize(1);
  rp.E1.resize(1);
  rp.E2.resize(1);
  Stage &A = rp.A[0], &B = rp.B[0], &C = rp.C;
  // z-pass: natural [z][y][x] -> ws [y][z][x]
  auto zpass = [&](Stage& Z) -> dfft_status_t {
    Z.in = {kUserOut, 0};
    Z.a.in.tstride = ny * nxc;
    Z.a.in.lstride = nxc;
    Z.out = {kWs, 0};
    Z.a.out.tstride = nxc;
    Z.a.out.lstride = nz * nxc;
    Z.a.scale = 1.0;
    return finish_stage(pl, Z, kStrided, (int)nz, nxc, ny, nullptr, nullptr);
  };
  if (pl->dir == DFFT_FORWARD) {
    A.in = {kUserIn, 0};
    A.a.in.tstride = 1;
    A.a.in.lstride = pl->r2c ? nx / 2 : nx;
    A.a.in_l0s = 1;
    A.a.in_l1s = ny;
    A.out = {kUserOut, 0};
    A.a.out.tstride = 1;
    A.a.out.lstride = nxc;
    A.a.out_l0s = 1;
    A.a.out_l1s = ny;
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, kContig, (int)(pl->r2c ? nx / 2 : nx), ny, nz, nullptr, nullptr));
    ST(zpass(B));
    C.in = {kWs, 0};
    C.a.in.tstride = nz * nxc;
    C.a.in.lstride = nxc;
    C.out = {kUserOut, 0};
    C.a.out.tstride = nxc;
    C.a.out.lstride = ny * nxc;
    C.a.scale = 1.0;
    ST(finish_stage(pl, C, kStrided, (int)ny, nxc, nz, nullptr, nullptr));
  } else {
    if (pl->r2c) return fail(DFFT_ERR_UNSUPPORTED, "C2R single-GPU path not built yet");
    A.in = {kUserIn, 0};
    A.a.in.tstride = nxc;
    A.a.in.lstride = ny * nxc;
    A.out = {kUserOut, 0};
    A.a.out.tstride = nxc;
    A.a.out.lstride = ny * nxc;
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, kStrided, (int)ny, nxc, nz, nullptr, nullptr));
    ST(zpass(B));
    C.in = {kWs, 0};
    C.a.in.tstride = 1;
    C.a.in.lstride = nxc;
    C.a.in_l0s = nz;  // line (y, z) of ws [y][z][x] is y·nz + z
    C.a.in_l1s = 1;
    C.out = {kUserOut, 0};
    C.a.out.tstride = 1;
    C.a.out.lstride = pl->r2c ? nx / 2 : nx;
    C.a.out_l0s = 1;
    C.a.out_l1s = ny;
    C.a.scale = 1.0 / ((double)nx * (double)ny * (double)nz);
    ST(finish_stage(pl, C, kContig, (int)(pl->r2c ? nx / 2 : nx), ny, nz, nullptr, nullptr));
  }
  return DFFT_SUCCESS;
}

// Inverse plan of one rank: z-IFFT (D3 in) → T2⁻¹ → y-IFFT → T1⁻¹ → x-IFFT ×1/N (D1 out).
dfft_status_t build_inverse(dfft_plan_t pl, const Geo& g, RankPlan& rp) {
  const long long i = rp.i, j = rp.j, K = g.K, es = (long long)pl->es;
  const long long Xn = g.Xn(i), Y1n = g.Y1n(i), Zn = g.Zn(j), Y3n = g.Y3n(j);
  // workspace: [S2' send][R2' recv][S1' send][R1' recv]
  const long long S2 = 0, S2n = Y3n * Xn * (g.nz - Zn);
  const long long R2 = S2 + S2n, R2n = g.ny * Zn * Xn;
  const long long S1 = R2 + R2n, S1n = Zn * Xn * (g.ny - Y1n);
  const long long R1 = S1 + S1n, R1n = g.nxc * Y1n * Zn;
  rp.ws_bytes = (size_t)(R1 + R1n) * es;
  auto s2off = [&](long long k, long long jp) {
    long long acc = 0;
    for (long long q = 0; q < jp; ++q)
      if (q != j) acc += g.Zn(q);
    return S2 + Y3n * (g.x0(i, k) * (g.nz - Zn) + g.xc(i, k) * acc);
  };
  auto s1off = [&](long long k, long long ip) {
    long long acc = 0;
    for (long long q = 0; q < ip; ++q)
      if (q != i) acc += g.Y1n(q);
    return S1 + Zn * (g.x0(i, k) * (g.ny - Y1n) + g.xc(i, k) * acc);
  };
  // recv1' block of (source row is, chunk k): [z][y ∈ Y1_me][xc_k(is)]
  auto r1off = [&](long long is, long long k) { return R1 + Zn * Y1n * (g.Xlo(is) + g.x0(is, k)); };
  rp.A.resize(K);
  rp.B.resize(K);
  rp.E1.resize(K);
  rp.E2.resize(K);
  for (long long k = 0; k < K; ++k) {
    const long long xc = g.xc(i, k), x0 = g.x0(i, k);
    // ---- stage A: z-IFFT of columns (xx, y') of `in`; out segmented by z-owner j'
    Stage& A = rp.A[k];
    A.in = {kUserIn, x0 * es};
    A.a.in.tstride = Y3n * Xn;
    A.a.in.lstride = Xn;
    A.out = {kWs, 0};
    std::vector<longlong2> at(g.nz);
    for (long long t = 0; t < g.nz; ++t) {
      long long jp = owner(t, g.nz, g.P2), tl = t - g.Zlo(jp);
      if (jp == j) at[t] = tent(0, R2 + g.ny * Zn * x0 + g.Y3lo(j) * Zn * xc + tl * xc, Zn * xc);
      else at[t] = tent(0, s2off(k, jp) + tl * xc, g.Zn(jp) * xc);
    }
    A.a.scale = 1.0;
    ST(finish_stage(pl, A, kStrided, (int)g.nz, xc, Y3n, nullptr, &at));
    // first exchange of the inverse = T2⁻¹ on the column group
    Exchange& E2 = rp.E1[k];
    E2.comm = 1;
    for (long long jp = 0; jp < g.P2; ++jp) {
      if (jp == j) continue;
      E2.sends.push_back({(int)jp, {kWs, s2off(k, jp) * es}, (size_t)(Y3n * g.Zn(jp) * xc * es)});
      E2.recvs.push_back({(int)jp, {kWs, (R2 + g.ny * Zn * x0 + g.Y3lo(jp) * Zn * xc) * es},
                          (size_t)(g.Y3n(jp) * Zn * xc * es)});
    }
    // ---- stage B: y-IFFT of columns (xx, z) of recv2' chunk k; out segmented by y-owner i'
    Stage& B = rp.B[k];
    B.in = {kWs, (R2 + g.ny * Zn * x0) * es};
    B.a.in.tstride = Zn * xc;
    B.a.in.lstride = xc;
    B.out = {kWs, 0};
    std::vector<longlong2> bt(g.ny);
    for (long long t = 0; t < g.ny; ++t) {
      long long ip = owner(t, g.ny, g.P1), tl = t - g.Y1lo(ip);
      if (ip == i) bt[t] = tent(0, r1off(i, k) + tl * xc, Y1n * xc);
      else bt[t] = tent(0, s1off(k, ip) + tl * xc, g.Y1n(ip) * xc);
    }
    B.a.scale = 1.0;
    ST(finish_stage(pl, B, kStrided, (int)g.ny, xc, Zn, nullptr, &bt));
    // second exchange of the inverse = T1⁻¹ on the row group
    Exchange& E1 = rp.E2[k];
    E1.comm = 0;
    for (long long ip = 0; ip < g.P1; ++ip) {
      if (ip == i) continue;
      E1.sends.push_back({(int)ip, {kWs, s1off(k, ip) * es}, (size_t)(Zn * g.Y1n(ip) * xc * es)});
      E1.recvs.push_back({(int)ip, {kWs, r1off(ip, k) * es}, (size_t)(Zn * Y1n * g.xc(ip, k) * es)});
    }
  }
  // ---- stage C: x-IFFT of lines (y, z); input segmented by (source row, chunk); ×1/N
  Stage& C = rp.C;
  C.in = {kWs, 0};
  C.a.in_l0s = 1;
  C.a.in_l1s = Y1n;
  std::vector<longlong2> ct(g.nxc);
  for (long long t = 0; t < g.nxc; ++t) {
    long long is = owner(t, g.nxc, g.P1), tl1 = t - g.Xlo(is);
    long long k = owner(tl1, g.Xn(is), K), tl = tl1 - g.x0(is, k);
    ct[t] = tent(0, r1off(is, k) + tl, g.xc(is, k));
  }
  C.out = {kUserOut, 0};
  C.a.out.tstride = 1;
  C.a.out.lstride = pl->r2c ? g.nx / 2 : g.nx;
  C.a.out_l0s = 1;
  C.a.out_l1s = Y1n;
  C.a.scale = 1.0 / ((double)g.nx * (double)g.ny * (double)g.nz);
  ST(finish_stage(pl, C, kContig, (int)(pl->r2c ? g.nx / 2 : g.nx), Y1n, Zn, &ct, nullptr));
  return DFFT_SUCCESS;
}

// ------------------------------------------------------------------------------ execution
void* resolve(const Ref& r, const void* in, void* out, void* ws) {
  switch (r.kind) {
    case kUserIn: return (char*)in + r.off;
    case kUserOut: return (char*)out + r.off;
    case kWs: return (char*)ws + r.off;
    default: return nullptr;
  }
}

dfft_status_t launch(const Stage& s, const void* in, void* out, void* ws, cudaStream_t st) {
  if (s.empty) return DFFT_SUCCESS;
  PassArgs a = s.a;
  a.in.base = resolve(s.in, in, out, ws);
  a.in.base1 = resolve(s.in1, in, out, ws);
  a.out.base = resolve(s.out, in, out, ws);
  a.out.base1 = resolve(s.out1, in, out, ws);
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
    CUtensorMap tin, tout;
    if (encode(&tin, a.in.base, a.in.tstride, a.in.lstride)) {
      bool use_st = g_tma_store && a.out.ttab == nullptr && ((uintptr_t)a.out.base & 15) == 0 &&
                (a.out.tstride * (long long)ces) % 16 == 0 && (a.L1 == 1 || (a.out.lstride * (long long)ces) % 16 == 0) &&
                encode(&tout, a.out.base, a.out.tstride, a.out.lstride);
      if (!use_st) tout = tin;  // unused by the non-TST variant
      void* targs[] = {&tin, &tout, &a};
      CU(cudaLaunchKernel(use_st ? s.k.tma_st_fn : s.k.tma_fn, dim3((unsigned)s.tma_grid), dim3(s.k.tma_threads), targs,
                          s.k.tma_smem, st));
      return DFFT_SUCCESS;
    }
  }
  void* args[] = {&a};
  CU(cudaLaunchKernel(s.k.fn, dim3((unsigned)s.grid), dim3(s.k.threads), args, s.k.smem, st));
  return DFFT_SUCCESS;
}

dfft_status_t exchange_nccl(dfft_plan_t pl, const Exchange& x, const void* in, void* out, void* ws,
                            cudaStream_t st) {
  if (x.empty()) return DFFT_SUCCESS;
  ncclComm_t c = x.comm == 0 ? pl->row : pl->col;
  NC(ncclGroupStart());
  for (const Xfer& s : x.sends) NC(ncclSend(resolve(s.ref, in, out, ws), s.bytes, ncclUint8, s.peer, c, st));
  for (const Xfer& r : x.recvs) NC(ncclRecv(resolve(r.ref, in, out, ws), r.bytes, ncclUint8, r.peer, c, st));
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
      void* sp = resolve(s.ref, ins[r], outs[r], src.ws);
      void* dp = resolve(rv->ref, ins[q], outs[q], dst.ws);
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
dfft_status_t launch_p(dfft_plan_t pl, int phase, const Stage& s, const void* in, void* out, void* ws,
                       cudaStream_t st) {
  if (s.empty) return DFFT_SUCCESS;
  size_t slot = 0;
  ST(prof_begin(pl, phase, st, &slot));
  ST(launch(s, in, out, ws, st));
  return prof_end(pl, slot, st);
}
dfft_status_t exchange_p(dfft_plan_t pl, int phase, const Exchange& x, const void* in, void* out, void* ws,
                         cudaStream_t st) {
  if (x.empty()) return DFFT_SUCCESS;
  size_t slot = 0;
  ST(prof_begin(pl, phase, st, &slot));
  ST(exchange_nccl(pl, x, in, out, ws, st));
  return prof_end(pl, slot, st);
}

dfft_status_t execute_rank(dfft_plan_t pl, const void* in, void* out, cudaStream_t user) {
  RankPlan& rp = pl->ranks[0];
  const size_t K = rp.A.size();
  void* ws = rp.ws;
  if (!pl->overlap) {
    // static-barrier ablation: every step in program order on the user's stream
    for (size_t k = 0; k < K; ++k) ST(launch_p(pl, 0, rp.A[k], in, out, ws, user));
    for (size_t k = 0; k < K; ++k) ST(exchange_p(pl, 1, rp.E1[k], in, out, ws, user));
    for (size_t k = 0; k < K; ++k) ST(launch_p(pl, 2, rp.B[k], in, out, ws, user));
    for (size_t k = 0; k < K; ++k) ST(exchange_p(pl, 3, rp.E2[k], in, out, ws, user));
    return launch_p(pl, 4, rp.C, in, out, ws, user);
  }
  cudaStream_t sc = pl->s_comp, sm = pl->s_comm;
  CU(cudaEventRecord(pl->ev_fork, user));
  CU(cudaStreamWaitEvent(sc, pl->ev_fork, 0));
  CU(cudaStreamWaitEvent(sm, pl->ev_fork, 0));
  // host issue order is a topological order of the chunk DAG, so every wait refers to the
  // record issued in this execute:  A0 E1_0 | A1 E1_1 B0 E2_0 | A2 E1_2 B1 E2_1 | ...
  auto do_A = [&](size_t k) -> dfft_status_t {
    ST(launch_p(pl, 0, rp.A[k], in, out, ws, sc));
    if (!rp.E1[k].empty()) {
      CU(cudaEventRecord(pl->evA[k], sc));
      CU(cudaStreamWaitEvent(sm, pl->evA[k], 0));
      ST(exchange_p(pl, 1, rp.E1[k], in, out, ws, sm));
      CU(cudaEventRecord(pl->evE1[k], sm));
    }
    return DFFT_SUCCESS;
  };
  ST(do_A(0));
  for (size_t k = 0; k < K; ++k) {
    if (k + 1 < K) ST(do_A(k + 1));
    if (!rp.E1[k].empty()) CU(cudaStreamWaitEvent(sc, pl->evE1[k], 0));
    ST(launch_p(pl, 2, rp.B[k], in, out, ws, sc));
    if (!rp.E2[k].empty()) {
      CU(cudaEventRecord(pl->evB[k], sc));
      CU(cudaStreamWaitEvent(sm, pl->evB[k], 0));
      ST(exchange_p(pl, 3, rp.E2[k], in, out, ws, sm));
      CU(cudaEventRecord(pl->evE2[k], sm));
    }
  }
  // stage C needs every chunk of exchange 2 (same comm stream => the last record suffices)
  if (!rp.E2[K - 1].empty()) CU(cudaStreamWaitEvent(sc, pl->evE2[K - 1], 0));
  ST(launch_p(pl, 4, rp.C, in, out, ws, sc));
  CU(cudaEventRecord(pl->ev_join_comp, sc));
  CU(cudaEventRecord(pl->ev_join_comm, sm));
  CU(cudaStreamWaitEvent(user, pl->ev_join_comp, 0));
  CU(cudaStreamWaitEvent(user, pl->ev_join_comm, 0));
  return DFFT_SUCCESS;
}

dfft_status_t execute_sim(dfft_plan_t pl, const void* const* ins, void* const* outs, cudaStream_t st) {
  const size_t P = pl->ranks.size(), K = pl->ranks[0].A.size();
  for (size_t k = 0; k < K; ++k)
    for (size_t r = 0; r < P; ++r) ST(launch(pl->ranks[r].A[k], ins[r], outs[r], pl->ranks[r].ws, st));
  for (size_t k = 0; k < K; ++k) ST(exchange_sim(pl, false, k, ins, outs, st));
  for (size_t k = 0; k < K; ++k)
    for (size_t r = 0; r < P; ++r) ST(launch(pl->ranks[r].B[k], ins[r], outs[r], pl->ranks[r].ws, st));
  for (size_t k = 0; k < K; ++k) ST(exchange_sim(pl, true, k, ins, outs, st));
  for (size_t r = 0; r < P; ++r) ST(launch(pl->ranks[r].C, ins[r], outs[r], pl->ranks[r].ws, st));
  return DFFT_SUCCESS;
}

void free_stage(Stage& s) {
  if (s.in_tab) cudaFree(s.in_tab);
  if (s.out_tab) cudaFree(s.out_tab);
  s.in_tab = s.out_tab = nullptr;
}

void free_plan(dfft_plan_t pl) {
  if (!pl) return;
  if (pl->s_comp) cudaStreamSynchronize(pl->s_comp);
  if (pl->s_comm) cudaStreamSynchronize(pl->s_comm);
  for (RankPlan& rp : pl->ranks) {
    for (Stage& s : rp.A) free_stage(s);
    for (Stage& s : rp.B) free_stage(s);
    free_stage(rp.C);
    if (rp.ws) cudaFree(rp.ws);
  }
  for (auto* v : {&pl->evA, &pl->evE1, &pl->evB, &pl->evE2})
    for (cudaEvent_t e : *v) cudaEventDestroy(e);
  for (cudaEvent_t e : pl->prof_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : {pl->ev_fork, pl->ev_join_comp, pl->ev_join_comm})
    if (e) cudaEventDestroy(e);
  if (pl->s_comp) cudaStreamDestroy(pl->s_comp);
  if (pl->s_comm) cudaStreamDestroy(pl->s_comm);
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

}  // namespace

// ================================================================================ C ABI
extern "C" {

int dfft_version(void) { return DFFT_VERSION; }

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
  if (type < DFFT_C2C_F32 || type > DFFT_R2C_F64) return fail(DFFT_ERR_INVALID_VALUE, "bad type");
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
  if (r2c && nx % 2) return fail(DFFT_ERR_UNSUPPORTED, "R2C needs even nx");
  long long nxc = r2c ? nx / 2 + 1 : nx;
  long long nfft_x = r2c ? nx / 2 : nx;
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
  Geo g{nx, ny, nz, r2c ? nx / 2 + 1 : nx, p1, p2, 1};
  long long i = rank / p2, j = rank % p2;
  int64_t d1lo[3] = {0, g.Y1lo(i), g.Zlo(j)}, d1n[3] = {nx, g.Y1n(i), g.Zn(j)};
  int64_t d3lo[3] = {g.Xlo(i), g.Y3lo(j), 0}, d3n[3] = {g.Xn(i), g.Y3n(j), nz};
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
  bool f64 = type == DFFT_C2C_F64 || type == DFFT_R2C_F64;
  if (r2c) return fail(DFFT_ERR_UNSUPPORTED, "R2C/C2R not available in this build yet");
  long long nxc = r2c ? nx / 2 + 1 : nx;
  int Kreq = (int)(flags & 0xff);
  bool overlap = !(flags & DFFT_FLAG_NO_OVERLAP);
  long long kmax = direction == DFFT_FORWARD ? nz / p2 : nxc / p1;
  long long K = Kreq > 0 ? Kreq : (P > 1 ? 4 : 1);
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
  pl->overlap = overlap;
  pl->es = f64 ? 16 : 8;
  Geo g{nx, ny, nz, nxc, p1, p2, K};

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
    int64_t d3lo[3] = {g.Xlo(rp.i), g.Y3lo(rp.j), 0}, d3n[3] = {g.Xn(rp.i), g.Y3n(rp.j), nz};
    size_t real_es = pl->es / 2;
    size_t d1b = (size_t)(d1n[0] * d1n[1] * d1n[2]) * (r2c ? real_es : pl->es);
    size_t d3b = (size_t)(d3n[0] * d3n[1] * d3n[2]) * pl->es;
    if (direction == DFFT_FORWARD) {
      memcpy(rp.in_lo, d1lo, sizeof d1lo);
      memcpy(rp.in_n, d1n, sizeof d1n);
      memcpy(rp.out_lo, d3lo, sizeof d3lo);
      memcpy(rp.out_n, d3n, sizeof d3n);
      rp.in_bytes = d1b;
      rp.out_bytes = d3b;
      ST(P == 1 ? build_single(pl, g, rp) : build_forward(pl, g, rp));
    } else {
      memcpy(rp.in_lo, d3lo, sizeof d3lo);
      memcpy(rp.in_n, d3n, sizeof d3n);
      memcpy(rp.out_lo, d1lo, sizeof d1lo);
      memcpy(rp.out_n, d1n, sizeof d1n);
      rp.in_bytes = d3b;
      rp.out_bytes = d1b;
      ST(P == 1 ? build_single(pl, g, rp) : build_inverse(pl, g, rp));
    }
    if (rp.ws_bytes) {
      cudaError_t e = cudaMalloc(&rp.ws, rp.ws_bytes);
      if (e != cudaSuccess) return fail(DFFT_ERR_ALLOC, "workspace of %zu bytes: %s", rp.ws_bytes, cudaGetErrorString(e));
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
  s.a.in.tstride = s.a.out.tstride = 1;
  s.a.in.lstride = s.a.out.lstride = n;
  s.a.in_l0s = s.a.out_l0s = 1;
  s.a.in_l1s = s.a.out_l1s = 0;
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
int length_schedule(int n, int rad[kMaxPass]) {
  Sched s = make_sched(n);
  for (int p = 0; p < kMaxPass; ++p) rad[p] = s.rad[p];
  return s.npass;
}
}  // namespace dfft
