// fft_kernels.cuh — sm_100a batched 1D FFT kernels of the distributed 3D FFT.
//
// Each stage of the paper's pipeline is "independent 1D FFTs" along one axis (P:101-105,
// §III-A; Alg. 1 stages 1-3).  Two kernel families compute a batch of length-N
// lines with a mixed-radix Stockham autosort FFT (radix 16/8/4/2 first, then 3/5/7):
//   * contig  — the FFT axis is unit stride on the read side (stage-1 x lines, and the
//               inverse's last x stage).  LPC lines per CTA, T threads per line.
//   * strided — the FFT axis is strided; W adjacent unit-stride columns per CTA so every
//               row access is a 64-128 B coalesced segment (stages 2-3, y and z).
// Pass p (radix R, Ns = product of earlier radices) maps butterfly b < N/R:
//     v[r] = X[b + r·N/R] · w_{Ns·R}^{(b mod Ns)·r},  V = DFT_R(v),
//     Y[(b/Ns)·Ns·R + (b mod Ns) + r·Ns] = V[r]
// so the first pass reads and the last pass writes consecutive addresses across threads
// (coalesced straight from/to HBM, no staging pass); the passes in between exchange through
// padded shared memory (conflict-free layouts chosen with tools/bank_sim.py).  Twiddles
// come from per-pass tables in HBM (long-double generated, [r-1][m] layout so a warp's
// loads coalesce), never from recurrences.
//
// The pack / unpack of the redistribution (Alg. 2 phases 3-5) is fused into
// the global side of the first and last pass through a SideMap: element t of line
// (l0, l1) lives at  base + toff(t) + Lidx·lstr(t) + c0  where (toff, lstr) come either
// from a closed form (unsegmented side) or from a per-t table (segmented side: t ranges
// owned by different peers land in different send blocks / buffers).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dfft {

// --------------------------------------------------------------------------------- types
template <typename Real> struct CT;
template <> struct CT<float> { using type = float2; };
template <> struct CT<double> { using type = double2; };

template <typename C> __device__ __forceinline__ C cadd(C a, C b) { return {a.x + b.x, a.y + b.y}; }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { return {a.x - b.x, a.y - b.y}; }
// Fixed contraction (a.x·b.x − a.y·b.y as one fma over a rounded product, likewise the imaginary
// part): every kernel rounds a twiddle multiply the same way whether the twiddle sits in a register
// or comes from a load, so the transports' outputs stay bit-identical (test_gpu_executor.py).
template <typename C> __device__ __forceinline__ C cmul(C a, C b) {
  if constexpr (sizeof(a.x) == 4)
    return {__fmaf_rn(a.x, b.x, -__fmul_rn(a.y, b.y)), __fmaf_rn(a.x, b.y, __fmul_rn(a.y, b.x))};
  else
    return {__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)), __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x))};
}
// a · (DIR·i):  forward (DIR=-1) multiplies by -i, inverse by +i
template <int DIR, typename C> __device__ __forceinline__ C mul_i(C a) {
  if (DIR < 0) return {a.y, -a.x};
  return {-a.y, a.x};
}

// --------------------------------------------------------------------------------- schedule
constexpr int kMaxPass = 8;
struct Sched {
  int n, npass, T;
  int rad[kMaxPass];
};
// radix-MAXR (16 or 32) passes first, then the 2^k remainder, then 3, 5, 7.
constexpr Sched make_sched(int n, int maxr = 16) {
  Sched s{n, 0, 1, {0, 0, 0, 0, 0, 0, 0, 0}};
  int m = n, odd[kMaxPass] = {0, 0, 0, 0, 0, 0, 0, 0}, nodd = 0;
  for (int p = 7; p >= 3; p -= 2)
    while (m % p == 0) { odd[nodd++] = p; m /= p; }
  while (m % maxr == 0) { s.rad[s.npass++] = maxr; m /= maxr; }
  if (m >= 32) { s.rad[s.npass++] = 16; m /= 16; }
  if (m > 1) s.rad[s.npass++] = m;  // 2, 4, 8 or 16
  for (int q = nodd - 1; q >= 0; --q) s.rad[s.npass++] = odd[q];
  int rmax = 1;
  for (int p = 0; p < s.npass; ++p) rmax = s.rad[p] > rmax ? s.rad[p] : rmax;
  s.T = n / rmax;
  return s;
}
constexpr int sched_ns(const Sched& s, int p) {
  int ns = 1;
  for (int q = 0; q < p; ++q) ns *= s.rad[q];
  return ns;
}
// offset (in complex elements) of pass p's twiddle table: Σ_{1<=q<p} (R_q - 1)·Ns_q
constexpr int sched_twoff(const Sched& s, int p) {
  int off = 0;
  for (int q = 1; q < p; ++q) off += (s.rad[q] - 1) * sched_ns(s, q);
  return off;
}
constexpr int sched_twlen(const Sched& s) { return sched_twoff(s, s.npass); }

// --------------------------------------------------------------------------------- butterflies
// exp(-2πi m/16) constants: cos and sin of 2πm/16 for m = 0..3 (the rest by symmetry)
#define DFFT_C16_1 0.92387953251128675613
#define DFFT_S16_1 0.38268343236508977173
#define DFFT_SQH 0.70710678118654752440

// cos(2πq/32), q ∈ [0, 8]
__host__ __device__ constexpr double cos32(int q) {
  return q == 0 ? 1.0 : q == 1 ? 0.98078528040323044913 : q == 2 ? 0.92387953251128675613
       : q == 3 ? 0.83146961230254523708 : q == 4 ? 0.70710678118654752440 : q == 5 ? 0.55557023301960222474
       : q == 6 ? 0.38268343236508977173 : q == 7 ? 0.19509032201612826785 : 0.0;
}
// a · w_32^q, w_32 = exp(DIR·2πi/32), q a compile-time constant after unrolling
template <int DIR, typename C>
__device__ __forceinline__ C tw32(C a, int q) {
  using Real = decltype(a.x);
  q &= 31;
  if (q == 0) return a;
  if (q == 16) return {-a.x, -a.y};
  if (q == 8) return mul_i<DIR>(a);
  if (q == 24) return mul_i<-DIR>(a);
  // cos/sin of 2πq/32 by quadrant
  const int r = q & 7, quad = q >> 3;
  const Real cb = (Real)cos32(r), sb = (Real)cos32(8 - r);
  Real c = quad == 0 ? cb : quad == 1 ? -sb : quad == 2 ? -cb : sb;
  Real sn = quad == 0 ? sb : quad == 1 ? cb : quad == 2 ? -sb : -cb;
  const Real ws = DIR < 0 ? -sn : sn;
  return {a.x * c - a.y * ws, a.x * ws + a.y * c};
}

// a · w_R^m with w_R = exp(DIR·2πi/R), R ∈ {2,4,8,16}; m is a compile-time constant after
// unrolling, so every branch folds.
template <int DIR, int R, typename C>
__device__ __forceinline__ C twc(C a, int m) {
  using Real = decltype(a.x);
  int q = (m * (16 / R)) & 15;  // index in 16ths of a turn
  if (q == 0) return a;
  if (q == 8) return {-a.x, -a.y};
  if (q == 4) return mul_i<DIR>(a);
  if (q == 12) return mul_i<-DIR>(a);
  // cos/sin of 2πq/16 for the remaining q
  Real c, s;
  int q4 = q & 3;
  Real cb = q4 == 1 ? (Real)DFFT_C16_1 : q4 == 2 ? (Real)DFFT_SQH : (Real)DFFT_S16_1;
  Real sb = q4 == 1 ? (Real)DFFT_S16_1 : q4 == 2 ? (Real)DFFT_SQH : (Real)DFFT_C16_1;
  if (q < 4) { c = cb; s = sb; }
  else if (q < 8) { c = -sb; s = cb; }
  else if (q < 12) { c = -cb; s = -sb; }
  else { c = sb; s = -cb; }
  // w = c + DIR·i·s
  Real ws = DIR < 0 ? -s : s;
  return {a.x * c - a.y * ws, a.x * ws + a.y * c};
}

template <int DIR, typename C> __device__ __forceinline__ void dft2(C& a, C& b) {
  C t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <int DIR, typename C> __device__ __forceinline__ void dft4(C& a0, C& a1, C& a2, C& a3) {
  C t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = mul_i<DIR>(csub(a1, a3));
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, t3);
  a3 = csub(t1, t3);
}

// odd prime radix by the symmetric-pair form:
//   X_k = a0 + Σ_m cos θ (a_m + a_{R-m}) + DIR·i Σ_m sin θ (a_m - a_{R-m}),  θ = 2π m k / R
// cos(2πq/R) and sin(2πq/R) for R ∈ {3,5,7}, q ∈ [0, R)
__host__ __device__ constexpr double odd_cos(int R, int q) {
  return q == 0 ? 1.0
       : R == 3 ? -0.5
       : R == 5 ? ((q == 1 || q == 4) ? 0.30901699437494742410 : -0.80901699437494742410)
       : ((q == 1 || q == 6) ? 0.62348980185873353053
          : (q == 2 || q == 5) ? -0.22252093395631440429 : -0.90096886790241912624);
}
__host__ __device__ constexpr double odd_sin(int R, int q) {
  return q == 0 ? 0.0
       : (2 * q > R ? -1.0 : 1.0) *
         (R == 3 ? 0.86602540378443864676
          : R == 5 ? ((q == 1 || q == 4) ? 0.95105651629515357212 : 0.58778525229247312917)
          : ((q == 1 || q == 6) ? 0.78183148246802980871
             : (q == 2 || q == 5) ? 0.97492791218182360702 : 0.43388373911755812048));
}

template <int DIR, int R, typename C> __device__ __forceinline__ void dft_odd(C* v) {
  using Real = decltype(v[0].x);
  constexpr int H = (R - 1) / 2;
  C sp[H + 1], sm[H + 1];
#pragma unroll
  for (int m = 1; m <= H; ++m) {
    sp[m] = cadd(v[m], v[R - m]);
    sm[m] = csub(v[m], v[R - m]);
  }
  C x0 = v[0];
  C sum = x0;
#pragma unroll
  for (int m = 1; m <= H; ++m) sum = cadd(sum, sp[m]);
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    C re = x0, im = {0, 0};
#pragma unroll
    for (int m = 1; m <= H; ++m) {
      const Real c = (Real)odd_cos(R, (m * k) % R), s = (Real)odd_sin(R, (m * k) % R);
      re.x += c * sp[m].x;
      re.y += c * sp[m].y;
      im.x += s * sm[m].x;
      im.y += s * sm[m].y;
    }
    // DIR·i·im
    C t = mul_i<DIR>(im);
    v[k] = cadd(re, t);
    v[R - k] = csub(re, t);
  }
  v[0] = sum;
}

template <int DIR, int R, typename C> __device__ __forceinline__ void dft(C* v);

// DFT_{A·B} by one Cooley-Tukey step: n = B·n1 + n2, k = k1 + A·k2,
//   X[k1 + A k2] = Σ_{n2} w_B^{n2 k2} · [w_{AB}^{n2 k1} · Σ_{n1} x[B n1 + n2] w_A^{n1 k1}]
template <int DIR, int A, int B, typename C> __device__ __forceinline__ void dft_ct(C* v) {
  constexpr int R = A * B;
  C t[R];
#pragma unroll
  for (int n2 = 0; n2 < B; ++n2) {
    C u[A];
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) u[n1] = v[B * n1 + n2];
    dft<DIR, A>(u);
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) t[n2 * A + k1] = tw32<DIR>(u[k1], (n2 * k1 * (32 / R)) & 31);
  }
#pragma unroll
  for (int k1 = 0; k1 < A; ++k1) {
    C u[B];
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) u[n2] = t[n2 * A + k1];
    dft<DIR, B>(u);
#pragma unroll
    for (int k2 = 0; k2 < B; ++k2) v[k1 + A * k2] = u[k2];
  }
}

// DFT_R in registers, in place, natural order in and out.
template <int DIR, int R, typename C> __device__ __forceinline__ void dft(C* v) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    dft2<DIR>(v[0], v[1]);
  } else if constexpr (R == 4) {
    dft4<DIR>(v[0], v[1], v[2], v[3]);
  } else if constexpr (R == 8) {
    // 8 = 2 (A) × 4 (B): n = 4 n1 + n2, k = k1 + 2 k2
    dft2<DIR>(v[0], v[4]);
    dft2<DIR>(v[1], v[5]);
    dft2<DIR>(v[2], v[6]);
    dft2<DIR>(v[3], v[7]);
    // Y[n2][k1] at v[n2 + 4 k1]; twiddle w8^{n2 k1}
    v[5] = twc<DIR, 8>(v[5], 1);
    v[6] = twc<DIR, 8>(v[6], 2);
    v[7] = twc<DIR, 8>(v[7], 3);
    dft4<DIR>(v[0], v[1], v[2], v[3]);  // k1 = 0 -> X[0,2,4,6]
    dft4<DIR>(v[4], v[5], v[6], v[7]);  // k1 = 1 -> X[1,3,5,7]
    C t[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) t[i] = v[i];
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      v[2 * k2] = t[k2];
      v[2 * k2 + 1] = t[4 + k2];
    }
  } else if constexpr (R == 16) {
    // 16 = 4 (A) × 4 (B): n = 4 n1 + n2, k = k1 + 4 k2
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4<DIR>(v[n2], v[n2 + 4], v[n2 + 8], v[n2 + 12]);
    // now v[n2 + 4 k1] = Y[n2][k1]; twiddle w16^{n2 k1}
#pragma unroll
    for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
      for (int k1 = 1; k1 < 4; ++k1) v[n2 + 4 * k1] = twc<DIR, 16>(v[n2 + 4 * k1], n2 * k1);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4<DIR>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
    // v[4 k1 + k2] = X[k1 + 4 k2]: transpose 4x4
    C t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = v[i];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = t[4 * k1 + k2];
  } else if constexpr (R == 32) {
    dft_ct<DIR, 4, 8>(v);
  } else {
    static_assert(R == 3 || R == 5 || R == 7, "unsupported radix");
    dft_odd<DIR, R>(v);
  }
}

// --------------------------------------------------------------------------------- side maps
// Where element t of a line lives on the global side of a pass (input of the first pass or
// output of the last pass).  Unsegmented: toff = t·tstride, lstr = lstride.  Segmented: a
// per-t table {toff, lstr} built at plan time (send-block routing = the fused pack/unpack).
constexpr int kMaxBases = 16;
// Element (t, l0, l1) of a side lives at  base + off(t) + l0·s0 + l1·s1  (complex elements):
//   unsegmented: off(t) = t·tstride, (s0, s1) from the map;
//   segmented:   a per-t table entry {sel<<56 | off(t), s0, s1} — t ranges owned by different
//                peers live in different send blocks / windows with their own layouts.
struct SegEnt {
  long long off;  // sel << 56 | element offset of (t, 0, 0) relative to bases[sel]
  int s0, s1;     // line strides of this segment
};
// One segment of a column-blocked segmented output side, as the persistent strided kernel's bulk
// epilogue sees it: rows t ∈ [tlo, tlo+tn) of a tile land contiguously at bases[sel] +
// off0 + (block·mT + l1)·s1 (requires t-stride == bw == tile width, column stride 1).
constexpr int kMaxBulk = 16;
struct BulkSeg {
  long long off0, s1;
  int tlo, tn, sel;
};
struct SideMap {
  void* base;                 // unsegmented: the side's pointer
  void* bases[kMaxBases];     // segmented: base pointer per selector (local buffers, peers' windows)
  const SegEnt* ttab;         // nullptr => unsegmented
  long long tstride, s0, s1;  // unsegmented strides (elements)
  // column-blocked layouts (bw > 0): column l0 lives in block l0/bw at position l0%bw, and the
  // block index strides like mT lines of l1:  off(t) + (l0%bw)·s0 + ((l0/bw)·mT + l1)·s1.
  // A warp's rows of one block are then contiguous (256 B pieces over NVLink).
  int bw;
  long long mT;
  // t-blocked unsegmented side (tb > 0, contig family): t lives at (t/tb)·tbs + t%tb — the
  // column-blocked receive windows seen along the FFT axis, without a per-t table
  int tb;
  long long tbs;
  // bulk epilogue (output side of the persistent strided kernel, OM = 2): one
  // cp.async.bulk shared→global copy per segment per tile instead of per-element stores
  int nbulk;
  BulkSeg bulk[kMaxBulk];
};

// effective (l0, l1) of a side for column l0 / line l1 (blocked layouts fold the block into l1)
__device__ __forceinline__ void side_lines(const SideMap& m, long long l0, long long l1, long long& e0, long long& e1) {
  if (m.bw > 0) {
    const long long xb = l0 / m.bw;
    e0 = l0 - xb * m.bw;
    e1 = xb * m.mT + l1;
  } else {
    e0 = l0;
    e1 = l1;
  }
}

template <typename C>
__device__ __forceinline__ C* seg_ptr(const SideMap& m, int t, long long l0, long long l1) {
  const longlong2 raw = __ldg(reinterpret_cast<const longlong2*>(m.ttab) + t);
  const int s0 = (int)(raw.y & 0xffffffffLL), s1 = (int)(raw.y >> 32);
  C* b = reinterpret_cast<C*>(m.bases[(unsigned long long)raw.x >> 56]);
  return b + ((raw.x & ((1LL << 56) - 1)) + l0 * s0 + l1 * s1);
}

// Global store of one complex value from the last pass (DFFT_STORE_CS: streaming hint, dev A/B).
template <typename C> __device__ __forceinline__ void st_out(C* p, C v) {
#ifdef DFFT_STORE_CS
  __stcs(p, v);
#else
  *p = v;
#endif
}

// Kernel arguments shared by both families.
struct PassArgs {
  SideMap in, out;
  const void* tw;    // per-pass twiddle tables (complex), sched_twoff layout
  const void* tw2;   // R2C/C2R: w^k = exp(DIR·2πi·k/(2N)), k < N (the split/merge twiddles)
  const void* tw3;   // R2R (DCT): c_k = exp(DIR·iπk/(2L)), k < L, L = the real line length
  long long L0, L1;  // line grid: lines (l0, l1), l0 < L0, l1 < L1 (strided: l0 = the column)
  double scale;      // applied to the outputs of the last pass (1 = none)
  // persistent strided kernels: tile order.  Tiles run in groups of g0 column tiles × all L1
  // (column tile fastest inside a group); g0 = 0 means one group (column tile fastest overall).
  // Concurrently resident CTAs then touch g0 adjacent column tiles × (#CTAs / g0) adjacent
  // lines: g0 = 1 suits a side where adjacent l1 are adjacent in memory (column-blocked
  // windows), a small g0 balances a blocked side against a natural one.
  int g0;
  // spectral multiplier of the last forward stage (dfft_plan_set_poisson): per-axis tables of
  // the discrete Laplacian's eigenvalues λ_d (Real, indexed by the local t / l0 / l1 of this stage,
  // already offset to the rank's global bins); each output is multiplied by 1/(λt+λ0+λ1), 0 at
  // k = 0.  spec[0] == nullptr: off.
  const void* spec[3];
  // R2R plans: a complex column l0 carries two real x columns (bins 2·l0 and 2·l0+1), so the x table
  // (spec[1]) holds one eigenvalue per real bin and re / im take their own factor
  int spec_pairs;
  // contig family: line order of consecutive CTAs — 0: l0 fastest, 1: l1 fastest (the host picks the
  // order whose consecutive lines are adjacent on the output side: scattered 8 KB writes cost more
  // than scattered 8 KB reads)
  int lorder;
  // generic kernels (lengths without a specialised instantiation): the radix schedule at run time
  // and the lines (contig) / columns (strided) per CTA
  Sched gen;
  int gen_per;
};

// tile -> (column tile tx, line l1) under the grouped order above
__device__ __forceinline__ void tile_coords(long long tile, long long ntile, long long L1, int g0, long long& tx,
                                            long long& l1) {
  if (g0 <= 0 || g0 >= ntile) {
    l1 = tile / ntile;
    tx = tile - l1 * ntile;
    return;
  }
  const long long grp = tile / ((long long)g0 * L1);
  const long long base = grp * g0;
  const long long gw = ntile - base < g0 ? ntile - base : g0;
  const long long r = tile - grp * g0 * L1;
  l1 = r / gw;
  tx = base + (r - l1 * gw);
}

// Twiddles of passes >= 1 held in registers.  In a persistent kernel a thread's butterflies are
// the same in every tile, so the table is read once per CTA instead of once per tile per pass
// (r02 ncu: the M = 128 z kernel's top stall was long_scoreboard on these loads).
struct TwNone {
  static constexpr bool kHoisted = false;
};
template <typename C, int N, int MAXR> struct TwHoist {
  static constexpr bool kHoisted = true;
  static constexpr Sched S = make_sched(N, MAXR);
  static constexpr int nb(int p) { return (N / S.rad[p] + S.T - 1) / S.T; }
  static constexpr int off(int p) {
    int o = 0;
    for (int q = 1; q < p; ++q) o += nb(q) * (S.rad[q] - 1);
    return o;
  }
  static constexpr int K = off(S.npass);
  C w[K > 0 ? K : 1];
  template <int P> __device__ __forceinline__ void fill(const C* __restrict__ tw, int j) {
    if constexpr (P < S.npass) {
      constexpr int R = S.rad[P], NR = N / R, Ns = sched_ns(S, P);
#pragma unroll
      for (int u = 0; u < nb(P); ++u) {
        const int b = j + S.T * u;
        const int m = (b < NR ? b : 0) % Ns;
#pragma unroll
        for (int r = 1; r < R; ++r) w[off(P) + u * (R - 1) + r - 1] = __ldg(tw + sched_twoff(S, P) + (r - 1) * Ns + m);
      }
      fill<P + 1>(tw, j);
    }
  }
  template <int P> __device__ __forceinline__ C get(int u, int r) const { return w[off(P) + u * (S.rad[P] - 1) + r - 1]; }
};

// --------------------------------------------------------------------------------- Stockham core
// One thread's part of the passes of one line.  IO supplies the global side:
//   C load(int t)  and  void store(int t, C v); SM maps t to a shared-memory slot.
template <typename C, int N, int DIR, int P, int MAXR = 16, class IO, class SM, class TWR = TwNone>
__device__ __forceinline__ void stockham_pass(IO& io, const SM& sm, C* smem, const C* __restrict__ tw, int j,
                                              bool active, const TWR& twr = TWR{}) {
  constexpr Sched S = make_sched(N, MAXR);
  constexpr int R = S.rad[P];
  constexpr int NR = N / R;
  constexpr int Ns = sched_ns(S, P);
  constexpr int NB = (NR + S.T - 1) / S.T;
  constexpr bool EXACT = (NR % S.T) == 0;
  constexpr bool LAST = (P == S.npass - 1);
  C v[NB][R];
  // ---- gather inputs
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    const int b = j + S.T * u;
    if (EXACT || b < NR) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (P == 0) {
          v[u][r] = active ? io.load(b + r * NR) : C{0, 0};
        } else {
          v[u][r] = smem[sm(b + r * NR)];
        }
      }
    }
  }
  // every read of this pass is done before anything is overwritten (also makes a single-pass
  // transform safe in place)
  // (IO::kLastBar = false: the last pass's outputs go to a buffer no thread is reading)
  if constexpr ((P > 0 && (!LAST || IO::kLastBar)) || (P == 0 && LAST) || IO::kSyncAfterLoad) io.bar();
  if constexpr (P == 0 && (IO::kSyncAfterLoad || IO::kRefillNoSync)) io.after_load();  // e.g. refill a TMA stage
  // ---- twiddle, butterfly, scatter
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    const int b = j + S.T * u;
    if (EXACT || b < NR) {
      const int m = b % Ns;
      if constexpr (P > 0 && TWR::kHoisted) {
#pragma unroll
        for (int r = 1; r < R; ++r) v[u][r] = cmul(v[u][r], twr.template get<P>(u, r));
      } else if constexpr (P > 0) {
        const C* twp = tw + sched_twoff(S, P);
#pragma unroll
        for (int r = 1; r < R; ++r) v[u][r] = cmul(v[u][r], __ldg(twp + (r - 1) * Ns + m));
      }
      dft<DIR, R>(v[u]);
      const int d = (b / Ns) * Ns * R + m;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (LAST) {
          if (active) io.store(d + r * Ns, v[u][r]);
        } else {
          smem[sm(d + r * Ns)] = v[u][r];
        }
      }
    }
  }
  if constexpr (!LAST) {
    io.bar();
    stockham_pass<C, N, DIR, P + 1, MAXR>(io, sm, smem, tw, j, active, twr);
  }
}

// ------------------------------------------------------------------ contiguous-axis family
// Global side of a pass for one line (l0, l1): loads of the first pass, stores of the last.
// UNIT_T: unsegmented sides have t-stride 1 (the contig family; the host guarantees it).
// SPEC / TB are compile-time features (runtime branches on them cost 8-30 % in the r01
// same-box A/B: the stores / loads of every other plan paid for them)
template <typename C, bool UNIT_T = false, bool SPEC = false, bool TB = false> struct GIO {
  static constexpr bool kSyncAfterLoad = false;
  static constexpr bool kRefillNoSync = false;
  static constexpr bool kLastBar = true;
  __device__ __forceinline__ void after_load() {}
  __device__ __forceinline__ void bar() const { __syncthreads(); }  // barrier among the threads of a tile
  const C* __restrict__ in;
  C* __restrict__ out;
  const SideMap* mi;
  const SideMap* mo;
  long long i0, i1, o0, o1;  // effective (l0, l1) per side
  long long lin, lout;       // unsegmented sides: l0·s0 + l1·s1
  decltype(C{}.x) scale;
  using R = decltype(C{}.x);
  const R* spt = nullptr;  // spectral multiplier (PassArgs::spec): λ table along t, and λ0[l0] + λ1[l1]
  R lam01 = 0;
  __device__ __forceinline__ void spectral(const PassArgs& a, long long l0_, long long l1_) {
    if (!SPEC || a.spec[0] == nullptr) return;
    spt = reinterpret_cast<const R*>(a.spec[0]);
    lam01 = __ldg(reinterpret_cast<const R*>(a.spec[1]) + l0_) + __ldg(reinterpret_cast<const R*>(a.spec[2]) + l1_);
  }
  __device__ __forceinline__ C apply_spec(int t, C v) const {
    if constexpr (SPEC) {
      const R lam = __ldg(spt + t) + lam01;
      const R g = lam != R(0) ? R(1) / lam : R(0);
      v.x *= g;
      v.y *= g;
    }
    return v;
  }
  __device__ __forceinline__ void init(const SideMap& i, const SideMap& o, long long l0_, long long l1_, double sc) {
    in = reinterpret_cast<const C*>(i.base);
    out = reinterpret_cast<C*>(o.base);
    mi = &i;
    mo = &o;
    side_lines(i, l0_, l1_, i0, i1);
    side_lines(o, l0_, l1_, o0, o1);
    lin = i0 * i.s0 + i1 * i.s1;
    lout = o0 * o.s0 + o1 * o.s1;
    scale = (decltype(C{}.x))sc;
  }
  __device__ __forceinline__ C load(int t) const {
    if (mi->ttab == nullptr) {
      if constexpr (TB) return in[lin + (long long)(t / mi->tb) * mi->tbs + t % mi->tb];
      return UNIT_T ? in[lin + t] : in[(long long)t * mi->tstride + lin];
    }
    return *seg_ptr<const C>(*mi, t, i0, i1);
  }
  // R2R lines are real: real element r of a line is component r&1 of complex element r>>1
  __device__ __forceinline__ R load_real(int r) const {
    const int t = r >> 1;
    const C* p = mi->ttab == nullptr ? in + (UNIT_T ? lin + t : (long long)t * mi->tstride + lin)
                                     : seg_ptr<const C>(*mi, t, i0, i1);
    return reinterpret_cast<const R*>(p)[r & 1];
  }
  __device__ __forceinline__ void store_real(int r, R v) const {
    const int t = r >> 1;
    C* p = mo->ttab == nullptr ? out + (UNIT_T ? lout + t : (long long)t * mo->tstride + lout) : seg_ptr<C>(*mo, t, o0, o1);
    reinterpret_cast<R*>(p)[r & 1] = v * scale;
  }
  __device__ __forceinline__ void store(int t, C v) const {
    if (scale != 1) { v.x *= scale; v.y *= scale; }
    v = apply_spec(t, v);
    if (mo->ttab == nullptr) st_out(out + (UNIT_T ? lout + t : (long long)t * mo->tstride + lout), v);
    else st_out(seg_ptr<C>(*mo, t, o0, o1), v);
  }
};

// shared-memory slot of element t of a line: one pad slot per 2^SH elements
template <int SH> struct PadSM {
  int base;
  __device__ __forceinline__ int operator()(int t) const { return base + t + (t >> SH); }
};

#ifndef DFFT_CONTIG_MAXR32
#define DFFT_CONTIG_MAXR32 1
#endif
template <int N, int ES, bool R32 = true> struct ContigCfg {
  // fp32 lines of >= 512 points: radix-32 passes (1024 = 32·32), as the xz8 and TMA kernels
  // (R32 = false: the radix-16 variant, for x-FFTs that store into peers' windows)
  static constexpr int MAXR = (R32 && DFFT_CONTIG_MAXR32 && ES == 8 && N >= 512 && N % 32 == 0) ? 32 : 16;
  static constexpr Sched S = make_sched(N, MAXR);
  static constexpr int SH = MAXR == 32 ? 5 : 4;  // one pad slot per 2^SH elements (see XZ8Cfg)
  static constexpr int LPC = S.T >= 256 ? 1 : 256 / S.T;  // lines per CTA
  static constexpr int THREADS = S.T * LPC;
  static constexpr int LS = N + (N >> SH);  // padded line stride in smem
  // resident CTAs the register budget allows: 64 registers a thread (f32, radix 16: what ptxas used
  // unbounded) or 128 (f64, radix 32).  A bare minBlocks = 1 lets ptxas take up to 255 and halves
  // the occupancy (r02: cfg5's f64 x-stages 0.97 -> 1.29 ms, 1.42 -> 2.26 ms)
  static constexpr int BUDGET = (ES == 16 || MAXR == 32) ? 128 : 64;
  static constexpr int MINB_RAW = 65536 / (THREADS * BUDGET);
  static constexpr int MINB = MINB_RAW < 1 ? 1 : MINB_RAW > 4 ? 4 : MINB_RAW;
};

// R2C / C2R (reading R8; "exploiting Hermitian symmetry"): a real line of nx = 2N samples
// is FFT'd as N complex points z[m] = x[2m] + i·x[2m+1].
//   R2C (MODE 1): Z = DFT_N(z) goes to shared memory; then for k = 0..N
//       E = (Z[k] + conj Z[N-k]) / 2,  O = (Z[k] - conj Z[N-k]) / (2i),  X[k] = E + w^k O,
//       w = exp(-2πi/nx), Z[N] ≡ Z[0]; the N+1 bins go out through the side map.
//   C2R (MODE 2): the first pass loads Z[t] = E + i·O with E = (X[t] + conj X[N-t]) / 2,
//       O = (X[t] - conj X[N-t])·w^{-t} / 2 (Im X[0] and Im X[N] dropped), and the inverse N-point
//       FFT yields N·(x[2m] + i·x[2m+1]); the host folds 2/(nx·ny·nz) into `scale`.
template <typename C> struct SmemZ : GIO<C, true> {  // R2C: the last pass stores Z to shared memory
  C* zb;
  __device__ __forceinline__ void store(int t, C v) const { zb[t] = v; }
};
template <typename C, int N> struct C2RIO : GIO<C, true> {
  const C* tw2;
  __device__ __forceinline__ C load(int t) const {
    C xt = GIO<C, true>::load(t), xn = GIO<C, true>::load(N - t);
    if (t == 0) {
      xt.y = 0;
      xn.y = 0;
    }
    const C w = __ldg(tw2 + t);  // exp(+2πi t / 2N)
    const C e = {(xt.x + xn.x) * 0.5f, (xt.y - xn.y) * 0.5f};
    const C d = {(xt.x - xn.x) * 0.5f, (xt.y + xn.y) * 0.5f};
    const C o = cmul(d, w);
    return {e.x - o.y, e.y + o.x};  // E + i·O
  }
};

// R2R (reading R21; DCT-II forward, DCT-III/(2L) inverse along every axis) by Makhoul's
// permutation: a real line x of even length L is reordered v_n = x_{2n}, v_{L-1-n} = x_{2n+1}
// (n < L/2), V = DFT_L(v), and X_k = 2·Re(c_k V_k), c_k = exp(-iπk/(2L)).  The inverse builds
// V_k = ½·conj(c_k)·(X_k − i·X_{L−k}) (X_L = 0), v = IDFT_L(V), x_{perm(n)} = v_n.
__host__ __device__ constexpr int dct_perm(int n, int L) { return n < L / 2 ? 2 * n : 2 * (L - 1 - n) + 1; }

// x lines (contig, MODE 3/4): L = 2N reals per line; the N-point complex FFT runs on the packed
// z_m = v_{2m} + i·v_{2m+1} (the R2C trick), so V comes from the R2C split / goes in through the
// C2R merge.  MODE 3 loads the permuted reals; MODE 4 loads X and builds the merged spectrum.
// The line is staged through shared memory in its natural order (coalesced 16 B accesses on the
// global side); the permutation and the X_k / X_{L-k} pairing then read shared memory.
// The inverse stages its line through shared memory with coalesced 16 B global accesses and does
// Makhoul's permutation on the shared-memory side with unit-stride (conflict-free) indices:
// complex element q of the line holds (x_{2q}, x_{2q+1}) = (v_q, v_{L-1-q}).
// (the forward reads its permuted reals straight from global memory: staging its line the same
// way measured slower, 1.58 vs 2.36 ms at 768x768x384 f64; the inverse gains, 2.07 -> 1.98 ms)
// DST (reading R22) by the identities  DST-II(x)_k = DCT-II(x')_{L-1-k},  x'_n = (-1)^n x_n,  and
// DST-III(X)_n = (-1)^n DCT-III(X')_n,  X'_k = X_{L-1-k}:  sign-flipped loads and a reversed
// output (forward), reversed loads and sign-flipped outputs (inverse).
template <bool DST, typename R> __device__ __forceinline__ R alt_sign(int n, R v) { return (DST && (n & 1)) ? -v : v; }

template <typename C, int N, bool DST = false> struct DctXFwdIO : GIO<C, true> {
  C* zb;  // the last pass's outputs
  __device__ __forceinline__ C load(int t) const {
    const int p0 = dct_perm(2 * t, 2 * N), p1 = dct_perm(2 * t + 1, 2 * N);
    return {alt_sign<DST>(p0, this->load_real(p0)), alt_sign<DST>(p1, this->load_real(p1))};
  }
  __device__ __forceinline__ void store(int t, C v) const { zb[t] = v; }
};
template <typename C, int N, bool DST = false> struct DctXInvIO : GIO<C, true> {
  using R = decltype(C{}.x);
  static constexpr bool kSyncAfterLoad = true;
  const C* tw2;  // exp(+2πi t / 2N)
  const C* tw3;  // exp(+iπk / (4N)), k < 2N
  const R* xr;   // the staged input line (2N reals)
  C* zb;         // the last pass's outputs z_t = (v_{2t}, v_{2t+1}) (times N)
  __device__ __forceinline__ C vk(int k) const {  // V_k = ½·conj(c_k)·(X_k − i·X_{L−k}), k ≤ N
    // (DST: X'_k = X_{L-1-k})
    const R xk = DST ? (k == 2 * N ? R(0) : xr[2 * N - 1 - k]) : xr[k];
    const R xl = k == 0 ? R(0) : DST ? xr[k - 1] : xr[2 * N - k];
    const C c = __ldg(tw3 + k);
    const C d = {xk * R(0.5), -xl * R(0.5)};
    return cmul(c, d);
  }
  __device__ __forceinline__ C load(int t) const {
    const C xt = vk(t), xn = vk(N - t);
    const C w = __ldg(tw2 + t);
    const C e = {(xt.x + xn.x) * R(0.5), (xt.y - xn.y) * R(0.5)};
    const C d = {(xt.x - xn.x) * R(0.5), (xt.y + xn.y) * R(0.5)};
    const C o = cmul(d, w);
    return {e.x - o.y, e.y + o.x};  // E + i·O  (IDFT_N of it = v_{2m} + i·v_{2m+1}, times N)
  }
  __device__ __forceinline__ void store(int t, C v) const { zb[t] = v; }
};

// MODE 0 c2c, 1 R2C, 2 C2R, 3 / 4 DCT-II / DCT-III of real x-lines, 5 / 6 DST-II / DST-III
template <typename Real, int N, int DIR, int MODE, bool TB = false, bool R32 = true>
__global__ void __launch_bounds__(ContigCfg<N, 2 * sizeof(Real), R32>::THREADS, ContigCfg<N, 2 * sizeof(Real), R32>::MINB)
fft_contig_kernel(const __grid_constant__ PassArgs a) {
  using C = typename CT<Real>::type;
  using Cfg = ContigCfg<N, 2 * sizeof(Real), R32>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  C* smem = reinterpret_cast<C*>(smem_raw);
  const int li = threadIdx.x / Cfg::S.T;
  const int j = threadIdx.x % Cfg::S.T;
  const long long line = (long long)blockIdx.x * Cfg::LPC + li;
  const bool active = line < a.L0 * a.L1;
  long long l0 = 0, l1 = 0;
  if (active) {
    if (a.lorder) {
      l0 = line / a.L1;
      l1 = line - l0 * a.L1;
    } else {
      l1 = line / a.L0;
      l0 = line - l1 * a.L0;
    }
  }
  PadSM<Cfg::SH> sm{li * Cfg::LS};
  const C* tw = reinterpret_cast<const C*>(a.tw);
  if constexpr (MODE == 0) {
    GIO<C, true, false, TB> io;
    io.init(a.in, a.out, l0, l1, a.scale);
    stockham_pass<C, N, DIR, 0, Cfg::MAXR>(io, sm, smem, tw, j, active);
  } else if constexpr (MODE == 1) {
    SmemZ<C> io;
    io.init(a.in, a.out, l0, l1, a.scale);
    C* zb = smem + li * Cfg::LS;
    io.zb = zb;
    stockham_pass<C, N, DIR, 0, Cfg::MAXR>(io, sm, smem, tw, j, active);
    __syncthreads();
    if (active) {
      const C* tw2 = reinterpret_cast<const C*>(a.tw2);
      for (int k = j; k <= N; k += Cfg::S.T) {
        const C zk = zb[k == N ? 0 : k], zn = zb[k == 0 ? 0 : N - k];
        const C e = {(zk.x + zn.x) * 0.5f, (zk.y - zn.y) * 0.5f};
        const C o = {(zk.y + zn.y) * 0.5f, (zn.x - zk.x) * 0.5f};  // (Z[k] - conj Z[N-k]) / 2i
        C w;
        if (k == N) w = {-1, 0};
        else w = __ldg(tw2 + k);
        io.GIO<C, true>::store(k, cadd(e, cmul(w, o)));
      }
    }
  } else if constexpr (MODE == 2) {
    C2RIO<C, N> io;
    io.init(a.in, a.out, l0, l1, a.scale);
    io.tw2 = reinterpret_cast<const C*>(a.tw2);
    stockham_pass<C, N, DIR, 0, Cfg::MAXR>(io, sm, smem, tw, j, active);
  } else if constexpr (MODE == 3 || MODE == 5) {  // forward DCT-II / DST-II of real x-lines of length 2N
    using R = Real;
    constexpr bool DST = MODE == 5;
    DctXFwdIO<C, N, DST> io;
    io.init(a.in, a.out, l0, l1, a.scale);
    C* zb = smem + li * Cfg::LS;
    io.zb = zb;
    stockham_pass<C, N, DIR, 0, Cfg::MAXR>(io, sm, smem, tw, j, active);
    __syncthreads();
    if (active) {
      const C* tw2 = reinterpret_cast<const C*>(a.tw2);  // exp(-2πi k / 2N)
      const C* tw3 = reinterpret_cast<const C*>(a.tw3);  // exp(-iπk / (4N)), k < 2N
      for (int k = j; k <= N; k += Cfg::S.T) {
        const C zk = zb[k == N ? 0 : k], zn = zb[k == 0 ? 0 : N - k];
        const C e = {(zk.x + zn.x) * R(0.5), (zk.y - zn.y) * R(0.5)};
        const C o = {(zk.y + zn.y) * R(0.5), (zn.x - zk.x) * R(0.5)};
        const C w = k == N ? C{-1, 0} : __ldg(tw2 + k);
        const C v = cadd(e, cmul(w, o));  // V_k of the real permuted line, k <= N
        const C ck = __ldg(tw3 + k);
        // X_k = 2 Re(c_k V_k)  (DST: stored at 2N-1-k)
        io.store_real(DST ? 2 * N - 1 - k : k, R(2) * (ck.x * v.x - ck.y * v.y));
        if (k > 0 && k < N) {  // X_{2N-k} = 2 Re(c_{2N-k} conj V_k)  (DST: at k-1)
          const C cl = __ldg(tw3 + 2 * N - k);
          io.store_real(DST ? k - 1 : 2 * N - k, R(2) * (cl.x * v.x + cl.y * v.y));
        }
      }
    }
  } else {  // MODE 4 / 6: inverse DCT-III / DST-III of real x-lines of length 2N (scale by the host)
    using R = Real;
    constexpr bool DST = MODE == 6;
    DctXInvIO<C, N, DST> io;
    io.init(a.in, a.out, l0, l1, a.scale);
    io.tw2 = reinterpret_cast<const C*>(a.tw2);
    io.tw3 = reinterpret_cast<const C*>(a.tw3);
    C* zb = smem + li * Cfg::LS;
    io.xr = reinterpret_cast<const R*>(zb);
    io.zb = zb;
    if (active)
      for (int t = j; t < N; t += Cfg::S.T) zb[t] = io.GIO<C, true>::load(t);
    __syncthreads();
    stockham_pass<C, N, DIR, 0, Cfg::MAXR>(io, sm, smem, tw, j, active);
    __syncthreads();
    if (active) {  // output element q = (x_{2q}, x_{2q+1}) = (v_q, v_{2N-1-q}); coalesced stores
      const R* vr = reinterpret_cast<const R*>(zb);
      for (int q = j; q < N; q += Cfg::S.T)
        io.GIO<C, true>::store(q, C{vr[q], DST ? -vr[2 * N - 1 - q] : vr[2 * N - 1 - q]});
    }
  }
}

// ------------------------------------------------------------------ x-FFT fused with a radix-8 z step
// The z axis of length Nz = 8·M is split by one Cooley-Tukey step (z = z1 + M·k, K = 8·m + q):
//   X[8m + q] = Σ_{z1} w_M^{z1·m} · Y_q[z1],    Y_q[z1] = w_Nz^{z1·q} · Σ_{k<8} x[z1 + M·k] · w_8^{k·q}
// Forward (DIR -1): a CTA takes the 8 x-lines (y, z1 + M·k), runs their x-FFT, then the radix-8 step
// across the lines and the twiddle, and writes Y_q as line q of the intermediate.  The remaining
// M-point z-FFTs run as a strided stage whose tiles are only M rows deep, so they are 256-512 B wide
// — the row width the DRAM wants at any pitch.  Inverse (DIR +1): the mirror — the 8
// lines q in, conjugate twiddle, inverse radix-8 step, then the x-IFFT of each line k.
// Line addressing (complex elements): line (l0, l1, r) starts at base + l0·s0 + l1·s1 + r·tstride,
// r = k or q; the t stride along a line is 1.
#ifndef DFFT_XZ8_MAXR32
#define DFFT_XZ8_MAXR32 1
#endif
template <int N, int ES> struct XZ8Cfg {
  // fp32 lines of >= 512 points: radix-32 passes (1024 = 32·32, two passes), as the TMA kernels
  static constexpr int MAXR = (DFFT_XZ8_MAXR32 && ES == 8 && N >= 512 && N % 32 == 0) ? 32 : 16;
  static constexpr Sched S = make_sched(N, MAXR);
  // one pad slot per 2^SH elements: the first pass scatters to b·MAXR + r, conflict-free per half-warp
  static constexpr int SH = MAXR == 32 ? 5 : 4;
  static constexpr int T = S.T, THREADS = 8 * T, LS = N + (N >> SH);
  static constexpr bool OK = THREADS <= 1024 && THREADS >= 64;
  // 8 padded lines in shared memory; minimum resident CTAs for __launch_bounds__: 2 where two
  // fit by shared memory and still leave 64 (f32, radix 16) / 128 (f64 or radix 32) registers a
  // thread — the budgets the butterflies compile in without spills — else 1
  static constexpr int SMEM = 8 * LS * ES;
  static constexpr bool FITS = SMEM <= 227 * 1024;
  static constexpr int MINB =
      2 * (SMEM + 1024) <= 228 * 1024 && 2 * THREADS * (ES == 16 || MAXR == 32 ? 128 : 64) <= 65536 ? 2 : 1;
};
template <typename C, int N, int DIR, int SH> struct XZ8IO : GIO<C, true> {
  static constexpr bool kSyncAfterLoad = DIR > 0;  // inverse: pass 0 reads the line from smem in place
  const C* src;  // forward: this line in global memory; inverse: unused (smem)
  C* dst;        // inverse: this line in global memory
  C* line;       // this line in shared memory, PadSM positions (base applied)
  __device__ __forceinline__ C load(int t) const {
    if constexpr (DIR < 0) return src[t];
    else return line[t + (t >> SH)];
  }
  __device__ __forceinline__ void store(int t, C v) const {
    if constexpr (DIR < 0) {
      line[t + (t >> SH)] = v;
    } else {
      if (this->scale != 1) {
        v.x *= this->scale;
        v.y *= this->scale;
      }
      dst[t] = v;
    }
  }
};

template <typename Real, int N, int DIR>
__global__ void __launch_bounds__(XZ8Cfg<N, 2 * sizeof(Real)>::THREADS, XZ8Cfg<N, 2 * sizeof(Real)>::MINB)
    fft_xz8_kernel(const __grid_constant__ PassArgs a) {
  using C = typename CT<Real>::type;
  using Cfg = XZ8Cfg<N, 2 * sizeof(Real)>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  C* smem = reinterpret_cast<C*>(smem_raw);
  const int li = threadIdx.x / Cfg::T, j = threadIdx.x % Cfg::T;
  const long long l1 = blockIdx.x / a.L0, l0 = blockIdx.x - l1 * a.L0;
  const C* in = reinterpret_cast<const C*>(a.in.base) + l0 * a.in.s0 + l1 * a.in.s1;
  C* out = reinterpret_cast<C*>(a.out.base) + l0 * a.out.s0 + l1 * a.out.s1;
  const C* tw = reinterpret_cast<const C*>(a.tw);
  const C* tw2 = reinterpret_cast<const C*>(a.tw2);  // w_Nz^e, e < Nz (sign DIR)
  C* line = smem + li * Cfg::LS;
  XZ8IO<C, N, DIR, Cfg::SH> io;
  io.scale = (Real)a.scale;
  io.line = line;
  PadSM<Cfg::SH> sm{li * Cfg::LS};
  if constexpr (DIR < 0) {
    io.src = in + li * a.in.tstride;  // x-line k = li
    stockham_pass<C, N, DIR, 0, Cfg::MAXR>(io, sm, smem, tw, j, true);
    __syncthreads();
    for (int t = threadIdx.x; t < N; t += Cfg::THREADS) {  // radix-8 step across the 8 lines
      C v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = smem[k * Cfg::LS + t + (t >> Cfg::SH)];
      dft<DIR, 8>(v);
      out[t] = v[0];
#pragma unroll
      for (int q = 1; q < 8; ++q) out[q * a.out.tstride + t] = cmul(v[q], __ldg(tw2 + l1 * q));
    }
  } else {
    // the 8 lines q at column t straight from global memory (8 loads in flight per column),
    // conjugate twiddle, inverse radix-8 step, lines k into shared memory
    constexpr int IT = (N + Cfg::THREADS - 1) / Cfg::THREADS;
    C v[IT][8];
#pragma unroll
    for (int it = 0; it < IT; ++it) {  // every load of the thread in flight at once
      const int t = threadIdx.x + it * Cfg::THREADS;
      if (t < N) {
#pragma unroll
        for (int q = 0; q < 8; ++q) v[it][q] = in[q * a.in.tstride + t];
      }
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int t = threadIdx.x + it * Cfg::THREADS;
      if (t < N) {
#pragma unroll
        for (int q = 1; q < 8; ++q) v[it][q] = cmul(v[it][q], __ldg(tw2 + l1 * q));
        dft<DIR, 8>(v[it]);
#pragma unroll
        for (int k = 0; k < 8; ++k) smem[k * Cfg::LS + t + (t >> Cfg::SH)] = v[it][k];
      }
    }
    __syncthreads();
    io.dst = out + li * a.out.tstride;  // x-line k = li
    stockham_pass<C, N, DIR, 0, Cfg::MAXR>(io, sm, smem, tw, j, true);
  }
}

// ------------------------------------------------------------------ strided-axis family
template <typename Real, int N> struct StridedCfg {
  static constexpr Sched S = make_sched(N);
  static constexpr int ES = (int)sizeof(Real) * 2;
  // W adjacent columns per CTA: 64-128 B row segments, at least 256 threads for short
  // lines, smem tile capped at 96 KB.
#ifndef DFFT_STRIDED_W0
#define DFFT_STRIDED_W0 64
#endif
  static constexpr int W0 = DFFT_STRIDED_W0 / ES;  // row segment bytes / element size
  // whole 32 B sectors per row (see TmaCfg: partial-sector stores cost a DRAM read each)
  static constexpr int Wthr = S.T * W0 >= 256 ? W0 : (256 / S.T + 32 / ES - 1) / (32 / ES) * (32 / ES);
  static constexpr int Wcap = (96 * 1024) / (N * ES) >= 1 ? (96 * 1024) / (N * ES) : 1;
  static constexpr int W = Wthr < Wcap ? Wthr : (Wcap >= 8 ? 8 : Wcap >= 4 ? 4 : Wcap >= 2 ? 2 : 1);
  static constexpr int THREADS = S.T * W;
  // pad W slots per R0 rows when a row is narrower than 128 B: 64-bit shared accesses resolve
  // conflicts per half-warp, so rows b and b+1 must land 64 B apart mod 128 (tools/bank_sim.py)
  static constexpr int PAD = (W * ES < 128) ? W : 0;
  static constexpr int R0 = S.rad[0];
  static constexpr int SMEM_ELEMS = N * W + (N / R0) * PAD;
};

template <int W, int R0, int PAD> struct StridedSM {
  int c;
  __device__ __forceinline__ int operator()(int t) const { return t * W + c + (t / R0) * PAD; }
};

template <typename Real, int N, int DIR, bool SPEC = false>
__global__ void __launch_bounds__(StridedCfg<Real, N>::THREADS)
fft_strided_kernel(const __grid_constant__ PassArgs a) {
  using C = typename CT<Real>::type;
  using Cfg = StridedCfg<Real, N>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  C* smem = reinterpret_cast<C*>(smem_raw);
  const int c = threadIdx.x % Cfg::W;
  const int j = threadIdx.x / Cfg::W;
  const long long ntile = (a.L0 + Cfg::W - 1) / Cfg::W;
  const long long l1 = blockIdx.x / ntile;
  const long long l0 = (blockIdx.x - l1 * ntile) * Cfg::W + c;
  const bool active = l0 < a.L0;
  GIO<C, false, SPEC> io;
  io.init(a.in, a.out, active ? l0 : 0, l1, a.scale);
  io.spectral(a, active ? l0 : 0, l1);
  StridedSM<Cfg::W, Cfg::R0, Cfg::PAD> sm{c};
  stockham_pass<C, N, DIR, 0>(io, sm, smem, reinterpret_cast<const C*>(a.tw), j, active);
}

// Strided R2R stage (y or z DCT, reading R21): the real array is viewed as complex pairs of
// adjacent x columns, so one complex column holds two real columns a (re) and b (im) and one
// N-point complex FFT serves both.  Forward: z_t = column[perm(t)], Z = DFT_N(z),
//   Va_k = (Z_k + conj Z_{N−k})/2, Vb_k = (Z_k − conj Z_{N−k})/(2i),
//   X_k = (2 Re(c_k Va_k), 2 Re(c_k Vb_k))  — the last pass goes to shared memory and each thread
// finishes the pairs (k, N−k).  Inverse: Z_t = Va_t + i·Vb_t with V from rows t and N−t, z =
// IDFT_N(Z) (unnormalised; the host folds 1/N), row perm(t) = z_t.
template <typename C, int N, int DIR, bool DST = false> struct DctStridedIO : GIO<C> {
  using R = decltype(C{}.x);
  const C* tw3;  // c_k = exp(DIR·iπk/(2N)), k < N
  C* tile;       // forward: the last pass's outputs, dense [t][W] at column c
  int W, c;
  __device__ __forceinline__ C load(int t) const {
    if constexpr (DIR < 0) {
      const int p = dct_perm(t, N);
      const C v = GIO<C>::load(p);
      return (DST && (p & 1)) ? C{-v.x, -v.y} : v;
    } else {
      const C xt = GIO<C>::load(DST ? N - 1 - t : t);
      const C xl = t == 0 ? C{0, 0} : GIO<C>::load(DST ? t - 1 : N - t);
      const C cc = __ldg(tw3 + t);  // conj(c_t) for the inverse table
      const C da = {xt.x * R(0.5), -xl.x * R(0.5)}, db = {xt.y * R(0.5), -xl.y * R(0.5)};
      const C va = cmul(cc, da), vb = cmul(cc, db);
      return {va.x - vb.y, va.y + vb.x};  // Va + i·Vb
    }
  }
  __device__ __forceinline__ void store(int t, C v) const {
    if constexpr (DIR < 0) {
      tile[t * W + c] = v;
    } else {
      const int p = dct_perm(t, N);
      GIO<C>::store(p, (DST && (p & 1)) ? C{-v.x, -v.y} : v);
    }
  }
};

// multiplier 1/λ of the Poisson solve on a DCT / DST output row (runtime: those stages only)
template <typename C> __device__ __forceinline__ C dct_spec(const PassArgs& a, int row, long long l0, long long l1, C v) {
  using R = decltype(C{}.x);
  if (a.spec[0] == nullptr) return v;
  const R* lx = reinterpret_cast<const R*>(a.spec[1]);
  const R base = __ldg(reinterpret_cast<const R*>(a.spec[0]) + row) + __ldg(reinterpret_cast<const R*>(a.spec[2]) + l1);
  const R lre = base + __ldg(lx + (a.spec_pairs ? 2 * l0 : l0));
  const R lim = base + __ldg(lx + (a.spec_pairs ? 2 * l0 + 1 : l0));
  return {lre != R(0) ? v.x / lre : R(0), lim != R(0) ? v.y / lim : R(0)};
}

template <typename Real, int N, int DIR, bool DST = false>
__global__ void __launch_bounds__(StridedCfg<Real, N>::THREADS)
fft_strided_dct_kernel(const __grid_constant__ PassArgs a) {
  using C = typename CT<Real>::type;
  using R = Real;
  using Cfg = StridedCfg<Real, N>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  C* smem = reinterpret_cast<C*>(smem_raw);
  C* tile = smem;  // dense [t][W] (forward): aliases the pass buffer (the last pass reads it first)
  const int c = threadIdx.x % Cfg::W;
  const int j = threadIdx.x / Cfg::W;
  const long long ntile = (a.L0 + Cfg::W - 1) / Cfg::W;
  const long long l1 = blockIdx.x / ntile;
  const long long l0 = (blockIdx.x - l1 * ntile) * Cfg::W + c;
  const bool active = l0 < a.L0;
  DctStridedIO<C, N, DIR, DST> io;
  io.init(a.in, a.out, active ? l0 : 0, l1, a.scale);
  io.tw3 = reinterpret_cast<const C*>(a.tw3);
  io.tile = tile;
  io.W = Cfg::W;
  io.c = c;
  StridedSM<Cfg::W, Cfg::R0, Cfg::PAD> sm{c};
  stockham_pass<C, N, DIR, 0>(io, sm, smem, reinterpret_cast<const C*>(a.tw), j, active);
  if constexpr (DIR < 0) {
    __syncthreads();
    if (active) {
      const C* tw3 = reinterpret_cast<const C*>(a.tw3);
      for (int k = j; k <= N / 2; k += Cfg::S.T) {
        const C zk = tile[k * Cfg::W + c], zn = tile[(k == 0 ? 0 : N - k) * Cfg::W + c];
        // s = Z_k + conj Z_{N-k} (= 2 Va_k),  d = Z_k − conj Z_{N-k} (= 2i Vb_k)
        const C sk = {zk.x + zn.x, zk.y - zn.y}, dk = {zk.x - zn.x, zk.y + zn.y};
        const C ck = __ldg(tw3 + k);
        // X^a_k = Re(c_k s), X^b_k = Re(c_k d / i) = Im(c_k d)   (DST: row N-1-k)
        const int rk = DST ? N - 1 - k : k;
        io.GIO<C>::store(rk, dct_spec(a, rk, l0, l1, C{ck.x * sk.x - ck.y * sk.y, ck.x * dk.y + ck.y * dk.x}));
        if (k > 0 && 2 * k != N) {  // the partner row N−k: s' = conj s, d' = −conj d   (DST: row k-1)
          const C cl = __ldg(tw3 + N - k);
          const C sl = {sk.x, -sk.y}, dl = {-dk.x, dk.y};
          const int rl = DST ? k - 1 : N - k;
          io.GIO<C>::store(rl, dct_spec(a, rl, l0, l1, C{cl.x * sl.x - cl.y * sl.y, cl.x * dl.y + cl.y * dl.x}));
        }
      }
    }
  }
}

// ------------------------------------------------------------------ strided family, TMA-staged
// Persistent CTAs; each tile (W columns × N rows) is brought into shared memory by TMA
// (cp.async.bulk.tensor, 3D box: 2W reals × BOXR rows × 1) into one of NS stages, completion
// tracked by an mbarrier with expect_tx.  Pass 0 reads the stage, the stage is refilled with the
// tile NS steps ahead right after (one elected thread), and the remaining passes run in a padded
// work buffer — HBM reads stay in flight while the CTA computes.  Stores go from registers
// through the SideMap (fused pack) as in the plain strided kernel.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const void* tmap, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
// a tile's box: 3D (reals, row, l1) or, for a column-blocked input, 4D (reals in block, row, l1,
// block) — the host encodes the matching tensor map
__device__ __forceinline__ void tma_load_tile(void* dst, const void* tmap, int bw, int c0, int row, int l1,
                                              uint64_t* bar) {
  if (bw > 0) tma_load_4d(dst, tmap, c0 % (2 * bw), row, l1, c0 / (2 * bw), bar);
  else tma_load_3d(dst, tmap, c0, row, l1, bar);
}
__device__ __forceinline__ void tma_store_3d(const void* tmap, int c0, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tmap), "r"(c0),
               "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const void* tmap, int c0, int c1, int c2, int c3, const void* src) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(tmap),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(src))
               : "memory");
}
// a tile's box on the store side: 3D, or 4D into a column-blocked output (as tma_load_tile)
__device__ __forceinline__ void tma_store_tile(const void* tmap, int bw, int c0, int row, int l1, const void* src) {
  if (bw > 0) tma_store_4d(tmap, c0 % (2 * bw), row, l1, c0 / (2 * bw), src);
  else tma_store_3d(tmap, c0, row, l1, src);
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

constexpr int largest_divisor_le(int n, int cap) {
  for (int d = cap; d >= 1; --d)
    if (n % d == 0) return d;
  return 1;
}

template <typename Real, int N> struct TmaCfg {
  static constexpr int ES = (int)sizeof(Real) * 2;
#ifndef DFFT_TMA_MAXR32
#define DFFT_TMA_MAXR32 1
#endif
  // fp32 lines of >= 512 points use radix-32 passes (1024 = 32·32: two passes, fewer barriers and
  // less shared-memory traffic per tile); fp64 keeps radix 16 (register budget)
  // fp64 lines with a factor 5 (480, 720): radix-8 passes.  A thread holds ceil(rmax/R)·R values of
  // a radix-R pass; at rmax = 16 the radix-3/5 passes of 720 need 18-20 complex doubles and the
  // kernel spilled 1.2 KB a thread (r02 ptxas), at rmax = 8 it needs 9-10.
  static constexpr int MAXR =
      (DFFT_TMA_MAXR32 && ES == 8 && N >= 512 && N % 32 == 0) ? 32 : (ES == 16 && N % 5 == 0) ? 8 : 16;
  static constexpr Sched S = make_sched(N, MAXR);
#ifndef DFFT_TMA_ROWB
#define DFFT_TMA_ROWB 64
#endif
#ifndef DFFT_TMA_MINTHR
#define DFFT_TMA_MINTHR 256
#endif
  static constexpr int W0 = DFFT_TMA_ROWB / ES;  // row segment of a tile (bytes / element size)
  static constexpr int NS = 2;
  static constexpr int R0 = S.rad[0];
  static constexpr size_t smem_for(int w) {
    return (size_t)(NS * N * w + N * w + (N / R0) * (w * ES < 128 ? w : 0)) * ES + NS * 8 + 16;
  }
  // at least DFFT_TMA_MINTHR threads, in whole 32 B sectors per tile row: a row that ends inside a
  // sector (f64 N = 768: 5 columns = 80 B) makes every tile store a partial-sector write, which
  // L2 completes with a DRAM read (r02: the f64 768 strided pass ran at 1.6 TB/s).  Round up to a
  // sector multiple while the tile fits, else down.
  static constexpr int SECT = 32 / ES;
  static constexpr int Wraw = S.T * W0 >= DFFT_TMA_MINTHR ? W0 : DFFT_TMA_MINTHR / S.T;
  static constexpr int Wup = (Wraw + SECT - 1) / SECT * SECT;
  static constexpr int Wdn = Wraw >= SECT ? Wraw / SECT * SECT : Wraw;
  static constexpr int W = (smem_for(Wup) <= 227 * 1024 && 2 * Wup <= 256 && S.T * Wup <= 1024) ? Wup : Wdn;
  static constexpr int THREADS = S.T * W;
  static constexpr int BOXR = largest_divisor_le(N, 256);
  static constexpr int NBOX = N / BOXR;
  static constexpr int PAD = (W * ES < 128) ? W : 0;
  static constexpr int STAGE_ELEMS = N * W;
  static constexpr int WORK_ELEMS = N * W + (N / R0) * PAD;
  static constexpr size_t SMEM = (size_t)(NS * STAGE_ELEMS + WORK_ELEMS) * ES + NS * 8 + 16;
  static constexpr bool OK = S.npass >= 2 && THREADS <= 1024 && SMEM <= 227 * 1024 && 2 * W <= 256;
  // in-place variant (IP): the passes run in the stage buffer itself (pass 0 reads the whole tile
  // before it writes), so the shared memory of the separate work tile buys another stage in flight
  static constexpr int BUF_IP = (WORK_ELEMS * ES + 127) / 128 * 128 / ES;
  static constexpr int NS_IP = 3 * BUF_IP * ES + 64 <= 227 * 1024 ? 3 : 2;
  static constexpr size_t SMEM_IP = (size_t)NS_IP * BUF_IP * ES + NS_IP * 8 + 16;
  // where it measured faster (r02 same-box A/B, tools/ab/tma_inplace_lengths.sh): f32 M = 96 / 192
  // (the xz8 plan's z passes: 1.43 -> 1.07 ms, 1.36 -> 1.26 ms), f64 128 (0.36 -> 0.34 ms); equal
  // or slower elsewhere (the 1024-row y pass 2.96 -> 3.05 ms)
  static constexpr bool IP_PREFER = (ES == 8 && (N == 96 || N == 192)) || (ES == 16 && N == 128);
};

// DCT (R2R strided stages on the TMA kernel, OM 1 only): -1 forward (permuted loads from the
// stage; the (k, N−k) post-processing runs on the output tile before the TMA store), +1 inverse
// (V from stage rows t and N−t in the loads, permuted rows in the stores).
// DCT (R2R strided stages, OM 1 only): 0 = c2c; -1 / +1 = DCT-II / DCT-III; -2 / +2 = DST-II / DST-III
template <typename C, int W, int OM, bool SPEC = false, int N_ = 0, int DCT = 0> struct TmaIO : GIO<C, false, SPEC> {
  static constexpr bool DSTV = DCT == 2 || DCT == -2;
  static constexpr bool kSyncAfterLoad = true;
  static constexpr bool kRefillNoSync = false;
  static constexpr bool kLastBar = true;
  const C* stage;  // this tile's stage buffer, dense [t][W]
  C* obuf;         // OM > 0: dense [t][W] output tile, written by a TMA tensor store (1) or bulk copies (2)
  int c;
  // refill: thread 0 issues the TMA for the tile NS steps ahead into the drained stage
  const void* tmap;
  uint64_t* mbar;
  C* stage_ptr;
  int next_c0, next_l1, nbox, boxr, in_bw;
  uint32_t bytes;
  bool refill;
  const C* tw3 = nullptr;  // DCT: c_k = exp(DCT·iπk/(2N))
  __device__ __forceinline__ C load(int t) const {
    if constexpr (DCT < 0) {
      const int p = dct_perm(t, N_);
      const C v = stage[p * W + c];
      return (DSTV && (p & 1)) ? C{-v.x, -v.y} : v;
    } else if constexpr (DCT > 0) {
      using R = decltype(C{}.x);
      const C xt = stage[(DSTV ? N_ - 1 - t : t) * W + c];
      const C xl = t == 0 ? C{0, 0} : stage[(DSTV ? t - 1 : N_ - t) * W + c];
      const C cc = __ldg(tw3 + t);
      const C da = {xt.x * R(0.5), -xl.x * R(0.5)}, db = {xt.y * R(0.5), -xl.y * R(0.5)};
      const C va = cmul(cc, da), vb = cmul(cc, db);
      return {va.x - vb.y, va.y + vb.x};
    } else {
      return stage[t * W + c];
    }
  }
  __device__ __forceinline__ void store(int t, C v) const {
    if constexpr (OM != 0) {
      if (this->scale != 1) { v.x *= this->scale; v.y *= this->scale; }
      if constexpr (DCT > 0) {
        const int p = dct_perm(t, N_);
        obuf[p * W + c] = (DSTV && (p & 1)) ? C{-v.x, -v.y} : v;
        return;
      }
      obuf[t * W + c] = this->apply_spec(t, v);
    } else {
      GIO<C, false, SPEC>::store(t, v);
    }
  }
  __device__ __forceinline__ void after_load() {
    if (refill && threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(mbar, bytes);
      for (int q = 0; q < nbox; ++q)
        tma_load_tile(stage_ptr + q * boxr * W, tmap, in_bw, next_c0, q * boxr, next_l1, mbar);
    }
  }
};

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}

// OM (output mode): 0 = per-element stores through the SideMap; 1 = the output side is
// unsegmented and written by TMA tensor stores (omap) from the work buffer — issuing 64 B row
// stores at a large stride from the SMs throttles the LSU (r01 ncu: lg_throttle); 2 = the
// output is segmented into column-blocked windows (possibly peers' over NVLink) and each
// segment of a tile leaves as one contiguous cp.async.bulk copy.
template <typename Real, int N, int DIR, int OM, bool SPEC = false, int DCT = 0, bool IP = false>
__global__ void __launch_bounds__(TmaCfg<Real, N>::THREADS)
fft_strided_tma_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap omap,
                       const __grid_constant__ PassArgs a) {
  constexpr bool TST = OM != 0;
  static_assert(!IP || (OM == 1 && DCT == 0), "the in-place variant stores its tile with TMA stores");
  using C = typename CT<Real>::type;
  using Cfg = TmaCfg<Real, N>;
  constexpr int NSK = IP ? Cfg::NS_IP : Cfg::NS;             // stages in flight
  constexpr int BUF = IP ? Cfg::BUF_IP : Cfg::STAGE_ELEMS;    // elements a stage
  // 1024-byte aligned: TMA destinations need 128 B alignment, and a cluster launch does not
  // otherwise guarantee it for the dynamic shared-memory base
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  C* stages = reinterpret_cast<C*>(smem_raw);
  C* work = stages + NSK * BUF;  // (IP: the current stage, set per tile)
  uint64_t* bars = reinterpret_cast<uint64_t*>(IP ? stages + NSK * BUF : work + Cfg::WORK_ELEMS);
  const int c = threadIdx.x % Cfg::W;
  const int j = threadIdx.x / Cfg::W;
  const long long ntile = (a.L0 + Cfg::W - 1) / Cfg::W;
  const long long total = ntile * a.L1;
  constexpr uint32_t kBytes = (uint32_t)(Cfg::STAGE_ELEMS * Cfg::ES);
  // TMA coordinates are in reals: column c -> 2c
  auto issue = [&](long long tile, int s) {
    long long tx, l1;
    tile_coords(tile, ntile, a.L1, a.g0, tx, l1);
    const int c0 = (int)(tx * Cfg::W * 2);
    mbar_expect_tx(&bars[s], kBytes);
    for (int q = 0; q < Cfg::NBOX; ++q)
      tma_load_tile(stages + s * BUF + q * Cfg::BOXR * Cfg::W, &tmap, a.in.bw, c0, q * Cfg::BOXR, (int)l1,
                    &bars[s]);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSK; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NSK; ++s) {
      long long tile = blockIdx.x + (long long)s * gridDim.x;
      if (tile < total) issue(tile, s);
    }
  }
  // twiddles in registers where they take at most 256 B a thread (32 in fp32: the 1024-row y pass
  // has 31, the M = 128 z pass 14; 16 in fp64) and the CTA is at most 256 threads (larger CTAs —
  // 840: 840 threads, 384: 288 — have no register room and spilled)
#ifndef DFFT_TW_HOIST_BYTES
#define DFFT_TW_HOIST_BYTES 256
#endif
  using TH = TwHoist<C, N, Cfg::MAXR>;
  constexpr bool kHoist = TH::K > 0 && TH::K * Cfg::ES <= DFFT_TW_HOIST_BYTES && Cfg::THREADS <= 256;
  TH twh;
  if constexpr (kHoist) twh.template fill<1>(reinterpret_cast<const C*>(a.tw), j);
  __syncthreads();
  int it = 0;
  for (long long tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
    const int s = it % NSK;
    const uint32_t parity = (uint32_t)((it / NSK) & 1);
    if constexpr (IP) work = stages + s * BUF;
    long long tx, l1;
    tile_coords(tile, ntile, a.L1, a.g0, tx, l1);
    const long long l0 = tx * Cfg::W + c;
    const bool active = l0 < a.L0;
    if (TST && !IP && threadIdx.x == 0) bulk_wait_read0();  // previous tile's TMA store has read `work`
    TmaIO<C, Cfg::W, OM, SPEC, N, DCT> io;
    io.tw3 = reinterpret_cast<const C*>(a.tw3);
    io.init(a.in, a.out, active ? l0 : 0, l1, a.scale);
    io.spectral(a, active ? l0 : 0, l1);
    io.stage = stages + s * BUF;
    io.obuf = work;
    io.c = c;
    // refill: the drained stage gets the tile NS steps ahead
    const int rs = s;
    const long long next = tile + (long long)NSK * gridDim.x;
    io.refill = !IP && next < total;  // (IP: the stage is the work tile; refilled after its store)
    io.tmap = &tmap;
    io.mbar = &bars[rs];
    io.stage_ptr = stages + rs * BUF;
    {
      long long ntx, nl1;
      tile_coords(next, ntile, a.L1, a.g0, ntx, nl1);
      io.next_l1 = (int)nl1;
      io.next_c0 = (int)(ntx * Cfg::W * 2);
    }
    io.nbox = Cfg::NBOX;
    io.boxr = Cfg::BOXR;
    io.in_bw = a.in.bw;
    io.bytes = kBytes;
    mbar_wait(&bars[s], parity);
    StridedSM<Cfg::W, Cfg::R0, Cfg::PAD> sm{c};
    if constexpr (kHoist) stockham_pass<C, N, DIR, 0, Cfg::MAXR>(io, sm, work, reinterpret_cast<const C*>(a.tw), j, active, twh);
    else stockham_pass<C, N, DIR, 0, Cfg::MAXR>(io, sm, work, reinterpret_cast<const C*>(a.tw), j, active);
    if constexpr (DCT < 0) {  // forward R2R: finish the row pairs (k, N−k) of the output tile
      constexpr bool DST = DCT == -2;
      constexpr int NP = (N / 2 + Cfg::S.T) / Cfg::S.T;  // pairs per thread (upper bound)
      __syncthreads();
      const C* tw3 = reinterpret_cast<const C*>(a.tw3);
      // all pairs are read before any is written: the DST's reversed rows cross pairs
      C ok[NP], ol[NP];
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        const int k = j + q * Cfg::S.T;
        if (active && k <= N / 2) {
          const C zk = work[k * Cfg::W + c], zn = work[(k == 0 ? 0 : N - k) * Cfg::W + c];
          const C sk = {zk.x + zn.x, zk.y - zn.y}, dk = {zk.x - zn.x, zk.y + zn.y};
          const C ck = __ldg(tw3 + k);
          ok[q] = C{ck.x * sk.x - ck.y * sk.y, ck.x * dk.y + ck.y * dk.x};
          const C cl = __ldg(tw3 + (k == 0 ? 0 : N - k));
          const C sl = {sk.x, -sk.y}, dl = {-dk.x, dk.y};
          ol[q] = C{cl.x * sl.x - cl.y * sl.y, cl.x * dl.y + cl.y * dl.x};
        }
      }
      if constexpr (DST) __syncthreads();
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        const int k = j + q * Cfg::S.T;
        if (active && k <= N / 2) {
          const int rk = DST ? N - 1 - k : k;
          work[rk * Cfg::W + c] = dct_spec(a, rk, l0, l1, ok[q]);
          if (k > 0 && 2 * k != N) {
            const int rl = DST ? k - 1 : N - k;
            work[rl * Cfg::W + c] = dct_spec(a, rl, l0, l1, ol[q]);
          }
        }
      }
    }
    if constexpr (TST) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
      __syncthreads();
      if (threadIdx.x == 0) {
        if constexpr (OM == 1) {
          const int c0 = (int)(tx * Cfg::W * 2);
          const C* src = work;
          for (int q = 0; q < Cfg::NBOX; ++q)
            tma_store_tile(&omap, a.out.bw, c0, q * Cfg::BOXR, (int)l1, src + q * Cfg::BOXR * Cfg::W);
        } else {
          const long long e1 = tx * a.out.mT + l1;  // block tx (bw == W), line l1
          for (int q = 0; q < a.out.nbulk; ++q) {
            const BulkSeg& g = a.out.bulk[q];
            C* dst = reinterpret_cast<C*>(a.out.bases[g.sel]) + (g.off0 + e1 * g.s1);
            bulk_store(dst, work + g.tlo * Cfg::W, (uint32_t)(g.tn * Cfg::W * Cfg::ES));
          }
        }
        bulk_commit();
        if constexpr (IP) {
          if (next < total) {  // the store has read the stage: the tile NSK steps ahead goes in
            bulk_wait_read0();
            issue(next, s);
          }
        }
      }
    }
  }
  if (TST && threadIdx.x == 0) bulk_wait0();
}

// ------------------------------------------------------------------ generic lengths
// Any 2^a 3^b 5^c 7^d length without a specialised instantiation: the same Stockham passes with the
// radix schedule read at run time (PassArgs::gen, make_sched), each pass dispatched to its
// compile-time butterfly, ping-pong through shared memory (one barrier per pass).  CONTIG: gen_per
// lines per CTA (t unit stride on the global side); strided: gen_per columns per CTA.
template <typename C, int DIR, int R, bool FIRST, bool LAST, class IO, class IDX>
__device__ __forceinline__ void gen_pass(IO& io, const IDX& idx, const C* src, C* dst, const C* tw, int n, int Ns,
                                         int j, int TP, bool active) {
  const int NR = n / R;
  for (int b = j; b < NR; b += TP) {
    C v[R];
    const int m = b % Ns;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if constexpr (FIRST) v[r] = active ? io.load(b + r * NR) : C{0, 0};
      else v[r] = src[idx(b + r * NR)];
    }
    if constexpr (!FIRST) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(tw + (r - 1) * Ns + m));
    }
    dft<DIR, R>(v);
    const int d = (b / Ns) * Ns * R + m;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if constexpr (LAST) {
        if (active) io.store(d + r * Ns, v[r]);
      } else {
        dst[idx(d + r * Ns)] = v[r];
      }
    }
  }
}
template <typename C, int DIR, bool FIRST, bool LAST, class IO, class IDX>
__device__ __forceinline__ void gen_pass_any(int R, IO& io, const IDX& idx, const C* src, C* dst, const C* tw, int n,
                                             int Ns, int j, int TP, bool active) {
  switch (R) {
    case 2: gen_pass<C, DIR, 2, FIRST, LAST>(io, idx, src, dst, tw, n, Ns, j, TP, active); break;
    case 3: gen_pass<C, DIR, 3, FIRST, LAST>(io, idx, src, dst, tw, n, Ns, j, TP, active); break;
    case 4: gen_pass<C, DIR, 4, FIRST, LAST>(io, idx, src, dst, tw, n, Ns, j, TP, active); break;
    case 5: gen_pass<C, DIR, 5, FIRST, LAST>(io, idx, src, dst, tw, n, Ns, j, TP, active); break;
    case 7: gen_pass<C, DIR, 7, FIRST, LAST>(io, idx, src, dst, tw, n, Ns, j, TP, active); break;
    case 8: gen_pass<C, DIR, 8, FIRST, LAST>(io, idx, src, dst, tw, n, Ns, j, TP, active); break;
    default: gen_pass<C, DIR, 16, FIRST, LAST>(io, idx, src, dst, tw, n, Ns, j, TP, active); break;
  }
}
struct GenLineIdx {
  int base;
  __device__ __forceinline__ int operator()(int t) const { return base + t; }
};
struct GenColIdx {
  int W, c;
  __device__ __forceinline__ int operator()(int t) const { return t * W + c; }
};

constexpr int kGenThreads = 256;

template <typename Real, int DIR, bool CONTIG, bool SPEC = false>
__global__ void __launch_bounds__(kGenThreads) fft_generic_kernel(const __grid_constant__ PassArgs a) {
  using C = typename CT<Real>::type;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int n = a.gen.n, per = a.gen_per;
  const int TP = kGenThreads / per;  // threads per line / column
  C* buf[2] = {reinterpret_cast<C*>(smem_raw), reinterpret_cast<C*>(smem_raw) + (size_t)per * n};
  int q, j;
  long long l0, l1;
  bool active;
  bool part;  // the thread has a line / column slot (per need not divide the CTA size)
  if constexpr (CONTIG) {
    q = threadIdx.x / TP;
    j = threadIdx.x % TP;
    part = q < per;
    const long long line = (long long)blockIdx.x * per + q;
    active = part && line < a.L0 * a.L1;
    l1 = active ? line / a.L0 : 0;
    l0 = active ? line - l1 * a.L0 : 0;
  } else {
    q = threadIdx.x % per;
    j = threadIdx.x / per;
    part = j < TP;
    const long long ntile = (a.L0 + per - 1) / per;
    l1 = blockIdx.x / ntile;
    l0 = (blockIdx.x - l1 * ntile) * per + q;
    active = part && l0 < a.L0;
    if (!active) l0 = 0;
  }
  if (!part) j = 1 << 30;  // no butterflies (the loops below start past the end); still at every barrier
  GIO<C, CONTIG, SPEC> io;
  io.init(a.in, a.out, l0, l1, a.scale);
  io.spectral(a, l0, l1);
  const C* tw = reinterpret_cast<const C*>(a.tw);
  const int np = a.gen.npass;
  int Ns = 1, twoff = 0;
  for (int p = 0; p < np; ++p) {
    const int R = a.gen.rad[p];
    const bool first = p == 0, last = p == np - 1;
    const C* src = buf[p & 1];
    C* dst = buf[(p + 1) & 1];
    const C* twp = tw + twoff;
    if constexpr (CONTIG) {
      GenLineIdx idx{q * n};
      if (first && last) gen_pass_any<C, DIR, true, true>(R, io, idx, src, dst, twp, n, Ns, j, TP, active);
      else if (first) gen_pass_any<C, DIR, true, false>(R, io, idx, src, dst, twp, n, Ns, j, TP, active);
      else if (last) gen_pass_any<C, DIR, false, true>(R, io, idx, src, dst, twp, n, Ns, j, TP, active);
      else gen_pass_any<C, DIR, false, false>(R, io, idx, src, dst, twp, n, Ns, j, TP, active);
    } else {
      GenColIdx idx{per, q};
      if (first && last) gen_pass_any<C, DIR, true, true>(R, io, idx, src, dst, twp, n, Ns, j, TP, active);
      else if (first) gen_pass_any<C, DIR, true, false>(R, io, idx, src, dst, twp, n, Ns, j, TP, active);
      else if (last) gen_pass_any<C, DIR, false, true>(R, io, idx, src, dst, twp, n, Ns, j, TP, active);
      else gen_pass_any<C, DIR, false, false>(R, io, idx, src, dst, twp, n, Ns, j, TP, active);
    }
    if (p > 0) twoff += (R - 1) * Ns;
    Ns *= R;
    if (!last) __syncthreads();
  }
}

}  // namespace dfft
