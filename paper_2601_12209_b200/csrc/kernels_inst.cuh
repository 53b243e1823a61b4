// kernels_inst.cuh — instantiation + registration of the FFT kernels for one precision.
// Included by kernels_f32.cu / kernels_f64.cu with DFFT_REAL and DFFT_LOOKUP defined.
#include "registry.h"

namespace dfft {

namespace {
template <typename Real, int N, int DIR, int MODE = 0>
KernelInfo make_contig() {
#ifndef DFFT_CONTIG_R32_ALLMODES
#define DFFT_CONTIG_R32_ALLMODES 0
#endif
  // radix-32 passes for c2c lines only (MODE 0); the R2C / C2R / DCT / DST modes keep radix 16
  constexpr bool R32 = MODE == 0 || DFFT_CONTIG_R32_ALLMODES;
  using Cfg = ContigCfg<N, (int)sizeof(Real) * 2, R32>;
  KernelInfo k;
  k.fn = (const void*)&fft_contig_kernel<Real, N, DIR, MODE, false, R32>;
  if constexpr (MODE == 0) k.fn_tb = (const void*)&fft_contig_kernel<Real, N, DIR, 0, true>;
  k.threads = Cfg::THREADS;
  k.per_cta = Cfg::LPC;
  k.smem = (Cfg::S.npass > 1 || MODE == 1 || MODE >= 3) ? (size_t)Cfg::LPC * Cfg::LS * sizeof(Real) * 2 : 0;
  k.twlen = sched_twlen(Cfg::S);
  k.tma_maxr = Cfg::MAXR;  // the twiddle tables follow its radix schedule
  if constexpr (MODE == 0 && Cfg::MAXR == 32) {
    using C16 = ContigCfg<N, (int)sizeof(Real) * 2, false>;
    k.r16_fn = (const void*)&fft_contig_kernel<Real, N, DIR, 0, false, false>;
    k.r16_fn_tb = (const void*)&fft_contig_kernel<Real, N, DIR, 0, true, false>;
    k.r16_threads = C16::THREADS;
    k.r16_per_cta = C16::LPC;
    k.r16_smem = (size_t)C16::LPC * C16::LS * sizeof(Real) * 2;
  }
  return k;
}
template <typename Real, int N, int DIR, bool DST = false>
KernelInfo make_strided_dct() {
  using Cfg = StridedCfg<Real, N>;
  KernelInfo k;
  k.fn = (const void*)&fft_strided_dct_kernel<Real, N, DIR, DST>;
  k.spec_fn = k.fn;  // the DCT / DST kernels apply the Poisson multiplier at run time (dct_spec)
  k.threads = Cfg::THREADS;
  k.per_cta = Cfg::W;
  k.smem = (size_t)Cfg::SMEM_ELEMS * sizeof(Real) * 2;
  k.twlen = sched_twlen(Cfg::S);
  using TC = TmaCfg<Real, N>;
  if constexpr (TC::OK) {  // TMA-staged variant, TMA stores only (unsegmented outputs)
    k.tma_fn = k.tma_st1_fn = (const void*)&fft_strided_tma_kernel<Real, N, DIR, 1, false, DST ? 2 * DIR : DIR>;
    k.tma_st_only = true;
    k.tma_threads = TC::THREADS;
    k.tma_w = TC::W;
    k.tma_boxr = TC::BOXR;
    k.tma_maxr = TC::MAXR;
    k.tma_smem = TC::SMEM;
  }
  return k;
}
template <typename Real, int N, int DIR>
KernelInfo make_strided() {
  using Cfg = StridedCfg<Real, N>;
  KernelInfo k;
  k.fn = (const void*)&fft_strided_kernel<Real, N, DIR>;
  if constexpr (DIR < 0) k.spec_fn = (const void*)&fft_strided_kernel<Real, N, DIR, true>;
  k.threads = Cfg::THREADS;
  k.per_cta = Cfg::W;
  k.smem = Cfg::S.npass > 1 ? (size_t)Cfg::SMEM_ELEMS * sizeof(Real) * 2 : 0;
  k.twlen = sched_twlen(Cfg::S);
  using TC = TmaCfg<Real, N>;
  if constexpr (TC::OK) {
    k.tma_fn = (const void*)&fft_strided_tma_kernel<Real, N, DIR, 0>;
    k.tma_st1_fn = (const void*)&fft_strided_tma_kernel<Real, N, DIR, 1>;  // TMA stores
    k.tma_bk_fn = (const void*)&fft_strided_tma_kernel<Real, N, DIR, 2>;
    if constexpr (TC::IP_PREFER) {  // in place in the stage, three stages in flight
      k.tma_ip_fn = (const void*)&fft_strided_tma_kernel<Real, N, DIR, 1, false, 0, true>;
      k.tma_ip_smem = TC::SMEM_IP;
    }
    if constexpr (DIR < 0) k.tma_st_spec_fn = (const void*)&fft_strided_tma_kernel<Real, N, DIR, 1, true>;
    k.tma_threads = TC::THREADS;
    k.tma_w = TC::W;
    k.tma_boxr = TC::BOXR;
    k.tma_maxr = TC::MAXR;
    k.tma_smem = TC::SMEM;
  }
  return k;
}
template <typename Real, int N, int DIR>
KernelInfo make_xz8() {
  KernelInfo k;
  using Cfg = XZ8Cfg<N, (int)sizeof(Real) * 2>;
  // only where two CTAs fit an SM: with one (f32 N = 2048, f64 N = 1024: 135-139 KB of lines) the
  // fused pass measured 1.3x slower than the plain x pass and the plan keeps the whole-axis passes
  if constexpr (Cfg::OK && Cfg::FITS && Cfg::MINB == 2) {
    k.fn = (const void*)&fft_xz8_kernel<Real, N, DIR>;
    k.threads = Cfg::THREADS;
    k.per_cta = 1;  // one (y, z1) pair of 8 lines per CTA
    k.smem = (size_t)Cfg::SMEM;
    k.twlen = sched_twlen(Cfg::S);
    k.tma_maxr = Cfg::MAXR;  // the twiddle tables follow its radix schedule
  }
  return k;
}

// generic lengths: lines (contig) or columns (strided) per CTA so that the ping-pong line buffers
// stay within 64 KB and every line keeps >= 32 threads
template <typename Real, int DIR, bool CONTIG, bool SPEC = false>
KernelInfo make_generic(int n) {
  KernelInfo k;
  k.generic = true;
  k.fn = (const void*)&fft_generic_kernel<Real, DIR, CONTIG>;
  if constexpr (!CONTIG && DIR < 0) k.spec_fn = (const void*)&fft_generic_kernel<Real, DIR, false, true>;
  const int es = (int)sizeof(Real) * 2;
  int per = 32768 / (n * es);
  per = per < 1 ? 1 : per > 8 ? 8 : per;
  k.threads = kGenThreads;
  k.per_cta = per;
  k.smem = (size_t)2 * per * n * es;
  return k;
}
}  // namespace

bool DFFT_LOOKUP(int family, int n, int dir, KernelInfo* out) {
#define DFFT_CASE(N)                                                                             \
  case N:                                                                                        \
    if (family == kContig) *out = dir < 0 ? make_contig<DFFT_REAL, N, -1>() : make_contig<DFFT_REAL, N, 1>(); \
    else if (family == kContigR2C) *out = make_contig<DFFT_REAL, N, -1, 1>();                  \
    else if (family == kContigC2R) *out = make_contig<DFFT_REAL, N, 1, 2>();                   \
    else if (family == kContigDct) *out = dir < 0 ? make_contig<DFFT_REAL, N, -1, 3>() : make_contig<DFFT_REAL, N, 1, 4>(); \
    else if (family == kStridedDct) *out = dir < 0 ? make_strided_dct<DFFT_REAL, N, -1>() : make_strided_dct<DFFT_REAL, N, 1>(); \
    else if (family == kContigDst) *out = dir < 0 ? make_contig<DFFT_REAL, N, -1, 5>() : make_contig<DFFT_REAL, N, 1, 6>(); \
    else if (family == kContigXZ8) { *out = dir < 0 ? make_xz8<DFFT_REAL, N, -1>() : make_xz8<DFFT_REAL, N, 1>(); return out->fn != nullptr; } \
    else if (family == kStridedDst) *out = dir < 0 ? make_strided_dct<DFFT_REAL, N, -1, true>() : make_strided_dct<DFFT_REAL, N, 1, true>(); \
    else *out = dir < 0 ? make_strided<DFFT_REAL, N, -1>() : make_strided<DFFT_REAL, N, 1>();    \
    return true;
  switch (n) {
    DFFT_LENGTHS(DFFT_CASE)
    default:
      if (!length_supported(n) || (family != kContig && family != kStrided)) return false;
      if (family == kContig) *out = dir < 0 ? make_generic<DFFT_REAL, -1, true>(n) : make_generic<DFFT_REAL, 1, true>(n);
      else *out = dir < 0 ? make_generic<DFFT_REAL, -1, false>(n) : make_generic<DFFT_REAL, 1, false>(n);
      return true;
  }
#undef DFFT_CASE
}

}  // namespace dfft
