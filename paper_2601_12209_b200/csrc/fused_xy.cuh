// fused_xy.cuh — the x-FFT and the y-FFT of every z-plane in one pass over HBM (single-GPU c2c).
//
// The paper's three stages of batched 1D FFTs (§III-A) cost one HBM round trip each when
// run as separate passes.  On one GPU nothing separates the x and y stages (the 2D transform of a
// z-plane is "the first two transforms performed locally"), so this kernel runs both over a
// plane while the plane lives in L2: X workers read W x-lines of a plane from HBM, transform them
// and store the tile into a ring of scratch planes (R planes, 8 MB each at 1024^2 c64 — L2-sized);
// Y workers read W-column tiles of a finished scratch plane, transform them along y and write the
// output plane.  HBM sees one read and one write per element for both axes.
//
// Workers.  CTAs [0, nx_ctas) run X items, the rest Y items; each group takes items from its own
// ticket counter in plane order, one item at a time per CTA (in place in one tile buffer; two
// CTAs per SM).  Per plane: done_x counts X tiles whose scratch stores completed, done_y counts Y
// tiles whose scratch loads landed.  A Y item's load waits for done_x[plane] == tpp; an X item's
// store into slot plane % R waits for done_y[plane - R] == tpp.  A CTA holds one item and has
// signalled everything before it when it waits, and tickets are taken in order, so the lowest
// unfinished item can always finish; the launch is cooperative so both groups are resident.
#pragma once
#include "fft_kernels.cuh"

namespace dfft {

struct XYArgs {
  const void* tw;                // per-pass twiddles of the TMA radix schedule (x and y share N)
  long long nplanes;             // z planes
  int tpp;                       // tiles per plane: N / W (X: W lines, Y: W columns)
  int nslots;                    // scratch planes in the ring
  int nx_ctas;                   // CTAs [0, nx_ctas) are X workers
  unsigned int* done_x;          // [nplanes]
  unsigned int* done_y;          // [nplanes]
  unsigned long long* tickets;   // [0] X items handed out, [1] Y items
  double scale;                  // on the final (y) outputs
  int nodep;                     // diagnostic (DFFT_XY_NODEP): skip the cross-group waits (wrong results)
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_u32(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// X item: W lines x N, dense [line][t] as the TMA lands it; the passes exchange in place through
// the same buffer in a layout padded one slot per R0 (all reads of a pass precede its writes), and
// the last pass writes dense [line][t] again for the TMA store.
template <typename C, int N> struct XLineIO : GIO<C> {
  static constexpr bool kSyncAfterLoad = true;
  static constexpr bool kRefillNoSync = false;
  static constexpr bool kLastBar = true;
  C* buf;
  int li;
  __device__ __forceinline__ void after_load() {}
  __device__ __forceinline__ C load(int t) const { return buf[li * N + t]; }
  __device__ __forceinline__ void store(int t, C v) const { buf[li * N + t] = v; }
};
template <int N, int R0> struct XLineSM {
  int base;
  __device__ __forceinline__ int operator()(int t) const { return base + t + t / R0; }
};
// Y item: W columns x N rows, dense [t][W] (the strided tile), in place the same way
template <typename C, int W> struct YColIO : GIO<C> {
  static constexpr bool kSyncAfterLoad = true;
  static constexpr bool kRefillNoSync = false;
  static constexpr bool kLastBar = true;
  C* buf;
  int c;
  __device__ __forceinline__ void after_load() {}
  __device__ __forceinline__ C load(int t) const { return buf[t * W + c]; }
  __device__ __forceinline__ void store(int t, C v) const {
    if (this->scale != 1) {
      v.x *= this->scale;
      v.y *= this->scale;
    }
    buf[t * W + c] = v;
  }
};

template <typename Real, int N> struct XYCfg {
  using Cfg = TmaCfg<Real, N>;
  static constexpr int XPAD = Cfg::W * (N + N / Cfg::R0);             // X exchange layout
  static constexpr int YPAD = N * Cfg::W + (N / Cfg::R0) * Cfg::PAD;  // Y exchange layout
  static constexpr int BUF = XPAD > YPAD ? XPAD : YPAD;
  // one in-place tile buffer per CTA, two CTAs per SM (16 warps: one CTA's load latency and
  // hand-offs overlap the other's passes; measured against one CTA with three stages: 6.3 vs 8.0 ms)
  static constexpr size_t SMEM = (size_t)BUF * Cfg::ES + 64;
  static constexpr bool OK = Cfg::OK && 2 * (SMEM + 1024) <= 228 * 1024 && N % Cfg::W == 0 && (N * Cfg::ES) % 256 == 0;
};

template <typename Real, int N, int DIR>
__global__ void __launch_bounds__(TmaCfg<Real, N>::THREADS, 2)
fft_xy_fused_kernel(const __grid_constant__ CUtensorMap xin, const __grid_constant__ CUtensorMap xsc,
                    const __grid_constant__ CUtensorMap ysc, const __grid_constant__ CUtensorMap yout,
                    const __grid_constant__ XYArgs a) {
  using C = typename CT<Real>::type;
  using Cfg = TmaCfg<Real, N>;
  constexpr int W = Cfg::W, R0 = Cfg::R0, T = Cfg::S.T;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  C* buf = reinterpret_cast<C*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + XYCfg<Real, N>::BUF);
  long long* item_sm = reinterpret_cast<long long*>(full + 1);
  const bool is_x = (int)blockIdx.x < a.nx_ctas;
  const long long total = a.nplanes * a.tpp;
  constexpr uint32_t kBytes = (uint32_t)(Cfg::STAGE_ELEMS * Cfg::ES);
  const C* tw = reinterpret_cast<const C*>(a.tw);
  long long prev_plane = -1;  // thread 0 (X): the last stored tile's plane, not yet counted in done_x
  long long ticket = -1;      // thread 0: the next item of this CTA, taken ahead of time
  auto grab = [&]() { ticket = (long long)atomicAdd(a.tickets + (is_x ? 0 : 1), 1ULL); };
  // thread 0: start the load of the pre-taken item (Y: once its plane is complete in the ring)
  auto start = [&]() {
    const long long t = ticket;
    *reinterpret_cast<volatile long long*>(item_sm) = t;
    if (t >= total) return;
    const long long plane = t / a.tpp;
    const int tile = (int)(t - plane * a.tpp);
    if (is_x) {
      mbar_expect_tx(full, kBytes);
      tma_load_4d(buf, &xin, 0, 0, tile * W, (int)plane, full);
    } else {
      while (!a.nodep && ld_acquire_u32(a.done_x + plane) < (unsigned)a.tpp) __nanosleep(64);
      asm volatile("fence.proxy.async.global;" ::: "memory");
      mbar_expect_tx(full, kBytes);
      for (int q = 0; q < Cfg::NBOX; ++q)
        tma_load_3d(buf + q * Cfg::BOXR * W, &ysc, tile * W * 2, q * Cfg::BOXR, (int)(plane % a.nslots), full);
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    grab();
    start();
  }
  __syncthreads();
  for (uint32_t parity = 0;; parity ^= 1) {
    const long long item = *reinterpret_cast<volatile long long*>(item_sm);
    if (item >= total) break;
    const long long plane = item / a.tpp;
    const int tile = (int)(item - plane * a.tpp);
    if (threadIdx.x == 0) grab();  // the next ticket's atomic overlaps this item's passes
    mbar_wait(full, parity);
    if (!is_x && threadIdx.x == 0) red_release_add_u32(a.done_y + plane, 1u);  // scratch tile read
    if (is_x) {
      XLineIO<C, N> io;
      io.buf = buf;
      io.li = threadIdx.x / T;
      XLineSM<N, R0> sm{io.li * (N + N / R0)};
      stockham_pass<C, N, DIR, 0, Cfg::MAXR>(io, sm, buf, tw, (int)(threadIdx.x % T), true);
    } else {
      YColIO<C, W> io;
      io.buf = buf;
      io.c = threadIdx.x % W;
      io.scale = (Real)a.scale;
      StridedSM<W, R0, Cfg::PAD> sm{io.c};
      stockham_pass<C, N, DIR, 0, Cfg::MAXR>(io, sm, buf, tw, (int)(threadIdx.x / W), true);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
    __syncthreads();
    if (threadIdx.x == 0) {
      if (is_x) {
        bulk_wait0();  // the previous scratch store is complete: count it, then (maybe) wait for a slot
        if (prev_plane >= 0) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          red_release_add_u32(a.done_x + prev_plane, 1u);
        }
        if (plane >= a.nslots && !a.nodep)
          while (ld_acquire_u32(a.done_y + (plane - a.nslots)) < (unsigned)a.tpp) __nanosleep(64);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        tma_store_4d(&xsc, 0, 0, tile * W, (int)(plane % a.nslots), buf);
        prev_plane = plane;
      } else {
        for (int q = 0; q < Cfg::NBOX; ++q)
          tma_store_3d(&yout, tile * W * 2, q * Cfg::BOXR, (int)plane, buf + q * Cfg::BOXR * W);
      }
      bulk_commit();
      bulk_wait_read0();  // the store has read the buffer: it may take the next tile
      start();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bulk_wait0();
    if (is_x && prev_plane >= 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      red_release_add_u32(a.done_x + prev_plane, 1u);
    }
  }
}

}  // namespace dfft
