// registry.h — host-side lookup of the instantiated FFT kernels (one per family × length ×
// precision × direction), with their launch shapes.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "fft_kernels.cuh"

namespace dfft {

enum Family {
  kContig = 0, kStrided = 1, kContigR2C = 2, kContigC2R = 3, kContigDct = 4, kStridedDct = 5, kContigDst = 6, kStridedDst = 7,
  kContigXZ8 = 8  // x-FFT fused with a radix-8 z step (fft_xz8_kernel; n = the x length)
};

struct KernelInfo {
  const void* fn = nullptr;
  const void* fn_tb = nullptr;    // contig c2c: t-blocked input side (SideMap::tb)
  const void* spec_fn = nullptr;  // strided forward: with the Poisson multiplier (PassArgs::spec)
  int threads = 0;       // CTA size
  int per_cta = 0;       // contig: lines per CTA; strided: columns per CTA (W)
  size_t smem = 0;       // dynamic shared memory bytes
  int twlen = 0;         // twiddle table length (complex elements)
  // strided family only: persistent TMA-staged variant (null if not instantiable for n)
  const void* tma_fn = nullptr;
  const void* tma_st1_fn = nullptr;  // same, with TMA stores (unsegmented output side)
  const void* tma_bk_fn = nullptr;  // same, with bulk-copy stores (column-blocked segmented output)
  const void* tma_st_spec_fn = nullptr;  // TMA stores + Poisson multiplier (forward only)
  bool tma_st_only = false;              // the TMA variant exists only with TMA stores (R2R)
  int tma_threads = 0, tma_w = 0, tma_boxr = 0, tma_maxr = 16;  // tma_maxr: its radix schedule
  size_t tma_smem = 0;
  const void* tma_ip_fn = nullptr;  // TMA stores, passes in place in the stage (one more stage in flight)
  size_t tma_ip_smem = 0;
  bool generic = false;  // fft_generic_kernel: the radix schedule is passed at run time (PassArgs::gen)
  // contig c2c with radix-32 passes: the radix-16 variant (x-FFTs whose epilogue stores to peers)
  const void* r16_fn = nullptr;
  const void* r16_fn_tb = nullptr;
  int r16_threads = 0, r16_per_cta = 0;
  size_t r16_smem = 0;
};

// Supported axis lengths: 2^a (2..4096), 3·2^a (3..3072), and the paper's
// GPU shapes 480/720/840 with radix 5 and 7.
#define DFFT_LENGTHS(X) \
  X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) \
  X(3) X(6) X(12) X(24) X(48) X(96) X(192) X(384) X(768) X(1536) X(3072) \
  X(5) X(7) X(480) X(720) X(840)

bool lookup_kernel_f32(int family, int n, int dir, KernelInfo* out);
bool lookup_kernel_f64(int family, int n, int dir, KernelInfo* out);
bool length_supported(long long n);    // c2c axis: specialised or generic (2^a 3^b 5^c 7^d <= 4096)
bool length_specialised(long long n);  // one of DFFT_LENGTHS (R2C / C2R / DCT / DST need it)
// radix schedule of length n (for twiddle generation): returns npass, fills rad[]
int length_schedule(int n, int rad[kMaxPass], int maxr = 16);

}  // namespace dfft
