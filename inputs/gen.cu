// inputs/gen.cu — device-side fill of the seeded synthetic input (libdfft_inputs.so).
// Holds none of the FFT's arithmetic; shared by tests and bench, never by the oracle.
// Bits: value(p, g) = ((splitmix64((seed<<32) ^ (2g+p)) >> 11) * 2^-52) - 1, g = x + nx(y + ny z);
// fp32 boxes round with __double2float_rn (see inputs/__init__.py for the recipe).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t sm64(uint64_t s) {
  uint64_t z = s + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double uni(uint64_t seed, int64_t g, int part) {
  uint64_t st = (seed << 32) ^ (uint64_t)(2 * g + part);
  return (double)(sm64(st) >> 11) * 0x1p-52 - 1.0;
}

template <typename T, bool CPLX>
__global__ void fill_kernel(T* out, uint64_t seed, int64_t gnx, int64_t gny, int64_t lx, int64_t ly,
                            int64_t lz, int64_t nx, int64_t ny, int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = i % nx, r = i / nx, y = r % ny, z = r / ny;
    int64_t g = (lx + x) + gnx * ((ly + y) + gny * (lz + z));
    double re = uni(seed, g, 0);
    if (CPLX) {
      double im = uni(seed, g, 1);
      out[2 * i] = (T)re;  // double->float conversion is round-to-nearest-even
      out[2 * i + 1] = (T)im;
    } else {
      out[i] = (T)re;
    }
  }
}

}  // namespace

extern "C" int dfft_inputs_fill_box(void* out, int f32, int cplx, uint64_t seed, int64_t gnx,
                                    int64_t gny, int64_t gnz, int64_t lx, int64_t ly, int64_t lz,
                                    int64_t nx, int64_t ny, int64_t nz, void* stream) {
  (void)gnz;
  int64_t total = nx * ny * nz;
  if (total == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  int blocks = (int)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32);
  if (f32 && cplx)
    fill_kernel<float, true><<<blocks, 256, 0, s>>>((float*)out, seed, gnx, gny, lx, ly, lz, nx, ny, total);
  else if (f32)
    fill_kernel<float, false><<<blocks, 256, 0, s>>>((float*)out, seed, gnx, gny, lx, ly, lz, nx, ny, total);
  else if (cplx)
    fill_kernel<double, true><<<blocks, 256, 0, s>>>((double*)out, seed, gnx, gny, lx, ly, lz, nx, ny, total);
  else
    fill_kernel<double, false><<<blocks, 256, 0, s>>>((double*)out, seed, gnx, gny, lx, ly, lz, nx, ny, total);
  return (int)cudaGetLastError();
}
