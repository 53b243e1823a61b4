// p2p_tma.cu — NVLink write microbenchmark for the fused-store epilogues (design aid):
// persistent CTAs (1 per SM) write 64 KB shared-memory tiles (8 complex64 columns x 1024 rows)
// into GPU 1's memory either as one contiguous cp.async.bulk copy, or as TMA tensor stores of
// 64 B rows at a given row pitch (the layouts a consumer-friendly receive window would need).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_tma tools/p2p_tma.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode 0: bulk contiguous 64 KB per tile; mode 1: TMA tensor stores through a 4D map
// (16 floats = 64 B, 1024 rows at `pitch`, slots = pitch/64 tiles side by side, blocks)
__global__ void __launch_bounds__(256) writer(const __grid_constant__ CUtensorMap map, float* dst, int tiles, int slots,
                                              int mode) {
  extern __shared__ __align__(128) float sm[];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = (float)i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      if (mode == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + (size_t)t * 16384),
                     "r"(su32(sm)), "r"(65536) : "memory");
      } else {
        for (int q = 0; q < 4; ++q)
          asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(&map),
                       "r"(0), "r"(q * 256), "r"(t % slots), "r"(t / slots), "r"(su32(sm + q * 256 * 16)) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  const size_t span = 8ull << 30;
  float* d1;
  CK(cudaSetDevice(1)); CK(cudaMalloc(&d1, span));
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0));
  float* d0; CK(cudaMalloc(&d0, span));
  CK(cudaFuncSetAttribute(writer, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int sms = 148;
  for (int peer = 0; peer < 2; ++peer)
    for (long long pitch : {64LL, 512LL, 4096LL, 65536LL}) {
      for (int mode = 0; mode < 2; ++mode) {
        if (mode == 0 && pitch != 64) continue;
        float* dst = peer ? d1 : d0;
        const long long slots = pitch / 64, rowspan = 1024 * pitch;
        const long long blocks = (span / 2) / rowspan;
        const int tiles = (int)(slots * blocks);
        CUtensorMap map;
        cuuint64_t dims[4] = {16, 1024, (cuuint64_t)slots, (cuuint64_t)blocks};
        cuuint64_t strides[3] = {(cuuint64_t)pitch, 64, (cuuint64_t)rowspan};
        cuuint32_t box[4] = {16, 256, 1, 1}, es[4] = {1, 1, 1, 1};
        CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dst, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d (pitch %lld)\n", (int)r, pitch); continue; }
        const int nt = tiles, reps = 1;
        for (int it = 0; it < 2; ++it) {
          CK(cudaEventRecord(e0));
          for (int rp = 0; rp < reps; ++rp) writer<<<sms, 256, 65536>>>(map, dst, nt, (int)slots, mode);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms = 0; CK(cudaEventElapsedTime(&ms, e0, e1));
          double bytes = (double)nt * reps * 65536;
          if (it) printf("%s %-6s pitch %6lld B: %8.1f GB/s (%.2f GB in %.3f ms)\n", peer ? "peer " : "local", mode ? "tma" : "bulk",
                         pitch, bytes / ms / 1e6, bytes / 1e9, ms);
        }
      }
    }
  return 0;
}
