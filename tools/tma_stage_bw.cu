// tma_stage_bw.cu — design aid: HBM bandwidth of the strided FFT's tile stream with no compute.
// Persistent CTAs (one per SM) move tiles of 1024 rows x 64 B (8 float2 columns): TMA load of the
// tile (rows `pitch` bytes apart) into one of NS shared-memory stages, then a TMA store of the
// tile to the output (rows at the output pitch).  Measures how the number of tiles in flight per
// SM (NS) and the pitch of each side set the achieved bandwidth — the question behind the
// large-pitch strided pass of the 1-GPU 1024^3 plan.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_stage_bw.cu -o tools/tma_stage_bw
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NS, int BW = 16>
__global__ void __launch_bounds__(128) stream_tiles(const __grid_constant__ CUtensorMap tin,
                                                    const __grid_constant__ CUtensorMap tout, int ntx, int nl1) {
  constexpr int ROWS = 65536 / (BW * 4), BOXR = ROWS < 256 ? ROWS : 256, NB = ROWS / BOXR;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + NS * 65536);
  const long long total = (long long)ntx * nl1;
  auto issue = [&](long long tile, int s) {
    const int tx = (int)(tile % ntx), l1 = (int)(tile / ntx);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(65536) : "memory");
    // tile = (column block tx, row block of ROWS rows, line): the row block is folded into l1
    const int rb = l1 % (1024 / ROWS), ln = l1 / (1024 / ROWS);
    for (int q = 0; q < NB; ++q)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              su32(smem + s * 65536 + q * BOXR * BW * 4)),
          "l"(&tin), "r"(tx * BW), "r"(rb * ROWS + q * BOXR), "r"(ln), "r"(su32(&bar[s]))
          : "memory");
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NS; ++s)
      if (blockIdx.x + (long long)s * gridDim.x < total) issue(blockIdx.x + (long long)s * gridDim.x, s);
  }
  __syncthreads();
  int it = 0;
  for (long long tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
    const int s = it % NS;
    const uint32_t par = (uint32_t)((it / NS) & 1);
    if (threadIdx.x == 0) {
      asm volatile(
          "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
              su32(&bar[s])),
          "r"(par)
          : "memory");
      const int tx = (int)(tile % ntx), l1 = (int)(tile / ntx);
      const int rb = l1 % (1024 / ROWS), ln = l1 / (1024 / ROWS);
      for (int q = 0; q < NB; ++q)
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&tout),
                     "r"(tx * BW), "r"(rb * ROWS + q * BOXR), "r"(ln), "r"(su32(smem + s * 65536 + q * BOXR * BW * 4))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      const long long next = tile + (long long)NS * gridDim.x;
      if (next < total) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        issue(next, s);
      }
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// CL CTAs per cluster take adjacent 64 B column tiles of the same rows; a cluster barrier before
// every load issue keeps their TMA row requests in lockstep (the DRAM sees CL*64 B per row)
template <int NS, int CL>
__global__ void __launch_bounds__(128) stream_tiles_cluster(const __grid_constant__ CUtensorMap tin,
                                                            const __grid_constant__ CUtensorMap tout, int ntx, int nl1) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + NS * 65536);
  const int rank = (int)(blockIdx.x % CL), cid = (int)(blockIdx.x / CL), ncl = (int)(gridDim.x / CL);
  const long long groups = (long long)(ntx / CL) * nl1;  // tile groups of CL adjacent column tiles
  auto coords = [&](long long g, int& tx, int& l1) {
    tx = (int)(g % (ntx / CL)) * CL + rank;
    l1 = (int)(g / (ntx / CL));
  };
  auto issue = [&](long long g, int s) {
    int tx, l1;
    coords(g, tx, l1);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(65536) : "memory");
    for (int q = 0; q < 4; ++q)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              su32(smem + s * 65536 + q * 16384)),
          "l"(&tin), "r"(tx * 16), "r"(q * 256), "r"(l1), "r"(su32(&bar[s]))
          : "memory");
  };
  auto csync = [] {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  csync();
  if (threadIdx.x == 0)
    for (int s = 0; s < NS; ++s)
      if (cid + (long long)s * ncl < groups) issue(cid + (long long)s * ncl, s);
  int it = 0;
  for (long long g = cid; g < groups; g += ncl, ++it) {
    const int s = it % NS;
    const uint32_t par = (uint32_t)((it / NS) & 1);
    if (threadIdx.x == 0) {
      asm volatile(
          "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
              su32(&bar[s])),
          "r"(par)
          : "memory");
      int tx, l1;
      coords(g, tx, l1);
      for (int q = 0; q < 4; ++q)
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&tout),
                     "r"(tx * 16), "r"(q * 256), "r"(l1), "r"(su32(smem + s * 65536 + q * 16384))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncwarp();
    const long long next = g + (long long)NS * ncl;
    csync();  // every CTA of the cluster issues its part of the next group together
    if (threadIdx.x == 0 && next < groups) issue(next, s);
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}

// 3D view in floats: (2 * ncol, 1024 rows, nl1) with row pitch rp and l1 pitch lp (bytes)
CUtensorMap make_map(void* base, long long ncol, long long rp, long long lp, int nl1, int bw = 16) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)(2 * ncol), 1024, (cuuint64_t)nl1};
  cuuint64_t str[2] = {(cuuint64_t)rp, (cuuint64_t)lp};
  const int rows = 65536 / (bw * 4);
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)(rows < 256 ? rows : 256), 1}, es[3] = {1, 1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return m;
}

int main() {
  // the 1024^3 c64 z-pass geometry: 1024 columns (x) x 1024 rows (z) x 1024 lines (y)
  const long long ncol = 1024, nl1 = 1024;
  const size_t bytes = (size_t)ncol * 1024 * nl1 * 8;  // 8 GiB
  void *a, *b;
  if (cudaMalloc(&a, bytes + (64 << 20)) != cudaSuccess || cudaMalloc(&b, bytes + (64 << 20)) != cudaSuccess) return 1;
  cudaMemset(a, 0, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // small pitch: [y][z][x] (row = z at 8 KB, l1 = y at 8 MB); large: [z][y][x] (row = z at 8 MB, l1 = y at 8 KB)
  const long long SMALL = ncol * 8, LARGE = ncol * 8 * nl1;
  auto run = [&](const char* name, long long irp, long long ilp, long long orp, long long olp, int ns, int bw) {
    const int lines = (int)nl1;
    CUtensorMap tin = make_map(a, ncol, irp, ilp, lines, bw);
    CUtensorMap tout = make_map(b, ncol, orp, olp, lines, bw);
    const size_t sm = (size_t)ns * 65536 + 64;
    const void* fn = bw == 16   ? (ns == 1 ? (const void*)stream_tiles<1, 16> : (const void*)stream_tiles<2, 16>)
                     : bw == 32 ? (ns == 1 ? (const void*)stream_tiles<1, 32> : (const void*)stream_tiles<2, 32>)
                     : bw == 64 ? (ns == 1 ? (const void*)stream_tiles<1, 64> : (const void*)stream_tiles<2, 64>)
                                : (ns == 1 ? (const void*)stream_tiles<1, 128> : (const void*)stream_tiles<2, 128>);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int grid = sms;
    const int rows = 65536 / (bw * 4);
    int ntx = (int)(2 * ncol / bw), nl = lines * (1024 / rows);
    void* args[] = {&tin, &tout, &ntx, &nl};
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      cudaLaunchKernel(fn, dim3(grid), dim3(128), args, sm, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) best = ms < best ? ms : best;
    }
    const double moved = 2.0 * ncol * 1024 * lines * 8;
    printf("%-18s row %4d B x %4d rows NS=%d: %7.3f ms  %6.0f GB/s\n", name, bw * 4, rows, ns, best, moved / (best * 1e6));
  };
  for (int bw : {16, 64})
    for (int ns : {2}) {
      run("small -> small", SMALL, LARGE, SMALL, LARGE, ns, bw);
      run("large -> small", LARGE, SMALL, SMALL, LARGE, ns, bw);
      run("small -> large", SMALL, LARGE, LARGE, SMALL, ns, bw);
    }
  auto runc = [&](const char* name, long long irp, long long ilp, long long orp, long long olp, int ns, int cl) {
    CUtensorMap tin = make_map(a, ncol, irp, ilp, (int)nl1, 16);
    CUtensorMap tout = make_map(b, ncol, orp, olp, (int)nl1, 16);
    const size_t sm = (size_t)ns * 65536 + 64;
    const void* fn = cl == 2 ? (ns == 2 ? (const void*)stream_tiles_cluster<2, 2> : (const void*)stream_tiles_cluster<3, 2>)
                     : cl == 4 ? (ns == 2 ? (const void*)stream_tiles_cluster<2, 4> : (const void*)stream_tiles_cluster<3, 4>)
                               : (ns == 2 ? (const void*)stream_tiles_cluster<2, 8> : (const void*)stream_tiles_cluster<3, 8>);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    int ncl = 0;
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = sm;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(sms);
    cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg);
    cfg.gridDim = dim3(ncl * cl);
    int ntx = (int)(ncol / 8), nl = (int)nl1;
    void* args[] = {&tin, &tout, &ntx, &nl};
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      cudaLaunchKernelExC(&cfg, fn, args);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) best = ms < best ? ms : best;
    }
    const double moved = 2.0 * ncol * 1024 * nl1 * 8;
    printf("%-18s cluster %d (%d clusters) NS=%d 64 B rows: %7.3f ms  %6.0f GB/s  %s\n", name, cl, ncl, ns, best,
           moved / (best * 1e6), cudaGetErrorString(cudaGetLastError()));
  };
  for (int cl : {2, 4, 8})
    for (int ns : {2, 3}) {
      runc("small -> small", SMALL, LARGE, SMALL, LARGE, ns, cl);
      runc("large -> small", LARGE, SMALL, SMALL, LARGE, ns, cl);
      runc("small -> large", SMALL, LARGE, LARGE, SMALL, ns, cl);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
