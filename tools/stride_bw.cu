// stride_bw.cu — local HBM bandwidth of the strided-FFT tile access pattern (design aid).
// A "tile" is 64 B x R rows; rows are `stride` bytes apart; consecutive CTAs take adjacent
// 64 B columns.  Variants: strided read + contiguous write, contiguous read + strided write.
#include <cuda_runtime.h>
#include <cstdio>

// each CTA (256 threads) moves tiles of 8 float2 columns x 1024 rows
__global__ void rd_strided(float2* __restrict__ dst, const float2* __restrict__ src, long long ncol_tiles,
                           long long stride_el, int rows) {
  long long tile = blockIdx.x % ncol_tiles, plane = blockIdx.x / ncol_tiles;
  src += plane * rows * stride_el;
  int c = threadIdx.x % 8, r0 = threadIdx.x / 8;
  for (int r = r0; r < rows; r += 32) {
    float2 v = src[(long long)r * stride_el + tile * 8 + c];
    dst[(tile * rows + r) * 8 + c] = v;
  }
}
__global__ void wr_strided(float2* __restrict__ dst, const float2* __restrict__ src, long long ncol_tiles,
                           long long stride_el, int rows) {
  long long tile = blockIdx.x % ncol_tiles, plane = blockIdx.x / ncol_tiles;
  dst += plane * rows * stride_el;
  int c = threadIdx.x % 8, r0 = threadIdx.x / 8;
  for (int r = r0; r < rows; r += 32) {
    float2 v = src[(tile * rows + r) * 8 + c];
    dst[(long long)r * stride_el + tile * 8 + c] = v;
  }
}

int main() {
  const size_t bytes = 1ull << 31;  // 2 GiB moved each way
  float2 *a, *b;
  cudaMalloc(&a, 9ull << 30);
  cudaMalloc(&b, 9ull << 30);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int rows = 1024;
  for (long long stride_b : {8192LL, 65536LL, 1LL << 20, 4LL << 20, 8LL << 20}) {
    long long stride_el = stride_b / 8;
    long long tiles = stride_el / 8;  // 64 B column tiles across the full row
    long long total = (long long)(bytes / 8) / ((long long)rows * 8);
    if (tiles > total) tiles = total;
    long long planes = total / tiles;
    long long moved = tiles * planes * rows * 64;
    for (int w = 0; w < 2; ++w) {
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (w) wr_strided<<<tiles * planes, 256>>>(a, b, tiles, stride_el, rows);
        else rd_strided<<<tiles * planes, 256>>>(b, a, tiles, stride_el, rows);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      printf("%s stride %8lld B: %6.0f GB/s (read+write), %.1f MB moved\n", w ? "strided WRITE" : "strided READ ",
             stride_b, 2.0 * moved / (best * 1e6), moved / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
