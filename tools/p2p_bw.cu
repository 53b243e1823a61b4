// p2p_bw.cu — NVLink peer-access microbenchmark on 2 GPUs of one box (design aid).
// Measures, GPU0 -> GPU1 and bidirectionally: copy engine (cudaMemcpyPeerAsync), kernel stores
// and loads with contiguous 16 B/lane, and the exchange pattern of the strided FFT epilogue
// (64 B row pieces at a 4 KB stride).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cuda_runtime.h>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

// contiguous: each thread moves 16 B per iteration, grid-stride
__global__ void st_contig(float4* __restrict__ dst, const float4* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) dst[i] = src[i];
}
// pieces of `piece` bytes (8 B per lane) at a `stride`-byte pitch on the destination side
__global__ void st_pieces(float2* __restrict__ dst, const float2* __restrict__ src, size_t nelem, int piece_el, int stride_el) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nelem; i += (size_t)gridDim.x * blockDim.x) {
    size_t row = i / piece_el, col = i % piece_el;
    dst[row * stride_el + col] = src[i];
  }
}
__global__ void ld_pieces(float2* __restrict__ dst, const float2* __restrict__ src, size_t nelem, int piece_el, int stride_el) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nelem; i += (size_t)gridDim.x * blockDim.x) {
    size_t row = i / piece_el, col = i % piece_el;
    dst[i] = src[row * stride_el + col];
  }
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  const size_t bytes = 1ull << 30;
  void *a0, *b0, *a1, *b1;
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0)); CK(cudaMalloc(&a0, 8 * bytes)); CK(cudaMalloc(&b0, 8 * bytes));
  CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0)); CK(cudaMalloc(&a1, 8 * bytes)); CK(cudaMalloc(&b1, 8 * bytes));
  cudaStream_t s0, s1; cudaEvent_t e0, e1, f0, f1;
  CK(cudaSetDevice(0)); CK(cudaStreamCreate(&s0)); CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaSetDevice(1)); CK(cudaStreamCreate(&s1)); CK(cudaEventCreate(&f0)); CK(cudaEventCreate(&f1));
  int sms = 148;
  size_t moved = bytes;
  auto run = [&](const char* name, bool bidir, auto&& launch) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaSetDevice(0); cudaDeviceSynchronize(); cudaSetDevice(1); cudaDeviceSynchronize();
      cudaSetDevice(0); cudaEventRecord(e0, s0); launch(0, s0); cudaEventRecord(e1, s0);
      if (bidir) { cudaSetDevice(1); cudaEventRecord(f0, s1); launch(1, s1); cudaEventRecord(f1, s1); }
      cudaSetDevice(0); cudaEventSynchronize(e1);
      float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
      float ms1 = 0;
      if (bidir) { cudaSetDevice(1); cudaEventSynchronize(f1); cudaEventElapsedTime(&ms1, f0, f1); }
      if (rep == 1) printf("%-48s %s  %7.1f GB/s per direction (%.3f ms%s)\n", name, bidir ? "bidir" : "uni  ",
                           moved / (ms * 1e6), ms, bidir ? "" : "");
      cudaError_t err = cudaGetLastError();
      if (err != cudaSuccess) printf("  error: %s\n", cudaGetErrorString(err));
    }
  };
  for (int bidir = 0; bidir < 2; ++bidir) {
    run("copy engine cudaMemcpyPeerAsync 1 GiB", bidir, [&](int d, cudaStream_t s) {
      if (d == 0) cudaMemcpyPeerAsync(a1, 1, a0, 0, bytes, s); else cudaMemcpyPeerAsync(b0, 0, b1, 1, bytes, s); });
    run("kernel store 16B/lane contiguous", bidir, [&](int d, cudaStream_t s) {
      if (d == 0) st_contig<<<sms * 8, 256, 0, s>>>((float4*)a1, (const float4*)a0, bytes / 16);
      else st_contig<<<sms * 8, 256, 0, s>>>((float4*)b0, (const float4*)b1, bytes / 16); });
    run("kernel load 16B/lane contiguous", bidir, [&](int d, cudaStream_t s) {
      if (d == 0) st_contig<<<sms * 8, 256, 0, s>>>((float4*)a0, (const float4*)a1, bytes / 16);
      else st_contig<<<sms * 8, 256, 0, s>>>((float4*)b1, (const float4*)b0, bytes / 16); });
    for (int piece : {64, 128, 256, 512}) {
      char nm[96];
      const size_t rows = (8 * bytes) / 4096;  // destination span fits the 8 GiB buffer
      moved = rows * piece;
      snprintf(nm, sizeof nm, "kernel store %3d B pieces, 4 KB pitch, 8B/lane", piece);
      run(nm, bidir, [&](int d, cudaStream_t s) {
        int pe = piece / 8;
        if (d == 0) st_pieces<<<sms * 8, 256, 0, s>>>((float2*)a1, (const float2*)a0, moved / 8, pe, 512);
        else st_pieces<<<sms * 8, 256, 0, s>>>((float2*)b0, (const float2*)b1, moved / 8, pe, 512); });
      snprintf(nm, sizeof nm, "kernel load  %3d B pieces, 4 KB pitch, 8B/lane", piece);
      run(nm, bidir, [&](int d, cudaStream_t s) {
        int pe = piece / 8;
        if (d == 0) ld_pieces<<<sms * 8, 256, 0, s>>>((float2*)a0, (const float2*)a1, moved / 8, pe, 512);
        else ld_pieces<<<sms * 8, 256, 0, s>>>((float2*)b1, (const float2*)b0, moved / 8, pe, 512); });
      moved = bytes;
    }
    run("local HBM copy 16B/lane (reference)", false, [&](int d, cudaStream_t s) {
      st_contig<<<sms * 8, 256, 0, s>>>((float4*)b0, (const float4*)a0, bytes / 16); });
  }
  return 0;
}
