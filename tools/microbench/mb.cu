// Microbenchmarks that decide the codec kernel design on B200 (sm_100a):
// SMEM histogram atomics, FP64 divide rate, cluster barrier cost, streaming read BW.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t mix32(uint32_t x){x^=x>>16;x*=0x7feb352dU;x^=x>>15;x*=0x846ca68bU;x^=x>>16;return x;}

__global__ void k_smem_hist(int iters, int nbins, uint32_t* out, int mode) {
  extern __shared__ uint32_t h[];
  for (int i = threadIdx.x; i < nbins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t s = mix32(threadIdx.x * 7919u + blockIdx.x);
  for (int it = 0; it < iters; ++it) {
    s = mix32(s + it);
    uint32_t b = (mode == 0) ? (s % nbins) : (mode == 1 ? (s % 64) : 0);
    atomicAdd(&h[b], 1u);
  }
  __syncthreads();
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < nbins; i += blockDim.x) acc += h[i];
  if (acc == 0xFFFFFFFF) out[0] = acc;
}
__global__ void k_hash_only(int iters, uint32_t* out) {
  uint32_t s = mix32(threadIdx.x * 7919u + blockIdx.x), acc = 0;
  for (int it = 0; it < iters; ++it) { s = mix32(s + it); acc += s % 2048; }
  if (acc == 0xFFFFFFFF) out[0] = acc;
}
__global__ void k_ddiv(int iters, double* out) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 3.0 + blockIdx.x * 1e-4, acc = 0;
  for (int it = 0; it < iters; ++it) { acc += __ddiv_rn(a, b); a += 1.0; }
  if (acc == -1.0) out[0] = acc;
}
__global__ void k_dfma(int iters, double* out) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 0.999999, c0=0,c1=0,c2=0,c3=0;
  for (int it = 0; it < iters; ++it) { c0 = fma(a,b,c0); c1 = fma(a,b,c1); c2=fma(a,b,c2); c3=fma(a,b,c3); }
  if (c0+c1+c2+c3 == -1.0) out[0] = c0;
}
__global__ void __cluster_dims__(4,1,1) k_cluster_sync(int iters, uint32_t* out) {
  cg::cluster_group cl = cg::this_cluster();
  for (int it = 0; it < iters; ++it) cl.sync();
  if (threadIdx.x == 9999) out[0] = 1;
}
__global__ void k_block_sync(int iters, uint32_t* out) {
  for (int it = 0; it < iters; ++it) __syncthreads();
  if (threadIdx.x == 9999) out[0] = 1;
}
__global__ void k_read(const uint4* __restrict__ p, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  uint32_t* out; cudaMalloc(&out, 64);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs=%d clock_khz=%d\n", nsm, clk);
  float ms;
  const int iters = 4096;
  for (int threads : {256, 512, 1024}) {
    for (int mode : {0, 1, 2}) {
      int grid = nsm * (2048 / threads);
      cudaFuncSetAttribute(k_smem_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048*4);
      k_smem_hist<<<grid, threads, 2048 * 4>>>(iters, 2048, out, mode);
      cudaEventRecord(e0);
      k_smem_hist<<<grid, threads, 2048 * 4>>>(iters, 2048, out, mode);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      double per = (double)grid * threads * iters / (ms * 1e-3);
      printf("smem_hist threads=%d mode=%d(0=2048 bins,1=64 bins,2=1 bin): %.3f ms, %.2f Gatom/s total, %.2f atom/clk/SM\n",
             threads, mode, ms, per / 1e9, per / nsm / (clk * 1e3));
    }
  }
  { int grid = nsm * 4, threads = 512;
    k_hash_only<<<grid, threads>>>(iters, out);
    cudaEventRecord(e0); k_hash_only<<<grid, threads>>>(iters, out); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double per = (double)grid * threads * iters / (ms * 1e-3);
    printf("hash_only baseline: %.3f ms, %.2f elem/clk/SM\n", ms, per / nsm / (clk * 1e3)); }
  { int grid = nsm * 4, threads = 512; double* d; cudaMalloc(&d, 64);
    k_ddiv<<<grid, threads>>>(1024, d);
    cudaEventRecord(e0); k_ddiv<<<grid, threads>>>(1024, d); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double per = (double)grid * threads * 1024 / (ms * 1e-3);
    printf("ddiv: %.3f ms, %.2f Gdiv/s, %.2f div/clk/SM\n", ms, per / 1e9, per / nsm / (clk * 1e3));
    k_dfma<<<grid, threads>>>(1024, d);
    cudaEventRecord(e0); k_dfma<<<grid, threads>>>(1024, d); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    per = (double)grid * threads * 1024 * 4 / (ms * 1e-3);
    printf("dfma: %.3f ms, %.2f TFLOP/s fp64, %.2f dfma/clk/SM\n", ms, 2*per / 1e12, per / nsm / (clk * 1e3)); }
  { int grid = (nsm / 4) * 4, threads = 512;
    k_cluster_sync<<<grid, threads>>>(10000, out);
    cudaEventRecord(e0); k_cluster_sync<<<grid, threads>>>(10000, out); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("cluster(4) sync: %.1f ns each; err=%s\n", ms * 1e6 / 10000, cudaGetErrorString(cudaGetLastError()));
    k_block_sync<<<nsm, threads>>>(10000, out);
    cudaEventRecord(e0); k_block_sync<<<nsm, threads>>>(10000, out); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("block(512) sync: %.1f ns each\n", ms * 1e6 / 10000); }
  { size_t bytes = 1ull << 30; uint4* p; cudaMalloc(&p, bytes); cudaMemset(p, 1, bytes);
    for (int bpsm : {1, 2, 4}) for (int threads : {512, 1024}) {
      int grid = nsm * bpsm;
      k_read<<<grid, threads>>>(p, bytes / 16, out);
      cudaEventRecord(e0); k_read<<<grid, threads>>>(p, bytes / 16, out); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      printf("stream read grid=%d threads=%d: %.1f GB/s\n", grid, threads, bytes / (ms * 1e-3) / 1e9);
    }
    cudaFree(p); }
  printf("last err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
