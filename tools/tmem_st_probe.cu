// tcgen05.st throughput: W warps per CTA (one CTA per SM) store 32 lanes x X columns of
// 32-bit words per instruction, `iters` times, with tcgen05.wait::st every `per_wait`
// stores. Reports bytes/cycle per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tmem_st_probe tools/tmem_st_probe.cu
#include <cstdio>
#include "../paper_2506_21411_b200/csrc/common.cuh"
using namespace dchag;

template <int X>
DEV void st_x(uint32_t taddr, uint32_t v) {
  if constexpr (X == 16) {
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = v + i;
    tmem_st16(taddr, r);
  } else {
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = v + i;
    tmem_st32(taddr, r);
  }
}

template <int X>
__global__ void __launch_bounds__(512, 1) probe(int iters, int per_wait, long long* out) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot + ((uint32_t)((warp & 3) * 32) << 16);
  const int colbase = (warp >> 2) * 128;  // 4 warps per lane quarter, separate columns
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    st_x<X>(tb + colbase + (i * X) % 128, (uint32_t)i);
    if ((i + 1) % per_wait == 0) tmem_st_wait();
  }
  tmem_st_wait();
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tslot, 512); }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  long long h[148];
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    for (int per_wait : {1, 4, 1000000}) {
      probe<16><<<148, warps * 32>>>(iters, per_wait, d);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double bytes = (double)warps * iters * 32 * 16 * 4;
      printf("x16 warps=%2d wait_every=%7d: %.1f B/cycle/SM\n", warps, per_wait, bytes / h[0]);
      probe<32><<<148, warps * 32>>>(iters, per_wait, d);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      bytes = (double)warps * iters * 32 * 32 * 4;
      printf("x32 warps=%2d wait_every=%7d: %.1f B/cycle/SM\n", warps, per_wait, bytes / h[0]);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
