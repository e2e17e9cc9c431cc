// Microbenchmark: tcgen05.mma issue/throughput for the shapes the D-CHAG kernels use.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_probe tools/mma_probe.cu
#include <cstdio>
#include "../paper_2506_21411_b200/csrc/common.cuh"
using namespace dchag;

template <int MODE>  // 0: TS N=64 same-acc runs of 4; 1: TS N=64 rotate 4 accs; 2: SS N=64;
                     // 3: TS N=256; 4: SS N=256; 5: TS N=128; 6: SS N=128 K-major swz128
__global__ void __launch_bounds__(128, 1) probe(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tslot, 512);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  long long t0 = 0, t1 = 0;
  if (warp == 1) {
    if (elect_one()) {
      const uint32_t saddr = smem_u32(smem);
      constexpr uint32_t N = (MODE == 3 || MODE == 4) ? 256 : ((MODE == 5 || MODE == 6) ? 128 : 64);
      const uint32_t idesc = idesc_bf16_f32(128, N);
      t0 = clock64();
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint64_t bd = smem_desc(saddr + (j & 3) * 2048, 1024, 128, 0);
          uint32_t acc;
          if (MODE == 0) acc = tb + (j >> 2) * 64;
          else if (MODE == 1) acc = tb + (j & 3) * 64;
          else if (MODE == 2) acc = tb + (j & 3) * 64;
          else acc = tb;
          if (MODE == 2 || MODE == 4 || MODE == 6) {
            const uint64_t ad = smem_desc(saddr + 65536 + (j & 3) * 2048, 1024, 128, 0);
            mma_ss(acc, ad, bd, idesc, 1u);
          } else {
            mma_ts(acc, tb + 256 + (j & 3) * 8, bd, idesc, 1u);
          }
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      t1 = clock64();
      out[blockIdx.x] = t1 - t0;
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tb, 512); }
}

template <int MODE>
void run(const char* name, double flops_per_mma) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int iters = 2000, smem = 140 * 1024;
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<MODE><<<148, 128, smem>>>(10, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<MODE><<<148, 128, smem>>>(iters, d);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double n = 16.0 * iters;
  printf("%-34s %s cyc/mma=%.1f  TFLOP/s=%.0f\n", name, cudaGetErrorString(e), h[0] / n,
         148 * n * flops_per_mma / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  run<0>("TS N=64 same acc x4", 2.0 * 128 * 64 * 16);
  run<1>("TS N=64 rotate 4 accs", 2.0 * 128 * 64 * 16);
  run<2>("SS N=64 rotate", 2.0 * 128 * 64 * 16);
  run<5>("TS N=128", 2.0 * 128 * 128 * 16);
  run<6>("SS N=128", 2.0 * 128 * 128 * 16);
  run<3>("TS N=256", 2.0 * 128 * 256 * 16);
  run<4>("SS N=256", 2.0 * 128 * 256 * 16);
  return 0;
}
