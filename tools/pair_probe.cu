// Correctness + rate probe for the CTA-pair (cta_group::2) TS MMA the level-0 kernel uses:
// A (bf16, K-major) in each CTA's TMEM lanes, B split by N across the pair's shared memory
// (each CTA holds 32 of the 64 output columns, canonical no-swizzle K-major blocks), one
// M256 x N64 x K16 MMA issued by the leader, commit multicast to both CTAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/pair_probe tools/pair_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2506_21411_b200/csrc/common.cuh"
using namespace dchag;

DEV void tmem_alloc2(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)), "r"(cols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
DEV void tmem_dealloc2(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
               : "memory");
}
DEV void mma_ts2(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
      "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
DEV void commit2_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

__host__ __device__ inline float aval(int row, int k) { return (float)(((row * 3 + k * 5) % 7) - 3); }
__host__ __device__ inline float bval(int n, int k) { return (float)(((n * 2 + k * 3) % 5) - 2); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(float* out, long long* cyc, int iters) {
  __shared__ __align__(1024) uint8_t sB[4096];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  if (warp == 0) tmem_alloc2(&tslot, 128);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  // B half: n in [32*rank, 32*rank+32), k in [0,16): [k/8][n_local/8][n%8][k%8]
  for (int i = threadIdx.x; i < 32 * 16; i += 128) {
    const int nl = i / 16, k = i % 16;
    const int off = ((k / 8) * 4 + nl / 8) * 64 + (nl % 8) * 8 + (k % 8);
    reinterpret_cast<__nv_bfloat16*>(sB)[off] = __float2bfloat16(bval(32 * rank + nl, k));
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tb = tslot;
  // A: row = 128*rank + thread, 16 bf16 = 8 TMEM columns at col 64
  {
    const int row = 128 * rank + threadIdx.x;
    uint32_t v[8];
    for (int j = 0; j < 8; ++j)
      v[j] = pack_bf16(aval(row, 2 * j), aval(row, 2 * j + 1));
    tmem_st8(tb + ((uint32_t)(warp * 32) << 16) + 64, v);
    tmem_st_wait();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (rank == 0 && warp == 1 && elect_one()) {
    const uint32_t idesc = idesc_bf16_f32(256, 64);
    const uint64_t bd = smem_desc(smem_u32(sB), 512, 128, 0);
    mma_ts2(tb, tb + 64, bd, idesc, 0u);
    commit2_mc(&bar, 3);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  {
    uint32_t v[32];
    for (int half = 0; half < 2; ++half) {
      tmem_ld32(tb + ((uint32_t)(warp * 32) << 16) + half * 32, v);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j)
        out[((long long)rank * 128 + threadIdx.x) * 64 + half * 32 + j] = __uint_as_float(v[j]);
    }
  }
  // rate: iters x 16 back-to-back M256 MMAs (accumulate into the same D)
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (rank == 0 && warp == 1 && elect_one()) {
    const uint32_t idesc = idesc_bf16_f32(256, 64);
    const uint64_t bd = smem_desc(smem_u32(sB), 512, 128, 0);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int j = 0; j < 16; ++j) mma_ts2(tb, tb + 64, bd, idesc, 1u);
    commit2_mc(&bar, 3);
    mbar_wait(&bar, 1);
    cyc[0] = clock64() - t0;
  }
  if (rank == 1 && warp == 1) mbar_wait(&bar, 1);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc2(tb, 128);
  }
}

int main() {
  float* d_out;
  long long* d_cyc;
  cudaMalloc(&d_out, 256 * 64 * sizeof(float));
  cudaMalloc(&d_cyc, sizeof(long long));
  const int iters = 256;
  probe<<<2, 128>>>(d_out, d_cyc, iters);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("launch failed: %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> out(256 * 64);
  long long cyc = 0;
  cudaMemcpy(out.data(), d_out, out.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 256; ++r)
    for (int n = 0; n < 64; ++n) {
      float ref = 0.f;
      for (int k = 0; k < 16; ++k) ref += aval(r, k) * bval(n, k);
      if (out[r * 64 + n] != ref) {
        if (bad < 8) printf("mismatch r=%d n=%d got %g want %g\n", r, n, out[r * 64 + n], ref);
        ++bad;
      }
    }
  printf("pair MMA M256xN64xK16 (A in TMEM, B split by N): %s (%d mismatches)\n",
         bad ? "FAIL" : "OK", bad);
  printf("rate: %.1f cycles per MMA (%d MMAs)\n", (double)cyc / (iters * 16), iters * 16);
  return bad ? 1 : 0;
}
