// Latency of the synchronisation primitives on the D-CHAG critical path (one CTA).
#include <cstdio>
#include "../paper_2506_21411_b200/csrc/common.cuh"
using namespace dchag;

__global__ void __launch_bounds__(128, 1) probe(long long* out) {
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tslot, 512);
  if (threadIdx.x == 32) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int N = 1000;
  long long t0, t1;
  if (threadIdx.x == 0) {
    // 1. try_wait on an already-completed phase
    mbar_arrive(&bar[0]);
    t0 = clock64();
    for (int i = 0; i < N; ++i) mbar_wait(&bar[0], 0);
    t1 = clock64();
    out[0] = (t1 - t0) / N;
    // 2. arrive + wait round trip on the same thread
    uint32_t ph = 0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) { mbar_arrive(&bar[1]); mbar_wait(&bar[1], ph); ph ^= 1; }
    t1 = clock64();
    out[1] = (t1 - t0) / N;
    // 3. tcgen05.commit (no MMA pending) -> wait
    ph = 0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) { mma_commit(&bar[2]); mbar_wait(&bar[2], ph); ph ^= 1; }
    t1 = clock64();
    out[2] = (t1 - t0) / N;
    // 4. one N=64 TS MMA + commit + wait
    ph = 0;
    const uint32_t idesc = idesc_bf16_f32(128, 64);
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
      mma_ts(tslot, tslot + 256, 0, idesc, 1u);
      mma_commit(&bar[3]);
      mbar_wait(&bar[3], ph);
      ph ^= 1;
    }
    t1 = clock64();
    out[3] = (t1 - t0) / N;
  }
  __syncthreads();
  // 5. bar.sync 128
  t0 = clock64();
  for (int i = 0; i < N; ++i) asm volatile("bar.sync 1, 128;" ::: "memory");
  t1 = clock64();
  if (threadIdx.x == 0) out[4] = (t1 - t0) / N;
  // 6. tcgen05.st x32 + wait::st per warp
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = i;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  t0 = clock64();
  for (int i = 0; i < N; ++i) { tmem_st32(tslot + lane_off + 256, r); tmem_st_wait(); }
  t1 = clock64();
  if (threadIdx.x == 0) out[5] = (t1 - t0) / N;
  // 7. 4 x tcgen05.st x32 then one wait
  t0 = clock64();
  for (int i = 0; i < N; ++i) {
    tmem_st32(tslot + lane_off + 256, r); tmem_st32(tslot + lane_off + 288, r);
    tmem_st32(tslot + lane_off + 320, r); tmem_st32(tslot + lane_off + 352, r);
    tmem_st_wait();
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[6] = (t1 - t0) / N;
  // 8. fence before + after pair
  t0 = clock64();
  for (int i = 0; i < N; ++i) { tc_fence_before(); tc_fence_after(); }
  t1 = clock64();
  if (threadIdx.x == 0) out[7] = (t1 - t0) / N;
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tslot, 512); }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  probe<<<1, 128>>>(d);
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"try_wait completed", "arrive+wait same thread", "commit(no mma)+wait",
                         "mma N64 + commit + wait", "bar.sync 128", "st.x32 + wait::st",
                         "4x st.x32 + wait::st", "fence before+after"};
  printf("%s\n", cudaGetErrorString(e));
  for (int i = 0; i < 8; ++i) printf("%-28s %lld cycles\n", names[i], h[i]);
  return 0;
}
