// Latency of one remote mbarrier arrive -> try_wait wake-up between the two CTAs of a
// cluster (the READY hop of the CTA-pair level-0 kernel). Ping-pong N rounds; report ns/hop.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/cluster_pingpong tools/cluster_pingpong.cu
#include <cstdio>
#include "../paper_2506_21411_b200/csrc/common.cuh"
using namespace dchag;

template <int MODE>  // 0: arrive default sem (.release.cta), 1: .release.cluster
__global__ void __cluster_dims__(2, 1, 1) pingpong(int rounds, long long* out) {
  __shared__ __align__(8) uint64_t bar;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  cluster_sync();
  if (threadIdx.x == 0) {
    const uint32_t other = rank ^ 1;
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&bar)), "r"(other));
    long long t0 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < rounds; ++i) {
      if (rank == 0) {
        if (MODE == 0) asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        else asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        mbar_wait(&bar, i & 1);
      } else {
        mbar_wait(&bar, i & 1);
        if (MODE == 0) asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        else asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
      }
    }
    long long t1 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (rank == 0) out[MODE] = t1 - t0;
  }
  __syncthreads();
  cluster_sync();
}

int main() {
  long long* d;
  cudaMalloc(&d, 2 * sizeof(long long));
  const int rounds = 10000;
  pingpong<0><<<2, 32>>>(rounds, d);
  pingpong<1><<<2, 32>>>(rounds, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("failed: %s\n", cudaGetErrorString(e)); return 1; }
  long long h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("remote mbarrier arrive -> wake, one hop: %.0f ns (default sem), %.0f ns (.release.cluster)\n",
         h[0] / (2.0 * rounds), h[1] / (2.0 * rounds));
  return 0;
}
