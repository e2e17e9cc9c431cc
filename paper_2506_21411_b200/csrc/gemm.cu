// Grouped projection GEMM on tcgen05 (K_gemm).
//
//   out[g][m, n] = sum_k A[g][m, k] * W[g][n, k] + bias[g][n] (+ rowbias[g][m % P][n])
//
// A and W are bf16, K-major, loaded by TMA with a K-wide swizzle (32/64/128 B);
// the fp32 accumulator lives in TMEM (two 256-column buffers so the epilogue of
// tile i overlaps the MMAs of tile i+1).  Columns n < Nv are written as bf16 to
// outV, columns Nv <= n < Nv+Nl as fp32 to outL: the "value" and "logit" halves
// of a D-CHAG node projection folded with its consumer (K_gemm).
//
// Persistent grid; warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer,
// warps 2..5 = epilogue (one TMEM lane quarter each).
#include "common.cuh"
#include "dchag_kernels.h"

namespace dchag {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BN_MAX = 256;
constexpr int GEMM_THREADS = 192;

template <int BK, int STAGES>
struct GemmSmem {
  static constexpr int A_BYTES = GEMM_BM * BK * 2;
  static constexpr int W_BYTES = GEMM_BN_MAX * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + W_BYTES;
  static constexpr int TOTAL = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BK>
DEV uint32_t swz_layout() {
  return BK == 64 ? 2u : (BK == 32 ? 4u : 6u);
}

template <int BK, int STAGES>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
                GemmArgs args) {
  using SM = GemmSmem<BK, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SM::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int n_tiles_n = (args.N + args.BN - 1) / args.BN;
  const int n_tiles_m = args.M / GEMM_BM;
  const int tiles_per_g = n_tiles_m * n_tiles_n;
  const int total_tiles = tiles_per_g * args.G;
  const int k_steps = args.K / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmW);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tslot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const int g = t / tiles_per_g;
        const int rem = t - g * tiles_per_g;
        const int mt = rem / n_tiles_n;
        const int nt = rem - mt * n_tiles_n;
        const int m0 = mt * GEMM_BM;
        const int mo = m0 / args.Mi, mi = m0 - mo * args.Mi;
        for (int ks = 0; ks < k_steps; ++ks) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * SM::STAGE_BYTES;
          uint8_t* sW = sA + SM::A_BYTES;
          mbar_expect_tx(&full[stage], SM::A_BYTES + args.BN * BK * 2);
          tma_load_4d(sA, &tmA, &full[stage], ks * BK, mi, mo, g);
          tma_load_3d(sW, &tmW, &full[stage], ks * BK, nt * args.BN, g);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    const uint32_t idesc = idesc_bf16_f32(GEMM_BM, args.BN);
    constexpr uint32_t SBO = 8 * BK * 2;  // 8 rows x swizzle width
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], acc_phase);  // epilogue warps pre-load bias into the buffer
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * GEMM_BN_MAX;
      for (int ks = 0; ks < k_steps; ++ks) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_addr = smem_u32(smem + stage * SM::STAGE_BYTES);
          const uint32_t w_addr = a_addr + SM::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = smem_desc(a_addr + kk * 32, 16, SBO, swz_layout<BK>());
            const uint64_t wd = smem_desc(w_addr + kk * 32, 16, SBO, swz_layout<BK>());
            mma_ss(d_tmem, ad, wd, idesc, 1u);
          }
          mma_commit(&empty[stage]);
          if (ks == k_steps - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..5)
    // The accumulator buffer of tile i is pre-loaded with bias (+ row bias) while the MMAs
    // of tile i-1 run, so the drain below is pure TMEM -> bf16/fp32 -> HBM.
    const int quarter = warp & 3;
    const int row_in_tile = quarter * 32 + lane;
    const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16);
    auto tile_coords = [&](int t, int& g, int& mo, int& mi, int& nt) {
      g = t / tiles_per_g;
      const int rem = t - g * tiles_per_g;
      const int mt = rem / n_tiles_n;
      nt = rem - mt * n_tiles_n;
      const int m = mt * GEMM_BM + row_in_tile;
      mo = m / args.Mi;
      mi = m - mo * args.Mi;
    };
    // Row bias of a tile: fetched into registers one tile ahead (all 16 chunks issued at
    // once, so the HBM/L2 latency overlaps the drain of the previous tile).
    constexpr int NCH = GEMM_BN_MAX / 16;
    const bool rb_vec = (args.rowbias_row & 7) == 0 && (args.rowbias_g & 7) == 0;
    auto fetch_rb = [&](int t, uint4 (&rbv)[NCH][2]) {
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) rbv[ch][0] = rbv[ch][1] = make_uint4(0, 0, 0, 0);
      if (!args.rowbias || t >= total_tiles) return;
      int g, mo, mi, nt;
      tile_coords(t, g, mo, mi, nt);
      const __nv_bfloat16* rb = args.rowbias + (size_t)g * args.rowbias_g +
                                (size_t)(mi % args.rowbias_period) * args.rowbias_row;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int n0 = nt * args.BN + ch * 16;
        if (ch * 16 < args.BN && n0 + 16 <= args.N && rb_vec) {
          rbv[ch][0] = __ldg(reinterpret_cast<const uint4*>(rb + n0));
          rbv[ch][1] = __ldg(reinterpret_cast<const uint4*>(rb + n0 + 8));
        } else if (ch * 16 < args.BN) {
          uint32_t w[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float lo = n0 + 2 * e < args.N ? __bfloat162float(rb[n0 + 2 * e]) : 0.f;
            const float hi = n0 + 2 * e + 1 < args.N ? __bfloat162float(rb[n0 + 2 * e + 1]) : 0.f;
            w[e] = pack_bf16(lo, hi);
          }
          rbv[ch][0] = make_uint4(w[0], w[1], w[2], w[3]);
          rbv[ch][1] = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
    };
    auto init_acc = [&](int t, int buf, const uint4 (&rbv)[NCH][2]) {
      int g, mo, mi, nt;
      tile_coords(t, g, mo, mi, nt);
      const float* bias = args.bias ? args.bias + (size_t)g * args.bias_g : nullptr;
      const bool bvec = (args.bias_g & 3) == 0;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        if (ch * 16 >= args.BN) break;
        const int n0 = nt * args.BN + ch * 16;
        float v[16];
        const uint32_t q[8] = {rbv[ch][0].x, rbv[ch][0].y, rbv[ch][0].z, rbv[ch][0].w,
                               rbv[ch][1].x, rbv[ch][1].y, rbv[ch][1].z, rbv[ch][1].w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          v[2 * e] = bf16lo(q[e]);
          v[2 * e + 1] = bf16hi(q[e]);
        }
        if (bias) {
          if (n0 + 16 <= args.N && bvec) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + n0 + j));
              v[j] += b4.x; v[j + 1] += b4.y; v[j + 2] += b4.z; v[j + 3] += b4.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (n0 + j < args.N) v[j] += __ldg(bias + n0 + j);
          }
        }
        uint32_t u[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) u[j] = __float_as_uint(v[j]);
        tmem_st16(lane_base + buf * GEMM_BN_MAX + ch * 16, u);
      }
      tmem_st_wait();
    };
    // prologue: pre-load the first two tiles' buffers
    uint4 rbv[NCH][2];
    {
      int i = 0;
      for (int t = blockIdx.x; t < total_tiles && i < 2; t += gridDim.x, ++i) {
        fetch_rb(t, rbv);
        init_acc(t, i, rbv);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[i]);
      }
    }
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      int g, mo, mi, nt;
      tile_coords(t, g, mo, mi, nt);
      const int t2 = t + 2 * gridDim.x;
      fetch_rb(t2, rbv);  // in flight while this tile's MMAs finish and it drains
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = lane_base + acc * GEMM_BN_MAX;
      for (int c0 = 0; c0 < args.BN; c0 += 16) {
        const int n0 = nt * args.BN + c0;
        if (n0 >= args.N) break;
        uint32_t r[16];
        tmem_ld16(t_row + c0, r);
        tmem_ld_wait();
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
        if (n0 < args.Nv) {
          if (args.outV_f32) {
            float* o = reinterpret_cast<float*>(args.outV) + (size_t)g * args.sVg +
                       (size_t)mo * args.sVmo + (size_t)mi * args.sVmi + n0;
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
            __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(args.outV) +
                               (size_t)g * args.sVg + (size_t)mo * args.sVmo +
                               (size_t)mi * args.sVmi + n0;
            uint4 q0, q1;
            q0.x = pack_bf16(v[0], v[1]); q0.y = pack_bf16(v[2], v[3]);
            q0.z = pack_bf16(v[4], v[5]); q0.w = pack_bf16(v[6], v[7]);
            q1.x = pack_bf16(v[8], v[9]); q1.y = pack_bf16(v[10], v[11]);
            q1.z = pack_bf16(v[12], v[13]); q1.w = pack_bf16(v[14], v[15]);
            reinterpret_cast<uint4*>(o)[0] = q0;
            reinterpret_cast<uint4*>(o)[1] = q1;
          }
        } else {
          float* o = args.outL + (size_t)g * args.sLg + (size_t)mo * args.sLmo +
                     (size_t)mi * args.sLmi + (n0 - args.Nv);
          if (n0 + 16 <= args.N && (args.sLmi & 3) == 0 && (args.sLg & 3) == 0 &&
              (args.sLmo & 3) == 0 && ((n0 - args.Nv) & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (n0 + j < args.N) o[j] = v[j];
          }
        }
      }
      // re-arm this buffer for the tile two steps ahead
      if (t2 < total_tiles) init_acc(t2, acc, rbv);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

template <int BK, int STAGES>
static cudaError_t launch_gemm_t(const CUtensorMap& tA, const CUtensorMap& tW,
                                 const GemmArgs& a, int num_sms, cudaStream_t st) {
  using SM = GemmSmem<BK, STAGES>;
  auto kern = gemm_kernel<BK, STAGES>;
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::TOTAL);
  if (e != cudaSuccess) return e;
  const int tiles = a.G * (a.M / GEMM_BM) * ((a.N + a.BN - 1) / a.BN);
  const int grid = tiles < num_sms ? tiles : num_sms;
  kern<<<grid, GEMM_THREADS, SM::TOTAL, st>>>(tA, tW, a);
  return cudaGetLastError();
}

cudaError_t launch_gemm(const CUtensorMap& tA, const CUtensorMap& tW, const GemmArgs& a,
                        int bk, int num_sms, cudaStream_t st) {
  switch (bk) {
    case 64: return launch_gemm_t<64, 4>(tA, tW, a, num_sms, st);
    case 32: return launch_gemm_t<32, 6>(tA, tW, a, num_sms, st);
    case 16: return launch_gemm_t<16, 8>(tA, tW, a, num_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace dchag
