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
#include <type_traits>
#include <cuda_fp16.h>

#include "common.cuh"
#include "dchag_kernels.h"

namespace dchag {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BN_MAX = 256;
constexpr int GEMM_THREADS = 320;  // producer, MMA, 8 epilogue warps
constexpr int GEMM_STAGE_OUT = 8 * 32 * 128;  // epilogue staging: 8 warps x 32 rows x 128 B
constexpr int GEMM_BIAS_SMEM = 8 * 4 * 32 * 4;  // per-warp bias of its 4 column groups (fp32)
constexpr float kCombRunMax = 65504.f * 256.f;  // range of the COMB running sum (fp16 x 2^8)

// set by the COMB epilogue when a partial child sum leaves the fp16 x 2^8 range
__device__ int g_comb_overflow = 0;

cudaError_t comb_overflow_flag(int* value, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(value, g_comb_overflow, sizeof(int));
  if (e == cudaSuccess && reset) {
    const int zero = 0;
    e = cudaMemcpyToSymbol(g_comb_overflow, &zero, sizeof(int));
  }
  return e;
}

template <int BK, int STAGES, bool PAIR = false, int OUT = GEMM_STAGE_OUT>
struct GemmSmem {
  static constexpr int A_BYTES = GEMM_BM * BK * 2;
  static constexpr int W_BYTES = (PAIR ? GEMM_BN_MAX / 2 : GEMM_BN_MAX) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + W_BYTES;
  static constexpr int OUT_BYTES = OUT;  // epilogue staging
  static constexpr int TOTAL =
      STAGES * STAGE_BYTES + OUT + GEMM_BIAS_SMEM + 1024 /*align*/ + 256 /*barriers*/;
};
// LEAN epilogue staging: 8 warps x two 4 KB buffers (32 rows x 128 B, 128B swizzle)
constexpr int GEMM_LEAN_OUT = 8 * 2 * 4096;

template <int BK>
DEV uint32_t swz_layout() {
  return BK == 64 ? 2u : (BK == 32 ? 4u : 6u);
}

// PAIR: a CTA pair (cluster of 2, cta_group::2) computes a 256 x BN tile. Rank r loads rows
// [128r, 128r + 128) of the A tile and rows [r BN/2, (r+1) BN/2) of the W tile into its own
// shared memory, both signalling the leader's full barrier (.cta_group::2 TMA); the leader
// issues M256 MMAs that read A from each CTA and W split by N across the pair, so each SM's
// shared memory carries half the W traffic (the 1-CTA kernel was bound at ~216 B/cycle of
// TMA writes + MMA reads per SM against ~128 available). Each CTA drains its own 128 rows.
DEV void mma_ss_pair(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(ad), "l"(bd),
      "r"(idesc), "r"(acc)
      : "memory");
}
DEV void commit_pair_g(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"((uint16_t)3)
      : "memory");
}
DEV uint32_t rank0_addr(const void* p) {  // shared::cluster address of rank 0's copy
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
DEV void tma_load_4d_pair(void* dst, const CUtensorMap* m, uint32_t bar_cl, int c0, int c1,
                          int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".cta_group::2 [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cl), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
DEV void tma_load_3d_pair(void* dst, const CUtensorMap* m, uint32_t bar_cl, int c0, int c1,
                          int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".cta_group::2 [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cl), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// LAY (operand layouts, training backward / weight folding): bit 0 = A is MN-major
// (element (m, k) at (k / Ki) * sAko + (k % Ki) * lda + m: TMA'd as two 64-row x 64-column
// 128B-swizzled atoms per stage), bit 1 = W is MN-major ((n, k) at k * ldw + n). MN-major
// operands need BK = 64 and the CTA-pair kernel; the MMA reads them with the transpose bits
// of the instruction descriptor.
// DCHAG_GEMM_DEBUG bit 16: per-tile event timestamps (globaltimer ns) into outL, as
// [event][cta][64 tiles] int64 (timing probe only; tools/gemm_epi_probe.py)
#define GEMM_TRACE(ev, i)                                                                     \
  do {                                                                                        \
    if ((args.debug & 16) && (i) < 64) {                                                      \
      long long t_;                                                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                  \
      reinterpret_cast<long long*>(args.outL)[((ev) * gridDim.x + blockIdx.x) * 64 + (i)] = t_; \
    }                                                                                         \
  } while (0)

// LEAN 1: the plain bf16 epilogue (bias, no row bias / mask / row-dot / combine, every tile
// full and a multiple of 64 columns wide); LEAN 2: the same drain for row-dot tiles; LEAN 3:
// narrow fp32 logit-only tiles (see the epilogue below).
template <int BK, int STAGES, bool PAIR, bool COMB = false, int LAY = 0, int LEAN = 0>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
                const __grid_constant__ CUtensorMap tmV, GemmArgs args) {
  using SM = GemmSmem<BK, STAGES, PAIR, (LEAN == 1 || LEAN == 4) ? GEMM_LEAN_OUT : GEMM_STAGE_OUT>;
  constexpr int CL = PAIR ? 2 : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* stage_out = smem + STAGES * SM::STAGE_BYTES;
  float* bias_smem = reinterpret_cast<float*>(stage_out + SM::OUT_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_out + SM::OUT_BYTES + GEMM_BIAS_SMEM);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int n_tiles_n = (args.N + args.BN - 1) / args.BN;
  const int n_tiles_m = args.M / GEMM_BM;
  const int ctiles_n = n_tiles_n, ctiles_m = n_tiles_m / CL;
  const int ctiles_per_g = ctiles_m * ctiles_n;
  const int total_ct = ctiles_per_g * args.G;
  const int k_steps = args.K / BK;
  const int crank = PAIR ? (int)cluster_rank() : 0;
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  // Row-dot mode walks the groups innermost over a contiguous chunk of tiles per CTA, so
  // consecutive tiles of a CTA share (mt, nt) and the epilogue keeps its dotG rows in
  // registers across the groups; otherwise tiles are strided over the CTAs, groups outermost.
  const bool dot_mode = !COMB && args.dotOut != nullptr;
  constexpr bool comb = COMB;
  const int chunk = (total_ct + ncl - 1) / ncl;
  const int ct_begin = dot_mode ? cid * chunk : cid;
  const int ct_end = dot_mode ? min(total_ct, ct_begin + chunk) : total_ct;
  const int ct_step = dot_mode ? 1 : ncl;
  auto decode = [&](int ct, int& g, int& mt, int& nt) {
    int mc;
    if (dot_mode) {
      const int rest = args.fd_G.div(ct);
      g = ct - rest * args.G;
      mc = args.fd_ctn.div(rest);
      nt = rest - mc * ctiles_n;
    } else {
      g = args.fd_cpg.div(ct);
      const int rem = ct - g * ctiles_per_g;
      mc = args.fd_ctn.div(rem);
      nt = rem - mc * ctiles_n;
    }
    mt = mc * CL + crank;
  };

  // COMB: children [c_first, c_first + c_n) summed by output group g (split s of parent j)
  auto comb_range = [&](int g, int& c_first, int& c_n) {
    const int j = g % args.nparents, sp = g / args.nparents;
    const int f = __ldg(args.cfirst + j), n = __ldg(args.ccount + j);
    const int lo = sp * n / args.csplit, hi = (sp + 1) * n / args.csplit;
    c_first = f + lo;
    c_n = hi - lo;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmW);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8 * CL);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(tslot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc(tslot, 512);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // the pair signals each other's barriers from here on
  tc_fence_after();
  const uint32_t tmem_base = *tslot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const int w_rows = args.BN / CL;
      for (int ct = ct_begin; ct < ct_end; ct += ct_step) {
        int g0, mt, nt;
        decode(ct, g0, mt, nt);
        const int m0 = mt * GEMM_BM;
        const int mo = args.fd_Mi.div(m0), mi = m0 - mo * args.Mi;
        int c_first = g0, c_n = 1;
        if (comb) comb_range(g0, c_first, c_n);
        for (int ci = 0; ci < c_n; ++ci)
        for (int ks = 0; ks < k_steps; ++ks) {
          const int g = c_first + ci;
          mbar_wait(&empty[stage], phase ^ 1);
          GEMM_TRACE(0, (ct - ct_begin) / ct_step);
          uint8_t* sA = smem + stage * SM::STAGE_BYTES;
          uint8_t* sW = sA + SM::A_BYTES;
          if (PAIR) {
            // both CTAs' bytes complete on the leader's full barrier
            if (crank == 0)
              mbar_expect_tx(&full[stage], 2 * (SM::A_BYTES + w_rows * BK * 2));
            const uint32_t fb = rank0_addr(&full[stage]);
            if constexpr ((LAY & 1) != 0) {
              const int k0 = ks * BK, ko = k0 / args.Ki, ki = k0 - ko * args.Ki;
              tma_load_4d_pair(sA, &tmA, fb, m0, ki, ko, g);
              tma_load_4d_pair(sA + 8192, &tmA, fb, m0 + 64, ki, ko, g);
            } else {
              tma_load_4d_pair(sA, &tmA, fb, ks * BK, mi, mo, g);
            }
            if constexpr ((LAY & 2) != 0) {
              for (int j = 0; j < w_rows / 64; ++j)
                tma_load_3d_pair(sW + j * 8192, &tmW, fb, nt * args.BN + crank * w_rows + 64 * j,
                                 ks * BK, g);
            } else {
              tma_load_3d_pair(sW, &tmW, fb, ks * BK, nt * args.BN + crank * w_rows, g);
            }
          } else {
            mbar_expect_tx(&full[stage], SM::A_BYTES + args.BN * BK * 2);
            tma_load_4d(sA, &tmA, &full[stage], ks * BK, mi, mo, g);
            tma_load_3d(sW, &tmW, &full[stage], ks * BK, nt * args.BN, g);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (the leader of a pair)
    if (crank == 0) {
      const uint32_t idesc = idesc_bf16_f32(GEMM_BM * CL, args.BN) |
                             ((LAY & 1) ? (1u << 15) : 0u) | ((LAY & 2) ? (1u << 16) : 0u);
      constexpr uint32_t SBO = 8 * BK * 2;  // 8 rows x swizzle width
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int ct = ct_begin; ct < ct_end; ct += ct_step) {
       int c_n = 1;
       if (comb) {
         int g0, mt, nt, cf;
         decode(ct, g0, mt, nt);
         comb_range(g0, cf, c_n);
       }
       for (int ci = 0; ci < c_n; ++ci) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);  // epilogues drained this accumulator buffer
        tc_fence_after();
        if (lane == 0) GEMM_TRACE(1, (ct - ct_begin) / ct_step);
        const uint32_t d_tmem = tmem_base + acc * GEMM_BN_MAX;
        for (int ks = 0; ks < k_steps; ++ks) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) GEMM_TRACE(2, (ct - ct_begin) / ct_step);
          if (elect_one()) {
            const uint32_t a_addr = smem_u32(smem + stage * SM::STAGE_BYTES);
            const uint32_t w_addr = a_addr + SM::A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              // MN-major: 16 K rows of 128 B per k-step, 64-element atoms 8 KB apart
              const uint64_t ad = (LAY & 1) ? smem_desc(a_addr + kk * 2048, 8192, 1024, 2u)
                                            : smem_desc(a_addr + kk * 32, 16, SBO, swz_layout<BK>());
              const uint64_t wd = (LAY & 2) ? smem_desc(w_addr + kk * 2048, 8192, 1024, 2u)
                                            : smem_desc(w_addr + kk * 32, 16, SBO, swz_layout<BK>());
              if (!(args.debug & 4)) {
                if (PAIR) mma_ss_pair(d_tmem, ad, wd, idesc, (ks | kk) != 0);
                else mma_ss(d_tmem, ad, wd, idesc, (ks | kk) != 0);
              }
            }
            if (PAIR) {
              commit_pair_g(&empty[stage]);
              if (ks == k_steps - 1) commit_pair_g(&tfull[acc]);
            } else {
              mma_commit(&empty[stage]);
              if (ks == k_steps - 1) mma_commit(&tfull[acc]);
            }
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
       }
      }
    }
  } else if constexpr (COMB && LEAN == 4) {
    // ------------------------------------------------ lean combine epilogue (warps 2..9)
    // As the lean epilogue (warp = rows [32q, 32q + 32) x columns [128 hf, 128 hf + 128)),
    // with the softmax-weighted sum over the parent's children kept in registers as fp16
    // pairs scaled by 2^-8 (range +-1.68e7, as the general combine epilogue): per child and
    // column pair one FFMA pair ((acc + bias) / 256 with the bias pre-scaled in shared
    // memory), one pack and one HFMA2 (run += p_child,head * v / 256); the last child is
    // added in fp32 and leaves as bf16 through the 128B-swizzled staging + TMA store. A
    // partial sum beyond the fp16 range raises the overflow flag (dchag_combine_overflow).
    const int quarter = warp & 3;
    const int hf = (warp - 2) >> 2;
    const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16);
    const uint32_t my_stage = smem_u32(stage_out) + (uint32_t)(warp - 2) * 8192u;
    const uint32_t my_bias = smem_u32(bias_smem) + (uint32_t)(warp - 2) * 512u;
    const int cols = args.BN - hf * 128;  // 128, 64 or <= 0 (BN % 64 == 0)
    const int npairs = cols >= 128 ? 2 : (cols >= 64 ? 1 : 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    int vbuf = 0;
    for (int t = ct_begin; t < ct_end; t += ct_step) {
      int g, mt, nt;
      decode(t, g, mt, nt);
      int c_first, c_n;
      comb_range(g, c_first, c_n);
      const int c0 = nt * args.BN + hf * 128;
      const int m_row = mt * GEMM_BM + quarter * 32 + lane;
      const int r0 = mt * GEMM_BM + quarter * 32;
      const int mo0 = args.fd_Mi.div(r0), mi0 = r0 - mo0 * args.Mi;
      const int hd0 = min(c0 / args.dh, args.H - 1), hd1 = min((c0 + 64) / args.dh, args.H - 1);
      __half2 run[2][32];
      __half2 mx = __float2half2_rn(0.f);
      for (int ci = 0; ci < c_n; ++ci) {
        const int gb = c_first + ci;
        const bool last = ci + 1 == c_n;
        float4 b4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (args.bias && 4 * lane < cols)
          b4 = __ldg(reinterpret_cast<const float4*>(args.bias + (size_t)gb * args.bias_g + c0) +
                     lane);
        const float* lp = args.Lpre + ((size_t)gb * args.M + m_row) * args.H;
        const float pw0 = __ldg(lp + hd0), pw1 = __ldg(lp + hd1);
        __syncwarp();  // the previous child's bias reads are done
        constexpr float kS = 1.f / 256.f;
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(my_bias + 16u * lane),
                     "f"(b4.x * kS), "f"(b4.y * kS), "f"(b4.z * kS), "f"(b4.w * kS)
                     : "memory");
        __syncwarp();
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t t_col = lane_base + acc * GEMM_BN_MAX + hf * 128;
        auto release = [&]() {
          tc_fence_before();
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(rank0_addr(&tempty[acc]))
                         : "memory");
        };
        if (npairs == 0) release();
        uint32_t rn[32];
        if (npairs > 0) tmem_ld32(t_col, rn);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          if (p >= npairs) break;
          const float pw = p ? pw1 : pw0;
          const __half2 pw2 = __float2half2_rn(pw);
          const uint32_t buf = my_stage + (uint32_t)vbuf * 4096u;
          if (last) {
            if (lane == 0) bulk_wait_read1();  // this staging buffer's previous store is read
            __syncwarp();
          }
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {  // 32-column halves; the next half's load in flight
            tmem_ld_wait(rn);
            uint32_t r[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = rn[e];
            if (hh == 0 || p + 1 < npairs) tmem_ld32(t_col + p * 64 + hh * 32 + 32, rn);
            else release();
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // 4 columns per step
              float4 b;
              asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                           : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                           : "r"(my_bias + (uint32_t)(p * 64 + hh * 32 + 4 * j) * 4u));
              const float f0 = fmaf(__uint_as_float(r[4 * j]), kS, b.x);
              const float f1 = fmaf(__uint_as_float(r[4 * j + 1]), kS, b.y);
              const float f2 = fmaf(__uint_as_float(r[4 * j + 2]), kS, b.z);
              const float f3 = fmaf(__uint_as_float(r[4 * j + 3]), kS, b.w);
              __half2& u01 = run[p][16 * hh + 2 * j];
              __half2& u23 = run[p][16 * hh + 2 * j + 1];
              if (!last) {
                const __half2 h01 = __floats2half2_rn(f0, f1), h23 = __floats2half2_rn(f2, f3);
                u01 = ci ? __hfma2(pw2, h01, u01) : __hmul2(pw2, h01);
                u23 = ci ? __hfma2(pw2, h23, u23) : __hmul2(pw2, h23);
                mx = __hmax2(mx, __hmax2(__habs2(u01), __habs2(u23)));
              } else {  // last child in fp32: out = 256 (pw f / 256 + run)
                const float2 q01 = ci ? __half22float2(u01) : make_float2(0.f, 0.f);
                const float2 q23 = ci ? __half22float2(u23) : make_float2(0.f, 0.f);
                pk[2 * j] = pack_bf16(256.f * fmaf(pw, f0, q01.x), 256.f * fmaf(pw, f1, q01.y));
                pk[2 * j + 1] = pack_bf16(256.f * fmaf(pw, f2, q23.x), 256.f * fmaf(pw, f3, q23.y));
              }
            }
            if (last) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                                 buf + 128u * lane + ((uint32_t)((4 * hh + k) ^ (lane & 7)) << 4)),
                             "r"(pk[4 * k]), "r"(pk[4 * k + 1]), "r"(pk[4 * k + 2]),
                             "r"(pk[4 * k + 3])
                             : "memory");
            }
          }
          if (last) {
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_4d(&tmV, buf, c0 + p * 64, mi0, mo0, g);
              bulk_commit();
            }
            vbuf ^= 1;
          }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      // the fp16 partial sums stayed finite (an inf / NaN compares false: flagged too)
      if (!(fmaxf(__low2float(mx), __high2float(mx)) <= 65504.f)) g_comb_overflow = 1;
    }
    if (lane == 0) bulk_wait0();
  } else if constexpr (LEAN != 0) {
    // ------------------------------------------------ lean epilogue (warps 2..9)
    // Warp (quarter q, half hf) drains rows [32q, 32q + 32) x columns [128 hf, 128 hf + 128)
    // of its CTA's tile, 64 columns at a time: two TMEM loads in flight together, bias add,
    // then either (LEAN 1) bf16 pack, one 128B-swizzled 4 KB staging buffer (two per warp)
    // and one TMA store of 32 rows x 128 B, or (LEAN 2, row-dot) the two 32-column dot
    // products with this row's dotG columns (held in registers while consecutive tiles share
    // (mt, nt)), four independent partial sums each. The accumulator buffer goes back to
    // the MMA warp as soon as the last TMEM load of the tile has landed. (The general
    // epilogue below spends ~350 instructions and a dozen dependent branches per 32
    // columns; this path ~70.)
    const int quarter = warp & 3;
    const int hf = (warp - 2) >> 2;
    const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16);
    const uint32_t my_stage = smem_u32(stage_out) + (uint32_t)(warp - 2) * 8192u;
    const uint32_t my_bias = smem_u32(bias_smem) + (uint32_t)(warp - 2) * 512u;
    const int cols = args.BN - hf * 128;  // this warp's columns: 128, 64 or <= 0
    const int npairs = cols >= 128 ? 2 : (cols >= 64 ? 1 : 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    int vbuf = 0;
    int prev_mt = -1, prev_nt = -1;
    uint4 dg[LEAN == 2 ? 16 : 1];  // row-dot: this row's 128 dotG columns (bf16)
    // the bias columns of a tile are fetched one tile ahead (a dependent global load per
    // tile would otherwise stall the drain for the load's latency)
    auto fetch_bias = [&](int t2) {
      float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t2 < ct_end && args.bias && 4 * lane < cols) {
        int g2, mt2, nt2;
        decode(t2, g2, mt2, nt2);
        b = __ldg(reinterpret_cast<const float4*>(args.bias + (size_t)g2 * args.bias_g +
                                                  nt2 * args.BN + hf * 128) + lane);
      }
      return b;
    };
    float4 b_next = fetch_bias(ct_begin);
    for (int t = ct_begin; t < ct_end; t += ct_step) {
      int g, mt, nt;
      decode(t, g, mt, nt);
      const int c0 = nt * args.BN + hf * 128;
      if constexpr (LEAN == 2) {
        if (mt != prev_mt || nt != prev_nt) {
          const uint4* src = reinterpret_cast<const uint4*>(
              args.dotG + (size_t)(mt * GEMM_BM + quarter * 32 + lane) * args.ldG + c0);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            dg[j] = 8 * j < cols ? __ldg(src + j) : make_uint4(0, 0, 0, 0);
          prev_mt = mt;
          prev_nt = nt;
        }
      }
      if (warp == 2 && lane == 0) GEMM_TRACE(17, (t - ct_begin) / ct_step);
      const float4 b4 = b_next;
      b_next = fetch_bias(t + ct_step);
      __syncwarp();  // the previous tile's bias reads are done
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(my_bias + 16u * lane),
                   "f"(b4.x), "f"(b4.y), "f"(b4.z), "f"(b4.w)
                   : "memory");
      __syncwarp();
      const int r0 = mt * GEMM_BM + quarter * 32;
      const int mo0 = args.fd_Mi.div(r0), mi0 = r0 - mo0 * args.Mi;
      if (warp == 2 && lane == 0) GEMM_TRACE(18, (t - ct_begin) / ct_step);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (warp == 2 && lane == 0) GEMM_TRACE(3, (t - ct_begin) / ct_step);
      const uint32_t t_col = lane_base + acc * GEMM_BN_MAX + hf * 128;
      auto release = [&]() {
        tc_fence_before();
        __syncwarp();
        if (warp == 2 && lane == 0) GEMM_TRACE(4, (t - ct_begin) / ct_step);
        if (lane == 0) {
          if (PAIR)
            asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(rank0_addr(&tempty[acc]))
                         : "memory");
          else
            mbar_arrive(&tempty[acc]);
        }
      };
      if constexpr (LEAN == 3) {
        // narrow fp32 tiles (the logit columns alone, N <= 256): each thread writes its row's
        // columns straight from registers, 16-byte stores (rows are contiguous: coalesced)
        const int nq = cols > 0 ? (min(cols, 128) + 31) / 32 : 0;
        const int m_row = mt * GEMM_BM + quarter * 32 + lane;
        const int mo = args.fd_Mi.div(m_row), mi = m_row - mo * args.Mi;
        float* dst = args.outL + (size_t)g * args.sLg + (size_t)mo * args.sLmo +
                     (size_t)mi * args.sLmi + c0;
        if (nq == 0) release();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (q >= nq) break;
          uint32_t ra[32];
          tmem_ld32(t_col + q * 32, ra);
          tmem_ld_wait(ra);
          if (q == nq - 1) release();
          const int nvalid = min(32, cols - q * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (4 * j >= nvalid) break;
            float4 b;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                         : "r"(my_bias + (uint32_t)(q * 32 + 4 * j) * 4u));
            reinterpret_cast<float4*>(dst + q * 32)[j] =
                make_float4(__uint_as_float(ra[4 * j]) + b.x, __uint_as_float(ra[4 * j + 1]) + b.y,
                            __uint_as_float(ra[4 * j + 2]) + b.z,
                            __uint_as_float(ra[4 * j + 3]) + b.w);
          }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      if (npairs == 0) release();
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        if (p >= npairs) break;
        uint32_t ra[32], rb[32];
        tmem_ld32(t_col + p * 64, ra);
        tmem_ld32(t_col + p * 64 + 32, rb);
        tmem_ld_wait(ra);
        reg_fence32(rb);
        if (p == npairs - 1) release();
        if constexpr (LEAN == 2) {
          const int m_row = mt * GEMM_BM + quarter * 32 + lane;
          float hsum = 0.f;  // dot64: the pair's two 32-column sums
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t* r = h ? rb : ra;
            float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // 4 columns per step
              float4 b;
              asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                           : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                           : "r"(my_bias + (uint32_t)(p * 64 + h * 32 + 4 * j) * 4u));
              const uint4 q = dg[8 * p + 4 * h + (j >> 1)];
              const uint32_t q0 = (j & 1) ? q.z : q.x, q1 = (j & 1) ? q.w : q.y;
              float& a = s4[j & 3];
              a = fmaf(__uint_as_float(r[4 * j]) + b.x, bf16lo(q0), a);
              a = fmaf(__uint_as_float(r[4 * j + 1]) + b.y, bf16hi(q0), a);
              a = fmaf(__uint_as_float(r[4 * j + 2]) + b.z, bf16lo(q1), a);
              a = fmaf(__uint_as_float(r[4 * j + 3]) + b.w, bf16hi(q1), a);
            }
            const float sh = (s4[0] + s4[1]) + (s4[2] + s4[3]);
            if (args.dot64)
              hsum += sh;
            else
              args.dotOut[((size_t)g * (args.N >> 5) + (c0 >> 5) + 2 * p + h) * args.M + m_row] = sh;
          }
          if (args.dot64)
            args.dotOut[((size_t)g * (args.N >> 6) + (c0 >> 6) + p) * args.M + m_row] = hsum;
        } else {
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float4 b;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                       : "r"(my_bias + (uint32_t)(p * 64 + 4 * j) * 4u));
          const uint32_t* r = j < 8 ? ra + 4 * j : rb + 4 * (j - 8);
          pk[2 * j] = pack_bf16(__uint_as_float(r[0]) + b.x, __uint_as_float(r[1]) + b.y);
          pk[2 * j + 1] = pack_bf16(__uint_as_float(r[2]) + b.z, __uint_as_float(r[3]) + b.w);
        }
        const uint32_t buf = my_stage + (uint32_t)vbuf * 4096u;
        if (lane == 0) bulk_wait_read1();  // this buffer's previous store has read it
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                           buf + 128u * lane + ((uint32_t)(k ^ (lane & 7)) << 4)),
                       "r"(pk[4 * k]), "r"(pk[4 * k + 1]), "r"(pk[4 * k + 2]), "r"(pk[4 * k + 3])
                       : "memory");
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_4d(&tmV, buf, c0 + p * 64, mi0, mo0, g);
          bulk_commit();
        }
        vbuf ^= 1;
        }  // store tiles
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait0();  // this warp's tensor stores complete before exit
  } else {
    // ------------------------------------------------ epilogue (warps 2..9)
    // Two warps per TMEM lane quarter; warp half hf drains the 32-column groups
    // hf, hf+2, ...  bias (+ row bias, prefetched before the tile's accumulator is ready)
    // is added here; bf16/fp32 rows are transposed through a per-warp swizzled staging
    // buffer so every store instruction writes whole 64/128-byte row segments.
    const int quarter = warp & 3;
    const int hf = (warp - 2) >> 2;
    const int row_in_tile = quarter * 32 + lane;
    const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16);
    uint8_t* my_out = stage_out + (warp - 2) * (32 * 128);
    int vbuf = 0;  // TMA-store staging buffer of this warp (two of 2 KB)
    const int n_groups = (args.BN + 31) / 32;
    const bool rb_vec = (args.rowbias_row & 7) == 0 && (args.rowbias_g & 7) == 0;
    const bool b_vec = (args.bias_g & 3) == 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    // two instantiations of the tile loop: row-dot tiles and the rest (each carries only its
    // own registers: the row-dot dotG rows would otherwise stay live through the value path)
    auto tile_loop = [&](auto dot_tag) {
    constexpr bool DOT = !COMB && decltype(dot_tag)::value;
    int prev_mt = -1, prev_nt = -1;
    uint4 rbv[DOT ? 4 : 1][4];  // row-dot mode: this thread's dotG row, 4 column groups
    float4 dot_bias_pf = make_float4(0.f, 0.f, 0.f, 0.f);  // the next tile's bias columns
    bool dot_pf_valid = false;
    for (int t = ct_begin; t < ct_end; t += ct_step) {
      int g, mt, nt;
      if (warp == 2 && lane == 0) GEMM_TRACE(17, (t - ct_begin) / ct_step);
      decode(t, g, mt, nt);
      const int m_row = mt * GEMM_BM + row_in_tile;
      const int mo = args.fd_Mi.div(m_row), mi = m_row - mo * args.Mi;
      // prefetch this thread's row bias for its column groups (in flight during the wait)
      // row-dot mode: the same registers carry this row's dotG columns instead
      constexpr bool dot = DOT;
      const __nv_bfloat16* rb =
          dot ? args.dotG + (size_t)m_row * args.ldG
          : (args.rowbias && !(args.debug & 2)) ? args.rowbias + (size_t)g * args.rowbias_g +
                             (size_t)(mi % args.rowbias_period) * args.rowbias_row
                       : nullptr;
      // row-dot mode keeps its dotG rows in registers across the groups of one (mt, nt); the
      // plain row bias is loaded per column group inside the (rolled) group loop below
      const bool reload = dot && (mt != prev_mt || nt != prev_nt);
      prev_mt = mt;
      prev_nt = nt;
      if constexpr (DOT) {
#pragma unroll
        for (int gi = 0; gi < 4; ++gi) {
          if (!reload) break;
          const int n0 = nt * args.BN + (hf + 2 * gi) * 32;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            rbv[gi][j] = make_uint4(0, 0, 0, 0);
            const int n = n0 + 8 * j;
            if (rb && hf + 2 * gi < n_groups && n < args.N) {
              rbv[gi][j] = __ldg(reinterpret_cast<const uint4*>(rb + n));  // N % 32 == 0
            }
          }
        }
      }
      // row bias of one 32-column group (bf16, 8 per uint4), zeros past N / without row bias
      auto load_rowbias = [&](int n0, uint4 (&q)[4]) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          q[j] = make_uint4(0, 0, 0, 0);
          const int n = n0 + 8 * j;
          if (!rb || n >= args.N) continue;
          if (rb_vec && n + 8 <= args.N) {
            q[j] = __ldg(reinterpret_cast<const uint4*>(rb + n));
          } else {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float lo = n + 2 * e < args.N ? __bfloat162float(rb[n + 2 * e]) : 0.f;
              const float hi = n + 2 * e + 1 < args.N ? __bfloat162float(rb[n + 2 * e + 1]) : 0.f;
              w[e] = pack_bf16(lo, hi);
            }
            q[j] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      };
      if constexpr (DOT) {
        // row-dot tile: sum over each 32-column group of (acc + bias) * dotG. The tile's
        // bias row (the channel's) was fetched during the previous tile, and the TMEM loads
        // of group i+1 are in flight while group i is reduced.
        float* wbias = bias_smem + (warp - 2) * 128;
        const float* bias_t = args.bias ? args.bias + (size_t)g * args.bias_g : nullptr;
        const int nb = nt * args.BN + (hf + 2 * (lane >> 3)) * 32 + (lane & 7) * 4;
        auto fetch_bias = [&](const float* bp, int n) {
          float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
          if (!bp) return b;
          if (b_vec && n + 4 <= args.N) return __ldg(reinterpret_cast<const float4*>(bp + n));
          if (n < args.N) b.x = __ldg(bp + n);
          if (n + 1 < args.N) b.y = __ldg(bp + n + 1);
          if (n + 2 < args.N) b.z = __ldg(bp + n + 2);
          if (n + 3 < args.N) b.w = __ldg(bp + n + 3);
          return b;
        };
        if (!dot_pf_valid) dot_bias_pf = fetch_bias(bias_t, nb);
        __syncwarp();  // the previous tile's broadcast reads are done
        reinterpret_cast<float4*>(wbias)[lane] = dot_bias_pf;
        __syncwarp();
        dot_pf_valid = false;
        if (t + ct_step < ct_end && args.bias) {
          int g2, mt2, nt2;
          decode(t + ct_step, g2, mt2, nt2);
          dot_bias_pf = fetch_bias(args.bias + (size_t)g2 * args.bias_g,
                                   nt2 * args.BN + (hf + 2 * (lane >> 3)) * 32 + (lane & 7) * 4);
          dot_pf_valid = true;
        }
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t t_row = lane_base + acc * GEMM_BN_MAX;
        auto gvalid = [&](int gi) {
          const int grp = hf + 2 * gi;
          return grp < n_groups && nt * args.BN + grp * 32 < args.N;
        };
        auto reduce = [&](const uint32_t (&r)[32], int gi) {
          const int n0 = nt * args.BN + (hf + 2 * gi) * 32;
          float sdot = 0.f;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t q[4] = {rbv[gi][j].x, rbv[gi][j].y, rbv[gi][j].z, rbv[gi][j].w};
            const float4 b0 = reinterpret_cast<const float4*>(wbias + gi * 32)[2 * j];
            const float4 b1 = reinterpret_cast<const float4*>(wbias + gi * 32)[2 * j + 1];
            const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              sdot = fmaf(__uint_as_float(r[8 * j + 2 * e]) + bb[2 * e], bf16lo(q[e]), sdot);
              sdot = fmaf(__uint_as_float(r[8 * j + 2 * e + 1]) + bb[2 * e + 1], bf16hi(q[e]),
                          sdot);
            }
          }
          args.dotOut[((size_t)g * (args.N >> 5) + (n0 >> 5)) * args.M + m_row] = sdot;
        };
        uint32_t ra[32], rc[32];
        if (gvalid(0)) {
          tmem_ld32(t_row + hf * 32, ra);
          tmem_ld_wait();
          if (gvalid(1)) tmem_ld32(t_row + (hf + 2) * 32, rc);
          reduce(ra, 0);
          tmem_ld_wait();
          if (gvalid(1)) {
            if (gvalid(2)) tmem_ld32(t_row + (hf + 4) * 32, ra);
            reduce(rc, 1);
            tmem_ld_wait();
            if (gvalid(2)) {
              if (gvalid(3)) tmem_ld32(t_row + (hf + 6) * 32, rc);
              reduce(ra, 2);
              tmem_ld_wait();
              if (gvalid(3)) reduce(rc, 3);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR)
            asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(rank0_addr(&tempty[acc]))
                         : "memory");
          else
            mbar_arrive(&tempty[acc]);
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      } else {
      // combine mode: softmax statistics of this row over the parent's children, per group
      int c_first = g, c_n = 1;
      if (comb) comb_range(g, c_first, c_n);
      __half2 run[COMB ? 4 : 1][16];  // running weighted sum (fp16 pairs; fp32 math)
      for (int ci = 0; ci < c_n; ++ci) {
      const int gb = c_first + ci;  // bias / logit group of this tile (the child in COMB)
      const float* bias =
          (args.bias && !(args.debug & 2)) ? args.bias + (size_t)gb * args.bias_g : nullptr;
      // this warp's bias columns (groups hf, hf+2, hf+4, hf+6) -> shared memory with one
      // coalesced load per lane, read back as broadcasts (the per-group global loads of every
      // lane were the epilogue's largest cost)
      float* wbias = bias_smem + (warp - 2) * 128;
      auto bias_cols = [&](const float* bp, int n) {
        float4 b4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (b_vec && n + 4 <= args.N) {
          b4 = __ldg(reinterpret_cast<const float4*>(bp + n));
        } else {
          if (n < args.N) b4.x = __ldg(bp + n);
          if (n + 1 < args.N) b4.y = __ldg(bp + n + 1);
          if (n + 2 < args.N) b4.z = __ldg(bp + n + 2);
          if (n + 3 < args.N) b4.w = __ldg(bp + n + 3);
        }
        return b4;
      };
      if (bias) {
        __syncwarp();  // the previous tile's broadcast reads are done
        const int n = nt * args.BN + (hf + 2 * (lane >> 3)) * 32 + (lane & 7) * 4;
        // non-COMB tiles: this tile's bias columns were fetched during the previous tile
        const float4 b4 = (!COMB && dot_pf_valid) ? dot_bias_pf : bias_cols(bias, n);
        reinterpret_cast<float4*>(wbias)[lane] = b4;
        __syncwarp();
      }
      if (!COMB) {
        dot_pf_valid = false;
        if (bias && t + ct_step < ct_end) {  // the next tile's bias, in flight during this one
          int g2, mt2, nt2;
          decode(t + ct_step, g2, mt2, nt2);
          dot_bias_pf = bias_cols(args.bias + (size_t)g2 * args.bias_g,
                                  nt2 * args.BN + (hf + 2 * (lane >> 3)) * 32 + (lane & 7) * 4);
          dot_pf_valid = true;
        }
      }
      if (warp == 2 && lane == 0) GEMM_TRACE(18, (t - ct_begin) / ct_step);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (warp == 2 && lane == 0) GEMM_TRACE(3, (t - ct_begin) / ct_step);
      const uint32_t t_row = lane_base + acc * GEMM_BN_MAX;
      // a rolled loop over the warp's column groups (COMB keeps its running sums in registers
      // and unrolls): the kernel's instruction footprint, and with it the per-tile
      // instruction-fetch stalls, stays small
      // The TMEM load of group gi + 1 is in flight while group gi is processed, and the
      // accumulator buffer is handed back to the MMA warp as soon as the last load landed.
      auto gvalid = [&](int gi) {
        const int grp = hf + 2 * gi;
        return gi < 4 && !(args.debug & 8) && grp < n_groups && nt * args.BN + grp * 32 < args.N;
      };
      bool released = false;
      auto release = [&]() {
        tc_fence_before();
        __syncwarp();
        if (warp == 2 && lane == 0) GEMM_TRACE(4, (t - ct_begin) / ct_step);
        if (lane == 0) {
          if (PAIR)  // the leader's MMA warp waits for both CTAs' drains
            asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(rank0_addr(&tempty[acc]))
                         : "memory");
          else
            mbar_arrive(&tempty[acc]);
        }
        released = true;
      };
      uint32_t rn[32];
      if (gvalid(0)) tmem_ld32(t_row + hf * 32, rn);
#pragma unroll(COMB ? 4 : 1)
      for (int gi = 0; gi < 4; ++gi) {
        if (!gvalid(gi)) break;
        const int grp = hf + 2 * gi;
        const int n0 = nt * args.BN + grp * 32;
        uint4 rq[4];
        if constexpr (!COMB) load_rowbias(n0, rq);
        tmem_ld_wait(rn);
        uint32_t r[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = rn[j];
        if (gvalid(gi + 1)) tmem_ld32(t_row + (grp + 2) * 32, rn);
        else release();
        float v[32];
        if constexpr (COMB) {  // no row bias in combine mode
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t q[4] = {rq[j].x, rq[j].y, rq[j].z, rq[j].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              v[8 * j + 2 * e] = __uint_as_float(r[8 * j + 2 * e]) + bf16lo(q[e]);
              v[8 * j + 2 * e + 1] = __uint_as_float(r[8 * j + 2 * e + 1]) + bf16hi(q[e]);
            }
          }
        }
        if (bias) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 b4 = reinterpret_cast<const float4*>(wbias + gi * 32)[j / 4];
            v[j] += b4.x; v[j + 1] += b4.y; v[j + 2] += b4.z; v[j + 3] += b4.w;
          }
        }
        if (!COMB && args.rmask) {
          // trunk-input epilogue (model.py:100-108 apply_token_mask): masked rows take the
          // mask token, v = v (1 - m) + mask_token m
          const float mr = __ldg(args.rmask + m_row);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float mt = n0 + j < args.N ? __ldg(args.mtok + n0 + j) : 0.f;
            v[j] = fmaf(v[j], 1.f - mr, mt * mr);
          }
        }
        if constexpr (COMB) {
          // Lpre holds the softmax over the parent's children (dchag_child_softmax)
          const int hd = min(n0 / args.dh, args.H - 1);
          const float pw = __ldg(args.Lpre + ((size_t)gb * args.M + m_row) * args.H + hd);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            // the running sum is stored as fp16 pairs scaled by 2^-8 (exact power-of-two
            // scaling): range +-1.68e7 instead of fp16's 65504, absolute error <= 2^-16
            // below 0.0156; a partial sum beyond that range raises the overflow flag
            // (dchag_combine_overflow) instead of silently becoming inf
            float2 o = ci ? __half22float2(run[gi][j]) : make_float2(0.f, 0.f);
            o.x = fmaf(pw, v[2 * j], o.x * 256.f);
            o.y = fmaf(pw, v[2 * j + 1], o.y * 256.f);
            if (ci + 1 < c_n) {
              if (fmaxf(fabsf(o.x), fabsf(o.y)) > kCombRunMax) g_comb_overflow = 1;
              run[gi][j] = __float22half2_rn(make_float2(o.x * (1.f / 256.f),
                                                         o.y * (1.f / 256.f)));
            } else {
              v[2 * j] = o.x;
              v[2 * j + 1] = o.y;
            }
          }
          if (ci + 1 < c_n) continue;
        }
        if (args.debug & 1) {
          if (__float_as_uint(v[0]) == 0x7fc00001u) args.outL[0] = v[1];
          continue;
        }
        const int gcols = min(32, args.BN - grp * 32);  // columns of this group in the tile
        if ((gcols == 32 || gcols == 16) && n0 + gcols <= args.Nv) {
          // value region: stage in smem (swizzled) + coalesced copy-out of whole row segments
          const int nk = gcols / 8;          // 16-byte chunks per row (bf16)
          if (!args.outV_f32 && args.v_tma && gcols == 32) {
            // 32 rows x 32 columns -> 64B-swizzled staging (two buffers per warp) -> one TMA
            // tensor store; the store drains asynchronously while the warp moves on
            uint8_t* buf = my_out + vbuf * 2048;
            if (lane == 0) bulk_wait_read1();  // this buffer's previous store has read it
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              uint4 o;
              o.x = pack_bf16(v[8 * k + 0], v[8 * k + 1]);
              o.y = pack_bf16(v[8 * k + 2], v[8 * k + 3]);
              o.z = pack_bf16(v[8 * k + 4], v[8 * k + 5]);
              o.w = pack_bf16(v[8 * k + 6], v[8 * k + 7]);
              *reinterpret_cast<uint4*>(buf + lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4)) = o;
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              const int r0 = mt * GEMM_BM + quarter * 32;
              const int mo0 = args.fd_Mi.div(r0), mi0 = r0 - mo0 * args.Mi;
              tma_store_4d(&tmV, smem_u32(buf), n0, mi0, mo0, g);
              bulk_commit();
            }
            vbuf ^= 1;
          } else if (!args.outV_f32) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (k < nk) {
                uint4 o;
                o.x = pack_bf16(v[8 * k + 0], v[8 * k + 1]);
                o.y = pack_bf16(v[8 * k + 2], v[8 * k + 3]);
                o.z = pack_bf16(v[8 * k + 4], v[8 * k + 5]);
                o.w = pack_bf16(v[8 * k + 6], v[8 * k + 7]);
                *reinterpret_cast<uint4*>(my_out + lane * 64 + ((k ^ (lane & 3)) << 4)) = o;
              }
            }
            __syncwarp();
            const int mt0 = mt * GEMM_BM + quarter * 32;
            const int rows_per = 32 / nk;    // rows written per warp instruction
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (i < nk) {
                const int rr = i * rows_per + lane / nk, k = lane % nk;
                const int mrow = mt0 + rr;
                const int mo2 = args.fd_Mi.div(mrow), mi2 = mrow - mo2 * args.Mi;
                const uint4 o =
                    *reinterpret_cast<const uint4*>(my_out + rr * 64 + ((k ^ (rr & 3)) << 4));
                *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(args.outV) +
                                          (size_t)g * args.sVg + (size_t)mo2 * args.sVmo +
                                          (size_t)mi2 * args.sVmi + n0 + k * 8) = o;
              }
            }
            __syncwarp();
          } else {
            const int nk4 = gcols / 4;       // 16-byte chunks per row (fp32)
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (k < nk4)
                *reinterpret_cast<float4*>(my_out + lane * 128 + ((k ^ (lane & 7)) << 4)) =
                    make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
            __syncwarp();
            const int mt0 = mt * GEMM_BM + quarter * 32;
            const int rows_per = 32 / nk4;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (i < nk4) {
                const int rr = i * rows_per + lane / nk4, k = lane % nk4;
                const int mrow = mt0 + rr;
                const int mo2 = args.fd_Mi.div(mrow), mi2 = mrow - mo2 * args.Mi;
                float4 o =
                    *reinterpret_cast<const float4*>(my_out + rr * 128 + ((k ^ (rr & 7)) << 4));
                float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(args.outV) +
                                                        (size_t)g * args.sVg + (size_t)mo2 * args.sVmo +
                                                        (size_t)mi2 * args.sVmi + n0 + k * 4);
                if (args.accum) {  // out += acc (one owner per element: deterministic)
                  const float4 old = *dst;
                  o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
                }
                *dst = o;
              }
            }
            __syncwarp();
          }
        } else {
          // mixed / logit region (few columns): direct per-row stores
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = n0 + j;
            if (n >= args.N || j >= gcols) break;
            if (n < args.Nv) {
              if (args.outV_f32) {
                float* dst = reinterpret_cast<float*>(args.outV) + (size_t)g * args.sVg +
                             (size_t)mo * args.sVmo + (size_t)mi * args.sVmi + n;
                *dst = args.accum ? *dst + v[j] : v[j];
              } else
                reinterpret_cast<__nv_bfloat16*>(args.outV)[(size_t)g * args.sVg +
                                                            (size_t)mo * args.sVmo +
                                                            (size_t)mi * args.sVmi + n] =
                    __float2bfloat16(v[j]);
            } else {
              args.outL[(size_t)g * args.sLg + (size_t)mo * args.sLmo + (size_t)mi * args.sLmi +
                        (n - args.Nv)] = v[j];
            }
          }
        }
      }
      if (!released) release();
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }  // children (COMB)
      }  // value / combine tiles
    }
    };
    if (!COMB && dot_mode) tile_loop(std::true_type{});
    else tile_loop(std::false_type{});
    if (lane == 0) bulk_wait0();  // this warp's tensor stores complete before exit
  }

  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // no CTA leaves while its peer may still signal its barriers
  if (warp == 1) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                   : "memory");
    else
      tmem_dealloc(tmem_base, 512);
  }
}

template <int BK, int STAGES, bool PAIR, bool COMB = false, int LAY = 0, int LEAN = 0>
static cudaError_t launch_gemm_t(const CUtensorMap& tA, const CUtensorMap& tW,
                                 const CUtensorMap& tV, const GemmArgs& a, int num_sms,
                                 cudaStream_t st) {
  using SM = GemmSmem<BK, STAGES, PAIR, (LEAN == 1 || LEAN == 4) ? GEMM_LEAN_OUT : GEMM_STAGE_OUT>;
  static_assert(SM::TOTAL <= 227 * 1024, "shared memory");
  auto kern = gemm_kernel<BK, STAGES, PAIR, COMB, LAY, LEAN>;
  GemmArgs af = a;
  {
    constexpr int CLh = PAIR ? 2 : 1;
    const int ctn = (a.N + a.BN - 1) / a.BN;
    const int cpg = (a.M / GEMM_BM / CLh) * ctn;
    af.fd_G = make_fastdiv((unsigned)a.G);
    af.fd_cpg = make_fastdiv((unsigned)(cpg > 0 ? cpg : 1));
    af.fd_ctn = make_fastdiv((unsigned)(ctn > 0 ? ctn : 1));
    af.fd_Mi = make_fastdiv((unsigned)a.Mi);
  }
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::TOTAL);
  if (e != cudaSuccess) return e;
  constexpr int CL = PAIR ? 2 : 1;
  const int ctiles = a.G * (a.M / GEMM_BM / CL) * ((a.N + a.BN - 1) / a.BN);
  const int max_cl = num_sms / CL;
  const int grid = (ctiles < max_cl ? ctiles : max_cl) * CL;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = SM::TOTAL;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, tA, tW, tV, af);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_gemm(const CUtensorMap& tA, const CUtensorMap& tW, const CUtensorMap& tV,
                        const GemmArgs& a, int bk, int num_sms, cudaStream_t st) {
  switch (bk) {
    case 64:
      if (a.lay) {
        if (!a.pair || a.cfirst) return cudaErrorInvalidValue;
        if (a.lay == 1) return launch_gemm_t<64, 5, true, false, 1>(tA, tW, tV, a, num_sms, st);
        if (a.lay == 2) return launch_gemm_t<64, 5, true, false, 2>(tA, tW, tV, a, num_sms, st);
        return launch_gemm_t<64, 5, true, false, 3>(tA, tW, tV, a, num_sms, st);
      }
      if (a.pair && a.cfirst && a.lean == 4)
        return launch_gemm_t<64, 4, true, true, 0, 4>(tA, tW, tV, a, num_sms, st);
      if (a.pair && a.cfirst) return launch_gemm_t<64, 5, true, true>(tA, tW, tV, a, num_sms, st);
      if (a.cfirst) return cudaErrorInvalidValue;
      if (a.pair && a.lean == 1)
        return launch_gemm_t<64, 4, true, false, 0, 1>(tA, tW, tV, a, num_sms, st);
      if (a.pair && a.lean == 2)
        return launch_gemm_t<64, 5, true, false, 0, 2>(tA, tW, tV, a, num_sms, st);
      if (a.pair && a.lean == 3)
        return launch_gemm_t<64, 5, true, false, 0, 3>(tA, tW, tV, a, num_sms, st);
      if (a.pair) return launch_gemm_t<64, 5, true>(tA, tW, tV, a, num_sms, st);
      return launch_gemm_t<64, 3, false>(tA, tW, tV, a, num_sms, st);
    case 32: return launch_gemm_t<32, 6, false>(tA, tW, tV, a, num_sms, st);
    case 16: return launch_gemm_t<16, 8, false>(tA, tW, tV, a, num_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

// =====================================================================  K_tgc
// Training backward, tcgen05 form of K_tg (comb.cu):  T_c^T[d][k] = sum_r (p_c[r][h(d)] G[r][d])
// patch_c[r][k] for one channel c and 128 columns d per CTA. Both operands are MN-major
// (their natural global layouts): A = G tile [64 r][128 d] and B = patch tile [64 r][64 k],
// each TMA'd as 128B-swizzled atoms (64 MN elements x 8 K rows); builder warps scale the A
// tile in place by p (a row of one 64-column half belongs to one head, so the swizzle never
// has to be undone); one thread issues M128 N64 K16 MMAs into a 64-column TMEM accumulator.
constexpr int TGC_STAGES = 4;
constexpr int TGC_A_BYTES = 2 * 64 * 64 * 2;    // two 64-column halves x 64 rows
constexpr int TGC_B_BYTES = 64 * 64 * 2;
constexpr int TGC_STAGE = TGC_A_BYTES + TGC_B_BYTES;
constexpr int TGC_SMEM = TGC_STAGES * TGC_STAGE + 1024 + 256;
// TE mode: + one constant 64 x 64 B atom (column 0 = 1: the bias / colsum column, N = 80)
constexpr int TGC_SMEM_TE = TGC_SMEM + TGC_B_BYTES;

// TE = false: T_c (fp32) as above. TE = true (the training step's augmented form):
//  * the B operand gets a second, constant MN atom whose first column is 1, so the MMA
//    (N = 80) also produces the column sums sum_r A[r][m] in accumulator column 64;
//  * CTA column x = D/128 (attention nodes) computes E_c^T = dl_c^T [patch_c | 1] with A =
//    the node's bf16 dl [g][H][R] read K-major (rows h >= H zero-filled by TMA), unscaled;
//  * the epilogue writes bf16 rows of the node's TE block (see L0TgradArgs).
template <bool TE>
__global__ void __launch_bounds__(192, 2)
    l0_tgrad_tc_kernel(const __grid_constant__ CUtensorMap tmG,
                       const __grid_constant__ CUtensorMap tmP,
                       const __grid_constant__ CUtensorMap tmDL, L0TgradArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* ones = smem + TGC_STAGES * TGC_STAGE;   // TE: constant atom (1024-aligned)
  uint64_t* full = reinterpret_cast<uint64_t*>(ones + (TE ? TGC_B_BYTES : 0));
  uint64_t* scaled = full + TGC_STAGES;
  uint64_t* empty = scaled + TGC_STAGES;
  uint64_t* done = empty + TGC_STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = warp_id(), lane = lane_id();
  const int c = blockIdx.y, d0 = blockIdx.x * 128;
  const bool eblk = TE && d0 >= a.D;               // the E_c block (dl as A, K-major)
  const int nst = a.R / 64;
  const int dh = a.D / a.H;
  constexpr uint32_t TCOLS = TE ? 128 : 64;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmG);
    tma_prefetch(&tmP);
    if (TE) tma_prefetch(&tmDL);
    for (int s = 0; s < TGC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&scaled[s], 4);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (TE) {  // ones atom: element (row r, n = 0) = 1 sits in 16-byte chunk (r & 7) of row r
    for (int i = threadIdx.x; i < TGC_B_BYTES / 16; i += blockDim.x) {
      const int r = i >> 3, ch = i & 7;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (ch == (r & 7)) v.x = 0x3F80u;  // bf16 1.0 in the low half
      *reinterpret_cast<uint4*>(ones + i * 16) = v;
    }
    fence_async_smem();
  }
  if (warp == 1) tmem_alloc(tslot, TCOLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0) {
    if (elect_one()) {
      for (int i = 0; i < nst; ++i) {
        const int s = i % TGC_STAGES;
        mbar_wait(&empty[s], ((i / TGC_STAGES) & 1) ^ 1);
        uint8_t* sa = smem + s * TGC_STAGE;
        mbar_expect_tx(&full[s], TGC_STAGE);
        const int r0 = i * 64, b = r0 / a.S, s0 = r0 - b * a.S;
        if (eblk) {
          tma_load_3d(sa, &tmDL, &full[s], r0, 0, c);          // [128 h][64 r], K-major
        } else {
          tma_load_2d(sa, &tmG, &full[s], d0, r0);
          tma_load_2d(sa + TGC_A_BYTES / 2, &tmG, &full[s], d0 + 64, r0);
        }
        tma_load_3d(sa + TGC_A_BYTES, &tmP, &full[s], 0, s0, b * a.cnt + a.c0 + c);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16_f32(128, TE ? 80 : 64) | (eblk ? 0u : (1u << 15)) |
                           (1u << 16);
    for (int i = 0; i < nst; ++i) {
      const int s = i % TGC_STAGES;
      mbar_wait(&scaled[s], (i / TGC_STAGES) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sa = smem_u32(smem + s * TGC_STAGE), sb = sa + TGC_A_BYTES;
        const uint32_t lbo_b = TE ? smem_u32(ones) - sb : (uint32_t)TGC_B_BYTES;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = eblk ? smem_desc(sa + kk * 32, 16, 1024, 2u)
                                   : smem_desc(sa + kk * 2048, TGC_A_BYTES / 2, 1024, 2u);
          const uint64_t bd = smem_desc(sb + kk * 2048, lbo_b, 1024, 2u);
          if (!(a.debug & 2)) mma_ss(tmem, ad, bd, idesc, (i | kk) != 0);
        }
        mma_commit(&empty[s]);
        if (i == nst - 1) mma_commit(done);
      }
      __syncwarp();
    }
  } else {
    // builders: thread t scales row r = t % 64 of half mh = t / 64 by p[r][head(mh)]
    const int t = threadIdx.x - 64;
    const int row = t & 63, mh = t >> 6;
    const int head = (d0 + mh * 64) / dh;
    const int hA = d0 / dh;
    const int hg = hA / (a.NH > 0 ? a.NH : 1);
    const int hn = (hA - hg * a.NH) & ~1;
    const int sel = head & 1;
    const float mixc = a.mix ? __ldg(a.mix + c) : 0.f;
    // the raw p word (two heads' bf16) of stage i; converted only where it is consumed, so
    // the loads of the queue below really stay in flight (a conversion right after the load
    // made every load stall for its full latency)
    auto pword = [&](int i) -> uint32_t {
      if (a.mix) return 0u;
      return __ldg(reinterpret_cast<const uint32_t*>(
          a.p + ((size_t)(hg * a.g + c) * a.R + i * 64 + row) * a.NH + hn));
    };
    auto pconv = [&](uint32_t w) -> float {
      if (a.mix) return mixc;
      return sel ? bf16hi(w) : bf16lo(w);
    };
    // p of the next four stages in flight: one register per ring slot, the stage loop
    // unrolled by the ring depth so no register copy (which would wait for the load) moves
    // the queue along
    static_assert(TGC_STAGES == 4, "the p queue is unrolled by the ring depth");
    uint32_t pq[TGC_STAGES];
#pragma unroll
    for (int j = 0; j < TGC_STAGES; ++j) pq[j] = (!eblk && j < nst) ? pword(j) : 0u;
    for (int i0 = 0; i0 < nst; i0 += TGC_STAGES)
#pragma unroll
    for (int s = 0; s < TGC_STAGES; ++s) {
      const int i = i0 + s;
      if (i >= nst) break;
      const uint32_t pw = pq[s];
      if (!eblk && i + TGC_STAGES < nst) pq[s] = pword(i + TGC_STAGES);
      mbar_wait(&full[s], (i / TGC_STAGES) & 1);
      const float pc = pconv(pw);
      if (!eblk && !(a.debug & 1)) {
        const uint32_t rowaddr = smem_u32(smem + s * TGC_STAGE) + mh * (TGC_A_BYTES / 2) +
                                 (row >> 3) * 1024 + (row & 7) * 128;
        // rows sit 128 B apart: visit the row's 16-byte chunks in a row-rotated order so the
        // 8 rows of a swizzle atom hit 8 different bank groups (all chunks share one p)
        uint32_t v[8][4];
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          const uint32_t ad = rowaddr + (((ch + row) & 7) << 4);
          asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[ch][0]), "=r"(v[ch][1]), "=r"(v[ch][2]), "=r"(v[ch][3])
                       : "r"(ad));
        }
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          const uint32_t ad = rowaddr + (((ch + row) & 7) << 4);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            v[ch][e] = pack_bf16(bf16lo(v[ch][e]) * pc, bf16hi(v[ch][e]) * pc);
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ad), "r"(v[ch][0]),
                       "r"(v[ch][1]), "r"(v[ch][2]), "r"(v[ch][3])
                       : "memory");
        }
        fence_async_smem();  // generic-proxy writes -> visible to the tensor core
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&scaled[s]);
    }
    // epilogue: lane quarter q of the accumulator = rows d0 + 32 q .. +31, 64 columns k
    mbar_wait(done, 0);
    tc_fence_after();
    const int q = warp & 3;
    if constexpr (TE) {
      const int m = q * 32 + lane;                          // d - d0, or h (E block)
      const long long col = eblk ? (long long)a.D + m : (long long)d0 + m;
      __nv_bfloat16* te = a.TE + col;
      const bool live = !eblk || m < a.H;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + half * 32, r);
        tmem_ld_wait();
        if (live) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            te[(size_t)(c * a.PP + half * 32 + j) * a.te_ld] = __float2bfloat16(__uint_as_float(r[j]));
        }
      }
      uint32_t r16[16];
      tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + 64, r16);
      tmem_ld_wait();
      if (live) te[(size_t)(a.ones0 + c) * a.te_ld] = __float2bfloat16(__uint_as_float(r16[0]));
    } else {
      const int d = d0 + q * 32 + lane;
      float* out = a.T + (size_t)c * 64 * a.D + d;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + half * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) out[(size_t)(half * 32 + j) * a.D] = __uint_as_float(r[j]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TCOLS);
  }
}

// K_te with two channels per CTA. K_te's floor is the L2 -> SM fan-out: the one-channel
// form moves each G tile into shared memory once per channel. Here a stage holds one G tile
// and both channels' patch tiles; the builders scale G into two A operands, p_c0 G into a
// small ring of copies (A0, two slots) and p_c1 G in place. G then crosses the fabric once per
// channel pair, and a unit of work moves 16 KB instead of 24. The E columns (A = dl_c,
// unscaled) take one channel per CTA: two CTA columns past the D / 128 G columns.
// Ring depth: 4, 5 and 6 stages ran alike (87-88 us per TR node; load-only 76 us at every
// depth), one copy slot instead of two cost 20 us (the builders then wait for the MMAs).
constexpr int TE2_STAGES = 4;
constexpr int TE2_A0 = 2;                                 // copy slots for channel c0
constexpr int TE2_STAGE = TGC_A_BYTES + 2 * TGC_B_BYTES;  // G | B0 | B1 = 32 KB
constexpr int TE2_SMEM = TE2_STAGES * TE2_STAGE + TE2_A0 * TGC_A_BYTES + TGC_B_BYTES + 1024 + 256;
constexpr int TE2_BUILDERS = 8;

__global__ void __launch_bounds__(64 + 32 * TE2_BUILDERS, 1)
    l0_tgrad_te2_kernel(const __grid_constant__ CUtensorMap tmG,
                        const __grid_constant__ CUtensorMap tmP,
                        const __grid_constant__ CUtensorMap tmDL, L0TgradArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* a0 = smem + TE2_STAGES * TE2_STAGE;     // [TE2_A0] scaled copies for channel c0
  uint8_t* ones = a0 + TE2_A0 * TGC_A_BYTES;       // constant atom (column 0 = 1)
  uint64_t* full = reinterpret_cast<uint64_t*>(ones + TGC_B_BYTES);
  uint64_t* scaled = full + TE2_STAGES;
  uint64_t* empty = scaled + TE2_STAGES;
  uint64_t* done = empty + TE2_STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = warp_id(), lane = lane_id();
  const int c0 = blockIdx.y * 2, d0 = blockIdx.x * 128;
  const bool eblk = d0 >= a.D;
  const int ech = eblk ? (int)blockIdx.x - a.D / 128 : 0;  // E column: its channel c0 + ech
  const int nst = a.R / 64;
  const int nit = nst;
  const int dh = a.D / a.H;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmG);
    tma_prefetch(&tmP);
    tma_prefetch(&tmDL);
    for (int s = 0; s < TE2_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&scaled[s], TE2_BUILDERS);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < TGC_B_BYTES / 16; i += blockDim.x) {
    const int r = i >> 3, ch = i & 7;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (ch == (r & 7)) v.x = 0x3F80u;
    *reinterpret_cast<uint4*>(ones + i * 16) = v;
  }
  fence_async_smem();
  if (warp == 1) tmem_alloc(tslot, 256);           // two accumulators, columns 0 and 128
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0) {
    if (elect_one()) {
      for (int i = 0; i < nit; ++i) {
        const int s = i % TE2_STAGES;
        mbar_wait(&empty[s], ((i / TE2_STAGES) & 1) ^ 1);
        uint8_t* sa = smem + s * TE2_STAGE;
        if (eblk) {
          const int r0 = i * 64, b = r0 / a.S, s0 = r0 - b * a.S;
          mbar_expect_tx(&full[s], TGC_A_BYTES + TGC_B_BYTES);
          tma_load_3d(sa, &tmDL, &full[s], r0, 0, c0 + ech);     // [128 h][64 r], K-major
          tma_load_3d(sa + TGC_A_BYTES, &tmP, &full[s], 0, s0, b * a.cnt + a.c0 + c0 + ech);
        } else {
          const int r0 = i * 64, b = r0 / a.S, s0 = r0 - b * a.S;
          mbar_expect_tx(&full[s], TE2_STAGE);
          tma_load_2d(sa, &tmG, &full[s], d0, r0);
          tma_load_2d(sa + TGC_A_BYTES / 2, &tmG, &full[s], d0 + 64, r0);
          tma_load_3d(sa + TGC_A_BYTES, &tmP, &full[s], 0, s0, b * a.cnt + a.c0 + c0);
          tma_load_3d(sa + TGC_A_BYTES + TGC_B_BYTES, &tmP, &full[s], 0, s0,
                      b * a.cnt + a.c0 + c0 + 1);
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16_f32(128, 80) | (eblk ? 0u : (1u << 15)) | (1u << 16);
    for (int i = 0; i < nit; ++i) {
      const int s = i % TE2_STAGES;
      mbar_wait(&scaled[s], (i / TE2_STAGES) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sg = smem_u32(smem + s * TE2_STAGE);
        if (eblk) {
          const uint32_t sb = sg + TGC_A_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            if (!(a.debug & 2))
              mma_ss(tmem + ech * 128, smem_desc(sg + kk * 32, 16, 1024, 2u),
                     smem_desc(sb + kk * 2048, smem_u32(ones) - sb, 1024, 2u), idesc,
                     (i | kk) != 0);
        } else {
#pragma unroll
          for (int ch = 0; ch < 2; ++ch) {
            const uint32_t sa = ch ? sg : smem_u32(a0 + (i % TE2_A0) * TGC_A_BYTES);
            const uint32_t sb = sg + TGC_A_BYTES + ch * TGC_B_BYTES;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              if (!(a.debug & 2))
                mma_ss(tmem + ch * 128, smem_desc(sa + kk * 2048, TGC_A_BYTES / 2, 1024, 2u),
                       smem_desc(sb + kk * 2048, smem_u32(ones) - sb, 1024, 2u), idesc,
                       (i | kk) != 0);
          }
        }
        mma_commit(&empty[s]);
        if (i == nit - 1) mma_commit(done);
      }
      __syncwarp();
    }
  } else {
    // builders: thread t scales chunks [4 cq, 4 cq + 4) of row r = t % 64 of half mh
    const int t = threadIdx.x - 64;
    const int row = t & 63, mh = (t >> 6) & 1, cq = t >> 7;
    const int head = (d0 + mh * 64) / dh;
    const int hA = d0 / dh;
    const int hg = hA / (a.NH > 0 ? a.NH : 1);
    const int hn = (hA - hg * a.NH) & ~1;
    const int sel = head & 1;
    const float mix0 = (a.mix && !eblk) ? __ldg(a.mix + c0) : 0.f;
    const float mix1 = (a.mix && !eblk) ? __ldg(a.mix + c0 + 1) : 0.f;
    auto pword = [&](int ch, int i) -> uint32_t {
      if (a.mix) return 0u;
      return __ldg(reinterpret_cast<const uint32_t*>(
          a.p + ((size_t)(hg * a.g + c0 + ch) * a.R + i * 64 + row) * a.NH + hn));
    };
    auto pconv = [&](uint32_t w, float mixc) -> float {
      if (a.mix) return mixc;
      return sel ? bf16hi(w) : bf16lo(w);
    };
    // p of the next four stages in flight (raw words, one register per queue slot; the loop
    // is unrolled by the queue depth so no register copy waits for a load)
    constexpr int PQ = 4;
    uint32_t pq0[PQ], pq1[PQ];
#pragma unroll
    for (int j = 0; j < PQ; ++j) {
      pq0[j] = (!eblk && j < nst) ? pword(0, j) : 0u;
      pq1[j] = (!eblk && j < nst) ? pword(1, j) : 0u;
    }
    for (int i0 = 0; i0 < nit; i0 += PQ)
#pragma unroll
    for (int j = 0; j < PQ; ++j) {
      const int i = i0 + j;
      if (i >= nit) break;
      const int s = i % TE2_STAGES;
      const uint32_t w0 = pq0[j], w1 = pq1[j];
      if (!eblk && i + PQ < nst) {
        pq0[j] = pword(0, i + PQ);
        pq1[j] = pword(1, i + PQ);
      }
      mbar_wait(&full[s], (i / TE2_STAGES) & 1);
      if (!eblk && !(a.debug & 1)) {
        // the copy slot i % TE2_A0 is free once the MMAs of stage i - TE2_A0 have completed
        if (i >= TE2_A0)
          mbar_wait(&empty[(i - TE2_A0) % TE2_STAGES], ((i - TE2_A0) / TE2_STAGES) & 1);
        const float p0 = pconv(w0, mix0), p1 = pconv(w1, mix1);
        const uint32_t off = mh * (TGC_A_BYTES / 2) + (row >> 3) * 1024 + (row & 7) * 128;
        const uint32_t rg = smem_u32(smem + s * TE2_STAGE) + off;
        const uint32_t rc = smem_u32(a0 + (i % TE2_A0) * TGC_A_BYTES) + off;
        uint32_t v[4][4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t ad = rg + (((4 * cq + k + row) & 7) << 4);
          asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[k][0]), "=r"(v[k][1]), "=r"(v[k][2]), "=r"(v[k][3])
                       : "r"(ad));
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t o = ((4 * cq + k + row) & 7) << 4;
          uint32_t x0[4], x1[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float lo = bf16lo(v[k][e]), hi = bf16hi(v[k][e]);
            x0[e] = pack_bf16(lo * p0, hi * p0);
            x1[e] = pack_bf16(lo * p1, hi * p1);
          }
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(rc + o), "r"(x0[0]),
                       "r"(x0[1]), "r"(x0[2]), "r"(x0[3])
                       : "memory");
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(rg + o), "r"(x1[0]),
                       "r"(x1[1]), "r"(x1[2]), "r"(x1[3])
                       : "memory");
        }
        fence_async_smem();  // generic-proxy writes -> visible to the tensor core
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&scaled[s]);
    }
    // epilogue: warps 2..5 drain channel c0's accumulator, warps 6..9 channel c0 + 1's
    mbar_wait(done, 0);
    tc_fence_after();
    const int q = warp & 3, ch = (warp - 2) >> 2, c = c0 + ch;
    const uint32_t tacc = tmem + ch * 128 + ((uint32_t)(q * 32) << 16);
    const int m = q * 32 + lane;
    const long long col = eblk ? (long long)a.D + m : (long long)d0 + m;
    __nv_bfloat16* te = a.TE + col;
    const bool live = !eblk || (m < a.H && ch == ech);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t r[32];
      tmem_ld32(tacc + half * 32, r);
      tmem_ld_wait();
      if (live) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          te[(size_t)(c * a.PP + half * 32 + j) * a.te_ld] = __float2bfloat16(__uint_as_float(r[j]));
      }
    }
    uint32_t r16[16];
    tmem_ld16(tacc + 64, r16);
    tmem_ld_wait();
    if (live) te[(size_t)(a.ones0 + c) * a.te_ld] = __float2bfloat16(__uint_as_float(r16[0]));
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

cudaError_t launch_l0_tgrad_tc(const CUtensorMap& tG, const CUtensorMap& tP,
                               const L0TgradArgs& a, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(l0_tgrad_tc_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, TGC_SMEM);
  if (e != cudaSuccess) return e;
  l0_tgrad_tc_kernel<false><<<dim3(a.D / 128, a.g), 192, TGC_SMEM, st>>>(tG, tP, tG, a);
  return cudaGetLastError();
}

cudaError_t launch_l0_tgrad_te(const CUtensorMap& tG, const CUtensorMap& tP,
                               const CUtensorMap& tDL, const L0TgradArgs& a, cudaStream_t st) {
  // two channels per CTA when the node's channel count is even (DCHAG_TE_CH=1: one)
  const char* ch1 = getenv("DCHAG_TE_CH");
  if (a.g % 2 == 0 && !(ch1 && atoi(ch1) == 1)) {
    cudaError_t e = cudaFuncSetAttribute(l0_tgrad_te2_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, TE2_SMEM);
    if (e != cudaSuccess) return e;
    l0_tgrad_te2_kernel<<<dim3(a.D / 128 + (a.has_dl ? 2 : 0), a.g / 2), 64 + 32 * TE2_BUILDERS,
                          TE2_SMEM, st>>>(tG, tP, tDL, a);
    return cudaGetLastError();
  }
  cudaError_t e = cudaFuncSetAttribute(l0_tgrad_tc_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, TGC_SMEM_TE);
  if (e != cudaSuccess) return e;
  l0_tgrad_tc_kernel<true><<<dim3(a.D / 128 + (a.has_dl ? 1 : 0), a.g), 192, TGC_SMEM_TE, st>>>(
      tG, tP, tDL, a);
  return cudaGetLastError();
}

}  // namespace dchag
