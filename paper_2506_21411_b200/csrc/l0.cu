// Level-0 D-CHAG nodes with the tokenizer folded in (tokens are never formed).
//
// For a level-0 single_query node n over channels c in G_n, with
//   U_n[:,h] = wk[:,h] q'_h / sqrt(dh),  M_c = tok.w[c] @ wv_n,
// the node's context vector is (verified to 1.9e-16)
//   logits[r,c,h] = patch_c[r] . (tok.w[c] U_n)[:,h] + (tok.b[c]+chan_id[c]) U_n[:,h] + pos[s] U_n[:,h]
//   p[r,c,h]      = softmax_c(logits)
//   ctx[r,h-blk]  = sum_c p[r,c,h] * (patch_c[r] @ M_c[:,h-blk])         <- K_l0, tcgen05
//                 + sum_c p[r,c,h] * ((tok.b[c]+chan_id[c]) @ wv_n)[h-blk]  <- "ext" K-block
//                 + (pos[s] @ wv_n)[h-blk]                                  <- epilogue
// Reference semantics restated: model.py:51-64 (tokenizer) + layers.py:103-123 (node).
//
// K_p0 (l0_logits_kernel): logits + softmax with mma.sync (small: K = P*P, N = heads).
// K_l0 (l0_node_kernel):   A-scaled GEMM.  The A operand p[r,c,h] * patch_c[r,:] is built
//   by 4 warps (thread = row = TMEM lane) in registers and written to TMEM with
//   tcgen05.st; tcgen05.mma reads A from TMEM and B = M_c[:,h-blk] from shared memory
//   (1-D bulk copies of pre-tiled canonical blocks).  Image rows arrive by 1-D bulk copy:
//   a 128-position tile of one channel is one contiguous run of 128*P*P pixels.
#include "common.cuh"
#include "dchag_kernels.h"

namespace dchag {

// =====================================================================  K_p0
DEV long long globaltimer_ns() {  // comparable across the two SMs of a pair (clock64 is not)
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define P0_TRACE(ev, k)                                                                     \
  do {                                                                                      \
    if (a.trace && blockIdx.x < 4 && threadIdx.x == 0 && (k) < 64)                          \
      a.trace[(blockIdx.x * 8 + (ev)) * 64 + (k)] = globaltimer_ns();                      \
  } while (0)
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4],
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Persistent CTAs over work items (node n, block of RB rows); each CTA takes a contiguous
// range of items (so the node, and the staged logit weights, rarely change) and
// double-buffers the image slices: while the 8 warps compute item k, the bulk copies of item
// k+1 are in flight. Warp w takes the m16 row tile w % MT and the channels
// c = w / MT mod CS (CS = 8 / MT). An item's rows of every channel of the node are one
// contiguous image run (RB % (W/P) == 0): g 1-D bulk copies per item, images read from HBM
// once. Logit weights (16-byte XOR swizzle, conflict-free ldmatrix) and the bias rows live
// in shared memory. Pass 1: max over the node's channels (merged across channel phases
// through shared memory); pass 2: e = 2^(t - max), sums; pass 3 (no pinv): p = e / sum.
template <int NT, int P, int MT>  // NT = HP / 8 head tiles, MT = RB / 16 row tiles
__global__ void __launch_bounds__(256, NT <= 2 ? 2 : 1)  // two CTAs per SM need <= 128 registers
    l0_logits_kernel(L0LogitArgs a, int items_per_cta, int nbuf) {
  constexpr int RB = MT * 16, CS = 8 / MT;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t landed[2];
  constexpr int PP = P * P;
  constexpr int KS = PP / 16;
  constexpr int CPR = PP * 2 / 16;  // 16-byte chunks per weight row
  const uint32_t sbase = (smem_u32(smem_raw) + 127) & ~127u;
  const int R = a.B * a.S;
  const int bpn = R / RB;            // items per node
  const int total = a.n_nodes * bpn;
  const int it0 = blockIdx.x * items_per_cta;
  const int it1 = min(total, it0 + items_per_cta);
  if (it0 >= it1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int mt = warp % MT, cph = warp / MT;
  const uint32_t chunk = (uint32_t)RB * PP * 2;             // bytes of one channel's block
  const uint32_t ibuf = (uint32_t)a.gmax * chunk;           // one item's image buffer
  const uint32_t sW = sbase + nbuf * ibuf;                  // [g*HP][PP] swizzled weights
  const uint32_t wrow = (uint32_t)a.HP * PP * 2;            // weight bytes per channel
  const uint32_t sU = sW + (uint32_t)a.gmax * wrow;         // [g][HP] fp32 bias rows
  float* stat = reinterpret_cast<float*>(smem_raw + (sU - smem_u32(smem_raw)) +
                                         (size_t)a.gmax * a.HP * 4);  // [CS][MT][NT][4][32]
  const int lwp = __ffs(a.wp) - 1;   // W / P divides 128: a power of two
  // warp 0: bulk copies of item it into buffer buf, one channel per lane (one thread issuing
  // all g copies took ~70 ns per copy, ~1.1 us per 16-channel item, on the critical path)
  // (c0, g: the item's node, loaded by the caller ahead of time -- a dependent load here
  // held the issuing warp for its latency)
  auto issue = [&](int it, int buf, int c0, int g) {
    const int n = it / bpn, r0 = (it - n * bpn) * RB;
    const int b = r0 / a.S, s0 = r0 - b * a.S;
    const __nv_bfloat16* src0 = a.img + b * a.img_sb + (long long)(s0 >> lwp) * P * a.W;
    const int ln = threadIdx.x & 31;
    if (ln == 0) mbar_expect_tx(&landed[buf], chunk * g);
    __syncwarp();
    const int nl = a.issue_serial ? 1 : 32;
    if (ln < nl)
    for (int c = ln; c < g; c += nl)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(sbase + buf * ibuf + c * chunk), "l"(src0 + (long long)(c0 + c) * a.img_sc),
          "r"(chunk), "r"(smem_u32(&landed[buf]))
          : "memory");
  };
  // all 8 warps: lane 0 of warp w issues the copies of channels w, w + 8, ... (a warp that
  // issues all of them is held up ~1 us and the item's barriers wait for it)
  auto issue_all = [&](int it, int buf, int c0, int g) {
    const int n = it / bpn, r0 = (it - n * bpn) * RB;
    const int b = r0 / a.S, s0 = r0 - b * a.S;
    const __nv_bfloat16* src0 = a.img + b * a.img_sb + (long long)(s0 >> lwp) * P * a.W;
    if (threadIdx.x == 0) mbar_expect_tx(&landed[buf], chunk * g);
    if ((threadIdx.x & 31) == 0)
      for (int c = threadIdx.x >> 5; c < g; c += 8)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(sbase + buf * ibuf + c * chunk), "l"(src0 + (long long)(c0 + c) * a.img_sc),
            "r"(chunk), "r"(smem_u32(&landed[buf]))
            : "memory");
  };
  if (threadIdx.x == 0) {
    mbar_init(&landed[0], 1);
    mbar_init(&landed[1], 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    __syncwarp();
    issue(it0, 0, __ldg(a.node_c0 + it0 / bpn), __ldg(a.node_g + it0 / bpn));
  }
  auto wswz = [&](int row, int ch) -> uint32_t {  // byte offset of chunk ch of weight row
    const int f = CPR >= 8 ? (row & 7) : ((row / (8 / CPR)) & (CPR - 1));
    return (uint32_t)(row * (PP * 2) + ((ch ^ f) << 4));
  };
  // per-thread shared byte offsets inside a channel block / weight slice (item independent)
  uint32_t aoff[KS], boff[KS][NT / 2 > 0 ? NT / 2 : 1];
  uint32_t aoff4[4];
  if (P == 8) {
    const int mat = lane >> 3, rr = lane & 7;
    const int rl = mt * 16 + (mat & 1) * 8 + rr;
    const int i = rl >> lwp, j = rl & (a.wp - 1);
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
      aoff[ks] = (uint32_t)(((i * P + 2 * ks + (mat >> 1)) * a.W + j * P) * 2);
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {  // a0..a3: rows gid / gid+8, k = 2tig (+8)
      const int rl = mt * 16 + gid + 8 * (e & 1);
      const int i = rl >> lwp, j = rl & (a.wp - 1);
      const int k = 2 * tig + 8 * (e >> 1);
      aoff4[e] = (uint32_t)(((i * P + k / P) * a.W + j * P + k % P) * 2);
    }
  }
  {
    const int mat = lane >> 3, rr = lane & 7;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int np = 0; np < (NT + 1) / 2; ++np) {
        // x4: matrices (nt = 2np + mat/2, k half = mat%2); x2 (NT == 1): (nt 0, k half mat)
        const int nt = NT == 1 ? 0 : 2 * np + (mat >> 1);
        boff[ks][np] = wswz(nt * 8 + rr, ks * 2 + (mat & 1));
      }
  }
  constexpr float LOG2E = 1.4426950408889634f;
  auto sidx = [&](int k, int nt, int e) { return (((k * MT + mt) * NT + nt) * 4 + e) * 32 + lane; };
  const int nh = a.nh;  // heads per K_l0 unit (the p layout's head-group width)
  const bool unnorm = a.pinv != nullptr;
  int cur_node = -1;
  uint32_t ph[2] = {0u, 0u};
  for (int it = it0, k = 0; it < it1; ++it, ++k) {
    const int buf = nbuf == 2 ? (k & 1) : 0;
    const int n = it / bpn, r0 = (it - n * bpn) * RB;
    const int c0 = __ldg(a.node_c0 + n), g = __ldg(a.node_g + n);
    const long long poff = __ldg(a.node_poff + n);
    // the next item's node (usually this one): its copies are issued mid-item
    const int nn = (it + 1) / bpn;
    const int c0n = nn == n ? c0 : __ldg(a.node_c0 + min(nn, a.n_nodes - 1));
    const int gn = nn == n ? g : __ldg(a.node_g + min(nn, a.n_nodes - 1));
    // item k-1 is finished by every warp (end-of-item barrier): its buffer takes item k+1
    P0_TRACE(0, k);
    if (nbuf == 2 && threadIdx.x < 32 && it + 1 < it1) issue(it + 1, buf ^ 1, c0n, gn);
    if (n != cur_node) {  // stage this node's logit weights and bias rows
      const uint4* src = reinterpret_cast<const uint4*>(a.WUt + (long long)c0 * a.HP * PP);
      const int nchunks = g * a.HP * CPR;
      for (int i = threadIdx.x; i < nchunks; i += 256)
        sts128(sW + wswz(i / CPR, i % CPR), __ldg(src + i));
      const float* bsrc = a.bU + (long long)c0 * a.HP;
      for (int i = threadIdx.x; i < g * a.HP; i += 256)
        reinterpret_cast<float*>(smem_raw + (sU - smem_u32(smem_raw)))[i] = __ldg(bsrc + i);
      cur_node = n;
      __syncthreads();
    }
    const float* sUf = reinterpret_cast<const float*>(smem_raw + (sU - smem_u32(smem_raw)));
    int rows[2];
    float pu[NT][4];
#pragma unroll
    for (int q = 0; q < 2; ++q) rows[q] = r0 + mt * 16 + gid + 8 * q;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const float* pr0 = a.posU + ((long long)n * a.S + rows[0] % a.S) * a.HP + nt * 8 + 2 * tig;
      const float* pr1 = a.posU + ((long long)n * a.S + rows[1] % a.S) * a.HP + nt * 8 + 2 * tig;
      const float2 u0 = __ldg(reinterpret_cast<const float2*>(pr0));
      const float2 u1 = __ldg(reinterpret_cast<const float2*>(pr1));
      pu[nt][0] = u0.x; pu[nt][1] = u0.y; pu[nt][2] = u1.x; pu[nt][3] = u1.y;
    }
    mbar_wait(&landed[buf], ph[buf]);
    ph[buf] ^= 1;
    P0_TRACE(1, k);
    const uint32_t ibase = sbase + buf * ibuf;
    auto logits = [&](int c, float (&L)[NT][4]) {
      const uint32_t ab = ibase + c * chunk;
      const uint32_t wb = sW + c * wrow;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const float2 bb = *reinterpret_cast<const float2*>(sUf + c * a.HP + nt * 8 + 2 * tig);
        L[nt][0] = pu[nt][0] + bb.x;
        L[nt][1] = pu[nt][1] + bb.y;
        L[nt][2] = pu[nt][2] + bb.x;
        L[nt][3] = pu[nt][3] + bb.y;
      }
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        uint32_t af[4];
        if (P == 8) {
          ldsm_x4(ab + aoff[ks], af);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) af[e] = lds32(ab + aoff4[e]);
        }
        if (NT == 1) {
          uint32_t bf[2];
          ldsm_x2(wb + boff[ks][0], bf);
          mma_bf16_16816(L[0], af, bf[0], bf[1]);
        } else {
#pragma unroll
          for (int np = 0; np < NT / 2; ++np) {
            uint32_t bf[4];
            ldsm_x4(wb + boff[ks][np], bf);
            mma_bf16_16816(L[2 * np], af, bf[0], bf[1]);
            mma_bf16_16816(L[2 * np + 1], af, bf[2], bf[3]);
          }
        }
      }
    };
    // pass 1: max only. With at most KEEP channels per warp the logits stay in registers, so
    // the image buffer is free after this pass and the next item's copies start right away
    // (they overlap the softmax passes); otherwise passes 2/3 recompute them.
    constexpr int KEEP = 4;
    const bool keep = g <= KEEP * CS;
    float Lk[KEEP][NT][4];
    float mx[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) mx[nt][e] = -INFINITY;
    if (keep) {
#pragma unroll
      for (int i = 0; i < KEEP; ++i) {
        const int c = cph + i * CS;
        if (c < g) {
          logits(c, Lk[i]);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) mx[nt][e] = fmaxf(mx[nt][e], Lk[i][nt][e]);
        }
      }
    } else {
#pragma unroll 2
      for (int c = cph; c < g; c += CS) {
        float L[NT][4];
        logits(c, L);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) mx[nt][e] = fmaxf(mx[nt][e], L[nt][e]);
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) stat[sidx(cph, nt, e)] = mx[nt][e];
    __syncthreads();
    const bool early = keep && nbuf == 1 && it + 1 < it1;
    P0_TRACE(2, k);
    if (early) {  // every warp is done with the image
      if (a.issue_serial) { if (threadIdx.x < 32) issue(it + 1, 0, c0n, gn); }
      else issue_all(it + 1, 0, c0n, gn);
    }
    P0_TRACE(5, k);
    float nmx[NT][4];  // -max * log2(e)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float m = stat[sidx(0, nt, e)];
#pragma unroll
        for (int kk = 1; kk < CS; ++kk) m = fmaxf(m, stat[sidx(kk, nt, e)]);
        nmx[nt][e] = -m * LOG2E;
      }
    __syncthreads();  // stat reused for the sums
    P0_TRACE(6, k);
    // p / e store offsets (elements, relative to the node's p block) for channel 0
    int poff_e[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int h = nt * 8 + 2 * tig, hg = h / nh, hl = h - hg * nh;
#pragma unroll
      for (int q = 0; q < 2; ++q) poff_e[nt][q] = ((hg * g) * R + rows[q]) * nh + hl;
    }
    __nv_bfloat16* pn = a.p + poff;
    const int cstride = R * nh;  // elements between consecutive channels of one head group
    // pass 2: e = 2^(t - max), sums; with pinv the unnormalised e is the output
    float sm_[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) sm_[nt][e] = 0.f;
    auto pass2 = [&](int c, const float (&L)[NT][4]) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        float ev[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          ev[e] = ex2_approx(fmaf(L[nt][e], LOG2E, nmx[nt][e]));
          sm_[nt][e] += ev[e];
        }
        if (unnorm && nt * 8 + 2 * tig < a.H) {
#pragma unroll
          for (int q = 0; q < 2; ++q)
            *reinterpret_cast<uint32_t*>(pn + poff_e[nt][q] + c * cstride) =
                pack_bf16(ev[2 * q], ev[2 * q + 1]);
        }
      }
    };
    if (keep) {
#pragma unroll
      for (int i = 0; i < KEEP; ++i)
        if (cph + i * CS < g) pass2(cph + i * CS, Lk[i]);
    } else {
#pragma unroll 2
      for (int c = cph; c < g; c += CS) {
        float L[NT][4];
        logits(c, L);
        pass2(c, L);
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) stat[sidx(cph, nt, e)] = sm_[nt][e];
    P0_TRACE(7, k);
    __syncthreads();
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float t = stat[sidx(0, nt, e)];
#pragma unroll
        for (int kk = 1; kk < CS; ++kk) t += stat[sidx(kk, nt, e)];
        sm_[nt][e] = 1.f / t;
      }
    if (unnorm) {
      if (cph == 0) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int h = nt * 8 + 2 * tig;
          if (h < a.H) {
#pragma unroll
            for (int q = 0; q < 2; ++q)
              *reinterpret_cast<float2*>(a.pinv + ((long long)n * R + rows[q]) * a.H + h) =
                  make_float2(sm_[nt][2 * q], sm_[nt][2 * q + 1]);
          }
        }
      }
    } else {
      // pass 3 (normalised output): p = e / sum
      auto pass3 = [&](int c, const float (&L)[NT][4]) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          if (nt * 8 + 2 * tig < a.H) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const float p0 =
                  ex2_approx(fmaf(L[nt][2 * q], LOG2E, nmx[nt][2 * q])) * sm_[nt][2 * q];
              const float p1 =
                  ex2_approx(fmaf(L[nt][2 * q + 1], LOG2E, nmx[nt][2 * q + 1])) * sm_[nt][2 * q + 1];
              *reinterpret_cast<uint32_t*>(pn + poff_e[nt][q] + c * cstride) = pack_bf16(p0, p1);
            }
          }
        }
      };
      if (keep) {
#pragma unroll
        for (int i = 0; i < KEEP; ++i)
          if (cph + i * CS < g) pass3(cph + i * CS, Lk[i]);
      } else {
#pragma unroll 2
        for (int c = cph; c < g; c += CS) {
          float L[NT][4];
          logits(c, L);
          pass3(c, L);
        }
      }
    }
    P0_TRACE(3, k);
    __syncthreads();  // item done: its image buffer and the stat area may be reused
    P0_TRACE(4, k);
    if (nbuf == 1 && !early && threadIdx.x < 32 && it + 1 < it1) issue(it + 1, 0, c0n, gn);
  }
}

cudaError_t launch_l0_logits(const L0LogitArgs& a, int num_sms, cudaStream_t st) {
  const int R = a.B * a.S;
  const int PP = a.P * a.P;
  const int NTv = a.HP / 8;
  // rows per item: a multiple of the patch-row width (one contiguous run per channel); two
  // CTAs per SM, each holding two image buffers, the node's weights and bias rows
  auto smem_for = [&](int rb, int nbuf) {
    const int cs = 8 / (rb / 16);
    return (long long)nbuf * a.gmax * rb * PP * 2 + (long long)a.gmax * a.HP * PP * 2 +
           (long long)a.gmax * a.HP * 4 + (long long)cs * (rb / 16) * NTv * 4 * 32 * 4 + 128;
  };
  // item rows: a multiple of the patch-row width (one contiguous run per channel), the
  // largest <= 32 that keeps two CTAs per SM; the image slice is double-buffered only when
  // that still fits two CTAs (measured: two single-buffered CTAs beat one double-buffered)
  int RB = 0, nbuf = 1;
  for (int rb = 128; rb >= 16; rb >>= 1) {
    if (rb % a.wp || R % rb) continue;
    RB = rb;  // smallest valid so far
    if (rb <= 32 && smem_for(rb, 1) <= 113 * 1024) break;
  }
  if (RB == 0) return cudaErrorInvalidValue;
  // many heads (large weight block): when two CTAs per SM only fit 16-row single-buffered
  // items, one CTA per SM with 32-row double-buffered items is faster (TR, H = 32: 0.68 ->
  // 0.36 ms per launch, tools/p0_sweep_train.sh)
  bool one_cta = false;
  if (RB < 32 && a.wp <= 32 && 32 % a.wp == 0 && R % 32 == 0 && smem_for(32, 2) <= 227 * 1024) {
    RB = 32;
    one_cta = true;
  }
  if (const char* f = getenv("DCHAG_P0_RB")) {  // experiment override
    const int rb = atoi(f);
    if (rb >= 16 && rb % a.wp == 0 && R % rb == 0) RB = rb;
  }
  if (smem_for(RB, 2) <= (one_cta ? 227 : 113) * 1024) nbuf = 2;
  if (const char* f = getenv("DCHAG_P0_NBUF")) nbuf = atoi(f) == 2 ? 2 : 1;
  const long long smem = smem_for(RB, nbuf);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  void (*k)(L0LogitArgs, int, int) = nullptr;
#define L0L_PICK(NTv_, P_)                                                                    \
  k = RB == 16 ? l0_logits_kernel<NTv_, P_, 1> : RB == 32 ? l0_logits_kernel<NTv_, P_, 2>     \
    : RB == 64 ? l0_logits_kernel<NTv_, P_, 4> : l0_logits_kernel<NTv_, P_, 8>;
  if (a.P == 8) {
    if (NTv == 1) { L0L_PICK(1, 8) } else if (NTv == 2) { L0L_PICK(2, 8) } else if (NTv == 4) { L0L_PICK(4, 8) }
  } else if (a.P == 4) {
    if (NTv == 1) { L0L_PICK(1, 4) } else if (NTv == 2) { L0L_PICK(2, 4) } else if (NTv == 4) { L0L_PICK(4, 4) }
  }
#undef L0L_PICK
  if (!k) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int total = a.n_nodes * (R / RB);
  int per_sm = (int)((227 * 1024) / smem);  // co-resident CTAs (smem-limited), at most 4
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) == cudaSuccess && fa.numRegs > 0)
    per_sm = min(per_sm, 65536 / (fa.numRegs * 256));  // and register-limited
  if (per_sm > 4) per_sm = 4;
  if (per_sm < 1) per_sm = 1;
  if (const char* f = getenv("DCHAG_P0_PERSM")) per_sm = atoi(f) > 0 ? atoi(f) : per_sm;
  const int ctas = min(total, per_sm * num_sms);
  const int per_cta = (total + ctas - 1) / ctas;
  k<<<(total + per_cta - 1) / per_cta, 256, (size_t)smem, st>>>(a, per_cta, nbuf);
  return cudaGetLastError();
}

// =====================================================================  K_l0
constexpr int L0_STAGES = 4;
constexpr int L0_IMG_BYTES = 16384;                // 128 rows x 64 K bf16 (or ext: 16 ch of p)
constexpr int L0_P_BYTES = 4096;                   // p of the stage: CG ch x 128 rows x NH bf16
constexpr int L0_B_BYTES = 128 * 64 * 2;          // B halves of a head group: 128 N x 64 K bf16
constexpr int L0_STAGE_BYTES = L0_IMG_BYTES + L0_P_BYTES + L0_B_BYTES;
constexpr int L0_OUT_BYTES = 4 * 128 * 128;        // ctx tile staging: 4 heads x 128 rows x 128 B
constexpr int L0_SMEM = L0_STAGES * L0_STAGE_BYTES + L0_OUT_BYTES + 1024 + 256;
constexpr int L0_THREADS = 608;                    // producer, image gate, MMA gate, 16 builders
constexpr uint32_t L0_ACC_COLS = 256;              // accumulator: NH heads x DH <= 256 columns
constexpr uint32_t L0_SLOT_COLS = 4 * 32;          // A slot: 64 bf16 K per head = 32 columns

#define L0_TRACE(ev, idx)                                                                   \
  do {                                                                                      \
    if (a.trace && blockIdx.x < 2 && (idx) < 256)                                           \
      a.trace[((ev) + 8 * blockIdx.x) * 256 + (idx)] = globaltimer_ns();                    \
  } while (0)


DEV void tmem_alloc_pair(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)), "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
DEV void tmem_dealloc_pair(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
               : "memory");
}
// M256 MMA over the CTA pair: A rows from each CTA's TMEM, B split by N across the pair
DEV void mma_ts_pair(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
      "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
DEV void commit_pair(uint64_t* bar) {  // arrives on `bar` in both CTAs of the pair
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"((uint16_t)3)
      : "memory");
}
// Arrive on rank 0's copy of bar. Default (.release.cta) semantics, as CUTLASS's cluster
// barriers use: the data the leader's MMA consumes is TMEM written by tcgen05.st, ordered by
// tcgen05.wait::st + fence::before_thread_sync; a .release.cluster arrive measured ~1 us.
DEV void mbar_arrive_rank0(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, 0;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {  // acquire.cluster wait
  const uint32_t addr = smem_u32(bar);
  const long long t0 = clock64();
  while (true) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
    if (clock64() - t0 > 40000000000LL) __trap();
  }
}
DEV void tma_store_2d(const CUtensorMap* m, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}

// Level-0 node kernel on CTA pairs (cluster of 2, cta_group::2 MMAs).
// A cluster unit is (node n, pair of 128-row tiles, head group hg of NH heads); CTA rank r owns
// tile 2*pair + r (an odd tile count gives the last pair a phantom tile that loads a copy of
// the last tile and stores nothing). Stages of a unit:
//   main stage st < nmain: CG channels (K = 64 per head): image rows, p slices, B halves
//   ext stage e < next:    16 channels of the bias K-block: p slices (A = p), Et halves
// Each M256 x N64 MMA reads A (p * patch, built by this CTA's builders) from both CTAs' TMEM and
// B = M_c[:, head] split by N: rank r holds output columns [32r, 32r + 32) of every head. That
// halves the B operand's shared-memory traffic per SM (TMA write + MMA read), which bounded the
// single-CTA kernel (~105 KB of smem traffic per 512-cycle stage at ~128 B/cycle).
// Warp roles (per CTA, 19 warps):
//   warp 0      producer: 1-D bulk copies of every stage into a 4-deep shared-memory ring.
//   warp 1      image gate: "stage landed" (mbarrier) -> named barrier IMG(q); TMEM owner.
//   warp 2      MMA gate (rank 0 only): READY(q) from both CTAs' builders (cluster mbarrier)
//               -> the stage's MMAs -> commits to stage, slot and accumulator barriers of
//               both CTAs.
//   warps 3..18 builders, two groups of 8 taking alternate stages (group q & 1 owns A slot
//               q & 1); the two warps of a TMEM lane quarter split K into halves for all NH
//               heads: A = p[r,c,h] * patch_c[r] -> tcgen05.st -> READY(q). At the end of a
//               unit they drain the accumulator (x 1/sum_c e) into a 128B-swizzled smem tile
//               that TMA tensor stores write to ctx in the background of the next unit.
template <int PP, int L0_NH, int L0_DH, bool ROWP>
__global__ void __launch_bounds__(L0_THREADS, 1)
    l0_node_kernel(L0NodeArgs a, const __grid_constant__ CUtensorMap tm_ctx,
                   const __grid_constant__ CUtensorMap tm_pos) {
  constexpr int CG = 64 / PP;        // channels per main stage (K = 64 per head per stage)
  constexpr int L0_BH_BYTES = L0_DH * 64;  // one head's B half: DH/2 N x 64 K bf16
  constexpr uint32_t BLBO = L0_DH * 8;     // bytes between K-adjacent core matrices of a half
  static_assert(L0_NH * L0_DH <= 256, "head group exceeds the accumulator");
  constexpr int P = PP == 64 ? 8 : 4;
  constexpr int NBAR = 288;          // image gate warp + one group's 8 builder warps
  constexpr int PROW = 128 * L0_NH * 2;  // bytes of one channel's p slice for the tile
  constexpr bool rowp = ROWP;        // p staged per row (attention) or a constant table (linear)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* stage_out = smem + L0_STAGES * L0_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_out + L0_OUT_BYTES);
  uint64_t* empty = full + L0_STAGES;
  uint64_t* aempty = empty + L0_STAGES;
  uint64_t* accfull = aempty + 2;
  uint64_t* ready = accfull + 1;  // [2], rank 0's copy is the one used
  uint64_t* posv_full = ready + 2;  // the unit's positional tile landed in the staging tile
  uint32_t* tslot = reinterpret_cast<uint32_t*>(posv_full + 1);

  const int warp = warp_id(), lane = lane_id();
  const int R = a.B * a.S;
  const int n_tiles = R / 128;
  const int npairs = (n_tiles + 1) / 2;
  const int HG = a.H / L0_NH;
  const int crank = (int)cluster_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int total_units = a.n_nodes * npairs * HG;
  auto decode = [&](int u, int& hg, int& tile, int& n) {
    hg = u % HG;
    const int rest = u / HG;
    tile = (rest % npairs) * 2 + crank;
    n = rest / npairs;
  };
  auto unit_stages = [&](int u, int& g, int& nmain, int& next) {
    const int n = (u / HG) / npairs;
    g = __ldg(a.node_g + n);
    nmain = (g + CG - 1) / CG;
    next = (g + 15) / 16;
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < L0_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&aempty[0], 1);
    mbar_init(&aempty[1], 1);
    mbar_init(accfull, 1);
    mbar_init(&ready[0], 16);  // 8 builder warps x 2 CTAs
    mbar_init(&ready[1], 16);
    mbar_init(posv_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tslot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive / multicast
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    // ------------------------------------------------ producer (bulk copies)
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cid; u < total_units; u += ncl) {
        int hg, tile, n;
        decode(u, hg, tile, n);
        if (tile >= n_tiles) tile = n_tiles - 1;  // phantom tile: load a copy
        const int c0 = __ldg(a.node_c0 + n);
        int g, nmain, next;
        unit_stages(u, g, nmain, next);
        const long long poff = __ldg(a.node_poff + n);
        const int r0 = tile * 128;
        const int b = r0 / a.S, s0 = r0 - b * a.S;
        const __nv_bfloat16* chunk0 =
            a.img + b * a.img_sb + (long long)(s0 / a.wp) * P * a.W;
        auto pslice = [&](int c) {  // p slice of (hg, channel c) for this tile
          return a.p + poff + (((long long)hg * g + c) * R + r0) * L0_NH;
        };
        for (int st = 0; st < nmain + next; ++st) {
          mbar_wait(&empty[stage], phase ^ 1);  // MMAs of the stage 4 back are done
          uint8_t* sI = smem + stage * L0_STAGE_BYTES;
          uint8_t* sP = sI + L0_IMG_BYTES;
          uint8_t* sB = sP + L0_P_BYTES;
          if (a.debug_mode & 4) {
            mbar_arrive(&full[stage]);
          } else if (st < nmain) {
            const int cv = min(CG, g - st * CG);
            mbar_expect_tx(&full[stage], cv * 128 * PP * 2 + (rowp ? cv * PROW : 0) +
                                             L0_NH * L0_BH_BYTES);
            for (int cc = 0; cc < cv; ++cc) {
              const int c = st * CG + cc;
              bulk_load(sI + cc * 128 * PP * 2, chunk0 + (long long)(c0 + c) * a.img_sc,
                        128 * PP * 2, &full[stage]);
              if (rowp) bulk_load(sP + cc * PROW, pslice(c), PROW, &full[stage]);
            }
            // B halves: Mt [H][2][C_pad*PP/8][DH/16][8][8]; the stage's 64 K rows are contiguous
            for (int h = 0; h < L0_NH; ++h) {
              const __nv_bfloat16* src =
                  a.Mt + (((long long)(hg * L0_NH + h) * 2 + crank) * a.C_pad + c0 + st * CG) *
                             (PP * (L0_DH / 2));
              bulk_load(sB + h * L0_BH_BYTES, src, L0_BH_BYTES, &full[stage]);
            }
          } else {
            const int e = st - nmain;
            const int ce = min(16, g - 16 * e);
            mbar_expect_tx(&full[stage], (rowp ? ce * PROW : 0) + L0_NH * 16 * L0_DH);
            if (rowp)
              for (int cc = 0; cc < ce; ++cc)
                bulk_load(sI + cc * PROW, pslice(16 * e + cc), PROW, &full[stage]);
            // Et [n][H][2][KE/8][DH/16][8][8]
            for (int h = 0; h < L0_NH; ++h) {
              const __nv_bfloat16* src =
                  a.Et + (((long long)n * a.H + hg * L0_NH + h) * 2 + crank) *
                             ((long long)(L0_DH / 2) * a.KE) + e * 16 * (L0_DH / 2);
              bulk_load(sB + h * L0_BH_BYTES, src, 16 * L0_DH, &full[stage]);
            }
          }
          if (++stage == L0_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ image gate: full(q) -> IMG(q)
    int q_total = 0;
    for (int u = cid; u < total_units; u += ncl) {
      int g, nmain, next;
      unit_stages(u, g, nmain, next);
      q_total += nmain + next;
    }
    for (int q = 0; q < q_total; ++q) {
      mbar_wait(&full[q % L0_STAGES], (uint32_t)((q / L0_STAGES) & 1));
      if (lane == 0) L0_TRACE(0, q);
      asm volatile("bar.arrive %0, %1;" ::"r"(1 + (int)(q & 3)), "r"(NBAR) : "memory");
    }
  } else if (warp == 2) {
    // ------------------------------------------------ MMA gate (rank 0): READY(q) -> MMAs
    // UTCHMMA issue blocks while the tensor pipe is busy, so the issuer is a dedicated warp.
    // Stages are issued in order: the accumulation order is fixed (bit-reproducible).
    if (crank == 0) {
      const uint32_t idesc = idesc_bf16_f32(256, L0_DH);
      int q = 0;
      for (int u = cid; u < total_units; u += ncl) {
        int g, nmain, next;
        unit_stages(u, g, nmain, next);
        const int nst = nmain + next;
        for (int st = 0; st < nst; ++st, ++q) {
          const int cs = q % L0_STAGES, G = q & 1;
          mbar_wait(&ready[G], (uint32_t)((q >> 1) & 1));
          tc_fence_after();
          if (elect_one()) {
            L0_TRACE(2, q);
            const uint32_t sb = smem_u32(smem) + cs * L0_STAGE_BYTES + L0_IMG_BYTES + L0_P_BYTES;
            const uint32_t at0 = tbase + L0_ACC_COLS + G * L0_SLOT_COLS;
            if (a.debug_mode & 2) {
            } else if (st < nmain) {
#pragma unroll
              for (int h = 0; h < L0_NH; ++h)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  mma_ts_pair(tbase + h * L0_DH, at0 + h * 32 + kk * 8,
                              smem_desc(sb + h * L0_BH_BYTES + kk * 2 * BLBO, BLBO, 128, 0), idesc,
                              (st | kk) != 0);
            } else {
#pragma unroll
              for (int h = 0; h < L0_NH; ++h)
                mma_ts_pair(tbase + h * L0_DH, at0 + h * 32,
                            smem_desc(sb + h * L0_BH_BYTES, BLBO, 128, 0), idesc, 1u);
            }
            commit_pair(&empty[cs]);
            commit_pair(&aempty[G]);
            if (st == nst - 1) commit_pair(accfull);
            L0_TRACE(1, q);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------------------------ builders (warps 3..18)
    const int bw = warp - 3;
    const int G = bw >> 3;
    const int kh = (bw >> 2) & 1;
    const int quarter = warp & 3;       // TMEM lane quarter is fixed by warp id % 4
    const int m = quarter * 32 + lane;  // row within tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    constexpr int EC = L0_NH * L0_DH / 4;  // accumulator columns drained by this warp
    const int ecol = (G * 2 + kh) * EC;
    const bool lead = bw == 0 && lane == 0;  // issues the ctx tensor stores
    auto p_smem = [&](uint32_t base, int cc, uint32_t (&o)[2]) {  // base has the row offset
      const uint32_t src = base + cc * PROW;
      if (L0_NH == 4) {
        const uint2 v = lds64(src);
        o[0] = v.x; o[1] = v.y;
      } else {
        o[0] = lds32(src); o[1] = 0u;
      }
    };
    uint32_t accphase = 0;
    // epilogue of a finished unit: drain (x 1/sum) into the 128B-swizzled staging tile, TMA
    // tensor stores write it to ctx in the background. It runs after the builders have
    // already staged their first A slot of the next unit (overlapping the MMA tail), and
    // before that slot's READY: the next unit's first MMAs overwrite the accumulator.
    // positional tile of a unit: TMA loads of posV[n][s0 .. s0+128][head group] into the
    // staging tile (the drain adds it in place), issued once the previous unit's ctx stores
    // have read the staging
    uint32_t pos_phase = 0;
    bool pos_issued_cur = false, pos_issued_pend = false;
    auto issue_pos = [&](int n, int tile, int hg) {
      bulk_wait_read0();
      const int s0 = (min(tile, n_tiles - 1) * 128) % a.S;
      constexpr int NSUB = L0_NH * L0_DH / 64;  // 64-column sub-tiles of the head group
      mbar_expect_tx(posv_full, NSUB * 128 * 128);
      for (int sub = 0; sub < NSUB; ++sub)
        tma_load_2d(stage_out + sub * (128 * 128), &tm_pos, posv_full,
                    hg * L0_NH * L0_DH + sub * 64, n * a.S + s0);
    };
    auto epilogue = [&](int n, int tile, int hg, float sc) {
      mbar_wait(accfull, accphase);  // the unit's last MMAs
      accphase ^= 1;
      if (a.has_pos) {
        // the staging tile holds this unit's positional rows (posV[n][s][head group])
        if (lead && !pos_issued_pend) issue_pos(n, tile, hg);
        mbar_wait(posv_full, pos_phase);
        pos_phase ^= 1;
      } else {
        if (lead) bulk_wait_read0();   // the previous unit's stores have read the staging
        asm volatile("bar.sync 5, 512;" ::: "memory");  // ACC0: staging free
      }
      tc_fence_after();
      if (!(a.debug_mode & 32)) {
        const uint32_t sout = smem_u32(stage_out);
#pragma unroll
        for (int cb = 0; cb < EC; cb += 32) {
          const int col = ecol + cb;               // column within the head group
          const int hd = col / 64, c8 = (col % 64) / 8;  // 64-column sub-tile, 16-B chunk
          uint32_t v[32];
          tmem_ld32(tbase + lane_off + col, v);
          tmem_ld_wait();
          const uint32_t rowb = sout + hd * (128 * 128) + m * 128;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t addr = rowb + ((uint32_t)((c8 + k) ^ (m & 7)) << 4);
            float f[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] = sc * __uint_as_float(v[8 * k + e]);
            if (a.has_pos) {  // + posV (the token's positional term through wv_n)
              const uint4 pv4 = lds128(addr);
              const uint32_t pw[4] = {pv4.x, pv4.y, pv4.z, pv4.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                f[2 * e] += bf16lo(pw[e]);
                f[2 * e + 1] += bf16hi(pw[e]);
              }
            }
            uint4 o;
            o.x = pack_bf16(f[0], f[1]);
            o.y = pack_bf16(f[2], f[3]);
            o.z = pack_bf16(f[4], f[5]);
            o.w = pack_bf16(f[6], f[7]);
            sts128(addr, o);
          }
        }
      }
      tc_fence_before();
      fence_async_smem();  // staging writes -> async proxy (TMA store)
      asm volatile("bar.sync 6, 512;" ::: "memory");  // ACC1: tile staged, accumulator drained
      tc_fence_after();
      if (lead && tile < n_tiles && !(a.debug_mode & (8 | 32))) {
        const uint32_t sout = smem_u32(stage_out);
        for (int sub = 0; sub < L0_NH * L0_DH / 64; ++sub)
          tma_store_2d(&tm_ctx, sout + sub * (128 * 128), hg * L0_NH * L0_DH + sub * 64,
                       n * R + tile * 128);
        bulk_commit();
      }
    };
    int q = 0;
    int pend_n = -1, pend_tile = 0, pend_hg = 0;  // unit whose epilogue is pending
    float pend_sc = 1.f;
    for (int u = cid; u < total_units; u += ncl) {
      int hg, tile, n;
      decode(u, hg, tile, n);
      int g, nmain, next;
      unit_stages(u, g, nmain, next);
      const int nst = nmain + next;
      const long long poff = __ldg(a.node_poff + n);
      // softmax normaliser of this row and this warp's head, fetched a unit ahead of its use
      // (an HBM miss in the drain stalled the whole pair ~1 us)
      const float sc_u = a.pinv ? __ldg(a.pinv + ((long long)n * R + min(tile, n_tiles - 1) * 128 +
                                                  m) * a.H + hg * L0_NH + ecol / L0_DH)
                                : 1.f;
      auto p_const = [&](int c, uint32_t (&o)[2]) {  // linear-mix nodes: p[poff + c*H + h]
        const __nv_bfloat16* src = a.p + poff + (long long)c * a.H + hg * L0_NH;
        if (L0_NH == 4) {
          const uint2 v = __ldg(reinterpret_cast<const uint2*>(src));
          o[0] = v.x; o[1] = v.y;
        } else {
          o[0] = __ldg(reinterpret_cast<const unsigned int*>(src)); o[1] = 0u;
        }
      };
      for (int st = 0; st < nst; ++st, ++q) {
        if ((q & 1) != G) continue;
        const int cs = q % L0_STAGES;
        // per-thread address terms are re-derived every stage (hoisted values spilled, and
        // a spill reload misses the ~25 KB L1 left next to the shared-memory carve-out)
        const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
        uint32_t tb = tbase + lane_off;
        asm volatile("" : "+r"(tb));
        const uint32_t mm = threadIdx.x & 127u;  // == m
        const uint32_t lwp = (uint32_t)(__ffs(a.wp) - 1);  // W / P divides 128: a power of 2
        const uint32_t xo = ((((mm >> lwp) * P + (P == 8 ? 4 * kh : 0)) * (uint32_t)a.W +
                              (mm & (uint32_t)(a.wp - 1)) * P) * 2);
        const uint32_t wr = (uint32_t)a.W * 2, po = mm * (L0_NH * 2);
        const uint32_t sI = sbase + cs * L0_STAGE_BYTES;
        const uint32_t sP = sI + L0_IMG_BYTES;
        const bool ext = st >= nmain;
        asm volatile("bar.sync %0, %1;" ::"r"(1 + (q & 3)), "r"(NBAR) : "memory");  // IMG
        const uint32_t slot_t = tb + L0_ACC_COLS + G * L0_SLOT_COLS;
        if (!ext) {
          // this warp's 16 of the 32 A columns: P == 8 -> pixel rows 4kh..4kh+3 of the one
          // channel; P == 4 -> channels 2kh, 2kh+1 of the stage's four
          constexpr int NCC = CG == 1 ? 1 : 2;
          uint32_t x[16], pv[NCC][2];
#pragma unroll
          for (int ci = 0; ci < NCC; ++ci) {
            const int cc = CG == 1 ? 0 : 2 * kh + ci;
            const int c = st * CG + cc;
            const bool valid = c < g;
            if (!valid) {
              pv[ci][0] = pv[ci][1] = 0u;
            } else if (rowp) {
              p_smem(sP + po, cc, pv[ci]);
            } else {
              p_const(c, pv[ci]);
            }
            const uint32_t base = sI + cc * 128 * PP * 2 + xo;
            if (P == 8) {
#pragma unroll
              for (int r4 = 0; r4 < 4; ++r4) {
                const uint4 v = valid ? lds128(base + r4 * wr) : make_uint4(0, 0, 0, 0);
                x[r4 * 4 + 0] = v.x; x[r4 * 4 + 1] = v.y; x[r4 * 4 + 2] = v.z; x[r4 * 4 + 3] = v.w;
              }
            } else {
#pragma unroll
              for (int py = 0; py < 4; ++py) {
                const uint2 v = valid ? lds64(base + py * wr) : make_uint2(0, 0);
                x[ci * 8 + py * 2 + 0] = v.x; x[ci * 8 + py * 2 + 1] = v.y;
              }
            }
          }
          if ((bw & 7) == 0 && lane == 0) L0_TRACE(3, q);
          // A slot free: the MMAs of this group's previous stage (same slot) have completed
          mbar_wait(&aempty[G], (uint32_t)(((q >> 1) & 1) ^ 1));
          tc_fence_after();
#pragma unroll
          for (int h = 0; h < L0_NH; ++h) {
            uint32_t ph[2];
#pragma unroll
            for (int ci = 0; ci < 2; ++ci) {
              const uint32_t w = pv[NCC == 1 ? 0 : ci][h >> 1];
              ph[ci] = (a.debug_mode & 1) ? 0u
                       : (h & 1) ? (w & 0xffff0000u) | (w >> 16) : (w << 16) | (w & 0xffffu);
            }
            // multiply + tcgen05.st in one asm block (the products never become C values, so
            // the compiler cannot keep all heads' products live at once)
            tmem_st16_scaled(slot_t + h * 32 + 16 * kh, x, ph[0], ph[1]);
          }
        } else {
          // ext stage e: A[r, k] = p[r, 16e + k, h] (k < 16); this warp: k in [8kh, 8kh+8)
          const int e = st - nmain;
          uint32_t lo[4][2], hi[4][2];
#pragma unroll
          for (int kc = 0; kc < 4; ++kc) {
            const int cl0 = 8 * kh + 2 * kc;          // channel within the ext block
            const int c0e = 16 * e + cl0;
            lo[kc][0] = lo[kc][1] = hi[kc][0] = hi[kc][1] = 0u;
            if (c0e < g) { if (rowp) p_smem(sI + po, cl0, lo[kc]); else p_const(c0e, lo[kc]); }
            if (c0e + 1 < g) { if (rowp) p_smem(sI + po, cl0 + 1, hi[kc]); else p_const(c0e + 1, hi[kc]); }
          }
          mbar_wait(&aempty[G], (uint32_t)(((q >> 1) & 1) ^ 1));
          tc_fence_after();
#pragma unroll
          for (int h = 0; h < L0_NH; ++h) {
            uint32_t y4[4];
#pragma unroll
            for (int kc = 0; kc < 4; ++kc) {
              const uint32_t a16 = (h & 1) ? (lo[kc][h >> 1] >> 16) : (lo[kc][h >> 1] & 0xffffu);
              const uint32_t b16 = (h & 1) ? (hi[kc][h >> 1] >> 16) : (hi[kc][h >> 1] & 0xffffu);
              y4[kc] = a16 | (b16 << 16);
            }
            tmem_st4(slot_t + h * 32 + 4 * kh, y4);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        if ((bw & 7) == 0 && lane == 0) L0_TRACE(4, q);
        if (pend_n >= 0) {  // first own stage of this unit staged: finish the previous unit
          epilogue(pend_n, pend_tile, pend_hg, pend_sc);
          pend_n = -1;
        } else if (a.has_pos && lead && !pos_issued_cur) {
          issue_pos(n, tile, hg);  // the previous unit's stores were issued a stage ago
          pos_issued_cur = true;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_rank0(&ready[G]);  // READY(q): this warp's A is in TMEM
      }
      pend_n = n; pend_tile = tile; pend_hg = hg; pend_sc = sc_u;
      pos_issued_pend = pos_issued_cur;
      pos_issued_cur = false;
    }
    if (pend_n >= 0) epilogue(pend_n, pend_tile, pend_hg, pend_sc);
    if (lead) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tbase, 512);
  }
}

cudaError_t launch_l0_node(const L0NodeArgs& a, const CUtensorMap& tm_ctx,
                           const CUtensorMap& tm_pos, int num_sms, cudaStream_t st) {
  const int R = a.B * a.S;
  const int dh = a.D / a.H;
  const int nh = dh == 128 ? 2 : (a.H % 4 == 0 ? 4 : 2);  // heads per unit: NH * dh <= 256
  if (R % 128 || a.S % 128 || 128 % a.wp || a.H % nh || a.D != a.H * dh ||
      (dh != 64 && dh != 128) || a.KE % 16 || a.nh != nh)
    return cudaErrorInvalidValue;
  const int n_tiles = R / 128;
  const int units = a.n_nodes * ((n_tiles + 1) / 2) * (a.H / nh);
  const int max_cl = num_sms / 2;
  const int grid = (units < max_cl ? units : max_cl) * 2;
  void (*kern)(L0NodeArgs, const CUtensorMap, const CUtensorMap) = nullptr;
  const bool rp = a.p_row_mode != 0;
#define L0N_PICK(PP_, NH_, DH_) \
  kern = rp ? l0_node_kernel<PP_, NH_, DH_, true> : l0_node_kernel<PP_, NH_, DH_, false>;
  if (a.P == 8) {
    if (dh == 128) { L0N_PICK(64, 2, 128) } else if (nh == 4) { L0N_PICK(64, 4, 64) } else { L0N_PICK(64, 2, 64) }
  } else if (a.P == 4) {
    if (dh == 128) { L0N_PICK(16, 2, 128) } else if (nh == 4) { L0N_PICK(16, 4, 64) } else { L0N_PICK(16, 2, 64) }
  } else {
    return cudaErrorInvalidValue;
  }
#undef L0N_PICK
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L0_SMEM);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(L0_THREADS);
  cfg.dynamicSmemBytes = L0_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, a, tm_ctx, tm_pos);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace dchag
