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
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4],
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// One CTA = (node n, block of RB rows), 8 warps: warp w takes the m16 row tile w % (RB/16)
// and the channels c = w / (RB/16) mod CS (CS = 128 / RB channel phases). The block's rows of
// every channel of the node are one contiguous image run each (RB % (W/P) == 0), so the node
// slice lands in shared memory with g 1-D bulk copies (images are read from HBM once); the
// logit weights are staged with a 16-byte XOR swizzle (conflict-free ldmatrix rows). Pass 1:
// per-warp online max/sum over its channels, merged through shared memory; pass 2: p.
// Fragments come from ldmatrix (P = 8: a 16-wide K step is two whole patch pixel rows) or
// 32-bit shared loads (P = 4), all on precomputed 32-bit shared addresses.
template <int NT, int P, int MT>  // NT = HP / 8 head tiles, MT = RB / 16 row tiles
__global__ void __launch_bounds__(256) l0_logits_kernel(L0LogitArgs a) {
  constexpr int RB = MT * 16, CS = 8 / MT;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t landed;
  constexpr int PP = P * P;
  constexpr int KS = PP / 16;
  constexpr int CPR = PP * 2 / 16;  // 16-byte chunks per weight row
  const uint32_t sbase = (smem_u32(smem_raw) + 127) & ~127u;
  const int R = a.B * a.S;
  const int blocks_per_node = R / RB;
  const int n = blockIdx.x / blocks_per_node;
  const int rblk = blockIdx.x - n * blocks_per_node;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int mt = warp % MT, cph = warp / MT;
  const int c0 = __ldg(a.node_c0 + n), g = __ldg(a.node_g + n);
  const long long poff = __ldg(a.node_poff + n);
  const int r0 = rblk * RB;
  const uint32_t chunk = (uint32_t)RB * PP * 2;            // bytes of one channel's image block
  const uint32_t sW = sbase + (uint32_t)a.gmax * chunk;    // [g*HP][PP] swizzled weights
  const uint32_t wrow = (uint32_t)a.HP * PP * 2;           // weight bytes per channel
  float2* stats = reinterpret_cast<float2*>(smem_raw + (sW - smem_u32(smem_raw)) +
                                            (size_t)a.gmax * wrow);
  if (threadIdx.x == 0) {
    mbar_init(&landed, 1);
    fence_barrier_init();
    const int b = r0 / a.S, s0 = r0 - b * a.S;
    const __nv_bfloat16* src0 = a.img + b * a.img_sb + (long long)(s0 / a.wp) * P * a.W;
    mbar_expect_tx(&landed, chunk * g);
    for (int c = 0; c < g; ++c) {
      const uint32_t dst = sbase + c * chunk;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(dst), "l"(src0 + (long long)(c0 + c) * a.img_sc), "r"(chunk),
          "r"(smem_u32(&landed))
          : "memory");
    }
  }
  auto wswz = [&](int row, int ch) -> uint32_t {  // byte offset of chunk ch of weight row
    const int f = CPR >= 8 ? (row & 7) : ((row / (8 / CPR)) & (CPR - 1));
    return (uint32_t)(row * (PP * 2) + ((ch ^ f) << 4));
  };
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.WUt + (long long)c0 * a.HP * PP);
    const int nchunks = g * a.HP * CPR;
    for (int i = threadIdx.x; i < nchunks; i += 256) sts128(sW + wswz(i / CPR, i % CPR), __ldg(src + i));
  }

  int rows[2], srow[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    rows[q] = r0 + mt * 16 + gid + 8 * q;
    srow[q] = rows[q] % a.S;
  }
  // per-thread shared byte offsets inside a channel block / weight slice
  uint32_t aoff[KS], boff[KS][NT / 2 > 0 ? NT / 2 : 1];
  uint32_t aoff4[4];
  if (P == 8) {
    const int mat = lane >> 3, rr = lane & 7;
    const int rl = mt * 16 + (mat & 1) * 8 + rr;
    const int i = rl / a.wp, j = rl - i * a.wp;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
      aoff[ks] = (uint32_t)(((i * P + 2 * ks + (mat >> 1)) * a.W + j * P) * 2);
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {  // a0..a3: rows gid / gid+8, k = 2tig (+8)
      const int rl = mt * 16 + gid + 8 * (e & 1);
      const int i = rl / a.wp, j = rl - i * a.wp;
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
        const int kh = NT == 1 ? (mat & 1) : (mat & 1);
        boff[ks][np] = wswz(nt * 8 + rr, ks * 2 + kh);
      }
  }
  float pu[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const float* pr0 = a.posU + ((long long)n * a.S + srow[0]) * a.HP + nt * 8 + 2 * tig;
    const float* pr1 = a.posU + ((long long)n * a.S + srow[1]) * a.HP + nt * 8 + 2 * tig;
    pu[nt][0] = pr0[0]; pu[nt][1] = pr0[1];
    pu[nt][2] = pr1[0]; pu[nt][3] = pr1[1];
  }
  __syncthreads();  // barrier init + weights visible
  mbar_wait(&landed, 0);

  auto logits = [&](int c, float (&L)[NT][4]) {
    const uint32_t ab = sbase + c * chunk;
    const uint32_t wb = sW + c * wrow;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const float* bu = a.bU + (long long)(c0 + c) * a.HP + nt * 8 + 2 * tig;
      const float2 bb = __ldg(reinterpret_cast<const float2*>(bu));
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

  // softmax over the node's channels in base 2: t = logit * log2(e)
  constexpr float LOG2E = 1.4426950408889634f;
  float* stat = reinterpret_cast<float*>(stats);  // [CS][MT][NT][4][32]
  auto sidx = [&](int k, int nt, int e) { return (((k * MT + mt) * NT + nt) * 4 + e) * 32 + lane; };
  // pass 1: max only
  float mx[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) mx[nt][e] = -INFINITY;
#pragma unroll 2
  for (int c = cph; c < g; c += CS) {
    float L[NT][4];
    logits(c, L);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) mx[nt][e] = fmaxf(mx[nt][e], L[nt][e]);
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) stat[sidx(cph, nt, e)] = mx[nt][e];
  __syncthreads();
  float nmx[NT][4];  // -max * log2(e)
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float m = stat[sidx(0, nt, e)];
#pragma unroll
      for (int k = 1; k < CS; ++k) m = fmaxf(m, stat[sidx(k, nt, e)]);
      nmx[nt][e] = -m * LOG2E;
    }
  __syncthreads();  // stat reused for the sums
  const int nh = (a.H % 4 == 0) ? 4 : 2;
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
  const bool unnorm = a.pinv != nullptr;
  // pass 2: e = 2^(t - max), sums; with pinv the unnormalised e is the output
  float sm_[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) sm_[nt][e] = 0.f;
#pragma unroll 2
  for (int c = cph; c < g; c += CS) {
    float L[NT][4];
    logits(c, L);
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
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) stat[sidx(cph, nt, e)] = sm_[nt][e];
  __syncthreads();
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float t = stat[sidx(0, nt, e)];
#pragma unroll
      for (int k = 1; k < CS; ++k) t += stat[sidx(k, nt, e)];
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
    return;
  }
  // pass 3 (normalised output): p = e / sum
#pragma unroll 2
  for (int c = cph; c < g; c += CS) {
    float L[NT][4];
    logits(c, L);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      if (nt * 8 + 2 * tig < a.H) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const float p0 = ex2_approx(fmaf(L[nt][2 * q], LOG2E, nmx[nt][2 * q])) * sm_[nt][2 * q];
          const float p1 =
              ex2_approx(fmaf(L[nt][2 * q + 1], LOG2E, nmx[nt][2 * q + 1])) * sm_[nt][2 * q + 1];
          *reinterpret_cast<uint32_t*>(pn + poff_e[nt][q] + c * cstride) = pack_bf16(p0, p1);
        }
      }
    }
  }
}

cudaError_t launch_l0_logits(const L0LogitArgs& a, cudaStream_t st) {
  const int R = a.B * a.S;
  const int PP = a.P * a.P;
  // rows per CTA: a multiple of the patch-row width (one contiguous run per channel), as
  // large as 64 while the node slice stays <= 64 KB (two CTAs per SM overlap copies)
  int RB = 0;
  for (int rb = 128; rb >= 16; rb >>= 1) {
    if (rb % a.wp || R % rb) continue;
    RB = rb;  // smallest valid so far
    if (rb <= 64 && (long long)a.gmax * rb * PP * 2 <= 64 * 1024) break;
  }
  if (RB == 0) return cudaErrorInvalidValue;
  const int NTv = a.HP / 8;
  const long long smem = (long long)a.gmax * RB * PP * 2 + (long long)a.gmax * a.HP * PP * 2 +
                         8LL * NTv * 4 * 32 * 8 + 128;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  const int grid = a.n_nodes * (R / RB);
  void (*k)(L0LogitArgs) = nullptr;
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
  k<<<grid, 256, (size_t)smem, st>>>(a);
  return cudaGetLastError();
}

// =====================================================================  K_l0
constexpr int L0_DH = 64;                          // head dim (MMA N)
constexpr int L0_STAGES = 4;
constexpr int L0_IMG_BYTES = 16384;                // 128 rows x 64 K bf16 (or ext: 16 ch of p)
constexpr int L0_P_BYTES = 4096;                   // p of the stage: CG ch x 128 rows x NH bf16
constexpr int L0_B_BYTES = 4 * L0_DH * 64 * 2;     // up to 4 heads x [64 x 64] bf16
constexpr int L0_STAGE_BYTES = L0_IMG_BYTES + L0_P_BYTES + L0_B_BYTES;
constexpr int L0_STAGE_OUT = 16 * 32 * 32;         // epilogue staging: 16 warps x 32 rows x 32 B
constexpr int L0_SMEM = L0_STAGES * L0_STAGE_BYTES + L0_STAGE_OUT + 1024 + 256;
constexpr int L0_THREADS = 576;                    // producer, image gate, 16 builders
constexpr uint32_t L0_ACC_COLS = 4 * L0_DH;        // accumulator region (NH * 64 used)
constexpr uint32_t L0_SLOT_COLS = 4 * 32;          // A slot: 64 bf16 K per head = 32 columns

#define L0_TRACE(ev, idx)                                                                   \
  do {                                                                                      \
    if (a.trace && blockIdx.x == 0 && (idx) < 256) a.trace[(ev) * 256 + (idx)] = clock64(); \
  } while (0)

// Stages of one unit (node n, 128-row tile, head group hg of NH heads):
//   main stage st < nmain: CG channels (K = 64 per head): image rows, p slices, B = M_c blocks
//   ext stage e < next:    16 channels of the bias K-block: p slices (A = p) and Et K-block
// Warp roles (one persistent CTA per SM, 18 warps):
//   warp 0      producer: 1-D bulk copies of every stage into a 4-deep shared-memory ring.
//   warp 1      image gate: waits "stage landed" (mbarrier) -> named barrier IMG(q).
//   warps 2..17 builders, two groups of 8 taking alternate stages (group q & 1 owns A slot
//               q & 1): A = p[r,c,h] * patch_c[r] (or p itself for ext) -> registers ->
//               tcgen05.st; the group's first warp then issues the stage's tcgen05.mma
//               (A from TMEM, B from smem) and commits stage, slot and accumulator barriers.
// The trace of the previous layout (one gate warp, 8 builders serialising every stage) showed
// ~1300 cycles per stage against 512 of MMA: the per-stage handshake chain (mbarrier try_wait
// ~157 cycles, tcgen05.st + wait ~137, named-barrier hops) ran back to back with the build.
// Two groups overlap one stage's chain with the next stage's build.
// CL = 2: a CTA pair (same node and head group, adjacent row tiles) splits the B blocks of
// every stage between its two producers and multicasts them, halving the weight fill per CTA
// (the kernel is L2->SMEM fill bound); empty[] then counts both CTAs' MMA commits.
template <int PP, int L0_NH, int CL>
__global__ void __launch_bounds__(L0_THREADS, 1) l0_node_kernel(L0NodeArgs a) {
  constexpr int CG = 64 / PP;        // channels per main stage (K = 64 per head per stage)
  constexpr int P = PP == 64 ? 8 : 4;
  constexpr int NBAR = 288;          // image gate warp + one group's 8 builder warps
  constexpr int PROW = 128 * L0_NH * 2;  // bytes of one channel's p slice for the tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* stage_out = smem + L0_STAGES * L0_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_out + L0_STAGE_OUT);
  uint64_t* empty = full + L0_STAGES;
  uint64_t* aempty = empty + L0_STAGES;
  uint64_t* accfull = aempty + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accfull + 1);

  const int warp = warp_id(), lane = lane_id();
  const int R = a.B * a.S;
  const int n_tiles = R / 128;
  const int HG = a.H / L0_NH;
  const int crank = CL > 1 ? (int)cluster_rank() : 0;
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const int total_units = a.n_nodes * (n_tiles / CL) * HG;  // cluster units
  const uint16_t cmask = (uint16_t)((1u << CL) - 1);
  const bool rowp = a.p_row_mode != 0;
  // cluster unit u -> (head group, this CTA's row tile, node)
  auto decode = [&](int u, int& hg, int& tile, int& n) {
    hg = u % HG;
    const int rest = u / HG;
    tile = (rest % (n_tiles / CL)) * CL + crank;
    n = rest / (n_tiles / CL);
  };
  auto unit_stages = [&](int u, int& g, int& nmain, int& next) {
    const int n = (u / HG) / (n_tiles / CL);
    g = __ldg(a.node_g + n);
    nmain = (g + CG - 1) / CG;
    next = (g + 15) / 16;
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < L0_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);
    }
    mbar_init(&aempty[0], 1);
    mbar_init(&aempty[1], 1);
    mbar_init(accfull, 2);  // one commit per builder group
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync();  // the peer multicasts into our barriers from here on
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
        const int c0 = __ldg(a.node_c0 + n);
        int g, nmain, next;
        unit_stages(u, g, nmain, next);
        const long long poff = __ldg(a.node_poff + n);
        const int r0 = tile * 128;
        const int b = r0 / a.S, s0 = r0 - b * a.S;
        const __nv_bfloat16* chunk0 =
            a.img + b * a.img_sb + (long long)(s0 / a.wp) * P * a.W;
        // p slice of (hg, channel c) for this tile
        auto pslice = [&](int c) {
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
                                             L0_NH * L0_DH * 64 * 2);
            for (int cc = 0; cc < cv; ++cc) {
              const int c = st * CG + cc;
              bulk_load(sI + cc * 128 * PP * 2, chunk0 + (long long)(c0 + c) * a.img_sc,
                        128 * PP * 2, &full[stage]);
              if (rowp) bulk_load(sP + cc * PROW, pslice(c), PROW, &full[stage]);
            }
            for (int h = crank * (L0_NH / CL); h < (crank + 1) * (L0_NH / CL); ++h) {
              const __nv_bfloat16* src =
                  a.Mt + ((long long)(hg * L0_NH + h) * a.C_pad + c0 + st * CG) * (L0_DH * PP);
              if (CL == 1) bulk_load(sB + h * (L0_DH * 64 * 2), src, L0_DH * 64 * 2, &full[stage]);
              else bulk_load_mc(sB + h * (L0_DH * 64 * 2), src, L0_DH * 64 * 2, &full[stage], cmask);
            }
          } else {
            const int e = st - nmain;
            const int ce = min(16, g - 16 * e);
            mbar_expect_tx(&full[stage], (rowp ? ce * PROW : 0) + L0_NH * L0_DH * 16 * 2);
            if (rowp)
              for (int cc = 0; cc < ce; ++cc)
                bulk_load(sI + cc * PROW, pslice(16 * e + cc), PROW, &full[stage]);
            for (int h = crank * (L0_NH / CL); h < (crank + 1) * (L0_NH / CL); ++h) {
              const __nv_bfloat16* src = a.Et + ((long long)n * a.H + hg * L0_NH + h) *
                                                    (L0_DH * a.KE) + e * 16 * L0_DH;
              if (CL == 1) bulk_load(sB + h * (L0_DH * 64 * 2), src, L0_DH * 16 * 2, &full[stage]);
              else bulk_load_mc(sB + h * (L0_DH * 64 * 2), src, L0_DH * 16 * 2, &full[stage], cmask);
            }
          }
          if (++stage == L0_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ image gate: full(q) -> IMG(q)
    long long q_total = 0;
    for (int u = cid; u < total_units; u += ncl) {
      int g, nmain, next;
      unit_stages(u, g, nmain, next);
      q_total += nmain + next;
    }
    for (long long q = 0; q < q_total; ++q) {
      mbar_wait(&full[q % L0_STAGES], (uint32_t)((q / L0_STAGES) & 1));
      if (lane == 0) L0_TRACE(0, q);
      asm volatile("bar.arrive %0, %1;" ::"r"(1 + (int)(q & 3)), "r"(NBAR) : "memory");
    }
  } else {
    // ------------------------------------------------ builders (warps 2..17)
    // Two groups of 8 warps take alternate stages (group G = q & 1 owns A slot G), so one
    // group's handshake latencies overlap the other group's build. Within a group the two
    // warps of a TMEM lane quarter split K = 64 into halves (kh) for all NH heads, so every
    // image row is read from shared memory once. The group's first warp issues the stage's
    // MMAs itself (no gate warp hop). The accumulator is zeroed by tcgen05.st after each
    // drain, so every MMA accumulates and the two groups' MMAs need no mutual ordering.
    const int bw = warp - 2;
    const int G = bw >> 3;
    const int kh = (bw >> 2) & 1;
    const int quarter = warp & 3;       // TMEM lane quarter is fixed by warp id % 4
    const bool issuer = (bw & 7) == 0;
    const int m = quarter * 32 + lane;  // row within tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    constexpr int EC = L0_NH * 16;      // accumulator columns drained by this warp
    const int ecol = (G * 2 + kh) * EC;
    uint8_t* my_out = stage_out + bw * 1024;
    const uint32_t idesc = idesc_bf16_f32(128, L0_DH);
    const int i_l = m / a.wp, jj = m - (m / a.wp) * a.wp;
    auto zero_acc = [&]() {
      uint32_t z[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) z[e] = 0u;
#pragma unroll
      for (int cb = 0; cb < EC; cb += 16) tmem_st16(tbase + lane_off + ecol + cb, z);
      tmem_st_wait();
      tc_fence_before();
      asm volatile("bar.sync 7, 512;" ::: "memory");  // ACC: whole accumulator zeroed
      tc_fence_after();
    };
    // all NH heads of one channel for this row, packed bf16 pairs (heads 0-1, 2-3)
    auto p_smem = [&](const uint8_t* base, int cc, uint32_t (&o)[2]) {
      const uint8_t* src = base + cc * PROW + m * L0_NH * 2;
      if (L0_NH == 4) {
        const uint2 v = *reinterpret_cast<const uint2*>(src);
        o[0] = v.x; o[1] = v.y;
      } else {
        o[0] = *reinterpret_cast<const uint32_t*>(src); o[1] = 0u;
      }
    };
    long long q_total = 0;
    for (int u = cid; u < total_units; u += ncl) {
      int g, nmain, next;
      unit_stages(u, g, nmain, next);
      q_total += nmain + next;
    }
    zero_acc();
    uint32_t accphase = 0;
    long long q = 0;
    for (int u = cid; u < total_units; u += ncl) {
      int hg, tile, n;
      decode(u, hg, tile, n);
      int g, nmain, next;
      unit_stages(u, g, nmain, next);
      const int nst = nmain + next;
      const long long poff = __ldg(a.node_poff + n);
      // constant p table (linear-mix nodes): p[poff + c*H + h]
      auto p_const = [&](int c, uint32_t (&o)[2]) {
        const __nv_bfloat16* src = a.p + poff + (long long)c * a.H + hg * L0_NH;
        if (L0_NH == 4) {
          const uint2 v = __ldg(reinterpret_cast<const uint2*>(src));
          o[0] = v.x; o[1] = v.y;
        } else {
          o[0] = __ldg(reinterpret_cast<const unsigned int*>(src)); o[1] = 0u;
        }
      };
      for (int st = 0; st < nst; ++st, ++q) {
        if ((int)(q & 1) != G) continue;
        const int cs = (int)(q % L0_STAGES);
        const uint8_t* sI = smem + cs * L0_STAGE_BYTES;
        const uint8_t* sP = sI + L0_IMG_BYTES;
        const bool ext = st >= nmain;
        asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(q & 3)), "r"(NBAR) : "memory");  // IMG
        if (bw == 0 && lane == 0) L0_TRACE(3, q);
        const uint32_t slot_t = tbase + lane_off + L0_ACC_COLS + G * L0_SLOT_COLS;
        if (!ext) {
          // this warp's 16 of the 32 A columns: P == 8 -> pixel rows 4kh..4kh+3 of the one
          // channel; P == 4 -> channels 2kh, 2kh+1 of the stage's four
          constexpr int NCC = CG == 1 ? 1 : 2;  // channels touched by this K half
          uint32_t x[16], pv[NCC][2];
#pragma unroll
          for (int ci = 0; ci < NCC; ++ci) {
            const int cc = CG == 1 ? 0 : 2 * kh + ci;
            const int c = st * CG + cc;
            const bool valid = c < g;
            if (!valid) {
              pv[ci][0] = pv[ci][1] = 0u;
            } else if (rowp) {
              p_smem(sP, cc, pv[ci]);
            } else {
              p_const(c, pv[ci]);
            }
            const __nv_bfloat16* base = reinterpret_cast<const __nv_bfloat16*>(
                                            sI + cc * 128 * PP * 2) +
                                        (i_l * P) * a.W + jj * P;
            if (P == 8) {
#pragma unroll
              for (int r4 = 0; r4 < 4; ++r4) {
                const int py = 4 * kh + r4;
                const uint4 v = valid ? *reinterpret_cast<const uint4*>(base + py * a.W)
                                      : make_uint4(0, 0, 0, 0);
                x[r4 * 4 + 0] = v.x; x[r4 * 4 + 1] = v.y; x[r4 * 4 + 2] = v.z; x[r4 * 4 + 3] = v.w;
              }
            } else {
#pragma unroll
              for (int py = 0; py < 4; ++py) {
                const uint2 v = valid ? *reinterpret_cast<const uint2*>(base + py * a.W)
                                      : make_uint2(0, 0);
                x[ci * 8 + py * 2 + 0] = v.x; x[ci * 8 + py * 2 + 1] = v.y;
              }
            }
          }
          // A slot free: the MMAs of this group's previous stage (same slot) have completed
          mbar_wait(&aempty[G], (uint32_t)(((q >> 1) & 1) ^ 1));
          tc_fence_after();
#pragma unroll
          for (int h = 0; h < L0_NH; ++h) {
            uint32_t y[16];
#pragma unroll
            for (int ci = 0; ci < NCC; ++ci) {
              const uint32_t w = pv[ci][h >> 1];
              const uint32_t ph = (h & 1) ? (w & 0xffff0000u) | (w >> 16)
                                          : (w << 16) | (w & 0xffffu);
#pragma unroll
              for (int e = 0; e < 16 / NCC; ++e)
                y[ci * (16 / NCC) + e] =
                    (a.debug_mode & 1) ? 0u : mul_bf16x2(x[ci * (16 / NCC) + e], ph);
            }
            tmem_st16(slot_t + h * 32 + 16 * kh, y);
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
            if (c0e < g) { if (rowp) p_smem(sI, cl0, lo[kc]); else p_const(c0e, lo[kc]); }
            if (c0e + 1 < g) { if (rowp) p_smem(sI, cl0 + 1, hi[kc]); else p_const(c0e + 1, hi[kc]); }
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
        if (bw == 0 && lane == 0) L0_TRACE(4, q);
        if (!issuer) {
          asm volatile("bar.arrive %0, 256;" ::"r"(5 + G) : "memory");  // GRP: slot written
        } else {
          asm volatile("bar.sync %0, 256;" ::"r"(5 + G) : "memory");
          // fixed MMA order across the two groups (bit-reproducible accumulation): wait
          // until the other group's issuer has issued stage q-1
          if (q > 0) asm volatile("bar.sync %0, 64;" ::"r"(8 + G) : "memory");
          tc_fence_after();
          if (elect_one()) {
            if (bw == 0) L0_TRACE(2, q);
            const uint64_t bd0 = smem_desc(smem_u32(sI + L0_IMG_BYTES + L0_P_BYTES), 1024, 128, 0);
            const uint32_t at0 = tbase + L0_ACC_COLS + G * L0_SLOT_COLS;
            if (a.debug_mode & 2) {
            } else if (!ext) {
#pragma unroll
              for (int h = 0; h < L0_NH; ++h)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  mma_ts(tbase + h * L0_DH, at0 + h * 32 + kk * 8,
                         bd0 + (uint64_t)((h * (L0_DH * 64 * 2) + kk * 2048) >> 4), idesc, 1u);
            } else {
#pragma unroll
              for (int h = 0; h < L0_NH; ++h)
                mma_ts(tbase + h * L0_DH, at0 + h * 32,
                       bd0 + (uint64_t)((h * (L0_DH * 64 * 2)) >> 4), idesc, 1u);
            }
            if (CL == 1) mma_commit(&empty[cs]);
            else mma_commit_mc(&empty[cs], cmask);  // the peer multicasts into this stage too
            mma_commit(&aempty[G]);
            if (st + 2 >= nst) mma_commit(accfull);  // this group's last stage of the unit
          }
          __syncwarp();
          if (q + 1 < q_total) asm volatile("bar.arrive %0, 64;" ::"r"(9 - G) : "memory");
        }
      }
      // epilogue: this warp's 32 rows x EC columns, TMEM -> bf16 -> swizzled smem (1 KB)
      // -> coalesced 32-byte row segments; then zero the columns for the next unit
      if (bw == 0 && lane == 0) L0_TRACE(6, q);
      // softmax normaliser of this row and this warp's head (unnormalised p from K_p0)
      const float sc = a.pinv ? __ldg(a.pinv + ((long long)n * R + tile * 128 + m) * a.H +
                                      hg * L0_NH + ecol / L0_DH)
                              : 1.f;
      mbar_wait(accfull, accphase);  // both groups' last MMAs of the unit (count 2)
      accphase ^= 1;
      if (bw == 0 && lane == 0) L0_TRACE(7, q);
      tc_fence_after();
      const long long row0 = (long long)n * R + tile * 128 + quarter * 32;
#pragma unroll 1
      for (int cb = 0; cb < ((a.debug_mode & 32) ? 0 : EC); cb += 16) {
        const int col = ecol + cb;  // column within this head group
        uint32_t v[16];
        tmem_ld16(tbase + lane_off + col, v);
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          uint4 o;
          o.x = pack_bf16(sc * __uint_as_float(v[8 * k + 0]), sc * __uint_as_float(v[8 * k + 1]));
          o.y = pack_bf16(sc * __uint_as_float(v[8 * k + 2]), sc * __uint_as_float(v[8 * k + 3]));
          o.z = pack_bf16(sc * __uint_as_float(v[8 * k + 4]), sc * __uint_as_float(v[8 * k + 5]));
          o.w = pack_bf16(sc * __uint_as_float(v[8 * k + 6]), sc * __uint_as_float(v[8 * k + 7]));
          *reinterpret_cast<uint4*>(my_out + lane * 32 + ((k ^ ((lane >> 2) & 1)) << 4)) = o;
        }
        __syncwarp();
        if (a.debug_mode & (64 | 128)) {
          // timing experiment: the same bytes as one contiguous 1 KB run per warp chunk
          __nv_bfloat16* dst = a.ctx + ((((long long)u * 16 + bw) * (EC / 16) + cb / 16) << 9);
          if (a.debug_mode & 64) {
#pragma unroll
            for (int i = 0; i < 2; ++i)
              *reinterpret_cast<uint4*>(dst + i * 256 + lane * 8) =
                  *reinterpret_cast<const uint4*>(my_out + i * 512 + lane * 16);
          } else {
            fence_async_smem();
            if (lane == 0) { bulk_store(dst, my_out, 1024); bulk_commit(); bulk_wait_read0(); }
          }
        } else if (!(a.debug_mode & 8)) {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int rr = i * 16 + (lane >> 1), k = lane & 1;
            const uint4 o =
                *reinterpret_cast<const uint4*>(my_out + rr * 32 + ((k ^ ((rr >> 2) & 1)) << 4));
            *reinterpret_cast<uint4*>(a.ctx + (row0 + rr) * a.D + hg * L0_NH * L0_DH + col +
                                      k * 8) = o;
          }
        }
        __syncwarp();
      }
      zero_acc();
    }
  }

  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

cudaError_t launch_l0_node(const L0NodeArgs& a, int num_sms, cudaStream_t st) {
  const int R = a.B * a.S;
  const int nh = a.H % 4 == 0 ? 4 : 2;
  if (R % 128 || a.S % 128 || 128 % a.wp || a.H % nh || a.D != a.H * L0_DH || a.KE % 16)
    return cudaErrorInvalidValue;
  const int n_tiles = R / 128;
  const int CL = (n_tiles % 2 == 0 && a.cluster != 1) ? 2 : 1;
  const int units = a.n_nodes * (n_tiles / CL) * (a.H / nh);
  const int max_cl = num_sms / CL;
  const int grid = (units < max_cl ? units : max_cl) * CL;
  void (*kern)(L0NodeArgs) = nullptr;
  if (a.P == 8)
    kern = nh == 4 ? (CL == 2 ? l0_node_kernel<64, 4, 2> : l0_node_kernel<64, 4, 1>)
                   : (CL == 2 ? l0_node_kernel<64, 2, 2> : l0_node_kernel<64, 2, 1>);
  else if (a.P == 4)
    kern = nh == 4 ? (CL == 2 ? l0_node_kernel<16, 4, 2> : l0_node_kernel<16, 4, 1>)
                   : (CL == 2 ? l0_node_kernel<16, 2, 2> : l0_node_kernel<16, 2, 1>);
  else
    return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L0_SMEM);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(L0_THREADS);
  cfg.dynamicSmemBytes = L0_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace dchag
