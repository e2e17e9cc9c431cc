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

template <int NT, int P>  // NT = HP / 8 head tiles; P compile-time so every load unrolls
__global__ void __launch_bounds__(128) l0_logits_kernel(L0LogitArgs a) {
  const int R = a.B * a.S;
  const int blocks_per_node = R / 64;
  const int n = blockIdx.x / blocks_per_node;
  const int rblk = blockIdx.x - n * blocks_per_node;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  constexpr int PP = P * P;
  const int c0 = __ldg(a.node_c0 + n), g = __ldg(a.node_g + n);
  const long long poff = __ldg(a.node_poff + n);

  int rows[2];
  rows[0] = rblk * 64 + warp * 16 + gid;
  rows[1] = rows[0] + 8;
  const __nv_bfloat16* rowimg[2];
  int srow[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int b = rows[q] / a.S, s = rows[q] - b * a.S;
    srow[q] = s;
    const int i = s / a.wp, j = s - i * a.wp;
    rowimg[q] = a.img + b * a.img_sb + (long long)(i * P) * a.W + j * P;
  }
  float pu[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const float* pr0 = a.posU + ((long long)n * a.S + srow[0]) * a.HP + nt * 8 + 2 * tig;
    const float* pr1 = a.posU + ((long long)n * a.S + srow[1]) * a.HP + nt * 8 + 2 * tig;
    pu[nt][0] = pr0[0]; pu[nt][1] = pr0[1];
    pu[nt][2] = pr1[0]; pu[nt][3] = pr1[1];
  }

  auto logits = [&](int c, float (&L)[NT][4]) {
    const long long coff = (long long)(c0 + c) * a.img_sc;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const float* bu = a.bU + (long long)(c0 + c) * a.HP + nt * 8 + 2 * tig;
      L[nt][0] = pu[nt][0] + bu[0];
      L[nt][1] = pu[nt][1] + bu[1];
      L[nt][2] = pu[nt][2] + bu[0];
      L[nt][3] = pu[nt][3] + bu[1];
    }
    uint32_t afs[PP / 16][4];
#pragma unroll
    for (int ks = 0; ks < PP / 16; ++ks) {
#pragma unroll
      for (int hk = 0; hk < 2; ++hk) {
        const int k = ks * 16 + hk * 8 + 2 * tig;
        const int py = k / P, px = k - py * P;
        const long long off = coff + (long long)py * a.W + px;
        afs[ks][hk * 2 + 0] = __ldg(reinterpret_cast<const unsigned int*>(rowimg[0] + off));
        afs[ks][hk * 2 + 1] = __ldg(reinterpret_cast<const unsigned int*>(rowimg[1] + off));
      }
    }
#pragma unroll
    for (int ks = 0; ks < PP / 16; ++ks) {
      const uint32_t (&af)[4] = afs[ks];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const __nv_bfloat16* wb = a.WUt + ((long long)(c0 + c) * a.HP + nt * 8 + gid) * PP +
                                  ks * 16 + 2 * tig;
        const uint32_t b0 = __ldg(reinterpret_cast<const unsigned int*>(wb));
        const uint32_t b1 = __ldg(reinterpret_cast<const unsigned int*>(wb + 8));
        mma_bf16_16816(L[nt], af, b0, b1);
      }
    }
  };

  float mx[NT][4], sm[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) { mx[nt][e] = -INFINITY; sm[nt][e] = 0.f; }
#pragma unroll 2
  for (int c = 0; c < g; ++c) {
    float L[NT][4];
    logits(c, L);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float m2 = fmaxf(mx[nt][e], L[nt][e]);
        sm[nt][e] = sm[nt][e] * __expf(mx[nt][e] - m2) + __expf(L[nt][e] - m2);
        mx[nt][e] = m2;
      }
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) sm[nt][e] = 1.f / sm[nt][e];
  for (int c = 0; c < g; ++c) {
    float L[NT][4];
    logits(c, L);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int h = nt * 8 + 2 * tig;
      if (h < a.H) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const float p0 = __expf(L[nt][2 * q] - mx[nt][2 * q]) * sm[nt][2 * q];
          const float p1 = __expf(L[nt][2 * q + 1] - mx[nt][2 * q + 1]) * sm[nt][2 * q + 1];
          const int nh = (a.H % 4 == 0) ? 4 : 2;
          const int hg = h / nh, hl = h - hg * nh;
          __nv_bfloat16* dst = a.p + poff + (((long long)hg * g + c) * R + rows[q]) * nh + hl;
          *reinterpret_cast<uint32_t*>(dst) = pack_bf16(p0, p1);
        }
      }
    }
  }
}

cudaError_t launch_l0_logits(const L0LogitArgs& a, cudaStream_t st) {
  const int R = a.B * a.S;
  if (R % 64) return cudaErrorInvalidValue;
  const int grid = a.n_nodes * (R / 64);
  void (*k)(L0LogitArgs) = nullptr;
  const int nt = a.HP / 8;
  if (a.P == 8) k = nt == 1 ? l0_logits_kernel<1, 8> : nt == 2 ? l0_logits_kernel<2, 8>
                                                      : nt == 4 ? l0_logits_kernel<4, 8> : nullptr;
  else if (a.P == 4) k = nt == 1 ? l0_logits_kernel<1, 4> : nt == 2 ? l0_logits_kernel<2, 4>
                                                           : nt == 4 ? l0_logits_kernel<4, 4> : nullptr;
  if (!k) return cudaErrorInvalidValue;
  k<<<grid, 128, 0, st>>>(a);
  return cudaGetLastError();
}

// =====================================================================  K_l0
constexpr int L0_DH = 64;                          // head dim (MMA N)
constexpr int L0_STAGES = 4;
constexpr int L0_IMG_BYTES = 16384;                // 128 rows x 64 K bf16 (or ext: 16 ch of p)
constexpr int L0_P_BYTES = 4096;                   // p of the stage: CG ch x 128 rows x NH bf16
constexpr int L0_B_BYTES = 4 * L0_DH * 64 * 2;     // up to 4 heads x [64 x 64] bf16
constexpr int L0_STAGE_BYTES = L0_IMG_BYTES + L0_P_BYTES + L0_B_BYTES;
constexpr int L0_STAGE_OUT = 8 * 32 * 64;          // epilogue staging: 8 warps x 32 rows x 64 B
constexpr int L0_SMEM = L0_STAGES * L0_STAGE_BYTES + L0_STAGE_OUT + 1024 + 256;
constexpr int L0_THREADS = 352;                    // producer, gate, image gate, 8 builders
constexpr uint32_t L0_ACC_COLS = 4 * L0_DH;        // accumulator region (NH * 64 used)
constexpr uint32_t L0_SLOT_COLS = 4 * 32;          // A slot: 64 bf16 K per head = 32 columns

#define L0_TRACE(ev, idx)                                                                   \
  do {                                                                                      \
    if (a.trace && blockIdx.x == 0 && (idx) < 256) a.trace[(ev) * 256 + (idx)] = clock64(); \
  } while (0)

// Stages of one unit (node n, 128-row tile, head group hg of NH heads):
//   main stage st < nmain: CG channels (K = 64 per head): image rows, p slices, B = M_c blocks
//   ext stage e < next:    16 channels of the bias K-block: p slices (A = p) and Et K-block
// Warp roles (one persistent CTA per SM):
//   warp 0      producer: 1-D bulk copies of every stage into a 4-deep shared-memory ring.
//   warp 1      gate: waits "A slot free" (mbarrier), releases builders (named barrier SLOT),
//               collects READY, issues the stage's tcgen05.mma (A from TMEM, B from smem).
//   warp 2      image gate: waits "stage landed" (mbarrier) -> named barrier IMG.
//   warps 3..10 builders, two per TMEM lane quarter (thread = row), HW = NH/2 heads each:
//               A = p[r,c,h] * patch_c[r] (or p itself for ext) -> registers -> tcgen05.st.
// Builders never touch an mbarrier or global memory inside the stage loop (p arrives with
// the stage): an already-completed mbarrier try_wait costs ~157 cycles on B200 against ~20
// for bar.sync, and a global load consumed one stage later still exposed ~800 cycles of L2
// latency per stage (tools/sync_probe.cu, tools/l0_trace.py).
// CL = 2: a CTA pair (same node and head group, adjacent row tiles) splits the B blocks of
// every stage between its two producers and multicasts them, halving the weight fill per CTA
// (the kernel is L2->SMEM fill bound); empty[] then counts both CTAs' MMA commits.
template <int PP, int L0_NH, int CL>
__global__ void __launch_bounds__(L0_THREADS, 1) l0_node_kernel(L0NodeArgs a) {
  constexpr int CG = 64 / PP;        // channels per main stage (K = 64 per head per stage)
  constexpr int P = PP == 64 ? 8 : 4;
  constexpr int NBAR = 288;          // gate (or image gate) warp + 8 builder warps
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
    mbar_init(accfull, 1);
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
    // ------------------------------------------------ gate: slot waits + MMA issue
    // Per stage q: READY(q) -> issue the stage's MMAs -> commit (stage + A slot).  The builders
    // wait on the A-slot mbarrier themselves, so a slot hand-off costs one commit->mbarrier
    // hop plus one named-barrier hop.
    const uint32_t idesc = idesc_bf16_f32(128, L0_DH);
    long long q_total = 0;
    for (int u = cid; u < total_units; u += ncl) {
      int g, nmain, next;
      unit_stages(u, g, nmain, next);
      q_total += nmain + next;
    }
    long long q = 0;
    for (int u = cid; u < total_units; u += ncl) {
      int g, nmain, next;
      unit_stages(u, g, nmain, next);
      for (int st = 0; st < nmain + next; ++st, ++q) {
        const int cs = (int)(q % L0_STAGES), cl = (int)(q & 1);
        asm volatile("bar.sync %0, %1;" ::"r"(7 + cl), "r"(NBAR) : "memory");  // READY(q)
        if (lane == 0) L0_TRACE(2, q);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t bd0 = smem_desc(
              smem_u32(smem + cs * L0_STAGE_BYTES + L0_IMG_BYTES + L0_P_BYTES), 1024, 128, 0);
          const uint32_t at0 = tbase + L0_ACC_COLS + cl * L0_SLOT_COLS;
          if (a.debug_mode & 2) {
          } else if (st < nmain) {
#pragma unroll
            for (int h = 0; h < L0_NH; ++h)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_ts(tbase + h * L0_DH, at0 + h * 32 + kk * 8,
                       bd0 + (uint64_t)((h * (L0_DH * 64 * 2) + kk * 2048) >> 4), idesc,
                       (st | kk) != 0);
          } else {
#pragma unroll
            for (int h = 0; h < L0_NH; ++h)
              mma_ts(tbase + h * L0_DH, at0 + h * 32,
                     bd0 + (uint64_t)((h * (L0_DH * 64 * 2)) >> 4), idesc, 1u);
          }
          if (CL == 1) mma_commit(&empty[cs]);
          else mma_commit_mc(&empty[cs], cmask);  // the peer multicasts into this stage too
          mma_commit(&aempty[cl]);
          if (st == nmain + next - 1) mma_commit(accfull);
        }
        __syncwarp();
      }
    }
  } else if (warp == 2) {
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
    // ------------------------------------------------ builders + epilogue (warps 3..10)
    // Two builder warps per TMEM lane quarter split each stage's K = 64 into halves
    // (kh = 0: K 0..31, kh = 1: K 32..63) for all NH heads, so every image row is read from
    // shared memory exactly once (smem bandwidth is shared with TMA writes and MMA reads).
    constexpr int HW = L0_NH / 2;       // epilogue: heads drained per warp
    const int quarter = warp & 3;
    const int hh = (warp - 3) >> 2;     // K half (build) / head half (epilogue)
    const int m = quarter * 32 + lane;  // row within tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    uint8_t* my_out = stage_out + (warp - 3) * (32 * 64);
    uint32_t accphase = 0;
    long long q = 0;
    const int i_l = m / a.wp, jj = m - (m / a.wp) * a.wp;
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
    for (int u = cid; u < total_units; u += ncl) {
      int hg, tile, n;
      decode(u, hg, tile, n);
      int g, nmain, next;
      unit_stages(u, g, nmain, next);
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
      for (int st = 0; st < nmain + next; ++st, ++q) {
        const int cs = (int)(q % L0_STAGES), cl = (int)(q & 1);
        const uint8_t* sI = smem + cs * L0_STAGE_BYTES;
        const uint8_t* sP = sI + L0_IMG_BYTES;
        uint32_t y[L0_NH][16];
        asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(q & 3)), "r"(NBAR) : "memory");  // IMG
        if (warp == 3 && lane == 0) L0_TRACE(3, q);
        const bool ext = st >= nmain;
        if (a.debug_mode & 1) {
#pragma unroll
          for (int h = 0; h < L0_NH; ++h)
#pragma unroll
            for (int e = 0; e < 16; ++e) y[h][e] = 0u;
        } else if (!ext) {
          // this warp's 16 of the 32 A columns: P == 8 -> pixel rows 4kh..4kh+3 of the one
          // channel; P == 4 -> channels 2kh, 2kh+1 of the stage's four
          constexpr int NCC = CG == 1 ? 1 : 2;  // channels touched by this K half
          uint32_t x[16], pv[NCC][2];
#pragma unroll
          for (int ci = 0; ci < NCC; ++ci) {
            const int cc = CG == 1 ? 0 : 2 * hh + ci;
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
                const int py = 4 * hh + r4;
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
#pragma unroll
          for (int h = 0; h < L0_NH; ++h) {
#pragma unroll
            for (int ci = 0; ci < NCC; ++ci) {
              const uint32_t w = pv[ci][h >> 1];
              const uint32_t ph = (h & 1) ? (w & 0xffff0000u) | (w >> 16)
                                          : (w << 16) | (w & 0xffffu);
#pragma unroll
              for (int e = 0; e < 16 / NCC; ++e)
                y[h][ci * (16 / NCC) + e] = mul_bf16x2(x[ci * (16 / NCC) + e], ph);
            }
          }
        } else {
          // ext stage e: A[r, k] = p[r, 16e + k, h] (k < 16); this warp: k in [8hh, 8hh+8)
          const int e = st - nmain;
#pragma unroll
          for (int kc = 0; kc < 4; ++kc) {
            const int cl0 = 8 * hh + 2 * kc;          // channel within the ext block
            const int c0e = 16 * e + cl0;
            uint32_t lo[2] = {0u, 0u}, hi[2] = {0u, 0u};
            if (c0e < g) { if (rowp) p_smem(sI, cl0, lo); else p_const(c0e, lo); }
            if (c0e + 1 < g) { if (rowp) p_smem(sI, cl0 + 1, hi); else p_const(c0e + 1, hi); }
#pragma unroll
            for (int h = 0; h < L0_NH; ++h) {
              const uint32_t a16 = (h & 1) ? (lo[h >> 1] >> 16) : (lo[h >> 1] & 0xffffu);
              const uint32_t b16 = (h & 1) ? (hi[h >> 1] >> 16) : (hi[h >> 1] & 0xffffu);
              y[h][kc] = a16 | (b16 << 16);
            }
          }
        }
        if (warp == 3 && lane == 0) L0_TRACE(4, q);
        // A slot free: the MMAs of stage q-2 (same slot) have completed
        mbar_wait(&aempty[cl], (uint32_t)(((q >> 1) & 1) ^ 1));
        if (warp == 3 && lane == 0) L0_TRACE(5, q);
        tc_fence_after();
        const uint32_t slot_t = tbase + lane_off + L0_ACC_COLS + cl * L0_SLOT_COLS;
        if (!ext) {
#pragma unroll
          for (int h = 0; h < L0_NH; ++h) tmem_st16(slot_t + h * 32 + 16 * hh, y[h]);
        } else {
#pragma unroll
          for (int h = 0; h < L0_NH; ++h) {
            uint32_t y4[4] = {y[h][0], y[h][1], y[h][2], y[h][3]};
            tmem_st4(slot_t + h * 32 + 4 * hh, y4);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        asm volatile("bar.arrive %0, %1;" ::"r"(7 + cl), "r"(NBAR) : "memory");  // READY
      }
      // epilogue: this warp's 32 rows x HW heads, TMEM -> bf16 -> swizzled smem -> coalesced
      // 16-byte stores (8 row segments of 64 B per warp instruction)
      if (warp == 3 && lane == 0) L0_TRACE(6, q);
      mbar_wait(accfull, accphase);
      if (warp == 3 && lane == 0) L0_TRACE(7, q);
      tc_fence_after();
      const long long row0 = (long long)n * R + tile * 128 + quarter * 32;
#pragma unroll 1
      for (int cb = 0; cb < ((a.debug_mode & 32) ? 0 : HW * L0_DH); cb += 32) {
        const int col = (hh * HW) * L0_DH + cb;  // column within this head group
        uint32_t v[32];
        tmem_ld32(tbase + lane_off + col, v);
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint4 o;
          o.x = pack_bf16(__uint_as_float(v[8 * k + 0]), __uint_as_float(v[8 * k + 1]));
          o.y = pack_bf16(__uint_as_float(v[8 * k + 2]), __uint_as_float(v[8 * k + 3]));
          o.z = pack_bf16(__uint_as_float(v[8 * k + 4]), __uint_as_float(v[8 * k + 5]));
          o.w = pack_bf16(__uint_as_float(v[8 * k + 6]), __uint_as_float(v[8 * k + 7]));
          *reinterpret_cast<uint4*>(my_out + lane * 64 + ((k ^ (lane & 3)) << 4)) = o;
        }
        __syncwarp();
        if (!(a.debug_mode & 8)) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rr = i * 8 + (lane >> 2), k = lane & 3;
            const uint4 o =
                *reinterpret_cast<const uint4*>(my_out + rr * 64 + ((k ^ (rr & 3)) << 4));
            *reinterpret_cast<uint4*>(a.ctx + (row0 + rr) * a.D + hg * L0_NH * L0_DH + col +
                                      k * 8) = o;
          }
        }
        __syncwarp();
      }
      tc_fence_before();  // acc reads precede the next unit's first MMA (via READY)
      accphase ^= 1;
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
