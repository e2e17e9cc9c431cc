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
          __nv_bfloat16* dst = a.p + poff + (((long long)hg * R + rows[q]) * g + c) * nh + hl;
          *reinterpret_cast<uint32_t*>(dst) = pack_bf16(p0, p1);
        }
      }
    }
  }
}

// K_p0 v2: the CTA stages every image row it needs (TR positions x g channels) in shared
// memory with 1-D bulk copies, recomputes the logits from shared memory in a second pass
// (mma.sync is cheap next to the HBM read), and writes p through a shared staging tile so
// the global stores are contiguous 16-byte vectors.
template <int NT, int TR>
__global__ void __launch_bounds__(TR * 2) l0_logits_smem_kernel(L0LogitArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                             ~uintptr_t(127));
  const int R = a.B * a.S;
  const int blocks_per_node = R / TR;
  const int n = blockIdx.x / blocks_per_node;
  const int rblk = blockIdx.x - n * blocks_per_node;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int PP = a.P * a.P;
  const int c0 = __ldg(a.node_c0 + n), g = __ldg(a.node_g + n);
  const long long poff = __ldg(a.node_poff + n);
  const int nh = (a.H % 4 == 0) ? 4 : 2;
  const int r0 = rblk * TR;
  const int b = r0 / a.S, s0 = r0 - b * a.S;
  const int chunk = TR * PP;  // elements per channel
  __nv_bfloat16* simg = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* sp = simg + (size_t)g * chunk;                 // [hg][TR][g][nh]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sp + (size_t)TR * g * a.H + 64);
  bar = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(bar) + 7) & ~uintptr_t(7));
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, (uint32_t)(g * chunk * 2));
    const __nv_bfloat16* src = a.img + b * a.img_sb + (long long)(s0 / a.wp) * a.P * a.W;
    for (int c = 0; c < g; ++c)
      bulk_load(simg + (size_t)c * chunk, src + (long long)(c0 + c) * a.img_sc, chunk * 2, bar);
  }
  const int rl[2] = {warp * 16 + gid, warp * 16 + gid + 8};  // rows within the tile
  int rowoff[2];
  float pu[NT][4];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int m = rl[q];
    const int i = m / a.wp, j = m - i * a.wp;
    rowoff[q] = i * a.P * a.W + j * a.P;
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const float* pr0 = a.posU + ((long long)n * a.S + s0 + rl[0]) * a.HP + nt * 8 + 2 * tig;
    const float* pr1 = a.posU + ((long long)n * a.S + s0 + rl[1]) * a.HP + nt * 8 + 2 * tig;
    pu[nt][0] = pr0[0]; pu[nt][1] = pr0[1];
    pu[nt][2] = pr1[0]; pu[nt][3] = pr1[1];
  }
  mbar_wait(bar, 0);

  auto logits = [&](int c, float (&L)[NT][4]) {
    const __nv_bfloat16* cimg = simg + (size_t)c * chunk;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const float* bu = a.bU + (long long)(c0 + c) * a.HP + nt * 8 + 2 * tig;
      const float b0 = __ldg(bu), b1 = __ldg(bu + 1);
      L[nt][0] = pu[nt][0] + b0;
      L[nt][1] = pu[nt][1] + b1;
      L[nt][2] = pu[nt][2] + b0;
      L[nt][3] = pu[nt][3] + b1;
    }
    for (int ks = 0; ks < PP / 16; ++ks) {
      uint32_t af[4];
#pragma unroll
      for (int hk = 0; hk < 2; ++hk) {
        const int k = ks * 16 + hk * 8 + 2 * tig;
        const int py = k / a.P, px = k - py * a.P;
        const int off = py * a.W + px;
        af[hk * 2 + 0] = *reinterpret_cast<const uint32_t*>(cimg + rowoff[0] + off);
        af[hk * 2 + 1] = *reinterpret_cast<const uint32_t*>(cimg + rowoff[1] + off);
      }
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
        const int hg = h / nh, hl = h - hg * nh;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const float p0 = __expf(L[nt][2 * q] - mx[nt][2 * q]) * sm[nt][2 * q];
          const float p1 = __expf(L[nt][2 * q + 1] - mx[nt][2 * q + 1]) * sm[nt][2 * q + 1];
          *reinterpret_cast<uint32_t*>(sp + (((size_t)hg * TR + rl[q]) * g + c) * nh + hl) =
              pack_bf16(p0, p1);
        }
      }
    }
  }
  __syncthreads();
  // copy out: per head group a contiguous run of TR*g*nh bf16
  const int run = TR * g * nh;  // elements, multiple of 8
  for (int hg = 0; hg < a.H / nh; ++hg) {
    const uint4* src = reinterpret_cast<const uint4*>(sp + (size_t)hg * run);
    uint4* dst = reinterpret_cast<uint4*>(a.p + poff + ((long long)hg * R + r0) * g * nh);
    for (int i = threadIdx.x; i < run / 8; i += blockDim.x) dst[i] = src[i];
  }
}

cudaError_t launch_l0_logits(const L0LogitArgs& a, cudaStream_t st) {
  const int R = a.B * a.S;
  const int PP = a.P * a.P;
  // fast path: shared-memory staged (needs whole patch rows per tile and g*PP*TR*2 <= 128 KB;
  // the node sizes are not known here, so the caller passes them bounded via H*?: use gmax)
  const int TR = (32 % a.wp == 0) ? 32 : ((64 % a.wp == 0) ? 64 : 0);
  if (a.p0_smem && TR && a.S % TR == 0 && a.gmax > 0 &&
      (long long)a.gmax * PP * TR * 2 + (long long)TR * a.gmax * a.H * 2 <= 200000 &&
      (TR * a.gmax * (a.H % 4 == 0 ? 4 : 2)) % 8 == 0) {
    const int smem = a.gmax * PP * TR * 2 + TR * a.gmax * a.H * 2 + 64 * 2 + 256;
    const int grid = a.n_nodes * (R / TR);
    void (*k)(L0LogitArgs) = nullptr;
    const int nt = a.HP / 8;
    if (TR == 32) k = nt == 1 ? l0_logits_smem_kernel<1, 32> : nt == 2 ? l0_logits_smem_kernel<2, 32>
                                                              : nt == 4 ? l0_logits_smem_kernel<4, 32> : nullptr;
    else k = nt == 1 ? l0_logits_smem_kernel<1, 64> : nt == 2 ? l0_logits_smem_kernel<2, 64>
                                                     : nt == 4 ? l0_logits_smem_kernel<4, 64> : nullptr;
    if (k) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      k<<<grid, TR * 2, smem, st>>>(a);
      return cudaGetLastError();
    }
  }
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
constexpr int L0_DH = 64;      // head dim (MMA N)
constexpr int L0_STAGES = 4;
constexpr int L0_IMG_BYTES = 16384;                 // 128 rows x 64 K (bf16) per stage
constexpr int L0_B_BYTES = 4 * L0_DH * 64 * 2;  // up to 4 heads x [64 x 64] bf16
constexpr int L0_STAGE_BYTES = L0_IMG_BYTES + L0_B_BYTES;
constexpr int L0_SMEM = L0_STAGES * L0_STAGE_BYTES + 1024 + 256;
constexpr int L0_THREADS = 224;  // producer, gate, 4 builders, image gate
constexpr uint32_t L0_ACC_COLS = 4 * L0_DH;  // accumulator region (NH * 64 used)
constexpr uint32_t L0_SLOT_COLS = 4 * 32;    // A slot: 64 bf16 K per head = 32 columns

// NH = heads per CTA (2 or 4): accumulator NH*64 TMEM columns, A slot NH*32 columns.
//
// Warp roles (one persistent CTA per SM, a "unit" = (node, 128-row tile, head group)):
//   warp 0      producer: 1-D bulk copies of the image rows and the pre-tiled B blocks of
//               every stage (one stage = K 64 per head) into a 4-deep shared-memory ring.
//   warp 1      control: the only warp that waits on mbarriers (full / A-slot free);
//               releases the builders with a named barrier (GO), collects them (READY) and
//               issues the stage's tcgen05.mma (A from TMEM, B from shared memory).
//   warps 2..5  builders (thread = row = TMEM lane): A = p[r,c,h] * patch_c[r] written to
//               one of two TMEM slots with tcgen05.st; then the unit's epilogue.
// Builders never wait on an mbarrier inside the stage loop: an already-completed
// mbarrier try_wait costs ~157 cycles on B200 against ~20 for bar.sync (tools/sync_probe),
// and two of them per stage made the first version handshake-bound.
template <int PP, int L0_NH>
__global__ void __launch_bounds__(L0_THREADS, 1) l0_node_kernel(L0NodeArgs a) {
  constexpr int CG = 64 / PP;        // channels per stage (K = 64 per head per stage)
  constexpr int P = PP == 64 ? 8 : 4;
  constexpr int NBAR = 160;          // control warp + 4 builder warps
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L0_STAGES * L0_STAGE_BYTES);
  uint64_t* empty = full + L0_STAGES;
  uint64_t* aempty = empty + L0_STAGES;
  uint64_t* accfull = aempty + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accfull + 1);

  const int warp = warp_id(), lane = lane_id();
  const int R = a.B * a.S;
  const int n_tiles = R / 128;
  const int HG = a.H / L0_NH;
  const int total_units = a.n_nodes * n_tiles * HG;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < L0_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&aempty[0], 1);
    mbar_init(&aempty[1], 1);
    mbar_init(accfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    // ------------------------------------------------ producer (bulk copies)
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
        const int hg = u % HG;
        const int rest = u / HG;
        const int tile = rest % n_tiles;
        const int n = rest / n_tiles;
        const int c0 = __ldg(a.node_c0 + n), g = __ldg(a.node_g + n);
        const int nmain = (g + CG - 1) / CG;
        const int r0 = tile * 128;
        const int b = r0 / a.S, s0 = r0 - b * a.S;
        const __nv_bfloat16* chunk0 =
            a.img + b * a.img_sb + (long long)(s0 / a.wp) * P * a.W;
        for (int st = 0; st <= nmain; ++st) {
          mbar_wait(&empty[stage], phase ^ 1);  // MMAs of the stage 4 back are done
          uint8_t* sI = smem + stage * L0_STAGE_BYTES;
          uint8_t* sB = sI + L0_IMG_BYTES;
          if (a.debug_mode & 4) {
            mbar_arrive(&full[stage]);
          } else if (st < nmain) {
            const int cv = min(CG, g - st * CG);
            mbar_expect_tx(&full[stage], cv * 128 * PP * 2 + L0_NH * L0_DH * 64 * 2);
            for (int cc = 0; cc < cv; ++cc)
              bulk_load(sI + cc * 128 * PP * 2,
                        chunk0 + (long long)(c0 + st * CG + cc) * a.img_sc, 128 * PP * 2,
                        &full[stage]);
            for (int h = 0; h < L0_NH; ++h)
              bulk_load(sB + h * (L0_DH * 64 * 2),
                        a.Mt + ((long long)(hg * L0_NH + h) * a.C_pad + c0 + st * CG) *
                                   (L0_DH * PP),
                        L0_DH * 64 * 2, &full[stage]);
          } else {
            const int eb = L0_DH * a.KE * 2;
            mbar_expect_tx(&full[stage], L0_NH * eb);
            for (int h = 0; h < L0_NH; ++h)
              bulk_load(sB + h * (L0_DH * 64 * 2),
                        a.Et + ((long long)n * a.H + hg * L0_NH + h) * (L0_DH * a.KE), eb,
                        &full[stage]);
          }
          if (++stage == L0_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ control ("gate"): waits + MMA issue
    // Named barriers (160 threads = this warp + 4 builder warps):
    //   IMG[k%4]   (ids 1..4) stage k's image/B landed   -> builders precompute A in registers
    //   SLOT[k%2]  (ids 5..6) stage k's TMEM A slot free  -> builders store A (4 x tcgen05.st)
    //   READY[k%2] (ids 7..8) stage k's A is in TMEM      -> this warp issues the MMAs
    // Order per stage k: READY(k) -> issue(k) -> wait slot of k+1 (MMAs of k-1 done) -> SLOT(k+1)
    // -> wait full(k+2) -> IMG(k+2).  The MMAs of k+1 are then issued while those of k run.
    const uint32_t idesc = idesc_bf16_f32(128, L0_DH);
    // global stage counter q: smem stage q % 4, A slot q % 2 (phase bits derived from q)
    long long q_total = 0;
    for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
      const int n = (u / HG) / n_tiles;
      q_total += (__ldg(a.node_g + n) + CG - 1) / CG + 1;
    }
    auto slot_free = [&](long long q) {
      if (q < q_total) {
        mbar_wait(&aempty[q & 1], (uint32_t)(((q >> 1) & 1) ^ 1));
        tc_fence_after();
        asm volatile("bar.arrive %0, %1;" ::"r"(5 + (int)(q & 1)), "r"(NBAR) : "memory");
      }
    };
    slot_free(0);
    long long q = 0;
    for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
      const int n = (u / HG) / n_tiles;
      const int g = __ldg(a.node_g + n);
      const int nmain = (g + CG - 1) / CG;
      for (int st = 0; st <= nmain; ++st, ++q) {
        const int cs = (int)(q % L0_STAGES), cl = (int)(q & 1);
        asm volatile("bar.sync %0, %1;" ::"r"(7 + cl), "r"(NBAR) : "memory");  // READY(q)
        tc_fence_after();
        if (elect_one()) {
          const int ksteps = (a.debug_mode & 2) ? 0 : (st < nmain ? 4 : a.KE / 16);
          const uint64_t bd0 =
              smem_desc(smem_u32(smem + cs * L0_STAGE_BYTES + L0_IMG_BYTES), 1024, 128, 0);
          const uint32_t at0 = tbase + L0_ACC_COLS + cl * L0_SLOT_COLS;
          if (ksteps == 4) {
#pragma unroll
            for (int h = 0; h < L0_NH; ++h)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_ts(tbase + h * L0_DH, at0 + h * 32 + kk * 8,
                       bd0 + (uint64_t)((h * (L0_DH * 64 * 2) + kk * 2048) >> 4), idesc,
                       (st | kk) != 0);
          } else {
            for (int h = 0; h < L0_NH; ++h)
              for (int kk = 0; kk < ksteps; ++kk)
                mma_ts(tbase + h * L0_DH, at0 + h * 32 + kk * 8,
                       bd0 + (uint64_t)((h * (L0_DH * 64 * 2) + kk * 2048) >> 4), idesc,
                       (st | kk) != 0);
          }
          mma_commit(&empty[cs]);
          mma_commit(&aempty[cl]);
          if (st == nmain) mma_commit(accfull);
        }
        __syncwarp();
        slot_free(q + 1);
      }
    }
  } else if (warp == 6) {
    // ------------------------------------------------ image gate: full(q) -> IMG(q)
    long long q_total = 0;
    for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
      const int n = (u / HG) / n_tiles;
      q_total += (__ldg(a.node_g + n) + CG - 1) / CG + 1;
    }
    for (long long q = 0; q < q_total; ++q) {
      mbar_wait(&full[q % L0_STAGES], (uint32_t)((q / L0_STAGES) & 1));
      asm volatile("bar.arrive %0, %1;" ::"r"(1 + (int)(q & 3)), "r"(NBAR) : "memory");
    }
  } else {
    // ------------------------------------------------ builders + epilogue (warps 2..5)
    const int quarter = warp & 3;
    const int m = quarter * 32 + lane;  // row within tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    uint32_t accphase = 0;
    long long q = 0;
    const int i_l = m / a.wp, jj = m - (m / a.wp) * a.wp;
    for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
      const int hg = u % HG;
      const int rest = u / HG;
      const int tile = rest % n_tiles;
      const int n = rest / n_tiles;
      const int g = __ldg(a.node_g + n);
      const long long poff = __ldg(a.node_poff + n);
      const int nmain = (g + CG - 1) / CG;
      const int r = tile * 128 + m;
      // p of this (row, head group): channel c at prow + c * pstride, NH heads contiguous
      const __nv_bfloat16* prow =
          a.p_row_mode ? a.p + poff + ((long long)(hg * R + r) * g) * L0_NH
                       : a.p + poff + hg * L0_NH;
      const int pstride = a.p_row_mode ? L0_NH : a.H;
      uint32_t pc[CG][2], pn[CG][2];
      auto load_p = [&](int st, uint32_t (&d)[CG][2]) {
#pragma unroll
        for (int cc = 0; cc < CG; ++cc) {
          const int c = st * CG + cc;
          d[cc][0] = 0u;
          d[cc][1] = 0u;
          if (st < nmain && c < g && !(a.debug_mode & 16)) {
            if (L0_NH == 4) {
              const uint2 v = __ldg(reinterpret_cast<const uint2*>(prow + (long long)c * pstride));
              d[cc][0] = v.x; d[cc][1] = v.y;
            } else {
              d[cc][0] = __ldg(reinterpret_cast<const unsigned int*>(prow + (long long)c * pstride));
            }
          }
        }
      };
      load_p(0, pc);
      for (int st = 0; st <= nmain; ++st, ++q) {
        load_p(st + 1, pn);
        const int cs = (int)(q % L0_STAGES), cl = (int)(q & 1);
        uint32_t y[L0_NH][32];
        asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(q & 3)), "r"(NBAR) : "memory");  // IMG
        if (a.debug_mode & 1) {
#pragma unroll
          for (int h = 0; h < L0_NH; ++h)
#pragma unroll
            for (int e = 0; e < 32; ++e) y[h][e] = 0u;
        } else if (st < nmain) {
          uint32_t x[32];
          const uint8_t* sI = smem + cs * L0_STAGE_BYTES;
#pragma unroll
          for (int cc = 0; cc < CG; ++cc) {
            const bool valid = st * CG + cc < g;
            const __nv_bfloat16* base = reinterpret_cast<const __nv_bfloat16*>(
                                            sI + cc * 128 * PP * 2) +
                                        (i_l * P) * a.W + jj * P;
#pragma unroll
            for (int py = 0; py < P; ++py) {
              if (P == 8) {
                uint4 v = valid ? *reinterpret_cast<const uint4*>(base + py * a.W)
                                : make_uint4(0, 0, 0, 0);
                x[cc * 32 + py * 4 + 0] = v.x; x[cc * 32 + py * 4 + 1] = v.y;
                x[cc * 32 + py * 4 + 2] = v.z; x[cc * 32 + py * 4 + 3] = v.w;
              } else {
                uint2 v = valid ? *reinterpret_cast<const uint2*>(base + py * a.W)
                                : make_uint2(0, 0);
                x[cc * 8 + py * 2 + 0] = v.x; x[cc * 8 + py * 2 + 1] = v.y;
              }
            }
          }
#pragma unroll
          for (int h = 0; h < L0_NH; ++h) {
#pragma unroll
            for (int cc = 0; cc < CG; ++cc) {
              const uint32_t w = pc[cc][h >> 1];
              const uint32_t ph = (h & 1) ? (w & 0xffff0000u) | (w >> 16)
                                          : (w << 16) | (w & 0xffffu);
#pragma unroll
              for (int e = 0; e < 32 / CG; ++e)
                y[h][cc * (32 / CG) + e] = mul_bf16x2(x[cc * (32 / CG) + e], ph);
            }
          }
        } else {
          // ext block: A[r, c] = p[r, c, h], zero-padded to 64 (the MMA reads KE)
          for (int kc = 0; kc < 32; ++kc) {
            const int c = 2 * kc;
            uint32_t lo[2] = {0u, 0u}, hi[2] = {0u, 0u};
            if (c < g) {
              if (L0_NH == 4) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(prow + (long long)c * pstride));
                lo[0] = v.x; lo[1] = v.y;
              } else {
                lo[0] = __ldg(reinterpret_cast<const unsigned int*>(prow + (long long)c * pstride));
              }
            }
            if (c + 1 < g) {
              if (L0_NH == 4) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(prow + (long long)(c + 1) * pstride));
                hi[0] = v.x; hi[1] = v.y;
              } else {
                hi[0] = __ldg(reinterpret_cast<const unsigned int*>(prow + (long long)(c + 1) * pstride));
              }
            }
#pragma unroll
            for (int h = 0; h < L0_NH; ++h) {
              const uint32_t a16 = (h & 1) ? (lo[h >> 1] >> 16) : (lo[h >> 1] & 0xffffu);
              const uint32_t b16 = (h & 1) ? (hi[h >> 1] >> 16) : (hi[h >> 1] & 0xffffu);
              y[h][kc] = a16 | (b16 << 16);
            }
          }
        }
        asm volatile("bar.sync %0, %1;" ::"r"(5 + cl), "r"(NBAR) : "memory");  // SLOT free
        tc_fence_after();
        const uint32_t slot_t = tbase + lane_off + L0_ACC_COLS + cl * L0_SLOT_COLS;
#pragma unroll
        for (int h = 0; h < L0_NH; ++h) tmem_st32(slot_t + h * 32, y[h]);
        tmem_st_wait();
        tc_fence_before();
        asm volatile("bar.arrive %0, %1;" ::"r"(7 + cl), "r"(NBAR) : "memory");  // READY
#pragma unroll
        for (int cc = 0; cc < CG; ++cc) { pc[cc][0] = pn[cc][0]; pc[cc][1] = pn[cc][1]; }
      }
      // epilogue: ctx (fp32 TMEM) -> bf16 HBM  (pos term folded into the next K_gemm)
      mbar_wait(accfull, accphase);
      tc_fence_after();
      __nv_bfloat16* out = a.ctx + ((long long)n * R + r) * a.D + hg * L0_NH * L0_DH;
#pragma unroll 1
      for (int cb = 0; cb < ((a.debug_mode & 32) ? 0 : L0_NH * L0_DH); cb += 32) {
        uint32_t v[32];
        tmem_ld32(tbase + lane_off + cb, v);
        tmem_ld_wait();
        if (a.debug_mode & 8) {
          if (v[0] == 0x7fffffffu && v[31] == 0x7fffffffu) out[cb] = __float2bfloat16(1.f);
          continue;
        }
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 o;
          o.x = pack_bf16(__uint_as_float(v[j + 0]), __uint_as_float(v[j + 1]));
          o.y = pack_bf16(__uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
          o.z = pack_bf16(__uint_as_float(v[j + 4]), __uint_as_float(v[j + 5]));
          o.w = pack_bf16(__uint_as_float(v[j + 6]), __uint_as_float(v[j + 7]));
          *reinterpret_cast<uint4*>(out + cb + j) = o;
        }
      }
      tc_fence_before();  // acc reads precede the next unit's first MMA (via READY)
      accphase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

cudaError_t launch_l0_node(const L0NodeArgs& a, int num_sms, cudaStream_t st) {
  const int R = a.B * a.S;
  const int nh = a.H % 4 == 0 ? 4 : 2;
  if (R % 128 || a.S % 128 || 128 % a.wp || a.H % nh || a.D != a.H * L0_DH || a.KE % 16 ||
      a.KE > 64)
    return cudaErrorInvalidValue;
  const int units = a.n_nodes * (R / 128) * (a.H / nh);
  const int grid = units < num_sms ? units : num_sms;
  void (*kern)(L0NodeArgs) = nullptr;
  if (a.P == 8) kern = nh == 4 ? l0_node_kernel<64, 4> : l0_node_kernel<64, 2>;
  else if (a.P == 4) kern = nh == 4 ? l0_node_kernel<16, 4> : l0_node_kernel<16, 2>;
  else return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L0_SMEM);
  if (e != cudaSuccess) return e;
  kern<<<grid, L0_THREADS, L0_SMEM, st>>>(a);
  return cudaGetLastError();
}

}  // namespace dchag
