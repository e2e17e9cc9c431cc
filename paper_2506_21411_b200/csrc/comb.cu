// Upper-level combine (K_comb) and the patch unfold used by tokenize_channels.
//
// A node above level 0 receives, per child j, the child's output already projected
// into this node's value space, V_j = y_j @ wv_n (folded into the child's K_gemm), and
// its logits L_j = y_j @ U_n.  The node's context is then a per-position weighted sum
//   ctx[r, h-blk] = sum_j softmax_j(L_j[r,h]) * V_j[r, h-blk]       (layers.py:103-123)
// or, for a linear node, ctx[r,:] = sum_j mix_j V_j[r,:]             (layers.py:141-146).
// HBM-bound: reads g*D bf16 + g*H fp32 per row, writes D bf16.
#include <cstdlib>

#include "common.cuh"
#include "dchag_kernels.h"

namespace dchag {

constexpr int COMB_PTAB = 1024;  // softmax table per warp: g * H <= 1024 floats
constexpr int COMB_MAXH = 32;

// One warp per (node, row).  Phase 1: lanes < H own one head each and compute the
// softmax over the g children from coalesced logit rows; weights go to shared memory.
// Phase 2: every lane owns CH 8-column (16-byte) chunks (D = 256 CH) and streams the g
// child rows two at a time, so each lane keeps 2 CH independent 16-byte loads in flight.
// CH is a template parameter so the register arrays are exactly sized (occupancy).
template <int CH>
__global__ void __launch_bounds__(256, CH >= 8 ? 1 : (CH >= 4 ? 2 : 4)) combine_kernel(CombineArgs a) {
  __shared__ float sp[8][COMB_PTAB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // item = (node, row, column segment of <= 2048 columns; D = 4096 rows take two warps)
  const int nseg = (a.D + 2047) / 2048;
  const long long item = (long long)blockIdx.x * 8 + warp;
  const long long nr = item / nseg;
  const int seg = (int)(item - nr * nseg);
  const int n = (int)(nr / a.R);
  const int r = (int)(nr - (long long)n * a.R);
  if (n >= a.n_nodes) return;
  const int first = __ldg(a.node_first + n), g = __ldg(a.node_g + n);
  const int H = a.H, dh = a.D / H;
  const int col0 = seg * 2048, dseg = min(2048, a.D - col0);
  // row r = (rb, rs) with rs < rows_inner: child rows may be interleaved with other channels
  const int rb = r / a.rows_inner, rs = r - rb * a.rows_inner;
  float* p = sp[warp];
  const long long ldv = a.ldv ? a.ldv : a.D;
  const __nv_bfloat16* vbase =
      a.V + (long long)first * a.sVj + (long long)rb * a.sVb + (long long)rs * ldv + col0;
  const int nchunk = dseg / 8;  // chunks of this segment; lanes past it idle (D < 256)
  const bool act = lane < nchunk;  // D >= 256 is a multiple of 256: all lanes active
  // the first two children's value rows are requested before the softmax phase, so their
  // HBM latency overlaps the logit loads
  uint4 v0[CH], v1[CH];
  {
    const uint4* r0 = reinterpret_cast<const uint4*>(vbase);
    const uint4* r1 = reinterpret_cast<const uint4*>(vbase + (g > 1 ? a.sVj : 0));
#pragma unroll
    for (int q = 0; q < CH; ++q) v0[q] = act ? __ldg(r0 + lane + 32 * q) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int q = 0; q < CH; ++q)
      v1[q] = act && g > 1 ? __ldg(r1 + lane + 32 * q) : make_uint4(0, 0, 0, 0);
  }
  if (a.W) {  // explicit per-(child, head) weights (full_cross)
    const float* wr = a.W + ((long long)n * a.R + r) * a.max_g * H;
    for (int i = lane; i < g * H; i += 32) p[i] = __ldg(wr + i);
  } else if (a.mix) {
    for (int j = lane; j < g; j += 32) p[j] = __ldg(a.mix + first + j);
  } else if (lane < H) {
    const float* lr = a.L + (long long)first * a.sLj + (long long)rb * a.sLb +
                      (long long)rs * H + lane;
    float m = -INFINITY;
    for (int j = 0; j < g; ++j) m = fmaxf(m, __ldg(lr + (long long)j * a.sLj));
    float ssum = 0.f;
    for (int j = 0; j < g; ++j) {
      const float e = __expf(__ldg(lr + (long long)j * a.sLj) - m);
      p[j * H + lane] = e;
      ssum += e;
    }
    const float inv = 1.f / ssum;
    for (int j = 0; j < g; ++j) p[j * H + lane] *= inv;
  }
  __syncwarp();
  float acc[CH][8];
#pragma unroll
  for (int q = 0; q < CH; ++q)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[q][e] = 0.f;
  int hq[CH];  // head of each of this lane's chunks
#pragma unroll
  for (int q = 0; q < CH; ++q) hq[q] = (col0 + (lane + 32 * q) * 8) / dh;
  auto accumulate = [&](const uint4 (&v)[CH], int j) {
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      const float pj = (a.mix && !a.W) ? p[j] : p[j * H + hq[q]];
      const uint32_t vv[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[q][2 * e] += pj * bf16lo(vv[e]);
        acc[q][2 * e + 1] += pj * bf16hi(vv[e]);
      }
    }
  };
  accumulate(v0, 0);
  if (g > 1) accumulate(v1, 1);
  int j = 2;
  for (; j + 2 <= g; j += 2) {
    const uint4* r0 = reinterpret_cast<const uint4*>(vbase + (long long)j * a.sVj);
    const uint4* r1 = reinterpret_cast<const uint4*>(vbase + (long long)(j + 1) * a.sVj);
#pragma unroll
    for (int q = 0; q < CH; ++q) v0[q] = act ? __ldg(r0 + lane + 32 * q) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int q = 0; q < CH; ++q) v1[q] = act ? __ldg(r1 + lane + 32 * q) : make_uint4(0, 0, 0, 0);
    accumulate(v0, j);
    accumulate(v1, j + 1);
  }
  if (j < g) {
    const uint4* r0 = reinterpret_cast<const uint4*>(vbase + (long long)j * a.sVj);
#pragma unroll
    for (int q = 0; q < CH; ++q) v0[q] = act ? __ldg(r0 + lane + 32 * q) : make_uint4(0, 0, 0, 0);
    accumulate(v0, j);
  }
  __nv_bfloat16* orow = a.ctx + ((long long)n * a.R + r) * a.D + col0;
  if (!act) return;
#pragma unroll
  for (int q = 0; q < CH; ++q) {
    uint4 o;
    o.x = pack_bf16(acc[q][0], acc[q][1]);
    o.y = pack_bf16(acc[q][2], acc[q][3]);
    o.z = pack_bf16(acc[q][4], acc[q][5]);
    o.w = pack_bf16(acc[q][6], acc[q][7]);
    reinterpret_cast<uint4*>(orow)[lane + 32 * q] = o;
  }
}

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t st) {
  if ((a.D > 256 ? a.D % 256 : a.D % 8) || (a.D > 2048 && a.D % 2048) || (a.D / a.H) % 8 ||
      a.H > COMB_MAXH ||
      a.max_g * (a.mix ? 1 : a.H) > COMB_PTAB)
    return cudaErrorInvalidValue;
  const long long items = (long long)a.n_nodes * a.R * ((a.D + 2047) / 2048);
  const int grid = (int)((items + 7) / 8);
  switch ((min(a.D, 2048) + 255) / 256) {
    case 1: combine_kernel<1><<<grid, 256, 0, st>>>(a); break;
    case 2: combine_kernel<2><<<grid, 256, 0, st>>>(a); break;
    case 4: combine_kernel<4><<<grid, 256, 0, st>>>(a); break;
    case 8: combine_kernel<8><<<grid, 256, 0, st>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// fp32 combine for the fp32 parity mode: ctx[n][r][:] = sum_j w_j(r,h) V_j[r][:] with fp32 V,
// logits / mix as in combine_kernel. One warp per (node, row); lanes over columns.
__global__ void __launch_bounds__(256) combine_f32_kernel(CombineF32Args a) {
  __shared__ float sp[8][COMB_PTAB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long item = (long long)blockIdx.x * 8 + warp;
  const int n = (int)(item / a.R);
  const int r = (int)(item - (long long)n * a.R);
  if (n >= a.n_nodes) return;
  const int first = __ldg(a.node_first + n), g = __ldg(a.node_g + n);
  const int H = a.H, dh = a.D / H;
  float* p = sp[warp];
  if (a.mix) {
    for (int j = lane; j < g; j += 32) p[j] = __ldg(a.mix + first + j);
  } else if (lane < H) {
    const float* lr = a.L + (long long)first * a.sLj + (long long)r * H + lane;
    float m = -INFINITY;
    for (int j = 0; j < g; ++j) m = fmaxf(m, __ldg(lr + (long long)j * a.sLj));
    float ssum = 0.f;
    for (int j = 0; j < g; ++j) {
      const float e = expf(__ldg(lr + (long long)j * a.sLj) - m);
      p[j * H + lane] = e;
      ssum += e;
    }
    for (int j = 0; j < g; ++j) p[j * H + lane] /= ssum;
  }
  __syncwarp();
  for (int c = lane; c < a.D; c += 32) {
    const int h = c / dh;
    float acc = 0.f;
    for (int j = 0; j < g; ++j)
      acc += (a.mix ? p[j] : p[j * H + h]) *
             __ldg(a.V + (long long)(first + j) * a.sVj + (long long)r * a.D + c);
    a.ctx[((long long)n * a.R + r) * a.D + c] = acc;
  }
}

cudaError_t launch_combine_f32(const CombineF32Args& a, cudaStream_t st) {
  if (a.H > COMB_MAXH || a.max_g * (a.mix ? 1 : a.H) > COMB_PTAB || a.D % a.H)
    return cudaErrorInvalidValue;
  const long long items = (long long)a.n_nodes * a.R;
  combine_f32_kernel<<<(unsigned)((items + 7) / 8), 256, 0, st>>>(a);
  return cudaGetLastError();
}

// Level-0 backward value gradient: dV[c][r][d] = p_c[r][h(d)] * G[r][d] (or mix[c] * G), and
// (posV != null) the positional part of dp, Gpos[r][h] = sum_{d in h} G[r][d] posV[r % S][d].
// One thread per (row, 8 columns): G is read once (16 B) and the node's g outputs are
// written as 16-byte stores, consecutive threads on consecutive columns; the dh/8 lanes of
// a head reduce Gpos with shuffles (a row's D/8 chunks and a head's chunks align with warps).
__global__ void __launch_bounds__(256) l0_dv_kernel(int g, int R, int D, int H, int NH,
                                                   const __nv_bfloat16* __restrict__ p,
                                                   const float* __restrict__ mix,
                                                   const __nv_bfloat16* __restrict__ G,
                                                   const float* __restrict__ posV,
                                                   long long ldpos, int S,
                                                   float* __restrict__ Gpos,
                                                   __nv_bfloat16* __restrict__ out) {
  const int dchunks = D >> 3;
  // 32-bit index math (R * D / 8 < 2^31, checked at launch): a 64-bit division per thread
  // was a visible share of this memory-bound kernel
  const unsigned idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (unsigned)R * (unsigned)dchunks) return;  // a multiple of 32: whole warps
  const int r = (int)(idx / (unsigned)dchunks);
  const int d0 = (int)(idx - (unsigned)r * dchunks) * 8;
  const uint4 gv = __ldg(reinterpret_cast<const uint4*>(G + (size_t)r * D + d0));
  const int dh = D / H;
  const int h = d0 / dh;
  const int hg = h / NH, hn = h - hg * NH;
  const float gf[8] = {bf16lo(gv.x), bf16hi(gv.x), bf16lo(gv.y), bf16hi(gv.y),
                       bf16lo(gv.z), bf16hi(gv.z), bf16lo(gv.w), bf16hi(gv.w)};
  if (posV) {
    const float4* pv = reinterpret_cast<const float4*>(posV + (size_t)(r % S) * ldpos + d0);
    const float4 a = __ldg(pv), b = __ldg(pv + 1);
    float acc = gf[0] * a.x + gf[1] * a.y + gf[2] * a.z + gf[3] * a.w +
                gf[4] * b.x + gf[5] * b.y + gf[6] * b.z + gf[7] * b.w;
    const int lanes = dh >> 3;  // 1..32, a power of two
    for (int off = lanes >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & (lanes - 1)) == 0) Gpos[(size_t)r * H + h] = acc;
  }
  if (!out) return;  // positional dp only
  for (int c = 0; c < g; ++c) {
    const float pc = mix ? __ldg(mix + c)
                         : __bfloat162float(p[((size_t)(hg * g + c) * R + r) * NH + hn]);
    uint4 o;
    o.x = pack_bf16(pc * gf[0], pc * gf[1]);
    o.y = pack_bf16(pc * gf[2], pc * gf[3]);
    o.z = pack_bf16(pc * gf[4], pc * gf[5]);
    o.w = pack_bf16(pc * gf[6], pc * gf[7]);
    *reinterpret_cast<uint4*>(out + ((size_t)c * R + r) * D + d0) = o;
  }
}

// Gpos alone (the training step's tcgen05 path), organised by position: a CTA takes one
// position s and a range of images b, so each thread reads its 8 posV columns once and
// reuses them for four images (posV rows were re-read from L2 once per image: 2x the bytes
// of G). The G chunks of BU images are requested before any is reduced.
constexpr int GPOS_BG = 4;   // images per CTA
__global__ void __launch_bounds__(256) l0_gpos_s_kernel(int R, int D, int H, int S,
                                                        const __nv_bfloat16* __restrict__ G,
                                                        const float* __restrict__ posV,
                                                        long long ldpos,
                                                        float* __restrict__ Gpos) {
  const int s = blockIdx.x, b0 = blockIdx.y * GPOS_BG;
  const int nb = min(GPOS_BG, R / S - b0);
  const int dh = D / H, lanes = dh >> 3;  // lanes per head (1..32, a power of two)
  for (int c = threadIdx.x; c < D / 8; c += blockDim.x) {  // D / 8 % 32 == 0: whole warps
    const int d0 = c * 8;
    const float4* pv = reinterpret_cast<const float4*>(posV + (size_t)s * ldpos + d0);
    const float4 pa = __ldg(pv), pb = __ldg(pv + 1);
    uint4 gv[GPOS_BG];
#pragma unroll
    for (int u = 0; u < GPOS_BG; ++u)
      gv[u] = u < nb ? __ldg(reinterpret_cast<const uint4*>(G + ((size_t)(b0 + u) * S + s) * D + d0))
                     : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < GPOS_BG; ++u) {
      float acc = bf16lo(gv[u].x) * pa.x + bf16hi(gv[u].x) * pa.y + bf16lo(gv[u].y) * pa.z +
                  bf16hi(gv[u].y) * pa.w + bf16lo(gv[u].z) * pb.x + bf16hi(gv[u].z) * pb.y +
                  bf16lo(gv[u].w) * pb.z + bf16hi(gv[u].w) * pb.w;
      for (int off = lanes >> 1; off > 0; off >>= 1)
        acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (u < nb && (threadIdx.x & (lanes - 1)) == 0)
        Gpos[((size_t)(b0 + u) * S + s) * H + d0 / dh] = acc;
    }
  }
}

cudaError_t launch_l0_dv(int g, int R, int D, int H, int NH, const __nv_bfloat16* p,
                         const float* mix, const __nv_bfloat16* G, const float* posV,
                         long long ldpos, int S, float* Gpos, __nv_bfloat16* out,
                         cudaStream_t st) {
  const int dh = D / H;
  if (D % H || dh % 8 || dh > 256 || ((dh / 8) & (dh / 8 - 1)) || ((long long)R * (D / 8)) % 32 ||
      (!mix && (NH < 1 || H % NH)) || (posV && (!Gpos || S < 1)))
    return cudaErrorInvalidValue;
  if (!out && posV && R % S == 0 && (D / 8) % 32 == 0 && dh % 8 == 0 && dh / 8 <= 32 &&
      ((ldpos > 0 ? ldpos : D) % 4) == 0) {
    const dim3 grid(S, (R / S + GPOS_BG - 1) / GPOS_BG);
    l0_gpos_s_kernel<<<grid, 256, 0, st>>>(R, D, H, S, G, posV, ldpos > 0 ? ldpos : D, Gpos);
    return cudaGetLastError();
  }
  const long long n = (long long)R * (D / 8);
  if (n >= (1ll << 31)) return cudaErrorInvalidValue;
  l0_dv_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, R, D, H, NH, p, mix, G, posV,
                                                             ldpos > 0 ? ldpos : D, S, Gpos, out);
  return cudaGetLastError();
}

// Metadata token rows of the trunk input (model.py:111-117): out[b][0][d] =
// sum_k meta[b][k] meta_w[k][d] + meta_b[d], written next to the aggregate rows the final
// GEMM's masked epilogue produced (dchag_final_vit).
__global__ void vit_meta_kernel(const float* __restrict__ meta, int kmeta,
                                const float* __restrict__ meta_w, const float* __restrict__ meta_b,
                                void* out, int f32, int S, int D) {
  const int b = blockIdx.y;
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= D) return;
  float a = __ldg(meta_b + d);
  for (int k = 0; k < kmeta; ++k) a = fmaf(__ldg(meta + (size_t)b * kmeta + k), __ldg(meta_w + (size_t)k * D + d), a);
  const size_t o = (size_t)b * (S + 1) * D + d;
  if (f32) reinterpret_cast<float*>(out)[o] = a;
  else reinterpret_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16(a);
}

cudaError_t launch_vit_meta(const float* meta, int kmeta, const float* meta_w,
                            const float* meta_b, void* out, int f32, int B, int S, int D,
                            cudaStream_t st) {
  vit_meta_kernel<<<dim3((D + 127) / 128, B), 128, 0, st>>>(meta, kmeta, meta_w, meta_b, out, f32,
                                                            S, D);
  return cudaGetLastError();
}

// ViT input tokens (model.py:100-117 up to the trunk): out[b][0] = meta_tok[b];
// out[b][1 + s] = agg[b][s] * (1 - mask[b][s]) + mask_token * mask[b][s]. One thread per
// 8 columns of an output row; rows are contiguous runs in both layouts.
template <typename T>
__global__ void __launch_bounds__(256) vit_tokens_kernel(const T* __restrict__ agg,
                                                        const float* __restrict__ mask,
                                                        const float* __restrict__ mask_token,
                                                        const float* __restrict__ meta_tok,
                                                        T* __restrict__ out, int B, int S, int D) {
  const int dchunks = D >> 3;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)B * (S + 1) * dchunks) return;
  const long long row = idx / dchunks;
  const int d0 = (int)(idx - row * dchunks) * 8;
  const int b = (int)(row / (S + 1)), j = (int)(row - (long long)b * (S + 1));
  float v[8];
  if (j == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldg(meta_tok + (size_t)b * D + d0 + i);
  } else {
    const int s = j - 1;
    const float m = __ldg(mask + (size_t)b * S + s);
    const T* src = agg + ((size_t)b * S + s) * D + d0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float a;
      if constexpr (sizeof(T) == 2) a = __bfloat162float(src[i]);
      else a = src[i];
      v[i] = a * (1.f - m) + __ldg(mask_token + d0 + i) * m;
    }
  }
  T* dst = out + row * D + d0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if constexpr (sizeof(T) == 2) dst[i] = __float2bfloat16(v[i]);
    else dst[i] = v[i];
  }
}

cudaError_t launch_vit_tokens(const void* agg, int f32, const float* mask,
                              const float* mask_token, const float* meta_tok, void* out, int B,
                              int S, int D, cudaStream_t st) {
  if (D % 8) return cudaErrorInvalidValue;
  const long long n = (long long)B * (S + 1) * (D / 8);
  const unsigned grid = (unsigned)((n + 255) / 256);
  if (f32)
    vit_tokens_kernel<float><<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(agg), mask,
                                                    mask_token, meta_tok,
                                                    reinterpret_cast<float*>(out), B, S, D);
  else
    vit_tokens_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(agg), mask, mask_token, meta_tok,
        reinterpret_cast<__nv_bfloat16*>(out), B, S, D);
  return cudaGetLastError();
}

// Level-0 backward token-weight gradient without dV in memory (training):
//   T_c[k][d] = sum_r patch_c[r][k] * p_c[r][h(d)] * G[r][d]      (= patch_c^T dV_c)
// One CTA per (channel c, 128 columns of d); 4 warps, warp = 32 k x 64 d (one head);
// the reduction over all R rows runs through 64-row chunks staged by cp.async (double
// buffered, 16-byte XOR swizzle for conflict-free ldmatrix). The A operand patch^T comes
// from ldmatrix.trans and is scaled by p of the warp's head in registers; B = G by
// ldmatrix.trans; mma.sync m16n8k16 bf16 -> fp32.
DEV void mma16816_tg(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
DEV void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
DEV void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
DEV void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
DEV uint32_t scale_bf16x2(uint32_t v, float s0, float s1) {
  return pack_bf16(bf16lo(v) * s0, bf16hi(v) * s1);
}

constexpr int TG_ROWS = 64;                               // rows per chunk
constexpr int TG_G_BYTES = TG_ROWS * 128 * 2;             // G tile: 64 rows x 128 d
constexpr int TG_P_BYTES = TG_ROWS * 64 * 2;              // patch tile: 64 rows x 64 k
constexpr int TG_S_BYTES = TG_ROWS * 4;                   // p word (2 heads, bf16) per row
constexpr int TG_BUF = TG_G_BYTES + TG_P_BYTES + TG_S_BYTES;
constexpr int TG_THREADS = 128;                           // 4 warps: 2 k halves x 2 heads
constexpr int TG_NW = 64;                                 // d columns per warp (one head)

__global__ void __launch_bounds__(TG_THREADS, 4) l0_tgrad_kernel(L0TgradArgs a) {
  extern __shared__ __align__(128) uint8_t tg_smem[];
  const int c = blockIdx.y;
  const int d0 = blockIdx.x * 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int dh = a.D / a.H;
  const int hA = d0 / dh;
  const uint32_t sbase = smem_u32(tg_smem);
  // row split: CTA z reduces chunks [z n / RS, (z+1) n / RS) and adds into T (pre-zeroed)
  const int nall = a.R / TG_ROWS, RS = gridDim.z;
  const int cbeg = (int)((long long)blockIdx.z * nall / RS);
  const int nchunks = (int)((long long)(blockIdx.z + 1) * nall / RS) - cbeg;
  auto load = [&](int i, int buf) {
    const uint32_t sg = sbase + buf * TG_BUF, sp = sg + TG_G_BYTES;
    const int r0 = (cbeg + i) * TG_ROWS;
#pragma unroll
    for (int t = 0; t < 1024 / TG_THREADS; ++t) {  // G: 64 rows x 16 chunks
      const int q = threadIdx.x + t * TG_THREADS, row = q >> 4, ch = q & 15;
      cp_async16(sg + row * 256 + ((ch ^ (row & 7)) << 4),
                 a.G + (size_t)(r0 + row) * a.D + d0 + ch * 8);
    }
    const int b = r0 / a.S, s0 = r0 - b * a.S;
    const __nv_bfloat16* pbase = a.patches + (((size_t)b * a.cnt + a.c0 + c) * a.S + s0) * 64;
#pragma unroll
    for (int t = 0; t < 512 / TG_THREADS; ++t) {  // patch: 64 rows x 8 chunks
      const int q = threadIdx.x + t * TG_THREADS, row = q >> 3, ch = q & 7;
      cp_async16(sp + row * 128 + ((ch ^ (row & 7)) << 4), pbase + (size_t)row * 64 + ch * 8);
    }
    if (!a.mix && threadIdx.x < TG_ROWS) {
      // p of the row's head pair (hA & ~1, +1): one 4-byte word of the [..][R][NH] layout
      const int row = threadIdx.x, hg = hA / a.NH, hn = (hA - hg * a.NH) & ~1;
      cp_async4(sg + TG_G_BYTES + TG_P_BYTES + row * 4,
                a.p + ((size_t)(hg * a.g + c) * a.R + r0 + row) * a.NH + hn);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int mbase = 32 * (warp & 1);   // k rows of this warp
  const int nbase = TG_NW * (warp >> 1);  // d columns (within the CTA's 128)
  // half of the row's p word this warp uses: its head's parity (the word holds hA & ~1, +1)
  const int hw = (d0 + nbase) / dh;
  const int sel = hw & 1;
  const float mixc = a.mix ? __ldg(a.mix + c) : 0.f;
  float acc[2][TG_NW / 8][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < TG_NW / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.f;
  load(0, 0);
  for (int i = 0; i < nchunks; ++i) {
    const int buf = i & 1;
    if (i + 1 < nchunks) {
      load(i + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const uint32_t sg = sbase + buf * TG_BUF, sp = sg + TG_G_BYTES;
    const uint32_t* ss = reinterpret_cast<const uint32_t*>(tg_smem + buf * TG_BUF +
                                                           TG_G_BYTES + TG_P_BYTES);
    auto pval = [&](int r) {
      if (a.mix) return mixc;
      const uint32_t w = ss[r];
      return sel ? bf16hi(w) : bf16lo(w);
    };
    const int j8 = lane >> 3, i8 = lane & 7;
#pragma unroll
    for (int kb = 0; kb < TG_ROWS; kb += 16) {
      // p of the 4 K indices this thread's A fragments carry
      const float p0 = pval(kb + 2 * tig), p1 = pval(kb + 2 * tig + 1);
      const float p8 = pval(kb + 2 * tig + 8), p9 = pval(kb + 2 * tig + 9);
      uint32_t af[2][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int r = kb + i8 + 8 * (j8 >> 1);
        const int col = mbase + mt * 16 + 8 * (j8 & 1);
        ldsm_x4_t(sp + r * 128 + (((col >> 3) ^ (r & 7)) << 4), af[mt]);
        af[mt][0] = scale_bf16x2(af[mt][0], p0, p1);
        af[mt][1] = scale_bf16x2(af[mt][1], p0, p1);
        af[mt][2] = scale_bf16x2(af[mt][2], p8, p9);
        af[mt][3] = scale_bf16x2(af[mt][3], p8, p9);
      }
#pragma unroll
      for (int np = 0; np < TG_NW / 16; ++np) {
        uint32_t bf[4];
        const int r = kb + i8 + 8 * (j8 & 1);
        const int col = nbase + np * 16 + 8 * (j8 >> 1);
        ldsm_x4_t(sg + r * 256 + (((col >> 3) ^ (r & 7)) << 4), bf);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          mma16816_tg(acc[mt][2 * np], af[mt], bf[0], bf[1]);
          mma16816_tg(acc[mt][2 * np + 1], af[mt], bf[2], bf[3]);
        }
      }
    }
    __syncthreads();  // the buffer is refilled by the next iteration's load
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < TG_NW / 8; ++nt) {
      const int m = mbase + mt * 16 + gid;
      const int d = d0 + nbase + nt * 8 + 2 * tig;
      float* o = a.T + ((size_t)c * 64 + m) * a.D + d;
      if (RS == 1) {
        *reinterpret_cast<float2*>(o) = make_float2(acc[mt][nt][0], acc[mt][nt][1]);
        *reinterpret_cast<float2*>(o + 8 * (size_t)a.D) =
            make_float2(acc[mt][nt][2], acc[mt][nt][3]);
      } else {
        atomicAdd(o, acc[mt][nt][0]);
        atomicAdd(o + 1, acc[mt][nt][1]);
        atomicAdd(o + 8 * (size_t)a.D, acc[mt][nt][2]);
        atomicAdd(o + 8 * (size_t)a.D + 1, acc[mt][nt][3]);
      }
    }
}

cudaError_t launch_l0_tgrad(const L0TgradArgs& a, cudaStream_t st) {
  const int dh = a.D / a.H;
  if (a.D % 128 || a.R % TG_ROWS || a.S % TG_ROWS || (dh != 64 && dh != 128) || a.PP != 64 ||
      (!a.mix && a.NH % 2))
    return cudaErrorInvalidValue;
  const int smem = 2 * TG_BUF;
  cudaError_t e = cudaFuncSetAttribute(l0_tgrad_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  // enough CTAs for ~3 per SM: split the row reduction (partials added atomically)
  const int base = (a.D / 128) * a.g;
  // measured (TR node, one B200, 4 warps x 32 k x 64 d): rs 2 0.168 ms, rs 4 0.151, rs 8 0.157
  // (8 warps x 32 x 32: rs 4 0.194)
  int rs = 1;
  while (rs < 4 && base * rs < 6 * 148 && (a.R / TG_ROWS) / (rs * 2) >= 8) rs *= 2;
  if (const char* f = getenv("DCHAG_TG_RS")) rs = atoi(f) > 0 ? atoi(f) : rs;
  if (rs > 1) {
    e = cudaMemsetAsync(a.T, 0, sizeof(float) * (size_t)a.g * a.PP * a.D, st);
    if (e != cudaSuccess) return e;
  }
  l0_tgrad_kernel<<<dim3(a.D / 128, a.g, rs), TG_THREADS, smem, st>>>(a);
  return cudaGetLastError();
}

// Softmax over each parent's children, in place: L[c][r][h] (c = first[j] .. +count[j]-1)
// -> p (layers.py:114-120 for a node above level 0; the operand of K_gemm's COMB epilogue).
// One thread per (parent, row, head); the children's logits of a (row, head) are strided.
__global__ void __launch_bounds__(256) child_softmax_kernel(float* __restrict__ L,
                                                           const int* __restrict__ first,
                                                           const int* __restrict__ count,
                                                           int n_parents, int R, int H) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)n_parents * R * H) return;
  const int j = (int)(idx / ((long long)R * H));
  const long long rh = idx - (long long)j * R * H;
  const int f = __ldg(first + j), g = __ldg(count + j);
  float* base = L + (size_t)f * R * H + rh;
  const size_t st = (size_t)R * H;
  if (g <= 16) {
    // up to 16 children: every logit loaded once, all loads in flight together, one store
    // each (the loop below reads each value three times)
    float v[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) v[c] = c < g ? base[c * st] : -INFINITY;
    float m = -INFINITY;
#pragma unroll
    for (int c = 0; c < 16; ++c) m = fmaxf(m, v[c]);
    float sum = 0.f;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      if (c < g) {
        v[c] = __expf(v[c] - m);
        sum += v[c];
      }
    }
    const float inv = 1.f / sum;
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c < g) base[c * st] = v[c] * inv;
    return;
  }
  float m = -INFINITY;
  for (int c = 0; c < g; ++c) m = fmaxf(m, base[c * st]);
  float sum = 0.f;
  for (int c = 0; c < g; ++c) {
    const float e = __expf(base[c * st] - m);
    base[c * st] = e;
    sum += e;
  }
  const float inv = 1.f / sum;
  for (int c = 0; c < g; ++c) base[c * st] *= inv;
}

cudaError_t launch_child_softmax(float* L, const int* first, const int* count, int n_parents,
                                 int R, int H, cudaStream_t st) {
  const long long n = (long long)n_parents * R * H;
  child_softmax_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(L, first, count, n_parents,
                                                                   R, H);
  return cudaGetLastError();
}

// Level-0 backward, softmax over the node's channels (layers.py:114-120 differentiated,
// tensor.py:201-203): dp_c[r][h] = sum of the row-dot GEMM's 32-column partials of head h
// (dpp [g][D/32][R]) + Gpos[r][h]; dl_c = p_c (dp_c - sum_c' p_c' dp_c'). One thread per
// (head, row), rows fastest (coalesced dpp / dl); dl written [g][H][R] fp32 and bf16.
__global__ void __launch_bounds__(256) l0_softmax_bwd_kernel(
    int g, int R, int H, int NH, int dh, const float* __restrict__ dpp,
    const float* __restrict__ Gpos, const __nv_bfloat16* __restrict__ p,
    float* __restrict__ dl, __nv_bfloat16* __restrict__ dlb) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)R * H) return;
  const int h = (int)(idx / R), r = (int)(idx - (long long)h * R);
  const int hg = h / NH, hn = h - hg * NH, np_ = dh / 32, D32 = H * np_;
  const float gp = __ldg(Gpos + (size_t)r * H + h);
  float sdp = 0.f;
  // channels four at a time: every load of a group is issued before any is consumed
  // (the kernel is load-latency bound; one channel at a time kept ~1 load in flight)
  auto dp_load = [&](int c) {
    float dp = gp;
#pragma unroll 4
    for (int k = 0; k < np_; ++k) dp += __ldg(dpp + ((size_t)c * D32 + h * np_ + k) * R + r);
    return dp;
  };
  auto p_load = [&](int c) {
    return __bfloat162float(p[((size_t)(hg * g + c) * R + r) * NH + hn]);
  };
  int c = 0;
  for (; c + 4 <= g; c += 4) {
    float dp[4], pc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      dp[u] = dp_load(c + u);
      pc[u] = p_load(c + u);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      sdp = fmaf(pc[u], dp[u], sdp);
      dl[((size_t)(c + u) * H + h) * R + r] = dp[u];  // dp for now; scaled below
    }
  }
  for (; c < g; ++c) {
    const float dp = dp_load(c), pc = p_load(c);
    sdp = fmaf(pc, dp, sdp);
    dl[((size_t)c * H + h) * R + r] = dp;
  }
  c = 0;
  for (; c + 4 <= g; c += 4) {
    float d[4], pc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      d[u] = dl[((size_t)(c + u) * H + h) * R + r];
      pc[u] = p_load(c + u);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t o = ((size_t)(c + u) * H + h) * R + r;
      const float v = pc[u] * (d[u] - sdp);
      dl[o] = v;
      dlb[o] = __float2bfloat16(v);
    }
  }
  for (; c < g; ++c) {
    const size_t o = ((size_t)c * H + h) * R + r;
    const float v = p_load(c) * (dl[o] - sdp);
    dl[o] = v;
    dlb[o] = __float2bfloat16(v);
  }
}

// Register-resident variant for g <= 16 channels and dh = 64: one thread per (head, row)
// as above, every dp_c / p_c of the thread in registers -- all loads issued before any is
// consumed, no dl round trip through memory; dl fp32 is optional (the tcgen05 TE path reads
// only the bf16 copy).
template <int GM, int NP>
__global__ void __launch_bounds__(256) l0_softmax_bwd_reg_kernel(
    int g, int R, int H, int NH, const float* __restrict__ dpp,
    const float* __restrict__ Gpos, const __nv_bfloat16* __restrict__ p,
    float* __restrict__ dl, __nv_bfloat16* __restrict__ dlb) {
  const unsigned idx = blockIdx.x * blockDim.x + threadIdx.x;  // R * H < 2^31 (launch)
  if (idx >= (unsigned)R * (unsigned)H) return;
  const int h = (int)(idx / (unsigned)R), r = (int)(idx - (unsigned)h * R);
  const int hg = h / NH, hn = h - hg * NH, D32 = H * NP;
  const float gp = __ldg(Gpos + (size_t)r * H + h);
  float dp[GM], pv[GM];
#pragma unroll
  for (int c = 0; c < GM; ++c) {
    dp[c] = gp;
    pv[c] = 0.f;
    if (c < g) {
#pragma unroll
      for (int k = 0; k < NP; ++k) dp[c] += __ldg(dpp + ((size_t)c * D32 + h * NP + k) * R + r);
      pv[c] = __bfloat162float(p[((size_t)(hg * g + c) * R + r) * NH + hn]);
    }
  }
  float sdp = 0.f;
#pragma unroll
  for (int c = 0; c < GM; ++c) sdp = fmaf(pv[c], dp[c], sdp);
#pragma unroll
  for (int c = 0; c < GM; ++c) {
    if (c < g) {
      const size_t o = ((size_t)c * H + h) * R + r;
      const float v = pv[c] * (dp[c] - sdp);
      if (dl) dl[o] = v;
      dlb[o] = __float2bfloat16(v);
    }
  }
}

// One dp partial per head, NH = 4: one thread per (head group, row) takes the group's four
// heads, so each channel's p is one 8-byte load (the per-head form read 2 bytes of every
// 8: a quarter of each sector) and Gpos one float4.
template <int GM>
__global__ void __launch_bounds__(256) l0_softmax_bwd_hg4_kernel(
    int g, int R, int H, const float* __restrict__ dpp, const float* __restrict__ Gpos,
    const __nv_bfloat16* __restrict__ p, float* __restrict__ dl,
    __nv_bfloat16* __restrict__ dlb) {
  const unsigned idx = blockIdx.x * blockDim.x + threadIdx.x;  // R * H / 4 < 2^31 (launch)
  const int HG = H / 4;
  if (idx >= (unsigned)R * (unsigned)HG) return;
  const int hg = (int)(idx / (unsigned)R), r = (int)(idx - (unsigned)hg * R);
  const float4 gp = __ldg(reinterpret_cast<const float4*>(Gpos + (size_t)r * H + hg * 4));
  float dp[GM][4];
  uint2 pw[GM];
#pragma unroll
  for (int c = 0; c < GM; ++c) {
    dp[c][0] = gp.x; dp[c][1] = gp.y; dp[c][2] = gp.z; dp[c][3] = gp.w;
    pw[c] = make_uint2(0u, 0u);
    if (c < g) {
#pragma unroll
      for (int hn = 0; hn < 4; ++hn)
        dp[c][hn] += __ldg(dpp + ((size_t)c * H + hg * 4 + hn) * R + r);
      pw[c] = __ldg(reinterpret_cast<const uint2*>(p + ((size_t)(hg * g + c) * R + r) * 4));
    }
  }
#pragma unroll
  for (int hn = 0; hn < 4; ++hn) {
    float sdp = 0.f;
#pragma unroll
    for (int c = 0; c < GM; ++c) {
      const uint32_t w = (hn < 2) ? pw[c].x : pw[c].y;
      sdp = fmaf((hn & 1) ? bf16hi(w) : bf16lo(w), dp[c][hn], sdp);
    }
#pragma unroll
    for (int c = 0; c < GM; ++c) {
      if (c < g) {
        const uint32_t w = (hn < 2) ? pw[c].x : pw[c].y;
        const float pc = (hn & 1) ? bf16hi(w) : bf16lo(w);
        const size_t o = ((size_t)c * H + hg * 4 + hn) * R + r;
        const float v = pc * (dp[c][hn] - sdp);
        if (dl) dl[o] = v;
        dlb[o] = __float2bfloat16(v);
      }
    }
  }
}

cudaError_t launch_l0_softmax_bwd(int g, int R, int H, int NH, int dh, const float* dpp,
                                  const float* Gpos, const __nv_bfloat16* p, float* dl,
                                  __nv_bfloat16* dlb, cudaStream_t st) {
  if (dh % 32 || NH < 1 || H % NH) return cudaErrorInvalidValue;
  if (g <= 16 && dh == 32 && NH == 4 && H % 4 == 0 && (long long)R * H < (1ll << 31) &&
      reinterpret_cast<uintptr_t>(p) % 8 == 0) {
    const long long n = (long long)R * (H / 4);
    l0_softmax_bwd_hg4_kernel<16><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        g, R, H, dpp, Gpos, p, dl, dlb);
    return cudaGetLastError();
  }
  if (g <= 16 && (dh == 64 || dh == 32) && (long long)R * H < (1ll << 31)) {
    const long long n = (long long)R * H;
    if (dh == 64)
      l0_softmax_bwd_reg_kernel<16, 2><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
          g, R, H, NH, dpp, Gpos, p, dl, dlb);
    else  // one partial per head (dchag_gemm_rowdot_heads with 64-column groups)
      l0_softmax_bwd_reg_kernel<16, 1><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
          g, R, H, NH, dpp, Gpos, p, dl, dlb);
    return cudaGetLastError();
  }
  if (!dl) return cudaErrorInvalidValue;  // the general kernel keeps dp in dl
  const long long n = (long long)R * H;
  l0_softmax_bwd_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, R, H, NH, dh, dpp,
                                                                     Gpos, p, dl, dlb);
  return cudaGetLastError();
}

// full_cross node weights (see FullCrossArgs; layers.py:125-138 with the rq reduce folded).
// One CTA per (node, row), one warp per head. The row's q and k of every child (g <= 32
// rows of D bf16 each) are staged in shared memory with 16-byte coalesced loads (row
// stride padded by 16 B: conflict-free ldmatrix); each head's g x g logits are tensor-core
// products (mma.sync m16n8k16: A = q_h [child i][dh], B = k_h [child j][dh]) that stay in
// registers through the softmax over j (quad shuffles), the u-weighted sums t_i,h, the
// head sum s_i (shared memory), p2 = softmax_i(s) and w_jh = sum_i p2_i S^h_ij
// (shuffles over the fragment rows).
DEV void mma_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int MI>  // MI = 1: g <= 16 children, 2: g <= 32
__global__ void __launch_bounds__(1024) fullcross_weights_kernel(FullCrossArgs a) {
  extern __shared__ __align__(16) uint8_t fsm_raw[];
  constexpr int NJ = 2 * MI;                       // 8-wide n-tiles over the children j
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const long long item = blockIdx.x;
  const int n = (int)(item / a.R);
  const int r = (int)(item - (long long)n * a.R);
  const int first = __ldg(a.node_first + n), g = __ldg(a.node_g + n);
  const int H = a.H, D = a.D, dh = D / H, h = warp;
  // q | k of child j (contiguous in HBM, 4D bytes) land in one padded smem row by a 1-D bulk
  // copy (no per-chunk address math or register staging); the 16-byte pad keeps the 8 rows
  // of an ldmatrix in different banks
  __shared__ __align__(8) uint64_t landed;
  const int pitch = 4 * D + 16;
  const int rows = 16 * MI;
  uint8_t* qk = fsm_raw;                                             // [rows][pitch]
  uint8_t* pqs = fsm_raw + rows * pitch;                             // positional query row
  float* tsm = reinterpret_cast<float*>(pqs + pitch);                // [H][32] t_i,h
  float* p2s = tsm + H * 32;                                         // [32]
  if (threadIdx.x == 0) {
    mbar_init(&landed, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0) {  // lane j issues child j's copy (lane g the posq row): parallel issue
    if (lane == 0) mbar_expect_tx(&landed, (uint32_t)g * 4 * D + (a.posq ? 2 * D : 0));
    __syncwarp();
    if (lane < g)
      bulk_load(qk + lane * pitch, a.QK + (long long)(first + lane) * a.sQj + (long long)r * a.ldq,
                4 * D, &landed);
    else if (lane == g && a.posq)
      bulk_load(pqs, a.posq + ((long long)n * a.S + r % a.S) * D, 2 * D, &landed);
  }
  // this lane's u values (independent of the copies: in flight during them)
  const float sc = rsqrtf((float)dh);
  float uj[2 * MI][2];
#pragma unroll
  for (int nj = 0; nj < 2 * MI; ++nj)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = nj * 8 + 2 * tig + e;
      uj[nj][e] = j < g ? __ldg(a.u + (long long)(first + j) * a.sUj + (long long)r * H + h) : 0.f;
    }
  mbar_wait(&landed, 0);
  __syncthreads();
  // logits S^h = q_h k_h^T / sqrt(dh) on the tensor cores
  float acc[MI][NJ][4];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[mi][nj][e] = 0.f;
  const int mat = lane >> 3, rr = lane & 7;
  for (int k0 = 0; k0 < dh; k0 += 16) {
    const int col = (h * dh + k0) * 2;
    uint32_t af[MI][4];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      // children beyond g read child 0's row (finite; their logits rows / columns are masked)
      int row = mi * 16 + rr + 8 * (mat & 1);
      row = row < g ? row : 0;
      ldsm_x4(smem_u32(qk + row * pitch + col + 16 * (mat >> 1)), af[mi]);
    }
    // the positional query (q_i + pos q) . k_j = q_i . k_j + posq . k_j: one more product
    // with the posq row broadcast to all 16 fragment rows (no in-place add over g rows)
    uint32_t pf[4];
    if (a.posq) ldsm_x4(smem_u32(pqs + col + 16 * (mat >> 1)), pf);
#pragma unroll
    for (int np = 0; np < NJ / 2; ++np) {
      uint32_t bf[4];
      int row = np * 16 + rr + 8 * (mat >> 1);
      row = row < g ? row : 0;
      ldsm_x4(smem_u32(qk + row * pitch + 2 * D + col + 16 * (mat & 1)), bf);
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        mma_16816(acc[mi][2 * np], af[mi], bf[0], bf[1]);
        mma_16816(acc[mi][2 * np + 1], af[mi], bf[2], bf[3]);
        if (a.posq) {
          mma_16816(acc[mi][2 * np], pf, bf[0], bf[1]);
          mma_16816(acc[mi][2 * np + 1], pf, bf[2], bf[3]);
        }
      }
    }
  }
  // softmax over j of every row i (quad shuffles), t_i = sum_j S_ij u_jh
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {             // fragment rows gid (hr 0) and gid + 8
      float m = -INFINITY;
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = nj * 8 + 2 * tig + e;
          const float v = acc[mi][nj][2 * hr + e] * sc;
          acc[mi][nj][2 * hr + e] = v;
          if (j < g) m = fmaxf(m, v);
        }
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
      float sum = 0.f;
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = nj * 8 + 2 * tig + e;
          const float ev = j < g ? __expf(acc[mi][nj][2 * hr + e] - m) : 0.f;
          acc[mi][nj][2 * hr + e] = ev;
          sum += ev;
        }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      const float inv = 1.f / sum;
      float tu = 0.f;
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          acc[mi][nj][2 * hr + e] *= inv;
          tu = fmaf(acc[mi][nj][2 * hr + e], uj[nj][e], tu);
        }
      tu += __shfl_xor_sync(0xffffffffu, tu, 1);
      tu += __shfl_xor_sync(0xffffffffu, tu, 2);
      if (tig == 0) tsm[h * 32 + mi * 16 + gid + 8 * hr] = tu;
    }
  __syncthreads();
  // s_i = sum_h t_i,h ; p2 = softmax_i(s)  (warp 0)
  if (warp == 0) {
    float sv = -INFINITY;
    if (lane < g) {
      sv = 0.f;
      for (int hh = 0; hh < H; ++hh) sv += tsm[hh * 32 + lane];
    }
    float m = sv;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float e = lane < g ? __expf(sv - m) : 0.f;
    float sum = e;
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    p2s[lane] = e / sum;
  }
  __syncthreads();
  // w_jh = sum_i p2_i S_ij : per column j, reduce over the fragment rows (gid, m-tiles)
  float pr[MI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) pr[mi][hr] = p2s[mi * 16 + gid + 8 * hr];  // 0 beyond g
#pragma unroll
  for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      float wj = 0.f;
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) wj = fmaf(pr[mi][hr], acc[mi][nj][2 * hr + e], wj);
      wj += __shfl_xor_sync(0xffffffffu, wj, 4);
      wj += __shfl_xor_sync(0xffffffffu, wj, 8);
      wj += __shfl_xor_sync(0xffffffffu, wj, 16);
      const int j = nj * 8 + 2 * tig + e;
      if (gid == 0 && j < g) {
        if (a.pout) {
          const int hg = h / a.nh;
          a.pout[__ldg(a.node_poff + n) + (((long long)hg * g + j) * a.R + r) * a.nh + h % a.nh] =
              __float2bfloat16(wj);
        } else {
          a.w[(((long long)n * a.R + r) * a.max_g + j) * H + h] = wj;
        }
      }
    }
}

cudaError_t launch_fullcross_weights(const FullCrossArgs& a, cudaStream_t st) {
  const int dh = a.D / a.H;
  if (a.max_g > 32 || a.H > 32 || dh % 16 || a.H < 1 || a.D % 8) return cudaErrorInvalidValue;
  const int MI = a.max_g > 16 ? 2 : 1;
  const size_t smem = (size_t)(16 * MI + 1) * (a.D * 4 + 16) + ((size_t)a.H * 32 + 32) * 4;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = MI == 2 ? fullcross_weights_kernel<2> : fullcross_weights_kernel<1>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)((long long)a.n_nodes * a.R), a.H * 32, smem, st>>>(a);
  return cudaGetLastError();
}

// Backward of a full_cross node (layers.py:125-138 with sdp_attention :49-64, the rq reduce
// folded as in fullcross_weights_kernel), one CTA per (node, row), one warp per head, g <= 16.
// Recomputes S^h = softmax_j(q_i k_j / sqrt(dh)) (tensor cores), t, p2, w, then with
// G = dLoss/dctx:  dw_jh = G_h . v_jh;  dp2_i = sum_hj S_ij dw_jh;  dt = p2 (dp2 - p2.dp2);
// dS_ij = p2_i dw_j + dt_i u_j;  du_j = sum_i dt_i S_ij;  dL = S (dS - rowsum(S dS));
// dq_i = sum_j dL_ij k_j / sqrt(dh);  dk_j = sum_i dL_ij q_i / sqrt(dh);
// dv_jh = w_jh G_h + du_jh a_h;  dA[row][h-blk] = sum_j du_jh v_jh  (-> d(wo rq)).
__global__ void __launch_bounds__(1024) fullcross_bwd_kernel(FullCrossBwdArgs a) {
  extern __shared__ __align__(16) uint8_t fsm_raw[];
  __shared__ __align__(8) uint64_t landed;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const long long item = blockIdx.x;
  const int n = (int)(item / a.R);
  const int r = (int)(item - (long long)n * a.R);
  const int first = __ldg(a.node_first + n), g = __ldg(a.node_g + n);
  const int H = a.H, D = a.D, dh = D / H, h = warp;
  const int pitch = 6 * D + 16;                    // q | k | v row of a child (+ pad)
  uint8_t* qkv = fsm_raw;                          // [16][pitch]
  float* Gs = reinterpret_cast<float*>(fsm_raw + 16 * pitch);       // [D]
  float* tsm = Gs + D;                             // [H][16] t_i,h, then dp2 parts
  float* p2s = tsm + H * 16;                       // [16]
  float* dts = p2s + 16;                           // [16]
  float* dw = dts + 16;                            // [H][16]
  float* dLs = dw + H * 16;                        // [H][16][17]
  if (threadIdx.x == 0) {
    mbar_init(&landed, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&landed, (uint32_t)g * 6 * D);
    for (int j = 0; j < g; ++j)
      bulk_load(qkv + j * pitch, a.QKV + (long long)(first + j) * a.sQj + (long long)r * a.ldq,
                6 * D, &landed);
  }
  for (int t = threadIdx.x; t < (16 - g) * (6 * D / 16); t += blockDim.x)
    *reinterpret_cast<uint4*>(qkv + (g + t / (6 * D / 16)) * pitch + (t % (6 * D / 16)) * 16) =
        make_uint4(0, 0, 0, 0);
  for (int d = threadIdx.x; d < D; d += blockDim.x)
    Gs[d] = __ldg(a.G + ((long long)n * a.R + r) * D + d);
  mbar_wait(&landed, 0);
  __syncthreads();
  auto qv = [&](int j, int d) {  // q (0), k (D), v (2D) element of child j
    return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(qkv + j * pitch + d * 2));
  };
  // ---- logits and S (as fullcross_weights_kernel, MI = 1)
  float acc[2][4];
#pragma unroll
  for (int nj = 0; nj < 2; ++nj)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nj][e] = 0.f;
  const int mat = lane >> 3, rr = lane & 7;
  for (int k0 = 0; k0 < dh; k0 += 16) {
    const int col = (h * dh + k0) * 2;
    uint32_t af[4], bf[4];
    ldsm_x4(smem_u32(qkv + (rr + 8 * (mat & 1)) * pitch + col + 16 * (mat >> 1)), af);
    ldsm_x4(smem_u32(qkv + (rr + 8 * (mat >> 1)) * pitch + 2 * D + col + 16 * (mat & 1)), bf);
    mma_16816(acc[0], af, bf[0], bf[1]);
    mma_16816(acc[1], af, bf[2], bf[3]);
  }
  const float sc = rsqrtf((float)dh);
  float uj[2][2];
#pragma unroll
  for (int nj = 0; nj < 2; ++nj)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = nj * 8 + 2 * tig + e;
      uj[nj][e] = j < g ? __ldg(a.u + (long long)(first + j) * a.R * H + (long long)r * H + h) : 0.f;
    }
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    float m = -INFINITY;
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = nj * 8 + 2 * tig + e;
        acc[nj][2 * hr + e] *= sc;
        if (j < g) m = fmaxf(m, acc[nj][2 * hr + e]);
      }
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
    float sum = 0.f;
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = nj * 8 + 2 * tig + e;
        const float ev = j < g ? __expf(acc[nj][2 * hr + e] - m) : 0.f;
        acc[nj][2 * hr + e] = ev;
        sum += ev;
      }
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    const float inv = 1.f / sum;
    float tu = 0.f;
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        acc[nj][2 * hr + e] *= inv;                         // S_ij
        tu = fmaf(acc[nj][2 * hr + e], uj[nj][e], tu);
      }
    tu += __shfl_xor_sync(0xffffffffu, tu, 1);
    tu += __shfl_xor_sync(0xffffffffu, tu, 2);
    if (tig == 0) tsm[h * 16 + gid + 8 * hr] = tu;
  }
  // dw_jh = G_h . v_jh  (lanes over the head's dh columns, one child at a time)
  for (int j = 0; j < 16; ++j) {
    float part = 0.f;
    if (j < g)
      for (int d = lane; d < dh; d += 32) part = fmaf(Gs[h * dh + d], qv(j, 2 * D + h * dh + d), part);
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) dw[h * 16 + j] = part;
  }
  __syncthreads();
  if (warp == 0) {  // p2 = softmax_i(sum_h t)
    float sv = -INFINITY;
    if (lane < g) {
      sv = 0.f;
      for (int hh = 0; hh < H; ++hh) sv += tsm[hh * 16 + lane];
    }
    float m = sv;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float e = lane < g ? __expf(sv - m) : 0.f;
    float sum = e;
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane < 16) p2s[lane] = e / sum;
  }
  __syncthreads();
  // w_jh = sum_i p2_i S_ij (kept per lane for its columns) and dp2 parts = sum_j S_ij dw_j
  float wj[2][2], dwj[2][2];
#pragma unroll
  for (int nj = 0; nj < 2; ++nj)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = nj * 8 + 2 * tig + e;
      dwj[nj][e] = dw[h * 16 + j];
      float x = p2s[gid] * acc[nj][e] + p2s[gid + 8] * acc[nj][2 + e];
      x += __shfl_xor_sync(0xffffffffu, x, 4);
      x += __shfl_xor_sync(0xffffffffu, x, 8);
      x += __shfl_xor_sync(0xffffffffu, x, 16);
      wj[nj][e] = x;
    }
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    float dpp = 0.f;
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) dpp = fmaf(acc[nj][2 * hr + e], dwj[nj][e], dpp);
    dpp += __shfl_xor_sync(0xffffffffu, dpp, 1);
    dpp += __shfl_xor_sync(0xffffffffu, dpp, 2);
    if (tig == 0) tsm[h * 16 + gid + 8 * hr] = dpp;   // t no longer needed
  }
  __syncthreads();
  if (warp == 0) {  // dt_i = p2_i (dp2_i - sum_i' p2_i' dp2_i')
    float dp2 = 0.f;
    if (lane < g)
      for (int hh = 0; hh < H; ++hh) dp2 += tsm[hh * 16 + lane];
    const float p2 = lane < 16 ? p2s[lane] : 0.f;
    float s = p2 * dp2;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane < 16) dts[lane] = lane < g ? p2 * (dp2 - s) : 0.f;
  }
  __syncthreads();
  // dS_ij = p2_i dw_j + dt_i u_j ; du_j = sum_i dt_i S_ij ; dL = S (dS - rowsum(S dS))
  float duj[2][2];
#pragma unroll
  for (int nj = 0; nj < 2; ++nj)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      float x = dts[gid] * acc[nj][e] + dts[gid + 8] * acc[nj][2 + e];
      x += __shfl_xor_sync(0xffffffffu, x, 4);
      x += __shfl_xor_sync(0xffffffffu, x, 8);
      x += __shfl_xor_sync(0xffffffffu, x, 16);
      duj[nj][e] = x;
    }
  float* dL = dLs + h * 16 * 17;
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int i = gid + 8 * hr;
    float dS[2][2], rs = 0.f;
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        dS[nj][e] = p2s[i] * dwj[nj][e] + dts[i] * uj[nj][e];
        rs = fmaf(acc[nj][2 * hr + e], dS[nj][e], rs);
      }
    rs += __shfl_xor_sync(0xffffffffu, rs, 1);
    rs += __shfl_xor_sync(0xffffffffu, rs, 2);
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = nj * 8 + 2 * tig + e;
        dL[i * 17 + j] = (i < g && j < g) ? acc[nj][2 * hr + e] * (dS[nj][e] - rs) * sc : 0.f;
      }
  }
  // per-child scalars of this head for the value gradient, broadcast via smem (reuse dw)
  __syncwarp();
  float* wsm = dw + h * 16;   // dw no longer needed: holds w_j, then du_j in the next slot
  if (gid == 0) {
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) wsm[nj * 8 + 2 * tig + e] = wj[nj][e];
  }
  float* dusm = dLs + H * 16 * 17 + h * 16;
  if (gid == 0) {
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) dusm[nj * 8 + 2 * tig + e] = duj[nj][e];
  }
  __syncwarp();
  // dq, dk, dv (bf16) and dA of this head's dh columns; lanes over columns
  for (int d = lane; d < dh; d += 32) {
    const int c = h * dh + d;
    const float ad = __ldg(a.a + (long long)n * D + c);
    float dAsum = 0.f;
    for (int j = 0; j < g; ++j) {
      float dq = 0.f, dk = 0.f;
      for (int jj = 0; jj < g; ++jj) {
        dq = fmaf(dL[j * 17 + jj], qv(jj, D + c), dq);     // dq_j = sum_jj dL[j][jj] k_jj
        dk = fmaf(dL[jj * 17 + j], qv(jj, c), dk);         // dk_j = sum_jj dL[jj][j] q_jj
      }
      const float vj = qv(j, 2 * D + c);
      const float dv = wsm[j] * Gs[c] + dusm[j] * ad;
      dAsum = fmaf(dusm[j], vj, dAsum);
      __nv_bfloat16* o = a.dQKV + (long long)(first + j) * a.sQj + (long long)r * a.ldq;
      o[c] = __float2bfloat16(dq);
      o[D + c] = __float2bfloat16(dk);
      o[2 * D + c] = __float2bfloat16(dv);
    }
    a.dA[((long long)n * a.R + r) * D + c] = dAsum;
  }
}

cudaError_t launch_fullcross_bwd(const FullCrossBwdArgs& a, cudaStream_t st) {
  const int dh = a.D / a.H;
  if (a.max_g > 16 || a.H > 32 || dh % 16 || a.D % 8) return cudaErrorInvalidValue;
  const size_t smem = (size_t)16 * (a.D * 6 + 16) + (size_t)a.D * 4 +
                      ((size_t)a.H * 16 * 2 + 32 + (size_t)a.H * 16 * 17 + (size_t)a.H * 16) * 4;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(fullcross_bwd_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fullcross_bwd_kernel<<<(unsigned)((long long)a.n_nodes * a.R), a.H * 32, smem, st>>>(a);
  return cudaGetLastError();
}

// Backward of the combine (layers.py:103-123 / :141-146 restated; reference tape
// tensor.py:168-205): given g = dLoss/dctx[n][r][:] (fp32) and the saved child values
// V_j (bf16) and logits L_j (fp32, attention) or mix (linear):
//   p_jh   = softmax_j(L_j[r,h])                    (recomputed)
//   dp_jh  = g[r, h-blk] . V_j[r, h-blk]
//   dL_jh  = p_jh (dp_jh - sum_j' p_j'h dp_j'h)      -> dL  [child][R][H]   (attention)
//   gV_j   = p_jh * g[r, h-blk]                      -> gV  [child][R][D]   bf16
//   dmix_j(r) = g[r] . V_j[r]                        -> dm  [child][R]      (linear)
// One warp per (node, row); lanes own 8-column chunks, head dot products reduced with
// shuffles inside the dh/8 lanes of a head.
// SPLIT = 2 (attention nodes): a row's D columns are shared by two warps (half the heads
// each), so a warp holds half the G row and half the value-row prefetch -- twice the warps
// per SM, twice the bytes in flight
template <int SPLIT>
__global__ void __launch_bounds__(128) combine_bwd_kernel(CombineBwdArgs a) {
  __shared__ float sp[4][COMB_PTAB];
  __shared__ float sd[4][COMB_PTAB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long item = ((long long)blockIdx.x * 4 + warp) / SPLIT;
  const int part_id = (int)(((long long)blockIdx.x * 4 + warp) % SPLIT);
  const int n = (int)(item / a.R);
  const int r = (int)(item - (long long)n * a.R);
  if (n >= a.n_nodes) return;
  const int first = __ldg(a.node_first + n), g = __ldg(a.node_g + n);
  const int H = a.H, dh = a.D / H, cpl = dh / 8;  // chunks per head
  float* p = sp[warp];
  float* dp = sd[warp];
  if (a.mix) {
    for (int j = lane; j < g; j += 32) p[j] = __ldg(a.mix + first + j);
  } else if (lane < H) {
    const float* lr = a.L + (long long)first * a.sLj + (long long)r * H + lane;
    float m = -INFINITY;
    for (int j = 0; j < g; ++j) m = fmaxf(m, __ldg(lr + (long long)j * a.sLj));
    float ssum = 0.f;
    for (int j = 0; j < g; ++j) {
      const float e = __expf(__ldg(lr + (long long)j * a.sLj) - m);
      p[j * H + lane] = e;
      ssum += e;
    }
    const float inv = 1.f / ssum;
    for (int j = 0; j < g; ++j) p[j * H + lane] *= inv;
  }
  __syncwarp();
  constexpr int QN = 8 / SPLIT;                 // 16-byte chunks per lane (D <= 2048)
  const int nchunk = a.D / 8 / SPLIT;           // this warp's chunks: [cbase, cbase + nchunk)
  const int cbase = part_id * nchunk;
  const int per_lane = (nchunk + 31) / 32;
  float gr[QN][8];
  const float* grow = a.G + ((long long)n * a.R + r) * a.D;
#pragma unroll
  for (int q = 0; q < QN; ++q) {
    if (q < per_lane && lane + 32 * q < nchunk) {
      const int ch = cbase + lane + 32 * q;
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(grow) + 2 * ch);
      const float4 g1 = __ldg(reinterpret_cast<const float4*>(grow) + 2 * ch + 1);
      gr[q][0] = g0.x; gr[q][1] = g0.y; gr[q][2] = g0.z; gr[q][3] = g0.w;
      gr[q][4] = g1.x; gr[q][5] = g1.y; gr[q][6] = g1.z; gr[q][7] = g1.w;
    }
  }
  // child j + 1's value row is requested while child j is reduced (software pipeline)
  auto load_v = [&](int j, uint4 (&v)[QN]) {
    const __nv_bfloat16* vrow = a.V + (long long)(first + j) * a.sVj + (long long)r * a.D;
#pragma unroll
    for (int q = 0; q < QN; ++q) {
      const int ch = lane + 32 * q;
      v[q] = (q < per_lane && ch < nchunk)
                 ? __ldg(reinterpret_cast<const uint4*>(vrow) + cbase + ch)
                 : make_uint4(0, 0, 0, 0);
    }
  };
  uint4 vcur[QN], vnext[QN];
  if (g > 0) load_v(0, vnext);
  for (int j = 0; j < g; ++j) {
#pragma unroll
    for (int q = 0; q < QN; ++q) vcur[q] = vnext[q];
    if (j + 1 < g) load_v(j + 1, vnext);
    __nv_bfloat16* gvrow = a.sGj ? a.gV + (long long)(first + j) * a.sGj + (long long)r * a.ldg
                                 : a.gV + (long long)(first + j) * a.sVj + (long long)r * a.D;
    float dm_part = 0.f;
#pragma unroll
    for (int q = 0; q < QN; ++q) {
      float part = 0.f;
      const int ch = cbase + lane + 32 * q;
      const bool ok = q < per_lane && lane + 32 * q < nchunk;
      if (ok) {
        const uint4 v = vcur[q];
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          part += gr[q][2 * e] * bf16lo(vv[e]) + gr[q][2 * e + 1] * bf16hi(vv[e]);
        const float pj = a.mix ? p[j] : p[j * H + (ch * 8) / dh];
        uint4 o;
        o.x = pack_bf16(pj * gr[q][0], pj * gr[q][1]);
        o.y = pack_bf16(pj * gr[q][2], pj * gr[q][3]);
        o.z = pack_bf16(pj * gr[q][4], pj * gr[q][5]);
        o.w = pack_bf16(pj * gr[q][6], pj * gr[q][7]);
        reinterpret_cast<uint4*>(gvrow)[ch] = o;
      }
      if (a.mix) {
        dm_part += part;
      } else {
        // reduce over the cpl lanes of one head (cpl divides 32: consecutive lanes)
        for (int off = cpl >> 1; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
        if (ok && (lane % cpl) == 0) dp[j * H + (ch * 8) / dh] = part;
      }
    }
    if (a.mix) {
      for (int off = 16; off > 0; off >>= 1) dm_part += __shfl_xor_sync(0xffffffffu, dm_part, off);
      if (lane == 0) a.dm[(long long)(first + j) * a.R + r] = dm_part;
    }
  }
  __syncwarp();
  const int hd = part_id * (H / SPLIT) + lane;  // this warp's heads
  if (!a.mix && lane < H / SPLIT) {
    float s = 0.f;
    for (int j = 0; j < g; ++j) s += p[j * H + hd] * dp[j * H + hd];
    for (int j = 0; j < g; ++j) {
      const float v = p[j * H + hd] * (dp[j * H + hd] - s);
      if (a.dL) a.dL[(long long)(first + j) * a.sLj + (long long)r * H + hd] = v;
      if (a.sGj)
        a.gV[(long long)(first + j) * a.sGj + (long long)r * a.ldg + a.D + hd] =
            __float2bfloat16(v);
    }
  }
}

cudaError_t launch_combine_bwd(const CombineBwdArgs& a, cudaStream_t st) {
  const int dh = a.D / a.H;
  if (a.D % 8 || a.D > 2048 || dh % 8 || 32 % (dh / 8 > 32 ? 64 : dh / 8) || a.H > COMB_MAXH ||
      a.max_g * (a.mix ? 1 : a.H) > COMB_PTAB)
    return cudaErrorInvalidValue;
  const long long items = (long long)a.n_nodes * a.R;
  // two warps per row for attention nodes whose head split keeps whole heads per warp
  if (!a.mix && a.H % 2 == 0 && (a.D / 16) % dh == 0 && a.D >= 512) {
    combine_bwd_kernel<2><<<(int)((2 * items + 3) / 4), 128, 0, st>>>(a);
  } else {
    combine_bwd_kernel<1><<<(int)((items + 3) / 4), 128, 0, st>>>(a);
  }
  return cudaGetLastError();
}

// images [B][C][H][W] (strided) -> patches [B][C][S][P*P]: one CTA per (b, c, patch row):
// the strip's P image rows are read with 16-byte coalesced loads into shared memory and its
// wp*P*P outputs, one contiguous run, written back with 16-byte coalesced stores.
__global__ void __launch_bounds__(256) unfold_kernel(const __nv_bfloat16* img, long long sb,
                                                     long long sc, int B, int C, int Himg, int W,
                                                     int P, __nv_bfloat16* out) {
  extern __shared__ __align__(16) __nv_bfloat16 strip[];   // [P][W]
  const int hp = Himg / P, wp = W / P, S = hp * wp;
  const int i = blockIdx.x % hp;
  const int bc = blockIdx.x / hp;
  const int c = bc % C, b = bc / C;
  const __nv_bfloat16* src = img + b * sb + c * sc + (long long)i * P * W;
  const int n = P * W;                       // elements of the strip (multiple of 8)
  for (int e = threadIdx.x * 8; e < n; e += blockDim.x * 8) {
    const int py = e / W, x = e - py * W;
    *reinterpret_cast<uint4*>(strip + e) =
        __ldg(reinterpret_cast<const uint4*>(src + (long long)py * W + x));
  }
  __syncthreads();
  __nv_bfloat16* dst = out + (((long long)b * C + c) * S + (long long)i * wp) * P * P;
  for (int e = threadIdx.x * 8; e < n; e += blockDim.x * 8) {
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int o = e + q, j = o / (P * P), k = o - j * P * P;
      v[q] = strip[(k / P) * W + j * P + (k % P)];
    }
    *reinterpret_cast<uint4*>(dst + e) = *reinterpret_cast<const uint4*>(v);
  }
}

// P = 8 / 16: a CTA takes ns consecutive strips of one image (one contiguous input run and
// one contiguous output run), and every 16-byte output chunk -- eight consecutive pixels of
// one patch row -- is a single 16-byte shared-memory read (shift / mask index math).
template <int P>
__global__ void __launch_bounds__(256) unfold_wide_kernel(const __nv_bfloat16* img,
                                                          long long sb, long long sc, int C,
                                                          int Himg, int W, int ns,
                                                          __nv_bfloat16* out) {
  extern __shared__ __align__(16) __nv_bfloat16 strip[];   // [ns * P][W]
  const int hp = Himg / P, wp = W / P, S = hp * wp, nblk = hp / ns;
  const int i0 = (blockIdx.x % nblk) * ns;
  const int bc = blockIdx.x / nblk;
  const int c = bc % C, b = bc / C;
  const __nv_bfloat16* src = img + b * sb + c * sc + (long long)i0 * P * W;
  const int n = ns * P * W;
  for (int e = threadIdx.x * 8; e < n; e += blockDim.x * 8)
    *reinterpret_cast<uint4*>(strip + e) = __ldg(reinterpret_cast<const uint4*>(src + e));
  __syncthreads();
  __nv_bfloat16* dst = out + (((long long)b * C + c) * S + (long long)i0 * wp) * P * P;
  const int PW = P * W;
  for (int e = threadIdx.x * 8; e < n; e += blockDim.x * 8) {
    const int si = e / PW, o = e - si * PW;      // strip, offset in the strip's output run
    const int j = o / (P * P), k = o % (P * P);  // patch, pixel (k % 8 == 0)
    const int py = k / P, px = k % P;
    *reinterpret_cast<uint4*>(dst + e) =
        *reinterpret_cast<const uint4*>(strip + si * PW + py * W + j * P + px);
  }
}

cudaError_t launch_unfold(const __nv_bfloat16* img, long long img_sb, long long img_sc, int B,
                          int C, int Himg, int W, int P, __nv_bfloat16* out, cudaStream_t st) {
  if ((P * W) % 8 || W % 8 || (img_sb | img_sc) % 8 ||
      (reinterpret_cast<uintptr_t>(img) | reinterpret_cast<uintptr_t>(out)) % 16)
    return cudaErrorInvalidValue;
  if ((P == 8 || P == 16) && P * W * 2 <= 32 * 1024) {
    // strips per CTA: the largest divisor of Himg / P within 32 KB of shared memory
    const int hp = Himg / P;
    int ns = 1;
    for (int d = 1; d <= hp; ++d)
      if (hp % d == 0 && d * P * W * 2 <= 32 * 1024) ns = d;
    const int smem = ns * P * W * 2;
    const unsigned grid = (unsigned)((long long)B * C * (hp / ns));
    if (P == 8)
      unfold_wide_kernel<8><<<grid, 256, smem, st>>>(img, img_sb, img_sc, C, Himg, W, ns, out);
    else
      unfold_wide_kernel<16><<<grid, 256, smem, st>>>(img, img_sb, img_sc, C, Himg, W, ns, out);
    return cudaGetLastError();
  }
  const int smem = P * W * 2;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(unfold_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  unfold_kernel<<<B * C * (Himg / P), 256, smem, st>>>(img, img_sb, img_sc, B, C, Himg, W, P,
                                                        out);
  return cudaGetLastError();
}

}  // namespace dchag
