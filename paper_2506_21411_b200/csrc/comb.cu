// Upper-level combine (K_comb) and the patch unfold used by tokenize_channels.
//
// A node above level 0 receives, per child j, the child's output already projected
// into this node's value space, V_j = y_j @ wv_n (folded into the child's K_gemm), and
// its logits L_j = y_j @ U_n.  The node's context is then a per-position weighted sum
//   ctx[r, h-blk] = sum_j softmax_j(L_j[r,h]) * V_j[r, h-blk]       (layers.py:103-123)
// or, for a linear node, ctx[r,:] = sum_j mix_j V_j[r,:]             (layers.py:141-146).
// HBM-bound: reads g*D bf16 + g*H fp32 per row, writes D bf16.
#include "common.cuh"
#include "dchag_kernels.h"

namespace dchag {

constexpr int COMB_MAXG = 128;

// one warp per (node, row); lane owns 8-column chunks lane, lane+32, ... (16-B vectors)
__global__ void __launch_bounds__(256) combine_kernel(CombineArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long item = (long long)blockIdx.x * 8 + warp;
  const int n = (int)(item / a.R);
  const int r = (int)(item - (long long)n * a.R);
  if (n >= a.n_nodes) return;
  const int first = __ldg(a.node_first + n), g = __ldg(a.node_g + n);
  const int dh = a.D / a.H;
  const int nchunk = a.D / 8;
  const int per_lane = (nchunk + 31) / 32;  // <= 8 for D <= 2048

  float acc[8][8];
#pragma unroll
  for (int q = 0; q < 8; ++q)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[q][e] = 0.f;

  // softmax statistics for the heads this lane touches (computed redundantly per lane)
  float mx[8], inv[8];
  if (!a.mix) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      mx[q] = -INFINITY;
      inv[q] = 0.f;
      if (q < per_lane) {
        const int ch = lane + 32 * q;
        if (ch < nchunk) {
          const int h = ch * 8 / dh;
          float m = -INFINITY;
          for (int j = 0; j < g; ++j)
            m = fmaxf(m, a.L[(long long)(first + j) * a.sLj + (long long)r * a.H + h]);
          float s = 0.f;
          for (int j = 0; j < g; ++j)
            s += __expf(a.L[(long long)(first + j) * a.sLj + (long long)r * a.H + h] - m);
          mx[q] = m;
          inv[q] = 1.f / s;
        }
      }
    }
  }
  for (int j = 0; j < g; ++j) {
    const __nv_bfloat16* vrow = a.V + (long long)(first + j) * a.sVj + (long long)r * a.D;
    const float* lrow = a.L ? a.L + (long long)(first + j) * a.sLj + (long long)r * a.H : nullptr;
    const float mixj = a.mix ? __ldg(a.mix + first + j) : 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q < per_lane) {
        const int ch = lane + 32 * q;
        if (ch < nchunk) {
          float pj;
          if (a.mix) {
            pj = mixj;
          } else {
            const int h = ch * 8 / dh;
            pj = __expf(lrow[h] - mx[q]) * inv[q];
          }
          const uint4 v = *reinterpret_cast<const uint4*>(vrow + ch * 8);
          const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc[q][2 * e] += pj * bf16lo(vv[e]);
            acc[q][2 * e + 1] += pj * bf16hi(vv[e]);
          }
        }
      }
    }
  }
  __nv_bfloat16* orow = a.ctx + ((long long)n * a.R + r) * a.D;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q < per_lane) {
      const int ch = lane + 32 * q;
      if (ch < nchunk) {
        uint4 o;
        o.x = pack_bf16(acc[q][0], acc[q][1]);
        o.y = pack_bf16(acc[q][2], acc[q][3]);
        o.z = pack_bf16(acc[q][4], acc[q][5]);
        o.w = pack_bf16(acc[q][6], acc[q][7]);
        *reinterpret_cast<uint4*>(orow + ch * 8) = o;
      }
    }
  }
}

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t st) {
  if (a.D % 8 || a.D > 2048 || (a.D / a.H) % 8) return cudaErrorInvalidValue;
  const long long items = (long long)a.n_nodes * a.R;
  const int grid = (int)((items + 7) / 8);
  combine_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// images [B][C][H][W] (strided) -> patches [B][C][S][P*P]; one thread per patch row (py)
__global__ void unfold_kernel(const __nv_bfloat16* img, long long sb, long long sc, int B, int C,
                              int Himg, int W, int P, __nv_bfloat16* out) {
  const int hp = Himg / P, wp = W / P, S = hp * wp;
  const long long total = (long long)B * C * S * P;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int py = (int)(t % P);
  long long rest = t / P;
  const int s = (int)(rest % S);
  rest /= S;
  const int c = (int)(rest % C);
  const int b = (int)(rest / C);
  const int i = s / wp, j = s - i * wp;
  const __nv_bfloat16* src = img + b * sb + c * sc + (long long)(i * P + py) * W + j * P;
  __nv_bfloat16* dst = out + (((long long)b * C + c) * S + s) * P * P + py * P;
  for (int px = 0; px < P; ++px) dst[px] = src[px];
}

cudaError_t launch_unfold(const __nv_bfloat16* img, long long img_sb, long long img_sc, int B,
                          int C, int Himg, int W, int P, __nv_bfloat16* out, cudaStream_t st) {
  const long long total = (long long)B * C * (Himg / P) * (W / P) * P;
  const int grid = (int)((total + 255) / 256);
  unfold_kernel<<<grid, 256, 0, st>>>(img, img_sb, img_sc, B, C, Himg, W, P, out);
  return cudaGetLastError();
}

}  // namespace dchag
