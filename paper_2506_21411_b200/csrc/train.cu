// Training-step support kernels (the non-GEMM parts of the backward and of the per-step
// weight preparation; every matrix product of the step runs on the tcgen05 GEMMs).
//
//   cast_multi      fp32 master weights -> bf16 operands (plain or transposed, strided /
//                   padded destinations), every tensor of the step in one launch
//   query_fold      U[:, h] = wk[:, h-blk] (q wq)[h-blk] / sqrt(dh)   (layers.py:103-120
//                   with the input-independent query folded: logits = x U)
//   query_fold_bwd  its backward: d wk, d wq, d q from dU (tensor.py:395-413 on that chain)
//   colsum          periodic column sums: bias gradients (period 1, every row) and the
//                   positional sums over the batch (period S), deterministic
//   rowsum          row sums (the channel-softmax logit gradient summed over positions)
#include "common.cuh"
#include "dchag_kernels.h"

namespace dchag {

// ------------------------------------------------------------------------- cast_multi
__global__ void __launch_bounds__(256) cast_multi_kernel(const CastJob* jobs, int n_jobs) {
  const CastJob j = jobs[blockIdx.y];
  const int tiles_c = (j.cols + 31) / 32;
  const int tiles = ((j.rows + 31) / 32) * tiles_c;
  __shared__ float tile[32][33];
  const bool vec = !j.trans && !j.dst_f32 && j.cols % 4 == 0 && j.lds % 4 == 0 &&
                   j.ldd % 4 == 0 && ((reinterpret_cast<uintptr_t>(j.src) |
                                       reinterpret_cast<uintptr_t>(j.dst)) & 15) == 0;
  if (vec) {  // 16-byte loads, 8-byte stores; one warp per row (no per-element division)
    const int c4 = (int)(j.cols / 4);
    const int lane = threadIdx.x & 31;
    const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = w0; r < j.rows; r += nw) {
      const float4* src = reinterpret_cast<const float4*>(j.src + r * j.lds);
      uint2* dst = reinterpret_cast<uint2*>(j.dst + r * j.ldd);
      for (int c = lane; c < c4; c += 32) {
        const float4 v = __ldg(src + c);
        uint2 o;
        o.x = pack_bf16(v.x, v.y);
        o.y = pack_bf16(v.z, v.w);
        dst[c] = o;
      }
    }
    return;
  }
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int r0 = (t / tiles_c) * 32, c0 = (t % tiles_c) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
    if (!j.trans) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = r0 + ty + 8 * k, c = c0 + tx;
        if (r < j.rows && c < j.cols) {
          const float v = __ldg(j.src + (size_t)r * j.lds + c);
          if (j.dst_f32) reinterpret_cast<float*>(j.dst)[(size_t)r * j.ldd + c] = v;
          else j.dst[(size_t)r * j.ldd + c] = __float2bfloat16(v);
        }
      }
    } else {  // dst[c][r] = src[r][c] through a padded smem tile (both sides coalesced)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = r0 + ty + 8 * k, c = c0 + tx;
        tile[ty + 8 * k][tx] = (r < j.rows && c < j.cols) ? j.src[(size_t)r * j.lds + c] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = c0 + ty + 8 * k, r = r0 + tx;
        if (r < j.rows && c < j.cols)
          j.dst[(size_t)c * j.ldd + r] = __float2bfloat16(tile[tx][ty + 8 * k]);
      }
      __syncthreads();
    }
  }
}

cudaError_t launch_cast_multi(const CastJob* jobs, int n_jobs, int max_tiles, cudaStream_t st) {
  if (n_jobs < 1) return cudaSuccess;
  const int gx = max_tiles < 1024 ? max_tiles : 1024;
  cast_multi_kernel<<<dim3(gx > 0 ? gx : 1, n_jobs), 256, 0, st>>>(jobs, n_jobs);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------- query_fold
// phase 1: partial q wq over 128-row chunks of wq: part[node][chunk][j]
constexpr int QF_CHUNK = 128;

// a thread takes 4 adjacent columns (16-byte loads), rows 8 at a time in flight; the sum
// order over i is unchanged (sequential per column)
__global__ void qf_partial_kernel(const QueryFoldJob* jobs, int D, float* part) {
  const QueryFoldJob jb = jobs[blockIdx.z];
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const int i0 = blockIdx.y * QF_CHUNK, i1 = min(D, i0 + QF_CHUNK);
  if (j >= D) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int i = i0;
  for (; i + 8 <= i1; i += 8) {
    float4 w[8];
    float qv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      w[u] = __ldg(reinterpret_cast<const float4*>(jb.wq + (size_t)(i + u) * D + j));
      qv[u] = __ldg(jb.q + i + u);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc.x = fmaf(qv[u], w[u].x, acc.x); acc.y = fmaf(qv[u], w[u].y, acc.y);
      acc.z = fmaf(qv[u], w[u].z, acc.z); acc.w = fmaf(qv[u], w[u].w, acc.w);
    }
  }
  for (; i < i1; ++i) {
    const float4 w = __ldg(reinterpret_cast<const float4*>(jb.wq + (size_t)i * D + j));
    const float qv = __ldg(jb.q + i);
    acc.x = fmaf(qv, w.x, acc.x); acc.y = fmaf(qv, w.y, acc.y);
    acc.z = fmaf(qv, w.z, acc.z); acc.w = fmaf(qv, w.w, acc.w);
  }
  *reinterpret_cast<float4*>(part + ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * D + j) = acc;
}

// phase 2: qp = sum of the partials (fixed order); U[d][h] = s sum_{j in h} wk[d][j] qp[j]
__global__ void qf_final_kernel(const QueryFoldJob* jobs, int D, int H, int nchunk,
                                const float* part) {
  const QueryFoldJob jb = jobs[blockIdx.z];
  extern __shared__ float qp_s[];
  for (int j = threadIdx.x; j < D; j += blockDim.x) {
    float a = 0.f;
    for (int c = 0; c < nchunk; ++c) a += part[((size_t)blockIdx.z * nchunk + c) * D + j];
    qp_s[j] = a;
    if (blockIdx.x == 0 && jb.qp) jb.qp[j] = a;
  }
  __syncthreads();
  const int dh = D / H;
  const float s = rsqrtf((float)dh);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int d = blockIdx.x * nw + warp; d < D; d += gridDim.x * nw) {
    const float* row = jb.wk + (size_t)d * D;
    for (int h = 0; h < H; ++h) {
      float a = 0.f;
      for (int j = h * dh + lane; j < (h + 1) * dh; j += 32) a = fmaf(__ldg(row + j), qp_s[j], a);
#pragma unroll
      for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) jb.U[(size_t)d * jb.ldU + h] = a * s;
    }
  }
}

cudaError_t launch_query_fold(const QueryFoldJob* jobs, int n_jobs, int D, int H, float* part,
                              cudaStream_t st) {
  const int nchunk = (D + QF_CHUNK - 1) / QF_CHUNK;
  if (D % 4) return cudaErrorInvalidValue;
  qf_partial_kernel<<<dim3((D / 4 + 127) / 128, nchunk, n_jobs), 128, 0, st>>>(jobs, D, part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int smem = D * 4;
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(qf_final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  qf_final_kernel<<<dim3(32, 1, n_jobs), 256, smem, st>>>(jobs, D, H, nchunk, part);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------- query_fold_bwd
// With qp = q wq and U[d][h] = s sum_{j in h} wk[d][j] qp[j]:
//   d wk[d][j] = s dU[d][h(j)] qp[j]
//   d qp[j]    = s sum_d wk[d][j] dU[d][h(j)]
//   d wq[i][j] = q[i] d qp[j],  d q[i] = sum_j wq[i][j] d qp[j]
__global__ void qfb_partial_kernel(const QueryFoldJob* jobs, int D, int H, float* part) {
  const QueryFoldJob jb = jobs[blockIdx.z];
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) * 4;   // 4 columns of one head
  const int d0 = blockIdx.y * QF_CHUNK, d1 = min(D, d0 + QF_CHUNK);
  if (j >= D) return;
  const int h = j / (D / H);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int d = d0;
  for (; d + 8 <= d1; d += 8) {
    float4 w[8];
    float g[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      w[u] = __ldg(reinterpret_cast<const float4*>(jb.wk + (size_t)(d + u) * D + j));
      g[u] = __ldg(jb.dU + (size_t)(d + u) * jb.ldU + h);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc.x = fmaf(w[u].x, g[u], acc.x); acc.y = fmaf(w[u].y, g[u], acc.y);
      acc.z = fmaf(w[u].z, g[u], acc.z); acc.w = fmaf(w[u].w, g[u], acc.w);
    }
  }
  for (; d < d1; ++d) {
    const float4 w = __ldg(reinterpret_cast<const float4*>(jb.wk + (size_t)d * D + j));
    const float g = __ldg(jb.dU + (size_t)d * jb.ldU + h);
    acc.x = fmaf(w.x, g, acc.x); acc.y = fmaf(w.y, g, acc.y);
    acc.z = fmaf(w.z, g, acc.z); acc.w = fmaf(w.w, g, acc.w);
  }
  *reinterpret_cast<float4*>(part + ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * D + j) = acc;
}

__global__ void qfb_dqp_kernel(const QueryFoldJob* jobs, int D, int H, int nchunk,
                               const float* part, float* dqp) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= D) return;
  const float s = rsqrtf((float)(D / H));
  float a = 0.f;
  for (int c = 0; c < nchunk; ++c) a += part[((size_t)blockIdx.z * nchunk + c) * D + j];
  dqp[(size_t)blockIdx.z * D + j] = a * s;
}

// one warp per row i: d wk row i, d wq row i, d q[i]
__global__ void qfb_rows_kernel(const QueryFoldJob* jobs, int D, int H, const float* dqp_all) {
  const QueryFoldJob jb = jobs[blockIdx.z];
  const float* dqp = dqp_all + (size_t)blockIdx.z * D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int dh = D / H;
  const float s = rsqrtf((float)dh);
  const bool vec = D % 128 == 0 && dh % 4 == 0;
  for (int i = blockIdx.x * nw + warp; i < D; i += gridDim.x * nw) {
    const float qi = __ldg(jb.q + i);
    float dq = 0.f;
    if (vec) {  // 4 adjacent columns (one head) per lane and step: 16-byte loads / stores
      const float4* wq4 = reinterpret_cast<const float4*>(jb.wq + (size_t)i * D);
      const float4* g4 = reinterpret_cast<const float4*>(dqp);
      const float4* qp4 = reinterpret_cast<const float4*>(jb.qp);
      float4* dwq4 = reinterpret_cast<float4*>(jb.dwq + (size_t)i * D);
      float4* dwk4 = reinterpret_cast<float4*>(jb.dwk + (size_t)i * D);
      for (int c = lane; c < D / 4; c += 32) {
        const float4 g = g4[c], w = __ldg(wq4 + c), qp = __ldg(qp4 + c);
        const float du = s * __ldg(jb.dU + (size_t)i * jb.ldU + (4 * c) / dh);
        dq = fmaf(w.x, g.x, dq); dq = fmaf(w.y, g.y, dq);
        dq = fmaf(w.z, g.z, dq); dq = fmaf(w.w, g.w, dq);
        dwq4[c] = make_float4(qi * g.x, qi * g.y, qi * g.z, qi * g.w);
        dwk4[c] = make_float4(du * qp.x, du * qp.y, du * qp.z, du * qp.w);
      }
    } else {
      for (int j = lane; j < D; j += 32) {
        const float g = dqp[j];
        dq = fmaf(__ldg(jb.wq + (size_t)i * D + j), g, dq);
        jb.dwq[(size_t)i * D + j] = qi * g;
        jb.dwk[(size_t)i * D + j] = s * __ldg(jb.dU + (size_t)i * jb.ldU + j / dh) * __ldg(jb.qp + j);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) dq += __shfl_xor_sync(0xffffffffu, dq, o);
    if (lane == 0) jb.dq[i] = dq;
  }
}

cudaError_t launch_query_fold_bwd(const QueryFoldJob* jobs, int n_jobs, int D, int H,
                                  float* part, float* dqp, cudaStream_t st) {
  const int nchunk = (D + QF_CHUNK - 1) / QF_CHUNK;
  if (D % 4 || (D / H) % 4) return cudaErrorInvalidValue;
  qfb_partial_kernel<<<dim3((D / 4 + 127) / 128, nchunk, n_jobs), 128, 0, st>>>(jobs, D, H, part);
  qfb_dqp_kernel<<<dim3((D + 127) / 128, 1, n_jobs), 128, 0, st>>>(jobs, D, H, nchunk, part, dqp);
  qfb_rows_kernel<<<dim3(64, 1, n_jobs), 256, 0, st>>>(jobs, D, H, dqp);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------- colsum
// out[g][p][n] (+)= sum over rows r = p, p + P, ... < R of X[g][r][n]; X bf16 or fp32
// (row stride ldx, group stride sxg). P == 1 takes two passes (partials over 64-row chunks,
// then their sum in chunk order), P > 1 one (each output sums R / P rows): both
// deterministic.
template <typename T>
DEV float ldf(const T* p);
template <>
DEV float ldf<float>(const float* p) { return __ldg(p); }
template <>
DEV float ldf<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

constexpr int CS_ROWS = 64;

struct ColsumOut {               // where / how a column sum is written
  void* out;
  long long sog, ldo;            // group stride, row stride (periodic sums)
  int bf16, accumulate;
  const float* gscale;           // optional per-group scale
  DEV void put(int g, int p, int n, float a) const {
    if (gscale) a *= __ldg(gscale + g);
    const size_t o = (size_t)g * sog + (size_t)p * ldo + n;
    if (bf16) {
      reinterpret_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16(a);
    } else {
      float* f = reinterpret_cast<float*>(out) + o;
      *f = accumulate ? *f + a : a;
    }
  }
};

template <typename T>
__global__ void colsum_direct_kernel(const T* X, long long ldx, long long sxg, int R, int N,
                                     int P, ColsumOut o) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const int p = blockIdx.y, g = blockIdx.z;
  if (n >= N) return;
  const T* x = X + (size_t)g * sxg + n;
  float a = 0.f;
  for (int r = p; r < R; r += P) a += ldf(x + (size_t)r * ldx);
  o.put(g, p, n, a);
}

template <typename T>
__global__ void colsum_partial_kernel(const T* X, long long ldx, long long sxg, int R, int N,
                                      float* part) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const int ch = blockIdx.y, g = blockIdx.z;
  if (n >= N) return;
  const T* x = X + (size_t)g * sxg + n;
  float a = 0.f;
  for (int r = ch * CS_ROWS; r < min(R, (ch + 1) * CS_ROWS); ++r) a += ldf(x + (size_t)r * ldx);
  part[((size_t)g * gridDim.y + ch) * N + n] = a;
}

__global__ void colsum_final_kernel(const float* part, int nch, int N, ColsumOut o) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const int g = blockIdx.z;
  if (n >= N) return;
  float a = 0.f;
  for (int c = 0; c < nch; ++c) a += part[((size_t)g * nch + c) * N + n];
  o.put(g, 0, n, a);
}

// vectorised forms: a thread sums VW adjacent columns (one 16-byte load per row), rows
// unrolled by 8 so eight loads are in flight per thread
template <typename T>
struct ColVec;
template <>
struct ColVec<float> {
  static constexpr int VW = 4;
  static DEV void load(const float* p, float (&v)[4]) {
    const float4 f = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  }
};
template <>
struct ColVec<__nv_bfloat16> {
  static constexpr int VW = 8;
  static DEV void load(const __nv_bfloat16* p, float (&v)[8]) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) { v[2 * e] = bf16lo(w[e]); v[2 * e + 1] = bf16hi(w[e]); }
  }
};

// rows r0, r0 + step, ... < r1 of VW columns starting at x (8 rows per round in flight)
template <typename T>
DEV void colsum_rows(const T* x, long long ldx, int r0, int r1, int step,
                     float (&a)[ColVec<T>::VW]) {
  constexpr int VW = ColVec<T>::VW;
#pragma unroll
  for (int e = 0; e < VW; ++e) a[e] = 0.f;
  int r = r0;
  for (; r + 7 * step < r1; r += 8 * step) {
    float v[8][VW];
#pragma unroll
    for (int u = 0; u < 8; ++u) ColVec<T>::load(x + (size_t)(r + u * step) * ldx, v[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int e = 0; e < VW; ++e) a[e] += v[u][e];
  }
  for (; r < r1; r += step) {
    float v[VW];
    ColVec<T>::load(x + (size_t)r * ldx, v);
#pragma unroll
    for (int e = 0; e < VW; ++e) a[e] += v[e];
  }
}

template <typename T>
__global__ void colsum_direct_vec_kernel(const T* X, long long ldx, long long sxg, int R, int N,
                                         int P, ColsumOut o) {
  constexpr int VW = ColVec<T>::VW;
  const int n = (blockIdx.x * blockDim.x + threadIdx.x) * VW;
  const int p = blockIdx.y, g = blockIdx.z;
  if (n >= N) return;
  float a[VW];
  colsum_rows<T>(X + (size_t)g * sxg + n, ldx, p, R, P, a);
#pragma unroll
  for (int e = 0; e < VW; ++e) o.put(g, p, n + e, a[e]);
}

template <typename T>
__global__ void colsum_partial_vec_kernel(const T* X, long long ldx, long long sxg, int R, int N,
                                          float* part) {
  constexpr int VW = ColVec<T>::VW;
  const int n = (blockIdx.x * blockDim.x + threadIdx.x) * VW;
  const int ch = blockIdx.y, g = blockIdx.z;
  if (n >= N) return;
  float a[VW];
  colsum_rows<T>(X + (size_t)g * sxg + n, ldx, ch * CS_ROWS, min(R, (ch + 1) * CS_ROWS), 1, a);
#pragma unroll
  for (int e = 0; e < VW; ++e) part[((size_t)g * gridDim.y + ch) * N + n + e] = a[e];
}

template <typename T>
static cudaError_t colsum_t(const T* X, long long ldx, long long sxg, int G, int R, int N, int P,
                            const ColsumOut& o, float* part, cudaStream_t st) {
  const dim3 blk(128);
  constexpr int VW = ColVec<T>::VW;
  const bool vec = N % VW == 0 && ldx % VW == 0 && sxg % VW == 0 &&
                   reinterpret_cast<uintptr_t>(X) % 16 == 0;
  if (vec) {
    const int nthr = N / VW;
    if (P > 1 || R <= CS_ROWS) {
      colsum_direct_vec_kernel<T><<<dim3((nthr + 127) / 128, P, G), blk, 0, st>>>(
          X, ldx, sxg, R, N, P, o);
      return cudaGetLastError();
    }
    const int nch = (R + CS_ROWS - 1) / CS_ROWS;
    colsum_partial_vec_kernel<T><<<dim3((nthr + 127) / 128, nch, G), blk, 0, st>>>(
        X, ldx, sxg, R, N, part);
    colsum_final_kernel<<<dim3((N + 127) / 128, 1, G), blk, 0, st>>>(part, nch, N, o);
    return cudaGetLastError();
  }
  if (P > 1 || R <= CS_ROWS) {
    colsum_direct_kernel<T><<<dim3((N + 127) / 128, P, G), blk, 0, st>>>(X, ldx, sxg, R, N, P,
                                                                         o);
    return cudaGetLastError();
  }
  const int nch = (R + CS_ROWS - 1) / CS_ROWS;
  colsum_partial_kernel<T><<<dim3((N + 127) / 128, nch, G), blk, 0, st>>>(X, ldx, sxg, R, N,
                                                                          part);
  colsum_final_kernel<<<dim3((N + 127) / 128, 1, G), blk, 0, st>>>(part, nch, N, o);
  return cudaGetLastError();
}

cudaError_t launch_colsum(const void* X, int x_f32, long long ldx, long long sxg, int G, int R,
                          int N, int P, void* out, long long sog, long long ldo, int out_bf16,
                          int accumulate, const float* gscale, float* part, cudaStream_t st) {
  ColsumOut o{out, sog, ldo > 0 ? ldo : N, out_bf16, accumulate, gscale};
  if (x_f32)
    return colsum_t(reinterpret_cast<const float*>(X), ldx, sxg, G, R, N, P, o, part, st);
  return colsum_t(reinterpret_cast<const __nv_bfloat16*>(X), ldx, sxg, G, R, N, P, o, part, st);
}

// ------------------------------------------------------------------------- rowsum
__global__ void rowsum_kernel(const float* X, long long ldx, int rows, int N, float* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const float* x = X + (size_t)warp * ldx;
  float a = 0.f;
  for (int j = lane; j < N; j += 32) a += x[j];
#pragma unroll
  for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if (lane == 0) out[warp] = a;
}

cudaError_t launch_rowsum(const float* X, long long ldx, int rows, int N, float* out,
                          cudaStream_t st) {
  rowsum_kernel<<<(rows * 32 + 255) / 256, 256, 0, st>>>(X, ldx, rows, N, out);
  return cudaGetLastError();
}

}  // namespace dchag

namespace dchag {

// ------------------------------------------------------------------------- level-0 pack
// The training step refolds level 0 every step with one grouped GEMM,
//   MT[n] = [Wv_n | U_n | 0]^T [tok.w rows of node n ; tok.b + chan_id rows ; 0]^T,
// fp32 [n0][Dp][Kn]: MT[n][d][l*PP + k] = M_c[k][d] (c = c0_n + l), MT[n][d][gmax*PP + l] =
// Cb_c[d], and rows D + h the logit weights (WU, bU). These kernels scatter it into the
// operand layouts of K_p0 / K_l0 / the row-dot GEMM (fold.pack_rank's layouts).
DEV long long tiled_off(int blk, int k, int n, int K, int N) {  // canonical K-major core mats
  return (long long)blk * K * N + ((long long)(k >> 3) * (N >> 3) + (n >> 3)) * 64 +
         (n & 7) * 8 + (k & 7);
}

// One pass over the slab's fold rows, k fastest so every MT row segment is read coalesced,
// written to both layouts that hold M_c: K_l0's tiled Mt [H*2][C_pad*PP][hw] (8-element
// runs) and the row-dot operand Mrow [C][D][PP], plus Cb [C][D]. Mt's padding channels
// [C, C_pad) are zero from allocation and never written.
__global__ void pack_rows_kernel(L0PackArgs a) {
  // one warp per group of four fold rows (channel c, columns d .. d+3): lanes sweep the PP
  // contiguous values of every row, all four rows' loads issued before any store (no
  // per-element 64-bit index division); lane 0 also moves the Cb terms
  constexpr int RW = 4;
  const int hw = a.D / a.H / 2, K = a.C_pad * a.PP;
  const int lane = threadIdx.x & 31;
  const long long rows = (long long)a.C * a.D;
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long w4 = w0 * RW; w4 < rows; w4 += nw * RW) {
    float v[RW][2];
    const float* rowp[RW];
    int cs[RW], ds[RW], ls[RW];
#pragma unroll
    for (int u = 0; u < RW; ++u) {
      const long long w = w4 + u;
      cs[u] = -1;
      if (w >= rows) continue;
      const int c = (int)(w / a.D), d = (int)(w - (long long)c * a.D);
      const int n = __ldg(a.chan_node + c), l = __ldg(a.chan_local + c);
      cs[u] = c; ds[u] = d; ls[u] = l;
      rowp[u] = a.MT + ((size_t)n * a.Dp + d) * a.Kn;
#pragma unroll
      for (int k2 = 0; k2 < 2; ++k2) {
        const int kk = lane + 32 * k2;
        v[u][k2] = kk < a.PP ? rowp[u][l * a.PP + kk] : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < RW; ++u) {
      if (cs[u] < 0) continue;
      const int c = cs[u], d = ds[u];
      const int blk = d / hw, nn = d - blk * hw;
      __nv_bfloat16* mrow = a.Mrow + ((size_t)c * a.D + d) * a.PP;
#pragma unroll
      for (int k2 = 0; k2 < 2; ++k2) {
        const int kk = lane + 32 * k2;
        if (kk >= a.PP) continue;
        const __nv_bfloat16 b = __float2bfloat16(v[u][k2]);
        mrow[kk] = b;
        a.Mt[tiled_off(blk, c * a.PP + kk, nn, K, hw)] = b;
      }
      if (lane == 0) a.Cb[(size_t)c * a.D + d] = rowp[u][a.ones0 + ls[u]];
    }
  }
}

__global__ void pack_et_kernel(L0PackArgs a) {  // Et [n0][H][2][KE][hw] tiled
  const int hw = a.D / a.H / 2;
  const long long per_node = (long long)a.H * 2 * a.KE * hw;
  const long long total = per_node * a.n0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(t / per_node);
    const long long rem0 = t - (long long)n * per_node;
    const int hb = (int)(rem0 / ((long long)a.KE * hw));          // h * 2 + half
    const int rem = (int)(rem0 - (long long)hb * a.KE * hw);
    const int k = rem / hw, nn = rem - (rem / hw) * hw;
    const int d = hb * hw + nn;
    const float v = k < __ldg(a.node_g + n)
                        ? a.MT[((size_t)n * a.Dp + d) * a.Kn + a.ones0 + k] : 0.f;
    a.Et[(long long)n * per_node + tiled_off(hb, k, nn, a.KE, hw)] = __float2bfloat16(v);
  }
}

__global__ void pack_logit_kernel(L0PackArgs a) {  // WUt [C][HP][PP] bf16, bU [C][HP] fp32
  const long long total = (long long)a.C * a.HP * (a.PP + 1);
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(t / ((long long)a.HP * (a.PP + 1)));
    const int rem = (int)(t - (long long)c * a.HP * (a.PP + 1));
    const int h = rem / (a.PP + 1), kk = rem - h * (a.PP + 1);
    const int n = __ldg(a.chan_node + c), l = __ldg(a.chan_local + c);
    const float* row = a.MT + ((size_t)n * a.Dp + a.D + h) * a.Kn;
    if (kk < a.PP)
      a.WUt[((size_t)c * a.HP + h) * a.PP + kk] = __float2bfloat16(h < a.H ? row[l * a.PP + kk] : 0.f);
    else
      a.bU[(size_t)c * a.HP + h] = h < a.H ? row[a.ones0 + l] : 0.f;
  }
}

// posVU fp32 [n0][S][Dp] (pos [Wv | U]) -> posV0 bf16 [n0][S][D] (x mixsum for linear
// nodes), posU fp32 [n0][S][HP]
__global__ void pack_pos_kernel(L0PackArgs a) {
  // one warp per positional row (node n, position s), lanes sweep its columns
  const int W = a.D + a.HP;
  const int lane = threadIdx.x & 31;
  const long long rows = (long long)a.n0 * a.S;
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long row = w0; row < rows; row += nw) {
    const float* src = a.posVU + row * a.Dp;
    const int n = (int)(row / a.S);
    const float sc = a.mixsum ? __ldg(a.mixsum + n) : 1.f;
    for (int col = lane; col < W; col += 32) {
      if (col < a.D) {
        a.posV0[row * a.D + col] = __float2bfloat16(src[col] * sc);
      } else if (a.posU) {
        const int h = col - a.D;
        a.posU[row * a.HP + h] = h < a.H ? src[a.D + h] : 0.f;
      }
    }
  }
}

// ------------------------------------------------------------------------- split3
// fp32 x [rows][K] (row stride ldx) -> bf16 out [rows][3K] (row stride ldo) = [hi | lo | hi]
// with hi = bf16(x), lo = bf16(x - hi): the A operand of the fp32 parity mode's split-bf16
// 3-term GEMM, in one pass (the torch form read x twice and wrote four intermediates).
__global__ void split3_kernel(const float* __restrict__ x, long long rows, int K, long long ldx,
                              __nv_bfloat16* __restrict__ out, long long ldo) {
  const int k4 = K / 4;
  const long long n = rows * k4;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / k4;
    const int c = (int)(i - r * k4) * 4;
    const float4 v = __ldg(reinterpret_cast<const float4*>(x + r * ldx + c));
    const float f[4] = {v.x, v.y, v.z, v.w};
    uint32_t hi[2], lo[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const __nv_bfloat16 h0 = __float2bfloat16(f[2 * e]), h1 = __float2bfloat16(f[2 * e + 1]);
      const float r0 = f[2 * e] - __bfloat162float(h0), r1 = f[2 * e + 1] - __bfloat162float(h1);
      hi[e] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
      lo[e] = pack_bf16(r0, r1);
    }
    __nv_bfloat16* o = out + r * ldo + c;
    *reinterpret_cast<uint2*>(o) = make_uint2(hi[0], hi[1]);
    *reinterpret_cast<uint2*>(o + K) = make_uint2(lo[0], lo[1]);
    *reinterpret_cast<uint2*>(o + 2 * K) = make_uint2(hi[0], hi[1]);
  }
}

cudaError_t launch_split3(const float* x, long long rows, int K, long long ldx,
                          __nv_bfloat16* out, long long ldo, cudaStream_t st) {
  if (K % 4 || ldx % 4 || ldo % 4 || (reinterpret_cast<uintptr_t>(x) % 16) ||
      (reinterpret_cast<uintptr_t>(out) % 8))
    return cudaErrorInvalidValue;
  const long long n = rows * (K / 4);
  const int blocks = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  split3_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(x, rows, K, ldx, out, ldo);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------- p normalise
// p[poff[n] + ((hg*g + c)*R + r)*NH + hn] = e[same] * pinv[(n*R + r)*H + hg*NH + hn]: the
// training backward's normalised level-0 softmax from the forward's K_p0 output (e and 1/sum
// e), instead of a second K_p0 pass over the images. One thread per 8 elements (16 bytes).
__global__ void l0_p_normalize_kernel(const __nv_bfloat16* __restrict__ e,
                                      const float* __restrict__ pinv,
                                      __nv_bfloat16* __restrict__ p,
                                      const long long* __restrict__ node_poff,
                                      const int* __restrict__ node_g, int R, int H, int NH) {
  const int n = blockIdx.y;
  const int g = __ldg(node_g + n);
  const long long base = __ldg(node_poff + n);
  const int nel = g * R * H;          // the node's elements (< 2^31, a multiple of 8)
  const int rows8 = 8 / NH;           // rows covered by one 8-element chunk
  const float* pin = pinv + (long long)n * R * H;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) * 8; i < nel;
       i += gridDim.x * blockDim.x * 8) {
    const int t0 = i / NH;            // (hg*g + c)*R + r0
    const int r0 = t0 % R, hg = t0 / R / g;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(e + base + i));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    float sc[8];
    if (NH == 4) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(pin + (r0 + u) * H + hg * 4));
        sc[4 * u] = q.x; sc[4 * u + 1] = q.y; sc[4 * u + 2] = q.z; sc[4 * u + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) sc[k] = __ldg(pin + (r0 + k / NH) * H + hg * NH + k % NH);
    }
    (void)rows8;
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      o[k] = pack_bf16(bf16lo(w[k]) * sc[2 * k], bf16hi(w[k]) * sc[2 * k + 1]);
    *reinterpret_cast<uint4*>(p + base + i) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

cudaError_t launch_l0_p_normalize(const __nv_bfloat16* e, const float* pinv, __nv_bfloat16* p,
                                  const long long* node_poff, const int* node_g, int n_nodes,
                                  int gmax, int R, int H, int NH, cudaStream_t st) {
  if ((R * H) % 8 || NH < 1 || H % NH || 8 % NH || R % (8 / NH) ||
      (long long)gmax * R * H >= (1ll << 31) || (NH == 4 && H % 4))
    return cudaErrorInvalidValue;
  const long long per = (long long)gmax * R * H / 8;
  const int bx = (int)((per + 255) / 256 < 2048 ? (per + 255) / 256 : 2048);
  l0_p_normalize_kernel<<<dim3(bx, n_nodes), 256, 0, st>>>(e, pinv, p, node_poff, node_g, R, H,
                                                           NH);
  return cudaGetLastError();
}

cudaError_t launch_l0_pack(const L0PackArgs& a, cudaStream_t st) {
  if (a.PP > 64) return cudaErrorInvalidValue;  // pack_rows: two 32-lane sweeps per row
  const int grid = 148 * 8;
  pack_rows_kernel<<<grid, 256, 0, st>>>(a);
  pack_et_kernel<<<grid, 256, 0, st>>>(a);
  if (a.WUt) pack_logit_kernel<<<grid, 256, 0, st>>>(a);
  if (a.posVU) pack_pos_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace dchag
