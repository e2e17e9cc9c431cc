// extern "C" boundary of libdchag.so (declared in include/dchag.h).
// Validates shapes, builds TMA tensor maps (driver entry point fetched at runtime, so the
// library links only the static CUDA runtime), and launches the kernels on the caller's
// stream.  No device allocation, no host synchronisation.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/dchag.h"
#include "common.cuh"
#include "dchag_kernels.h"

using namespace dchag;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return DCHAG_OK;
  if (e == cudaErrorInvalidValue)
    return fail(DCHAG_ERR_SHAPE, "%s: unsupported shape/arguments", what);
  return fail(DCHAG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int num_sms_cached() {
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  return sms[dev] > 0 ? sms[dev] : 148;
}

// bf16 tensor map, dims[0] contiguous; strides in bytes for dims 1..rank-1
int make_map(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims,
             const cuuint64_t* strides_bytes, const cuuint32_t* box, CUtensorMapSwizzle swz) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(DCHAG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims,
                   strides_bytes, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DCHAG_ERR_SHAPE, "tensor map encode failed (%d)", (int)r);
  return DCHAG_OK;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

// ===================================================================== tiling kernel
namespace dchag {
__global__ void tile_weights_kernel(const float* src, int nblk, int K, int N, __nv_bfloat16* dst) {
  const long long total = (long long)nblk * K * N;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int b = (int)(t / ((long long)K * N));
  const int rem = (int)(t - (long long)b * K * N);
  const int k = rem / N, n = rem % N;
  const long long off =
      (long long)b * K * N + ((k / 8) * (N / 8) + (n / 8)) * 64 + (n % 8) * 8 + (k % 8);
  dst[off] = __float2bfloat16(src[t]);
}
}  // namespace dchag

extern "C" {

const char* dchag_version(void) { return "dchag-b200 0.1.0 (sm_100a)"; }
const char* dchag_last_error(void) { return g_err.c_str(); }
int dchag_num_sms(void) { return num_sms_cached(); }

int dchag_l0_tgrad_te(const void* patches, int cnt, int c0, int g, int R, int seq, int D,
                      int H, int nh, int PP, const void* p, const float* mix, const void* G,
                      const void* dlb, void* TE, long long te_ld, int ones0, void* stream) {
  if (!mix && !p) return fail(DCHAG_ERR_SHAPE, "l0_tgrad_te: need p or mix");
  if (H < 1 || H > 128 || D % H || D % 128 || R % 64 || seq % 64 || R % seq || PP != 64 ||
      (D / H != 64 && D / H != 128) || (!mix && (nh < 2 || nh % 2 || H % nh)) || !TE ||
      te_ld < D + (dlb ? H : 0) || te_ld % 8 ||
      (reinterpret_cast<uintptr_t>(patches) | reinterpret_cast<uintptr_t>(G) |
       reinterpret_cast<uintptr_t>(dlb)) % 16)
    return fail(DCHAG_ERR_SHAPE, "l0_tgrad_te: bad shape R=%d S=%d D=%d H=%d PP=%d", R, seq, D,
                H, PP);
  L0TgradArgs a;
  memset(&a, 0, sizeof(a));
  a.debug = getenv("DCHAG_TE_DEBUG") ? atoi(getenv("DCHAG_TE_DEBUG")) : 0;
  a.patches = reinterpret_cast<const __nv_bfloat16*>(patches);
  a.cnt = cnt; a.c0 = c0; a.g = g; a.R = R; a.S = seq; a.D = D; a.H = H; a.NH = nh; a.PP = PP;
  a.p = reinterpret_cast<const __nv_bfloat16*>(p); a.mix = mix;
  a.G = reinterpret_cast<const __nv_bfloat16*>(G);
  a.TE = reinterpret_cast<__nv_bfloat16*>(TE); a.te_ld = te_ld; a.ones0 = ones0;
  a.has_dl = dlb != nullptr;
  const int B = R / seq;
  CUtensorMap tG, tP, tDL;
  cuuint64_t gd[2] = {(cuuint64_t)D, (cuuint64_t)R};
  cuuint64_t gs[1] = {(cuuint64_t)D * 2};
  cuuint32_t gb[2] = {64u, 64u};
  int rc = make_map(&tG, G, 2, gd, gs, gb, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  cuuint64_t pd[3] = {64u, (cuuint64_t)seq, (cuuint64_t)B * cnt};
  cuuint64_t ps[2] = {64u * 2, (cuuint64_t)seq * 64 * 2};
  cuuint32_t pb[3] = {64u, 64u, 1u};
  rc = make_map(&tP, patches, 3, pd, ps, pb, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  tDL = tG;
  if (dlb) {
    cuuint64_t dd[3] = {(cuuint64_t)R, (cuuint64_t)H, (cuuint64_t)g};
    cuuint64_t ds[2] = {(cuuint64_t)R * 2, (cuuint64_t)R * H * 2};
    cuuint32_t db[3] = {64u, 128u, 1u};
    rc = make_map(&tDL, dlb, 3, dd, ds, db, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  return cuda_status(launch_l0_tgrad_te(tG, tP, tDL, a, S(stream)), "l0_tgrad_te");
}

int dchag_l0_pack(const float* MT, int n0, int C, int C_pad, int D, int H, int HP, int PP,
                  int gmax, int ones0, int KE, int seq, long long Dp, long long Kn,
                  const int* chan_node,
                  const int* chan_local, const int* node_g, void* Mt, void* Et, void* Mrow,
                  float* Cb, void* WUt, float* bU, const float* posVU, const float* mixsum,
                  void* posV0, float* posU, void* stream) {
  if (!MT || n0 < 1 || C < 1 || C_pad < C || H < 1 || D % (2 * H) || ((D / H / 2) % 8) ||
      PP % 8 || KE % 8 || Dp < D + (WUt ? H : 0) || ones0 < gmax * PP || Kn < ones0 + gmax ||
      !chan_node || !chan_local || !node_g || !Mt || !Et || !Mrow || !Cb ||
      (WUt && (!bU || HP < H)) || (posVU && !posV0))
    return fail(DCHAG_ERR_SHAPE, "l0_pack: bad arguments");
  L0PackArgs a;
  memset(&a, 0, sizeof(a));
  a.MT = MT; a.n0 = n0; a.C = C; a.C_pad = C_pad; a.D = D; a.H = H; a.HP = HP; a.PP = PP;
  a.gmax = gmax; a.ones0 = ones0; a.KE = KE; a.S = seq; a.Dp = Dp; a.Kn = Kn;
  a.chan_node = chan_node; a.chan_local = chan_local; a.node_g = node_g;
  a.Mt = reinterpret_cast<__nv_bfloat16*>(Mt); a.Et = reinterpret_cast<__nv_bfloat16*>(Et);
  a.Mrow = reinterpret_cast<__nv_bfloat16*>(Mrow); a.Cb = Cb;
  a.WUt = reinterpret_cast<__nv_bfloat16*>(WUt); a.bU = bU;
  a.posVU = posVU; a.mixsum = mixsum; a.posV0 = reinterpret_cast<__nv_bfloat16*>(posV0);
  a.posU = posU;
  return cuda_status(launch_l0_pack(a, S(stream)), "l0_pack");
}

int dchag_cast_multi(const void* jobs, int n_jobs, int max_tiles, void* stream) {
  if (n_jobs < 0 || (n_jobs && !jobs)) return fail(DCHAG_ERR_SHAPE, "cast_multi: bad table");
  return cuda_status(launch_cast_multi(reinterpret_cast<const CastJob*>(jobs), n_jobs, max_tiles,
                                       S(stream)), "cast_multi");
}

int dchag_query_fold(const void* jobs, int n_jobs, int D, int H, float* work, void* stream) {
  if (n_jobs < 1 || !jobs || !work || H < 1 || D % H || (D / H) < 1)
    return fail(DCHAG_ERR_SHAPE, "query_fold: bad arguments D=%d H=%d", D, H);
  return cuda_status(launch_query_fold(reinterpret_cast<const QueryFoldJob*>(jobs), n_jobs, D, H,
                                       work, S(stream)), "query_fold");
}

int dchag_query_fold_bwd(const void* jobs, int n_jobs, int D, int H, float* work, float* dqp,
                         void* stream) {
  if (n_jobs < 1 || !jobs || !work || !dqp || H < 1 || D % H)
    return fail(DCHAG_ERR_SHAPE, "query_fold_bwd: bad arguments D=%d H=%d", D, H);
  return cuda_status(launch_query_fold_bwd(reinterpret_cast<const QueryFoldJob*>(jobs), n_jobs, D,
                                           H, work, dqp, S(stream)), "query_fold_bwd");
}

int dchag_colsum(const void* X, int x_f32, long long ldx, long long sxg, int G, int R, int N,
                 int P, void* out, long long sog, long long ldo, int out_bf16, int accumulate,
                 const float* gscale, float* work, void* stream) {
  if (!X || !out || G < 1 || R < 1 || N < 1 || P < 1 || P > 65535 ||
      (P == 1 && R > 64 && !work) || (out_bf16 && accumulate))
    return fail(DCHAG_ERR_SHAPE, "colsum: bad arguments G=%d R=%d N=%d P=%d", G, R, N, P);
  return cuda_status(launch_colsum(X, x_f32, ldx, sxg, G, R, N, P, out, sog, ldo, out_bf16,
                                   accumulate, gscale, work, S(stream)), "colsum");
}

int dchag_rowsum(const float* X, long long ldx, int rows, int N, float* out, void* stream) {
  if (!X || !out || rows < 1 || N < 1) return fail(DCHAG_ERR_SHAPE, "rowsum: bad arguments");
  return cuda_status(launch_rowsum(X, ldx, rows, N, out, S(stream)), "rowsum");
}

int dchag_split3_bf16(const float* x, long long rows, int K, long long ldx, void* out,
                      long long ldo, void* stream) {
  if (!x || !out || rows < 1 || K < 4 || K % 4 || ldx < K || ldo < 3LL * K)
    return fail(DCHAG_ERR_SHAPE, "split3_bf16: bad arguments rows=%lld K=%d", rows, K);
  return cuda_status(launch_split3(x, rows, K, ldx, reinterpret_cast<__nv_bfloat16*>(out), ldo,
                                   S(stream)),
                     "split3_bf16");
}

int dchag_l0_p_normalize(const void* e, const float* pinv, void* p, const long long* node_poff,
                         const int* node_g, int n_nodes, int gmax, int R, int H, int nh,
                         void* stream) {
  if (!e || !pinv || !p || !node_poff || !node_g || n_nodes < 1 || gmax < 1 || R < 1 ||
      H < 1 || nh < 1 || H % nh || (R * H) % 8)
    return fail(DCHAG_ERR_SHAPE, "l0_p_normalize: bad arguments");
  return cuda_status(launch_l0_p_normalize(reinterpret_cast<const __nv_bfloat16*>(e), pinv,
                                           reinterpret_cast<__nv_bfloat16*>(p), node_poff,
                                           node_g, n_nodes, gmax, R, H, nh, S(stream)),
                     "l0_p_normalize");
}

int dchag_combine_overflow(int* flag, int reset) {
  if (!flag) return fail(DCHAG_ERR_SHAPE, "combine_overflow: null flag");
  return cuda_status(comb_overflow_flag(flag, reset), "combine_overflow");
}

static int gemm_impl(const void* A, int G, int Mo, int Mi, int K, long long sAg, long long sAmo,
                     long long sAmi, const void* W, int N, long long sWg, int Nv,
                     const float* bias, long long bias_g, const void* rowbias,
                     long long rowbias_g, long long rowbias_row, int rowbias_period, void* outV,
                     int outV_f32, long long sVg, long long sVmo, long long sVmi, float* outL,
                     long long sLg, long long sLmo, long long sLmi, const void* dotG,
                     long long ldG, float* dotOut, void* stream, const float* rmask = nullptr,
                     const float* mtok = nullptr, int dot_group = 32) {
  const bool dot = dotOut != nullptr;
  if (G < 1 || Mo < 1 || Mi < 128 || Mi % 128 || K < 16 || K % 16 || N < 16 || Nv < 0 ||
      Nv > N || Nv % 16)
    return fail(DCHAG_ERR_SHAPE, "gemm: bad shape G=%d Mo=%d Mi=%d K=%d N=%d Nv=%d", G, Mo, Mi,
                K, N, Nv);
  if (!dot && Nv < N && !outL) return fail(DCHAG_ERR_SHAPE, "gemm: N > Nv needs outL");
  if (!dot && Nv > 0 && !outV) return fail(DCHAG_ERR_SHAPE, "gemm: Nv > 0 needs outV");
  if ((sAmi * 2) % 16 || (sAmo * 2) % 16 || (sAg * 2) % 16 || (sWg * 2) % 16)
    return fail(DCHAG_ERR_SHAPE, "gemm: strides must be multiples of 16 bytes");
  const int bk = (K % 64 == 0) ? 64 : (K % 32 == 0 ? 32 : 16);
  // N tiling: <= 256 columns per tile, as even as possible (N = 1040 -> 5 x 208)
  const int ntn = (N + 255) / 256;
  const int bn = ((N + ntn - 1) / ntn + 15) / 16 * 16;
  const int ntm = Mo * Mi / 128;
  // CTA pairs (M = 256 tiles, W split across the pair) on the K-64 path when the M tiles pair
  // up; DCHAG_GEMM_PAIR=0 selects the single-CTA kernel (A/B probes)
  int pair = bk == 64 && ntm % 2 == 0 && (bn / 2) % 8 == 0;
  if (const char* f = getenv("DCHAG_GEMM_PAIR")) pair = pair && atoi(f) != 0;
  const CUtensorMapSwizzle swz = bk == 64   ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : bk == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                            : CU_TENSOR_MAP_SWIZZLE_32B;
  CUtensorMap tA, tW;
  {
    cuuint64_t dims[4] = {(cuuint64_t)K, (cuuint64_t)Mi, (cuuint64_t)Mo, (cuuint64_t)G};
    cuuint64_t str[3] = {(cuuint64_t)sAmi * 2, (cuuint64_t)sAmo * 2, (cuuint64_t)sAg * 2};
    cuuint32_t box[4] = {(cuuint32_t)bk, 128u, 1, 1};
    int rc = make_map(&tA, A, 4, dims, str, box, swz);
    if (rc) return rc;
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)N, (cuuint64_t)G};
    cuuint64_t str[2] = {(cuuint64_t)K * 2, (cuuint64_t)sWg * 2};
    cuuint32_t box[3] = {(cuuint32_t)bk, (cuuint32_t)(pair ? bn / 2 : bn), 1};
    int rc = make_map(&tW, W, 3, dims, str, box, swz);
    if (rc) return rc;
  }
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.G = G; a.M = Mo * Mi; a.Mi = Mi; a.N = N; a.Nv = Nv; a.K = K; a.BN = bn;
  a.pair = pair;
  // value columns by TMA tensor store (bf16 output, 16-byte aligned strides, 32-row boxes)
  CUtensorMap tV;
  memset(&tV, 0, sizeof(tV));
  a.debug = getenv("DCHAG_GEMM_DEBUG") ? atoi(getenv("DCHAG_GEMM_DEBUG")) : 0;
  // the lean epilogue: plain bf16 tiles, all full and 64-column aligned (DCHAG_GEMM_LEAN=0
  // selects the general epilogue, for A/B probes)
  const char* lean_env = getenv("DCHAG_GEMM_LEAN");
  const bool lean = pair && !dot && !rowbias && !rmask && outV && !outV_f32 && Nv == N &&
                    bn % 64 == 0 && N % bn == 0 && Mi % 32 == 0 && a.debug == 0 &&
                    (!bias || (bias_g % 4 == 0 && reinterpret_cast<uintptr_t>(bias) % 16 == 0)) &&
                    !(lean_env && atoi(lean_env) == 0);
  // narrow fp32 logit-only GEMMs (the full_cross u columns): lean drain, direct row stores
  if (pair && !dot && !rowbias && !rmask && Nv == 0 && outL && N <= 256 && N % 16 == 0 &&
      bn == N && a.debug == 0 && !(lean_env && atoi(lean_env) == 0) &&
      ((reinterpret_cast<uintptr_t>(outL) | (uintptr_t)(sLmi * 4) | (uintptr_t)(sLmo * 4) |
        (uintptr_t)(sLg * 4)) % 16) == 0 &&
      (!bias || (bias_g % 4 == 0 && reinterpret_cast<uintptr_t>(bias) % 16 == 0)))
    a.lean = 3;
  if (outV && !outV_f32 && Nv >= 32 && Mi % 32 == 0 &&
      ((reinterpret_cast<uintptr_t>(outV) | (uintptr_t)(sVmi * 2) | (uintptr_t)(sVmo * 2) |
        (uintptr_t)(sVg * 2)) % 16) == 0 && !getenv("DCHAG_GEMM_NO_TMA_STORE")) {
    cuuint64_t dims[4] = {(cuuint64_t)Nv, (cuuint64_t)Mi, (cuuint64_t)Mo, (cuuint64_t)G};
    cuuint64_t str[3] = {(cuuint64_t)sVmi * 2, (cuuint64_t)(Mo > 1 ? sVmo : Mi * sVmi) * 2,
                         (cuuint64_t)(G > 1 ? sVg : Mo * (Mo > 1 ? sVmo : Mi * sVmi)) * 2};
    cuuint32_t box[4] = {lean ? 64u : 32u, 32, 1, 1};
    if (make_map(&tV, outV, 4, dims, str, box,
                 lean ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B) == DCHAG_OK) {
      a.v_tma = 1;
      a.lean = lean;
    }
  }
  a.bias = bias; a.bias_g = bias_g;
  a.rowbias = reinterpret_cast<const __nv_bfloat16*>(rowbias);
  a.rowbias_g = rowbias_g; a.rowbias_row = rowbias_row;
  a.rowbias_period = rowbias_period > 0 ? rowbias_period : 1;
  a.outV = outV; a.outV_f32 = outV_f32; a.sVg = sVg; a.sVmo = sVmo; a.sVmi = sVmi;
  a.outL = outL; a.sLg = sLg; a.sLmo = sLmo; a.sLmi = sLmi;
  a.rmask = rmask; a.mtok = mtok;
  if (dot) {
    if (N % 32 || bn % 32 || ldG % 8 || !dotG || (reinterpret_cast<uintptr_t>(dotG) % 16))
      return fail(DCHAG_ERR_SHAPE, "gemm_rowdot: N, tile width and ldG must suit 32-column "
                                   "groups of 16-byte aligned rows (N=%d ldG=%lld)", N, ldG);
    a.v_tma = 0; a.rowbias = nullptr; a.outV = nullptr; a.outL = nullptr; a.Nv = N;
    a.dotG = reinterpret_cast<const __nv_bfloat16*>(dotG); a.ldG = ldG; a.dotOut = dotOut;
    // lean row-dot drain: full tiles, 64-column aligned (DCHAG_GEMM_LEAN=0: general drain)
    if ((a.debug & 16) && getenv("DCHAG_GEMM_TRACE_BUF"))  // timing probe: trace buffer
      a.outL = reinterpret_cast<float*>(strtoull(getenv("DCHAG_GEMM_TRACE_BUF"), nullptr, 0));
    a.lean = (pair && bn % 64 == 0 && N % bn == 0 && (a.debug & ~20) == 0 &&
              (!bias || (bias_g % 4 == 0 && reinterpret_cast<uintptr_t>(bias) % 16 == 0)) &&
              !(lean_env && atoi(lean_env) == 0)) ? 2 : 0;
    a.dot64 = dot_group == 64;
    if (a.dot64 && (a.lean != 2 || N % 64))
      return fail(DCHAG_ERR_SHAPE, "gemm_rowdot_heads: 64-column groups need the lean row-dot "
                                   "drain (CTA pairs, 64-column tiles; N=%d)", N);
  }
  return cuda_status(launch_gemm(tA, tW, tV, a, bk, num_sms_cached(), S(stream)), "gemm");
}

int dchag_gemm_bf16(const void* A, int G, int Mo, int Mi, int K, long long sAg, long long sAmo,
                    long long sAmi, const void* W, int N, long long sWg, int Nv,
                    const float* bias, long long bias_g, const void* rowbias,
                    long long rowbias_g, long long rowbias_row, int rowbias_period, void* outV,
                    int outV_f32, long long sVg, long long sVmo, long long sVmi, float* outL,
                    long long sLg, long long sLmo, long long sLmi, void* stream) {
  return gemm_impl(A, G, Mo, Mi, K, sAg, sAmo, sAmi, W, N, sWg, Nv, bias, bias_g, rowbias,
                   rowbias_g, rowbias_row, rowbias_period, outV, outV_f32, sVg, sVmo, sVmi, outL,
                   sLg, sLmo, sLmi, nullptr, 0, nullptr, stream);
}

int dchag_gemm_nt(const void* A, int a_mn, long long lda, long long sAko, int Ki,
                  long long sAg, const void* B, int b_mn, long long ldb, long long sBg, int G,
                  int M, int N, int K, const float* bias, long long bias_g, void* out,
                  int out_f32, int accumulate, long long ldc, long long sCg, void* stream) {
  if (G < 1 || M < 128 || M % 128 || N < 16 || N % 16 || K < 64 || K % 64 || !A || !B ||
      !out || (a_mn && (Ki < 64 || Ki % 64 || K % Ki)) || (accumulate && !out_f32))
    return fail(DCHAG_ERR_SHAPE, "gemm_nt: bad shape G=%d M=%d N=%d K=%d Ki=%d", G, M, N, K, Ki);
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) % 16 ||
      (lda * 2) % 16 || (sAko * 2) % 16 || (sAg * 2) % 16 || (ldb * 2) % 16 || (sBg * 2) % 16)
    return fail(DCHAG_ERR_SHAPE, "gemm_nt: operand pointers / strides must be 16-byte aligned");
  const int lay = (a_mn ? 1 : 0) | (b_mn ? 2 : 0);
  const int ntm = M / 128;
  const int pair = ntm % 2 == 0;
  if (lay && !pair) return fail(DCHAG_ERR_SHAPE, "gemm_nt: MN-major operands need M %% 256 == 0");
  // N tiles of 256 (128 when that is needed to fill the SMs, or for small N)
  int bn = N >= 256 ? 256 : (N + 15) / 16 * 16;
  if (b_mn) bn = N >= 256 ? 256 : 128;
  const int sms = num_sms_cached();
  auto units = [&](int b) { return G * (ntm / (pair ? 2 : 1)) * ((N + b - 1) / b); };
  if (bn == 256 && units(256) < sms / (pair ? 2 : 1) && N > 128) bn = 128;
  CUtensorMap tA, tW, tV;
  memset(&tV, 0, sizeof(tV));
  int rc;
  if (a_mn) {
    cuuint64_t dims[4] = {(cuuint64_t)M, (cuuint64_t)Ki, (cuuint64_t)(K / Ki), (cuuint64_t)G};
    cuuint64_t str[3] = {(cuuint64_t)lda * 2, (cuuint64_t)sAko * 2, (cuuint64_t)sAg * 2};
    cuuint32_t box[4] = {64u, 64u, 1, 1};
    rc = make_map(&tA, A, 4, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
  } else {
    cuuint64_t dims[4] = {(cuuint64_t)K, (cuuint64_t)M, 1, (cuuint64_t)G};
    cuuint64_t str[3] = {(cuuint64_t)lda * 2, (cuuint64_t)lda * M * 2, (cuuint64_t)sAg * 2};
    cuuint32_t box[4] = {64u, 128u, 1, 1};
    rc = make_map(&tA, A, 4, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  if (rc) return rc;
  if (b_mn) {
    cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)K, (cuuint64_t)G};
    cuuint64_t str[2] = {(cuuint64_t)ldb * 2, (cuuint64_t)sBg * 2};
    cuuint32_t box[3] = {64u, 64u, 1};
    rc = make_map(&tW, B, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
  } else {
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)N, (cuuint64_t)G};
    cuuint64_t str[2] = {(cuuint64_t)ldb * 2, (cuuint64_t)sBg * 2};
    cuuint32_t box[3] = {64u, (cuuint32_t)(pair ? bn / 2 : bn), 1};
    rc = make_map(&tW, B, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  if (rc) return rc;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.G = G; a.M = M; a.Mi = M; a.N = N; a.Nv = N; a.K = K; a.BN = bn;
  a.pair = pair; a.lay = lay; a.Ki = a_mn ? Ki : K; a.accum = accumulate;
  a.bias = bias; a.bias_g = bias_g; a.rowbias_period = 1;
  a.outV = out; a.outV_f32 = out_f32; a.sVg = sCg; a.sVmo = 0; a.sVmi = ldc;
  const char* lean_env = getenv("DCHAG_GEMM_LEAN");
  const bool lean = pair && !lay && !out_f32 && bn % 64 == 0 && N % bn == 0 &&
                    (!bias || (bias_g % 4 == 0 && reinterpret_cast<uintptr_t>(bias) % 16 == 0)) &&
                    !getenv("DCHAG_GEMM_DEBUG") && !(lean_env && atoi(lean_env) == 0);
  if (!out_f32 && N >= 32 &&
      ((reinterpret_cast<uintptr_t>(out) | (uintptr_t)(ldc * 2) | (uintptr_t)(sCg * 2)) % 16) == 0) {
    cuuint64_t dims[4] = {(cuuint64_t)N, (cuuint64_t)M, 1, (cuuint64_t)G};
    cuuint64_t str[3] = {(cuuint64_t)ldc * 2, (cuuint64_t)M * ldc * 2,
                         (cuuint64_t)(G > 1 ? sCg : M * ldc) * 2};
    cuuint32_t box[4] = {lean ? 64u : 32u, 32, 1, 1};
    if (make_map(&tV, out, 4, dims, str, box,
                 lean ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B) == DCHAG_OK) {
      a.v_tma = 1;
      a.lean = lean;
    }
  }
  return cuda_status(launch_gemm(tA, tW, tV, a, 64, sms, S(stream)), "gemm_nt");
}

int dchag_final_vit(const void* ctx, int B, int seq, int K, const void* W, int D,
                    const float* bias, const float* mask, const float* mask_token,
                    const float* meta, int kmeta, const float* meta_w, const float* meta_b,
                    void* out, int out_f32, void* stream) {
  if (!ctx || !W || !mask || !mask_token || !out || B < 1 || seq < 128 || seq % 128 || D % 16 ||
      kmeta < 0 || (kmeta && (!meta || !meta_w)) || !meta_b)
    return fail(DCHAG_ERR_SHAPE, "final_vit: bad arguments B=%d S=%d D=%d", B, seq, D);
  const size_t es = out_f32 ? 4 : 2;
  void* rows = reinterpret_cast<uint8_t*>(out) + (size_t)D * es;  // out[b][1 + s]
  int rc = gemm_impl(ctx, 1, B, seq, K, (long long)B * seq * K, (long long)seq * K, K, W, D,
                     (long long)D * K, D, bias, D, nullptr, 0, 0, 1, rows, out_f32, 0,
                     (long long)(seq + 1) * D, D, nullptr, 0, 0, 0, nullptr, 0, nullptr, stream,
                     mask, mask_token);
  if (rc) return rc;
  return cuda_status(launch_vit_meta(meta, kmeta, meta_w, meta_b, out, out_f32, B, seq, D,
                                     S(stream)), "final_vit");
}

int dchag_gemm_rowdot(const void* A, int G, int Mo, int Mi, int K, long long sAg,
                      long long sAmo, long long sAmi, const void* W, int N, long long sWg,
                      const float* bias, long long bias_g, const void* Gmat, long long ldG,
                      float* dot_out, void* stream) {
  if (!dot_out) return fail(DCHAG_ERR_SHAPE, "gemm_rowdot: dot_out is null");
  return gemm_impl(A, G, Mo, Mi, K, sAg, sAmo, sAmi, W, N, sWg, N, bias, bias_g, nullptr, 0, 0,
                   1, nullptr, 0, 0, 0, 0, nullptr, 0, 0, 0, Gmat, ldG, dot_out, stream);
}

int dchag_gemm_rowdot_heads(const void* A, int G, int Mo, int Mi, int K, long long sAg,
                            long long sAmo, long long sAmi, const void* W, int N, long long sWg,
                            const float* bias, long long bias_g, const void* Gmat, long long ldG,
                            int group, float* dot_out, void* stream) {
  if (!dot_out) return fail(DCHAG_ERR_SHAPE, "gemm_rowdot_heads: dot_out is null");
  if (group != 32 && group != 64)
    return fail(DCHAG_ERR_SHAPE, "gemm_rowdot_heads: group must be 32 or 64 (got %d)", group);
  return gemm_impl(A, G, Mo, Mi, K, sAg, sAmo, sAmi, W, N, sWg, N, bias, bias_g, nullptr, 0, 0,
                   1, nullptr, 0, 0, 0, 0, nullptr, 0, 0, 0, Gmat, ldG, dot_out, stream, nullptr,
                   nullptr, group);
}

int dchag_gemm_combine(const void* ctx, int n_children, int R, int D, int H, const void* W,
                       long long sWg, const float* bias, long long bias_g, const float* Lpre,
                       const int* first, const int* count, int n_parents, int csplit,
                       void* out, void* stream) {
  if (csplit != 1 && csplit != 2)
    return fail(DCHAG_ERR_SHAPE, "gemm_combine: csplit must be 1 or 2");
  if (n_children < 1 || n_parents < 1 || R < 256 || R % 256 || D < 256 || D % 256 || H < 1 ||
      D % H || (D / H) % 32 || !Lpre || !first || !count || !out)
    return fail(DCHAG_ERR_SHAPE, "gemm_combine: bad shape R=%d D=%d H=%d", R, D, H);
  if ((reinterpret_cast<uintptr_t>(ctx) | reinterpret_cast<uintptr_t>(W) |
       reinterpret_cast<uintptr_t>(out) | (uintptr_t)(sWg * 2)) % 16)
    return fail(DCHAG_ERR_SHAPE, "gemm_combine: pointers / strides must be 16-byte aligned");
  const int bn = 256;
  CUtensorMap tA, tW, tV;
  {
    cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)R, 1, (cuuint64_t)n_children};
    cuuint64_t str[3] = {(cuuint64_t)D * 2, (cuuint64_t)R * D * 2, (cuuint64_t)R * D * 2};
    cuuint32_t box[4] = {64u, 128u, 1, 1};
    int rc = make_map(&tA, ctx, 4, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)D, (cuuint64_t)n_children};
    cuuint64_t str[2] = {(cuuint64_t)D * 2, (cuuint64_t)sWg * 2};
    cuuint32_t box[3] = {64u, (cuuint32_t)(bn / 2), 1};
    int rc = make_map(&tW, W, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  // lean combine drain (heads of >= 64 columns, 64-column aligned; DCHAG_GEMM_LEAN=0 or a
  // timing probe selects the general epilogue)
  const char* lean_env = getenv("DCHAG_GEMM_LEAN");
  const int dbg = getenv("DCHAG_GEMM_DEBUG") ? atoi(getenv("DCHAG_GEMM_DEBUG")) : 0;
  const bool lean = (D / H) % 64 == 0 && dbg == 0 && !(lean_env && atoi(lean_env) == 0) &&
                    (!bias || (bias_g % 4 == 0 && reinterpret_cast<uintptr_t>(bias) % 16 == 0));
  {
    cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)R, 1, (cuuint64_t)n_parents * csplit};
    cuuint64_t str[3] = {(cuuint64_t)D * 2, (cuuint64_t)R * D * 2, (cuuint64_t)R * D * 2};
    cuuint32_t box[4] = {lean ? 64u : 32u, 32, 1, 1};
    int rc = make_map(&tV, out, 4, dims, str, box,
                      lean ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.G = n_parents * csplit; a.M = R; a.Mi = R; a.N = D; a.Nv = D; a.K = D; a.BN = bn;
  a.nparents = n_parents; a.csplit = csplit;
  a.pair = 1; a.v_tma = 1;
  a.bias = bias; a.bias_g = bias_g;
  a.rowbias_period = 1;
  a.outV = out; a.sVg = (long long)R * D; a.sVmo = 0; a.sVmi = D;
  a.cfirst = first; a.ccount = count; a.Lpre = Lpre; a.H = H; a.dh = D / H;
  a.debug = dbg;
  a.lean = lean ? 4 : 0;
  return cuda_status(launch_gemm(tA, tW, tV, a, 64, num_sms_cached(), S(stream)),
                     "gemm_combine");
}

int dchag_l0_logits(const void* img, long long img_sb, long long img_sc, int B, int Himg, int W,
                    int P, int H, int HP, int nh, int n_nodes, int gmax, const int* node_c0,
                    const int* node_g,
                    const long long* node_poff, const void* WUt, const float* bU,
                    const float* posU, void* p, float* pinv, void* stream) {
  if (Himg % P || W % P || HP % 8 || HP < H || H % 2 || (P * P) % 16 || (nh != 2 && nh != 4) ||
      H % nh)
    return fail(DCHAG_ERR_SHAPE, "l0_logits: bad shape");
  L0LogitArgs a;
  memset(&a, 0, sizeof(a));
  if (const char* tr = getenv("DCHAG_P0_TRACE_PTR"))
    a.trace = reinterpret_cast<long long*>(strtoull(tr, nullptr, 0));
  if (const char* is = getenv("DCHAG_P0_ISSUE")) a.issue_serial = atoi(is) == 1;
  a.img = reinterpret_cast<const __nv_bfloat16*>(img);
  a.img_sb = img_sb; a.img_sc = img_sc;
  a.B = B; a.S = (Himg / P) * (W / P); a.W = W; a.P = P; a.wp = W / P; a.H = H; a.HP = HP;
  a.n_nodes = n_nodes; a.gmax = gmax;
  a.nh = nh;
  a.node_c0 = node_c0; a.node_g = node_g; a.node_poff = node_poff;
  a.WUt = reinterpret_cast<const __nv_bfloat16*>(WUt);
  a.bU = bU; a.posU = posU;
  a.p = reinterpret_cast<__nv_bfloat16*>(p);
  a.pinv = pinv;
  if ((B * a.S) % 16) return fail(DCHAG_ERR_SHAPE, "l0_logits: B*S must be a multiple of 16");
  if ((reinterpret_cast<uintptr_t>(img) | (uintptr_t)(img_sb * 2) | (uintptr_t)(img_sc * 2) |
       (uintptr_t)(W * 2)) % 16)
    return fail(DCHAG_ERR_SHAPE, "l0_logits: image base/strides must be 16-byte aligned");
  return cuda_status(launch_l0_logits(a, num_sms_cached(), S(stream)), "l0_logits");
}

int dchag_l0_node(const void* img, long long img_sb, long long img_sc, int B, int Himg, int W,
                  int P, int H, int D, int n_nodes, const int* node_c0, const int* node_g,
                  const long long* node_poff, int p_row_mode, const void* p, const float* pinv,
                  const void* Mt, int C_pad, const void* Et, int KE, const void* posV, void* ctx,
                  void* stream) {
  if (Himg % P || W % P) return fail(DCHAG_ERR_SHAPE, "l0_node: image not divisible by patch");
  L0NodeArgs a;
  memset(&a, 0, sizeof(a));
  a.img = reinterpret_cast<const __nv_bfloat16*>(img);
  a.img_sb = img_sb; a.img_sc = img_sc;
  a.B = B; a.S = (Himg / P) * (W / P); a.W = W; a.P = P; a.wp = W / P; a.H = H; a.D = D;
  a.n_nodes = n_nodes; a.node_c0 = node_c0; a.node_g = node_g; a.node_poff = node_poff;
  a.nh = (H > 0 && D / H == 128) ? 2 : (H % 4 == 0 ? 4 : 2);
  a.p_row_mode = p_row_mode;
  a.p = reinterpret_cast<const __nv_bfloat16*>(p);
  a.pinv = pinv;
  a.Mt = reinterpret_cast<const __nv_bfloat16*>(Mt);
  a.C_pad = C_pad;
  a.Et = reinterpret_cast<const __nv_bfloat16*>(Et);
  a.KE = KE;
  a.ctx = reinterpret_cast<__nv_bfloat16*>(ctx);
  {
    const char* dbg = getenv("DCHAG_L0_DEBUG");
    a.debug_mode = dbg ? atoi(dbg) : 0;
    const char* tr = getenv("DCHAG_L0_TRACE_PTR");
    a.trace = tr ? reinterpret_cast<long long*>(strtoull(tr, nullptr, 0)) : nullptr;
  }
  if ((reinterpret_cast<uintptr_t>(img) | (uintptr_t)(img_sb * 2) | (uintptr_t)(img_sc * 2)) % 16)
    return fail(DCHAG_ERR_SHAPE, "l0_node: image base/strides must be 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(ctx) % 16 || (D * 2) % 16)
    return fail(DCHAG_ERR_SHAPE, "l0_node: ctx must be 16-byte aligned");
  // ctx [n_nodes * R rows][D] bf16; one store box = 64 columns (a head) x 128 rows, 128B swizzle
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)n_nodes * B * a.S};
  const cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  const cuuint32_t box[2] = {64, 128};
  if (int rc = make_map(&tm, ctx, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  // posV [n_nodes * S rows][D] bf16, same box geometry (loaded into the staging tile)
  CUtensorMap tp;
  memset(&tp, 0, sizeof(tp));
  a.has_pos = posV != nullptr;
  if (posV) {
    if (reinterpret_cast<uintptr_t>(posV) % 16)
      return fail(DCHAG_ERR_SHAPE, "l0_node: posV must be 16-byte aligned");
    const cuuint64_t pdims[2] = {(cuuint64_t)D, (cuuint64_t)n_nodes * a.S};
    if (int rc = make_map(&tp, posV, 2, pdims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
  }
  return cuda_status(launch_l0_node(a, tm, tp, num_sms_cached(), S(stream)), "l0_node");
}

int dchag_combine(int n_nodes, int R, int D, int H, const int* node_first, const int* node_g,
                  int max_g, const void* V, long long sVj, const float* L, long long sLj,
                  const float* mix, void* ctx, void* stream) {
  return dchag_combine_strided(n_nodes, R, D, H, node_first, node_g, max_g, V, sVj, 0, L, sLj,
                               0, R, mix, ctx, stream);
}

int dchag_combine_strided(int n_nodes, int R, int D, int H, const int* node_first,
                          const int* node_g, int max_g, const void* V, long long sVj,
                          long long sVb, const float* L, long long sLj, long long sLb,
                          int rows_inner, const float* mix, void* ctx, void* stream) {
  if (!mix && !L) return fail(DCHAG_ERR_SHAPE, "combine: need logits or mix");
  if (rows_inner < 1) return fail(DCHAG_ERR_SHAPE, "combine: rows_inner must be >= 1");
  CombineArgs a;
  memset(&a, 0, sizeof(a));
  a.n_nodes = n_nodes; a.R = R; a.D = D; a.H = H; a.max_g = max_g;
  a.rows_inner = rows_inner; a.sVb = sVb; a.sLb = sLb;
  a.node_first = node_first; a.node_g = node_g;
  a.V = reinterpret_cast<const __nv_bfloat16*>(V); a.sVj = sVj;
  a.L = L; a.sLj = sLj; a.mix = mix;
  a.ctx = reinterpret_cast<__nv_bfloat16*>(ctx);
  return cuda_status(launch_combine(a, S(stream)), "combine");
}

int dchag_l0_dv(int g, int R, int D, int H, int nh, const void* p, const float* mix,
                const void* G, const float* posV, long long ldpos, int period, float* Gpos,
                void* dV, void* stream) {
  if (!mix && !p && dV) return fail(DCHAG_ERR_SHAPE, "l0_dv: need p or mix");
  if (!dV && !posV) return fail(DCHAG_ERR_SHAPE, "l0_dv: nothing to compute");
  const int dh = H > 0 ? D / H : 0;
  if (H < 1 || D % H || dh % 8 || dh > 256 || ((dh / 8) & (dh / 8 - 1)) ||
      ((long long)R * (D / 8)) % 32 || (!mix && (nh < 1 || H % nh)) ||
      (posV && (!Gpos || period < 1 || R % period || (ldpos && (ldpos < D || ldpos % 4)))) ||
      (reinterpret_cast<uintptr_t>(G) | reinterpret_cast<uintptr_t>(dV) |
       reinterpret_cast<uintptr_t>(posV)) % 16)
    return fail(DCHAG_ERR_SHAPE, "l0_dv: bad shape R=%d D=%d H=%d nh=%d", R, D, H, nh);
  return cuda_status(launch_l0_dv(g, R, D, H, nh, reinterpret_cast<const __nv_bfloat16*>(p), mix,
                                  reinterpret_cast<const __nv_bfloat16*>(G), posV, ldpos, period,
                                  Gpos,
                                  reinterpret_cast<__nv_bfloat16*>(dV), S(stream)),
                     "l0_dv");
}

int dchag_vit_tokens(const void* agg, int agg_f32, int B, int seq, int D, const float* mask,
                     const float* mask_token, const float* meta_tok, void* out, void* stream) {
  if (B < 1 || seq < 1 || D < 8 || D % 8 || !agg || !mask || !mask_token || !meta_tok || !out)
    return fail(DCHAG_ERR_SHAPE, "vit_tokens: bad shape B=%d S=%d D=%d", B, seq, D);
  return cuda_status(launch_vit_tokens(agg, agg_f32, mask, mask_token, meta_tok, out, B, seq, D,
                                       S(stream)),
                     "vit_tokens");
}

int dchag_l0_tgrad(const void* patches, int cnt, int c0, int g, int R, int seq, int D, int H,
                   int nh, int PP, const void* p, const float* mix, const void* G, float* T,
                   void* stream) {
  if (!mix && !p) return fail(DCHAG_ERR_SHAPE, "l0_tgrad: need p or mix");
  if (H < 1 || D % H || D % 128 || R % 64 || seq % 64 || R % seq || PP != 64 ||
      (D / H != 64 && D / H != 128) || (!mix && (nh < 2 || nh % 2 || H % nh)) ||
      (reinterpret_cast<uintptr_t>(patches) | reinterpret_cast<uintptr_t>(G)) % 16)
    return fail(DCHAG_ERR_SHAPE, "l0_tgrad: bad shape R=%d S=%d D=%d H=%d PP=%d", R, seq, D, H,
                PP);
  L0TgradArgs a;
  memset(&a, 0, sizeof(a));  // every field defined (timing-probe bits included)
  a.debug = getenv("DCHAG_TE_DEBUG") ? atoi(getenv("DCHAG_TE_DEBUG")) : 0;
  a.patches = reinterpret_cast<const __nv_bfloat16*>(patches);
  a.cnt = cnt; a.c0 = c0; a.g = g; a.R = R; a.S = seq; a.D = D; a.H = H; a.NH = nh; a.PP = PP;
  a.p = reinterpret_cast<const __nv_bfloat16*>(p); a.mix = mix;
  a.G = reinterpret_cast<const __nv_bfloat16*>(G); a.T = T;
  // tcgen05 form (K_tgc: both operands MN-major straight from their global layouts) unless
  // DCHAG_TG_TC=0 selects the mma.sync kernel
  const char* tc = getenv("DCHAG_TG_TC");
  if (!(tc && atoi(tc) == 0)) {
    const int B = R / seq;
    CUtensorMap tG, tP;
    cuuint64_t gd[2] = {(cuuint64_t)D, (cuuint64_t)R};
    cuuint64_t gs[1] = {(cuuint64_t)D * 2};
    cuuint32_t gb[2] = {64u, 64u};
    int rc = make_map(&tG, G, 2, gd, gs, gb, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    cuuint64_t pd[3] = {64u, (cuuint64_t)seq, (cuuint64_t)B * cnt};
    cuuint64_t ps[2] = {64u * 2, (cuuint64_t)seq * 64 * 2};
    cuuint32_t pb[3] = {64u, 64u, 1u};
    rc = make_map(&tP, patches, 3, pd, ps, pb, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    return cuda_status(launch_l0_tgrad_tc(tG, tP, a, S(stream)), "l0_tgrad_tc");
  }
  return cuda_status(launch_l0_tgrad(a, S(stream)), "l0_tgrad");
}

int dchag_child_softmax(float* L, const int* first, const int* count, int n_parents, int R,
                        int H, void* stream) {
  if (!L || !first || !count || n_parents < 1 || R < 1 || H < 1)
    return fail(DCHAG_ERR_SHAPE, "child_softmax: bad arguments");
  return cuda_status(launch_child_softmax(L, first, count, n_parents, R, H, S(stream)),
                     "child_softmax");
}

int dchag_l0_softmax_bwd(int g, int R, int H, int nh, int dh, const float* dpp,
                         const float* Gpos, const void* p, float* dl, void* dlb, void* stream) {
  if (g < 1 || R < 1 || H < 1 || dh % 32 || nh < 1 || H % nh || !dpp || !Gpos || !p ||
      (!dl && (g > 16 || (dh != 64 && dh != 32))) || !dlb)
    return fail(DCHAG_ERR_SHAPE, "l0_softmax_bwd: bad arguments");
  return cuda_status(launch_l0_softmax_bwd(g, R, H, nh, dh, dpp, Gpos,
                                           reinterpret_cast<const __nv_bfloat16*>(p), dl,
                                           reinterpret_cast<__nv_bfloat16*>(dlb), S(stream)),
                     "l0_softmax_bwd");
}

int dchag_combine_f32(int n_nodes, int R, int D, int H, const int* node_first, const int* node_g,
                      int max_g, const float* V, long long sVj, const float* L, long long sLj,
                      const float* mix, float* ctx, void* stream) {
  if (!mix && !L) return fail(DCHAG_ERR_SHAPE, "combine_f32: need logits or mix");
  CombineF32Args a;
  memset(&a, 0, sizeof(a));
  a.n_nodes = n_nodes; a.R = R; a.D = D; a.H = H; a.max_g = max_g;
  a.node_first = node_first; a.node_g = node_g;
  a.V = V; a.sVj = sVj; a.L = L; a.sLj = sLj; a.mix = mix; a.ctx = ctx;
  return cuda_status(launch_combine_f32(a, S(stream)), "combine_f32");
}

int dchag_fullcross_weights(int n_nodes, int R, int D, int H, const int* node_first,
                            const int* node_g, int max_g, const void* QK, long long sQj,
                            long long ldq, const float* u, long long sUj, float* w,
                            const void* posq, int seq, void* pout, const long long* node_poff,
                            int nh, void* stream) {
  if (D % H || (D / H) % 16 || max_g < 1 || max_g > 32 || H > 32 || ldq < 2 * D || (ldq * 2) % 16 ||
      (sQj * 2) % 16 || reinterpret_cast<uintptr_t>(QK) % 16)
    return fail(DCHAG_ERR_SHAPE, "fullcross_weights: bad shape");
  FullCrossArgs a;
  memset(&a, 0, sizeof(a));
  a.n_nodes = n_nodes; a.R = R; a.D = D; a.H = H; a.max_g = max_g;
  a.node_first = node_first; a.node_g = node_g;
  a.QK = reinterpret_cast<const __nv_bfloat16*>(QK); a.sQj = sQj; a.ldq = ldq;
  a.u = u; a.sUj = sUj; a.w = w;
  a.posq = reinterpret_cast<const __nv_bfloat16*>(posq); a.S = seq > 0 ? seq : 1;
  a.pout = reinterpret_cast<__nv_bfloat16*>(pout); a.node_poff = node_poff; a.nh = nh;
  if (pout && (!node_poff || nh < 1 || H % nh))
    return fail(DCHAG_ERR_SHAPE, "fullcross_weights: p output needs node_poff and nh | H");
  if (!pout && !w) return fail(DCHAG_ERR_SHAPE, "fullcross_weights: no output");
  if (posq && (seq < 1 || R % seq)) return fail(DCHAG_ERR_SHAPE, "fullcross_weights: bad seq");
  return cuda_status(launch_fullcross_weights(a, S(stream)), "fullcross_weights");
}

int dchag_fullcross_bwd(int n_nodes, int R, int D, int H, const int* node_first,
                        const int* node_g, int max_g, const void* QKV, long long sQj,
                        long long ldq, const float* u, const float* G, const float* a_vec,
                        void* dQKV, float* dA, void* stream) {
  if (D % H || (D / H) % 16 || max_g < 1 || max_g > 16 || H > 32 || ldq < 3 * D ||
      (ldq * 2) % 16 || (sQj * 2) % 16 || reinterpret_cast<uintptr_t>(QKV) % 16 || !u || !G ||
      !a_vec || !dQKV || !dA)
    return fail(DCHAG_ERR_SHAPE, "fullcross_bwd: bad shape");
  FullCrossBwdArgs a;
  memset(&a, 0, sizeof(a));
  a.n_nodes = n_nodes; a.R = R; a.D = D; a.H = H; a.max_g = max_g;
  a.node_first = node_first; a.node_g = node_g;
  a.QKV = reinterpret_cast<const __nv_bfloat16*>(QKV); a.sQj = sQj; a.ldq = ldq;
  a.u = u; a.G = G; a.a = a_vec; a.dQKV = reinterpret_cast<__nv_bfloat16*>(dQKV); a.dA = dA;
  return cuda_status(launch_fullcross_bwd(a, S(stream)), "fullcross_bwd");
}

int dchag_combine_weighted(int n_nodes, int R, int D, int H, const int* node_first,
                           const int* node_g, int max_g, const void* V, long long sVj,
                           long long ldv, const float* w, void* ctx, void* stream) {
  CombineArgs a;
  memset(&a, 0, sizeof(a));
  a.n_nodes = n_nodes; a.R = R; a.D = D; a.H = H; a.max_g = max_g;
  a.rows_inner = R; a.node_first = node_first; a.node_g = node_g;
  a.V = reinterpret_cast<const __nv_bfloat16*>(V); a.sVj = sVj; a.ldv = ldv;
  a.W = w;
  a.ctx = reinterpret_cast<__nv_bfloat16*>(ctx);
  if (!w || (ldv * 2) % 16) return fail(DCHAG_ERR_SHAPE, "combine_weighted: bad arguments");
  return cuda_status(launch_combine(a, S(stream)), "combine_weighted");
}

int dchag_combine_bwd(int n_nodes, int R, int D, int H, const int* node_first, const int* node_g,
                      int max_g, const void* V, long long sVj, const float* L, long long sLj,
                      const float* mix, const float* G, float* dL, void* gV, float* dm,
                      void* stream) {
  if (!mix && (!L || !dL)) return fail(DCHAG_ERR_SHAPE, "combine_bwd: attention needs L and dL");
  if (mix && !dm) return fail(DCHAG_ERR_SHAPE, "combine_bwd: linear needs dm");
  CombineBwdArgs a;
  memset(&a, 0, sizeof(a));
  a.n_nodes = n_nodes; a.R = R; a.D = D; a.H = H; a.max_g = max_g;
  a.node_first = node_first; a.node_g = node_g;
  a.V = reinterpret_cast<const __nv_bfloat16*>(V); a.sVj = sVj;
  a.L = L; a.sLj = sLj; a.mix = mix; a.G = G; a.dL = dL;
  a.gV = reinterpret_cast<__nv_bfloat16*>(gV); a.dm = dm;
  return cuda_status(launch_combine_bwd(a, S(stream)), "combine_bwd");
}

int dchag_combine_bwd_packed(int n_nodes, int R, int D, int H, const int* node_first,
                             const int* node_g, int max_g, const void* V, long long sVj,
                             const float* L, long long sLj, const float* mix, const float* G,
                             void* gVL, long long sGj, long long ldg, float* dm, void* stream) {
  if (!mix && !L) return fail(DCHAG_ERR_SHAPE, "combine_bwd_packed: attention needs L");
  if (mix && !dm) return fail(DCHAG_ERR_SHAPE, "combine_bwd_packed: linear needs dm");
  if (ldg < D + (mix ? 0 : H) || ldg % 8 || sGj < (long long)R * ldg)
    return fail(DCHAG_ERR_SHAPE, "combine_bwd_packed: row stride %lld too small", ldg);
  CombineBwdArgs a;
  memset(&a, 0, sizeof(a));
  a.n_nodes = n_nodes; a.R = R; a.D = D; a.H = H; a.max_g = max_g;
  a.node_first = node_first; a.node_g = node_g;
  a.V = reinterpret_cast<const __nv_bfloat16*>(V); a.sVj = sVj;
  a.L = L; a.sLj = sLj; a.mix = mix; a.G = G; a.dL = nullptr;
  a.gV = reinterpret_cast<__nv_bfloat16*>(gVL); a.dm = dm; a.sGj = sGj; a.ldg = ldg;
  return cuda_status(launch_combine_bwd(a, S(stream)), "combine_bwd_packed");
}

int dchag_unfold(const void* img, long long img_sb, long long img_sc, int B, int C, int Himg,
                 int W, int P, void* out, void* stream) {
  if (Himg % P || W % P) return fail(DCHAG_ERR_SHAPE, "unfold: image not divisible by patch");
  return cuda_status(launch_unfold(reinterpret_cast<const __nv_bfloat16*>(img), img_sb, img_sc,
                                   B, C, Himg, W, P, reinterpret_cast<__nv_bfloat16*>(out),
                                   S(stream)),
                     "unfold");
}

int dchag_tile_weights(const float* src, int nblk, int K, int N, void* dst, void* stream) {
  if (K % 8 || N % 8 || N <= 0) return fail(DCHAG_ERR_SHAPE, "tile_weights: K, N must be multiples of 8");
  const long long total = (long long)nblk * K * N;
  if (total == 0) return DCHAG_OK;
  tile_weights_kernel<<<(unsigned)((total + 255) / 256), 256, 0, S(stream)>>>(
      src, nblk, K, N, reinterpret_cast<__nv_bfloat16*>(dst));
  return cuda_status(cudaGetLastError(), "tile_weights");
}

}  // extern "C"
