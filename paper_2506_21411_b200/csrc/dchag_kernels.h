// Internal (C++) launch interface shared by the kernel translation units and
// the C-ABI layer (capi.cu).  Not part of the public ABI: see include/dchag.h.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dchag {

// n / d for 0 <= n < 2^31 by a multiply-high with a host-computed magic number
// (Granlund-Montgomery: m = ceil(2^(31+l) / d), l = ceil(log2 d)): two instructions instead
// of a ~30-instruction integer division in the per-tile index math of the GEMM kernels
struct FastDiv {
  unsigned int m, s, d;
#ifdef __CUDACC__
  __host__ __device__ __forceinline__ int div(int n) const {
    return (int)(((unsigned long long)(unsigned int)n * m) >> s);
  }
#endif
};
inline FastDiv make_fastdiv(unsigned int d) {
  unsigned int l = 0;
  while ((1ull << l) < d) ++l;
  const unsigned long long num = 1ull << (31 + l);
  FastDiv f;
  f.m = (unsigned int)((num + d - 1) / d);
  f.s = 31 + l;
  f.d = d;
  return f;
}

struct GemmArgs {
  int G, M, Mi, N, Nv, K, BN;   // M = Mo * Mi rows per group
  int debug;                    // timing probes (DCHAG_GEMM_DEBUG)
  int pair;                     // 1: CTA-pair kernel (W TMA box built with BN/2 rows)
  int v_tma;                    // 1: bf16 value columns leave through TMA stores (tensor map
                                //    over outV, box 32 columns x 32 rows, 64B swizzle)
  const float* bias;            // [G][bias_g] fp32 or null
  long long bias_g;
  const __nv_bfloat16* rowbias; // [G][rowbias_g] with row (mi % period) * rowbias_row, or null
  long long rowbias_g, rowbias_row;
  int rowbias_period;
  void* outV;                   // columns [0, Nv): bf16 (or fp32 if outV_f32)
  int outV_f32;
  long long sVg, sVmo, sVmi;
  float* outL;                  // columns [Nv, N): fp32
  long long sLg, sLmo, sLmi;
  // row-dot mode (dotOut != null): nothing is stored; each 32-column group's
  // sum_n (acc + bias)[m][n] * dotG[m][n] goes to dotOut[(g * N/32 + n/32) * M + m]
  const __nv_bfloat16* dotG;    // [M][ldG] bf16, shared by all groups
  long long ldG;
  float* dotOut;
  // combine mode (the COMB kernel instance): G counts parents; output group j is the
  // softmax-weighted sum over its children g = cfirst[j] .. +ccount[j]-1 (the A / W / bias
  // groups) of the child tiles, weights softmax_c(Lpre[g][m][n / dh]) (layers.py:114-122)
  const int* cfirst;
  const int* ccount;
  const float* Lpre;            // [children][M][H] fp32 logits
  int H, dh;
  int nparents;                 // COMB: G = nparents * csplit; group g = split s * nparents + j
  int csplit;                   // 1, or 2: split s sums children [s c/2, (s+1) c/2) (partials)
  int lay;                      // operand layouts: bit 0 A MN-major, bit 1 W MN-major
  FastDiv fd_G, fd_cpg, fd_ctn, fd_Mi;  // set by launch_gemm: G, tiles per group, N tiles, Mi
  int dot64;                    // row-dot: one sum per 64 columns (dot_out [G][N/64][M])
  int lean;                     // 1: lean bf16 epilogue (tV box 64 columns x 32 rows, 128B
                                //    swizzle; see gemm_kernel)
  int Ki;                       // MN-major A: K = Ko * Ki rows, (k / Ki) * sAko + (k % Ki) * lda
  int accum;                    // fp32 output: out += acc instead of out = acc
  const float* rmask;           // optional [M] row mask m: v = v (1 - m) + mtok[n] m (epilogue)
  const float* mtok;            // [N] mask token
};

// host read (and optional reset) of the COMB overflow flag (synchronous)
cudaError_t comb_overflow_flag(int* value, int reset);

cudaError_t launch_gemm(const CUtensorMap& tA, const CUtensorMap& tW, const CUtensorMap& tV,
                        const GemmArgs& a, int bk, int num_sms, cudaStream_t st);

// Level-0 node: logits + softmax over the node's channels (tensor cores via mma.sync)
struct L0LogitArgs {
  const __nv_bfloat16* img;  // [B][*][H][W]; channel c of the slab at img + c*img_sc
  long long img_sb, img_sc;
  int B, S, W, P, wp, H, HP;  // H heads, HP = H padded to a multiple of 8
  int n_nodes, gmax;          // gmax >= every node_g (host-known)
  int nh;                     // heads per K_l0 unit: 2 if dh == 128, else 4 if H % 4 == 0, else 2
  const int* node_c0;         // first slab channel of node n
  const int* node_g;          // channel count of node n
  const long long* node_poff; // element offset of node n in p
  const __nv_bfloat16* WUt;   // [C][HP][PP]  logit weights tok.w[c] @ U_n, transposed
  const float* bU;            // [C][HP]      (tok.b[c]+chan_id[c]) @ U_n
  const float* posU;          // [n_nodes][S][HP]
  float* pinv;                // optional [n_nodes][R][H]: with it p holds the unnormalised
                              // e = exp(l - max) and pinv = 1 / sum_c e (K_l0 scales ctx)
  __nv_bfloat16* p;           // p[poff[n] + ((hg*g + c)*R + r)*NH + h%NH], hg = h/NH,
                              // NH = 4 if H % 4 == 0 else 2 (head group of one K_l0 CTA);
                              // a 128-row tile's slice of (hg, c) is one contiguous 1 KB run
  long long* trace;           // timing probe (DCHAG_P0_TRACE_PTR): CTAs 0..3, 64 items
  int issue_serial;           // A/B probe (DCHAG_P0_ISSUE=1): one thread issues every copy
};
cudaError_t launch_l0_logits(const L0LogitArgs& a, int num_sms, cudaStream_t st);

// Level-0 node: ctx[n][r][h*dh:(h+1)*dh] = sum_c p[r,c,h] * (patch_c[r] @ M_c[:,h]) + ext
struct L0NodeArgs {
  const __nv_bfloat16* img;
  long long img_sb, img_sc;
  int B, S, W, P, wp, H, D;
  int nh;                      // heads per unit (NH * dh <= 256), matches L0LogitArgs::nh
  int n_nodes;
  const int* node_c0;
  const int* node_g;
  const long long* node_poff;
  int p_row_mode;              // 1: K_p0 layout (see L0LogitArgs); 0: constant p[poff + c*H + h]
  const __nv_bfloat16* p;
  const float* pinv;           // optional [n_nodes][R][H] row/head scale of ctx (K_p0 output)
  const __nv_bfloat16* Mt;     // [H][2][C_pad*PP/8][dh/16][8][8]: per head, the two dh/2-column
                               // halves of M_c (one per CTA of a pair) as canonical no-swizzle
                               // K-major core-matrix blocks, channels consecutive along K
  int C_pad;
  const __nv_bfloat16* Et;     // [n_nodes][H][2][KE/8][dh/16][8][8] ext (bias) blocks, same split
  int KE;
  __nv_bfloat16* ctx;          // [n_nodes][R][D]
  int has_pos;                 // 1: ctx += posV[n][s] (tensor map tm_pos over [n_nodes*S][D])
  int debug_mode;              // timing probes: 1 no A build, 2 no MMA, 4 no copies,
                               // 8 no ctx stores, 32 no drain
  long long* trace;            // optional [8][256] clock64 timeline of CTA 0 (debug)
};
cudaError_t launch_l0_node(const L0NodeArgs& a, const CUtensorMap& tm_ctx,
                           const CUtensorMap& tm_pos, int num_sms, cudaStream_t st);

// Upper-level combine: ctx[n][r][:] = sum_j p_jh(r) * V_child(j)[r][:]
struct CombineArgs {
  int n_nodes, R, D, H, max_g;
  const int* node_first;       // first child index of node n
  const int* node_g;           // child count
  const __nv_bfloat16* V;      // child j at V + j*sVj + r*D
  long long sVj;
  const float* L;              // child j logits at L + j*sLj + r*H (attention mode)
  long long sLj;
  const float* mix;            // linear mode: p_j = mix[node_first[n] + j] (L ignored)
  int rows_inner;              // row r = rb * rows_inner + rs; child row offset
  long long sVb, sLb;          //   = j*sVj + rb*sVb + rs*D   (L: j*sLj + rb*sLb + rs*H)
  __nv_bfloat16* ctx;          // [n][R][D]
  long long ldv;               // elements between a child's V rows (0: D)
  const float* W;              // explicit weights [n][R][max_g][H] (full_cross), or null
};
cudaError_t launch_combine(const CombineArgs& a, cudaStream_t st);

// fp32 combine (fp32 parity mode): V, L, ctx fp32; rows contiguous (child j row r at j*sVj + r*D)
struct CombineF32Args {
  int n_nodes, R, D, H, max_g;
  const int* node_first;
  const int* node_g;
  const float* V;
  long long sVj;
  const float* L;
  long long sLj;
  const float* mix;
  float* ctx;
};
cudaError_t launch_combine_f32(const CombineF32Args& a, cudaStream_t st);

// Level-0 backward: T_c = patch_c^T (p_c * G) without dV in memory (comb.cu, l0_tgrad_kernel)
struct L0TgradArgs {
  const __nv_bfloat16* patches;  // [B][cnt][S][PP] bf16 (unfold_patches layout)
  int cnt, c0;                   // slab channels in `patches`, first channel of the node
  int g, R, S, D, H, NH, PP;
  const __nv_bfloat16* p;        // node block of the normalised K_p0 output [H/NH][g][R][NH]
  const float* mix;              // linear nodes: mix[g] (then p is unused)
  const __nv_bfloat16* G;        // [R][D] bf16
  float* T;                      // [g][PP][D] fp32
  // TE mode (dchag_l0_tgrad_te): the augmented products, one bf16 block per node
  //   TE[c*PP + k][d]      = T_c[k][d]                 (d < D)
  //   TE[c*PP + k][D + h]  = E_c[k][h] = sum_r patch_c[r][k] dl_c[r][h]
  //   TE[ones0 + c][d]     = sum_r p_c[r][h(d)] G[r][d]   (the bias row: colsum of dV_c)
  //   TE[ones0 + c][D + h] = sum_r dl_c[r][h]
  __nv_bfloat16* TE;
  long long te_ld;               // row stride of TE (elements)
  int ones0;                     // first bias row
  int has_dl;                    // dl given (attention nodes): one extra CTA column for E
  int debug;                     // timing probes (DCHAG_TE_DEBUG): 1 no scaling, 2 no MMA
};
cudaError_t launch_l0_tgrad(const L0TgradArgs& a, cudaStream_t st);
cudaError_t launch_l0_softmax_bwd(int g, int R, int H, int NH, int dh, const float* dpp,
                                  const float* Gpos, const __nv_bfloat16* p, float* dl,
                                  __nv_bfloat16* dlb, cudaStream_t st);
cudaError_t launch_child_softmax(float* L, const int* first, const int* count, int n_parents,
                                 int R, int H, cudaStream_t st);
cudaError_t launch_l0_tgrad_tc(const CUtensorMap& tG, const CUtensorMap& tP,
                               const L0TgradArgs& a, cudaStream_t st);
cudaError_t launch_l0_tgrad_te(const CUtensorMap& tG, const CUtensorMap& tP,
                               const CUtensorMap& tDL, const L0TgradArgs& a, cudaStream_t st);
cudaError_t launch_vit_meta(const float* meta, int kmeta, const float* meta_w,
                            const float* meta_b, void* out, int f32, int B, int S, int D,
                            cudaStream_t st);
cudaError_t launch_vit_tokens(const void* agg, int f32, const float* mask,
                              const float* mask_token, const float* meta_tok, void* out, int B,
                              int S, int D, cudaStream_t st);
cudaError_t launch_l0_dv(int g, int R, int D, int H, int NH, const __nv_bfloat16* p,
                         const float* mix, const __nv_bfloat16* G, const float* posV,
                         long long ldpos, int S, float* Gpos, __nv_bfloat16* out,
                         cudaStream_t st);

// full_cross node weights (layers.py:125-138 folded): per (node, row), heads h:
//   S^h = softmax_j(q_i,h . k_j,h / sqrt(dh)),  s_i = sum_h sum_j S^h_ij u_jh,
//   p2 = softmax_i(s),  w_jh = sum_i p2_i S^h_ij        (ctx_h = sum_j w_jh V_j,h)
struct FullCrossArgs {
  int n_nodes, R, D, H, max_g;
  const int* node_first;
  const int* node_g;
  const __nv_bfloat16* QK;     // child j row r: q at QK + j*sQj + r*ldq, k at + D
  long long sQj, ldq;
  const float* u;              // child j row r: u at u + j*sUj + r*H  (V_j,h . (wo rq)_h / sqrt D)
  long long sUj;
  float* w;                    // [n][R][max_g][H]
  // optional positional query (level 0 with the tokenizer folded): q_i += posq[n][r % S]
  // while staging (the key/value/u positional terms cancel in the softmaxes)
  const __nv_bfloat16* posq;   // [n][S][D] bf16 or null
  int S;
  // optional: w written as K_l0's bf16 p operand (dchag_l0_logits layout, normalised) instead
  // of the fp32 table: pout[poff[n] + ((h/nh * g + j) * R + r) * nh + h % nh]
  __nv_bfloat16* pout;
  const long long* node_poff;
  int nh;
};
cudaError_t launch_fullcross_weights(const FullCrossArgs& a, cudaStream_t st);

// Backward of a full_cross node per (node, row) given G = dLoss/dctx (see comb.cu).
struct FullCrossBwdArgs {
  int n_nodes, R, D, H, max_g;
  const int* node_first;
  const int* node_g;
  const __nv_bfloat16* QKV;    // child j row r: q | k | v at QKV + j*sQj + r*ldq
  long long sQj, ldq;
  const float* u;              // [child][R][H] (forward's u)
  const float* G;              // [n][R][D] fp32
  const float* a;              // [n][D] fp32: (wo rq) / sqrt(D) of the node
  __nv_bfloat16* dQKV;         // child j row r: dq | dk | dv at dQKV + j*sQj + r*ldq
  float* dA;                   // [n][R][D] fp32: sum_j du_jh v_j,h (per head block)
};
cudaError_t launch_fullcross_bwd(const FullCrossBwdArgs& a, cudaStream_t st);

// Backward of the combine: dL, gV (and dmix for linear nodes) from g = dLoss/dctx
struct CombineBwdArgs {
  int n_nodes, R, D, H, max_g;
  const int* node_first;
  const int* node_g;
  const __nv_bfloat16* V;      // child j at V + j*sVj + r*D (same strides for gV)
  long long sVj;
  const float* L;              // child logits, j*sLj + r*H (same strides for dL)
  long long sLj;
  const float* mix;            // linear mode
  const float* G;              // [n][R][D] fp32 upstream gradient of ctx
  float* dL;                   // attention: [child][R][H]
  __nv_bfloat16* gV;           // [child][R][D]
  float* dm;                   // linear: [child][R] row dots g . V_j
  // packed mode (the training step): gV child j row r at gV + j*sGj + r*ldg, and dL as bf16
  // in the same row at column D + h (the K-concatenated operand [gV | dL] of the backward
  // GEMMs); sGj = 0 keeps the V strides
  long long sGj, ldg;
};
cudaError_t launch_combine_bwd(const CombineBwdArgs& a, cudaStream_t st);

// images [B][C][H][W] -> patches [B][C][S][P*P] (bf16)
cudaError_t launch_unfold(const __nv_bfloat16* img, long long img_sb, long long img_sc, int B,
                          int C, int Himg, int W, int P, __nv_bfloat16* out, cudaStream_t st);

// ---- training-step support kernels (train.cu)
struct CastJob {                 // dst (bf16) <- src (fp32): rows x cols of src
  const float* src;
  __nv_bfloat16* dst;
  long long rows, cols, lds, ldd;
  long long trans;               // 1: dst[c * ldd + r] = src[r * lds + c]
  long long dst_f32;             // 1: dst is fp32 (a plain strided copy, e.g. stacked biases)
};
cudaError_t launch_cast_multi(const CastJob* jobs, int n_jobs, int max_tiles, cudaStream_t st);

struct QueryFoldJob {            // one single_query node: U = fold(wq, wk, q) and its backward
  const float* wq;
  const float* wk;
  const float* q;
  float* U;                      // [D][ldU] (forward output)
  long long ldU;
  float* qp;                     // [D] q wq (written by the forward, read by the backward)
  const float* dU;               // [D][ldU] (backward input)
  float* dwk;                    // [D][D] (backward outputs)
  float* dwq;
  float* dq;                     // [D]
};
cudaError_t launch_query_fold(const QueryFoldJob* jobs, int n_jobs, int D, int H, float* part,
                              cudaStream_t st);
cudaError_t launch_query_fold_bwd(const QueryFoldJob* jobs, int n_jobs, int D, int H,
                                  float* part, float* dqp, cudaStream_t st);
cudaError_t launch_colsum(const void* X, int x_f32, long long ldx, long long sxg, int G, int R,
                          int N, int P, void* out, long long sog, long long ldo, int out_bf16,
                          int accumulate, const float* gscale, float* part, cudaStream_t st);
cudaError_t launch_rowsum(const float* X, long long ldx, int rows, int N, float* out,
                          cudaStream_t st);

struct L0PackArgs {             // level-0 refold scatter (train.cu pack kernels)
  const float* MT;              // [n0][Dp][Kn]
  int n0, C, C_pad, D, H, HP, PP, gmax, KE, S;
  int ones0;                    // first tb row of a node block (MT column)
  long long Dp, Kn;
  const int* chan_node;         // [C] node of slab channel c
  const int* chan_local;        // [C] channel index inside its node
  const int* node_g;            // [n0]
  __nv_bfloat16* Mt;            // K_l0 tiled value weights
  __nv_bfloat16* Et;            // K_l0 tiled bias blocks
  __nv_bfloat16* Mrow;          // [C][D][PP] (row-dot GEMM operand)
  float* Cb;                    // [C][D]
  __nv_bfloat16* WUt;           // attention: [C][HP][PP]
  float* bU;                    //            [C][HP]
  const float* posVU;           // optional [n0][S][Dp] = pos [Wv | U]
  const float* mixsum;          // linear nodes: [n0] sum of mix (posV scale), else null
  __nv_bfloat16* posV0;         // [n0][S][D]
  float* posU;                  // attention: [n0][S][HP]
};
cudaError_t launch_l0_pack(const L0PackArgs& a, cudaStream_t st);
cudaError_t launch_split3(const float* x, long long rows, int K, long long ldx,
                          __nv_bfloat16* out, long long ldo, cudaStream_t st);
cudaError_t launch_l0_p_normalize(const __nv_bfloat16* e, const float* pinv, __nv_bfloat16* p,
                                  const long long* node_poff, const int* node_g, int n_nodes,
                                  int gmax, int R, int H, int NH, cudaStream_t st);

}  // namespace dchag
