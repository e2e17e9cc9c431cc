/* D-CHAG channel front end on B200 (sm_100a) -- C ABI of libdchag.so.
 *
 * The reference (/root/reference/pkg/src/dchag) is pure Python/numpy and has no
 * FFI; its drop-in boundary for this path is the functional API
 *   tokenize_channels (model.py:51-64), tree_aggregate (model.py:76-97),
 *   flat_aggregate (model.py:67-73), cross_attention_aggregate (layers.py:94-138),
 *   linear_mix_aggregate (layers.py:141-146), and the AllGather of gather_shards
 *   (strategies.py:83-96).
 * The Python host (paper_2506_21411_b200/ops.py) keeps those names and signatures and
 * lowers them onto the entry points below; INTEGRATION.md shows the ctypes binding.
 *
 * Conventions: every pointer is a device pointer unless noted; bf16 tensors are
 * uint16 storage; strides/offsets are in ELEMENTS; every launch is stream-ordered on
 * `stream` (a cudaStream_t, may be NULL = legacy default stream) and performs no
 * host synchronisation and no device allocation.  Return 0 on success, else a
 * DCHAG_ERR_* code; dchag_last_error() gives the message (thread-local).
 */
#ifndef DCHAG_H_
#define DCHAG_H_

#ifdef __cplusplus
extern "C" {
#endif

#define DCHAG_OK 0
#define DCHAG_ERR_SHAPE 1  /* maps to ShapeError / ConfigError in the host layer */
#define DCHAG_ERR_CONFIG 2
#define DCHAG_ERR_CUDA 3

const char* dchag_version(void);
const char* dchag_last_error(void);

/* Grouped projection GEMM (K_gemm), replaces the per-node `matmul(ctx, wo) + bo`
 * chain of layers.py:103-123 / :141-146 (folded with the consumer's wv/U):
 *   out[g][m][n] = sum_k A[g][m][k] * W[g][n][k] + bias[g][n] + rowbias[g][(mi % period)][n]
 * rows m = mo*Mi + mi (Mi % 128 == 0); A is bf16 with strides (sAg, sAmo, sAmi=row);
 * W is bf16 [G][N][K] contiguous rows; columns n < Nv go to outV (bf16, or fp32 if
 * outV_f32) at g*sVg + mo*sVmo + mi*sVmi + n; columns Nv <= n < N go to outL (fp32). */
int dchag_gemm_bf16(const void* A, int G, int Mo, int Mi, int K, long long sAg, long long sAmo,
                    long long sAmi, const void* W, int N, long long sWg, int Nv,
                    const float* bias, long long bias_g, const void* rowbias,
                    long long rowbias_g, long long rowbias_row, int rowbias_period, void* outV,
                    int outV_f32, long long sVg, long long sVmo, long long sVmi, float* outL,
                    long long sLg, long long sLmo, long long sLmi, void* stream);

/* General tcgen05 GEMM with explicit operand layouts (training backward and weight
 * folding: the reference's matmul backward, tensor.py:168-188 differentiated by
 * tensor.py:395-413, i.e. dW = X^T G and dX = G W^T without transposed copies):
 *   out[g][m][n] (+)= sum_k A_g(m, k) * B_g(n, k) + bias[g][n]
 * A: a_mn = 0 K-major, (m, k) at g*sAg + m*lda + k;
 *    a_mn = 1 MN-major, (m, k) at g*sAg + (k / Ki)*sAko + (k % Ki)*lda + m   (Ki % 64 == 0)
 * B: b_mn = 0 K-major, (n, k) at g*sBg + n*ldb + k;  b_mn = 1 MN-major, (n, k) at g*sBg + k*ldb + n
 * out: fp32 (out_f32 = 1; accumulate = 1 adds the product to the existing values) or bf16,
 * (m, n) at g*sCg + m*ldc + n. bias (fp32, optional) at g*bias_g + n.
 * M % 128 == 0 (M % 256 == 0 with an MN-major operand), N % 16 == 0, K % 64 == 0;
 * operands 16-byte aligned. Deterministic (fixed accumulation order, no split-K). */
int dchag_gemm_nt(const void* A, int a_mn, long long lda, long long sAko, int Ki,
                  long long sAg, const void* B, int b_mn, long long ldb, long long sBg, int G,
                  int M, int N, int K, const float* bias, long long bias_g, void* out,
                  int out_f32, int accumulate, long long ldc, long long sCg, void* stream);

/* The shared final layer's projection fused with the trunk's input assembly (
 * model.py:100-108 apply_token_mask, :111-117 metadata token + concat):
 *   out[b][1 + s][n] = (ctx[b*S + s] . W[n] + bias[n]) (1 - mask[b][s]) + mask_token[n] mask[b][s]
 *   out[b][0][n]     = sum_k meta[b][k] meta_w[k][n] + meta_b[n]
 * ctx bf16 [B*S][K], W bf16 [D][K] (n-major, as dchag_gemm_bf16), bias / mask / mask_token /
 * meta fp32; out [B][S+1][D] bf16 (or fp32 if out_f32). The mask is applied in the GEMM
 * epilogue and the rows land at their trunk positions: the aggregate is never written twice. */
int dchag_final_vit(const void* ctx, int B, int seq, int K, const void* W, int D,
                    const float* bias, const float* mask, const float* mask_token,
                    const float* meta, int kmeta, const float* meta_w, const float* meta_b,
                    void* out, int out_f32, void* stream);

/* Row-dot GEMM for the level-0 backward (the `dp = G . V` term of the softmax backward,
 * layers.py:103-121 differentiated by tensor.py:395-413): the product rows
 * V[g][m][:] = A[g][m][:] W[g]^T + bias[g] are never stored; for every 32-column group
 * dot_out[(g*N/32 + n/32)*M + m] = sum_{n in group} V[g][m][n] * Gmat[m][n] (fp32),
 * M = Mo*Mi, Gmat bf16 [M][ldG] shared by all g. A, W, strides as dchag_gemm_bf16;
 * N % 32 == 0. */
int dchag_gemm_rowdot(const void* A, int G, int Mo, int Mi, int K, long long sAg,
                      long long sAmo, long long sAmi, const void* W, int N, long long sWg,
                      const float* bias, long long bias_g, const void* Gmat, long long ldG,
                      float* dot_out, void* stream);

/* As dchag_gemm_rowdot with `group` (32 or 64) columns per dot: group = 64 gives one sum per
 * 64-column block, dot_out [G][N/64][M] (a head of 64 columns: the per-head dp partial the
 * softmax backward reads with dh = 32, i.e. one partial per head). 64-column groups need the
 * lean row-dot drain (CTA pairs, N % 64 == 0). */
int dchag_gemm_rowdot_heads(const void* A, int G, int Mo, int Mi, int K, long long sAg,
                            long long sAmo, long long sAmi, const void* W, int N, long long sWg,
                            const float* bias, long long bias_g, const void* Gmat, long long ldG,
                            int group, float* dot_out, void* stream);

/* Tree level >= 1 fused (K_gemm COMB instance): each child's folded value projection
 * V_c = ctx_c W_c^T + bias_c (layers.py:123 output projection folded with the parent's
 * value projection) and the parent's softmax-weighted child sum (layers.py:114-122) in one
 * kernel; V never reaches memory. ctx bf16 [n_children][R][D]; W bf16 rows [D][D] per child
 * at stride sWg elements (the value rows of the folded [N][D] weights); bias fp32 at
 * stride bias_g; Lpre fp32 [n_children][R][H] = the children's softmax weights (a
 * dchag_gemm_bf16 over the logit rows, then dchag_child_softmax); parent j owns children first[j] ..
 * first[j]+count[j]-1 (device int32). out bf16 [csplit][n_parents][R][D]: with csplit 2
 * (every parent with >= 2 children) split s holds the sum over children
 * [s c/2, (s+1) c/2) with the full softmax, and out[0] + out[1] is the result (more, smaller
 * work units when parents are few). R % 256 == 0, D % 256 == 0, (D/H) % 32 == 0. The
 * running sum is kept as fp16 pairs scaled by 2^-8 (fp32 math): partial child sums up to
 * +-1.68e7 in magnitude; beyond that the kernel raises a device flag that
 * dchag_combine_overflow reports. */
int dchag_gemm_combine(const void* ctx, int n_children, int R, int D, int H, const void* W,
                       long long sWg, const float* bias, long long bias_g, const float* Lpre,
                       const int* first, const int* count, int n_parents, int csplit,
                       void* out, void* stream);

/* Level-0 backward in the augmented form the training step uses (dchag_l0_tgrad plus the
 * bias and logit-weight terms): with x_c = [patch_c | 1] [tok.w[c]; tok.b[c] + chan_id[c]]
 * (model.py:51-64), one launch per node writes the bf16 block TE (row stride te_ld):
 *   TE[c*PP + k][d]      = sum_r patch_c[r][k] p_c[r][h(d)] G[r][d]     (d < D)
 *   TE[ones0 + c][d]     = sum_r p_c[r][h(d)] G[r][d]
 *   TE[c*PP + k][D + h]  = sum_r patch_c[r][k] dl_c[r][h]               (dlb given, h < H)
 *   TE[ones0 + c][D + h] = sum_r dl_c[r][h]
 * c = node-local channel; dlb = the node's bf16 [g][H][R] softmax-logit gradient
 * (dchag_l0_softmax_bwd) or NULL (linear nodes). The ones column is a constant shared-memory
 * operand atom (MMA N = 80). Other arguments as dchag_l0_tgrad; H <= 128. */
int dchag_l0_tgrad_te(const void* patches, int cnt, int c0, int g, int R, int seq, int D,
                      int H, int nh, int PP, const void* p, const float* mix, const void* G,
                      const void* dlb, void* TE, long long te_ld, int ones0, void* stream);

/* ---- training-step support (train.cu). Device tables are arrays of 8-byte fields. */

/* fp32 -> bf16 of many tensors in one launch: jobs[i] = {src, dst, rows, cols, lds, ldd,
 * trans, dst_f32} (int64 each; trans = 1 writes dst[c*ldd + r]; dst_f32 = 1 copies into an
 * fp32 dst, trans must be 0); the per-step refresh of the bf16 operand copies of the fp32
 * master weights. max_tiles = max over jobs of 32x32 tiles. */
int dchag_cast_multi(const void* jobs, int n_jobs, int max_tiles, void* stream);

/* Query fold of single_query nodes (layers.py:103-120): qp = q @ wq,
 * U[d][h] = sum_{j in head h} wk[d][j] qp[j] / sqrt(D/H). jobs[i] = {wq, wk, q, U, ldU, qp,
 * dU, dwk, dwq, dq} (fp32 device pointers / int64); writes U and qp. work: fp32
 * [n_jobs][ceil(D/128)][D]. */
int dchag_query_fold(const void* jobs, int n_jobs, int D, int H, float* work, void* stream);

/* Backward of the query fold (tensor.py:395-413 through that chain): from dU (and the
 * forward's qp) writes dwk, dwq [D][D] and dq [D]. work as dchag_query_fold, dqp fp32
 * [n_jobs][D]. */
int dchag_query_fold_bwd(const void* jobs, int n_jobs, int D, int H, float* work, float* dqp,
                         void* stream);

/* Periodic column sums: out[g][p][n] (+)= scale[g] * sum_{r = p, p+P, ... < R} X[g][r][n]
 * (X fp32 if x_f32 else bf16, row stride ldx, group stride sxg; out fp32, or bf16 if
 * out_bf16 (no accumulate), group stride sog, row stride ldo (0: N); gscale optional fp32
 * [G]). Bias gradients (P = 1) and sums over the batch of [B*S] rows (P = S).
 * Deterministic. work: fp32 [G][ceil(R/64)][N] when P == 1. */
int dchag_colsum(const void* X, int x_f32, long long ldx, long long sxg, int G, int R, int N,
                 int P, void* out, long long sog, long long ldo, int out_bf16, int accumulate,
                 const float* gscale, float* work, void* stream);

/* out[i] = sum_j X[i*ldx + j], j < N (fp32). */
int dchag_rowsum(const float* X, long long ldx, int rows, int N, float* out, void* stream);

/* Level-0 refold scatter (the training step refolds level 0 every step, fold.py's algebra):
 * MT fp32 [n0][Dp][Kn] is the grouped GEMM product [Wv_n | U_n]^T x [tok.w rows ; tok.b +
 * chan_id rows]^T of every level-0 node n (MT[n][d][l*PP + k] = (tok.w[c] Wv_n)[k][d] for
 * node-local channel l of slab channel c, MT[n][d][ones0 + l] = ((tok.b + chan_id)[c] Wv_n)[d] (ones0 >= gmax*PP),
 * rows D + h the logit weights). Writes the K_l0 operands Mt / Et (dchag_l0_node layouts),
 * Mrow bf16 [C][D][PP] and Cb fp32 [C][D] (row-dot GEMM operand and bias), and for attention
 * nodes WUt / bU (dchag_l0_logits layouts). With posVU (fp32 [n0][S][Dp] = pos [Wv_n | U_n])
 * also posV0 bf16 [n0][S][D] (scaled by mixsum[n] for linear nodes) and posU fp32
 * [n0][S][HP]. chan_node / chan_local / node_g: int32 device tables. */
int dchag_l0_pack(const float* MT, int n0, int C, int C_pad, int D, int H, int HP, int PP,
                  int gmax, int ones0, int KE, int S, long long Dp, long long Kn,
                  const int* chan_node,
                  const int* chan_local, const int* node_g, void* Mt, void* Et, void* Mrow,
                  float* Cb, void* WUt, float* bU, const float* posVU, const float* mixsum,
                  void* posV0, float* posU, void* stream);

/* Range guard of dchag_gemm_combine: *flag = 1 if any launch since the last reset saw a
 * partial child sum beyond +-1.68e7 (its fp16 x 2^8 running-sum range), else 0; reset != 0
 * clears it. Host-synchronous (reads a device symbol); not a kernel launch. */
int dchag_combine_overflow(int* flag, int reset);

/* Level-0 logits + softmax over each node's channels (K_p0): replaces the
 * q@wq / x@wk / logits / softmax part of layers.py:103-121 for tree level 0 with the
 * tokenizer (model.py:51-64) folded in.  img: bf16 [B][*][Himg][W] with batch stride
 * img_sb and channel stride img_sc (slab channel c at img + c*img_sc).
 * node_c0/node_g (int32) and node_poff (int64) are device arrays of n_nodes; gmax >= all node_g.
 * WUt bf16 [C][HP][P*P], bU fp32 [C][HP], posU fp32 [n_nodes][S][HP]; HP = H rounded up
 * to a multiple of 8.  Output p bf16, head-group then channel major (a 128-row tile's
 * slice for one (head group, channel) is contiguous, so K_l0 stages it with one bulk copy):
 * p[poff[n] + ((hg*g + c)*R + r)*NH + h%NH], hg = h/NH, NH = nh = dchag_l0_node's heads per
 * unit: 2 if the head dim is 128, else 4 if H%4==0, else 2.
 * pinv (optional, fp32 [n_nodes][R][H]): when given, p holds the unnormalised
 * e = exp(logit - max_c logit) and pinv = 1 / sum_c e; dchag_l0_node then applies pinv to
 * its accumulator (one exp per logit instead of three).  NULL: p is the normalised softmax. */
int dchag_l0_logits(const void* img, long long img_sb, long long img_sc, int B, int Himg, int W,
                    int P, int H, int HP, int nh, int n_nodes, int gmax, const int* node_c0,
                    const int* node_g,
                    const long long* node_poff, const void* WUt, const float* bU,
                    const float* posU, void* p, float* pinv, void* stream);

/* fp32 parity mode operand split: x fp32 [rows][K] (row stride ldx) -> out bf16 [rows][3K]
 * (row stride ldo) = [hi | lo | hi], hi = bf16(x), lo = bf16(x - hi); with the weights as
 * [hi | hi | lo] one bf16 GEMM over 3K gives x W to ~2^-16 relative. K % 4 == 0, x 16-byte
 * and out 8-byte aligned. */
int dchag_split3_bf16(const float* x, long long rows, int K, long long ldx, void* out,
                      long long ldo, void* stream);

/* The normalised level-0 softmax from dchag_l0_logits' pinv form (training backward):
 * p[i] = e[i] * pinv[(n*R + r)*H + h] over each node's block (layout as dchag_l0_logits'
 * p: poff[n] + ((hg*g + c)*R + r)*nh + h%nh). node_poff (int64) / node_g (int32) are device
 * arrays of n_nodes; gmax >= all node_g. (R*H) % 8 == 0; e and p 16-byte aligned. */
int dchag_l0_p_normalize(const void* e, const float* pinv, void* p, const long long* node_poff,
                         const int* node_g, int n_nodes, int gmax, int R, int H, int nh,
                         void* stream);

/* Level-0 node context (K_l0, tcgen05 with A in TMEM):
 *   ctx[n][r][h*64:(h+1)*64] = sum_c p[r,c,h] * (patch_c[r] @ M_c[:, h-block])
 *                             + sum_c p[r,c,h] * E_n[c, h-block]
 * Mt bf16 [H][2][32*C_pad*P*P] and Et bf16 [n_nodes][H][2][32*KE] are pre-tiled canonical
 * UMMA blocks (dchag_tile_weights, N = 32 halves; K runs over channel-major c*P*P + k); p_row_mode = 1 reads the dchag_l0_logits layout, 0 a constant
 * table p[poff + c*H + h]
 * (linear-mix nodes).  Requires head dim 64 or 128, S % 128 == 0, 128 % (W/P) == 0,
 * P in {4, 8}.  pinv (optional, the dchag_l0_logits output): ctx row r, head h is scaled by
 * pinv[n][r][h].  posV (optional, bf16 [n_nodes][S][D]): the node's positional term
 * pos[s] @ wv_n (x sum(mix) for linear nodes), added to ctx row r = (b, s). */
int dchag_l0_node(const void* img, long long img_sb, long long img_sc, int B, int Himg, int W,
                  int P, int H, int D, int n_nodes, const int* node_c0, const int* node_g,
                  const long long* node_poff, int p_row_mode, const void* p, const float* pinv,
                  const void* Mt, int C_pad, const void* Et, int KE, const void* posV, void* ctx,
                  void* stream);

/* Level-0 node backward, value gradient (training): dV[c][r][d] = p_c[r][h] * G[r][d]
 * for the node's g channels, p = the node's block of the normalised dchag_l0_logits output
 * ([H/nh][g][R][nh] bf16), or dV[c] = mix[c] * G for linear nodes (mix != NULL). With posV
 * (fp32 [S][D], row r uses r % S) also Gpos[r][h] = sum_{d in head h} G[r][d] posV[r % S][d]
 * (fp32 [R][H]), the positional part of dp = G . V; posV rows ldpos apart (0: D). G, dV bf16 [R][D] / [g][R][D], 16-byte
 * aligned; D/H a power of two in 8..256. dV == NULL computes Gpos only. */
int dchag_l0_dv(int g, int R, int D, int H, int nh, const void* p, const float* mix,
                const void* G, const float* posV, long long ldpos, int period, float* Gpos,
                void* dV, void* stream);

/* ViT input tokens after the front end (model.py:100-108 apply_token_mask, :111-117 meta
 * token + concat): out[b][0] = meta_tok[b], out[b][1+s] = agg[b][s] (1 - mask[b][s]) +
 * mask_token mask[b][s]. agg [B][S][D] and out [B][S+1][D] bf16 (or fp32 if agg_f32);
 * mask fp32 [B][S], mask_token fp32 [D], meta_tok fp32 [B][D] (= meta @ meta_w + meta_b).
 * D % 8 == 0. */
int dchag_vit_tokens(const void* agg, int agg_f32, int B, int seq, int D, const float* mask,
                     const float* mask_token, const float* meta_tok, void* out, void* stream);

/* Level-0 node backward, token-weight gradient (training; the patches^T . dtokens of
 * tensor.py:168-188 differentiated, with the node's dV = p . G folded in so dV is never
 * stored): T[c][k][d] = sum_r patch_c[r][k] p_c[r][h(d)] G[r][d] for the node's channels
 * c0 .. c0+g-1 of `patches` ([B][cnt][S][PP] bf16), p as dchag_l0_dv (or mix for linear
 * nodes), G bf16 [R][D], T fp32 [g][PP][D]. PP == 64, D % 128 == 0, S % 64 == 0,
 * D/H in {64, 128}, nh even. */
int dchag_l0_tgrad(const void* patches, int cnt, int c0, int g, int R, int seq, int D, int H,
                   int nh, int PP, const void* p, const float* mix, const void* G, float* T,
                   void* stream);

/* Softmax over each parent's children in place (layers.py:114-120 above level 0):
 * L fp32 [children][R][H] logits -> p, parent j's children first[j] .. first[j]+count[j]-1
 * (device int32). The weights dchag_gemm_combine applies. */
int dchag_child_softmax(float* L, const int* first, const int* count, int n_parents, int R,
                        int H, void* stream);

/* Level-0 node backward, channel softmax (training; layers.py:114-120 through
 * tensor.py:201-203): dp_c[r][h] = sum of dchag_gemm_rowdot's 32-column partials of head h
 * (dpp fp32 [g][H*dh/32][R]) + Gpos[r][h] (dchag_l0_dv), then
 * dl_c = p_c (dp_c - sum_c' p_c' dp_c'); p as dchag_l0_dv. dl fp32 and dlb bf16, both
 * [g][H][R]. dh % 32 == 0: dpp holds dh / 32 partials per head (pass dh = 32 for one partial
 * per head, dchag_gemm_rowdot_heads with group 64). dl may be NULL when g <= 16 and dh is 32
 * or 64 (only the bf16 copy is written). */
int dchag_l0_softmax_bwd(int g, int R, int H, int nh, int dh, const float* dpp,
                         const float* Gpos, const void* p, float* dl, void* dlb, void* stream);

/* fp32 parity mode combine: as dchag_combine with fp32 child values V (row r of child j at
 * V + j*sVj + r*D) and an fp32 context (precise expf, fp32 accumulation). */
int dchag_combine_f32(int n_nodes, int R, int D, int H, const int* node_first, const int* node_g,
                      int max_g, const float* V, long long sVj, const float* L, long long sLj,
                      const float* mix, float* ctx, void* stream);

/* full_cross node weights (layers.py:125-138 with sdp_attention layers.py:49-64): per node
 * and row, with q/k of child j at QK + j*sQj + r*ldq (k at +D, bf16) and u_jh = V_j,h .
 * (wo rq)_h / sqrt(D) at u + j*sUj + r*H (fp32):  S^h = softmax_j(q_i,h . k_j,h / sqrt(dh)),
 * s_i = sum_h sum_j S^h_ij u_jh,  p2 = softmax_i(s),  w[n][r][j][h] = sum_i p2_i S^h_ij.
 * The node output is then (sum_j w_jh V_j,h) @ wo + bo (dchag_combine_weighted + GEMM).
 * posq (optional, bf16 [n_nodes][seq][D]): added to every q of row r at position r % seq
 * (level 0 with the tokenizer folded: the positional parts of k, v and u cancel in the
 * softmaxes or are added to the context, so only the query's enters here).
 * pout (optional): the weights go out as dchag_l0_node's bf16 p operand instead of w
 * (pout[node_poff[n] + ((h/nh * g + j)*R + r)*nh + h%nh]): level 0 then sums the children's
 * values on the tensor cores from the patches (the single_query K_l0, p = w).
 * max_g <= 32, H <= 32, (D/H) % 16 == 0. */
int dchag_fullcross_weights(int n_nodes, int R, int D, int H, const int* node_first,
                            const int* node_g, int max_g, const void* QK, long long sQj,
                            long long ldq, const float* u, long long sUj, float* w,
                            const void* posq, int seq, void* pout, const long long* node_poff,
                            int nh, void* stream);

/* ctx[n][r][h-blk] = sum_j w[n][r][j][h] V_j[r][h-blk]; V_j row r at V + j*sVj + r*ldv (bf16). */
int dchag_combine_weighted(int n_nodes, int R, int D, int H, const int* node_first,
                           const int* node_g, int max_g, const void* V, long long sVj,
                           long long ldv, const float* w, void* ctx, void* stream);

/* Upper-level / final combine (K_comb): ctx[n][r][:] = sum_j w_j(r,h) V_{first+j}[r][:],
 * w = softmax_j(L_{first+j}[r][h]) (attention; mix == NULL) or mix[first+j] (linear).
 * Child j's V at V + j*sVj + r*D (bf16), logits at L + j*sLj + r*H (fp32).
 * max_g >= every node_g; requires max_g * H <= 1024 (attention). */
int dchag_combine(int n_nodes, int R, int D, int H, const int* node_first, const int* node_g,
                  int max_g, const void* V, long long sVj, const float* L, long long sLj,
                  const float* mix, void* ctx, void* stream);

/* Same, with child rows interleaved: row r = rb*rows_inner + rs lives at
 * V + j*sVj + rb*sVb + rs*D (L: L + j*sLj + rb*sLb + rs*H) -- e.g. tokens [B][C][S][D]
 * (tree_aggregate on tokens, model.py:76-97). */
int dchag_combine_strided(int n_nodes, int R, int D, int H, const int* node_first,
                          const int* node_g, int max_g, const void* V, long long sVj,
                          long long sVb, const float* L, long long sLj, long long sLb,
                          int rows_inner, const float* mix, void* ctx, void* stream);

/* Backward of dchag_combine (training; reference tape tensor.py:168-205 through
 * layers.py:103-123 / :141-146).  G fp32 [n][R][D] = dLoss/dctx.  Writes, per child j:
 * gV_j = p_jh * G[h-blk] (bf16, V's strides), and dL_j = p (dp - sum p dp) (fp32, L's
 * strides; attention) or dm_j[r] = G[r] . V_j[r] (fp32 [child][R]; linear). */
/* Backward of full_cross nodes (layers.py:125-138 through tensor.py:395-413), one CTA per
 * (node, row), g <= 16: recomputes the channel attention S^h, p2 and w from q | k | v
 * (child j row r at QKV + j*sQj + r*ldq, bf16) and u (fp32 [child][R][H]), and from
 * G = dLoss/dctx (fp32 [n][R][D]) and a = (wo rq)/sqrt(D) (fp32 [n][D]) writes
 * dq | dk | dv (bf16, the QKV layout at dQKV) and dA[n][r][:] = sum_j du_jh v_j,h (fp32; its
 * column sum is the gradient of a). */
int dchag_fullcross_bwd(int n_nodes, int R, int D, int H, const int* node_first,
                        const int* node_g, int max_g, const void* QKV, long long sQj,
                        long long ldq, const float* u, const float* G, const float* a_vec,
                        void* dQKV, float* dA, void* stream);

int dchag_combine_bwd(int n_nodes, int R, int D, int H, const int* node_first, const int* node_g,
                      int max_g, const void* V, long long sVj, const float* L, long long sLj,
                      const float* mix, const float* G, float* dL, void* gV, float* dm,
                      void* stream);

/* dchag_combine_bwd writing the K-concatenated operand of the training step's backward
 * GEMMs: gVL child j row r at gVL + j*sGj + r*ldg holds [gV_j (D bf16) | dL_j (H bf16)]
 * (attention) or gV_j (linear, with dm). ldg >= D + H, multiple of 8. */
int dchag_combine_bwd_packed(int n_nodes, int R, int D, int H, const int* node_first,
                             const int* node_g, int max_g, const void* V, long long sVj,
                             const float* L, long long sLj, const float* mix, const float* G,
                             void* gVL, long long sGj, long long ldg, float* dm, void* stream);

/* unfold_patches (tensor.py:303-323): img [B][C][Himg][W] -> out [B][C][S][P*P] bf16. */
int dchag_unfold(const void* img, long long img_sb, long long img_sc, int B, int C, int Himg,
                 int W, int P, void* out, void* stream);

/* Re-tile fp32 folded weights into the canonical no-swizzle K-major UMMA blocks read by
 * dchag_l0_node: src fp32 [nblk][K][N] (block b is a K x N matrix, column = output feature)
 * -> dst bf16 [nblk][K*N] in [K/8][N/8][8 rows][8 k] core-matrix order.  dchag_l0_node reads
 * Mt / Et as N = 32 blocks: each head's 64 output columns split into the two halves the CTAs
 * of a pair hold (block order [head][half]). */
int dchag_tile_weights(const float* src, int nblk, int K, int N, void* dst, void* stream);

/* Number of SMs the kernels size their persistent grids for (device of `stream`). */
int dchag_num_sms(void);

#ifdef __cplusplus
}
#endif
#endif /* DCHAG_H_ */
