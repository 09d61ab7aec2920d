/*
 * smpk.h — C ABI of libsmpk.so, the B200 (sm_100a) kernel library behind the
 * tensor-parallel hot path of the SageMaker model-parallelism design
 * (arXiv 2111.05972).
 *
 * The reference (/root/reference) has no FFI for this path: its tensor-parallel
 * operators exist only as the SPEC's free functions over a TpGroup
 * and as the paper's smp.nn API.  Every
 * entry point below names the SPEC/PAPER operation whose per-rank local compute
 * it performs; the collectives between them are issued by the host layer
 * (paper_2111_05972_b200/collectives.py) or by the peer-memory entry points at
 * the end of this header.
 *
 * Conventions
 *   - All pointers are raw device pointers (host pointers only where stated).
 *   - Tensors are bf16 unless the name says f32 / i64.  Leading dimensions and
 *     strides are in ELEMENTS.
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous on
 *     it and never allocates device memory.
 *   - Every function returns 0 (SMPK_OK) or an SMPK_ERR_* code; the message is
 *     available from smpk_last_error() (thread-local).
 */
#ifndef SMPK_H_
#define SMPK_H_

#include <stdint.h>

#if defined(__GNUC__)
#define SMPK_API __attribute__((visibility("default")))
#else
#define SMPK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes (SPEC.md:417,426,435,444 name the error classes) ---- */
#define SMPK_OK 0
#define SMPK_ERR_BAD_SHAPE 1     /* SPEC "shape mismatch" */
#define SMPK_ERR_NOT_DIVISIBLE 2 /* SPEC "non-divisible dimension" */
#define SMPK_ERR_OOB_INDEX 3     /* SPEC "out-of-range index -- reported with position" */
#define SMPK_ERR_PEER_TIMEOUT 4
#define SMPK_ERR_CUDA 5
#define SMPK_ERR_BAD_ARG 6
#define SMPK_ERR_UNSUPPORTED 7

/* ---- activations ("activation (gelu|relu)") ---- */
#define SMPK_ACT_NONE 0
#define SMPK_ACT_GELU_ERF 1  /* BERT gelu */
#define SMPK_ACT_GELU_TANH 2 /* GPT-2/3 gelu_new */
#define SMPK_ACT_RELU 3

/* ---- GEMM epilogues ---- */
#define SMPK_EPI_NONE 0     /* C = alpha*acc + beta*C                          */
#define SMPK_EPI_BIAS 1     /* C = alpha*acc + bias[n] (+ beta*C)               */
#define SMPK_EPI_BIAS_ACT 2 /* aux = acc + bias[n] (pre-activation); C = act(aux) */
#define SMPK_EPI_DACT 3     /* C = acc * act'(aux[m,n])  (activation backward)  */
#define SMPK_EPI_ADD 4      /* C = acc + aux[m,n]        (residual add)         */

SMPK_API const char* smpk_last_error(void);
SMPK_API int smpk_version(void);
/* number of SMs of the current device and whether it is an sm_100 part */
SMPK_API int smpk_device_info(int* num_sms, int* cc_major, int* cc_minor);

/*
 * smpk_gemm — batched C[m,n] = epi(alpha * sum_k A[m,k] * B[n,k]), tcgen05/TMEM/TMA.
 *
 * Replaces the local affine map inside dist_linear_forward/backward
 * (Fig 5) and the column/row-parallel linears and
 * attention contractions of dist_attention_forward / dist_mlp_forward
 * (PAPER.md:699-717).
 *
 *   A: a_mn_major == 0 -> A[m,k] = a[m*lda + k]   (row-major M x K)
 *      a_mn_major == 1 -> A[m,k] = a[k*lda + m]   (row-major K x M)
 *   B: b_mn_major == 0 -> B[n,k] = b[n*ldb + k]   (row-major N x K, i.e. nn.Linear weight)
 *      b_mn_major == 1 -> B[n,k] = b[k*ldb + n]   (row-major K x N)
 *   C: row-major M x N with ldc; bf16, or fp32 when c_f32 != 0.
 *   Batch: nb1 x nb2 problems; problem (i1,i2) offsets every operand by
 *   i1*x_bs1 + i2*x_bs2 elements (a zero A / B batch stride broadcasts that operand).
 *   aux (for BIAS_ACT / DACT / ADD) is bf16, row-major with ldaux and the same batch
 *   strides as C.
 */
SMPK_API int smpk_gemm(const void* a, int a_mn_major, int64_t lda, int64_t a_bs1, int64_t a_bs2,
              const void* b, int b_mn_major, int64_t ldb, int64_t b_bs1, int64_t b_bs2,
              void* c, int c_f32, int64_t ldc, int64_t c_bs1, int64_t c_bs2,
              int M, int N, int K, int nb1, int nb2,
              float alpha, float beta, int epilogue, int act,
              const void* bias, void* aux, int64_t ldaux, void* stream);

/*
 * smpk_gemm_ex — smpk_gemm with a split-K workspace.  When the output has too few
 * 128 x BN tiles to fill the SMs (the weight-gradient GEMMs dW = dY^T X, whose K is the
 * token count), the K range is split across CTAs; every split stores an fp32 partial
 * tile into `workspace` and the tile's splits then reduce it in split order
 * (deterministic) and apply the epilogue.  smpk_gemm_workspace returns the bytes the
 * chosen split needs (0: no split); a NULL / smaller workspace runs unsplit.
 */
SMPK_API int64_t smpk_gemm_workspace(int M, int N, int K, int nb1, int nb2);
/* smpk_set_sm_limits — cap the persistent grids of the GEMM (gemm_sms) and row / exchange kernels
 * (row_sms) launched after this call (0 = whole GPU), so kernels on two streams can share the SMs. */
SMPK_API int smpk_set_sm_limits(int gemm_sms, int row_sms);
SMPK_API int smpk_gemm_ex(const void* a, int a_mn_major, int64_t lda, int64_t a_bs1, int64_t a_bs2,
                          const void* b, int b_mn_major, int64_t ldb, int64_t b_bs1, int64_t b_bs2,
                          void* c, int c_f32, int64_t ldc, int64_t c_bs1, int64_t c_bs2,
                          int M, int N, int K, int nb1, int nb2,
                          float alpha, float beta, int epilogue, int act,
                          const void* bias, void* aux, int64_t ldaux, void* workspace, int64_t workspace_bytes,
                          void* stream);

/*
 * smpk_gemm_ex2 — smpk_gemm_ex that also emits the output's column sums (the bias gradient of the
 * layer whose input gradient it produces): colsum_part [smpk_gemm_colsum_rows(M)][N] fp32 receives
 * the sum of every 32-row output box (bf16 values as stored); smpk_colsum_partials reduces the
 * partial rows in order.  bf16, unbatched, unsplit outputs on the TMA-store path only.
 */
SMPK_API int64_t smpk_gemm_colsum_rows(int M);
SMPK_API int smpk_gemm_ex2(const void* a, int a_mn_major, int64_t lda, int64_t a_bs1, int64_t a_bs2,
                           const void* b, int b_mn_major, int64_t ldb, int64_t b_bs1, int64_t b_bs2,
                           void* c, int c_f32, int64_t ldc, int64_t c_bs1, int64_t c_bs2,
                           int M, int N, int K, int nb1, int nb2,
                           float alpha, float beta, int epilogue, int act,
                           const void* bias, void* aux, int64_t ldaux, void* workspace, int64_t workspace_bytes,
                           float* colsum_part, void* stream);
SMPK_API int smpk_colsum_partials(const float* part, int P, int N, void* out, int out_f32, void* stream);

/*
 * smpk_bdr_ln_fwd — r = residual + dropout(x + bias); y = LayerNorm(r; gamma, beta, eps).
 *
 * The epilogue of every sub-layer of dist_transformer_layer_forward
 * ("attention -> residual -> norm"), i.e. the bias, hidden
 * dropout (PAPER.md:818 hidden_dropout_prob), residual add and replicated
 * LayerNorm of speed mode.  bias/residual may be NULL; with
 * gamma == NULL no LayerNorm is applied (only r is produced); with r_out == NULL
 * r is not stored.  x, r_out, y_out: [M, H]; mean/rstd: fp32 [M].  Dropout keeps
 * element (row, col) per Philox4x32-10 with counter (col>>2, row_offset+row,
 * layer, site) and key `seed + *rng_step * 0x9E3779B97F4A7C15` (oracle/philox.py step_key;
 * rng_step may be null = step 0; it is the per-forward snapshot written by smpk_rng_next).  H must be a multiple of 256.
 */
SMPK_API int smpk_bdr_ln_fwd(const void* x, const void* bias, const void* residual, void* r_out,
                             const void* gamma, const void* beta, void* y_out, float* mean, float* rstd,
                             int M, int H, float eps, float p_drop, uint64_t seed, const uint64_t* rng_step, int layer, int site,
                             int64_t row_offset, void* stream);

/*
 * smpk_ln_bwd — backward of smpk_bdr_ln_fwd.
 *   dr   = LN'(dy; r, mean, rstd, gamma) + dres          (dres may be NULL)
 *   dsub = dropout'(dr)  (written only when p_drop > 0; otherwise dsub == dr)
 *   dgamma = colsum(dy * xhat), dbeta = colsum(dy), dbias = colsum(dsub)
 * Column sums are deterministic (fixed-order two-stage reduction) and written as
 * fp32 (grads_f32) or bf16, overwriting or accumulating.  Any of dgamma / dbeta /
 * dbias may be NULL.  workspace >= smpk_ln_bwd_workspace(M, H) bytes.
 */
SMPK_API int64_t smpk_ln_bwd_workspace(int M, int H);
SMPK_API int smpk_ln_bwd(const void* dy, const void* r, const float* mean, const float* rstd, const void* gamma,
                         const void* dres, void* dr_out, void* dsub_out, void* dgamma, void* dbeta, void* dbias,
                         int grads_f32, int accumulate, int M, int H, float p_drop, uint64_t seed, const uint64_t* rng_step, int layer,
                         int site, int64_t row_offset, void* workspace, int64_t workspace_bytes, void* stream);

/*
 * smpk_softmax_fwd / smpk_softmax_bwd — masked, scaled softmax over attention
 * scores with attention-probability dropout (the "scaled dot-product attention
 * with softmax over masked scores" of dist_attention_forward).
 *   scores, probs, probs_drop: [B, nh, sq, sk] bf16 contiguous.
 *   P  = softmax(scale * S + mask_add[b, k]  (+ -inf where k > q + sk - sq if causal))
 *   Pd = P * keep / (1 - p)   (written when p_drop > 0)
 *   backward: dS = scale * (Pd * dPd - P * sum_k(Pd * dPd))  (dscores may alias dprobs_drop)
 * Fully masked rows give P = 0.  Dropout row coordinate is
 * ((sample_offset + b) * nh_global + head_offset + h) * sq + q, site 0.
 */
SMPK_API int smpk_softmax_fwd(const void* scores, void* probs, void* probs_drop, const float* mask_add, int B,
                              int nh, int sq, int sk, float scale, int causal, float p_drop, uint64_t seed, const uint64_t* rng_step,
                              int layer, int64_t sample_offset, int head_offset, int nh_global, void* stream);
SMPK_API int smpk_softmax_bwd(const void* probs, const void* dprobs_drop, void* dscores, int B, int nh, int sq,
                              int sk, float scale, float p_drop, uint64_t seed, const uint64_t* rng_step, int layer, int64_t sample_offset,
                              int head_offset, int nh_global, void* stream);

/* smpk_colsum — out[n] (+)= sum_m x[m, n] (bias gradients), deterministic. */
SMPK_API int64_t smpk_colsum_workspace(int M, int N);
SMPK_API int smpk_colsum(const void* x, int M, int N, int64_t ldx, void* out, int out_f32, int accumulate,
                         void* workspace, int64_t workspace_bytes, void* stream);

/*
 * smpk_embed_fwd — embedding lookup of the rank's table slice.
 *   Vocab-parallel (builder-defined extension): the rank owns global
 *   rows [row_offset, row_offset + rows_local); non-owned ids give 0 (the TP combine
 *   is an allreduce / reduce-scatter).  Embedding-dim sharded DistributedEmbedding
 *   (SPEC.md:440-448): row_offset = 0, rows_local = vocab, table holds
 *   the rank's D/T columns.  out[t, :dim] = lookup (+ pos_table[t % seq] if non-NULL).
 *   Ids outside [0, vocab) set *err_pos = min(position) ("reported with
 *   position"); err_pos must be initialised to UINT64_MAX by the caller.
 */
SMPK_API int smpk_embed_fwd(const int64_t* ids, int64_t n, const void* table, int64_t ld_table,
                            int64_t row_offset, int64_t rows_local, int64_t vocab, int dim, void* out,
                            int64_t ld_out, const void* pos_table, int64_t ld_pos, int seq,
                            unsigned long long* err_pos, void* stream);
/*
 * smpk_embed_bwd — dtable[r] (+)= sum of dy[t] over tokens t with ids[t] == row_offset + r,
 * accumulated in token order (bit-deterministic, no float atomics); rows equal to
 * padding_row get no gradient (torch padding_idx semantics; pass -1 for none).
 */
SMPK_API int smpk_embed_bwd(const int64_t* ids, int64_t n, const void* dy, int64_t ld_dy, int64_t row_offset,
                            int64_t rows_local, int dim, void* dtable, int64_t ld_dt, int out_f32,
                            int accumulate, int64_t padding_row, void* stream);
/*
 * smpk_embed_bwd_sorted — the same gradient for tables much larger than the batch (NCF:
 * 10^8 rows): stable LSD radix sort of (local row, token position), then fixed-order
 * segmented sums with one read-modify-write per unique row; O(n log rows), no float atomics
 * (bit-deterministic).  accumulate = 0 zeroes dtable first.  dim, ld_dy, ld_dt multiples of 8.
 * Workspace: smpk_embed_bwd_sorted_workspace(n, rows_local, dim) bytes.
 */
SMPK_API int64_t smpk_embed_bwd_sorted_workspace(int64_t n, int64_t rows_local, int dim);
SMPK_API int smpk_embed_bwd_sorted(const int64_t* ids, int64_t n, const void* dy, int64_t ld_dy,
                                   int64_t row_offset, int64_t rows_local, int dim, void* dtable, int64_t ld_dt,
                                   int out_f32, int accumulate, int64_t padding_row, void* workspace,
                                   int64_t workspace_bytes, void* stream);
/*
 * Vocab-parallel softmax cross-entropy (builder-defined).
 *   fwd_local: stats[N][4] = {m_j, S_j = sum_{real cols} exp(l - m_j), l[target] if owned, owned}
 *              for the shard covering global columns [col_offset, col_offset + v_local); columns
 *              >= vocab are padding (-inf).
 *   combine:   stats_all [T][N][4] (allgathered, rank order) -> loss[N] = log S + m - l_tgt with
 *              m = max m_j, S = sum_j S_j e^{m_j - m}; ms[N][2] = (m, S).  Ignored rows -> 0.
 *   bwd:       dlogits = (exp(l - m) / S - onehot(target)) * grad_loss[row] * grad_scale.
 */
SMPK_API int smpk_vocab_ce_fwd_local(const void* logits, int64_t ld, int64_t N, int v_local, int64_t col_offset,
                                     int64_t vocab, const int64_t* targets, int64_t ignore_index, float* stats,
                                     void* stream);
SMPK_API int smpk_vocab_ce_combine(const float* stats_all, int T, int64_t N, const int64_t* targets,
                                   int64_t ignore_index, float* loss, float* ms, void* stream);
SMPK_API int smpk_vocab_ce_bwd(const void* logits, int64_t ld, int64_t N, int v_local, int64_t col_offset,
                               int64_t vocab, const int64_t* targets, int64_t ignore_index, const float* ms,
                               const float* grad_loss, float grad_scale, void* dlogits, int64_t ld_out,
                               void* stream);

/*
 * smpk_flash_attn_fwd — fused attention of one TP rank's local heads ("per-rank
 * scaled dot-product attention with softmax over masked scores"), on the
 * packed QKV buffer produced by the column-parallel QKV GEMM:
 *   qkv [B*s, ld] with q | k | v blocks of nh*dh columns, head h at column h*dh of each block;
 *   out [B*s, ld_out] (head h at column h*dh) = dropout(softmax(scale*QK^T + mask [+causal])) V;
 *   lse [B, nh, s] = log2-sum-exp2 of the scaled masked scores (for the backward).
 * dh in {64, 128}; s a multiple of 128.  Dropout (p_drop > 0) zeroes the probabilities whose
 * keep bit is clear in keep_bits (from smpk_attn_dropout_bits; the same bits smpk_softmax_fwd
 * draws) and scales the kept ones by 1/(1-p).
 */
SMPK_API int smpk_flash_attn_fwd(const void* qkv, int64_t ld, int B, int nh, int s, int dh, void* out,
                                 int64_t ld_out, float* lse, const float* mask_add, float scale, int causal,
                                 float p_drop, const uint32_t* keep_bits, void* stream);

/*
 * smpk_attn_dropout_bits — attention-probability dropout keep bits of one TP rank's local
 * heads: word ((b*nh + h)*sq + q)*(sk/32) + k/32, bit k%32 = keep(q, k) of the Philox4x32-10
 * stream (site 0, row = ((sample_offset+b)*nh_global + head_offset+h)*sq + q, col = k) that
 * oracle/philox.py restates.  Generated once per layer and read by the forward and backward.
 * causal != 0: words whose 128-key tile lies after the query's 128-row tile are not written
 * (the fused kernels never read them).
 */
SMPK_API int smpk_attn_dropout_bits(int B, int nh, int sq, int sk, float p_drop, uint64_t seed, const uint64_t* rng_step, int layer,
                                    int64_t sample_offset, int head_offset, int nh_global, uint32_t* bits,
                                    int causal, void* stream);
/* ... with the B samples in blocks of sample_block consecutive global samples, block_stride apart
 * (sample b -> sample_offset + (b / sample_block) * block_stride + b % sample_block): the
 * rank-major gathered samples of one overlapped micro-batch (tp_exchange = "overlap"). */
SMPK_API int smpk_attn_dropout_bits_blocked(int B, int nh, int sq, int sk, float p_drop, uint64_t seed,
                                            const uint64_t* rng_step, int layer, int64_t sample_offset,
                                            int sample_block, int64_t block_stride, int head_offset, int nh_global,
                                            uint32_t* bits, int causal, void* stream);

/*
 * smpk_flash_attn_bwd — backward of smpk_flash_attn_fwd: from dout (grad of out, same layout),
 * the forward's out and lse, writes dQ | dK | dV into dqkv (same layout as qkv).  P is
 * recomputed from lse (never stored); dQ partials of the key tiles are reduced in order
 * (deterministic).  workspace >= smpk_flash_attn_bwd_workspace(B, nh, s, dh) bytes.
 */
SMPK_API int64_t smpk_flash_attn_bwd_workspace(int B, int nh, int s, int dh);
SMPK_API int smpk_flash_attn_bwd(const void* qkv, int64_t ld, const void* out, int64_t ld_out, const void* dout,
                                 int64_t ld_dout, const float* lse, int B, int nh, int s, int dh, void* dqkv,
                                 const float* mask_add, float scale, int causal, float p_drop,
                                 const uint32_t* keep_bits, void* workspace, int64_t workspace_bytes, void* stream);

/*
 * Fused tensor-parallel collectives over peer-mapped (symmetric) memory — the row-parallel
 * "partial-sum allreduce fused into the GEMM epilogue through NVLink peer stores" of the
 * north_star, in the reduce-scatter + allgather form used with row-sharded activations
 * (fwd_allreduce_for_tp / reduce_scatter_for_tp / fused_allgather_for_tp).
 *   smpk_gemm_rs        C = A B^T with row r stored (TMA bulk stores over NVLink) to
 *                       peers[r / rows_per_owner] + peer_slot_off; peers is a HOST array of the
 *                       npeers peer-mapped base addresses, M = npeers * rows_per_owner;
 *                       row r lands at element (r % rows_per_owner) * ldc of the owner's slot
 *   smpk_bdr_ln_fwd_ex  smpk_bdr_ln_fwd reading x as the ascending-rank sum of nslots partial slots
 *                       (slot_stride elements apart) and storing its output to every out_peers[j]
 *                       + peer_off (allgather producer)
 *   smpk_ln_bwd_ex      smpk_ln_bwd with the same slot-sum input / peer-store output for dy / dsub
 *                       keep_out (forward, may be NULL) stores the hidden-dropout keep bits as
 *                       [M][H/8] bytes (bit j = column 8c+j); keep_in (backward) reads them
 *                       instead of re-drawing the Philox stream; x_peers / dy_peers (device table
 *                       of the T peer-mapped pool bases, may be NULL) make the input the
 *                       ascending-rank sum of the nslots peers' rows at element offset
 *                       x_peer_off (reduce-scatter consumer pulling the partials over NVLink)
 *   smpk_symm_export    IPC handle + offset of a pointer inside its allocation
 *   smpk_symm_barrier   epoch barrier over the group (system-scope release/acquire flag words);
 *                       the epoch counter is device-resident (local_flags[32]) so a barrier
 *                       captured in a CUDA graph advances on every replay.  After timeout_s
 *                       without a peer's signal the kernel records 1 + that peer in pinned
 *                       mapped host memory and traps (a sticky CUDA error: no stale peer data is
 *                       ever consumed); smpk_symm_timeout_peer reads the record without a CUDA
 *                       call, so the host can raise PEER_TIMEOUT naming the stuck peer
 */
/*
 * smpk_gemm_grouped — several independent GEMMs in one launch (currently n <= 2 are fused).
 * Each smpk_gemm_desc carries the arguments of smpk_gemm_ex2.  Two problems are fused into one
 * persistent CTA-pair grid when one of them is a plain bf16 GEMM (no epilogue, no column sums)
 * and both tile as 256 x 256 unsplit pairs: the plain problem's units (the long weight-gradient
 * tiles of a backward) run first, the other's (with its fused epilogue) fill in behind them, so
 * neither exposes its own wave tail or epilogue.  Otherwise the problems run one after the other.
 * Used by the transformer backward for (dW, dX) pairs that read the same upstream gradient.
 */
typedef struct smpk_gemm_desc {
  const void* a;
  int a_mn_major;
  int64_t lda, a_bs1, a_bs2;
  const void* b;
  int b_mn_major;
  int64_t ldb, b_bs1, b_bs2;
  void* c;
  int c_f32;
  int64_t ldc, c_bs1, c_bs2;
  int M, N, K, nb1, nb2;
  float alpha, beta;
  int epilogue, act;
  const void* bias;
  void* aux;
  int64_t ldaux;
  void* workspace;
  int64_t workspace_bytes;
  float* colsum_part;
} smpk_gemm_desc;
SMPK_API int smpk_gemm_grouped(const smpk_gemm_desc* descs, int n, void* stream);
SMPK_API int smpk_gemm_rs(const void* a, int a_mn_major, int64_t lda, const void* b, int b_mn_major, int64_t ldb,
                          void* const* peers, int npeers, int64_t ldc, int64_t rows_per_owner,
                          int64_t peer_slot_off, int M, int N, int K, void* stream);
SMPK_API int smpk_bdr_ln_fwd_ex(const void* x, int nslots, int64_t slot_stride, const void* bias, const void* residual,
                                void* r_out, const void* gamma, const void* beta, void* y_out, float* mean,
                                float* rstd, void* const* out_peers, int npeers, int64_t peer_off, int M, int H,
                                float eps, float p_drop, uint64_t seed, const uint64_t* rng_step, int layer, int site, int64_t row_offset,
                                void* keep_out, void* const* x_peers, int64_t x_peer_off, void* stream);
SMPK_API int smpk_ln_bwd_ex(const void* dy, int nslots, int64_t slot_stride, const void* r, const float* mean,
                            const float* rstd, const void* gamma, const void* dres, void* dr_out, void* dsub_out,
                            void* const* out_peers, int npeers, int64_t peer_off, void* dgamma, void* dbeta,
                            void* dbias, int grads_f32, int accumulate, int M, int H, float p_drop, uint64_t seed, const uint64_t* rng_step,
                            int layer, int site, int64_t row_offset, const void* keep_in, void* const* dy_peers,
                            int64_t dy_peer_off, void* workspace, int64_t workspace_bytes, void* stream);
/*
 * Channel-sharded (memory-mode) LayerNorm, "local sum x, sum x^2 -> scalar
 * allreduce -> ApplyLayerNorm": activations hold H/T of the H_total channels.
 *   smpk_bdr_ln_fwd_dist  as smpk_bdr_ln_fwd on the local columns, with the hidden-dropout column
 *                         index offset by col_offset; row_sums_out != NULL stores the partial
 *                         [M][2] (sum r, sum r^2); ext_sums != NULL normalises with the group's
 *                         sums (mean = S1/H_total, var = S2/H_total - mean^2).
 *   smpk_ln_bwd_dist      as smpk_ln_bwd; row_sums_out != NULL is a sums-only pass storing the
 *                         partial [M][2] (sum g, sum g*xhat; g = dy*gamma); ext_sums != NULL uses
 *                         the group's sums for the row means of the LayerNorm backward.
 * The [M][2] partials are summed across the TP group (NCCL allreduce) between the passes.
 */
SMPK_API int smpk_bdr_ln_fwd_dist(const void* x, const void* bias, const void* residual, void* r_out,
                                  const void* gamma, const void* beta, void* y_out, float* mean, float* rstd, int M,
                                  int H, float eps, float p_drop, uint64_t seed, const uint64_t* rng_step, int layer, int site,
                                  int64_t row_offset, int64_t col_offset, float* row_sums_out, const float* ext_sums,
                                  int H_total, void* stream);
SMPK_API int smpk_ln_bwd_dist(const void* dy, const void* r, const float* mean, const float* rstd, const void* gamma,
                              const void* dres, void* dr_out, void* dsub_out, void* dgamma, void* dbeta, void* dbias,
                              int grads_f32, int M, int H, float p_drop, uint64_t seed, const uint64_t* rng_step, int layer, int site,
                              int64_t row_offset, int64_t col_offset, float* row_sums_out, const float* ext_sums,
                              int H_total, void* workspace, int64_t workspace_bytes, void* stream);
/*
 * smpk_bias_act_fwd — pre = bf16(x + bias) (bias per column), y = act(pre); [M, N] row-major.
 * smpk_act_bwd      — dx = dy * act'(pre).  The MLP activation of memory mode, which follows a
 * reduce-scatter and so cannot be fused into the GEMM epilogue.
 */
SMPK_API int smpk_bias_act_fwd(const void* x, const void* bias, int M, int N, int act, void* pre_out, void* y,
                               void* stream);
SMPK_API int smpk_act_bwd(const void* dy, const void* pre, int M, int N, int act, void* dx, void* stream);
/* smpk_copy_async — stream-ordered device-to-device copy (copy engine; dst may be peer-mapped). */
SMPK_API int smpk_copy_async(void* dst, const void* src, int64_t bytes, void* stream);

/* smpk_stream_flag — stream-ordered 32-bit flag word (cuStreamWaitValue32 / cuStreamWriteValue32,
 * no SM): op 0 waits until *word == value, op 1 writes *word = value after the stream's prior work
 * (fenced: a preceding copy into a peer slot is visible first).  The mailbox handshake of the
 * chunked TP exchange (PAPER.md:281 AG/RS of TP-across-DP, split into per-owner chunks so the
 * copy engines move chunk c while the SMs compute chunk c+1). */
SMPK_API int smpk_stream_flag(void* word, uint32_t value, int op, void* stream);

/* Mailbox copies of the overlapped TP exchanges (tp_exchange = "overlap" / "chunks"; PAPER.md:281
 * AG/RS of TP across DP moved while the other micro-batch computes).  smpk_peer_put copies up to
 * SMPK_PUT_MAX_RANGES 16-byte-aligned ranges into peer-mapped slots with ordinary vector stores
 * (a few CTAs, SMPK_PUT_CTAS, default 32), then raises each destination group's ready word
 * (release.sys after the group's last CTA); a group with an ack word first waits for ack == 0
 * (the receiver released the previous round) and sets ack = 1.  counter: SMPK_PUT_MAX_GROUPS
 * zeroed words owned by this stream.  smpk_flag_wait spins until every word == value, then
 * re-arms it to 0 (timeout: records who[i] + 1 -- the signalling peer -- for smpk_symm_timeout_peer
 * and traps);
 * smpk_flag_set release-stores value into every word. */
#define SMPK_PUT_MAX_RANGES 16
#define SMPK_PUT_MAX_GROUPS 8
typedef struct {
  const void* src;
  void* dst;
  int64_t bytes;
  int group;
} smpk_put_range;
typedef struct {
  uint32_t* ready;
  uint32_t* ack;
} smpk_put_group;
SMPK_API int smpk_peer_put(const smpk_put_range* ranges, int nr, const smpk_put_group* groups, int ng, void* counter,
                           double timeout_s, void* stream);
SMPK_API int smpk_flag_wait(void* const* words, const int* who, int n, uint32_t value, double timeout_s, void* stream);
SMPK_API int smpk_flag_set(void* const* words, int n, uint32_t value, void* stream);
SMPK_API int smpk_symm_export(void* ptr, void* handle_out, int64_t* offset);
SMPK_API int smpk_symm_barrier(void* const* peer_flags, void* local_flags, int T, int rank, double timeout_s,
                               void* stream);
SMPK_API int smpk_symm_timeout_peer(void);

/*
 * Pipeline stage send/recv over NVLink peer memory — the D2D communicator of the
 * module server; replaces the simulated hop
 * mpsim pipeline.py:653-712 (_transfer / _send_request / _send_response) whose routing
 * and persistent-buffer accounting are comm.py:157-225.
 *   smpk_p2p_alloc/free       persistent receive ring (slots + sequence words), zeroed
 *   smpk_p2p_export/import    CUDA IPC handle (64 bytes) exchanged once per peer pair
 *   smpk_p2p_send             [wait local_free >= wait_free] -> copy to peer slot ->
 *                             peer_ready = seq + 1            (all stream-ordered)
 *   smpk_p2p_recv             wait local_ready >= seq + 1 -> copy slot -> dst ->
 *                             peer_free = seq + 1
 */
SMPK_API int smpk_p2p_alloc(int64_t bytes, void** ptr);
SMPK_API int smpk_p2p_free(void* ptr);
SMPK_API int smpk_p2p_export(void* ptr, void* handle_out);
SMPK_API int smpk_p2p_import(const void* handle, void** ptr);
SMPK_API int smpk_p2p_close(void* ptr);
SMPK_API int smpk_p2p_send(void* peer_slot, const void* src, int64_t bytes, void* peer_ready, const void* local_free,
                           uint32_t wait_free, uint32_t seq, void* stream);
SMPK_API int smpk_p2p_recv(void* dst, const void* local_slot, int64_t bytes, const void* local_ready,
                           void* peer_free, uint32_t seq, void* stream);


/* Per-step dropout RNG (PAPER.md:818 dropout 0.1).  Every dropout-drawing
 * call takes `const uint64_t* rng_step`: the Philox key is seed + (*rng_step) * 0x9E3779B97F4A7C15.
 * smpk_rng_next copies the device counter into *snapshot and increments the counter, on `stream`
 * (one tiny kernel: CUDA-graph capturable, so every replay of a captured training step draws new
 * masks).  A forward passes its snapshot to every kernel it launches and its backward re-reads
 * the same snapshot, so interleaved microbatches (pipeline schedules) stay consistent. */
SMPK_API int smpk_rng_next(uint64_t* counter, uint64_t* snapshot, void* stream);

/* smpk_adam_step — fused AdamW on one slice of fp32 master parameters (data-parallel optimizer,
 * PAPER.md:765 "shard_optimizer_state"): g = grad * grad_scale; m = b1 m + (1-b1) g;
 * v = b2 v + (1-b2) g^2; master -= lr * ((m / (1-b1^step)) / (sqrt(v / (1-b2^step)) + eps) + wd * master);
 * param_bf16 = bf16(master).  n % 4 == 0, 16-B aligned fp32 buffers. */
SMPK_API int smpk_adam_step(float* master, void* param_bf16, const float* grad, float* m, float* v, int64_t n,
                            float lr, float beta1, float beta2, float eps, float weight_decay, int step,
                            float grad_scale, void* stream);

/* Debug: per-CTA globaltimer records of the last fused-attention forward launched with
 * SMPK_FA_TRACE=1 in the environment (20 u64 per CTA; see csrc/flash_attn.cu).  Diagnostics only. */
SMPK_API int smpk_debug_fa_trace(void* host_out, int n_cta);
SMPK_API int smpk_debug_fb_trace(void* host_out, int n_cta); /* backward: 32 u64 per CTA */
SMPK_API int smpk_debug_gemm_trace(void* host_out, int n_cta); /* GEMM (SMPK_GEMM_TRACE=1): 40 u64 per CTA */

#ifdef __cplusplus
}
#endif

#endif /* SMPK_H_ */
