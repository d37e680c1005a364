/*
 * icepop.h -- C ABI of the B200-native (sm_100a) IcePop policy-gradient objective.
 *
 * This library replaces the reference's hot path, mismatchlab's
 *   objective_and_grad(groups, theta, theta_old, ref, cfg, bounds, temperature)
 *   (/root/reference/pkg/src/mismatchlab/objective.py:172-298)
 * together with the numerics it calls,
 *   batched_train_logits  (policy.py:279-289)   -> the lm_head contraction Z = H.W / T
 *   batched_log_softmax   (policy.py:350-355)   -> online log-sum-exp, gather, entropy
 *   group_advantages      (objective.py:153-159)
 * The reference has no FFI of its own (it is pure numpy); the Python host layer
 * (paper_2510_18855_b200.objective / .loss) binds these entry points with ctypes,
 * exactly as INTEGRATION.md shows for a maintainer wiring it into mismatchlab.
 *
 * Conventions
 *   - Plain pointers and sizes; every pointer is DEVICE memory unless stated.
 *   - Every call is stream-ordered on `stream` (a cudaStream_t passed as void*).
 *     Nothing synchronises the host except icepop_*_finish, which reads the
 *     device error word once.
 *   - Gradients are the reference's ASCENT gradient dJ/dW (objective.py:250-266)
 *     multiplied by `grad_scale`; a torch loss = -J passes grad_scale = -dL/dloss.
 *   - Reductions are fixed-order (no floating-point atomics): results are
 *     bit-stable run to run for a fixed shape and device count.
 *   - Return codes mirror the reference's exceptions:
 *       ICEPOP_OK       0
 *       ICEPOP_EINVAL   1  -> ValueError  (objective.py:190-193, 205-213)
 *       ICEPOP_ENUMERIC 2  -> NumericError (objective.py:228-229, 241-242, 279-280)
 *       ICEPOP_ECUDA    3  -> RuntimeError (CUDA launch / runtime failure)
 *       ICEPOP_EARCH    4  -> RuntimeError (device is not sm_100)
 *     icepop_last_error() returns a per-thread message for the last failure.
 */
#ifndef ICEPOP_B200_H_
#define ICEPOP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ICEPOP_ABI_VERSION 4

enum icepop_status {
  ICEPOP_OK = 0,
  ICEPOP_EINVAL = 1,
  ICEPOP_ENUMERIC = 2,
  ICEPOP_ECUDA = 3,
  ICEPOP_EARCH = 4
};

/* objective.py:41-44 (Algo) */
enum icepop_algo { ICEPOP_ALGO_ICEPOP = 0, ICEPOP_ALGO_GRPO = 1, ICEPOP_ALGO_TIS = 2 };

/* Weight layouts. [d,V] is the reference PolicyParams layout (policy.py:132-155,
 * weights[n_features, vocab]); [V,d] is the usual lm_head (nn.Linear) layout. */
enum icepop_weight_layout { ICEPOP_W_DV = 0, ICEPOP_W_VD = 1 };

/* Device error word bits (read by icepop_*_finish). */
#define ICEPOP_ERR_CALIB_OVERFLOW 1u  /* objective.py:228-229 */
#define ICEPOP_ERR_RATIO_OVERFLOW 2u  /* objective.py:241-242 */
#define ICEPOP_ERR_NONFINITE      4u  /* objective.py:279-280, policy.py:287-288 */

/* Layout of the per-rank fp64 statistics vector (summed across ranks by the caller). */
enum icepop_stat {
  ICEPOP_STAT_OBJECTIVE = 0,        /* sum_t w_t * (s_t - gamma*kl_t)            objective.py:268-278 */
  ICEPOP_STAT_N_POPPED = 1,         /* #(not kept)                               objective.py:284     */
  ICEPOP_STAT_TOKENS = 2,           /* token count                               objective.py:291     */
  ICEPOP_STAT_SUM_ENTROPY = 3,      /* sum_t entropy_t                           objective.py:293     */
  ICEPOP_STAT_SUM_ENTROPY_POPPED = 4,/* sum over popped tokens of entropy_t      objective.py:294     */
  ICEPOP_STAT_SUM_LOGP = 5,         /* sum_t lp_cur_t                            objective.py:292     */
  ICEPOP_STAT_SUM_KL = 6,           /* sum_t kl_t                                objective.py:290     */
  ICEPOP_STAT_ERRORS = 7,           /* OR of ICEPOP_ERR_* (as a double)                               */
  ICEPOP_NSTATS = 8
};

/* objective.py:47-82 (MaskingBounds, ObjectiveConfig) + the temperature argument. */
typedef struct icepop_config {
  double alpha;        /* inclusive lower calibration bound  (default 0.5) */
  double beta;         /* inclusive upper calibration bound  (default 5.0) */
  double clip_eps;     /* PPO clip epsilon                   (default 0.2) */
  double tis_cap;      /* TIS truncation cap                 (default 2.0) */
  double temperature;  /* logits are divided by it           (default 1.0) */
  double kl_coeff;     /* gamma of the KL-to-ref penalty     (default 0.0) */
  int32_t algo;        /* enum icepop_algo */
  int32_t _pad;
} icepop_config;

/* Batch geometry. Tokens are packed sequence-major in the reference's order
 * (group-major, then rollout, then token: objective.py:271-276). A rank owns the
 * contiguous global token range [token_offset, token_offset + n_tokens). */
typedef struct icepop_shape {
  int64_t n_tokens;      /* local tokens on this rank (rows of hidden)         */
  int64_t token_offset;  /* global index of the first local token              */
  int64_t hidden;        /* d  (n_features in the reference)                   */
  int64_t vocab;         /* V                                                  */
  int32_t n_seqs;        /* S, sequences (rollouts) in the GLOBAL batch        */
  int32_t n_groups;      /* prompt groups in the GLOBAL batch                  */
  int32_t weight_layout; /* enum icepop_weight_layout                          */
  int32_t _pad;
} icepop_shape;

/* Per-sequence metadata, replicated on every rank (device pointers). */
typedef struct icepop_batch {
  const int32_t* tokens;        /* [n_tokens]     sampled token id y_t (local)          */
  const double* lp_train_old;   /* [n_tokens]     TokenRecord.logp_train_old (local)    */
  const double* lp_infer_old;   /* [n_tokens]     TokenRecord.logp_infer_old (local)    */
  const int32_t* cu_seqlens;    /* [n_seqs+1]     global token offsets of sequences     */
  const int32_t* group_offsets; /* [n_groups+1]   sequence offsets of prompt groups     */
  const double* advantages;     /* [n_seqs]       PromptGroup.advantages, or NULL       */
  const double* rewards;        /* [n_seqs]       used (with group_advantages) if advantages == NULL */
  /* [n_tokens] (local) the calibration ratio c_t = exp(lp_train_old - lp_infer_old) computed by
   * the caller, or NULL (then computed on the device with CUDA's exp, which may differ from
   * numpy's by 1 ulp). The drop-in passes numpy's own values so that the mask is the
   * reference's bit for bit even for a c_t within 1 ulp of alpha or beta (objective.py:227). */
  const double* calib;
} icepop_batch;

/* ---- library ---------------------------------------------------------------------- */
int icepop_abi_version(void);
const char* icepop_last_error(void);
/* 0 on an sm_100 device with the kernels loadable; ICEPOP_EARCH otherwise. */
int icepop_device_check(int device);

/* ---- K0: group advantages (objective.py:153-159) ---------------------------------- */
/* adv[i] = (R_i - mean_g R) / max(std_pop,g(R), 1e-6) for every sequence i of group g.
 * A group of fewer than 2 sequences yields NaN advantages (the host layers reject it with
 * ValueError first, as objective.py:156-157 does). */
int icepop_group_advantages(const double* rewards, const int32_t* group_offsets, int32_t n_groups,
                            int32_t n_seqs, double* advantages, void* stream);

/* ---- bf16 tensor-core path (production) ------------------------------------------- */
/* hidden: [n_tokens, d] bf16 row-major. weight (and weight_ref): bf16 in `weight_layout`.
 * Workspace sizes (bytes) for icepop_fwd_bf16 / icepop_bwd_bf16 (with_ref: a weight_ref
 * will be passed). The backward materialises bf16 dZ chunks of at most `max_chunk_tokens`
 * rows (0 = all rows) and each chunk's hidden rows transposed (dW's GEMM reads them K-major):
 * 2 (V + d) bytes per chunk row; a smaller workspace than recommended shrinks the chunk
 * (>= 128 rows). max_chunk_tokens < 0: the stored-probabilities backward's workspace (block
 * lists, row scales, s H transposed, the one-hot sort: ~2 n_tokens d bytes; without it that
 * backward forms dZ in place for every row). */
int icepop_workspace_bytes(const icepop_shape* shape, int64_t max_chunk_tokens, int32_t with_ref,
                           size_t* fwd_bytes, size_t* bwd_bytes);

typedef struct icepop_fwd_out {
  float* lse;          /* [n_tokens] log-sum-exp of z = H.W/T (saved for backward)      */
  double* lp_cur;      /* [n_tokens] log pi_theta(y_t)  (objective.py:223-225)           */
  float* entropy;      /* [n_tokens] -sum p log p       (objective.py:274)               */
  uint8_t* kept;       /* [n_tokens] IcePop mask        (objective.py:230-238)           */
  double* calib;       /* [n_tokens] c_t                (objective.py:227)               */
  double* surrogate;   /* [n_tokens] s_t                (objective.py:246)               */
  float* coeff;        /* [n_tokens] dJ/dlogit scale    (objective.py:250)  (for bwd)     */
  double* stats;       /* [ICEPOP_NSTATS] this rank's partial sums                        */
  /* KL-to-ref outputs (objective.py:254-263), written when weight_ref != NULL; may be NULL */
  float* kl;           /* [n_tokens] kl_t = sum_v p (log p - log p_ref)                    */
  float* lse_ref;      /* [n_tokens] log-sum-exp of z_ref = H.W_ref/T                      */
  float* kl_w;         /* [n_tokens] w_t * gamma / T (the KL gradient's coefficient)       */
  /* Stored-probabilities mode (optional; both NULL = the backward recomputes the logits):
   * probs    [n_tokens, vocab] bf16, q = 2^(u - R), u = z log2(e), with one reference R per
   *          ICEPOP_PROBS_SLAB-column vocab slab: R = 0 while the slab's maximum of u lies within
   *          +-ICEPOP_PROBS_REF_RANGE (then p = q 2^(-lse log2 e) needs one scale per row), else R
   *          = that maximum. Needs vocab % 8 == 0 and no weight_ref. 2*n_tokens*vocab bytes of
   *          HBM buy a backward without the K3 GEMM.
   * tile_max [n_tokens, ICEPOP_TILE_MAX_LD(vocab)] f32: R of slab j at column j; columns past
   *          ceil(vocab / ICEPOP_PROBS_SLAB) are padding (0). */
  void* probs;
  float* tile_max;
} icepop_fwd_out;

#define ICEPOP_PROBS_SLAB 64
#define ICEPOP_PROBS_REF_RANGE 60.0f
#define ICEPOP_TILE_MAX_LD(vocab) (4 * (((vocab) + 255) / 256))

/* Forward: fused lm_head GEMM + online log-softmax/gather/entropy (tcgen05), then the
 * IcePop epilogue. Logits are never written to HBM (only the bf16 probabilities when
 * out->probs is set). With weight_ref != NULL a second B
 * operand shares every hidden tile (dual accumulators) and kl_t enters J as -gamma*kl_t. */
int icepop_fwd_bf16(const icepop_shape* shape, const icepop_config* cfg, const void* hidden,
                    const void* weight, const void* weight_ref, const icepop_batch* batch,
                    const icepop_fwd_out* out, void* workspace, size_t workspace_bytes, void* stream);

/* The IcePop epilogue alone (K2 + the stats reduction), re-run over the K1 partials that the
 * last icepop_fwd_bf16 call left in `workspace` (same shape, same weight_ref-ness `with_ref`,
 * same temperature): other bounds, algorithm, clip epsilon or advantages without another GEMM
 * (e.g. a mask-bound sweep). Writes the same outputs as the forward except probs / tile_max. */
int icepop_fwd_epilogue_bf16(const icepop_shape* shape, const icepop_config* cfg, const icepop_batch* batch,
                             int32_t with_ref, const icepop_fwd_out* out, void* workspace, size_t workspace_bytes,
                             void* stream);

/* On-policy forward (theta == theta_old, as in the reference's own loop, scheduler.py:540-541,
 * with lp_train_old recorded by icepop_logprob_bf16 under the same weights): then
 * lp_cur == lp_train_old exactly and r == 1 (objective.py:240), so no GEMM runs -- the IcePop
 * epilogue uses the recorded lse/entropy and out->lse receives lse_old for the backward.
 * Cuts the loss step from 8.d.V to 6.d.V executed FLOPs per token. No KL-to-ref term. */
int icepop_fwd_onpolicy(const icepop_shape* shape, const icepop_config* cfg, const icepop_batch* batch,
                        const float* lse_old, const float* entropy_old, const icepop_fwd_out* out,
                        void* workspace, size_t workspace_bytes, void* stream);

/* Log-prob only (no IcePop epilogue): lse, lp = z[y]-lse, entropy. Used to record
 * lp_train_old (scheduler.py:296-311) with the same kernel. Any output may be NULL. */
int icepop_logprob_bf16(const icepop_shape* shape, double temperature, const void* hidden,
                        const void* weight, const int32_t* tokens, float* lse, double* lp,
                        float* entropy, void* workspace, size_t workspace_bytes, void* stream);

/* What the backward reads from the forward (device pointers). */
typedef struct icepop_saved {
  const int32_t* tokens;  /* [n_tokens] */
  const float* lse;       /* [n_tokens] */
  const float* coeff;     /* [n_tokens] */
  const float* lse_ref;   /* [n_tokens] KL gradient inputs: used when gamma > 0 and       */
  const float* kl;        /* [n_tokens] weight_ref != NULL, else may be NULL              */
  const float* kl_w;      /* [n_tokens]                                                   */
  void* probs;            /* out->probs / out->tile_max of the forward, or NULL. CONSUMED: the */
  const float* tile_max;  /* backward may overwrite rows of probs (a second backward passes NULL) */
  /* [n_tokens] out->lp_cur of the forward. The sampled token's term of dZ, c (1 - p_y), is
   * formed as c * -expm1(lp_cur) in fp64: with probs it enters the GEMMs as a one-hot term
   * (q_y zeroed in probs), in the recompute mode it is K3's y entry. Required with probs;
   * recommended always: forming it by cancellation, c - c p_y, loses 2^-9 p_y / (1 - p_y) of
   * it against the bf16 q_y (12% on tokens with p_y = 0.98) and the absolute precision of the
   * fp32 logits against the recomputed p_y. The forward keeps 1 - p_y to fp32 relative
   * precision in lp_cur (log1p of the probability mass of the other tokens). */
  const double* lp_cur;
} icepop_saved;

/* Backward: recompute logits tile by tile, dZ = grad_scale*coeff_t*(e_y - softmax(z_t))
 * [- grad_scale*kl_w_t*p*(log p - log p_ref - kl_t) when gamma > 0] (bf16 chunk), then
 * grad_hidden = dZ.W^T and grad_weight (+)= H^T.dZ on tcgen05. With saved->probs there is no
 * logit recompute (not with gamma > 0). Given its workspace (icepop_workspace_bytes with
 * max_chunk_tokens < 0) the backward is row-scaled: dH = s (Q.W) + c (1 - p_y) W[y] and
 * dW = Q^T.(s H) + scatter_y(c (1 - p_y) H), s = -c 2^(-lse2), c = grad_scale coeff, with
 * q_y zeroed in probs and p_y = exp(saved->lp_cur). Rows with a
 * reference R != 0 get their dZ formed in place in probs first. Blocks without an active row
 * are skipped. With a NULL or smaller workspace, dZ is formed in place for every row
 * instead; probs is consumed either way.
 * grad_hidden: [n_tokens, d], bf16 if grad_hidden_f32 == 0 else f32; may be NULL.
 * grad_weight: f32 in the weight's layout; accumulate != 0 adds into it; may be NULL. */
int icepop_bwd_bf16(const icepop_shape* shape, const icepop_config* cfg, const void* hidden,
                    const void* weight, const void* weight_ref, const icepop_saved* saved,
                    double grad_scale, void* grad_hidden, int32_t grad_hidden_f32,
                    float* grad_weight, int32_t accumulate, void* workspace, size_t workspace_bytes,
                    void* stream);

/* ---- fused dW reduce-scatter over NVLink (the step after K5) ---------------- */
/* grad_weight rows (V for ICEPOP_W_VD, d for ICEPOP_W_DV) are owned ZeRO-style: rank o owns
 * rows [o*shard_rows, (o+1)*shard_rows). slots[o] is rank o's slot buffer, peer-mapped into
 * this process (icepop_peer_import): world x shard_rows x row_len floats, row_len = d (VD) or
 * V (DV). icepop_bwd_bf16_rs is icepop_bwd_bf16 whose last K5 epilogue stores each dW row
 * (+ this rank's earlier-chunk partial, kept in grad_weight_scratch) straight into the owner's
 * slot at row rank*shard_rows + (r - o*shard_rows) -- the transfer overlaps the GEMM tile by
 * tile; the row-scaled backward then adds its one-hot part into the touched rows of those slots. After a cross-rank barrier each owner calls icepop_rs_fold on its own slot buffer:
 * out = sum over ranks in rank order (deterministic). */
typedef struct icepop_rs_target {
  int32_t world;      /* 1..8 */
  int32_t rank;
  int64_t shard_rows;
  float* slots[8];
} icepop_rs_target;

int icepop_bwd_bf16_rs(const icepop_shape* shape, const icepop_config* cfg, const void* hidden,
                       const void* weight, const void* weight_ref, const icepop_saved* saved,
                       double grad_scale, void* grad_hidden, int32_t grad_hidden_f32,
                       const icepop_rs_target* rs, float* grad_weight_scratch, void* workspace,
                       size_t workspace_bytes, void* stream);
int icepop_rs_fold(const float* slots, int32_t world, int64_t shard_elems, float* out, void* stream);

/* Peer-mapped buffers (CUDA IPC over NVLink): allocate, export a 64-byte handle, import a
 * peer's handle into this process, close / free. */
int icepop_peer_alloc(size_t bytes, void** ptr);
int icepop_peer_free(void* ptr);
int icepop_peer_export(void* ptr, void* handle64);
int icepop_peer_import(const void* handle64, void** ptr);
int icepop_peer_close(void* ptr);

/* K3 alone: dZ[t, v] = grad_scale * coeff_t * (e_{y_t} - softmax(z_t))_v for the
 * shape->n_tokens rows of `hidden`, written as bf16 to dz[t * ldz + v]. The building
 * block icepop_bwd_bf16 chains with K4/K5 (icepop_gemm_bf16); exposed so callers can
 * interleave V-slab dW reductions with it. */
int icepop_dz_bf16(const icepop_shape* shape, double temperature, const void* hidden,
                   const void* weight, const void* weight_ref, const icepop_saved* saved,
                   double grad_scale, void* dz, int64_t ldz, void* stream);

/* ---- discrepancy probe (discrepancy.py:132-161) -------------------------- */
/* kl[t] = KL(softmax(H.W_p/T)_t || softmax(H.W_q/T)_t) per row (e.g. p = the inference
 * engine's weights, q = the training weights: delta_t of Theorem 1) with the dual-accumulator
 * GEMM; *mean_kl (device) = mean over rows. Any output pointer may be NULL. Workspace: the
 * forward size of icepop_workspace_bytes(with_ref = 1). */
int icepop_kl_bf16(const icepop_shape* shape, double temperature, const void* hidden,
                   const void* weight_p, const void* weight_q, float* kl, float* lse_p, float* lse_q,
                   double* mean_kl, void* workspace, size_t workspace_bytes, void* stream);

/* delta_and_gap (discrepancy.py:132-141) against caller-supplied inference-engine logits:
 * infer_logits [n_tokens, vocab] row-major, already divided by the temperature (the
 * reference perturbs the scaled train logits, policy.py:341-347); the train logits are
 * H.W / temperature from the lm_head GEMM. Per row: kl_rows[t] = KL(p_infer || p_train),
 * gap_rows[t] = max_v |p_infer - p_train|; *delta = mean_t kl_rows, *max_gap = max_t gap_rows
 * (device scalars; any output may be NULL). fp64 arithmetic after the GEMM, fixed-order
 * reductions. n_tokens == 0 -> EINVAL (an empty probe set). Workspace:
 * icepop_delta_gap_workspace_bytes (f64 != 0 for the fp64 variant). */
int icepop_delta_gap_workspace_bytes(const icepop_shape* shape, int32_t f64, size_t* bytes);
int icepop_delta_gap_bf16(const icepop_shape* shape, double temperature, const void* hidden, const void* weight,
                          const float* infer_logits, double* kl_rows, double* gap_rows, double* delta,
                          double* max_gap, void* workspace, size_t workspace_bytes, void* stream);
int icepop_delta_gap_f64(const icepop_shape* shape, double temperature, const double* hidden, const double* weight,
                         const double* infer_logits, double* kl_rows, double* gap_rows, double* delta,
                         double* max_gap, void* workspace, size_t workspace_bytes, void* stream);

/* ---- optimizer step (objective.py:301-326) --------------------------------- */
/* Gradient ascent on an fp32 master copy: v = beta v + g (velocity != NULL) or v = g;
 * w += lr v; weight_bf16 (may be NULL) receives the bf16 copy the GEMMs read. Non-finite
 * weights set ICEPOP_ERR_NONFINITE in stats[ICEPOP_STAT_ERRORS] (stats may be NULL);
 * icepop_finish(stats) maps it to NumericError. lr <= 0 or beta outside [0,1) -> EINVAL. */
int icepop_sgd_update_f32(float* weight, const float* grad, float* velocity, void* weight_bf16,
                          int64_t n, double lr, double beta, double* stats, void* stream);

/* The reference's own fp64 ascent step, bit for bit (objective.py:301-326; numpy rounds the
 * product and the sum separately): v_out = beta velocity + grad when velocity != NULL (then
 * the step is v_out) else the step is grad; weight_out = weight + lr step. Outputs may alias
 * their inputs. Non-finite weights set ICEPOP_ERR_NONFINITE in stats (may be NULL; map with
 * icepop_finish). lr <= 0 or beta outside [0, 1) -> EINVAL. */
int icepop_sgd_update_f64(double* weight_out, const double* weight, const double* grad, const double* velocity,
                          double* velocity_out, int64_t n, double lr, double beta, double* stats, void* stream);

/* ---- diagnostics ----------------------------------------------------------------------- */
/* Number of long-K GEMM launches on the current device whose wave barriers were abandoned
 * because a unit waited longer than ICEPOP_WAVE_TIMEOUT_US (default 10000): a concurrent kernel
 * held SMs, so part of the grid started late. The result is unaffected (the barrier only keeps
 * operand slices in L2); the count says the GEMM ran without that alignment. Synchronous. */
int icepop_wave_barrier_abandons(int64_t* count);

/* ---- fp64 SIMT validation path ----------------------------------------------------- */
/* Same semantics in fp64 on CUDA cores (still CUDA, no CPU fallback), so the
 * reference's exact-identity and finite-difference tests run unchanged on the GPU.
 * Supports the KL-to-ref term (objective.py:254-263) when weight_ref != NULL.
 * hidden [n_tokens, d] f64; weight / weight_ref f64 in `weight_layout`. */
int icepop_workspace_bytes_f64(const icepop_shape* shape, int32_t with_ref, size_t* bytes);

typedef struct icepop_f64_out {
  double* lse;         /* [n_tokens]                                                     */
  double* lp_cur;      /* [n_tokens]                                                     */
  double* entropy;     /* [n_tokens]                                                     */
  double* kl;          /* [n_tokens] kl_t (0 when weight_ref == NULL)                    */
  double* lse_ref;     /* [n_tokens] (written when weight_ref != NULL)                   */
  uint8_t* kept;
  double* calib;
  double* surrogate;
  double* coeff;       /* [n_tokens] objective.py:250                                   */
  double* stats;       /* [ICEPOP_NSTATS]                                                */
} icepop_f64_out;

int icepop_fwd_f64(const icepop_shape* shape, const icepop_config* cfg, const double* hidden,
                   const double* weight, const double* weight_ref, const icepop_batch* batch,
                   const icepop_f64_out* out, void* workspace, size_t workspace_bytes, void* stream);

/* grad_hidden [n_tokens,d] f64 (may be NULL); grad_weight f64 in weight layout (may be NULL).
 * kl/lse_ref/coeff/lse come from icepop_fwd_f64. */
int icepop_bwd_f64(const icepop_shape* shape, const icepop_config* cfg, const double* hidden,
                   const double* weight, const double* weight_ref, const icepop_batch* batch,
                   const icepop_f64_out* fwd, double grad_scale, double* grad_hidden,
                   double* grad_weight, int32_t accumulate, void* workspace,
                   size_t workspace_bytes, void* stream);

/* ---- completion --------------------------------------------------------------------- */
/* Synchronises `stream` once, reads stats[ICEPOP_STAT_ERRORS] and maps it to
 * ICEPOP_ENUMERIC with the reference's message; `stats` may be a host or device pointer
 * to the (already all-reduced) statistics vector. */
int icepop_finish(const double* stats, void* stream);

/* ---- building blocks exposed for tests / benchmarks --------------------------------- */
/* C[M,N] = A.B with bf16 operands on tcgen05, f32 accumulate, f32 or bf16 output.
 * a_mn_major: A stored [K,M] (M contiguous) instead of [M,K]; b_mn_major: B stored
 * [K,N] instead of [N,K]. ldc in elements. accumulate adds into C (f32 only). */
int icepop_gemm_bf16(const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K,
                     int32_t a_mn_major, int32_t b_mn_major, int32_t c_f32, int32_t accumulate,
                     void* stream);

/* Tile configuration of the tcgen05 GEMMs: 2 (default) = CTA pairs with cta_group::2
 * MMAs on 256 x 256 tiles, 1 = single-CTA 128 x 256 tiles. Process-wide; the
 * ICEPOP_CTA_GROUP environment variable sets the initial value. */
int icepop_set_cta_group(int32_t cta_group);

/* Tile shape of the long-K plain GEMMs (K4, K5) on CTA pairs: 1 (default) = 256 x 512 tiles
 * (two N = 256 MMAs per k step into one TMEM accumulator) unless the output is too small to
 * fill the GPU with them (then 256 x 256), 2 = 256 x 512 always, 0 = 256 x 256 always.
 * Process-wide; the ICEPOP_WIDE_TILES environment variable sets the initial value. */
int icepop_set_wide_tiles(int32_t enable);

/* Tile shape of K1 (the forward GEMM with the softmax epilogue) on CTA pairs: 0 (default) =
 * 256 x 256 with a double-buffered TMEM accumulator, 1 = 256 x 512 with one accumulator whose
 * halves are released separately (a quarter fewer operand bytes; measured equal on B200).
 * The stored probabilities and slab references are the same bits either way; the statistics
 * differ only by the summation grouping. Process-wide; ICEPOP_K1_WIDE sets the initial value. */
int icepop_set_k1_wide(int32_t enable);

/* K1 run length: the consecutive vocabulary tiles one CTA pair processes for one block of
 * tokens, merging the softmax statistics in registers and writing one partial per run (K2
 * merges ceil(V / (256 run)) partials per token instead of ceil(V / 256)). 0 (default) =
 * automatic (16, shorter when the problem has too few tiles to keep every pair busy), else 1..64.
 * Process-wide; ICEPOP_K1_RUN sets the initial value. */
int icepop_set_k1_run(int32_t run);

/* Backward row skipping: rows whose gradient coefficient is exactly zero (popped tokens,
 * clip-inactive tokens, zero-advantage sequences; objective.py:250) contribute nothing to
 * dW and get dHidden = 0, so icepop_bwd_bf16 compacts the active rows on the device and
 * runs K3-K5 on them only (1 = default; ICEPOP_SKIP_INACTIVE=0 sets the initial value 0). */
int icepop_set_skip_inactive(int32_t enable);

#ifdef __cplusplus
}
#endif
#endif /* ICEPOP_B200_H_ */
