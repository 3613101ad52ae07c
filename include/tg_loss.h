/*
 * tg_loss.h -- C ABI of the B200-native RFT trainer loss path ("tg" = task group).
 *
 * Drop-in boundary for Trinity-RFT's (reference: `triad`) trainer loss path:
 *
 *   reference entry point (file:line under /root/reference/pkg/src/triad)   replaced by
 *   ----------------------------------------------------------------------  ---------------------
 *   algorithms.group_loss           algorithms.py:351-365                  tg_loss_fwd_bwd
 *     loss_opmd_simple              algorithms.py:220-253   (GRPO analogue) TG_PG_VANILLA + TG_ADV_OPMD
 *     loss_opmd_kimi                algorithms.py:118-153                   TG_PG_OPMD_KIMI
 *     loss_opmd_pairwise            algorithms.py:156-190                   TG_PG_OPMD_PAIRWISE
 *     regularizer_g (anchor KL)     algorithms.py:193-217                   TgConfig.anchor_beta
 *   algorithms.loss_sft             algorithms.py:256-274                   TG_PG_SFT / seq_kind = 1
 *   algorithms.loss_dpo             algorithms.py:277-315                   TG_PG_DPO
 *   algorithms.combine_reports      algorithms.py:368-379                   stats[] (sums + group count)
 *   algorithms.experience_logprob   algorithms.py:81-85                     tg_logprob_fwd
 *   (hidden states, no logits)      policy.py:194-212 behind an LM head     tg_lmhead_logprob_fwd
 *   policy.logprob / grad_logprob   policy.py:194-212, 253-270              (fused into both)
 *   policy.scored_states            policy.py:181-191 (toy-table adapter)   tg_scored_states (host)
 *   ExperienceBuffer.sample_batch   buffer.py:240-264 (group indexing)      tg_group_by_task (host)
 *   algorithms.apply_update         algorithms.py:329-348 (SGD step)        tg_apply_update
 *   (LLM-scale optimizer step)      SURVEY.md 8f rank 4 (fused AdamW)        tg_adamw_step
 *
 * plus the north_star registry pieces the reference does not have (GRPO std
 * advantage, RLOO, PPO clip / dual clip, k1/k2/k3(low_var_kl)/abs KL,
 * entropy bonus, token / sequence aggregation modes).
 *
 * Conventions
 *  - Plain pointers + sizes; all array pointers in TgBatch / TgOut are DEVICE
 *    pointers (cudaMalloc / torch CUDA tensors).  `stream` is a cudaStream_t
 *    passed as void*.  Calls are stream-ordered and never synchronise the host.
 *  - The library never allocates device memory: the caller provides a
 *    workspace of tg_workspace_size() bytes (256-byte aligned).
 *  - Row t of `logits` scores `target[t]` (the host does the HF shift and drops
 *    mask-false positions).  Rows of one sequence are contiguous; sequences of
 *    one group are contiguous (seq_offsets / group_offsets are prefix sums).
 *  - dlogits = d loss / d logits, written once per element; it MAY alias
 *    `logits` (in place) when ld_out == ld and row_index == NULL.
 *  - Errors: every entry point returns TG_OK or a TG_E* code; tg_last_error()
 *    gives a message for the calling thread.  Data-dependent problems found on
 *    the device (target outside [0, V), non-finite loss/gradient, pairwise
 *    group of size < 2, DPO group of size != 2) are reported as counts in
 *    stats[TG_S_INVALID] and stats[TG_S_NONFINITE]; the Python layer raises
 *    AlgorithmError for them exactly where LossReport.__post_init__
 *    (algorithms.py:65-69) or policy._check_generated_tokens (policy.py:175-178)
 *    would have raised.
 */
#ifndef TG_LOSS_H_
#define TG_LOSS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TG_ABI_VERSION 5

/* return codes */
enum { TG_OK = 0, TG_EINVAL = 1, TG_ECUDA = 2, TG_EUNSUPPORTED = 3, TG_EWORKSPACE = 4 };

/* element type of logits / anchor_logits / dlogits (arithmetic is fp32) */
enum { TG_DTYPE_BF16 = 0, TG_DTYPE_F32 = 1 };

/* advantage_fn registry */
enum {
  TG_ADV_GIVEN = 0,     /* use TgBatch.advantage[seq]                                 */
  TG_ADV_GRPO = 1,      /* (r - mean_g) / (std_g(unbiased) + std_eps); K = 1 -> 0     */
  TG_ADV_RLOO = 2,      /* r_i - mean_{j != i} r_j; K = 1 -> 0                         */
  TG_ADV_OPMD = 3,      /* (r - mean_g) / (1 + tau)      algorithms.py:234-242         */
  TG_ADV_REINFORCE = 4  /* r                                                           */
};

/* policy_loss_fn registry */
enum {
  TG_PG_VANILLA = 0,        /* -A * lp                           (OPMD_SIMPLE form)     */
  TG_PG_PPO_CLIP = 1,       /* max(-A rho, -A clip(rho)) [dual clip c]                   */
  TG_PG_SFT = 2,            /* -lp (NLL)                          algorithms.py:256-274  */
  TG_PG_OPMD_KIMI = 3,      /* sum_i (r_i - zeta - tau(LP_i - ref_i))^2   :118-153       */
  TG_PG_OPMD_PAIRWISE = 4,  /* sum_{i<j} (a_i - a_j)^2                    :156-190       */
  TG_PG_DPO = 5,            /* mean softplus(-beta margin); groups are (chosen, rejected) */
  TG_PG_GIVEN = 6           /* caller-supplied per-row policy loss l_t (TgBatch.pg_loss) and
                               coefficient -d l_t / d lp_t (TgBatch.pg_coef): a policy loss
                               registered from Python, evaluated on the rows' lp before the
                               call; weighted by the aggregation weight like the built-ins,
                               token KL / entropy / SFT rows / anchor KL unchanged      */
};
/* The sequence-coupled losses (OPMD_KIMI, OPMD_PAIRWISE, DPO) are whole-sequence
   objectives: with them kl_fn / kl_coef, the entropy bonus, a loss_agg_mode other
   than TG_AGG_SEQ_SUM and a seq_kind array (SFT rows) are refused with TG_EINVAL
   instead of being silently dropped.  The anchor KL (anchor_beta) is allowed. */

/* kl_fn registry: token-level penalty kl_coef * kl(lp, ref_lp) */
enum { TG_KL_NONE = 0, TG_KL_K1 = 1, TG_KL_K2 = 2, TG_KL_K3 = 3 /* low_var_kl */, TG_KL_ABS = 4 };

/* entropy_loss_fn registry: loss -= entropy_coef * agg(H) */
enum { TG_ENT_NONE = 0, TG_ENT_DEFAULT = 1 };

/* loss_agg_mode registry: per-row weight w of RL rows */
enum {
  TG_AGG_SEQ_SUM = 0,                 /* w = 1 (the reference's semantics)             */
  TG_AGG_TOKEN_MEAN = 1,              /* w = 1 / N_tok(RL, global)                     */
  TG_AGG_SEQ_MEAN_TOKEN_SUM = 2,      /* w = 1 / B(RL, global)                         */
  TG_AGG_SEQ_MEAN_TOKEN_MEAN = 3,     /* w = 1 / (B * n_i)                             */
  TG_AGG_SEQ_MEAN_TOKEN_SUM_NORM = 4  /* w = 1 / agg_norm                              */
};

/* flags */
enum {
  TG_FLAG_FORCE_TWO_PASS = 1,  /* use the forward + backward streaming kernels even when
                                  the fused single-pass kernel applies (testing / A-B)  */
  TG_FLAG_NO_FUSED_TMA = 2,    /* alias kept for clarity: same effect                   */
  TG_FLAG_ROWS_GIVEN = 4,      /* forward-only loss from precomputed per-row values: out.lp,
                                  out.entropy, out.lse are INPUTS (e.g. from
                                  tg_lmhead_logprob_fwd); no logits are read (batch.logits
                                  may be NULL) and out.dlogits must be NULL               */
  TG_FLAG_UNSCALED_GRAD = 8    /* sequence-coupled losses (OPMD_KIMI / OPMD_PAIRWISE / DPO)
                                  in ONE pass over the logits (4V bytes per row instead
                                  of 6V): out.dlogits receives the unscaled p - e_y and
                                  out.row_coef (required) the per-row scale s_t in its
                                  third block, d loss / d z_t = s_t (p_t - e_y) -- the
                                  caller folds diag(s) into its LM-head backward
                                  (d hidden rows and the hidden rows of d W scale by s_t;
                                  SURVEY.md 7, hard part 3).  No anchor KL.  Layouts
                                  the single pass cannot take (unaligned pitch, forced
                                  two-pass) give the same outputs over two passes.   */
};

/* stats[] layout (double).  Sums are over this call's rows / groups; the
   caller allreduces (sum) across ranks, then divides by n_groups for the
   reference's averaged metrics (algorithms.py:377-378). */
enum {
  TG_S_LOSS = 0, TG_S_PG_LOSS, TG_S_KL_LOSS, TG_S_ENTROPY_LOSS, TG_S_ANCHOR_LOSS, TG_S_SFT_LOSS,
  TG_S_N_GROUPS, TG_S_SUM_MEAN_REWARD, TG_S_SUM_BASELINE, TG_S_SUM_KL_ESTIMATE, TG_S_SUM_GROUP_SIZE,
  TG_S_N_TOK, TG_S_N_TOK_RL, TG_S_CLIP_COUNT, TG_S_SUM_ENTROPY, TG_S_SUM_KL, TG_S_SUM_PPO_KL,
  TG_S_SUM_LP, TG_S_NONFINITE, TG_S_N_SEQS, TG_S_SUM_ADV, TG_S_SUM_RATIO, TG_S_N_SFT_SEQS,
  TG_S_SUM_SFT_REWARD, TG_S_SUM_DPO_MARGIN, TG_S_DUAL_CLIP_COUNT, TG_S_SUM_ANCHOR_KL,
  TG_S_INVALID, TG_S_RESERVED28, TG_S_RESERVED29, TG_S_RESERVED30, TG_S_RESERVED31,
  TG_NSTAT = 32
};

typedef struct TgConfig {
  int32_t advantage_fn;     /* TG_ADV_*  */
  int32_t policy_loss_fn;   /* TG_PG_*   */
  int32_t kl_fn;            /* TG_KL_*   */
  int32_t entropy_loss_fn;  /* TG_ENT_*  */
  int32_t loss_agg_mode;    /* TG_AGG_*  */
  int32_t flags;            /* TG_FLAG_* */
  double tau;               /* OPMD temperature (>= 0; > 0 for KIMI / PAIRWISE)   */
  double clip_lo, clip_hi;  /* PPO ratio clip range [1 - clip_lo, 1 + clip_hi]    */
  double clip_c;            /* dual-clip constant (> 1), 0 = off                  */
  double kl_coef;           /* token KL penalty coefficient                       */
  double entropy_coef;      /* entropy bonus coefficient                          */
  double std_eps;           /* GRPO std epsilon                                   */
  double sft_weight;        /* weight of SFT (seq_kind = 1) rows: w = sft_weight / n_sft */
  double anchor_beta;       /* beta of regularizer_g (needs anchor_logits)        */
  double dpo_beta;          /* DPO beta (> 0)                                     */
  double agg_norm;          /* divisor of TG_AGG_SEQ_MEAN_TOKEN_SUM_NORM          */
  int64_t n_tok_global;     /* RL rows over all ranks (token-mean); 0 = this call's */
  int64_t n_seq_global;     /* RL sequences over all ranks; 0 = this call's         */
  int64_t n_sft_seq_global; /* SFT sequences over all ranks; 0 = this call's        */
} TgConfig;

typedef struct TgBatch {
  int32_t dtype;                 /* TG_DTYPE_*                                           */
  int32_t n_seqs;                /* B                                                    */
  int32_t n_groups;              /* G                                                    */
  int32_t reserved0;
  int64_t n_rows;                /* T (trainable rows)                                   */
  int64_t vocab;                 /* V                                                    */
  int64_t ld;                    /* row pitch of logits, in elements (>= V)              */
  const void* logits;            /* [*, ld]                                              */
  const int64_t* row_index;      /* optional [T]: row t reads logits row row_index[t]    */
  const void* anchor_logits;     /* optional [T, ld_anchor] (same dtype)                 */
  int64_t ld_anchor;
  const int32_t* target;         /* [T] token scored by row t                            */
  const float* old_lp;           /* optional [T] behaviour logprob (PPO ratio, KL metric)*/
  const float* ref_lp;           /* optional [T] reference-policy logprob (token KL)     */
  const int32_t* seq_offsets;    /* [B+1] row prefix sums                                */
  const int32_t* group_offsets;  /* [G+1] sequence prefix sums                           */
  const float* reward;           /* [B]                                                  */
  const float* seq_ref_lp;       /* optional [B] sequence reference logprob (OPMD / DPO);
                                    default = sum of old_lp over the sequence
                                    (records.py:119-121)                                 */
  const float* advantage;        /* [B] for TG_ADV_GIVEN                                 */
  const uint8_t* seq_kind;       /* optional [B]: 0 RL rollout, 1 SFT / expert           */
  const float* pg_coef;          /* [T] for TG_PG_GIVEN: -d l_t / d lp_t (unweighted)     */
  const float* pg_loss;          /* [T] for TG_PG_GIVEN: l_t (unweighted)                 */
} TgBatch;

typedef struct TgOut {
  void* dlogits;     /* [T, ld_out] d loss / d logits, or NULL (forward only)   */
  int64_t ld_out;
  float* lp;         /* optional [T] current-policy logprob of target          */
  float* entropy;    /* optional [T] H_t                                        */
  float* lse;        /* optional [T] log-sum-exp                                */
  float* seq_lp;     /* optional [B] sum of lp over each sequence               */
  float* seq_adv;    /* optional [B] advantage (or coupled coefficient)         */
  double* stats;     /* [TG_NSTAT] device, required                             */
  float* row_coef;   /* optional [3, T] per-row gradient coefficients (a, hz, s):
                        d loss / d z_tv = p_tv (a_t + hz_t z_tv) - s_t [v = y_t],
                        p = exp(z - lse).  Requesting them selects the two-pass
                        route (the fused kernel keeps them on chip); with
                        TG_FLAG_ROWS_GIVEN they feed tg_lmhead_dlogits.        */
} TgOut;

/* Workspace bytes needed by tg_loss_fwd_bwd / tg_logprob_fwd for this batch. */
size_t tg_workspace_size(const TgBatch* batch, const TgConfig* cfg);

/* Loss + gradient.  Replaces group_loss over a batch of groups followed by
   combine_reports (orchestrator.py:299-308, without apply_update). */
int tg_loss_fwd_bwd(const TgBatch* batch, const TgConfig* cfg, TgOut* out,
                    void* workspace, size_t workspace_bytes, void* stream);

/* Forward-only logprob / entropy / lse (+ seq_lp) -- experience_logprob
   (algorithms.py:81-85) for old / ref logprob recompute.  stats may be NULL. */
int tg_logprob_fwd(const TgBatch* batch, TgOut* out, void* workspace,
                   size_t workspace_bytes, void* stream);

/* Fused LM-head + log-softmax forward on the tensor cores:
   z = hidden [n_rows, dim] x weight [vocab, dim]^T (bf16, row-major, pitches
   ld_hidden / ld_weight elements, multiples of 8; dim a multiple of 64) is
   folded tile by tile into per-row lse / entropy and lp = z[target] - lse
   without writing the logits.  Replaces policy.logprob (policy.py:194-212)
   when the caller holds hidden states instead of logits.  lp / target may be
   NULL (entropy / lse only).  fp32 accumulation.  When the row blocks alone
   cannot fill the SMs the vocabulary is split across CTAs and merged in a
   fixed order: the workspace (tg_lmhead_workspace_size bytes, 16-byte
   aligned; 0 bytes for large n_rows) holds the per-split partials. */
size_t tg_lmhead_workspace_size(int64_t n_rows, int64_t vocab);
int tg_lmhead_logprob_fwd(const void* hidden, int64_t ld_hidden, const void* weight,
                          int64_t ld_weight, int64_t n_rows, int64_t vocab, int64_t dim,
                          const int32_t* target, float* lp, float* entropy, float* lse,
                          void* workspace, size_t workspace_bytes, void* stream);

/* Backward half of the fused LM head (vocabulary chunked):
   recomputes z = hidden x weight[col0 : col0 + n_cols]^T on the tensor cores
   and writes, for every row t and chunk column j (v = col0 + j),
       dz[t, j] = exp(z_tv - lse_t) * (a_t + hz_t * z_tv) - s_t * [v == target_t]
   in bf16 to dz [n_rows, ld_dz] (ld_dz >= n_cols, a multiple of 8) -- the
   d loss / d logits of one vocabulary chunk, from the row coefficients
   TgOut.row_coef (a = row_coef[0:T], hz = [T:2T], s = [2T:3T]) and lse of the
   forward.  The caller turns each chunk into d hidden += dz . W_chunk and
   d W_chunk = dz^T . hidden (plain GEMMs), so the [T, V] logits never exist:
   peak memory is T x n_cols.  Replaces policy.grad_logprob (policy.py:253-270)
   behind an LM head.  Same size rules as tg_lmhead_logprob_fwd. */
int tg_lmhead_dlogits(const void* hidden, int64_t ld_hidden, const void* weight,
                      int64_t ld_weight, int64_t n_rows, int64_t vocab, int64_t dim,
                      int64_t col0, int64_t n_cols, const int32_t* target, const float* lse,
                      const float* row_coef, void* dz, int64_t ld_dz, void* stream);

/* The two gradient GEMMs of one vocabulary chunk, on the tensor cores (no
   cuBLAS): dz [n_rows, ld_dz] bf16 is the chunk written by tg_lmhead_dlogits.
     tg_lmhead_grad_hidden:  d_hidden [n_rows, ld_dh] fp32 (+)= dz . weight[col0 : col0 + n_cols]
                             (accumulate != 0 adds to d_hidden -- the chunks of one
                             step -- else overwrites it)
     tg_lmhead_grad_weight:  d_weight [n_cols, ld_dw] bf16 = dz^T . hidden
                             (the chunk's rows of d W; pass d_weight + col0 * ld_dw)
   fp32 accumulation over the whole chunk / all rows.  Together with
   tg_lmhead_logprob_fwd and tg_lmhead_dlogits they are the RFT loss's
   backward through an LM head: the SparseGrad.add_row / apply_update
   analogue (policy.py:215-250, algorithms.py:329-348) for a dense head.  Size
   rules as tg_lmhead_logprob_fwd; ld_dh a multiple of 4, ld_dw of 8, all
   pointers 16-byte aligned. */
int tg_lmhead_grad_hidden(const void* dz, int64_t ld_dz, const void* weight, int64_t ld_weight,
                          int64_t n_rows, int64_t vocab, int64_t dim, int64_t col0,
                          int64_t n_cols, float* d_hidden, int64_t ld_dh, int accumulate,
                          void* stream);
int tg_lmhead_grad_weight(const void* dz, int64_t ld_dz, const void* hidden, int64_t ld_hidden,
                          int64_t n_rows, int64_t dim, int64_t n_cols, void* d_weight,
                          int64_t ld_dw, void* stream);
/* Both GEMMs of one chunk in one launch (one tile queue over the two
   outputs, so neither GEMM's partial last wave leaves SMs idle); the same
   arguments and results as the two calls above. */
int tg_lmhead_grad_chunk(const void* dz, int64_t ld_dz, const void* hidden, int64_t ld_hidden,
                         const void* weight, int64_t ld_weight, int64_t n_rows, int64_t vocab,
                         int64_t dim, int64_t col0, int64_t n_cols, float* d_hidden,
                         int64_t ld_dh, int accumulate, void* d_weight, int64_t ld_dw,
                         void* stream);

/* Optimizer step: algorithms.apply_update (algorithms.py:329-348) on the
   device.  table [n_states, ld_table] fp32 (updated in place) gets
   table[s] -= learning_rate * sum of the gradient rows of state s, where the
   gradient rows are dlogits rows [*, ld_grad] (dtype TG_DTYPE_*) grouped by
   state in CSR form: state_ids[n_touched], state_offsets[n_touched + 1] into
   row_order[n_rows] (rows in row order within a state).  Per-state sums are
   f64 in row order (deterministic).  *status (device int32) becomes 0, or 1
   when any gradient element is non-finite, 2 when a state is outside
   [0, n_states) -- and then nothing is written (the reference refuses
   before it updates).  Stream-ordered; the caller reads status when it syncs. */
int tg_apply_update(float* table, int64_t ld_table, int64_t n_states, int64_t vocab,
                    const void* grad, int dtype, int64_t ld_grad, const int64_t* state_ids,
                    const int64_t* state_offsets, const int64_t* row_order, int64_t n_touched,
                    int64_t n_rows, double learning_rate, int32_t* status, void* stream);

/* Fused AdamW step of a [rows, cols] parameter block -- the LM head after its
   backward GEMMs ("LM-head backward GEMM plus a fused
   AdamW"; the LLM-scale counterpart of algorithms.apply_update,
   algorithms.py:329-348).  torch.optim.AdamW semantics, decoupled weight decay,
   step = the 1-based step count t:
     exp_avg    = exp_avg + (1 - beta1) (grad - exp_avg)
     exp_avg_sq = beta2 exp_avg_sq + (1 - beta2) grad^2
     param      = param (1 - lr wd) - lr / (1 - beta1^t) * exp_avg /
                  (sqrt(exp_avg_sq) / sqrt(1 - beta2^t) + eps)
   param (bf16 or fp32, row pitch ld_param) and grad (bf16 or fp32, row pitch
   ld_grad) are device arrays; exp_avg / exp_avg_sq fp32 [rows, cols]
   contiguous.  One HBM pass (22 bytes per bf16 parameter).  With `status`
   non-NULL a read-only pass over grad runs first and a non-finite element sets
   *status = 1 and leaves param and both moments untouched (apply_update's
   refusal, algorithms.py:337-338); status may be NULL to skip the check. */
int tg_adamw_step(void* param, int param_dtype, int64_t ld_param, const void* grad,
                  int grad_dtype, int64_t ld_grad, float* exp_avg, float* exp_avg_sq,
                  int64_t rows, int64_t cols, double lr, double beta1, double beta2, double eps,
                  double weight_decay, int64_t step, int32_t* status, void* stream);

/* Which kernel route tg_loss_fwd_bwd takes for this input: 1 = fused single
   pass (4V bytes/row; 6V with the anchor KL of regularizer_g, whose anchor
   rows ride the same pass), 2 = forward + backward streaming (6V; 10V with
   the anchor), 3 = coupled (6V), 4 = coupled with TG_FLAG_UNSCALED_GRAD
   (single pass, 4V). */
int tg_route(const TgBatch* batch, const TgConfig* cfg);

/* Thread-block cluster size of the fused single-pass kernel (k_fused_tma<T, CL>)
   that tg_loss_fwd_bwd launches for this input on the current device (routes 1
   and 4), or 0 when the call takes a streaming route.  Introspection only. */
int tg_fused_cluster_size(const TgBatch* batch, const TgConfig* cfg);

/* Timing hook (measurement only): when both are non-NULL cudaEvent_t handles,
   the next tg_loss_fwd_bwd call on this thread records ev_begin on its stream
   before its first kernel and ev_end after its last one (the whole call: the
   group prologue, the row kernels and the tail -- an event between kernels
   chained by programmatic dependent launch would serialise them).  The hook
   is consumed by that call. */
int tg_set_timing_events(void* ev_begin, void* ev_end);

/* Total CUDA kernel launches issued by this library in this process. */
int64_t tg_launch_count(void);

const char* tg_strerror(int code);
const char* tg_last_error(void);
int tg_abi_version(void);

/* ---- on-device packer ----------------------------------------------------- */

/* Padded token batch -> packed rows, on the device.
   mask[B*L] marks trainable TARGET positions; row r for target position
   (b, l), l >= 1, gets row_index[r] = b*L + l - 1 (HF shift into the
   [B*L, V] logits), target[r] = ids[b*L + l] and, when the dense inputs are
   given, old_out[r] / ref_out[r] from old_dense / ref_dense[b*L + l].  Rows
   keep (b, l) order; seq_offsets[B+1] and *n_rows (device int64) are written.
   Rows beyond `capacity` are counted but not written.  Workspace: 4*B bytes.
   Replaces the per-token Python assembly of Experience / TaskGroup records
   (records.py:21-131, workflows.py:128-183). */
int tg_pack_rows(const uint8_t* mask, const void* ids, int ids_is_int64, int32_t B, int32_t L,
                 const float* old_dense, const float* ref_dense, int64_t* row_index,
                 int32_t* target, float* old_out, float* ref_out, int64_t capacity,
                 int32_t* seq_offsets, int64_t* n_rows, void* workspace,
                 size_t workspace_bytes, void* stream);

/* ---- host helpers (no device access) ------------------------------------ */

/* Toy-table policy adapter (policy.py:152-161, 181-191; encoding.py:19-35):
   for each experience e (tokens[tok_off[e]:tok_off[e+1]], mask likewise,
   prompt length prompt_len[e]) write the bucket state and target token of
   every mask-true position, in order.  Returns the number of rows written
   (must equal the caller's capacity check) or -1 on error. */
int64_t tg_scored_states(const int64_t* tokens, const uint8_t* mask, const int64_t* tok_off,
                         const int64_t* prompt_len, int64_t n_exp, int64_t num_buckets,
                         int64_t* states_out, int32_t* target_out, int64_t capacity);

/* ExperienceBuffer.sample_batch(group_by_task=True) group indexing
   (buffer.py:240-264) over READY experiences given in insertion order:
   policy 0 = FIFO, 1 = PRIORITY (descending priority, ties by sample_id rank
   given in `id_rank`).  Writes up to n_take groups of group_size indices into
   groups_out and returns the number of groups. */
int64_t tg_group_by_task(const int64_t* task_key, const double* priority,
                         const int64_t* id_rank, const uint8_t* ready, int64_t n,
                         int64_t group_size, int64_t n_take, int32_t policy,
                         int64_t* groups_out);

#ifdef __cplusplus
}
#endif
#endif /* TG_LOSS_H_ */
