/*
 * ckrl.h — C ABI of the B200-native rollout -> advantage -> loss hot path.
 *
 * Drop-in boundary for the chunkrl reference (/root/reference/proj/src/chunkrl).
 * The reference exposes plain C++20 free functions over an AoS TrajectorySlab;
 * this ABI exposes the same operators over a caller-owned structure-of-arrays
 * slab in device memory (HBM), with explicit cudaStream_t, caller-provided
 * workspace (no allocation on the hot call) and status codes 1:1 with the
 * reference's exception types. Each entry point cites the reference interface
 * it replaces. There is no CPU fallback: every compute entry point launches
 * sm_100a kernels and fails with CKRL_ERR_CUDA when no device is usable.
 *
 * SoA slab layout (row-major, innermost last):
 *   record r = e*Tc + t      slot s = r*C + j      token k = s*M + m
 *   tokens       [E][Tc][C][M]      u8 (V <= 256) or i32
 *   old_logprob  [E][Tc][C][M]      f32   (TokenLogprobs, core/types.hpp:29-38)
 *   reward       [E][Tc][C]         f32
 *   flags        [E][Tc][C]         u8    bit0 terminated, bit1 truncated, bit2 valid
 *   episode_id   [E][Tc][C]         i32   uid & 0xffffffff (envsim/vec_env.cpp:14-16), -1 frozen
 *   value_scalar [E][Tc]            f32   StepRecord::value_scalar
 *   value_vector [E][Tc][C]         f32   StepRecord::value_vector
 *   bootstrap    [E][Tc][C]         f32   V_snapshot(post_obs[slot]) of the advantage-level
 *                                         head (scalar at chunk level, vector[0] at action
 *                                         level; assembler.cpp:114-118, 148-152)
 *   logits       [E][Tc][C][M][V]   f32 or bf16, current policy (forward_logits)
 *   new values   [E][Tc] (chunk value level) or [E][Tc][C] (action value level), f32
 */
#ifndef CKRL_H
#define CKRL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef struct CUstream_st* ckrl_stream_t; /* == cudaStream_t */

/* Status codes, 1:1 with chunkrl/core/errors.hpp:9-48 (+ CUDA / argument errors). */
typedef enum {
  CKRL_OK = 0,
  CKRL_ERR_UNSUPPORTED_COMBINATION = 1,  /* UnsupportedCombination */
  CKRL_ERR_GRANULARITY_ORDER = 2,        /* GranularityOrderViolation */
  CKRL_ERR_LENGTH_MISMATCH = 3,          /* LengthMismatch */
  CKRL_ERR_BAD_RESET_ID = 4,             /* BadResetId */
  CKRL_ERR_HEAD_MISMATCH = 5,            /* HeadMismatch */
  CKRL_ERR_NON_FINITE = 6,               /* NonFinite */
  CKRL_ERR_DEGENERATE_GROUP = 7,         /* DegenerateGroup */
  CKRL_ERR_SKIP_UPDATE = 8,              /* SkipUpdate */
  CKRL_ERR_INVALID_PLAN = 9,             /* InvalidPlan */
  CKRL_ERR_MEMORY_OVERFLOW = 10,         /* MemoryOverflow */
  CKRL_ERR_EMPTY_TRACE = 11,             /* EmptyTrace */
  CKRL_ERR_CONFIG = 12,                  /* ConfigError */
  CKRL_ERR_GENERIC = 13,                 /* chunkrl::Error */
  CKRL_ERR_CUDA = 14,                    /* device / launch failure */
  CKRL_ERR_INVALID_ARGUMENT = 15,        /* null pointer, bad dims, workspace too small */
  CKRL_ERR_NCCL = 16
} ckrl_status;

/* core/granularity.hpp:8 enum class Level { Chunk, Action, Token } */
enum { CKRL_LEVEL_CHUNK = 0, CKRL_LEVEL_ACTION = 1, CKRL_LEVEL_TOKEN = 2 };
enum { CKRL_DTYPE_F32 = 0, CKRL_DTYPE_BF16 = 1, CKRL_DTYPE_U8 = 2, CKRL_DTYPE_I32 = 3, CKRL_DTYPE_F64 = 4,
       CKRL_DTYPE_TOKEN_ROWS = 5 /* ckrl_token_row per position (ckrl_project_token_stats) */ };

/* One position's finished token statistics: the sampled token's log-prob (fp64) and the
 * entropy of the position's distribution (evaluate_chunk's token_logprobs / entropy,
 * policy/policy_net.cpp:333-357). Written by ckrl_project_token_stats; consumed by the losses
 * in place of logits when ckrl_policy_outputs.logits_dtype == CKRL_DTYPE_TOKEN_ROWS. */
typedef struct {
  double logprob;
  float entropy;
  uint32_t reserved; /* 0 */
} ckrl_token_row;

/* Communicator of a multi-rank job: peer-memory exchange buffers (+ optional NCCL), below. */
typedef struct ckrl_comm ckrl_comm;
enum { CKRL_FLAG_TERMINATED = 1, CKRL_FLAG_TRUNCATED = 2, CKRL_FLAG_VALID = 4 };

/* Diagnostics slots written to device memory (optim/losses.hpp:31-39 LossDiagnostics). */
enum {
  CKRL_DIAG_LOSS = 0, CKRL_DIAG_SURROGATE, CKRL_DIAG_VALUE_LOSS, CKRL_DIAG_ENTROPY,
  CKRL_DIAG_CLIP_FRAC, CKRL_DIAG_APPROX_KL, CKRL_DIAG_UNITS, CKRL_DIAG_STATUS,
  CKRL_DIAG_COUNT = 8
};

typedef struct {
  int32_t advantage_level, logprob_level, value_level;
} ckrl_granularity; /* GranularitySpec, core/granularity.hpp:21-27 */

typedef struct {
  double gamma, lambda;
} ckrl_gae_params; /* advantage/gae.hpp:8-13 */

typedef struct {
  double clip_eps, value_loss_coef, entropy_coef;
  int32_t advantage_normalization; /* applied once before the loss (optim/update.cpp:66-67) */
} ckrl_ppo_params; /* optim/losses.hpp:12-21 (optimizer fields are out of scope) */

typedef struct {
  double clip_eps;
} ckrl_grpo_params; /* optim/losses.hpp:23-29 */

typedef struct {
  double eps_std;
  int32_t apply_filter;
  double filter_lower, filter_upper;
  int32_t length_normalized;
  int32_t min_group_size;
} ckrl_grpo_options; /* advantage/assembler.hpp:76-83 */

/* The SoA rollout buffer (replaces TrajectorySlab, core/types.hpp:89-104). Device pointers. */
typedef struct {
  int32_t num_envs, num_chunks, chunk_len, tokens_per_action, vocab;
  int32_t token_dtype; /* CKRL_DTYPE_U8 | CKRL_DTYPE_I32 */
  const void* tokens;
  const float* old_logprob;
  const float* reward;
  const uint8_t* flags;
  const int32_t* episode_id;
  const float* value_scalar;
  const float* value_vector;
  const float* bootstrap;
} ckrl_rollout;

/* Current-policy outputs consumed by the loss (what ppo_loss recomputes through
 * PolicyNet::evaluate_chunk / value, losses.cpp:115, 196). Device pointers. */
typedef struct {
  int32_t logits_dtype; /* CKRL_DTYPE_F32 | CKRL_DTYPE_BF16 | CKRL_DTYPE_TOKEN_ROWS (logits then
                           points at [E][Tc][C][M] ckrl_token_row: the policy head already
                           reduced on the tensor cores, ckrl_project_token_stats) */
  const void* logits;
  const float* values;  /* new values at the value level; may be NULL if value_loss_coef == 0 */
} ckrl_policy_outputs;

/* Episode table (EpisodeInfo, core/types.hpp:72-85) as SoA, device pointers. */
typedef struct {
  int32_t count;
  const int32_t* env_id;
  const int32_t* episode_id;
  const int32_t* start_step;
  const int32_t* length;
  const double* total_reward;
  const int32_t* first_success;
  const uint8_t* complete;
  const int32_t* task_id;
  const int32_t* reset_state_id;
} ckrl_episodes;

/* PpoBatch (advantage/assembler.hpp:16-37) as SoA, device pointers (outputs of assembly). */
typedef struct {
  uint8_t* counted;    /* [E][Tc][C] */
  double* advantages;  /* [E][Tc] (chunk) or [E][Tc][C] (action); raw GAE, fp64 as the
                          reference's PpoBatch (assembler.hpp:16-37) */
  double* returns;     /* same shape */
} ckrl_ppo_batch;

/* GrpoBatch (advantage/assembler.hpp:40-62) as SoA: each env owns at most one retained
 * trajectory (only complete episodes starting at step 0 are grouped). Device pointers. */
typedef struct {
  int32_t* env_group;       /* [E] retained-group ordinal in GroupKey order, -1 none */
  int32_t* env_member;      /* [E] member index inside its group */
  int32_t* env_episode;     /* [E] episode_id of the trajectory */
  double* env_advantage;    /* [E] group-relative advantage */
  int32_t* env_group_size;  /* [E] trajectories in the group */
  double* slot_weight;      /* [E][Tc][C] per-step weight, f64 as the reference's TrajChunk::slot_weights
                               (0 outside the trajectory / masked, grpo.cpp:57-79) */
  uint8_t* slot_member;     /* [E][Tc][C] slot belongs to the trajectory */
  int32_t* group_counts;    /* [2] groups_total, groups_retained (device) */
} ckrl_grpo_batch;

/* Optional per-token / per-unit outputs of the loss (device, may be NULL each). */
typedef struct {
  float* coeff_logprob;  /* [E][Tc][C][M]  dLoss/dlogprob per position (accumulate_chunk_gradient) */
  float* coeff_entropy;  /* [E][Tc][C][M]  dLoss/dentropy per position */
  float* coeff_value;    /* value level shape, dLoss/dV */
  float* token_logprob;  /* [E][Tc][C][M]  new log-probs (evaluate_chunk) */
  float* token_entropy;  /* [E][Tc][C][M]  new entropies */
  void* dlogits;         /* [E][Tc][C][M][V] optional, logits dtype: the softmax-backward seam
                            (accumulate_chunk_gradient's dlogits, policy_net.cpp:431-456) fused
                            into the loss launch (V = 256; ckrl_logits_grad otherwise) */
  double* action_entropy; /* [E][Tc][C] entropy at action granularity: sum of the slot's token
                             entropies (ascending j) on unit-active slots (PPO: counted; GRPO:
                             weighted trajectory slots), 0 elsewhere */
  double* chunk_entropy;  /* [E][Tc] sum of the record's action entropies (ascending i) */
} ckrl_loss_outputs;

/* ---- host-only helpers (no device work) ---------------------------------------------- */
const char* ckrl_version(void);
const char* ckrl_status_string(int32_t status);
const char* ckrl_last_error(void); /* thread-local message of the last failing call */

/* validate_granularity (core/granularity.cpp:47-60). */
int32_t ckrl_validate_granularity(const ckrl_granularity* spec);

/* Workspace bytes for a slab of this shape (whole step; the cross-rank records live in the
 * communicator, so `world` does not change the size). Caller allocates device memory of at
 * least this size once. */
size_t ckrl_workspace_bytes(int32_t num_envs, int32_t num_chunks, int32_t chunk_len,
                            int32_t tokens_per_action, int32_t world);

/* Zero the workspace once after allocating it (its last-CTA counters self-reset). */
int32_t ckrl_workspace_init(void* workspace, size_t workspace_bytes, ckrl_stream_t stream);

/* Merge `world` per-rank whitening/normaliser stats records (host memory, the layout
 * ckrl_stats_record_bytes() describes) in rank order (Chan's pairwise moment update).
 * Exposed for the multi-rank host tests; the device path merges the same records in the
 * same order inside the loss kernel. */
size_t ckrl_stats_record_bytes(void);
int32_t ckrl_merge_stats_host(const void* records, int32_t world, double* out_mean,
                              double* out_denom, int64_t* out_counts /* n_adv,n_val,n_pos */);

/* ---- (c) advantage -------------------------------------------------------------------- */

/* compute_gae (advantage/gae.cpp:7-37) over `num_seqs` independent flat unit sequences
 * packed back to back; seq_offsets[num_seqs+1] (device) delimits them. flags use the
 * CKRL_FLAG_* bits (valid ignored). Outputs in fp64 (the reference's precision). */
int32_t ckrl_compute_gae(int32_t num_seqs, const int32_t* seq_offsets, const double* rewards,
                         const double* values, const double* bootstrap, const uint8_t* flags,
                         const ckrl_gae_params* params, double* advantages, double* returns,
                         ckrl_stream_t stream);

/* assemble_ppo_batch (advantage/assembler.cpp:78-195): segmentation, chunk/action units,
 * counted masks, bootstraps, GAE (warp-segmented reverse scan), plus the rank-local
 * normaliser / whitening stats record left in `workspace`. */
int32_t ckrl_assemble_ppo_batch(const ckrl_rollout* rollout, const ckrl_gae_params* gae,
                                const ckrl_granularity* spec, ckrl_ppo_batch* batch,
                                void* workspace, size_t workspace_bytes, ckrl_stream_t stream);

/* normalize_advantages (optim/update.cpp:14-45), materialised in place over the counted
 * units, using the stats left in `workspace` by ckrl_assemble_ppo_batch. The stats record
 * is then marked whitened: a following ckrl_ppo_loss uses the advantages as they are (as
 * the reference's ppo_loss does after update_ppo's normalize_advantages), and a second
 * ckrl_normalize_advantages re-whitens with the moments of the whitened values, as the
 * reference's recomputation does. */
int32_t ckrl_normalize_advantages(const ckrl_rollout* rollout, const ckrl_granularity* spec,
                                  ckrl_ppo_batch* batch, void* workspace,
                                  size_t workspace_bytes, ckrl_stream_t stream);

/* assemble_grpo_batch (advantage/assembler.cpp:197-267): eligibility, GroupKey-ordered
 * grouping (std::map order), min size, strict success-rate filter, group-relative
 * advantages, valid-action masks and length-normalised per-step weights. */
int32_t ckrl_assemble_grpo_batch(const ckrl_rollout* rollout, const ckrl_episodes* episodes,
                                 const ckrl_granularity* spec, const ckrl_grpo_options* options,
                                 ckrl_grpo_batch* batch, void* workspace, size_t workspace_bytes,
                                 ckrl_stream_t stream);

/* Per-group / per-episode GRPO helpers (advantage/grpo.hpp:32-53), batched: groups are
 * back-to-back segments of `returns` delimited by group_offsets[num_groups+1]; episodes are
 * segments of the per-step outputs delimited by step_offsets[num_episodes+1]. All device
 * pointers; bit-identical to the reference's fp64 arithmetic. Device-side errors
 * (DegenerateGroup: a group smaller than 2, or zero std with eps_std == 0) are written to
 * *status (device int32, first error wins; may be NULL). */
int32_t ckrl_grpo_group_advantage(int32_t num_groups, const int32_t* group_offsets,
                                  const double* returns, double eps_std, double* advantages,
                                  int32_t* status, ckrl_stream_t stream);
/* keep[g] = lower < group_mean_return < upper (strict); group_mean (nullable) receives the
 * means of group_mean_return (grpo.cpp:30-46). */
int32_t ckrl_success_rate_filter(int32_t num_groups, const int32_t* group_offsets,
                                 const double* returns, double lower, double upper,
                                 uint8_t* keep, double* group_mean, ckrl_stream_t stream);
/* valid_action_mask / length_norm_weights (grpo.cpp:48-79) per episode; either output may
 * be NULL. */
int32_t ckrl_valid_action_mask(int32_t num_episodes, const int64_t* step_offsets,
                               const uint8_t* success, const int64_t* first_success_step,
                               uint8_t* mask, ckrl_stream_t stream);
int32_t ckrl_length_norm_weights(int32_t num_episodes, const int64_t* step_offsets,
                                 const uint8_t* success, const int64_t* first_success_step,
                                 int32_t length_normalized, double* weights,
                                 ckrl_stream_t stream);
/* slab_success_rate (advantage/assembler.cpp:269-278): success_once fraction over complete
 * episodes, into *out (device f64). */
int32_t ckrl_slab_success_rate(const ckrl_episodes* episodes, double* out, ckrl_stream_t stream);

/* Minibatches. optim::ppo_loss / grpo_loss evaluate a subset of the batch (record_indices /
 * group_indices, losses.hpp:54-65; drawn by update_ppo / update_grpo, update.cpp:83-160).
 *
 * ckrl_select_records gathers records record_index[i] = env * num_chunks + chunk (device
 * int64, n entries) of (src, src_batch, src_policy) into the caller-allocated buffers of
 * (dst, dst_batch, dst_policy), laid out as num_envs = n, num_chunks = 1 (the dst arrays
 * are written; dims/dtypes must match src), and writes the subset's normalisers
 * (n_adv, n_val, n_pos) into `workspace` (sized for n envs). A following ckrl_ppo_loss on
 * the dst view with advantage_normalization = 0 is the minibatch loss.
 *
 * ckrl_select_groups keeps the envs of the n groups group_index[] (retained-group ordinals,
 * device int32) in dst_env_group (others -1) and sets the loss's group count to n in
 * `workspace` (the workspace that holds the GRPO assembly). */
int32_t ckrl_select_records(const ckrl_rollout* src, const ckrl_ppo_batch* src_batch,
                            const ckrl_policy_outputs* src_policy, const ckrl_granularity* spec,
                            int64_t n, const int64_t* record_index, const ckrl_rollout* dst,
                            const ckrl_ppo_batch* dst_batch, const ckrl_policy_outputs* dst_policy,
                            void* workspace, size_t workspace_bytes, ckrl_stream_t stream);
/* (src_policy->logits / ->values may be NULL when the dst buffers are already filled, e.g.
 * by a caller that evaluated its policy only on the selected records.) */
int32_t ckrl_select_groups(int32_t num_envs, const int32_t* src_env_group, int32_t* dst_env_group,
                           int32_t n, const int32_t* group_index, void* workspace,
                           size_t workspace_bytes, ckrl_stream_t stream);

/* Reads the rank's 64-byte stats record from a workspace after an assembly (synchronises
 * `stream`): the advantage-unit moments {mean, M2 = sum of squared deviations} (f64) and
 * {n_adv, n_adv, n_val, n_pos, groups_retained, status} (int64). Returns the device-detected
 * status (e.g. DegenerateGroup from the GRPO assembly, assembler.cpp:247-252) as the call's
 * status. */
int32_t ckrl_read_stats(const void* workspace, size_t workspace_bytes, int32_t num_envs,
                        double* moments_out /* [2] */, int64_t* counts_out /* [6] */,
                        ckrl_stream_t stream);

/* ---- (b) fused action-token kernel ---------------------------------------------------- */

/* PolicyNet::evaluate_chunk (policy/policy_net.cpp:333-357) + aggregate_logprob
 * (core/granularity.cpp:83-113): per-token log-prob and entropy from logits rows, and the
 * action / chunk log-prob aggregates in canonical order. Entropy at action and chunk
 * granularity: per slot the sum of its M token entropies (ascending j), per chunk the sum of
 * its slots' (ascending i), over the slots slot_mask ([num_chunks][chunk_len] u8, nonzero =
 * valid action; NULL = all) selects, 0 elsewhere. Any output may be NULL. */
int32_t ckrl_token_stats(int64_t num_chunks, int32_t chunk_len, int32_t tokens_per_action,
                         int32_t vocab, int32_t logits_dtype, const void* logits,
                         int32_t token_dtype, const void* tokens, float* token_logprob,
                         float* token_entropy, double* action_logprob, double* chunk_logprob,
                         const uint8_t* slot_mask, double* action_entropy, double* chunk_entropy,
                         ckrl_stream_t stream);

/* The policy head: PolicyNet::logits_from_feature (policy/policy_net.cpp:265-274),
 * logits[v] = sum_h W_pol[v][h] * feature[h] + b_pol[v], over the trunk feature of every
 * position (the hidden state forward_logits feeds it, :276-284). */
typedef struct {
  int32_t hidden;        /* H: a multiple of 64, 64 .. 16384 */
  int32_t vocab;         /* bins: 256 */
  const void* feature;   /* [rows][H] bf16, 16-byte aligned, row pitch H */
  const void* w_pol;     /* [vocab][H] bf16 (the reference's row-major W_pol block) */
  const float* b_pol;    /* [vocab] f32; NULL = zero bias */
} ckrl_policy_head;

/* Row N2: the hidden -> action-bin projection on the tensor cores (tcgen05.mma, bf16 inputs,
 * f32 accumulators in TMEM) fused with evaluate_chunk's per-position reduction
 * (policy_net.cpp:90-102, 333-357): per position the sampled token's log-prob and the
 * entropy, without the [rows][256] logits ever reaching HBM. Outputs (each nullable):
 * token_rows ([rows] ckrl_token_row, the losses' CKRL_DTYPE_TOKEN_ROWS input), token_logprob
 * (f64), token_entropy (f32), and the logits themselves (logits_dtype F32 | BF16, [rows][256])
 * for callers that still want them. Asynchronous on `stream`. */
int32_t ckrl_project_token_stats(int64_t rows, const ckrl_policy_head* head, int32_t token_dtype,
                                 const void* tokens, ckrl_token_row* token_rows,
                                 double* token_logprob, float* token_entropy, int32_t logits_dtype,
                                 void* logits, ckrl_stream_t stream);

/* ---- (f1) softmax-backward seam --------------------------------------------------------- */

/* The per-position logits gradient PolicyNet::accumulate_chunk_gradient forms before its
 * outer_add / trunk backward (policy/policy_net.cpp:431-456):
 *   dlogits[k][v] = coeff_lp[k] * ([v == tok_k] - p_kv) + coeff_ent[k] * (-p_kv * (ls_kv + H_k)),
 * ls = log_softmax(logits[k]), p = exp(ls), H_k = -sum_v p_kv ls_kv, for `rows` positions of
 * `vocab` bins. coeff_lp / coeff_ent are the loss outputs (ckrl_loss_outputs; coeff_ent may be
 * NULL = all zero). Positions with both coefficients zero are skipped by the reference; their
 * row is written as zeros. A non-finite coefficient is the reference's NonFinite (:437-438):
 * the row is zeroed and *status_device (optional, caller-zeroed int32) is set to
 * CKRL_ERR_NON_FINITE; read it with ckrl_read_status. dlogits may alias logits when both
 * dtypes match (in place). Asynchronous on `stream`. */
int32_t ckrl_logits_grad(int64_t rows, int32_t vocab, int32_t logits_dtype, const void* logits,
                         int32_t token_dtype, const void* tokens, const float* coeff_lp,
                         const float* coeff_ent, int32_t out_dtype, void* dlogits,
                         int32_t* status_device, ckrl_stream_t stream);

/* Synchronises `stream`, reads a device status word written by an asynchronous entry point
 * and returns it as the call's status (0 when clear). */
int32_t ckrl_read_status(const int32_t* status_device, ckrl_stream_t stream);

/* ---- (f4) optimizer step --------------------------------------------------------------- */

/* optim::Adam (optim/adam.hpp:10-27, adam.cpp:15-41). */
typedef struct ckrl_adam_params {
  double learning_rate;
  double max_grad_norm; /* <= 0: no clipping */
  double beta1;         /* reference default 0.9 */
  double beta2;         /* 0.999 */
  double eps;           /* 1e-8 */
} ckrl_adam_params;

/* Scratch for ckrl_adam_step (zero it once after allocating; its counter self-resets). */
size_t ckrl_adam_workspace_bytes(void);

/* Adam::step on `n` parameters (dtype CKRL_DTYPE_F32 or a double-precision step with
 * dtype = 4, CKRL_DTYPE_F64): ||grad|| (fp64 accumulate; all-reduced over `comm` when the
 * parameters are sharded across ranks), NonFinite if it is not finite (nothing is modified,
 * *status_device set; read it with ckrl_read_status), grad clipped in place to max_grad_norm,
 * then m / v / params updated with bias corrections for step `t` (>= 1, the count after this
 * step: the reference's ++t_). *norm_device receives the pre-clip norm. Asynchronous on
 * `stream`; two launches (the update a programmatic dependent of the norm). */
int32_t ckrl_adam_step(int32_t dtype, int64_t n, void* params, void* grad, void* exp_avg,
                       void* exp_avg_sq, const ckrl_adam_params* p, int64_t t, double* norm_device,
                       int32_t* status_device, void* workspace, size_t workspace_bytes,
                       ckrl_comm* comm, ckrl_stream_t stream);

/* ---- (d) losses ----------------------------------------------------------------------- */

/* ppo_loss (optim/losses.cpp:62-232) over every record (full batch), fused with the token
 * kernel: one pass over the logits computes log-softmax, gather, entropy, the clipped
 * surrogate at logprob granularity, value and entropy terms and all coefficients.
 * Diagnostics go to `diag_device` (double[CKRL_DIAG_COUNT], device) without host sync.
 * Requires the stats record produced by ckrl_assemble_ppo_batch in `workspace`
 * (whitening applied on the fly when params->advantage_normalization). */
int32_t ckrl_ppo_loss(const ckrl_rollout* rollout, const ckrl_ppo_batch* batch,
                      const ckrl_policy_outputs* policy, const ckrl_granularity* spec,
                      const ckrl_ppo_params* params, ckrl_loss_outputs* outputs,
                      double* diag_device, void* workspace, size_t workspace_bytes,
                      ckrl_stream_t stream);

/* grpo_loss (optim/losses.cpp:234-331) over every retained group. */
int32_t ckrl_grpo_loss(const ckrl_rollout* rollout, const ckrl_grpo_batch* batch,
                       const ckrl_policy_outputs* policy, const ckrl_granularity* spec,
                       const ckrl_grpo_params* params, ckrl_loss_outputs* outputs,
                       double* diag_device, void* workspace, size_t workspace_bytes,
                       ckrl_stream_t stream);

/* Whole step (the measured hot path): assemble -> fused loss, two launches (the loss a
 * programmatic dependent of the assembly). comm may be NULL (single rank); with a multi-rank
 * comm the stats record and loss sums cross ranks inside the two kernels (see ckrl_comm_*
 * below) and diag_device holds the job-wide diagnostics on every rank. */
int32_t ckrl_ppo_step(const ckrl_rollout* rollout, const ckrl_policy_outputs* policy,
                      const ckrl_gae_params* gae, const ckrl_granularity* spec,
                      const ckrl_ppo_params* params, ckrl_ppo_batch* batch,
                      ckrl_loss_outputs* outputs, double* diag_device, void* workspace,
                      size_t workspace_bytes, ckrl_comm* comm, ckrl_stream_t stream);
int32_t ckrl_grpo_step(const ckrl_rollout* rollout, const ckrl_episodes* episodes,
                       const ckrl_policy_outputs* policy, const ckrl_granularity* spec,
                       const ckrl_grpo_options* options, const ckrl_grpo_params* params,
                       ckrl_grpo_batch* batch, ckrl_loss_outputs* outputs, double* diag_device,
                       void* workspace, size_t workspace_bytes, ckrl_comm* comm,
                       ckrl_stream_t stream);

/* The two halves of ckrl_ppo_step / ckrl_grpo_step (same kernels and cross-rank exchange), for
 * callers that pipeline batches: e.g. batch i+1's assembly on one stream while batch i's loss
 * runs on another, each batch with its own workspace and batch buffers. The loss must follow
 * its own assembly (stream order or an event); an assembly may start once the loss of the
 * batch two before it has completed (the exchange keeps two batches in flight). */
int32_t ckrl_ppo_step_assemble(const ckrl_rollout* rollout, const ckrl_gae_params* gae,
                               const ckrl_granularity* spec, ckrl_ppo_batch* batch,
                               void* workspace, size_t workspace_bytes, ckrl_comm* comm,
                               ckrl_stream_t stream);
int32_t ckrl_ppo_step_loss(const ckrl_rollout* rollout, const ckrl_policy_outputs* policy,
                           const ckrl_granularity* spec, const ckrl_ppo_params* params,
                           const ckrl_ppo_batch* batch, ckrl_loss_outputs* outputs,
                           double* diag_device, void* workspace, size_t workspace_bytes,
                           ckrl_comm* comm, ckrl_stream_t stream);
int32_t ckrl_grpo_step_assemble(const ckrl_rollout* rollout, const ckrl_episodes* episodes,
                                const ckrl_granularity* spec, const ckrl_grpo_options* options,
                                ckrl_grpo_batch* batch, void* workspace, size_t workspace_bytes,
                                ckrl_comm* comm, ckrl_stream_t stream);
int32_t ckrl_grpo_step_loss(const ckrl_rollout* rollout, const ckrl_policy_outputs* policy,
                            const ckrl_granularity* spec, const ckrl_grpo_params* params,
                            const ckrl_grpo_batch* batch, ckrl_loss_outputs* outputs,
                            double* diag_device, void* workspace, size_t workspace_bytes,
                            ckrl_comm* comm, ckrl_stream_t stream);

/* Copy the device diagnostics to the host (synchronises `stream`) and map the device
 * status word to the reference's exceptions: SkipUpdate (no retained groups),
 * DegenerateGroup, NonFinite (losses.cpp:229-230, 326-327). */
int32_t ckrl_read_diagnostics(const double* diag_device, double* diag_host, ckrl_stream_t stream);

/* Profiling aid: %globaltimer stamps (ns) of CTA 0 from the last TMA loss / fused-step
 * launch: [0] start, [1] GAE phase done, [2] grid barrier passed, [3] constants ready,
 * [4..7] first unit phase of each buffer warp, [8] last row tile, [9] all roles done,
 * [10] reduction done. Synchronises the device. The stamps exist only in a library built
 * with -DCKRL_PROBES (they cost ~1 us per step); otherwise this reads back zeros. */
int32_t ckrl_debug_timeline(uint64_t* out, int32_t n);
/* Profiling aid: per-CTA %globaltimer stamps of the last TMA loss launch, [3][1184]: start,
 * roles done, exit. Synchronises the device. Zeros unless built with -DCKRL_PROBES. */
int32_t ckrl_debug_cta_times(uint64_t* out, int32_t n);

/* ---- (e) rollout pipeline on CUDA streams / events (cfg5) ----------------------------- */

/* VecEnvConfig (envsim/vec_env.hpp:16-35) + the rollout's reset mode. */
typedef struct {
  int32_t kind; /* 0 toy_reach, 1 scripted */
  int32_t num_envs, max_episode_steps, auto_reset, ignore_terminations, use_fixed_reset_state_ids;
  int32_t chunk_len, grid_size, reward_shaping, num_reset_states, success_step;
  int32_t deferred_reset; /* ResetMode::Deferred (rollout.hpp:19) */
  uint64_t seed;
} ckrl_env_config;

/* PolicyDescriptor (policy/policy_net.hpp:15-26); parameters are the reference's flat f64
 * layout (policy_net.cpp:107-152), device memory. */
typedef struct {
  int32_t obs_dim, hidden, trunk_layers, value_hidden, vocab, chunk_len, tokens_per_action;
} ckrl_policy_desc;

/* Samplers of StageGen (policy_net.cpp:286-331). REFERENCE sums the 256 exponentials and
 * walks the inverse CDF serially in the reference's order (bit-exact with sample_chunk);
 * PARALLEL does both as fixed-order block reductions / scans (warp shuffles), so the draw is
 * the same for every k and placement but may differ from the reference's in the last ulp of
 * the log-sum-exp (and, at a CDF boundary within an ulp of u, in the token). */
enum { CKRL_SAMPLER_REFERENCE = 0, CKRL_SAMPLER_PARALLEL = 1 };

/* RolloutSpec (placement/rollout.hpp:16-22) + pipeline depth k (PlacementPlan::pipeline_stage_num)
 * + placement. placed = 0 (a zero-initialised spec): colocated (PlacementMode::Colocated,
 * plan.cpp:60-68): env and generation kernels share the calling device. placed = 1: the
 * generation role runs on gen_device (hybrid / disaggregated placement; it may equal the env
 * device, which keeps the hand-offs): every chunk the stage's observation batch is copied env -> gen and its action
 * batch (tokens, log-probs, values, optional logits) gen -> env over NVLink peer copies, the
 * reference's obs / act channels (real_backend.cpp:15-37, 59-138), with per-stage events on
 * both devices. The slab is bit-identical across k and placement. */
typedef struct {
  ckrl_env_config env;
  ckrl_policy_desc policy;
  int32_t num_chunks;
  int32_t stages;                 /* k: env partitions, must divide num_envs */
  uint64_t sample_seed;
  const int32_t* reset_state_ids; /* [num_envs] device, or NULL */
  int32_t sampler;                /* CKRL_SAMPLER_* */
  int32_t placed;                 /* 0 colocated, 1 generation on gen_device */
  int32_t gen_device;             /* placed: the generation device */
  void* gen_workspace;            /* placed: ckrl_pipeline_gen_workspace_bytes on gen_device */
  size_t gen_workspace_bytes;
} ckrl_pipeline_spec;

/* derive_mode (placement/plan.cpp:60-68) after validate_plan (:49-58) of a PlacementPlan
 * given as inclusive slot ranges: 0 colocated, 1 disaggregated, 2 hybrid; negative on an
 * invalid plan (CKRL_ERR_INVALID_PLAN in *status). */
enum { CKRL_PLACEMENT_COLOCATED = 0, CKRL_PLACEMENT_DISAGGREGATED = 1, CKRL_PLACEMENT_HYBRID = 2 };
int32_t ckrl_placement_mode(int32_t num_slots, int32_t env_begin, int32_t env_end, int32_t rollout_begin,
                            int32_t rollout_end, int32_t actor_begin, int32_t actor_end,
                            int32_t pipeline_stage_num, int32_t* status);

/* The epoch's slab in the ckrl_rollout layout (f32 for the loss, f64 copies for exact
 * comparison with the reference) + the merged episode table. Device pointers. */
typedef struct {
  int32_t* tokens;            /* [E][T][C][M] */
  float* old_logprob;         /* [E][T][C][M] */
  double* old_logprob_f64;
  float* reward;              /* [E][T][C] */
  double* reward_f64;
  uint8_t* flags;             /* [E][T][C] */
  int32_t* episode_id;        /* [E][T][C] */
  float* value_scalar;        /* [E][T] */
  double* value_scalar_f64;
  float* value_vector;        /* [E][T][C] */
  double* value_vector_f64;
  float* boot_scalar;         /* [E][T][C] scalar head on post_obs */
  double* boot_scalar_f64;
  float* boot_vector0;        /* [E][T][C] vector head [0] on post_obs */
  double* boot_vector0_f64;
  int32_t* episode_count;     /* [1] */
  int32_t *ep_env_id, *ep_episode_id, *ep_start, *ep_length; /* [E*(T*C+1)] capacity */
  double* ep_total_reward;
  int32_t* ep_first_success;
  uint8_t* ep_complete;
  int32_t *ep_task, *ep_reset_id;
  int32_t* status;            /* [1] device error word (BadResetId) */
  float* logits;              /* optional [E][T][C][M][V]: the rollout policy's logits (the
                                 current policy's at the first PPO epoch), or NULL */
} ckrl_pipeline_outputs;

int64_t ckrl_policy_num_params(const ckrl_policy_desc* desc);
size_t ckrl_pipeline_workspace_bytes(const ckrl_pipeline_spec* spec);
/* Generation-side scratch of a placed pipeline (policy copy, sampling streams, obs / action
 * staging), allocated by the caller on gen_device. */
size_t ckrl_pipeline_gen_workspace_bytes(const ckrl_pipeline_spec* spec);
/* One rollout epoch (StageSim / StageGen / merge_stages, placement/rollout.cpp:11-109;
 * RealBackend::run_rollout_epoch, real_backend.cpp:59-138): k stage partitions, gen and
 * sim kernels on two streams with per-stage event hand-offs; the slab is identical for
 * every k. Work is ordered after prior work on `stream`, and `stream` waits for it. */
int32_t ckrl_pipeline_run(const ckrl_pipeline_spec* spec, const double* params,
                          ckrl_pipeline_outputs* out, void* workspace, size_t workspace_bytes,
                          ckrl_stream_t stream);

/* ---- (f3) wire and on-disk formats (host) ------------------------------------------------ */

/* dump_slab (core/types.cpp:9-28) of an SoA slab in HOST memory: the reference's
 * trajectories.txt text ("# env_id episode_uid step tokens[M] reward terminated truncated
 * valid" then one line per atomic slot: env_id is the slab row; uid = (first_env_id + row)
 * << 32 | episode_id, the global env id of a VecEnv partition or rank shard (vec_env.cpp:94),
 * -1 frozen; reward as %.17g of the f64 reward, e.g. ckrl_pipeline_outputs.reward_f64).
 * Writes at most `capacity` bytes (NUL-terminated when it fits) and the full text length to
 * *length (capacity 0 / out NULL: size query). */
int32_t ckrl_dump_slab(int32_t num_envs, int32_t num_chunks, int32_t chunk_len,
                       int32_t tokens_per_action, int32_t token_dtype, const void* tokens,
                       const double* reward, const uint8_t* flags, const int32_t* episode_id,
                       int32_t first_env_id, char* out, size_t capacity, size_t* length);

/* save_checkpoint / load_checkpoint (policy/checkpoint.cpp:37-83): the CKRL v1 file of a
 * policy descriptor + its flat f64 parameters (host memory). Load with params NULL queries
 * the descriptor and count; errors are the reference's chunkrl::Error cases (bad magic,
 * version, count mismatch, truncation) as CKRL_ERR_GENERIC with the reference's message. */
int32_t ckrl_save_checkpoint(const ckrl_policy_desc* desc, const double* params, const char* path);
int32_t ckrl_load_checkpoint(const char* path, ckrl_policy_desc* desc, double* params,
                             int64_t capacity, int64_t* count);

/* ---- multi-GPU: stats record + loss scalars over NVLink peer memory ------------------------
 * The path shards by env (PPO) / whole group (GRPO); its only cross-rank values are the
 * 64-byte stats record before the loss (whitening moments, n_adv / n_val / n_pos, retained
 * groups: optim/update.cpp:14-45, optim/losses.cpp:75-87, 246) and the raw loss sums after
 * it (losses.cpp:221-227). Each rank owns a small exchange buffer in its HBM; inside
 * ckrl_*_step the assembly kernel stores the rank's record into every rank's buffer and the
 * loss kernel's last CTA does the same with its sums (P2P stores + system-scope flags), so a
 * multi-rank step is the same two launches as a single-rank one. Every rank must run the
 * same sequence of steps (the exchange is collective).
 *
 * ckrl_comm_create: a rank of a `world`-rank job on the current device; unique_id (from
 * ckrl_comm_unique_id on one rank, 128 bytes) additionally creates an NCCL communicator,
 * used only by a sharded ckrl_adam_step; NULL skips NCCL. Before the first step the peers'
 * buffers must be mapped: across processes, all-gather every rank's ckrl_comm_ipc_handle
 * (CUDA IPC, CKRL_IPC_HANDLE_BYTES each, rank order) and pass them to ckrl_comm_open_peers;
 * in one process driving several ranks, ckrl_comm_set_peers with the ranks' communicators. */
#define CKRL_IPC_HANDLE_BYTES 64
int32_t ckrl_comm_unique_id(void* out_id /* 128 bytes */);
int32_t ckrl_comm_create(int32_t world, int32_t rank, const void* unique_id, ckrl_comm** out);
int32_t ckrl_comm_ipc_handle(ckrl_comm* comm, void* out_handle /* CKRL_IPC_HANDLE_BYTES */);
int32_t ckrl_comm_open_peers(ckrl_comm* comm, const void* handles /* world x CKRL_IPC_HANDLE_BYTES */);
int32_t ckrl_comm_set_peers(ckrl_comm* comm, ckrl_comm* const* comms /* [world], rank order */);
int32_t ckrl_comm_destroy(ckrl_comm* comm);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* CKRL_H */
