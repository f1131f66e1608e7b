// Launchers shared between the kernel translation units and the C-ABI layer.
#pragma once

#include <string>

#include "common.cuh"

namespace ckrl {

enum LossMode { MODE_STATS = 0, MODE_PPO = 1, MODE_GRPO = 2 };

struct LossArgs {
  int mode;
  int E, Tc, C, M, V;
  int64_t n_rec;        // records (E*Tc), or chunks for MODE_STATS
  int rec_per_tile;
  int64_t n_tiles;
  int logits_bf16, tok_i32;
  const void* logits;
  const void* tokens;
  const float* old_lp;
  // PPO
  const uint8_t* counted;
  const double* adv;
  const double* ret;
  const float* new_values;
  int adv_level, lp_level, val_level;
  double clip, vcoef, ecoef;
  int normalize;
  // GRPO
  const int32_t* env_group;
  const double* env_adv;
  const int32_t* env_group_size;
  const double* slot_weight;
  const uint8_t* slot_member;
  // outputs (nullable)
  float* coeff_lp;
  float* coeff_ent;
  float* coeff_val;
  float* tok_lp;
  float* tok_ent;
  double* action_lp;
  double* chunk_lp;
  double* action_ent;        // [slots] canonical-order sum of the slot's token entropies (masked)
  double* chunk_ent;         // [records] sum of the record's action entropies (masked)
  const uint8_t* stats_mask; // MODE_STATS: per-slot valid mask for the entropy aggregates (NULL: all)
  int all_rows;  // evaluate every row (token outputs requested / MODE_STATS)
  // stats: the rank's own record (single rank), or every rank's through the exchange
  const StatsRecord* recs;
  int world;
  ExchangeView ex;   // ex.world > 1: records and raw sums cross ranks over peer memory
  int max_ctas;      // > 0: loss grid cap (several ranks of one job share this device)
  char* ws;
  WsLayout L;
  double* diag;      // finalised diagnostics; raw sums also go to ws.loss_raw
  int finalize;      // 1: last CTA finalises into diag
  // fused PPO step (assembly inside the loss launch)
  ckrl_rollout ro;
  double gamma, lambda;
  // overlapped step: the assembly kernel is still running on `reserved_sms` SMs when this
  // kernel starts (programmatic dependent launch)
  int pdl;
  int reserved_sms;
  int nbuf;      // TMA kernel: row-partial buffers (multiple of 4, <= kMaxRowBufs)
  int rows_cap;  // TMA kernel: rows per buffer (rec_per_tile * C * M, rounded up to 8)
  int slots_cap; // TMA kernel: slots per buffer (rec_per_tile * C, rounded up to 8)
  void* dlogits; // optional fused softmax-backward output [positions][V] (logits dtype)
  const ckrl_token_row* rows_in;  // finished per-position {lp, H} instead of logits (row N2)
};

cudaError_t launch_ppo_assemble(const ckrl_rollout& ro, int action_level, double gamma,
                                double lambda, ckrl_ppo_batch& b, char* ws, const WsLayout& L,
                                cudaStream_t s, const ExchangeView& ex = ExchangeView{});
cudaError_t launch_flat_gae(int num_seqs, const int32_t* offs, const double* r, const double* v,
                            const double* b, const uint8_t* f, double gamma, double lambda,
                            double* adv, double* ret, cudaStream_t s);
cudaError_t launch_normalize(const ckrl_rollout& ro, int action_level, const uint8_t* counted,
                             double* adv, StatsRecord* recs, int world, uint32_t* ticket, cudaStream_t s);
cudaError_t launch_grpo_assemble(const ckrl_rollout& ro, const ckrl_episodes& ep,
                                 const ckrl_grpo_options& opt, ckrl_grpo_batch& gb, char* ws,
                                 const WsLayout& L, cudaStream_t s,
                                 const ExchangeView& ex = ExchangeView{});
cudaError_t launch_tile(LossArgs& a, cudaStream_t s, int* grid_out);
cudaError_t debug_cta_times(uint64_t* out, int n);
int32_t format_slab(int32_t E, int32_t Tc, int32_t C, int32_t M, int32_t token_dtype, const void* tokens,
                    const double* reward, const uint8_t* flags, const int32_t* episode_id, int32_t first_env_id,
                    std::string& out);
int32_t write_checkpoint(const ckrl_policy_desc& d, const double* params, int64_t count, const char* path,
                         std::string& err);
int32_t read_checkpoint(const char* path, ckrl_policy_desc* d, double* params, int64_t capacity,
                        int64_t* count_out, std::string& err);
size_t adam_workspace_bytes();
double* adam_norm_sq_slot(char* ws);
cudaError_t launch_adam_norm(int f64, const void* g, int64_t n, char* ws, cudaStream_t s);
cudaError_t launch_adam_update(int f64, void* p, void* g, void* m, void* v, int64_t n, double lr,
                               double max_norm, double b1, double b2, double eps, double bc1, double bc2,
                               char* ws, double* norm_out, int32_t* status, int pdl, cudaStream_t s);
cudaError_t launch_logits_grad(const void* logits, int logits_bf16, const void* tokens, int tok_i32,
                               const float* coeff_lp, const float* coeff_ent, int64_t rows, int V,
                               void* out, int out_bf16, int32_t* status, cudaStream_t s);
cudaError_t launch_ppo_fused(LossArgs& a, cudaStream_t s, int* grid_out);
cudaError_t launch_proj_stats(int64_t rows, int H, const void* feature, const void* w_pol, const float* b_pol,
                              const void* tokens, int tok_i32, ckrl_token_row* out, double* lp, float* ent,
                              void* logits, int logits_bf16, int max_ctas, cudaStream_t s);
cudaError_t read_timeline(uint64_t* out, int n);
size_t pipeline_ws_bytes(const ckrl_pipeline_spec& sp);
size_t pipeline_gen_ws_bytes(const ckrl_pipeline_spec& sp);
cudaError_t launch_select_records(const ckrl_rollout& src, const ckrl_ppo_batch& sb, const ckrl_policy_outputs& sp,
                                  int action_level, int value_action, int64_t n, const int64_t* idx,
                                  const ckrl_rollout& dst, const ckrl_ppo_batch& db,
                                  const ckrl_policy_outputs& dp, char* ws, cudaStream_t s);
cudaError_t launch_select_groups(int E, const int32_t* src_group, int32_t* dst_group, int n, const int32_t* sel,
                                 char* ws, cudaStream_t s);
cudaError_t launch_group_advantage(int G, const int32_t* off, const double* R, double eps, double* adv,
                                   int32_t* status, cudaStream_t s);
cudaError_t launch_success_filter(int G, const int32_t* off, const double* R, double lower, double upper,
                                  uint8_t* keep, double* mean_out, cudaStream_t s);
cudaError_t launch_mask_weights(int n_eps, const int64_t* off, const uint8_t* success, const int64_t* fs,
                                int normalized, uint8_t* mask, double* w, cudaStream_t s);
cudaError_t launch_success_rate(int n, const uint8_t* complete, const int32_t* fs, double* out, cudaStream_t s);
int64_t policy_num_params(const ckrl_policy_desc& d);
cudaError_t pipeline_run(const ckrl_pipeline_spec& sp, const double* params, ckrl_pipeline_outputs& out,
                         char* ws, cudaStream_t stream);

}  // namespace ckrl
