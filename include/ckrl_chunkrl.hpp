// C++ drop-in for the reference's hot-path operator API (chunkrl::advantage / chunkrl::optim),
// implemented on the B200 through the C ABI of ckrl.h (libckrl_host.so -> libckrl.so).
//
// Names, argument meaning and exception types follow the reference headers:
//   core/types.hpp:12-104        Observation, TokenAction, ActionChunk, TokenLogprobs, GroupKey,
//                                StepRecord, EpisodeInfo, TrajectorySlab (same fields)
//   core/granularity.hpp:9-35    Level, GranularitySpec, validate_granularity, level names
//   core/errors.hpp:9-48         the exception hierarchy (Error and its 12 subclasses)
//   advantage/gae.hpp:10-45      GaeParams, GaeResult, compute_gae (both overloads)
//   advantage/grpo.hpp:10-53     GroupBatch, FilterBounds, grpo_group_advantage,
//                                group_mean_return, success_rate_filter, valid_action_mask,
//                                length_norm_weights
//   advantage/assembler.hpp:14-107  PpoRecordView, PpoBatch, TrajChunk, GrpoTrajectory,
//                                GrpoGroup, GrpoBatch, Ppo/GrpoAssemblyOptions,
//                                GrpoAssemblyResult, assemble_ppo_batch, assemble_grpo_batch,
//                                slab_success_rate
//   optim/losses.hpp:12-65       PpoParams, GrpoParams, LossDiagnostics, ppo_loss, grpo_loss
//   optim/update.hpp:33          normalize_advantages
//
// The one unavoidable change: the reference's assembler and losses take a
// PolicyNet and call it internally (snapshot.value(post_obs) for bootstraps,
// assembler.cpp:114-118; evaluate_chunk / value for the new log-probs and values,
// losses.cpp:115, 196, 257). Here the network is passed as its two public calls —
// `ValueFn` (PolicyNet::value) and `LogitsFn` (PolicyNet::forward_logits) — or, on the
// production path, as a view of the current policy's logits / values already in HBM.
// Parameter gradients (grad_out) are the model backward and out of scope: the losses
// return the per-position coefficients that PolicyNet::accumulate_chunk_gradient /
// accumulate_value_gradient consume (losses.cpp:192-218) instead.
//
// Everything runs on the current CUDA device; calls are synchronous like the reference's.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "ckrl.h"

namespace ckrl::chunkrl {

// ---- core/errors.hpp ------------------------------------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
#define CKRL_CHUNKRL_ERROR(name)   \
  struct name : Error {            \
    using Error::Error;            \
  };
CKRL_CHUNKRL_ERROR(UnsupportedCombination)
CKRL_CHUNKRL_ERROR(GranularityOrderViolation)
CKRL_CHUNKRL_ERROR(LengthMismatch)
CKRL_CHUNKRL_ERROR(BadResetId)
CKRL_CHUNKRL_ERROR(HeadMismatch)
CKRL_CHUNKRL_ERROR(NonFinite)
CKRL_CHUNKRL_ERROR(DegenerateGroup)
CKRL_CHUNKRL_ERROR(SkipUpdate)
CKRL_CHUNKRL_ERROR(InvalidPlan)
CKRL_CHUNKRL_ERROR(MemoryOverflow)
CKRL_CHUNKRL_ERROR(EmptyTrace)
CKRL_CHUNKRL_ERROR(ConfigError)
#undef CKRL_CHUNKRL_ERROR

/// Throws the reference exception matching a ckrl status code (no-op for CKRL_OK).
void throw_if_error(int32_t status);

// ---- core/types.hpp ---------------------------------------------------------------------------
using Observation = std::vector<double>;

struct TokenAction {
  std::vector<int> tokens;
  bool operator==(const TokenAction&) const = default;
};

struct ActionChunk {
  std::vector<TokenAction> actions;
  int chunk_length() const { return static_cast<int>(actions.size()); }
  bool operator==(const ActionChunk&) const = default;
};

struct TokenLogprobs {
  int C = 0;
  int M = 0;
  std::vector<double> values;  // C*M, action-major
  double& at(int action, int token) { return values[static_cast<std::size_t>(action) * M + token]; }
  double at(int action, int token) const { return values[static_cast<std::size_t>(action) * M + token]; }
  bool operator==(const TokenLogprobs&) const = default;
};

struct GroupKey {
  int task_id = 0;
  int reset_state_id = -1;
  bool operator==(const GroupKey&) const = default;
  bool operator<(const GroupKey& o) const {
    return std::tie(task_id, reset_state_id) < std::tie(o.task_id, o.reset_state_id);
  }
};

struct StepRecord {
  Observation obs;
  ActionChunk chunk;
  TokenLogprobs token_logprobs;
  std::vector<double> rewards;
  std::vector<bool> terminated;
  std::vector<bool> truncated;
  std::vector<bool> valid;
  std::vector<std::int64_t> episode_uid;
  std::vector<Observation> post_obs;
  double value_scalar = 0.0;
  std::vector<double> value_vector;
  bool operator==(const StepRecord&) const = default;
};

struct EpisodeInfo {
  std::int64_t uid = -1;
  int env_id = -1;
  std::int64_t start_step = 0;
  std::int64_t length = 0;
  double total_reward = 0.0;
  bool success = false;
  std::int64_t first_success_step = -1;
  bool ended_by_truncation = false;
  bool complete = false;
  GroupKey group_key;
  bool operator==(const EpisodeInfo&) const = default;
};

struct TrajectorySlab {
  int num_envs = 0;
  int chunk_length = 0;
  int tokens_per_action = 0;
  std::vector<std::vector<StepRecord>> records;  // [env][chunk]
  std::vector<EpisodeInfo> episodes;
  bool operator==(const TrajectorySlab&) const = default;
  std::int64_t total_frames() const {
    std::int64_t n = 0;
    for (const auto& r : records) n += static_cast<std::int64_t>(r.size()) * chunk_length;
    return n;
  }
};

/// dump_slab (core/types.cpp:9-28): the trajectories.txt text of a slab (through
/// ckrl_dump_slab). Episode uids must be the reference's env << 32 | k (vec_env.cpp:14-16);
/// every env must hold the same number of records.
std::string dump_slab(const TrajectorySlab& slab);

// ---- core/granularity.hpp -------------------------------------------------------------------
enum class Level { Chunk, Action, Token };
const char* level_name(Level level);
Level level_from_name(const std::string& name);
bool coarser_than(Level a, Level b);

struct GranularitySpec {
  Level advantage_level = Level::Chunk;
  Level logprob_level = Level::Chunk;
  Level value_level = Level::Chunk;
  bool operator==(const GranularitySpec&) const = default;
};

void validate_granularity(const GranularitySpec& spec);

namespace policy {
enum class ValueHeadKind { Scalar, Vector };

/// policy::PolicyDescriptor (policy_net.hpp:15-26).
struct PolicyDescriptor {
  int obs_dim = 1;
  int hidden = 32;
  int trunk_layers = 2;
  int value_hidden = 32;
  int vocab = 4;
  int C = 4;
  int M = 2;
  bool operator==(const PolicyDescriptor&) const = default;
};
/// save_checkpoint / load_checkpoint (policy/checkpoint.cpp:37-83) over a descriptor and its
/// flat f64 parameters (the layout of policy_net.cpp:107-152); the same CKRL v1 bytes, and the
/// reference's Error cases.
void save_checkpoint(const PolicyDescriptor& desc, std::span<const double> params, const std::string& path);
std::pair<PolicyDescriptor, std::vector<double>> load_checkpoint(const std::string& path);

/// The per-position logits gradient PolicyNet::accumulate_chunk_gradient forms before its
/// outer_add / trunk backward (policy/policy_net.cpp:431-456), on the device: logits rows
/// [P][vocab] (e.g. forward_logits outputs), tokens [P], coefficients [P] (ppo_loss's
/// LossCoefficients or GRPO's, entropy optional) -> dlogits [P][vocab]. Positions with both
/// coefficients zero give zero rows; a non-finite coefficient throws NonFinite (:437-438).
std::vector<double> chunk_logits_gradient(std::span<const double> logits, int vocab,
                                          std::span<const int> tokens,
                                          std::span<const double> coeff_logprob,
                                          std::span<const double> coeff_entropy = {});
}  // namespace policy

/// PolicyNet::value (policy_net.hpp:82): 1 entry for the scalar head, C for the vector head.
using ValueFn = std::function<std::vector<double>(const Observation&, policy::ValueHeadKind)>;
/// PolicyNet::forward_logits (policy_net.hpp:64-65): vocab logits given the chunk prefix.
using LogitsFn = std::function<std::vector<double>(const Observation&, std::span<const int>)>;

namespace detail {
struct DeviceSlab;  // the slab in the ckrl_rollout SoA layout, in HBM
}

// ---- advantage ----------------------------------------------------------------------------------
namespace advantage {

struct GaeParams {
  double gamma = 0.99;
  double lambda = 0.95;
  bool operator==(const GaeParams&) const = default;
};

struct GaeResult {
  std::vector<double> advantages;
  std::vector<double> returns;
};

GaeResult compute_gae(std::span<const double> rewards, std::span<const double> values,
                      std::span<const double> bootstrap, const std::vector<bool>& terminated,
                      const std::vector<bool>& truncated, const GaeParams& params);
GaeResult compute_gae(std::span<const double> rewards, std::span<const double> values,
                      double bootstrap, const std::vector<bool>& terminated,
                      const std::vector<bool>& truncated, const GaeParams& params);

struct GroupBatch {
  GroupKey key;
  std::vector<double> total_rewards;
  std::vector<std::int64_t> lengths;
  std::vector<std::int64_t> first_success;
  std::vector<std::int64_t> episode_uids;
  std::vector<int> env_ids;
  std::size_t size() const { return total_rewards.size(); }
};

struct FilterBounds {
  double lower = 0.0;
  double upper = 1.0;
  bool operator==(const FilterBounds&) const = default;
};

std::vector<double> grpo_group_advantage(const GroupBatch& batch, double eps_std);
double group_mean_return(const GroupBatch& batch);
std::vector<GroupBatch> success_rate_filter(const std::vector<GroupBatch>& groups,
                                            const FilterBounds& bounds);
std::vector<bool> valid_action_mask(std::int64_t length, bool success, std::int64_t first_success_step);
std::vector<double> length_norm_weights(std::int64_t length, bool success,
                                        std::int64_t first_success_step, bool length_normalized);

struct PpoRecordView {
  const StepRecord* rec = nullptr;
  int env = 0;
  int chunk_index = 0;
  std::vector<bool> counted;
  std::vector<double> advantages;  // f32 on the device, widened
  std::vector<double> returns;
};

struct PpoBatch {
  GranularitySpec spec;
  int C = 0, M = 0;
  std::vector<PpoRecordView> records;  // [env * num_chunks + chunk]
  std::int64_t advantage_unit_count() const;
  std::shared_ptr<detail::DeviceSlab> device;  // SoA slab + batch arrays + workspace in HBM
};

struct TrajChunk {
  const StepRecord* rec = nullptr;
  std::vector<int> slots;
  std::vector<double> slot_weights;
};

struct GrpoTrajectory {
  std::int64_t episode_uid = -1;
  int env = 0;
  double advantage = 0.0;
  std::vector<TrajChunk> chunks;
};

struct GrpoGroup {
  GroupKey key;
  std::vector<GrpoTrajectory> trajectories;
};

struct GrpoBatch {
  GranularitySpec spec;
  int C = 0, M = 0;
  std::vector<GrpoGroup> groups;
  std::shared_ptr<detail::DeviceSlab> device;
};

struct PpoAssemblyOptions {
  GaeParams gae;
  GranularitySpec spec;
};

/// assemble_ppo_batch (assembler.cpp:78-195) on the device. `snapshot_value` is the snapshot
/// policy's value(); it is called for the post_obs of truncated slots and of the last slot
/// of every open segment, exactly where the reference bootstraps.
PpoBatch assemble_ppo_batch(const TrajectorySlab& slab, const ValueFn& snapshot_value,
                            const PpoAssemblyOptions& options);

struct GrpoAssemblyOptions {
  GranularitySpec spec;
  double eps_std = 1e-8;
  bool apply_filter = true;
  FilterBounds filter_bounds;
  bool length_normalized = true;
  int min_group_size = 2;
};

struct GrpoAssemblyResult {
  GrpoBatch batch;
  int groups_total = 0;
  int groups_retained = 0;
};

GrpoAssemblyResult assemble_grpo_batch(const TrajectorySlab& slab, const GrpoAssemblyOptions& options);

double slab_success_rate(const TrajectorySlab& slab);

}  // namespace advantage

// ---- optim --------------------------------------------------------------------------------------
namespace optim {

struct PpoParams {
  double clip_eps = 0.2;
  double value_loss_coef = 0.5;
  double entropy_coef = 0.0;
  int epochs_per_batch = 4;
  int minibatch_size = 64;
  double learning_rate = 3e-4;
  double max_grad_norm = 1.0;
  bool advantage_normalization = true;
};

struct GrpoParams {
  double clip_eps = 0.2;
  int epochs_per_batch = 1;
  int minibatch_groups = 0;
  double learning_rate = 3e-4;
  double max_grad_norm = 1.0;
};

struct LossDiagnostics {
  double loss = 0.0;
  double surrogate = 0.0;
  double value_loss = 0.0;
  double entropy = 0.0;
  double clip_frac = 0.0;
  double approx_kl = 0.0;
  std::int64_t units = 0;
};

/// The current policy as the loss sees it. Either its two public calls (filled for the
/// selected records only, like the reference's evaluate_chunk / value), or a view of its
/// logits [E][Tc][C][M][V] (f32 or bf16) and new values (value-level shape, f32) for every
/// record, on the device (`device = true`) or in host memory. With logits_dtype =
/// CKRL_DTYPE_TOKEN_ROWS the view is [E][Tc][C][M] ckrl_token_row instead: the policy head
/// already reduced on the tensor cores (ckrl_project_token_stats over the trunk features,
/// PolicyNet::logits_from_feature + evaluate_chunk, policy_net.cpp:265-284, 333-357).
struct CurrentPolicy {
  LogitsFn forward_logits;
  ValueFn value;
  const void* logits = nullptr;
  int32_t logits_dtype = CKRL_DTYPE_F32;
  const float* values = nullptr;
  int vocab = 0;
  bool device = true;
};

/// Per-position loss coefficients of the evaluated records, in selection order
/// ([n][C][M] and value-level shape): what accumulate_chunk_gradient /
/// accumulate_value_gradient receive (losses.cpp:192-218).
struct LossCoefficients {
  std::vector<double> coeff_logprob, coeff_entropy, coeff_value;
};

void normalize_advantages(advantage::PpoBatch& batch);

/// optim::Adam (optim/adam.hpp:10-27) with its moments resident on the device (float64, the
/// reference's precision). step() takes host spans like the reference — grad is clipped in
/// place, the pre-clip norm is returned, NonFinite leaves everything untouched;
/// step_device() runs on device-resident params / grad (n doubles each) with no copies.
class Adam {
 public:
  Adam(std::size_t num_params, double learning_rate, double max_grad_norm = 0.0, double beta1 = 0.9,
       double beta2 = 0.999, double eps = 1e-8);
  ~Adam();
  Adam(const Adam&) = delete;
  Adam& operator=(const Adam&) = delete;
  double step(std::span<double> params, std::span<double> grad);
  double step_device(double* params, double* grad);

 private:
  struct State;
  State* s_;
};

LossDiagnostics ppo_loss(const CurrentPolicy& net, const advantage::PpoBatch& batch,
                         std::span<const std::size_t> record_indices, const PpoParams& params,
                         LossCoefficients* coefficients = nullptr);

LossDiagnostics grpo_loss(const CurrentPolicy& net, const advantage::GrpoBatch& batch,
                          std::span<const std::size_t> group_indices, const GrpoParams& params);

}  // namespace optim

}  // namespace ckrl::chunkrl
