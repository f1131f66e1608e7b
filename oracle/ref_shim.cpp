// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference ("chunkrl", /root/reference/proj/src),
// compiled together with the reference's own sources by oracle/Makefile into
// oracle/_ref/libchunkrl_ref.so. It lets the Python fixture generator, the CPU
// tests and bench.py's reference arm drive the reference through its public API:
//
//   rollout     placement::StageSim / StageGen / merge_stages   (placement/rollout.cpp:11-109)
//   advantage   advantage::assemble_ppo_batch / assemble_grpo_batch (advantage/assembler.cpp:78-267)
//   update      optim::normalize_advantages                     (optim/update.cpp:14-45)
//   loss        optim::ppo_loss / grpo_loss                     (optim/losses.cpp:62-331)
//   policy      PolicyNet::evaluate_chunk / forward_logits / value (policy/policy_net.cpp)
//
// Everything the reference computes internally from its PolicyNet (current-policy
// logits, new values, bootstrap values) is exported as plain arrays in the SoA
// layout that include/ckrl.h defines, so the same inputs can be replayed through
// the oracle restatement and the CUDA path.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <thread>
#include <vector>

#include "chunkrl/advantage/assembler.hpp"
#include "chunkrl/core/errors.hpp"
#include "chunkrl/core/rng.hpp"
#include "chunkrl/optim/adam.hpp"
#include "chunkrl/policy/checkpoint.hpp"
#include "chunkrl/optim/losses.hpp"
#include "chunkrl/optim/update.hpp"
#include "chunkrl/placement/rollout.hpp"
#include "chunkrl/policy/policy_net.hpp"

using namespace chunkrl;

namespace {

struct Scenario {
  policy::PolicyNet snapshot; // rollout (old) policy: sampled tokens, old logprobs, bootstraps
  policy::PolicyNet current;  // policy under optimisation: new logits / values
  TrajectorySlab slab;
  std::vector<int> reset_ids; // RolloutSpec::reset_state_ids (empty: none)
  int E = 0, Tc = 0, C = 0, M = 0, V = 0;
};

// Status codes mirror include/ckrl.h (1:1 with chunkrl/core/errors.hpp).
int status_of(const std::exception& ex) {
  if (dynamic_cast<const UnsupportedCombination*>(&ex)) return 1;
  if (dynamic_cast<const GranularityOrderViolation*>(&ex)) return 2;
  if (dynamic_cast<const LengthMismatch*>(&ex)) return 3;
  if (dynamic_cast<const BadResetId*>(&ex)) return 4;
  if (dynamic_cast<const HeadMismatch*>(&ex)) return 5;
  if (dynamic_cast<const NonFinite*>(&ex)) return 6;
  if (dynamic_cast<const DegenerateGroup*>(&ex)) return 7;
  if (dynamic_cast<const SkipUpdate*>(&ex)) return 8;
  if (dynamic_cast<const InvalidPlan*>(&ex)) return 9;
  if (dynamic_cast<const MemoryOverflow*>(&ex)) return 10;
  if (dynamic_cast<const EmptyTrace*>(&ex)) return 11;
  if (dynamic_cast<const ConfigError*>(&ex)) return 12;
  if (dynamic_cast<const Error*>(&ex)) return 13;
  return 99;
}

Level level_of(int l) { return l == 0 ? Level::Chunk : (l == 1 ? Level::Action : Level::Token); }

void diag_out(const optim::LossDiagnostics& d, double* out) {
  out[0] = d.loss;
  out[1] = d.surrogate;
  out[2] = d.value_loss;
  out[3] = d.entropy;
  out[4] = d.clip_frac;
  out[5] = d.approx_kl;
  out[6] = static_cast<double>(d.units);
}

} // namespace

extern "C" {

struct refx_cfg {
  int env_kind; // 0 toy_reach, 1 scripted
  int num_envs;
  int max_episode_steps;
  int auto_reset;
  int ignore_terminations;
  int use_fixed_reset_state_ids;
  int chunk_length;
  int grid_size;
  int num_reset_states;
  int success_step;
  int reward_shaping;
  int num_chunks;
  int deferred_reset;
  int group_size;        // fixed ids: envs [g*G, (g+1)*G) share one id
  int ids_with_replacement; // 1: draw ids like train.cpp:92-101; 0: id = g % table
  int vocab;
  int tokens_per_action;
  int hidden;
  int trunk_layers;
  int value_hidden;
  unsigned long long env_seed;
  unsigned long long sample_seed;
  unsigned long long net_seed;
  double perturb; // N(0,1)*perturb added to every parameter of the current policy
};

static thread_local std::string g_err;

const char* refx_last_error() { return g_err.c_str(); }

void* refx_create(const refx_cfg* cfg, int* status) {
  try {
    placement::RolloutSpec spec;
    envsim::VecEnvConfig& ec = spec.env_config;
    ec.kind = cfg->env_kind == 0 ? envsim::EnvKind::ToyReach : envsim::EnvKind::Scripted;
    ec.num_envs = cfg->num_envs;
    ec.max_episode_steps = cfg->max_episode_steps;
    ec.auto_reset = cfg->auto_reset != 0;
    ec.ignore_terminations = cfg->ignore_terminations != 0;
    ec.use_fixed_reset_state_ids = cfg->use_fixed_reset_state_ids != 0;
    ec.seed = cfg->env_seed;
    ec.chunk_length = cfg->chunk_length;
    ec.grid_size = cfg->grid_size;
    ec.reward_shaping = cfg->reward_shaping != 0;
    ec.num_reset_states = cfg->num_reset_states;
    ec.success_step = cfg->success_step;
    spec.num_chunks = cfg->num_chunks;
    spec.reset_mode = cfg->deferred_reset ? envsim::ResetMode::Deferred : envsim::ResetMode::Immediate;
    spec.sample_seed = cfg->sample_seed;
    if (ec.use_fixed_reset_state_ids) {
      std::vector<int> ids(static_cast<std::size_t>(ec.num_envs), 0);
      Rng rid(mix_seed(cfg->env_seed, 0x1d5ull));
      int G = std::max(1, cfg->group_size);
      for (int g = 0; g * G < ec.num_envs; ++g) {
        int id = cfg->ids_with_replacement
                     ? static_cast<int>(rid.next_below(static_cast<std::uint64_t>(ec.num_reset_states)))
                     : g % ec.num_reset_states;
        for (int m = 0; m < G && g * G + m < ec.num_envs; ++m)
          ids[static_cast<std::size_t>(g * G + m)] = id;
      }
      spec.reset_state_ids = std::move(ids);
    }

    envsim::VecEnv probe(ec, 0, 1);
    policy::PolicyDescriptor desc;
    desc.obs_dim = probe.observation_dim();
    desc.hidden = cfg->hidden;
    desc.trunk_layers = cfg->trunk_layers;
    desc.value_hidden = cfg->value_hidden;
    desc.vocab = cfg->vocab;
    desc.C = cfg->chunk_length;
    desc.M = cfg->tokens_per_action;

    // The reference initialises output layers to zero (uniform policy, zero
    // values); perturb every parameter so logits, values and ratios are generic.
    policy::PolicyNet snap = policy::PolicyNet::initialized(desc, cfg->net_seed);
    {
      Rng r(mix_seed(cfg->net_seed, 0x5eedull));
      std::vector<double> p = snap.params();
      for (double& x : p)
        x += 0.3 * r.next_normal();
      snap.set_params(std::move(p));
    }
    policy::PolicyNet cur = snap;
    {
      Rng r(mix_seed(cfg->net_seed, 0xc0ffeeull));
      std::vector<double> p = cur.params();
      for (double& x : p)
        x += cfg->perturb * r.next_normal();
      cur.set_params(std::move(p));
    }

    std::vector<placement::StageSim> stages;
    stages.emplace_back(spec, 0, 1);
    placement::StageGen gen(snap, spec);
    std::vector<Observation> obs = stages[0].initial_obs();
    for (int t = 0; t < spec.num_chunks; ++t) {
      placement::GenBatch b = gen.generate(stages[0].first_env_id(), obs);
      obs = stages[0].execute(b);
    }
    auto* s = new Scenario{snap, cur, placement::merge_stages(spec, stages),
                           spec.reset_state_ids.value_or(std::vector<int>{})};
    // merge_stages probes M from the env (hard-coded 2); the policy defines it here.
    s->slab.tokens_per_action = desc.M;
    s->E = ec.num_envs;
    s->Tc = spec.num_chunks;
    s->C = desc.C;
    s->M = desc.M;
    s->V = desc.vocab;
    *status = 0;
    return s;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    *status = status_of(ex);
    return nullptr;
  }
}

// The reference's own optim::Adam (optim/adam.cpp) for `steps` steps; grads[s*n + i] is the
// gradient of step s (clipped in place, as the reference does). Returns the status of the
// first failing step; norms[s] the pre-clip norm of each step.
int refx_adam(long long n, int steps, double* params, double* grads, double lr, double max_grad_norm,
              double beta1, double beta2, double eps, double* norms) {
  try {
    optim::Adam adam(static_cast<std::size_t>(n), lr, max_grad_norm, beta1, beta2, eps);
    for (int s = 0; s < steps; ++s)
      norms[s] = adam.step(std::span<double>(params, static_cast<std::size_t>(n)),
                           std::span<double>(grads + static_cast<std::size_t>(s) * n, static_cast<std::size_t>(n)));
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return status_of(ex);
  }
}

// The policy head through the reference's public PolicyNet API, per position: a net with
// obs_dim 1, no trunk layers and C = M = 1, whose input bias b_in is set to the position's
// feature h (pos_bias and the embeddings zero, obs = {0}), so trunk_forward's x is exactly h
// (policy_net.cpp:206-210) and forward_logits returns logits_from_feature(h) = W_pol h + b_pol
// (:265-284); evaluate_chunk then gives the token's log-prob and entropy (:333-357).
// Parameter offsets follow PolicyNet::Layout (:114-143). logits [rows][V], lp / ent [rows].
int refx_project_token_stats(long long rows, int H, int V, const double* feature, const double* W,
                             const double* b, const int* tokens, double* logits, double* lp, double* ent) {
  try {
    policy::PolicyDescriptor d;
    d.obs_dim = 1;
    d.hidden = H;
    d.trunk_layers = 0;
    d.value_hidden = 1;
    d.vocab = V;
    d.C = 1;
    d.M = 1;
    policy::PolicyNet net(d);
    std::vector<double> p(net.num_params(), 0.0);
    const std::size_t b_in = static_cast<std::size_t>(H), emb = 3 * static_cast<std::size_t>(H);
    const std::size_t w_pol = emb + static_cast<std::size_t>(V) * H, b_pol = w_pol + static_cast<std::size_t>(V) * H;
    std::copy(W, W + static_cast<std::size_t>(V) * H, p.begin() + static_cast<std::ptrdiff_t>(w_pol));
    if (b) std::copy(b, b + V, p.begin() + static_cast<std::ptrdiff_t>(b_pol));
    const Observation obs{0.0};
    for (long long k = 0; k < rows; ++k) {
      std::copy(feature + k * H, feature + (k + 1) * H, p.begin() + static_cast<std::ptrdiff_t>(b_in));
      net.set_params(p);
      const std::vector<double> lg = net.forward_logits(obs, {});
      std::copy(lg.begin(), lg.end(), logits + k * V);
      ActionChunk ch;
      ch.actions.resize(1);
      ch.actions[0].tokens = {tokens[k]};
      const policy::ChunkEval ev = net.evaluate_chunk(obs, ch);
      lp[k] = ev.token_logprobs.values[0];
      ent[k] = ev.entropy[0];
    }
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return status_of(ex);
  }
}

// The reference's own dump_slab (core/types.cpp:9-28) of the scenario's slab; *len gets the
// full length, at most cap bytes are copied.
int refx_dump_slab(void* h, char* out, size_t cap, size_t* len) {
  const std::string text = dump_slab(static_cast<Scenario*>(h)->slab);
  *len = text.size();
  if (out && cap) std::memcpy(out, text.data(), std::min(cap, text.size()));
  return 0;
}

// save_checkpoint / load_checkpoint (policy/checkpoint.cpp:37-83) of the rollout snapshot.
int refx_save_checkpoint(void* h, const char* path) {
  try {
    policy::save_checkpoint(static_cast<Scenario*>(h)->snapshot, path);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return status_of(ex);
  }
}
int refx_load_checkpoint(const char* path, int* desc7, double* params, long long cap, long long* count) {
  try {
    policy::PolicyNet net = policy::load_checkpoint(path);
    const policy::PolicyDescriptor& d = net.descriptor();
    const int f[7] = {d.obs_dim, d.hidden, d.trunk_layers, d.value_hidden, d.vocab, d.C, d.M};
    std::memcpy(desc7, f, sizeof f);
    *count = static_cast<long long>(net.num_params());
    if (params && *count <= cap) std::memcpy(params, net.params().data(), sizeof(double) * net.num_params());
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return status_of(ex);
  }
}

void refx_destroy(void* h) { delete static_cast<Scenario*>(h); }

// Offset of the policy-head bias b_pol in the flat parameter vector (policy_net.cpp:107-152
// order: w_in, b_in, pos_bias, emb, trunk, w_pol, b_pol, ...). Its gradient slice is the sum
// over evaluated positions of the per-position logits gradient (outer_add, :451-452).
long long refx_bpol_offset(void* h) {
  const policy::PolicyDescriptor& d = static_cast<Scenario*>(h)->current.descriptor();
  const long long H = d.hidden, D = d.obs_dim, L = d.trunk_layers, V = d.vocab, P = d.positions();
  return H * D + H + P * H + P * V * H + L * (H * H + H) + V * H;
}

void refx_dims(void* h, long long* dims) {
  auto* s = static_cast<Scenario*>(h);
  dims[0] = s->E;
  dims[1] = s->Tc;
  dims[2] = s->C;
  dims[3] = s->M;
  dims[4] = s->V;
  dims[5] = static_cast<long long>(s->slab.episodes.size());
  dims[6] = static_cast<long long>(s->current.num_params());
}

// The rollout policy's flat parameter vector (policy_net.cpp:107-152 order) and the
// spec's reset ids, so the CUDA pipeline can replay the same rollout.
int refx_export_params(void* h, double* snapshot_params, int32_t* reset_ids) {
  auto* s = static_cast<Scenario*>(h);
  const std::vector<double>& p = s->snapshot.params();
  std::memcpy(snapshot_params, p.data(), sizeof(double) * p.size());
  if (reset_ids)
    for (int e = 0; e < s->E; ++e)
      reset_ids[e] = s->reset_ids.empty() ? -1 : s->reset_ids[static_cast<std::size_t>(e)];
  return s->reset_ids.empty() ? 0 : 1;
}

// SoA export. Layout per include/ckrl.h: [E][Tc][C][M](...[V]).
int refx_export(void* h, int32_t* tokens, double* old_lp, double* reward, uint8_t* flags,
                int32_t* episode_id, double* value_scalar, double* value_vector,
                double* boot_scalar, double* boot_vector0, double* logits,
                double* new_value_scalar, double* new_value_vector, double* lp_cur,
                double* ent_cur) {
  auto* s = static_cast<Scenario*>(h);
  try {
    const int C = s->C, M = s->M, V = s->V;
    for (int e = 0; e < s->E; ++e) {
      const auto& recs = s->slab.records[static_cast<std::size_t>(e)];
      for (int t = 0; t < s->Tc; ++t) {
        const StepRecord& rec = recs[static_cast<std::size_t>(t)];
        std::size_t rt = static_cast<std::size_t>(e) * s->Tc + t;
        value_scalar[rt] = rec.value_scalar;
        std::vector<double> nvs = s->current.value(rec.obs, policy::ValueHeadKind::Scalar);
        std::vector<double> nvv = s->current.value(rec.obs, policy::ValueHeadKind::Vector);
        new_value_scalar[rt] = nvs[0];
        policy::ChunkEval ev = s->current.evaluate_chunk(rec.obs, rec.chunk);
        std::vector<int> prefix;
        for (int j = 0; j < C; ++j) {
          std::size_t sl = rt * C + j;
          reward[sl] = rec.rewards[static_cast<std::size_t>(j)];
          flags[sl] = static_cast<uint8_t>((rec.terminated[static_cast<std::size_t>(j)] ? 1 : 0) |
                                           (rec.truncated[static_cast<std::size_t>(j)] ? 2 : 0) |
                                           (rec.valid[static_cast<std::size_t>(j)] ? 4 : 0));
          std::int64_t uid = rec.episode_uid[static_cast<std::size_t>(j)];
          episode_id[sl] = uid < 0 ? -1 : static_cast<int32_t>(uid & 0xffffffff);
          value_vector[sl] = rec.value_vector[static_cast<std::size_t>(j)];
          new_value_vector[sl] = nvv[static_cast<std::size_t>(j)];
          boot_scalar[sl] = s->snapshot.value(rec.post_obs[static_cast<std::size_t>(j)],
                                              policy::ValueHeadKind::Scalar)[0];
          boot_vector0[sl] = s->snapshot.value(rec.post_obs[static_cast<std::size_t>(j)],
                                               policy::ValueHeadKind::Vector)[0];
          for (int m = 0; m < M; ++m) {
            std::size_t tk = sl * M + m;
            int tok = rec.chunk.actions[static_cast<std::size_t>(j)].tokens[static_cast<std::size_t>(m)];
            tokens[tk] = tok;
            old_lp[tk] = rec.token_logprobs.at(j, m);
            std::vector<double> lg = s->current.forward_logits(rec.obs, prefix);
            std::memcpy(logits + tk * V, lg.data(), sizeof(double) * V);
            lp_cur[tk] = ev.token_logprobs.at(j, m);
            ent_cur[tk] = ev.entropy[static_cast<std::size_t>(j * M + m)];
            prefix.push_back(tok);
          }
        }
      }
    }
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return status_of(ex);
  }
}

int refx_export_episodes(void* h, int32_t* env_id, int32_t* episode_id, int64_t* start,
                         int64_t* length, double* total_reward, int64_t* first_success,
                         uint8_t* success, uint8_t* complete, int32_t* task, int32_t* reset_id) {
  auto* s = static_cast<Scenario*>(h);
  for (std::size_t i = 0; i < s->slab.episodes.size(); ++i) {
    const EpisodeInfo& ep = s->slab.episodes[i];
    env_id[i] = ep.env_id;
    episode_id[i] = static_cast<int32_t>(ep.uid & 0xffffffff);
    start[i] = ep.start_step;
    length[i] = ep.length;
    total_reward[i] = ep.total_reward;
    first_success[i] = ep.first_success_step;
    success[i] = ep.success ? 1 : 0;
    complete[i] = ep.complete ? 1 : 0;
    task[i] = ep.group_key.task_id;
    reset_id[i] = ep.group_key.reset_state_id;
  }
  return 0;
}

// assemble_ppo_batch -> [normalize_advantages] -> ppo_loss over every record in
// batch order (the full-batch step). grad (optional) receives ppo_loss's grad_out.
int refx_ppo(void* h, int adv_level, int lp_level, int val_level, double gamma, double lambda,
             int normalize, double clip_eps, double vcoef, double ecoef, uint8_t* counted,
             double* adv_raw, double* ret, double* adv_norm, double* diag, double* grad) {
  auto* s = static_cast<Scenario*>(h);
  try {
    advantage::PpoAssemblyOptions opts;
    opts.gae = advantage::GaeParams{gamma, lambda};
    opts.spec = GranularitySpec{level_of(adv_level), level_of(lp_level), level_of(val_level)};
    advantage::PpoBatch batch = advantage::assemble_ppo_batch(s->slab, s->snapshot, opts);
    const int C = s->C;
    const bool action = opts.spec.advantage_level == Level::Action;
    auto dump = [&](double* out, bool from_returns) {
      for (std::size_t r = 0; r < batch.records.size(); ++r) {
        const auto& v = batch.records[r];
        const auto& src = from_returns ? v.returns : v.advantages;
        if (action)
          for (int j = 0; j < C; ++j)
            out[r * C + j] = src[static_cast<std::size_t>(j)];
        else
          out[r] = src[0];
      }
    };
    for (std::size_t r = 0; r < batch.records.size(); ++r)
      for (int j = 0; j < C; ++j)
        counted[r * C + j] = batch.records[r].counted[static_cast<std::size_t>(j)] ? 1 : 0;
    dump(adv_raw, false);
    dump(ret, true);
    if (normalize)
      optim::normalize_advantages(batch);
    dump(adv_norm, false);
    optim::PpoParams params;
    params.clip_eps = clip_eps;
    params.value_loss_coef = vcoef;
    params.entropy_coef = ecoef;
    std::vector<std::size_t> idx(batch.records.size());
    for (std::size_t i = 0; i < idx.size(); ++i)
      idx[i] = i;
    std::vector<double> g;
    if (grad)
      g.assign(s->current.num_params(), 0.0);
    optim::LossDiagnostics d = optim::ppo_loss(s->current, batch, idx, params, grad ? &g : nullptr);
    diag_out(d, diag);
    if (grad)
      std::memcpy(grad, g.data(), sizeof(double) * g.size());
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return status_of(ex);
  }
}

// Replays per-position / per-unit coefficients through the reference's public
// gradient seam in ppo_loss's order (losses.cpp:259-285): per record with any
// counted slot, accumulate_chunk_gradient then accumulate_value_gradient.
int refx_replay_ppo_grad(void* h, int val_level, const uint8_t* counted, const double* coeff_lp,
                         const double* coeff_ent, const double* coeff_val, double* grad) {
  auto* s = static_cast<Scenario*>(h);
  try {
    const int C = s->C, P = s->C * s->M;
    std::vector<double> g(s->current.num_params(), 0.0);
    for (int e = 0; e < s->E; ++e)
      for (int t = 0; t < s->Tc; ++t) {
        std::size_t rt = static_cast<std::size_t>(e) * s->Tc + t;
        bool any = false;
        for (int j = 0; j < C; ++j)
          any = any || counted[rt * C + j];
        if (!any)
          continue;
        const StepRecord& rec = s->slab.records[static_cast<std::size_t>(e)][static_cast<std::size_t>(t)];
        s->current.accumulate_chunk_gradient(rec.obs, rec.chunk,
                                             std::span<const double>(coeff_lp + rt * P, P),
                                             std::span<const double>(coeff_ent + rt * P, P), g);
        if (val_level == 0) {
          s->current.accumulate_value_gradient(rec.obs, policy::ValueHeadKind::Scalar,
                                               std::span<const double>(coeff_val + rt, 1), g);
        } else {
          bool any_val = false;
          for (int j = 0; j < C; ++j)
            any_val = any_val || counted[rt * C + j];
          if (any_val)
            s->current.accumulate_value_gradient(rec.obs, policy::ValueHeadKind::Vector,
                                                 std::span<const double>(coeff_val + rt * C, C), g);
        }
      }
    std::memcpy(grad, g.data(), sizeof(double) * g.size());
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return status_of(ex);
  }
}

// Minibatch forms: ppo_loss over record_indices (whitening once over the whole batch first,
// update.cpp:66-67) and grpo_loss over group_indices, in the given order.
int refx_ppo_subset(void* h, int adv_level, int lp_level, int val_level, double gamma, double lambda,
                    int normalize, double clip_eps, double vcoef, double ecoef, long long n,
                    const long long* idx, double* diag) {
  auto* s = static_cast<Scenario*>(h);
  try {
    advantage::PpoAssemblyOptions opts;
    opts.gae = advantage::GaeParams{gamma, lambda};
    opts.spec = GranularitySpec{level_of(adv_level), level_of(lp_level), level_of(val_level)};
    advantage::PpoBatch batch = advantage::assemble_ppo_batch(s->slab, s->snapshot, opts);
    if (normalize)
      optim::normalize_advantages(batch);
    optim::PpoParams params;
    params.clip_eps = clip_eps;
    params.value_loss_coef = vcoef;
    params.entropy_coef = ecoef;
    std::vector<std::size_t> sel(static_cast<std::size_t>(n));
    for (long long i = 0; i < n; ++i)
      sel[static_cast<std::size_t>(i)] = static_cast<std::size_t>(idx[i]);
    diag_out(optim::ppo_loss(s->current, batch, sel, params, nullptr), diag);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return status_of(ex);
  }
}

int refx_grpo_subset(void* h, int adv_level, int lp_level, int val_level, double eps_std, int apply_filter,
                     double lower, double upper, int length_normalized, int min_group_size,
                     double clip_eps, long long n, const long long* idx, double* diag) {
  auto* s = static_cast<Scenario*>(h);
  try {
    advantage::GrpoAssemblyOptions o;
    o.spec = GranularitySpec{level_of(adv_level), level_of(lp_level), level_of(val_level)};
    o.eps_std = eps_std;
    o.apply_filter = apply_filter != 0;
    o.filter_bounds = advantage::FilterBounds{lower, upper};
    o.length_normalized = length_normalized != 0;
    o.min_group_size = min_group_size;
    advantage::GrpoAssemblyResult res = advantage::assemble_grpo_batch(s->slab, o);
    optim::GrpoParams p;
    p.clip_eps = clip_eps;
    std::vector<std::size_t> sel(static_cast<std::size_t>(n));
    for (long long i = 0; i < n; ++i)
      sel[static_cast<std::size_t>(i)] = static_cast<std::size_t>(idx[i]);
    diag_out(optim::grpo_loss(s->current, res.batch, sel, p, nullptr), diag);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return status_of(ex);
  }
}

// assemble_grpo_batch -> grpo_loss over every retained group. Per-env outputs
// describe the (at most one) retained trajectory each env owns; slot_weight is
// the trajectory's per-slot weight (0 outside it).
int refx_grpo(void* h, int adv_level, int lp_level, int val_level, double eps_std, int apply_filter,
              double lower, double upper, int length_normalized, int min_group_size,
              double clip_eps, int* groups_total, int* groups_retained, int32_t* env_group,
              int32_t* env_member, int32_t* env_episode, double* env_adv, int32_t* env_group_size,
              double* slot_weight, uint8_t* slot_member, double* diag, double* grad) {
  auto* s = static_cast<Scenario*>(h);
  try {
    advantage::GrpoAssemblyOptions o;
    o.spec = GranularitySpec{level_of(adv_level), level_of(lp_level), level_of(val_level)};
    o.eps_std = eps_std;
    o.apply_filter = apply_filter != 0;
    o.filter_bounds = advantage::FilterBounds{lower, upper};
    o.length_normalized = length_normalized != 0;
    o.min_group_size = min_group_size;
    advantage::GrpoAssemblyResult res = advantage::assemble_grpo_batch(s->slab, o);
    *groups_total = res.groups_total;
    *groups_retained = res.groups_retained;
    const int C = s->C;
    for (int e = 0; e < s->E; ++e) {
      env_group[e] = -1;
      env_member[e] = -1;
      env_episode[e] = -1;
      env_adv[e] = 0.0;
      env_group_size[e] = 0;
    }
    std::size_t nslot = static_cast<std::size_t>(s->E) * s->Tc * C;
    std::fill(slot_weight, slot_weight + nslot, 0.0);
    std::fill(slot_member, slot_member + nslot, 0);
    for (std::size_t gi = 0; gi < res.batch.groups.size(); ++gi) {
      const auto& grp = res.batch.groups[gi];
      for (std::size_t ti = 0; ti < grp.trajectories.size(); ++ti) {
        const auto& tr = grp.trajectories[ti];
        if (env_group[tr.env] >= 0) {
          g_err = "env owns two retained trajectories";
          return 13;
        }
        env_group[tr.env] = static_cast<int32_t>(gi);
        env_member[tr.env] = static_cast<int32_t>(ti);
        env_episode[tr.env] = static_cast<int32_t>(tr.episode_uid & 0xffffffff);
        env_adv[tr.env] = tr.advantage;
        env_group_size[tr.env] = static_cast<int32_t>(grp.trajectories.size());
        const auto& recs = s->slab.records[static_cast<std::size_t>(tr.env)];
        for (const auto& ch : tr.chunks) {
          std::size_t t = static_cast<std::size_t>(ch.rec - recs.data());
          for (std::size_t k = 0; k < ch.slots.size(); ++k) {
            std::size_t sl = (static_cast<std::size_t>(tr.env) * s->Tc + t) * C + ch.slots[k];
            slot_weight[sl] = ch.slot_weights[k];
            slot_member[sl] = 1;
          }
        }
      }
    }
    std::vector<std::size_t> idx(res.batch.groups.size());
    for (std::size_t i = 0; i < idx.size(); ++i)
      idx[i] = i;
    optim::GrpoParams p;
    p.clip_eps = clip_eps;
    std::vector<double> g;
    if (grad)
      g.assign(s->current.num_params(), 0.0);
    optim::LossDiagnostics d = optim::grpo_loss(s->current, res.batch, idx, p, grad ? &g : nullptr);
    diag_out(d, diag);
    if (grad)
      std::memcpy(grad, g.data(), sizeof(double) * g.size());
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return status_of(ex);
  }
}

// GRPO replay in grpo_loss's traversal order (groups -> trajectories -> chunks,
// losses.cpp:318-384); coefficients come from the caller's SoA arrays.
int refx_replay_grpo_grad(void* h, int adv_level, int lp_level, double eps_std, int apply_filter,
                          double lower, double upper, int length_normalized, int min_group_size,
                          const double* coeff_lp, double* grad) {
  auto* s = static_cast<Scenario*>(h);
  try {
    advantage::GrpoAssemblyOptions o;
    o.spec = GranularitySpec{level_of(adv_level), level_of(lp_level), level_of(adv_level)};
    o.eps_std = eps_std;
    o.apply_filter = apply_filter != 0;
    o.filter_bounds = advantage::FilterBounds{lower, upper};
    o.length_normalized = length_normalized != 0;
    o.min_group_size = min_group_size;
    advantage::GrpoAssemblyResult res = advantage::assemble_grpo_batch(s->slab, o);
    const int P = s->C * s->M;
    std::vector<double> g(s->current.num_params(), 0.0), zeros(static_cast<std::size_t>(P), 0.0);
    for (const auto& grp : res.batch.groups)
      for (const auto& tr : grp.trajectories) {
        const auto& recs = s->slab.records[static_cast<std::size_t>(tr.env)];
        for (const auto& ch : tr.chunks) {
          bool any = false;
          for (double w : ch.slot_weights)
            any = any || w != 0.0;
          if (!any)
            continue;
          std::size_t t = static_cast<std::size_t>(ch.rec - recs.data());
          std::size_t rt = static_cast<std::size_t>(tr.env) * s->Tc + t;
          s->current.accumulate_chunk_gradient(ch.rec->obs, ch.rec->chunk,
                                               std::span<const double>(coeff_lp + rt * P, P),
                                               zeros, g);
        }
      }
    std::memcpy(grad, g.data(), sizeof(double) * g.size());
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return status_of(ex);
  }
}

// ---------------------------------------------------------------------------
// Reference arm timing (bench.py --impl reference). The reference hot path is
// single-threaded; the ops are pure, so the batch is sharded
// by env across `threads` std::threads (GRPO: by whole groups, here env blocks
// of group_size). Timed: assembly (+ whitening) + the loss forward over the full
// batch; grad_out = nullptr (the backward through the toy trunk is not on the
// B200 path). Returns seconds per iteration; diag receives the recombined loss.
// ---------------------------------------------------------------------------
namespace {
TrajectorySlab sub_slab(const TrajectorySlab& slab, int e0, int e1) {
  TrajectorySlab s;
  s.num_envs = e1 - e0;
  s.chunk_length = slab.chunk_length;
  s.tokens_per_action = slab.tokens_per_action;
  s.records.assign(slab.records.begin() + e0, slab.records.begin() + e1);
  for (const auto& ep : slab.episodes)
    if (ep.env_id >= e0 && ep.env_id < e1) {
      s.episodes.push_back(ep);
      s.episodes.back().env_id -= e0;  // records are re-indexed from 0 in the shard
    }
  return s;
}
} // namespace

double refx_bench_ppo(void* h, int adv_level, int lp_level, int val_level, double gamma,
                      double lambda, double clip_eps, double vcoef, double ecoef, int threads,
                      int iters, int align, double* diag) {
  auto* s = static_cast<Scenario*>(h);
  try {
    threads = std::max(1, std::min(threads, s->E));
    align = std::max(1, align);
    std::vector<TrajectorySlab> shards;
    int per = (s->E + threads - 1) / threads;
    per = (per + align - 1) / align * align;
    for (int e0 = 0; e0 < s->E; e0 += per)
      shards.push_back(sub_slab(s->slab, e0, std::min(s->E, e0 + per)));
    advantage::PpoAssemblyOptions opts;
    opts.gae = advantage::GaeParams{gamma, lambda};
    opts.spec = GranularitySpec{level_of(adv_level), level_of(lp_level), level_of(val_level)};
    optim::PpoParams params;
    params.clip_eps = clip_eps;
    params.value_loss_coef = vcoef;
    params.entropy_coef = ecoef;
    const int P = static_cast<int>(shards.size());
    double total = 0.0;
    for (int it = 0; it < iters; ++it) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<advantage::PpoBatch> parts(static_cast<std::size_t>(P));
      {
        std::vector<std::thread> pool;
        for (int p = 0; p < P; ++p)
          pool.emplace_back([&, p] {
            parts[static_cast<std::size_t>(p)] =
                advantage::assemble_ppo_batch(shards[static_cast<std::size_t>(p)], s->snapshot, opts);
          });
        for (auto& th : pool)
          th.join();
      }
      advantage::PpoBatch all;
      all.spec = opts.spec;
      all.C = s->C;
      all.M = s->M;
      std::vector<std::size_t> bounds{0};
      for (auto& part : parts) {
        for (auto& v : part.records)
          all.records.push_back(std::move(v));
        bounds.push_back(all.records.size());
      }
      optim::normalize_advantages(all);
      std::vector<optim::LossDiagnostics> ds(static_cast<std::size_t>(P));
      std::vector<std::int64_t> nadv(static_cast<std::size_t>(P), 0);
      {
        std::vector<std::thread> pool;
        for (int p = 0; p < P; ++p)
          pool.emplace_back([&, p] {
            std::vector<std::size_t> idx;
            for (std::size_t i = bounds[static_cast<std::size_t>(p)]; i < bounds[static_cast<std::size_t>(p) + 1]; ++i)
              idx.push_back(i);
            ds[static_cast<std::size_t>(p)] = optim::ppo_loss(s->current, all, idx, params, nullptr);
          });
        for (auto& th : pool)
          th.join();
      }
      auto t1 = std::chrono::steady_clock::now();
      total += std::chrono::duration<double>(t1 - t0).count();
      if (diag && it == iters - 1)
        diag_out(ds[0], diag); // shard 0's diagnostics (timing run; parity lives in the tests)
    }
    return total / std::max(1, iters);
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -static_cast<double>(status_of(ex));
  }
}

double refx_bench_grpo(void* h, int adv_level, int lp_level, double eps_std, int length_normalized,
                       double clip_eps, int threads, int iters, int align, double* diag, int apply_filter) {
  auto* s = static_cast<Scenario*>(h);
  try {
    threads = std::max(1, std::min(threads, s->E));
    align = std::max(1, align);
    std::vector<TrajectorySlab> shards;
    int per = (s->E + threads - 1) / threads;
    per = (per + align - 1) / align * align;
    for (int e0 = 0; e0 < s->E; e0 += per)
      shards.push_back(sub_slab(s->slab, e0, std::min(s->E, e0 + per)));
    advantage::GrpoAssemblyOptions o;
    o.spec = GranularitySpec{level_of(adv_level), level_of(lp_level), level_of(adv_level)};
    o.eps_std = eps_std;
    o.length_normalized = length_normalized != 0;
    o.apply_filter = apply_filter != 0;
    optim::GrpoParams gp;
    gp.clip_eps = clip_eps;
    const int P = static_cast<int>(shards.size());
    double total = 0.0;
    for (int it = 0; it < iters; ++it) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<optim::LossDiagnostics> ds(static_cast<std::size_t>(P));
      std::vector<std::thread> pool;
      for (int p = 0; p < P; ++p)
        pool.emplace_back([&, p] {
          advantage::GrpoAssemblyResult r = advantage::assemble_grpo_batch(shards[static_cast<std::size_t>(p)], o);
          std::vector<std::size_t> idx(r.batch.groups.size());
          for (std::size_t i = 0; i < idx.size(); ++i)
            idx[i] = i;
          if (!idx.empty())
            ds[static_cast<std::size_t>(p)] = optim::grpo_loss(s->current, r.batch, idx, gp, nullptr);
        });
      for (auto& th : pool)
        th.join();
      auto t1 = std::chrono::steady_clock::now();
      total += std::chrono::duration<double>(t1 - t0).count();
      if (diag && it == iters - 1)
        diag_out(ds[0], diag);
    }
    return total / std::max(1, iters);
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -static_cast<double>(status_of(ex));
  }
}

} // extern "C"
