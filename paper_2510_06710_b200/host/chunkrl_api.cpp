// C++ drop-in for the reference's operator API (include/ckrl_chunkrl.hpp) on top of the C ABI.
//
// The host side only marshals: the reference's AoS TrajectorySlab is laid out once as the SoA
// rollout buffer of ckrl.h in HBM, every computation (GAE, segmentation, whitening, GRPO
// grouping / advantages / weights, the fused losses) runs in the CUDA kernels behind ckrl_*,
// and the results are returned in the reference's types. There is no CPU fallback: without a
// CUDA device every call throws.
#include "ckrl_chunkrl.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <utility>

namespace ckrl::chunkrl {

void throw_if_error(int32_t st) {
  if (st == CKRL_OK) return;
  const std::string msg = ckrl_last_error();
  switch (st) {
    case CKRL_ERR_UNSUPPORTED_COMBINATION: throw UnsupportedCombination(msg);
    case CKRL_ERR_GRANULARITY_ORDER: throw GranularityOrderViolation(msg);
    case CKRL_ERR_LENGTH_MISMATCH: throw LengthMismatch(msg);
    case CKRL_ERR_BAD_RESET_ID: throw BadResetId(msg);
    case CKRL_ERR_HEAD_MISMATCH: throw HeadMismatch(msg);
    case CKRL_ERR_NON_FINITE: throw NonFinite(msg);
    case CKRL_ERR_DEGENERATE_GROUP: throw DegenerateGroup(msg);
    case CKRL_ERR_SKIP_UPDATE: throw SkipUpdate(msg);
    case CKRL_ERR_INVALID_PLAN: throw InvalidPlan(msg);
    case CKRL_ERR_MEMORY_OVERFLOW: throw MemoryOverflow(msg);
    case CKRL_ERR_EMPTY_TRACE: throw EmptyTrace(msg);
    case CKRL_ERR_CONFIG: throw ConfigError(msg);
    default: throw Error(std::string(ckrl_status_string(st)) + ": " + msg);
  }
}

namespace {

void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) throw Error(std::string("CUDA: ") + cudaGetErrorString(e));
}

template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(std::size_t n) { alloc(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p_ = std::exchange(o.p_, nullptr);
    n_ = std::exchange(o.n_, 0);
    return *this;
  }
  ~DevBuf() { release(); }

  void alloc(std::size_t n) {
    release();
    n_ = n;
    if (n) cuda_check(cudaMalloc(reinterpret_cast<void**>(&p_), n * sizeof(T)));
  }
  void upload(const std::vector<T>& h) {
    alloc(h.size());
    if (n_) cuda_check(cudaMemcpy(p_, h.data(), n_ * sizeof(T), cudaMemcpyHostToDevice));
  }
  void upload(const T* h, std::size_t n) {
    alloc(n);
    if (n_) cuda_check(cudaMemcpy(p_, h, n_ * sizeof(T), cudaMemcpyHostToDevice));
  }
  std::vector<T> download() const {
    std::vector<T> h(n_);
    if (n_) cuda_check(cudaMemcpy(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost));
    return h;
  }
  void zero() {
    if (n_) cuda_check(cudaMemset(p_, 0, n_ * sizeof(T)));
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }

 private:
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

ckrl_granularity to_c(const GranularitySpec& s) {
  return ckrl_granularity{static_cast<int32_t>(s.advantage_level), static_cast<int32_t>(s.logprob_level),
                          static_cast<int32_t>(s.value_level)};
}


}  // namespace

namespace detail {

// The slab in HBM (ckrl_rollout layout) + the batch arrays of whichever assembly ran on it.
struct DeviceSlab {
  const TrajectorySlab* slab = nullptr;
  int E = 0, Tc = 0, C = 0, M = 0;
  GranularitySpec spec;
  DevBuf<int32_t> tokens;
  DevBuf<float> old_lp, reward, value_scalar, value_vector, bootstrap;
  DevBuf<uint8_t> flags;
  DevBuf<int32_t> episode_id;
  // PPO batch
  DevBuf<uint8_t> counted;
  DevBuf<double> adv, ret;
  // GRPO batch + episode table
  DevBuf<int32_t> env_group, env_member, env_episode, env_group_size, group_counts;
  DevBuf<double> env_adv;
  DevBuf<double> slot_weight;
  DevBuf<uint8_t> slot_member;
  DevBuf<unsigned char> ws;

  ckrl_rollout rollout(int vocab) const {
    ckrl_rollout r;
    r.num_envs = E;
    r.num_chunks = Tc;
    r.chunk_len = C;
    r.tokens_per_action = M;
    r.vocab = vocab < 1 ? 1 : vocab;
    r.token_dtype = CKRL_DTYPE_I32;
    r.tokens = tokens.get();
    r.old_logprob = old_lp.get();
    r.reward = reward.get();
    r.flags = flags.get();
    r.episode_id = episode_id.get();
    r.value_scalar = value_scalar.get();
    r.value_vector = value_vector.get();
    r.bootstrap = bootstrap.get();
    return r;
  }
  ckrl_ppo_batch ppo() const { return ckrl_ppo_batch{counted.get(), adv.get(), ret.get()}; }
  ckrl_grpo_batch grpo() const {
    return ckrl_grpo_batch{env_group.get(), env_member.get(), env_episode.get(), env_adv.get(),
                           env_group_size.get(), slot_weight.get(), slot_member.get(), group_counts.get()};
  }
  void alloc_ws(int envs) {
    ws.alloc(ckrl_workspace_bytes(envs, 0, 1, 1, 1));
    throw_if_error(ckrl_workspace_init(ws.get(), ws.size(), nullptr));
  }
};

}  // namespace detail

namespace {

using detail::DeviceSlab;

int32_t low_id(std::int64_t uid) { return uid < 0 ? -1 : static_cast<int32_t>(uid & 0xffffffff); }

// TrajectorySlab (AoS, core/types.hpp:54-104) -> SoA in HBM. `boot` (may be empty) holds the
// per-slot bootstrap values.
std::shared_ptr<DeviceSlab> upload(const TrajectorySlab& slab, const std::vector<float>& boot) {
  auto d = std::make_shared<DeviceSlab>();
  d->slab = &slab;
  d->E = slab.num_envs;
  d->C = slab.chunk_length;
  d->M = slab.tokens_per_action;
  if (static_cast<int>(slab.records.size()) != d->E) throw LengthMismatch("slab.records must have num_envs rows");
  d->Tc = d->E ? static_cast<int>(slab.records[0].size()) : 0;
  const int E = d->E, Tc = d->Tc, C = d->C, M = d->M;
  const std::size_t nr = static_cast<std::size_t>(E) * Tc, ns = nr * C, nk = ns * M;
  std::vector<int32_t> tok(nk, 0), eid(ns, -1);
  std::vector<float> olp(nk, 0.0f), rew(ns, 0.0f), vs(nr, 0.0f), vv(ns, 0.0f);
  std::vector<uint8_t> fl(ns, 0);
  for (int e = 0; e < E; ++e) {
    const auto& recs = slab.records[static_cast<std::size_t>(e)];
    if (static_cast<int>(recs.size()) != Tc) throw LengthMismatch("every env needs the same number of chunks");
    for (int t = 0; t < Tc; ++t) {
      const StepRecord& r = recs[static_cast<std::size_t>(t)];
      const std::size_t rt = static_cast<std::size_t>(e) * Tc + t;
      if (static_cast<int>(r.rewards.size()) != C || static_cast<int>(r.valid.size()) != C ||
          static_cast<int>(r.terminated.size()) != C || static_cast<int>(r.truncated.size()) != C ||
          static_cast<int>(r.episode_uid.size()) != C)
        throw LengthMismatch("StepRecord per-slot arrays must have chunk_length entries");
      vs[rt] = static_cast<float>(r.value_scalar);
      for (int j = 0; j < C; ++j) {
        const std::size_t sl = rt * C + j;
        rew[sl] = static_cast<float>(r.rewards[static_cast<std::size_t>(j)]);
        fl[sl] = static_cast<uint8_t>((r.terminated[static_cast<std::size_t>(j)] ? CKRL_FLAG_TERMINATED : 0) |
                                      (r.truncated[static_cast<std::size_t>(j)] ? CKRL_FLAG_TRUNCATED : 0) |
                                      (r.valid[static_cast<std::size_t>(j)] ? CKRL_FLAG_VALID : 0));
        eid[sl] = low_id(r.episode_uid[static_cast<std::size_t>(j)]);
        if (static_cast<std::size_t>(j) < r.value_vector.size())
          vv[sl] = static_cast<float>(r.value_vector[static_cast<std::size_t>(j)]);
        for (int m = 0; m < M; ++m) {
          const std::size_t k = sl * M + m;
          if (static_cast<std::size_t>(j) < r.chunk.actions.size() &&
              static_cast<std::size_t>(m) < r.chunk.actions[static_cast<std::size_t>(j)].tokens.size())
            tok[k] = r.chunk.actions[static_cast<std::size_t>(j)].tokens[static_cast<std::size_t>(m)];
          if (r.token_logprobs.values.size() == static_cast<std::size_t>(C) * M)
            olp[k] = static_cast<float>(r.token_logprobs.at(j, m));
        }
      }
    }
  }
  d->tokens.upload(tok);
  d->old_lp.upload(olp);
  d->reward.upload(rew);
  d->flags.upload(fl);
  d->episode_id.upload(eid);
  d->value_scalar.upload(vs);
  d->value_vector.upload(vv);
  std::vector<float> b = boot.empty() ? std::vector<float>(ns, 0.0f) : boot;
  d->bootstrap.upload(b);
  return d;
}

struct EpisodeTableDev {
  DevBuf<int32_t> env, eid, start, len, fs, task, rid;
  DevBuf<double> rew;
  DevBuf<uint8_t> complete;
  int32_t count = 0;
  ckrl_episodes c() const {
    return ckrl_episodes{count, env.get(), eid.get(), start.get(), len.get(), rew.get(), fs.get(),
                         complete.get(), task.get(), rid.get()};
  }
};

// success_from_flag: first_success := success ? max(fs, 0) : -1 (slab_success_rate reads the
// success flag, assembler.cpp:272-276).
EpisodeTableDev upload_episodes(const TrajectorySlab& slab, bool success_from_flag) {
  EpisodeTableDev t;
  const std::size_t n = slab.episodes.size();
  t.count = static_cast<int32_t>(n);
  std::vector<int32_t> env(n), eid(n), start(n), len(n), fs(n), task(n), rid(n);
  std::vector<double> rew(n);
  std::vector<uint8_t> comp(n);
  for (std::size_t i = 0; i < n; ++i) {
    const EpisodeInfo& ep = slab.episodes[i];
    env[i] = ep.env_id;
    eid[i] = low_id(ep.uid);
    start[i] = static_cast<int32_t>(ep.start_step);
    len[i] = static_cast<int32_t>(ep.length);
    rew[i] = ep.total_reward;
    fs[i] = success_from_flag ? (ep.success ? static_cast<int32_t>(std::max<std::int64_t>(ep.first_success_step, 0)) : -1)
                              : static_cast<int32_t>(ep.first_success_step);
    comp[i] = ep.complete ? 1 : 0;
    task[i] = ep.group_key.task_id;
    rid[i] = ep.group_key.reset_state_id;
  }
  t.env.upload(env);
  t.eid.upload(eid);
  t.start.upload(start);
  t.len.upload(len);
  t.fs.upload(fs);
  t.task.upload(task);
  t.rid.upload(rid);
  t.rew.upload(rew);
  t.complete.upload(comp);
  return t;
}

}  // namespace

// ---- core/granularity -----------------------------------------------------------------------
const char* level_name(Level l) {
  switch (l) {
    case Level::Chunk: return "chunk_level";
    case Level::Action: return "action_level";
    default: return "token_level";
  }
}

Level level_from_name(const std::string& n) {
  if (n == "chunk_level" || n == "chunk") return Level::Chunk;
  if (n == "action_level" || n == "action") return Level::Action;
  if (n == "token_level" || n == "token") return Level::Token;
  throw ConfigError("unknown granularity level: " + n);
}

bool coarser_than(Level a, Level b) { return static_cast<int>(a) < static_cast<int>(b); }

void validate_granularity(const GranularitySpec& spec) {
  const ckrl_granularity g = to_c(spec);
  throw_if_error(ckrl_validate_granularity(&g));
}

// ---- advantage ----------------------------------------------------------------------------------
namespace advantage {

GaeResult compute_gae(std::span<const double> rewards, std::span<const double> values,
                      std::span<const double> bootstrap, const std::vector<bool>& terminated,
                      const std::vector<bool>& truncated, const GaeParams& params) {
  const std::size_t n = rewards.size();
  if (values.size() != n || bootstrap.size() != n || terminated.size() != n || truncated.size() != n)
    throw LengthMismatch("compute_gae: rewards, values, bootstrap and flags must have equal length");
  GaeResult res;
  if (n == 0) return res;
  std::vector<uint8_t> flags(n);
  for (std::size_t i = 0; i < n; ++i)
    flags[i] = static_cast<uint8_t>((terminated[i] ? CKRL_FLAG_TERMINATED : 0) | (truncated[i] ? CKRL_FLAG_TRUNCATED : 0));
  DevBuf<double> r, v, b, adv(n), ret(n);
  r.upload(rewards.data(), n);
  v.upload(values.data(), n);
  b.upload(bootstrap.data(), n);
  DevBuf<uint8_t> f;
  f.upload(flags);
  DevBuf<int32_t> off;
  off.upload(std::vector<int32_t>{0, static_cast<int32_t>(n)});
  const ckrl_gae_params p{params.gamma, params.lambda};
  throw_if_error(ckrl_compute_gae(1, off.get(), r.get(), v.get(), b.get(), f.get(), &p, adv.get(), ret.get(), nullptr));
  res.advantages = adv.download();
  res.returns = ret.download();
  return res;
}

GaeResult compute_gae(std::span<const double> rewards, std::span<const double> values, double bootstrap,
                      const std::vector<bool>& terminated, const std::vector<bool>& truncated,
                      const GaeParams& params) {
  std::vector<double> boot(rewards.size(), 0.0);
  if (!boot.empty()) boot.back() = bootstrap;  // gae.cpp:39-46
  return compute_gae(rewards, values, boot, terminated, truncated, params);
}

std::vector<double> grpo_group_advantage(const GroupBatch& batch, double eps_std) {
  const std::size_t g = batch.size();
  DevBuf<double> R, adv(g);
  R.upload(batch.total_rewards);
  DevBuf<int32_t> off, status(1);
  off.upload(std::vector<int32_t>{0, static_cast<int32_t>(g)});
  status.zero();
  throw_if_error(ckrl_grpo_group_advantage(1, off.get(), R.get(), eps_std, adv.get(), status.get(), nullptr));
  const int32_t st = status.download()[0];
  if (st == CKRL_ERR_DEGENERATE_GROUP)
    throw DegenerateGroup(g < 2 ? "GRPO group needs at least 2 trajectories"
                                : "all trajectories in the group have equal return");
  throw_if_error(st);
  return adv.download();
}

namespace {
// batched group means + strict filter decisions (grpo.cpp:30-46)
void group_means(const std::vector<GroupBatch>& groups, const FilterBounds& b, std::vector<double>* means,
                 std::vector<uint8_t>* keep) {
  const std::size_t G = groups.size();
  if (G == 0) return;
  std::vector<int32_t> off{0};
  std::vector<double> R;
  for (const auto& g : groups) {
    R.insert(R.end(), g.total_rewards.begin(), g.total_rewards.end());
    off.push_back(static_cast<int32_t>(R.size()));
  }
  DevBuf<double> dR, dmean(G);
  dR.upload(R.empty() ? std::vector<double>{0.0} : R);
  DevBuf<int32_t> doff;
  doff.upload(off);
  DevBuf<uint8_t> dkeep(G);
  throw_if_error(ckrl_success_rate_filter(static_cast<int32_t>(G), doff.get(), dR.get(), b.lower, b.upper,
                                          dkeep.get(), dmean.get(), nullptr));
  if (means) *means = dmean.download();
  if (keep) *keep = dkeep.download();
}

std::vector<double> episode_weights(std::int64_t length, bool success, std::int64_t fs, bool normalized,
                                    std::vector<bool>* mask) {
  std::vector<double> w(static_cast<std::size_t>(std::max<std::int64_t>(length, 0)), 0.0);
  if (mask) mask->assign(w.size(), true);
  if (w.empty()) return w;
  DevBuf<int64_t> off, dfs;
  off.upload(std::vector<int64_t>{0, length});
  dfs.upload(std::vector<int64_t>{fs});
  DevBuf<uint8_t> succ;
  succ.upload(std::vector<uint8_t>{static_cast<uint8_t>(success ? 1 : 0)});
  if (mask) {
    DevBuf<uint8_t> m(w.size());
    throw_if_error(ckrl_valid_action_mask(1, off.get(), succ.get(), dfs.get(), m.get(), nullptr));
    const auto h = m.download();
    for (std::size_t i = 0; i < h.size(); ++i) (*mask)[i] = h[i] != 0;
    return w;
  }
  DevBuf<double> dw(w.size());
  throw_if_error(ckrl_length_norm_weights(1, off.get(), succ.get(), dfs.get(), normalized ? 1 : 0, dw.get(), nullptr));
  return dw.download();
}
}  // namespace

double group_mean_return(const GroupBatch& batch) {
  std::vector<double> m;
  group_means({batch}, FilterBounds{}, &m, nullptr);
  return m.at(0);
}

std::vector<GroupBatch> success_rate_filter(const std::vector<GroupBatch>& groups, const FilterBounds& bounds) {
  std::vector<uint8_t> keep;
  group_means(groups, bounds, nullptr, &keep);
  std::vector<GroupBatch> kept;
  for (std::size_t i = 0; i < groups.size(); ++i)
    if (keep[i]) kept.push_back(groups[i]);
  return kept;
}

std::vector<bool> valid_action_mask(std::int64_t length, bool success, std::int64_t first_success_step) {
  std::vector<bool> mask;
  episode_weights(length, success, first_success_step, true, &mask);
  return mask;
}

std::vector<double> length_norm_weights(std::int64_t length, bool success, std::int64_t first_success_step,
                                        bool length_normalized) {
  return episode_weights(length, success, first_success_step, length_normalized, nullptr);
}

std::int64_t PpoBatch::advantage_unit_count() const {
  std::int64_t n = 0;
  const bool action = spec.advantage_level == Level::Action;
  for (const auto& v : records) {
    if (action)
      n += std::count(v.counted.begin(), v.counted.end(), true);
    else
      n += std::any_of(v.counted.begin(), v.counted.end(), [](bool b) { return b; }) ? 1 : 0;
  }
  return n;
}

namespace {
// Where assemble_ppo_batch bootstraps (flush_segment, assembler.cpp:42-53): truncated units
// and the open end of every segment (a uid change or the end of the env's timeline). The
// unit's bootstrap slot is the slot itself (action level) or its last counted slot (chunk
// level, assembler.cpp:162-175).
std::vector<float> bootstrap_values(const TrajectorySlab& slab, const ValueFn& value, bool action) {
  const int E = slab.num_envs, C = slab.chunk_length;
  const int Tc = E ? static_cast<int>(slab.records[0].size()) : 0;
  std::vector<float> boot(static_cast<std::size_t>(E) * Tc * C, 0.0f);
  if (!value) return boot;
  auto eval = [&](int e, int t, int j) {
    const StepRecord& r = slab.records[static_cast<std::size_t>(e)][static_cast<std::size_t>(t)];
    const auto v = value(r.post_obs.at(static_cast<std::size_t>(j)),
                         action ? policy::ValueHeadKind::Vector : policy::ValueHeadKind::Scalar);
    boot[(static_cast<std::size_t>(e) * Tc + t) * C + j] = static_cast<float>(v.at(0));
  };
  for (int e = 0; e < E; ++e) {
    const auto& recs = slab.records[static_cast<std::size_t>(e)];
    struct U {
      int t, j;
      std::int64_t uid;
      bool term, trunc;
    };
    std::vector<U> units;
    for (int t = 0; t < Tc; ++t) {
      const StepRecord& r = recs[static_cast<std::size_t>(t)];
      if (action) {
        for (int j = 0; j < C; ++j)
          if (r.valid[static_cast<std::size_t>(j)])
            units.push_back({t, j, r.episode_uid[static_cast<std::size_t>(j)], (bool)r.terminated[static_cast<std::size_t>(j)],
                             (bool)r.truncated[static_cast<std::size_t>(j)]});
      } else {
        int first = -1;
        for (int j = 0; j < C && first < 0; ++j)
          if (r.valid[static_cast<std::size_t>(j)]) first = j;
        if (first < 0) continue;
        U u{t, first, r.episode_uid[static_cast<std::size_t>(first)], false, false};
        for (int j = first; j < C; ++j) {
          if (!r.valid[static_cast<std::size_t>(j)] || r.episode_uid[static_cast<std::size_t>(j)] != u.uid) break;
          u.term = u.term || r.terminated[static_cast<std::size_t>(j)];
          u.trunc = u.trunc || r.truncated[static_cast<std::size_t>(j)];
          u.j = j;
        }
        units.push_back(u);
      }
    }
    for (std::size_t i = 0; i < units.size(); ++i) {
      const U& u = units[i];
      const bool open_end = !u.term && !u.trunc && (i + 1 == units.size() || units[i + 1].uid != u.uid);
      if (u.trunc || open_end) eval(e, u.t, u.j);
    }
  }
  return boot;
}
}  // namespace

PpoBatch assemble_ppo_batch(const TrajectorySlab& slab, const ValueFn& snapshot_value,
                            const PpoAssemblyOptions& options) {
  validate_granularity(options.spec);
  if (options.spec.value_level != options.spec.advantage_level)  // assembler.cpp:81-82
    throw ConfigError("value_type must match reward_type for GAE assembly");
  const bool action = options.spec.advantage_level == Level::Action;
  auto d = upload(slab, bootstrap_values(slab, snapshot_value, action));
  d->spec = options.spec;
  const int E = d->E, Tc = d->Tc, C = d->C;
  const std::size_t nr = static_cast<std::size_t>(E) * Tc, U = action ? static_cast<std::size_t>(C) : 1;
  d->counted.alloc(nr * C);
  d->adv.alloc(nr * U);
  d->ret.alloc(nr * U);
  d->alloc_ws(E);
  const ckrl_rollout ro = d->rollout(1);
  const ckrl_gae_params gae{options.gae.gamma, options.gae.lambda};
  const ckrl_granularity g = to_c(options.spec);
  ckrl_ppo_batch b = d->ppo();
  throw_if_error(ckrl_assemble_ppo_batch(&ro, &gae, &g, &b, d->ws.get(), d->ws.size(), nullptr));
  cuda_check(cudaDeviceSynchronize());
  const auto counted = d->counted.download();
  const auto adv = d->adv.download();
  const auto ret = d->ret.download();
  PpoBatch batch;
  batch.spec = options.spec;
  batch.C = C;
  batch.M = d->M;
  batch.records.reserve(nr);
  for (int e = 0; e < E; ++e)
    for (int t = 0; t < Tc; ++t) {
      const std::size_t rt = static_cast<std::size_t>(e) * Tc + t;
      PpoRecordView v;
      v.rec = &slab.records[static_cast<std::size_t>(e)][static_cast<std::size_t>(t)];
      v.env = e;
      v.chunk_index = t;
      v.counted.resize(static_cast<std::size_t>(C));
      for (int j = 0; j < C; ++j) v.counted[static_cast<std::size_t>(j)] = counted[rt * C + j] != 0;
      v.advantages.resize(U);
      v.returns.resize(U);
      for (std::size_t u = 0; u < U; ++u) {
        // entries are meaningful only where counted (assembler.hpp:25-27); the rest are 0
        const bool on = action ? v.counted[u] : std::any_of(v.counted.begin(), v.counted.end(), [](bool x) { return x; });
        v.advantages[u] = on ? adv[rt * U + u] : 0.0;
        v.returns[u] = on ? ret[rt * U + u] : 0.0;
      }
      batch.records.push_back(std::move(v));
    }
  batch.device = d;
  return batch;
}

GrpoAssemblyResult assemble_grpo_batch(const TrajectorySlab& slab, const GrpoAssemblyOptions& options) {
  validate_granularity(options.spec);
  auto d = upload(slab, {});
  d->spec = options.spec;
  const int E = d->E, Tc = d->Tc, C = d->C;
  const std::size_t ns = static_cast<std::size_t>(E) * Tc * C;
  d->env_group.alloc(E);
  d->env_member.alloc(E);
  d->env_episode.alloc(E);
  d->env_group_size.alloc(E);
  d->env_adv.alloc(E);
  d->slot_weight.alloc(ns);
  d->slot_member.alloc(ns);
  d->group_counts.alloc(2);
  d->alloc_ws(E);
  EpisodeTableDev eps = upload_episodes(slab, false);
  const ckrl_rollout ro = d->rollout(1);
  const ckrl_episodes ec = eps.c();
  const ckrl_granularity g = to_c(options.spec);
  const ckrl_grpo_options o{options.eps_std, options.apply_filter ? 1 : 0, options.filter_bounds.lower,
                            options.filter_bounds.upper, options.length_normalized ? 1 : 0,
                            options.min_group_size};
  ckrl_grpo_batch gb = d->grpo();
  throw_if_error(ckrl_assemble_grpo_batch(&ro, &ec, &g, &o, &gb, d->ws.get(), d->ws.size(), nullptr));
  throw_if_error(ckrl_read_stats(d->ws.get(), d->ws.size(), E, nullptr, nullptr, nullptr));  // DegenerateGroup
  const auto counts = d->group_counts.download();
  const auto grp = d->env_group.download();
  const auto mem = d->env_member.download();
  const auto epi = d->env_episode.download();
  const auto adv = d->env_adv.download();
  const auto member = d->slot_member.download();

  GrpoAssemblyResult res;
  res.groups_total = counts[0];
  res.groups_retained = counts[1];
  res.batch.spec = options.spec;
  res.batch.C = C;
  res.batch.M = d->M;
  res.batch.groups.resize(static_cast<std::size_t>(std::max(0, counts[1])));
  std::vector<std::vector<std::pair<int, int>>> members(res.batch.groups.size());  // (member, env)
  for (int e = 0; e < E; ++e)
    if (grp[static_cast<std::size_t>(e)] >= 0)
      members[static_cast<std::size_t>(grp[static_cast<std::size_t>(e)])].push_back({mem[static_cast<std::size_t>(e)], e});
  for (std::size_t gi = 0; gi < members.size(); ++gi) {
    auto& ms = members[gi];
    std::sort(ms.begin(), ms.end());
    GrpoGroup& group = res.batch.groups[gi];
    for (const auto& [m, e] : ms) {
      (void)m;
      const EpisodeInfo* ep = nullptr;
      for (const auto& x : slab.episodes)
        if (x.env_id == e && low_id(x.uid) == epi[static_cast<std::size_t>(e)] && x.complete && x.start_step == 0) ep = &x;
      if (!ep) throw Error("GRPO assembly: trajectory without an episode");
      group.key = ep->group_key;
      GrpoTrajectory tr;
      tr.episode_uid = ep->uid;
      tr.env = e;
      tr.advantage = adv[static_cast<std::size_t>(e)];
      // the fp64 weights of the trajectory (grpo.cpp:57-79), in atomic order
      const std::vector<double> w =
          length_norm_weights(ep->length, ep->first_success_step >= 0, ep->first_success_step, options.length_normalized);
      std::size_t atomic = 0;
      for (int t = 0; t < Tc; ++t) {
        TrajChunk ch;
        ch.rec = &slab.records[static_cast<std::size_t>(e)][static_cast<std::size_t>(t)];
        for (int j = 0; j < C; ++j)
          if (member[(static_cast<std::size_t>(e) * Tc + t) * C + j]) {
            ch.slots.push_back(j);
            ch.slot_weights.push_back(atomic < w.size() ? w[atomic] : 0.0);
            ++atomic;
          }
        if (!ch.slots.empty()) tr.chunks.push_back(std::move(ch));
      }
      group.trajectories.push_back(std::move(tr));
    }
  }
  res.batch.device = d;
  return res;
}

double slab_success_rate(const TrajectorySlab& slab) {
  EpisodeTableDev eps = upload_episodes(slab, true);
  const ckrl_episodes ec = eps.c();
  DevBuf<double> out(1);
  throw_if_error(ckrl_slab_success_rate(&ec, out.get(), nullptr));
  return out.download()[0];
}

}  // namespace advantage

// ---- optim --------------------------------------------------------------------------------------
namespace optim {

namespace {

LossDiagnostics read_diag(const DevBuf<double>& diag) {
  double h[CKRL_DIAG_COUNT];
  throw_if_error(ckrl_read_diagnostics(diag.get(), h, nullptr));
  LossDiagnostics d;
  d.loss = h[CKRL_DIAG_LOSS];
  d.surrogate = h[CKRL_DIAG_SURROGATE];
  d.value_loss = h[CKRL_DIAG_VALUE_LOSS];
  d.entropy = h[CKRL_DIAG_ENTROPY];
  d.clip_frac = h[CKRL_DIAG_CLIP_FRAC];
  d.approx_kl = h[CKRL_DIAG_APPROX_KL];
  d.units = static_cast<std::int64_t>(h[CKRL_DIAG_UNITS]);
  return d;
}

int vocab_of(const CurrentPolicy& net, const Observation& probe) {
  if (net.logits) {
    if (net.vocab < 1) throw ConfigError("CurrentPolicy: vocab is required with a logits view");
    return net.vocab;
  }
  if (!net.forward_logits) throw ConfigError("CurrentPolicy: forward_logits or a logits view is required");
  return static_cast<int>(net.forward_logits(probe, {}).size());
}

// PolicyNet::evaluate_chunk's logits for one record (policy_net.cpp:333-357): position
// p = j*M + m sees the chunk's tokens before it.
void fill_record_logits(const CurrentPolicy& net, const StepRecord& rec, int C, int M, int V, float* dst) {
  std::vector<int> prefix;
  for (int j = 0; j < C; ++j)
    for (int m = 0; m < M; ++m) {
      const auto lg = net.forward_logits(rec.obs, prefix);
      if (static_cast<int>(lg.size()) != V) throw LengthMismatch("forward_logits: vocab changed");
      for (int v = 0; v < V; ++v) dst[static_cast<std::size_t>(j * M + m) * V + v] = static_cast<float>(lg[static_cast<std::size_t>(v)]);
      prefix.push_back(rec.chunk.actions.at(static_cast<std::size_t>(j)).tokens.at(static_cast<std::size_t>(m)));
    }
}

void fill_record_values(const CurrentPolicy& net, const StepRecord& rec, bool vector_head, int C, float* dst) {
  const auto v = net.value(rec.obs, vector_head ? policy::ValueHeadKind::Vector : policy::ValueHeadKind::Scalar);
  const int n = vector_head ? C : 1;
  if (static_cast<int>(v.size()) < n) throw HeadMismatch("value head size");
  for (int i = 0; i < n; ++i) dst[i] = static_cast<float>(v[static_cast<std::size_t>(i)]);
}

}  // namespace

void normalize_advantages(advantage::PpoBatch& batch) {
  auto& d = *batch.device;
  const ckrl_rollout ro = d.rollout(1);
  const ckrl_granularity g = to_c(batch.spec);
  ckrl_ppo_batch b = d.ppo();
  throw_if_error(ckrl_normalize_advantages(&ro, &g, &b, d.ws.get(), d.ws.size(), nullptr));
  const auto adv = d.adv.download();
  const std::size_t U = batch.spec.advantage_level == Level::Action ? static_cast<std::size_t>(batch.C) : 1;
  for (std::size_t r = 0; r < batch.records.size(); ++r) {
    auto& v = batch.records[r];
    for (std::size_t u = 0; u < U; ++u) {
      const bool on = U > 1 ? v.counted[u] : std::any_of(v.counted.begin(), v.counted.end(), [](bool x) { return x; });
      if (on) v.advantages[u] = adv[r * U + u];
    }
  }
}

LossDiagnostics ppo_loss(const CurrentPolicy& net, const advantage::PpoBatch& batch,
                         std::span<const std::size_t> record_indices, const PpoParams& params,
                         LossCoefficients* coefficients) {
  const int C = batch.C, M = batch.M;
  const int64_t n = static_cast<int64_t>(record_indices.size());
  if (n == 0) throw ConfigError("ppo_loss: empty record selection");
  if (C < 1 || M < 1) throw LengthMismatch("ppo_loss: batch C / M not set");
  for (std::size_t r : record_indices)
    if (r >= batch.records.size()) throw LengthMismatch("ppo_loss: record index out of range");
  const bool vec = batch.spec.value_level == Level::Action;
  const bool action = batch.spec.advantage_level == Level::Action;
  const int V = vocab_of(net, batch.records[record_indices[0]].rec->obs);
  const std::size_t P = static_cast<std::size_t>(C) * M;
  const int NV = vec ? C : 1, U = action ? C : 1;
  // bytes per position of the policy view: a V-bin logits row, or one finished token row
  // (CKRL_DTYPE_TOKEN_ROWS, the tensor-core policy head's output: ckrl_project_token_stats)
  const std::size_t pb = net.logits_dtype == CKRL_DTYPE_TOKEN_ROWS ? sizeof(ckrl_token_row)
                         : static_cast<std::size_t>(V) * (net.logits_dtype == CKRL_DTYPE_BF16 ? 2 : 4);
  if (net.logits && !batch.device)
    throw ConfigError("ppo_loss: a logits view needs a batch assembled by this library (record order)");

  // The selected records as a compact [n][1] SoA view, read from the batch's views and
  // their StepRecords as they are now (the reference reads them live, losses.cpp:100-120).
  std::vector<int32_t> tok(n * P, 0), eid(n * C, -1);
  std::vector<float> olp(n * P, 0.0f), rew(n * C, 0.0f), vs(n, 0.0f), vv(n * C, 0.0f), hv(n * NV, 0.0f);
  std::vector<double> adv(n * U, 0.0), ret(n * U, 0.0);
  std::vector<uint8_t> fl(n * C, 0), cnt(n * C, 0);
  std::vector<float> hl;
  if (!net.logits) {
    if (net.logits_dtype != CKRL_DTYPE_F32) throw ConfigError("forward_logits fills f32 logits");
    hl.assign(static_cast<std::size_t>(n) * P * V, 0.0f);
  }
  for (int64_t i = 0; i < n; ++i) {
    const advantage::PpoRecordView& v = batch.records[record_indices[static_cast<std::size_t>(i)]];
    const StepRecord& r = *v.rec;
    vs[i] = static_cast<float>(r.value_scalar);
    for (int j = 0; j < C; ++j) {
      const std::size_t sl = static_cast<std::size_t>(i) * C + j;
      const std::size_t jj = static_cast<std::size_t>(j);
      rew[sl] = jj < r.rewards.size() ? static_cast<float>(r.rewards[jj]) : 0.0f;
      const bool valid = jj < r.valid.size() && r.valid[jj];
      fl[sl] = static_cast<uint8_t>((valid ? CKRL_FLAG_VALID : 0) |
                                    (jj < r.terminated.size() && r.terminated[jj] ? CKRL_FLAG_TERMINATED : 0) |
                                    (jj < r.truncated.size() && r.truncated[jj] ? CKRL_FLAG_TRUNCATED : 0));
      eid[sl] = jj < r.episode_uid.size() ? low_id(r.episode_uid[jj]) : -1;
      if (jj < r.value_vector.size()) vv[sl] = static_cast<float>(r.value_vector[jj]);
      cnt[sl] = jj < v.counted.size() && v.counted[jj] ? 1 : 0;
      for (int m = 0; m < M; ++m) {
        tok[sl * M + m] = r.chunk.actions.at(jj).tokens.at(static_cast<std::size_t>(m));
        olp[sl * M + m] = static_cast<float>(r.token_logprobs.at(j, m));
      }
    }
    for (int u = 0; u < U; ++u) {
      adv[static_cast<std::size_t>(i) * U + u] = v.advantages.at(static_cast<std::size_t>(u));
      ret[static_cast<std::size_t>(i) * U + u] = v.returns.at(static_cast<std::size_t>(u));
    }
    if (!net.logits) {
      fill_record_logits(net, r, C, M, V, hl.data() + static_cast<std::size_t>(i) * P * V);
      if (net.value && params.value_loss_coef != 0.0) fill_record_values(net, r, vec, C, hv.data() + i * NV);
    }
  }
  DevBuf<int32_t> stok, seid, dtok(n * P), deid(n * C);
  DevBuf<float> solp, srew, svs, svv, sboot(n * C), dolp(n * P), drew(n * C), dvs(n), dvv(n * C),
      dboot(n * C), dvals(n * NV);
  DevBuf<double> sadv, sret, dadv(n * U), dret(n * U);
  DevBuf<uint8_t> sfl, scnt, dfl(n * C), dcnt(n * C);
  stok.upload(tok);
  seid.upload(eid);
  solp.upload(olp);
  srew.upload(rew);
  svs.upload(vs);
  svv.upload(vv);
  sadv.upload(adv);
  sret.upload(ret);
  sfl.upload(fl);
  scnt.upload(cnt);
  sboot.zero();
  DevBuf<unsigned char> logits(static_cast<std::size_t>(n) * P * pb);
  ckrl_policy_outputs src_pol{net.logits_dtype, nullptr, nullptr};
  ckrl_rollout src{static_cast<int32_t>(n), 1, C, M, V, CKRL_DTYPE_I32, stok.get(), solp.get(), srew.get(), sfl.get(),
                   seid.get(), svs.get(), svv.get(), sboot.get()};
  ckrl_ppo_batch sb{scnt.get(), sadv.get(), sret.get()};
  std::vector<int64_t> idx(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) idx[static_cast<std::size_t>(i)] = i;
  DevBuf<unsigned char> full_logits;
  DevBuf<float> full_values;
  if (net.logits) {
    // gather the selected rows of the [records][C][M][V] view on the device
    auto& d = *batch.device;
    const std::size_t nr = batch.records.size();
    if (net.device) {
      src_pol.logits = net.logits;
      src_pol.values = net.values;
    } else {
      full_logits.upload(static_cast<const unsigned char*>(net.logits), nr * P * pb);
      src_pol.logits = full_logits.get();
      if (net.values) {
        full_values.upload(net.values, nr * NV);
        src_pol.values = full_values.get();
      }
    }
    // the gather runs over the full device slab; the batch arrays are refreshed from the
    // host views first (normalize_advantages / caller edits)
    std::vector<uint8_t> fc(nr * C, 0);
    std::vector<double> fa(nr * U, 0.0), fr(nr * U, 0.0);
    for (std::size_t r = 0; r < nr; ++r) {
      const auto& v = batch.records[r];
      for (int j = 0; j < C; ++j) fc[r * C + j] = v.counted[static_cast<std::size_t>(j)] ? 1 : 0;
      for (int u = 0; u < U; ++u) {
        fa[r * U + u] = v.advantages[static_cast<std::size_t>(u)];
        fr[r * U + u] = v.returns[static_cast<std::size_t>(u)];
      }
    }
    d.counted.upload(fc);
    d.adv.upload(fa);
    d.ret.upload(fr);
    src = d.rollout(V);
    sb = d.ppo();
    idx.assign(record_indices.begin(), record_indices.end());
  } else {
    cuda_check(cudaMemcpy(logits.get(), hl.data(), hl.size() * 4, cudaMemcpyHostToDevice));
    cuda_check(cudaMemcpy(dvals.get(), hv.data(), hv.size() * 4, cudaMemcpyHostToDevice));
  }
  DevBuf<int64_t> didx;
  didx.upload(idx);
  DevBuf<unsigned char> ws(ckrl_workspace_bytes(static_cast<int32_t>(n), 0, 1, 1, 1));
  throw_if_error(ckrl_workspace_init(ws.get(), ws.size(), nullptr));
  ckrl_rollout dst{static_cast<int32_t>(n), 1, C, M, V, CKRL_DTYPE_I32, dtok.get(), dolp.get(), drew.get(), dfl.get(),
                   deid.get(), dvs.get(), dvv.get(), dboot.get()};
  ckrl_ppo_batch db{dcnt.get(), dadv.get(), dret.get()};
  ckrl_policy_outputs dp{net.logits_dtype, logits.get(), dvals.get()};
  const ckrl_granularity g = to_c(batch.spec);
  throw_if_error(ckrl_select_records(&src, &sb, &src_pol, &g, n, didx.get(), &dst, &db, &dp, ws.get(), ws.size(), nullptr));
  // the reference's ppo_loss takes the batch's advantages as they are (whitening happens
  // once in update_ppo / normalize_advantages)
  const ckrl_ppo_params pp{params.clip_eps, params.value_loss_coef, params.entropy_coef, 0};
  DevBuf<float> clp, cent, cval;
  ckrl_loss_outputs outs{};
  if (coefficients) {
    clp.alloc(n * P);
    cent.alloc(n * P);
    cval.alloc(n * NV);
    outs.coeff_logprob = clp.get();
    outs.coeff_entropy = cent.get();
    outs.coeff_value = cval.get();
  }
  DevBuf<double> diag(CKRL_DIAG_COUNT);
  throw_if_error(ckrl_ppo_loss(&dst, &db, &dp, &g, &pp, coefficients ? &outs : nullptr, diag.get(), ws.get(),
                               ws.size(), nullptr));
  LossDiagnostics out = read_diag(diag);
  if (coefficients) {
    const auto a = clp.download(), b2 = cent.download(), c = cval.download();
    coefficients->coeff_logprob.assign(a.begin(), a.end());
    coefficients->coeff_entropy.assign(b2.begin(), b2.end());
    coefficients->coeff_value.assign(c.begin(), c.end());
  }
  return out;
}

LossDiagnostics grpo_loss(const CurrentPolicy& net, const advantage::GrpoBatch& batch,
                          std::span<const std::size_t> group_indices, const GrpoParams& params) {
  if (group_indices.empty()) throw SkipUpdate("grpo_loss: no groups selected");  // losses.cpp:238
  if (!batch.device) throw ConfigError("grpo_loss: batch was not assembled by this library");
  auto& d = *batch.device;
  const int E = d.E, Tc = d.Tc, C = d.C, M = d.M;
  const std::size_t P = static_cast<std::size_t>(C) * M, nr = static_cast<std::size_t>(E) * Tc;
  for (std::size_t g : group_indices)
    if (g >= batch.groups.size()) throw LengthMismatch("grpo_loss: group index out of range");
  const Observation probe = E && Tc ? d.slab->records[0][0].obs : Observation{};
  const int V = vocab_of(net, probe);
  const std::size_t pb = net.logits_dtype == CKRL_DTYPE_TOKEN_ROWS ? sizeof(ckrl_token_row)
                         : static_cast<std::size_t>(V) * (net.logits_dtype == CKRL_DTYPE_BF16 ? 2 : 4);
  DevBuf<unsigned char> logits;
  const void* lp = net.logits;
  if (!net.logits || !net.device) {
    logits.alloc(nr * P * pb);
    if (net.logits) {
      cuda_check(cudaMemcpy(logits.get(), net.logits, nr * P * pb, cudaMemcpyHostToDevice));
    } else {
      if (net.logits_dtype != CKRL_DTYPE_F32) throw ConfigError("forward_logits fills f32 logits");
      std::vector<float> hl(nr * P * V, 0.0f);  // unselected envs never reach the loss
      for (std::size_t g : group_indices)
        for (const auto& tr : batch.groups[g].trajectories)
          for (int t = 0; t < Tc; ++t)
            fill_record_logits(net, d.slab->records[static_cast<std::size_t>(tr.env)][static_cast<std::size_t>(t)], C, M,
                               V, hl.data() + (static_cast<std::size_t>(tr.env) * Tc + t) * P * V);
      cuda_check(cudaMemcpy(logits.get(), hl.data(), hl.size() * 4, cudaMemcpyHostToDevice));
    }
    lp = logits.get();
  }
  // group selection on a copy of the assembly workspace (losses.cpp:240-246)
  DevBuf<unsigned char> ws(d.ws.size());
  cuda_check(cudaMemcpy(ws.get(), d.ws.get(), d.ws.size(), cudaMemcpyDeviceToDevice));
  std::vector<int32_t> sel(group_indices.begin(), group_indices.end());
  DevBuf<int32_t> dsel, env_group(E);
  dsel.upload(sel);
  throw_if_error(ckrl_select_groups(E, d.env_group.get(), env_group.get(), static_cast<int32_t>(sel.size()), dsel.get(),
                                    ws.get(), ws.size(), nullptr));
  ckrl_grpo_batch gb = d.grpo();
  gb.env_group = env_group.get();
  const ckrl_rollout ro = d.rollout(V);
  const ckrl_policy_outputs po{net.logits_dtype, lp, nullptr};
  const ckrl_granularity g = to_c(batch.spec);
  const ckrl_grpo_params gp{params.clip_eps};
  DevBuf<double> diag(CKRL_DIAG_COUNT);
  throw_if_error(ckrl_grpo_loss(&ro, &gb, &po, &g, &gp, nullptr, diag.get(), ws.get(), ws.size(), nullptr));
  return read_diag(diag);
}

}  // namespace optim

namespace policy {

std::vector<double> chunk_logits_gradient(std::span<const double> logits, int vocab,
                                          std::span<const int> tokens,
                                          std::span<const double> coeff_logprob,
                                          std::span<const double> coeff_entropy) {
  const std::size_t P = tokens.size();
  if (vocab < 1 || logits.size() != P * static_cast<std::size_t>(vocab) || coeff_logprob.size() != P ||
      (!coeff_entropy.empty() && coeff_entropy.size() != P))
    throw LengthMismatch("coefficient length must be C*M");
  if (P == 0) return {};
  std::vector<float> lg(logits.begin(), logits.end());
  std::vector<int32_t> tk(tokens.begin(), tokens.end());
  std::vector<float> kl(coeff_logprob.begin(), coeff_logprob.end());
  std::vector<float> ke(coeff_entropy.begin(), coeff_entropy.end());
  DevBuf<float> d_lg, d_kl, d_ke, d_out(lg.size());
  DevBuf<int32_t> d_tk, d_st(1);
  d_lg.upload(lg);
  d_tk.upload(tk);
  d_kl.upload(kl);
  if (!ke.empty()) d_ke.upload(ke);
  d_st.zero();
  throw_if_error(ckrl_logits_grad(static_cast<int64_t>(P), vocab, CKRL_DTYPE_F32, d_lg.get(), CKRL_DTYPE_I32,
                                  d_tk.get(), d_kl.get(), ke.empty() ? nullptr : d_ke.get(), CKRL_DTYPE_F32,
                                  d_out.get(), d_st.get(), nullptr));
  throw_if_error(ckrl_read_status(d_st.get(), nullptr));
  std::vector<float> out = d_out.download();
  return std::vector<double>(out.begin(), out.end());
}

}  // namespace policy

namespace optim {

struct Adam::State {
  std::size_t n = 0;
  ckrl_adam_params p{};
  std::int64_t t = 0;
  DevBuf<double> m, v, norm, params, grad;
  DevBuf<int32_t> status;
  DevBuf<unsigned char> ws;
};

Adam::Adam(std::size_t num_params, double learning_rate, double max_grad_norm, double beta1, double beta2,
           double eps)
    : s_(new State) {
  s_->n = num_params;
  s_->p = ckrl_adam_params{learning_rate, max_grad_norm, beta1, beta2, eps};
  s_->m.alloc(num_params);
  s_->v.alloc(num_params);
  s_->m.zero();
  s_->v.zero();
  s_->norm.alloc(1);
  s_->status.alloc(1);
  s_->ws.alloc(ckrl_adam_workspace_bytes());
  s_->ws.zero();
}

Adam::~Adam() { delete s_; }

double Adam::step_device(double* params, double* grad) {
  s_->status.zero();
  throw_if_error(ckrl_adam_step(CKRL_DTYPE_F64, static_cast<int64_t>(s_->n), params, grad, s_->m.get(),
                                s_->v.get(), &s_->p, s_->t + 1, s_->norm.get(), s_->status.get(), s_->ws.get(),
                                s_->ws.size(), nullptr, nullptr));
  throw_if_error(ckrl_read_status(s_->status.get(), nullptr));  // NonFinite: t_ unchanged (adam.cpp:21-28)
  ++s_->t;
  return s_->norm.download()[0];
}

double Adam::step(std::span<double> params, std::span<double> grad) {
  if (params.size() != s_->n || grad.size() != s_->n) throw LengthMismatch("Adam buffer size mismatch");
  s_->params.upload(params.data(), params.size());
  s_->grad.upload(grad.data(), grad.size());
  const double norm = step_device(s_->params.get(), s_->grad.get());
  std::vector<double> p = s_->params.download(), g = s_->grad.download();
  std::copy(p.begin(), p.end(), params.begin());
  std::copy(g.begin(), g.end(), grad.begin());
  return norm;
}

}  // namespace optim

std::string dump_slab(const TrajectorySlab& slab) {
  const int E = slab.num_envs, C = slab.chunk_length, M = slab.tokens_per_action;
  const int Tc = E > 0 ? static_cast<int>(slab.records[0].size()) : 0;
  for (const auto& r : slab.records)
    if (static_cast<int>(r.size()) != Tc) throw LengthMismatch("dump_slab: ragged records");
  const std::size_t S = static_cast<std::size_t>(E) * Tc * C;
  std::vector<int32_t> tok(S * M), ids(S);
  std::vector<double> rw(S);
  std::vector<uint8_t> fl(S);
  // the SoA keeps uid & 0xffffffff; the high word is the global env id first_env_id + row
  // (vec_env.cpp:94), recovered from the first live uid and checked for every slot
  int64_t first_env = -1;
  for (int e = 0; e < E; ++e)
    for (int t = 0; t < Tc; ++t) {
      const StepRecord& rec = slab.records[static_cast<std::size_t>(e)][static_cast<std::size_t>(t)];
      for (int j = 0; j < C; ++j) {
        const std::size_t s = (static_cast<std::size_t>(e) * Tc + t) * C + j;
        const std::size_t jj = static_cast<std::size_t>(j);
        for (int m = 0; m < M; ++m) tok[s * M + m] = rec.chunk.actions[jj].tokens[static_cast<std::size_t>(m)];
        rw[s] = rec.rewards[jj];
        fl[s] = static_cast<uint8_t>((rec.terminated[jj] ? CKRL_FLAG_TERMINATED : 0) |
                                     (rec.truncated[jj] ? CKRL_FLAG_TRUNCATED : 0) |
                                     (rec.valid[jj] ? CKRL_FLAG_VALID : 0));
        const std::int64_t uid = rec.episode_uid[jj];
        ids[s] = uid < 0 ? -1 : static_cast<int32_t>(uid & 0xffffffff);
        if (uid >= 0) {
          const int64_t env = (uid >> 32) - e;
          if (first_env < 0) first_env = env;
          if (env != first_env || env < 0)
            throw ConfigError("dump_slab: episode uids must be (first_env_id + env) << 32 | k");
        }
      }
    }
  const int32_t off = first_env < 0 ? 0 : static_cast<int32_t>(first_env);
  std::size_t n = 0;
  throw_if_error(ckrl_dump_slab(E, Tc, C, M, CKRL_DTYPE_I32, tok.data(), rw.data(), fl.data(), ids.data(), off,
                                nullptr, 0, &n));
  std::string out(n, '\0');
  throw_if_error(ckrl_dump_slab(E, Tc, C, M, CKRL_DTYPE_I32, tok.data(), rw.data(), fl.data(), ids.data(), off,
                                out.data(), n, &n));
  return out;
}

namespace policy {

void save_checkpoint(const PolicyDescriptor& d, std::span<const double> params, const std::string& path) {
  const ckrl_policy_desc cd{d.obs_dim, d.hidden, d.trunk_layers, d.value_hidden, d.vocab, d.C, d.M};
  if (ckrl_policy_num_params(&cd) != static_cast<int64_t>(params.size()))
    throw LengthMismatch("checkpoint parameter count mismatch");
  throw_if_error(ckrl_save_checkpoint(&cd, params.data(), path.c_str()));
}

std::pair<PolicyDescriptor, std::vector<double>> load_checkpoint(const std::string& path) {
  ckrl_policy_desc cd{};
  int64_t n = 0;
  throw_if_error(ckrl_load_checkpoint(path.c_str(), &cd, nullptr, 0, &n));
  std::vector<double> p(static_cast<std::size_t>(n));
  throw_if_error(ckrl_load_checkpoint(path.c_str(), &cd, p.data(), n, &n));
  return {PolicyDescriptor{cd.obs_dim, cd.hidden, cd.trunk_layers, cd.value_hidden, cd.vocab, cd.chunk_len,
                           cd.tokens_per_action},
          std::move(p)};
}

}  // namespace policy

}  // namespace ckrl::chunkrl
