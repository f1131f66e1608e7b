// C++ drop-in tests: the reference's own known-answer cases (tests/test_advantage.cpp,
// tests/test_optim.cpp) restated against include/ckrl_chunkrl.hpp, so a reference-style
// caller is checked through the same signatures and exception types on the B200.
//
//   ./test_dropin            run every case (needs a CUDA device)
//   ./test_dropin --list     list the cases (no device needed)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "ckrl_chunkrl.hpp"

using namespace ckrl::chunkrl;
using namespace ckrl::chunkrl::advantage;
using namespace ckrl::chunkrl::optim;

// ---- a minimal test harness ----------------------------------------------------------------
namespace {
struct Case {
  const char* name;
  std::function<void()> fn;
};
std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
int g_failures = 0;
struct Reg {
  Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
bool approx(double a, double b, double rel) { return std::fabs(a - b) <= rel * std::max(1.0, std::max(std::fabs(a), std::fabs(b))); }
}  // namespace

#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE(name)                                 \
  static void CAT(test_, __LINE__)();                   \
  static Reg CAT(reg_, __LINE__)(name, CAT(test_, __LINE__)); \
  static void CAT(test_, __LINE__)()
#define CHECK(cond)                                                              \
  do {                                                                           \
    if (!(cond)) {                                                               \
      ++g_failures;                                                              \
      std::fprintf(stderr, "  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
    }                                                                            \
  } while (0)
#define CHECK_APPROX(a, b, rel) CHECK(approx((a), (b), (rel)))
#define CHECK_THROWS_AS(expr, type)          \
  do {                                       \
    bool caught_ = false;                    \
    try {                                    \
      (void)(expr);                          \
    } catch (const type&) {                  \
      caught_ = true;                        \
    } catch (...) {                          \
    }                                        \
    CHECK(caught_ && #type);                 \
  } while (0)

// splitmix64 (the reference's Rng, core/rng.hpp) for the randomized cases
struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
  double normal() {
    double u1 = uniform(), u2 = uniform();
    if (u1 < 1e-300) u1 = 1e-300;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
  uint64_t below(uint64_t n) { return next() % n; }
};

// ---- GAE (test_advantage.cpp:16-100) -------------------------------------------------------
TEST_CASE("undiscounted reward-to-go with terminal end") {
  std::vector<double> r{0.0, 0.0, 1.0}, v{0.0, 0.0, 0.0};
  GaeResult res = compute_gae(r, v, 0.0, {false, false, true}, {false, false, false}, GaeParams{1.0, 1.0});
  CHECK((res.advantages == std::vector<double>{1.0, 1.0, 1.0}));
  CHECK((res.returns == std::vector<double>{1.0, 1.0, 1.0}));
}

TEST_CASE("all-zero rewards and values give zero advantages") {
  std::vector<double> z(5, 0.0);
  std::vector<bool> f(5, false);
  for (double a : compute_gae(z, z, 0.0, f, f, GaeParams{0.9, 0.8}).advantages) CHECK(a == 0.0);
}

TEST_CASE("bootstrapped two-step case") {
  std::vector<double> r{1.0, 1.0}, v{0.5, 0.5};
  std::vector<bool> f(2, false);
  GaeResult res = compute_gae(r, v, 0.5, f, f, GaeParams{0.5, 0.5});
  CHECK_APPROX(res.advantages[0], 0.9375, 1e-12);
  CHECK_APPROX(res.advantages[1], 0.75, 1e-12);
}

TEST_CASE("length mismatch is rejected") {
  std::vector<double> r{1.0, 2.0}, v{0.0};
  std::vector<bool> f{false, false};
  CHECK_THROWS_AS(compute_gae(r, v, 0.0, f, f, GaeParams{0.9, 0.9}), LengthMismatch);
}

TEST_CASE("lambda = gamma = 1 with zero values is the reward-to-go") {
  Rng rng(31);
  for (int trial = 0; trial < 20; ++trial) {
    const std::size_t n = 1 + rng.below(10);
    std::vector<double> r(n), v(n, 0.0);
    for (double& x : r) x = rng.normal();
    std::vector<bool> term(n, false), trunc(n, false);
    term[n - 1] = true;
    GaeResult res = compute_gae(r, v, 0.0, term, trunc, GaeParams{1.0, 1.0});
    double tail = 0.0;
    for (std::size_t t = n; t-- > 0;) {
      tail += r[t];
      CHECK_APPROX(res.advantages[t], tail, 1e-12);
    }
  }
}

TEST_CASE("GAE linearity") {
  Rng rng(33);
  const std::size_t n = 8;
  std::vector<double> r(n), v(n), b(n);
  std::vector<bool> term(n, false), trunc(n, false);
  for (std::size_t t = 0; t < n; ++t) {
    r[t] = rng.normal();
    v[t] = rng.normal();
    b[t] = rng.normal();
    term[t] = rng.uniform() < 0.2;
  }
  const GaeParams p{0.97, 0.9};
  GaeResult base = compute_gae(r, v, b, term, trunc, p);
  for (std::size_t t = 0; t < n; ++t) {
    r[t] *= 3.5;
    v[t] *= 3.5;
    b[t] *= 3.5;
  }
  GaeResult scaled = compute_gae(r, v, b, term, trunc, p);
  for (std::size_t t = 0; t < n; ++t) CHECK_APPROX(scaled.advantages[t], 3.5 * base.advantages[t], 1e-12);
}

// ---- GRPO helpers (test_advantage.cpp:102-230) ---------------------------------------------
GroupBatch group_of(std::vector<double> r) {
  GroupBatch g;
  g.total_rewards = std::move(r);
  return g;
}

TEST_CASE("GRPO group advantages") {
  auto a = grpo_group_advantage(group_of({1.0, 0.0}), 0.0);
  CHECK_APPROX(a[0], 1.0, 1e-12);
  CHECK_APPROX(a[1], -1.0, 1e-12);
  CHECK_THROWS_AS(grpo_group_advantage(group_of({1.0, 1.0, 1.0}), 0.0), DegenerateGroup);
  for (double x : grpo_group_advantage(group_of({1.0, 1.0, 1.0}), 1e-8)) CHECK(x == 0.0);
  const double sd = std::sqrt(0.5);
  a = grpo_group_advantage(group_of({3.0, 1.0, 2.0, 2.0}), 0.0);
  CHECK_APPROX(a[0], 1.0 / sd, 1e-12);
  CHECK_APPROX(a[1], -1.0 / sd, 1e-12);
  CHECK(a[2] == 0.0 && a[3] == 0.0);
  CHECK_THROWS_AS(grpo_group_advantage(group_of({1.0}), 0.0), DegenerateGroup);
  Rng rng(35);
  for (int trial = 0; trial < 50; ++trial) {
    std::vector<double> r(2 + rng.below(6));
    for (double& x : r) x = rng.normal();
    auto adv = grpo_group_advantage(group_of(r), 0.0);
    double mean = 0.0, var = 0.0;
    for (double x : adv) mean += x;
    mean /= (double)adv.size();
    for (double x : adv) var += (x - mean) * (x - mean);
    var /= (double)adv.size();
    CHECK(std::fabs(mean) <= 1e-12);
    CHECK(std::fabs(std::sqrt(var) - 1.0) <= 1e-9);
  }
}

TEST_CASE("valid action mask and length-norm weights") {
  auto m = valid_action_mask(10, true, 3);
  CHECK((m == std::vector<bool>{true, true, true, true, false, false, false, false, false, false}));
  CHECK((valid_action_mask(6, false, -1) == std::vector<bool>(6, true)));
  auto w = length_norm_weights(10, true, 3, true);
  for (int t = 0; t < 4; ++t) CHECK(w[t] == 0.25);
  for (int t = 4; t < 10; ++t) CHECK(w[t] == 0.0);
  for (double x : length_norm_weights(8, true, 3, false)) CHECK_APPROX(x, 0.125, 1e-15);
  for (bool normalized : {false, true}) {
    double tot = 0.0;
    for (double x : length_norm_weights(7, true, 2, normalized)) tot += x;
    CHECK_APPROX(tot, 1.0, 1e-12);
  }
}

TEST_CASE("success-rate filter") {
  CHECK(success_rate_filter({group_of({1, 1, 1, 1})}, FilterBounds{0.0, 1.0}).empty());
  CHECK(success_rate_filter({group_of({1, 0, 1, 0})}, FilterBounds{0.0, 1.0}).size() == 1);
  for (int g = 2; g <= 4; ++g)
    for (int bits = 0; bits < (1 << g); ++bits) {
      std::vector<double> r;
      int ones = 0;
      for (int i = 0; i < g; ++i) {
        r.push_back((bits >> i) & 1);
        ones += (bits >> i) & 1;
      }
      const bool kept = !success_rate_filter({group_of(r)}, FilterBounds{0.0, 1.0}).empty();
      CHECK(kept == (ones > 0 && ones < g));
    }
  CHECK_APPROX(group_mean_return(group_of({1.0, 2.0, 4.0})), 7.0 / 3.0, 1e-15);
}

// ---- assemblers (test_advantage.cpp:230-492) ------------------------------------------------
// One env, C-slot chunks of 1-token actions, zero logprobs; uids count episodes.
TrajectorySlab tiny_slab(const std::vector<double>& rewards, const std::vector<bool>& term, int C) {
  TrajectorySlab slab;
  slab.num_envs = 1;
  slab.chunk_length = C;
  slab.tokens_per_action = 1;
  slab.records.resize(1);
  std::int64_t uid = 0, start = 0, pos = 0, first = -1;
  double total = 0.0;
  bool open = true;
  auto close = [&](bool complete, std::int64_t end_next) {
    EpisodeInfo ep;
    ep.uid = uid;
    ep.env_id = 0;
    ep.start_step = start;
    ep.length = pos;
    ep.total_reward = total;
    ep.success = first >= 0;
    ep.first_success_step = first;
    ep.complete = complete;
    slab.episodes.push_back(ep);
    ++uid;
    start = end_next;
    pos = 0;
    total = 0.0;
    first = -1;
  };
  for (int t = 0; t < (int)rewards.size(); t += C) {
    StepRecord rec;
    rec.obs = {(double)t};
    rec.chunk.actions.assign(C, TokenAction{{0}});
    rec.token_logprobs = TokenLogprobs{C, 1, std::vector<double>(C, 0.0)};
    for (int j = 0; j < C; ++j) {
      const int i = t + j;
      rec.rewards.push_back(rewards[i]);
      rec.terminated.push_back(term[i]);
      rec.truncated.push_back(false);
      rec.valid.push_back(true);
      rec.episode_uid.push_back(uid);
      rec.post_obs.push_back({(double)(i + 1)});
      total += rewards[i];
      if (rewards[i] > 0 && first < 0) first = pos;
      ++pos;
      open = !term[i];
      if (term[i]) close(true, i + 1);
    }
    rec.value_vector.assign(C, 0.0);
    slab.records[0].push_back(std::move(rec));
  }
  if (open) close(false, 0);
  return slab;
}

const ValueFn zero_values = [](const Observation&, policy::ValueHeadKind k) {
  return std::vector<double>(k == policy::ValueHeadKind::Scalar ? 1 : 2, 0.0);
};

TEST_CASE("PPO assembler: action-level GAE over a terminal episode") {
  TrajectorySlab slab = tiny_slab({0.0, 0.0, 1.0, 0.0}, {false, false, true, false}, 2);
  PpoAssemblyOptions o;
  o.gae = GaeParams{1.0, 1.0};
  o.spec = GranularitySpec{Level::Action, Level::Action, Level::Action};
  PpoBatch b = assemble_ppo_batch(slab, zero_values, o);
  CHECK(b.records.size() == 2);
  CHECK_APPROX(b.records[0].advantages[0], 1.0, 1e-12);
  CHECK_APPROX(b.records[0].advantages[1], 1.0, 1e-12);
  CHECK_APPROX(b.records[1].advantages[0], 1.0, 1e-12);
  CHECK_APPROX(b.records[1].advantages[1], 0.0, 1e-12);
  CHECK(b.advantage_unit_count() == 4);
}

TEST_CASE("PPO assembler: chunk level drops post-reset tail slots") {
  TrajectorySlab slab = tiny_slab({1.0, 0.0, 0.0, 0.0}, {true, false, false, false}, 2);
  PpoAssemblyOptions o;
  o.gae = GaeParams{1.0, 1.0};
  PpoBatch b = assemble_ppo_batch(slab, zero_values, o);
  CHECK(b.records.size() == 2);
  CHECK((b.records[0].counted == std::vector<bool>{true, false}));
  CHECK_APPROX(b.records[0].advantages[0], 1.0, 1e-12);
  CHECK((b.records[1].counted == std::vector<bool>{true, true}));
  CHECK_APPROX(b.records[1].advantages[0], 0.0, 1e-12);
  o.spec = GranularitySpec{Level::Chunk, Level::Chunk, Level::Action};
  CHECK_THROWS_AS(assemble_ppo_batch(slab, zero_values, o), ConfigError);
  o.spec = GranularitySpec{Level::Action, Level::Chunk, Level::Action};
  CHECK_THROWS_AS(assemble_ppo_batch(slab, zero_values, o), UnsupportedCombination);
}

TEST_CASE("PPO assembler: truncation and open-end bootstraps come from the snapshot") {
  // one env, one chunk of 3 slots: truncation at slot 1 (fresh episode on slot 2, open end)
  TrajectorySlab slab;
  slab.num_envs = 1;
  slab.chunk_length = 3;
  slab.tokens_per_action = 1;
  StepRecord rec;
  rec.obs = {0.0};
  rec.chunk.actions.assign(3, TokenAction{{0}});
  rec.token_logprobs = TokenLogprobs{3, 1, {0.0, 0.0, 0.0}};
  rec.rewards = {1.0, 2.0, 4.0};
  rec.terminated = {false, false, false};
  rec.truncated = {false, true, false};
  rec.valid = {true, true, true};
  rec.episode_uid = {0, 0, 1};
  rec.post_obs = {{10.0}, {20.0}, {30.0}};
  rec.value_vector = {0.0, 0.0, 0.0};
  slab.records = {{rec}};
  const ValueFn v = [](const Observation& o, policy::ValueHeadKind) { return std::vector<double>(3, o[0]); };
  PpoAssemblyOptions opt;
  opt.gae = GaeParams{0.5, 1.0};
  opt.spec = GranularitySpec{Level::Action, Level::Action, Level::Action};
  PpoBatch b = assemble_ppo_batch(slab, v, opt);
  // slot 1: 2 + 0.5*20; slot 0: 1 + 0.5*A1; slot 2 (open end): 4 + 0.5*30
  CHECK_APPROX(b.records[0].advantages[1], 12.0, 1e-6);
  CHECK_APPROX(b.records[0].advantages[0], 7.0, 1e-6);
  CHECK_APPROX(b.records[0].advantages[2], 19.0, 1e-6);
}

TrajectorySlab grpo_slab(bool frozen_tail) {
  TrajectorySlab slab;
  slab.num_envs = 2;
  slab.chunk_length = 2;
  slab.tokens_per_action = 1;
  slab.records.resize(2);
  for (int e = 0; e < 2; ++e) {
    const bool ok = e == 0;
    StepRecord rec;
    rec.obs = {0.0};
    rec.chunk.actions.assign(2, TokenAction{{0}});
    rec.token_logprobs = TokenLogprobs{2, 1, {0.0, 0.0}};
    if (frozen_tail) {
      rec.rewards = {ok ? 1.0 : 0.0, 0.0};
      rec.terminated = {ok, ok};
      rec.truncated = {!ok, !ok};
      rec.valid = {true, false};
      rec.episode_uid = {e, -1};
    } else {
      rec.rewards = {0.0, ok ? 1.0 : 0.0};
      rec.terminated = {false, ok};
      rec.truncated = {false, !ok};
      rec.valid = {true, true};
      rec.episode_uid = {e, e};
    }
    rec.post_obs = {{1.0}, {2.0}};
    rec.value_vector = {0.0, 0.0};
    slab.records[e].push_back(rec);
    EpisodeInfo ep;
    ep.uid = e;
    ep.env_id = e;
    ep.length = frozen_tail ? 1 : 2;
    ep.total_reward = ok ? 1.0 : 0.0;
    ep.success = ok;
    ep.first_success_step = ok ? (frozen_tail ? 0 : 1) : -1;
    ep.complete = true;
    ep.group_key = GroupKey{0, frozen_tail ? 4 : 5};
    slab.episodes.push_back(ep);
  }
  return slab;
}

TEST_CASE("GRPO assembler groups episodes and broadcasts advantages") {
  TrajectorySlab slab = grpo_slab(false);
  GrpoAssemblyOptions o;
  o.spec = GranularitySpec{Level::Chunk, Level::Token, Level::Chunk};
  o.eps_std = 0.0;
  GrpoAssemblyResult res = assemble_grpo_batch(slab, o);
  CHECK(res.groups_total == 1 && res.groups_retained == 1);
  CHECK(res.batch.groups.size() == 1);
  const auto& g = res.batch.groups.at(0);
  CHECK(g.trajectories.size() == 2);
  CHECK((g.key == GroupKey{0, 5}));
  CHECK_APPROX(g.trajectories.at(0).advantage, 1.0, 1e-12);
  CHECK_APPROX(g.trajectories.at(1).advantage, -1.0, 1e-12);
  CHECK((g.trajectories.at(0).chunks.at(0).slot_weights == std::vector<double>{0.5, 0.5}));
}

TEST_CASE("GRPO assembler: frozen slots never enter a trajectory") {
  GrpoAssemblyOptions o;
  o.spec = GranularitySpec{Level::Chunk, Level::Token, Level::Chunk};
  o.eps_std = 0.0;
  GrpoAssemblyResult res = assemble_grpo_batch(grpo_slab(true), o);
  CHECK(res.batch.groups.size() == 1);
  for (const auto& tr : res.batch.groups.at(0).trajectories) {
    CHECK(tr.chunks.size() == 1);
    CHECK((tr.chunks.at(0).slots == std::vector<int>{0}));
  }
}

TEST_CASE("GRPO assembler: all-degenerate groups retain nothing; eps 0 raises") {
  TrajectorySlab slab;
  slab.num_envs = 2;
  slab.chunk_length = 1;
  slab.tokens_per_action = 1;
  slab.records.resize(2);
  for (int e = 0; e < 2; ++e) {
    StepRecord rec;
    rec.obs = {0.0};
    rec.chunk.actions.assign(1, TokenAction{{0}});
    rec.token_logprobs = TokenLogprobs{1, 1, {0.0}};
    rec.rewards = {1.0};
    rec.terminated = {true};
    rec.truncated = {false};
    rec.valid = {true};
    rec.episode_uid = {e};
    rec.post_obs = {{0.0}};
    rec.value_vector = {0.0};
    slab.records[e].push_back(rec);
    EpisodeInfo ep;
    ep.uid = e;
    ep.env_id = e;
    ep.length = 1;
    ep.total_reward = 1.0;
    ep.success = true;
    ep.first_success_step = 0;
    ep.complete = true;
    ep.group_key = GroupKey{0, 3};
    slab.episodes.push_back(ep);
  }
  GrpoAssemblyOptions o;
  GrpoAssemblyResult res = assemble_grpo_batch(slab, o);
  CHECK(res.groups_total == 1 && res.groups_retained == 0 && res.batch.groups.empty());
  o.apply_filter = false;
  o.eps_std = 0.0;
  CHECK_THROWS_AS(assemble_grpo_batch(slab, o), DegenerateGroup);
  CHECK_APPROX(slab_success_rate(slab), 1.0, 0.0);
}

// ---- losses (test_optim.cpp:115-180) ---------------------------------------------------------
// A deterministic stand-in policy (vocab 3, C = 2, M = 2) with exact host log-softmax for the
// stored log-probs.
struct ToyNet {
  double shift = 0.0;
  std::vector<double> logits(const Observation& o, std::span<const int> prefix) const {
    std::vector<double> l(3);
    for (int v = 0; v < 3; ++v)
      l[v] = 0.8 * std::sin(1.3 * v + 0.7 * o[0] - 0.4 * o[1] + 0.9 * (double)prefix.size() +
                            0.5 * (prefix.empty() ? 0 : prefix.back()) + shift);
    return l;
  }
  double logprob(const Observation& o, std::span<const int> prefix, int tok) const {
    auto l = logits(o, prefix);
    double mx = l[0];
    for (double x : l) mx = std::max(mx, x);
    double s = 0.0;
    for (double x : l) s += std::exp(x - mx);
    return l[tok] - (mx + std::log(s));
  }
  CurrentPolicy current() const {
    CurrentPolicy p;
    p.forward_logits = [this](const Observation& o, std::span<const int> pre) { return logits(o, pre); };
    p.value = [](const Observation& o, policy::ValueHeadKind k) {
      return std::vector<double>(k == policy::ValueHeadKind::Scalar ? 1 : 2, 0.25 * o[0]);
    };
    return p;
  }
};

struct Fixture {
  std::vector<StepRecord> storage;
  Fixture(uint64_t seed, int records, const ToyNet& old_net) {
    Rng rng(seed);
    for (int r = 0; r < records; ++r) {
      StepRecord rec;
      rec.obs = {rng.normal(), rng.normal()};
      rec.chunk.actions.resize(2);
      for (auto& a : rec.chunk.actions) a.tokens = {(int)rng.below(3), (int)rng.below(3)};
      rec.token_logprobs = TokenLogprobs{2, 2, std::vector<double>(4)};
      std::vector<int> prefix;
      for (int j = 0; j < 2; ++j)
        for (int m = 0; m < 2; ++m) {
          rec.token_logprobs.at(j, m) = old_net.logprob(rec.obs, prefix, rec.chunk.actions[j].tokens[m]);
          prefix.push_back(rec.chunk.actions[j].tokens[m]);
        }
      rec.rewards.assign(2, 0.0);
      rec.terminated.assign(2, false);
      rec.truncated.assign(2, false);
      rec.valid.assign(2, true);
      rec.episode_uid.assign(2, 0);
      rec.post_obs.assign(2, rec.obs);
      rec.value_vector.assign(2, 0.0);
      storage.push_back(rec);
    }
  }
  PpoBatch batch(const GranularitySpec& spec, Rng& rng) const {
    PpoBatch b;
    b.spec = spec;
    b.C = 2;
    b.M = 2;
    const std::size_t U = spec.advantage_level == Level::Chunk ? 1 : 2;
    for (std::size_t r = 0; r < storage.size(); ++r) {
      PpoRecordView v;
      v.rec = &storage[r];
      v.env = (int)r;
      v.counted.assign(2, true);
      v.advantages.resize(U);
      v.returns.resize(U);
      for (double& a : v.advantages) a = rng.normal();
      for (double& x : v.returns) x = rng.normal();
      b.records.push_back(v);
    }
    return b;
  }
};

std::vector<std::size_t> all(std::size_t n) {
  std::vector<std::size_t> i(n);
  for (std::size_t k = 0; k < n; ++k) i[k] = k;
  return i;
}

TEST_CASE("PPO surrogate with rho == 1 equals minus the mean advantage") {
  ToyNet net;
  Fixture f(100, 4, net);
  Rng rng(200);
  PpoBatch b = f.batch({Level::Chunk, Level::Chunk, Level::Chunk}, rng);
  PpoParams p;
  p.value_loss_coef = 0.0;
  p.entropy_coef = 0.0;
  LossDiagnostics d = ppo_loss(net.current(), b, all(4), p);
  double mean = 0.0;
  for (const auto& v : b.records) mean += (float)v.advantages[0];
  mean /= 4.0;
  CHECK_APPROX(d.surrogate, -mean, 1e-6);
  CHECK(d.clip_frac == 0.0);
  CHECK(d.units == 4);
}

TEST_CASE("forced clipping: positive advantage, rho = 2, eps = 0.2") {
  ToyNet net;
  Fixture f(101, 1, net);
  Rng rng(201);
  PpoBatch b = f.batch({Level::Chunk, Level::Chunk, Level::Chunk}, rng);
  b.records[0].advantages[0] = 2.5;
  for (double& v : f.storage[0].token_logprobs.values) v -= std::log(2.0) / 4.0;
  PpoParams p;
  p.value_loss_coef = 0.0;
  p.entropy_coef = 0.0;
  LossDiagnostics d = ppo_loss(net.current(), b, all(1), p);
  CHECK_APPROX(d.surrogate, -1.2 * 2.5, 1e-6);
  CHECK(d.clip_frac == 1.0);
}

TEST_CASE("clip inactivity: surrogate equals the importance-weighted sum at every lp level") {
  ToyNet cur, old;
  old.shift = 0.15;
  Fixture f(102, 4, old);
  Rng rng(202);
  for (Level lp : {Level::Chunk, Level::Action, Level::Token}) {
    PpoBatch b = f.batch({Level::Chunk, lp, Level::Chunk}, rng);
    PpoParams p;
    p.clip_eps = 1e6;
    p.value_loss_coef = 0.0;
    p.entropy_coef = 0.0;
    LossDiagnostics d = ppo_loss(cur.current(), b, all(4), p);
    double direct = 0.0;
    for (const auto& v : b.records) {
      std::vector<double> nl, ol;
      std::vector<int> prefix;
      for (int j = 0; j < 2; ++j)
        for (int m = 0; m < 2; ++m) {
          nl.push_back(cur.logprob(v.rec->obs, prefix, v.rec->chunk.actions[j].tokens[m]));
          ol.push_back(v.rec->token_logprobs.at(j, m));
          prefix.push_back(v.rec->chunk.actions[j].tokens[m]);
        }
      auto agg = [&](const std::vector<double>& x) {
        if (lp == Level::Token) return x;
        if (lp == Level::Action) return std::vector<double>{x[0] + x[1], x[2] + x[3]};
        return std::vector<double>{(x[0] + x[1]) + (x[2] + x[3])};
      };
      auto a = agg(nl), o = agg(ol);
      for (std::size_t u = 0; u < a.size(); ++u) direct += std::exp(a[u] - o[u]) * (float)v.advantages[0];
    }
    CHECK_APPROX(d.surrogate, -direct / 4.0, 1e-5);
    CHECK(d.clip_frac == 0.0);
  }
}

TEST_CASE("minibatch: record order does not change the loss; subsets normalise by their own units") {
  ToyNet cur, old;
  old.shift = 0.05;
  Fixture f(103, 6, old);
  Rng rng(203);
  PpoBatch b = f.batch({Level::Action, Level::Token, Level::Action}, rng);
  PpoParams p;
  const std::vector<std::size_t> fwd{0, 1, 2, 3, 4, 5}, rev{5, 4, 3, 2, 1, 0}, sub{1, 4};
  LossDiagnostics a = ppo_loss(cur.current(), b, fwd, p), c = ppo_loss(cur.current(), b, rev, p);
  CHECK_APPROX(a.loss, c.loss, 1e-6);
  CHECK(a.units == 24 && c.units == 24);
  LossCoefficients k;
  LossDiagnostics s = ppo_loss(cur.current(), b, sub, p, &k);
  CHECK(s.units == 8);
  CHECK(k.coeff_logprob.size() == 8 && k.coeff_value.size() == 4);
  // an assembled batch accepts a device-resident logits view in record order
  TrajectorySlab slab;
  slab.num_envs = 1;
  slab.chunk_length = 2;
  slab.tokens_per_action = 2;
  slab.records = {std::vector<StepRecord>(f.storage.begin(), f.storage.end())};
  PpoAssemblyOptions o;
  o.spec = GranularitySpec{Level::Chunk, Level::Chunk, Level::Chunk};
  PpoBatch ab = assemble_ppo_batch(slab, zero_values, o);
  std::vector<float> lg;
  for (const auto& rec : slab.records[0]) {
    std::vector<int> prefix;
    for (int j = 0; j < 2; ++j)
      for (int m = 0; m < 2; ++m) {
        for (double x : cur.logits(rec.obs, prefix)) lg.push_back((float)x);
        prefix.push_back(rec.chunk.actions[j].tokens[m]);
      }
  }
  std::vector<float> vals(6, 0.0f);
  for (int r = 0; r < 6; ++r) vals[r] = (float)(0.25 * slab.records[0][r].obs[0]);
  CurrentPolicy view;
  view.logits = lg.data();
  view.values = vals.data();
  view.vocab = 3;
  view.device = false;
  LossDiagnostics v1 = ppo_loss(view, ab, fwd, p);
  LossDiagnostics v2 = ppo_loss(cur.current(), ab, fwd, p);
  CHECK_APPROX(v1.loss, v2.loss, 1e-6);
  CHECK(v1.units == v2.units);
  // the same policy as finished token rows (the tensor-core head's output format)
  std::vector<ckrl_token_row> rows;
  for (const auto& rec : slab.records[0]) {
    std::vector<int> prefix;
    for (int j = 0; j < 2; ++j)
      for (int m = 0; m < 2; ++m) {
        std::vector<double> l;
        for (double x : cur.logits(rec.obs, prefix)) l.push_back((float)x);  // as the f32 view
        double mx = l[0], s = 0.0, h = 0.0;
        for (double x : l) mx = std::max(mx, x);
        for (double x : l) s += std::exp(x - mx);
        const double lse = mx + std::log(s);
        for (double x : l) h -= std::exp(x - lse) * (x - lse);
        const int tok = rec.chunk.actions[j].tokens[m];
        rows.push_back(ckrl_token_row{l[tok] - lse, (float)h, 0u});
        prefix.push_back(tok);
      }
  }
  CurrentPolicy rview = view;
  rview.logits = rows.data();
  rview.logits_dtype = CKRL_DTYPE_TOKEN_ROWS;
  LossDiagnostics v3 = ppo_loss(rview, ab, fwd, p);
  CHECK_APPROX(v3.loss, v1.loss, 1e-6);
  CHECK_APPROX(v3.entropy, v1.entropy, 1e-6);
  CHECK(v3.units == v1.units);
}

TEST_CASE("errors keep the reference's types") {
  CHECK_THROWS_AS(validate_granularity({Level::Action, Level::Chunk, Level::Action}), UnsupportedCombination);
  CHECK_THROWS_AS(validate_granularity({Level::Token, Level::Token, Level::Chunk}), UnsupportedCombination);
  CHECK(level_from_name("action_level") == Level::Action);
  CHECK_THROWS_AS(level_from_name("bogus"), ConfigError);
  ToyNet net;
  GrpoAssemblyResult empty;
  empty.batch.C = 1;
  CHECK_THROWS_AS(grpo_loss(net.current(), empty.batch, std::vector<std::size_t>{}, GrpoParams{}), SkipUpdate);
}

TEST_CASE("GRPO loss: two-member group, equal weights") {
  TrajectorySlab slab = grpo_slab(false);
  GrpoAssemblyOptions o;
  o.spec = GranularitySpec{Level::Chunk, Level::Chunk, Level::Chunk};
  o.eps_std = 0.0;
  GrpoAssemblyResult res = assemble_grpo_batch(slab, o);
  // rho == 1 (stored lps are 0 and the policy puts all mass on token 0): surrogate =
  // (1/G) * sum_i w_i * A_i = 0.5 * (1 - 1) = 0
  CurrentPolicy p;
  p.forward_logits = [](const Observation&, std::span<const int>) { return std::vector<double>{0.0, -1e4}; };
  LossDiagnostics d = grpo_loss(p, res.batch, std::vector<std::size_t>{0}, GrpoParams{});
  CHECK(std::fabs(d.loss) <= 1e-6);
  CHECK(d.units == 2);
}

TEST_CASE("logits gradient seam matches the reference's per-position formula") {
  // policy_net.cpp:444-456 restated in double on the host for a 3-position chunk of 5 bins
  const int V = 5;
  const std::vector<double> lg = {0.1, -1.2, 2.0, 0.3, 0.0, 1.5, 1.5, -0.5, 0.2, 3.0, -2.0, 0.0, 0.7, 0.1, -0.4};
  const std::vector<int> tok = {2, 4, 0};
  const std::vector<double> klp = {0.25, 0.0, -1.5}, kent = {0.01, 0.0, 0.02};
  std::vector<double> got = policy::chunk_logits_gradient(lg, V, tok, klp, kent);
  CHECK(got.size() == lg.size());
  for (int k = 0; k < 3; ++k) {
    double mx = lg[k * V];
    for (int v = 0; v < V; ++v) mx = std::max(mx, lg[k * V + v]);
    double s = 0.0;
    for (int v = 0; v < V; ++v) s += std::exp(lg[k * V + v] - mx);
    const double lse = mx + std::log(s);
    double H = 0.0;
    for (int v = 0; v < V; ++v) H -= std::exp(lg[k * V + v] - lse) * (lg[k * V + v] - lse);
    for (int v = 0; v < V; ++v) {
      const double ls = lg[k * V + v] - lse, p = std::exp(ls);
      double want = klp[k] * ((v == tok[k] ? 1.0 : 0.0) - p) + kent[k] * (-p * (ls + H));
      if (klp[k] == 0.0 && kent[k] == 0.0) want = 0.0;
      CHECK(std::fabs(got[k * V + v] - want) <= 1e-6 * std::max(1.0, std::fabs(want)));
    }
  }
  std::vector<double> bad = klp;
  bad[2] = std::nan("");
  CHECK_THROWS_AS(policy::chunk_logits_gradient(lg, V, tok, bad, kent), NonFinite);
  CHECK_THROWS_AS(policy::chunk_logits_gradient(lg, V, tok, std::vector<double>{1.0}, kent), LengthMismatch);
}

TEST_CASE("Adam on the quadratic probe drives parameters toward zero") {
  // tests/test_optim.cpp:464-475
  std::vector<double> theta{1.0, -2.0, 3.0};
  Adam adam(3, 0.1);
  for (int i = 0; i < 200; ++i) {
    std::vector<double> grad = theta;
    adam.step(theta, grad);
  }
  for (double v : theta) CHECK(std::abs(v) < 0.05);
}

TEST_CASE("Adam gradient norm clipping") {
  // tests/test_optim.cpp:477-484
  std::vector<double> theta{0.0, 0.0};
  Adam adam(2, 0.1, 1.0);
  std::vector<double> grad{30.0, 40.0};
  double norm = adam.step(theta, grad);
  CHECK_APPROX(norm, 50.0, 1e-12);
  CHECK_APPROX(std::sqrt(grad[0] * grad[0] + grad[1] * grad[1]), 1.0, 1e-9);
  std::vector<double> bad{std::nan(""), 1.0};
  CHECK_THROWS_AS(adam.step(theta, bad), NonFinite);
  std::vector<double> short_grad{1.0};
  CHECK_THROWS_AS(adam.step(theta, short_grad), LengthMismatch);
}

TEST_CASE("dump_slab and the CKRL checkpoint keep the reference's formats") {
  // core/types.cpp:9-28 on a 1-env, 2-record, C = 2 slab (uid = env << 32 | k)
  TrajectorySlab slab;
  slab.num_envs = 1;
  slab.chunk_length = 2;
  slab.tokens_per_action = 2;
  slab.records.resize(1);
  for (int t = 0; t < 2; ++t) {
    StepRecord r;
    r.chunk.actions.resize(2);
    for (int j = 0; j < 2; ++j) r.chunk.actions[static_cast<std::size_t>(j)].tokens = {t + j, 3};
    r.rewards = {0.1, t == 1 ? 1.1 : 0.0};
    r.terminated = {false, t == 1};
    r.truncated = {false, false};
    r.valid = {true, true};
    r.episode_uid = {0, 0};
    slab.records[0].push_back(r);
  }
  const std::string want =
      "# env_id episode_uid step tokens[2] reward terminated truncated valid\n"
      "0 0 0 0 3 0.10000000000000001 0 0 1\n"
      "0 0 1 1 3 0 0 0 1\n"
      "0 0 2 1 3 0.10000000000000001 0 0 1\n"
      "0 0 3 2 3 1.1000000000000001 1 0 1\n";
  CHECK(dump_slab(slab) == want);
  // checkpoint round trip; a count mismatch is the reference's Error
  policy::PolicyDescriptor d{6, 4, 1, 3, 5, 2, 2};
  const ckrl_policy_desc cd{6, 4, 1, 3, 5, 2, 2};
  std::vector<double> p(static_cast<std::size_t>(ckrl_policy_num_params(&cd)));
  for (std::size_t i = 0; i < p.size(); ++i) p[i] = 0.25 * static_cast<double>(i) - 3.0;
  const std::string path = "/tmp/ckrl_dropin_test.ckrl";
  policy::save_checkpoint(d, p, path);
  auto [d2, p2] = policy::load_checkpoint(path);
  CHECK(d2 == d);
  CHECK(p2 == p);
  CHECK_THROWS_AS(policy::save_checkpoint(d, std::vector<double>(3, 0.0), path), LengthMismatch);
  CHECK_THROWS_AS(policy::load_checkpoint("/tmp/ckrl_dropin_missing.ckrl"), Error);
}

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "--list") == 0) {
    for (const auto& c : cases()) std::printf("%s\n", c.name);
    return 0;
  }
  int failed_cases = 0;
  for (const auto& c : cases()) {
    if (argc > 1 && std::strstr(c.name, argv[1]) == nullptr) continue;  // optional name filter
    const int before = g_failures;
    try {
      c.fn();
    } catch (const std::exception& ex) {
      ++g_failures;
      std::fprintf(stderr, "  EXCEPTION: %s\n", ex.what());
    }
    const bool ok = g_failures == before;
    failed_cases += ok ? 0 : 1;
    std::printf("[%s] %s\n", ok ? " ok " : "FAIL", c.name);
  }
  std::printf("%zu cases, %d failed, %d failed checks\n", cases().size(), failed_cases, g_failures);
  return failed_cases ? 1 : 0;
}
