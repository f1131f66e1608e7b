// (e) The hybrid fine-grained rollout pipeline on CUDA streams and events (cfg5).
//
// Reference: placement/rollout.cpp:11-109 (StageSim / StageGen / merge_stages),
// placement/real_backend.cpp:59-138 (two workers exchanging obs / action batches over FIFO
// channels), envsim/vec_env.cpp:31-288 (ToyReach / Scripted dynamics, resets, chunk_step),
// policy/policy_net.cpp:197-403 (trunk, log-softmax, inverse-CDF sampling, value heads).
//
// B200 form: the env partitions of the k pipeline stages live in HBM; "sim" (env chunk
// step, one thread per env) and "gen" (policy sampling, one warp per env) are kernels on
// two streams; per-stage CUDA events replace the channels: gen(s,t) waits sim(s,t-1),
// sim(s,t) waits gen(s,t). With k >= 2, stage s's env step overlaps stage s+1's policy
// inference. Every random draw comes from splitmix64 streams keyed by the global env id
// (env dynamics: mix_seed(seed, gid); sampling: mix_seed(sample_seed, 0xac7100f + gid)),
// so the slab is bit-identical for every k — the reference's scheduling-invariance
// contract (tests/acceptance.cpp:245-311).
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace ckrl {

// ---- core/rng.hpp:11-57 ------------------------------------------------------------------
__host__ __device__ inline uint64_t rng_next(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t rng_make(uint64_t seed) {
  uint64_t s = seed;
  rng_next(s);
  rng_next(s);
  return s;
}
__host__ __device__ inline double rng_double(uint64_t& s) {
  return (double)(rng_next(s) >> 11) * 0x1.0p-53;
}
__host__ __device__ inline uint64_t rng_below(uint64_t& s, uint64_t n) { return rng_next(s) % n; }
__host__ __device__ inline uint64_t mix_seed(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9e3779b97f4a7c15ull * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// ---- PolicyNet parameter layout (policy/policy_net.cpp:107-152) --------------------------
struct PolicyLayout {
  int D, H, L, Hv, V, C, M, P;
  int64_t w_in, b_in, pos_bias, emb, trunk, w_pol, b_pol;
  int64_t v1_w, v1_b, v2_w, v2_b, v3_w, v3_b, c1_w, c1_b, c2_w, c2_b, c3_w, c3_b, total;
};

PolicyLayout make_layout(const ckrl_policy_desc& d) {
  PolicyLayout L;
  L.D = d.obs_dim;
  L.H = d.hidden;
  L.L = d.trunk_layers;
  L.Hv = d.value_hidden;
  L.V = d.vocab;
  L.C = d.chunk_len;
  L.M = d.tokens_per_action;
  L.P = L.C * L.M;
  int64_t off = 0;
  auto take = [&](int64_t n) {
    int64_t at = off;
    off += n;
    return at;
  };
  L.w_in = take((int64_t)L.H * L.D);
  L.b_in = take(L.H);
  L.pos_bias = take((int64_t)L.P * L.H);
  L.emb = take((int64_t)L.P * L.V * L.H);
  L.trunk = take((int64_t)L.L * ((int64_t)L.H * L.H + L.H));
  L.w_pol = take((int64_t)L.V * L.H);
  L.b_pol = take(L.V);
  L.v1_w = take((int64_t)L.Hv * L.H);
  L.v1_b = take(L.Hv);
  L.v2_w = take((int64_t)L.Hv * L.Hv);
  L.v2_b = take(L.Hv);
  L.v3_w = take(L.Hv);
  L.v3_b = take(1);
  L.c1_w = take((int64_t)L.Hv * L.H);
  L.c1_b = take(L.Hv);
  L.c2_w = take((int64_t)L.Hv * L.Hv);
  L.c2_b = take(L.Hv);
  L.c3_w = take((int64_t)L.C * L.Hv);
  L.c3_b = take(L.C);
  L.total = off;
  return L;
}

// ---- env state (envsim/vec_env.hpp:107-125), SoA in the pipeline workspace --------------
struct EnvState {
  int32_t *ax, *ay, *tx, *ty;
  int64_t *episode_step, *global_step, *episode_start;
  int64_t* ep_index;       // per-env episode counter (uid low half), -1 before the first reset
  int32_t* first_success;  // in-episode index, -1
  uint8_t *term, *trunc, *awaiting;
  int32_t* reset_id;
  double* episode_reward;
  uint64_t* rng;      // env dynamics stream
  uint64_t* samp;     // sampling stream (StageGen)
  double* obs;        // [E][D]
  int32_t* ep_count;  // closed episodes per env
  // per-env episode regions, capacity cap_ep each
  int32_t *ep_idx, *ep_len, *ep_fs;
  int64_t* ep_start;
  double* ep_rew;
  int32_t* ep_rid;
  uint8_t* ep_complete;
};

struct PipeArgs {
  ckrl_env_config env;
  PolicyLayout pl;
  const double* params;
  int T;        // chunks in the epoch
  int cap_ep;   // episode capacity per env
  uint64_t sample_seed;
  const int32_t* reset_ids;
  EnvState st;
  ckrl_pipeline_outputs out;
  double* post_obs;  // [E][T][C][D]
};

__device__ void observe(const PipeArgs& a, int e, double* o) {
  const EnvState& s = a.st;
  if (a.env.kind == 0) {
    double d = (double)(a.env.grid_size - 1);
    if (d <= 0.0) d = 1.0;
    o[0] = s.ax[e] / d;
    o[1] = s.ay[e] / d;
    o[2] = s.tx[e] / d;
    o[3] = s.ty[e] / d;
    o[4] = (s.tx[e] - s.ax[e]) / d;
    o[5] = (s.ty[e] - s.ay[e]) / d;
  } else {
    const double id_norm = s.reset_id[e] >= 0 ? (double)(s.reset_id[e] + 1) / (a.env.num_reset_states + 1) : 0.0;
    o[0] = (double)s.episode_step[e] / a.env.max_episode_steps;
    o[1] = id_norm;
  }
}

__device__ void layout_for_id(const PipeArgs& a, int rid, int& ax, int& ay, int& tx, int& ty) {
  uint64_t r = rng_make(mix_seed(mix_seed(a.env.seed, 0x7ab1e5eedull), (uint64_t)rid));
  const uint64_t g = (uint64_t)a.env.grid_size;
  ax = (int)rng_below(r, g);
  ay = (int)rng_below(r, g);
  do {
    tx = (int)rng_below(r, g);
    ty = (int)rng_below(r, g);
  } while (tx == ax && ty == ay);
}

// vec_env.cpp:74-102 (reset_env); returns false on BadResetId
__device__ bool reset_env(const PipeArgs& a, int e, int given_id) {
  EnvState& s = const_cast<EnvState&>(a.st);
  if (a.env.use_fixed_reset_state_ids && given_id < 0 && s.reset_id[e] < 0) return false;
  if (given_id >= 0) {
    if (given_id >= a.env.num_reset_states) return false;
    s.reset_id[e] = given_id;
  } else if (!a.env.use_fixed_reset_state_ids) {
    s.reset_id[e] = -1;
  }
  int ax, ay, tx, ty;
  if (s.reset_id[e] >= 0) {
    layout_for_id(a, s.reset_id[e], ax, ay, tx, ty);
  } else {
    uint64_t r = s.rng[e];
    const uint64_t g = (uint64_t)a.env.grid_size;
    ax = (int)rng_below(r, g);
    ay = (int)rng_below(r, g);
    do {
      tx = (int)rng_below(r, g);
      ty = (int)rng_below(r, g);
    } while (tx == ax && ty == ay);
    s.rng[e] = r;
  }
  s.ax[e] = ax;
  s.ay[e] = ay;
  s.tx[e] = tx;
  s.ty[e] = ty;
  s.ep_index[e] = s.ep_index[e] < 0 ? 0 : s.ep_index[e] + 1;
  s.episode_start[e] = s.global_step[e];
  s.episode_step[e] = 0;
  s.episode_reward[e] = 0.0;
  s.first_success[e] = -1;
  s.term[e] = s.trunc[e] = 0;
  s.awaiting[e] = 0;
  return true;
}

__device__ void close_episode(const PipeArgs& a, int e, bool complete) {
  EnvState& s = const_cast<EnvState&>(a.st);
  const int n = s.ep_count[e];
  if (n >= a.cap_ep) return;
  const int64_t q = (int64_t)e * a.cap_ep + n;
  s.ep_idx[q] = (int32_t)s.ep_index[e];
  s.ep_start[q] = s.episode_start[e];
  s.ep_len[q] = (int32_t)s.episode_step[e];
  s.ep_rew[q] = s.episode_reward[e];
  s.ep_fs[q] = s.first_success[e];
  s.ep_rid[q] = s.reset_id[e];
  s.ep_complete[q] = complete ? 1 : 0;
  s.ep_count[e] = n + 1;
}

// initial reset of a stage's envs (StageSim::initial_obs, rollout.cpp:19-32)
__global__ void env_reset_kernel(PipeArgs a, int first, int count) {
  const int e = first + blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= first + count) return;
  EnvState& s = a.st;
  s.rng[e] = rng_make(mix_seed(a.env.seed, (uint64_t)e));
  s.samp[e] = rng_make(mix_seed(a.sample_seed, 0xac7100full + (uint64_t)e));
  s.ep_index[e] = -1;
  s.global_step[e] = 0;
  s.reset_id[e] = -1;
  s.ep_count[e] = 0;
  s.awaiting[e] = 1;
  if (!reset_env(a, e, a.reset_ids ? a.reset_ids[e] : -1)) a.out.status[0] = CKRL_ERR_BAD_RESET_ID;
  observe(a, e, a.st.obs + (int64_t)e * a.pl.D);
}

// vec_env.cpp:137-199 (step_env) + 250-288 (chunk_step), one thread per env
__global__ void env_chunk_kernel(PipeArgs a, int first, int count, int t) {
  const int e = first + blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= first + count) return;
  EnvState& s = a.st;
  const int C = a.env.chunk_len, M = a.pl.M, D = a.pl.D;
  const bool immediate = !a.env.deferred_reset;
  for (int j = 0; j < C; ++j) {
    if (s.awaiting[e] && a.env.auto_reset && immediate)
      if (!reset_env(a, e, -1)) a.out.status[0] = CKRL_ERR_BAD_RESET_ID;
    const int64_t sl = ((int64_t)e * a.T + t) * C + j;
    double* po = a.post_obs + sl * D;
    float reward = 0.0f;
    uint8_t fl;
    int32_t uid;
    if (s.awaiting[e]) {  // frozen sub-env: flags stay latched, nothing executes
      fl = (s.term[e] ? CKRL_FLAG_TERMINATED : 0) | (s.trunc[e] ? CKRL_FLAG_TRUNCATED : 0);
      uid = -1;
      observe(a, e, po);
    } else {
      const int32_t* tok = a.out.tokens + sl * M;
      double r = 0.0;
      bool success_now;
      const int64_t step_index = s.episode_step[e];
      if (a.env.kind == 0) {
        const int axis = tok[0] % 2;
        const int delta = (tok[1] % 3) - 1;
        const int before = abs(s.ax[e] - s.tx[e]) + abs(s.ay[e] - s.ty[e]);
        const int g = a.env.grid_size;
        if (axis == 0)
          s.ax[e] = min(max(s.ax[e] + delta, 0), g - 1);
        else
          s.ay[e] = min(max(s.ay[e] + delta, 0), g - 1);
        const int after = abs(s.ax[e] - s.tx[e]) + abs(s.ay[e] - s.ty[e]);
        if (a.env.reward_shaping) r += 0.1 * (before - after);
        success_now = after == 0;
        if (success_now) r += 1.0;
      } else {
        success_now = (step_index + 1) == a.env.success_step;
        if (success_now) r = 1.0;
      }
      s.episode_step[e] += 1;
      s.global_step[e] += 1;
      s.episode_reward[e] += r;
      if (success_now && s.first_success[e] < 0) s.first_success[e] = (int32_t)step_index;
      const bool terminated = success_now && !a.env.ignore_terminations;
      bool truncated = s.episode_step[e] >= a.env.max_episode_steps;
      if (terminated) truncated = false;
      reward = (float)r;
      a.out.reward_f64[sl] = r;
      fl = CKRL_FLAG_VALID | (terminated ? CKRL_FLAG_TERMINATED : 0) | (truncated ? CKRL_FLAG_TRUNCATED : 0);
      uid = (int32_t)s.ep_index[e];
      observe(a, e, po);
      if (terminated || truncated) {
        close_episode(a, e, true);
        s.term[e] = terminated;
        s.trunc[e] = truncated;
        s.awaiting[e] = 1;
      }
    }
    if (!(fl & CKRL_FLAG_VALID)) a.out.reward_f64[sl] = 0.0;
    a.out.reward[sl] = reward;
    a.out.flags[sl] = fl;
    a.out.episode_id[sl] = uid;
  }
  if (s.awaiting[e] && a.env.auto_reset)
    if (!reset_env(a, e, -1)) a.out.status[0] = CKRL_ERR_BAD_RESET_ID;
  observe(a, e, s.obs + (int64_t)e * D);
}

// ---- policy (policy_net.cpp:197-403), one warp per env --------------------------------
// Row r of a matvec is owned by lane r % 32 and summed in column order (the reference's
// order); vectors are exchanged through the warp's shared-memory slice.
struct WarpScratch {
  double *x, *h, *lg, *u1, *u2;
  int32_t* prefix;
};

__device__ void matvec_rows(const double* W, const double* bias, int rows, int cols, const double* in,
                            double* out, bool tanh_act, int lane) {
  for (int r = lane; r < rows; r += 32) {
    const double* row = W + (int64_t)r * cols;
    double s = 0.0;
    for (int c = 0; c < cols; ++c) s += row[c] * in[c];
    out[r] = tanh_act ? tanh(s + bias[r]) : s + (bias ? bias[r] : 0.0);
  }
  __syncwarp();
}

// trunk_forward (policy_net.cpp:197-228): feature into ws.h (or ws.x when L == 0)
__device__ const double* trunk(const PipeArgs& a, const double* p, const double* obs, int pos,
                               const WarpScratch& w, int lane) {
  const PolicyLayout& L = a.pl;
  for (int hh = lane; hh < L.H; hh += 32) {
    const double* row = p + L.w_in + (int64_t)hh * L.D;
    double s = 0.0;
    for (int c = 0; c < L.D; ++c) s += row[c] * obs[c];
    s += p[L.b_in + hh] + p[L.pos_bias + (int64_t)pos * L.H + hh];
    for (int k = 0; k < pos; ++k) s += p[L.emb + ((int64_t)k * L.V + w.prefix[k]) * L.H + hh];
    w.x[hh] = s;
  }
  __syncwarp();
  const double* in = w.x;
  double* out = w.h;
  for (int l = 0; l < L.L; ++l) {
    const int64_t base = L.trunk + (int64_t)l * ((int64_t)L.H * L.H + L.H);
    matvec_rows(p + base, p + base + (int64_t)L.H * L.H, L.H, L.H, in, out, true, lane);
    const double* tmp = in;
    in = out;
    out = const_cast<double*>(tmp);
  }
  return in;
}

__device__ void value_head(const PipeArgs& a, const double* p, const double* f, bool scalar,
                           const WarpScratch& w, int lane, double* out) {
  const PolicyLayout& L = a.pl;
  const int64_t w1 = scalar ? L.v1_w : L.c1_w, b1 = scalar ? L.v1_b : L.c1_b;
  const int64_t w2 = scalar ? L.v2_w : L.c2_w, b2 = scalar ? L.v2_b : L.c2_b;
  const int64_t w3 = scalar ? L.v3_w : L.c3_w, b3 = scalar ? L.v3_b : L.c3_b;
  matvec_rows(p + w1, p + b1, L.Hv, L.H, f, w.u1, true, lane);
  matvec_rows(p + w2, p + b2, L.Hv, L.Hv, w.u1, w.u2, true, lane);
  matvec_rows(p + w3, p + b3, scalar ? 1 : L.C, L.Hv, w.u2, out, false, lane);
}

// StageGen::generate (rollout.cpp:68-83): sample_chunk + scalar and vector values
__global__ void gen_kernel(PipeArgs a, int first, int count, int t) {
  extern __shared__ __align__(16) unsigned char smem[];
  const PolicyLayout& L = a.pl;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = first + blockIdx.x * (blockDim.x >> 5) + warp;
  const int per_warp = 2 * L.H + L.V + 2 * L.Hv + L.C + 1;
  WarpScratch w;
  double* base = reinterpret_cast<double*>(smem) + (int64_t)warp * (per_warp + (L.P + 1) / 2 + 1);
  w.x = base;
  w.h = w.x + L.H;
  w.lg = w.h + L.H;
  w.u1 = w.lg + L.V;
  w.u2 = w.u1 + L.Hv;
  w.prefix = reinterpret_cast<int32_t*>(w.u2 + L.Hv + L.C + 1);
  if (e >= first + count) return;
  const double* p = a.params;
  const double* obs = a.st.obs + (int64_t)e * L.D;
  uint64_t rng = a.st.samp[e];
  const int64_t rec = (int64_t)e * a.T + t;
  for (int pos = 0; pos < L.P; ++pos) {
    const double* f = trunk(a, p, obs, pos, w, lane);
    matvec_rows(p + L.w_pol, p + L.b_pol, L.V, L.H, f, w.lg, false, lane);
    // log_softmax (policy_net.cpp:90-102) and inverse-CDF draw (:306-316), in order
    int tok = L.V - 1;
    double lp = 0.0;
    if (lane == 0) {
      double mx = w.lg[0];
      for (int v = 0; v < L.V; ++v) mx = w.lg[v] > mx ? w.lg[v] : mx;
      double sum = 0.0;
      for (int v = 0; v < L.V; ++v) sum += exp(w.lg[v] - mx);
      const double lse = mx + log(sum);
      const double u = rng_double(rng);
      double acc = 0.0;
      for (int v = 0; v < L.V; ++v) {
        acc += exp(w.lg[v] - lse);
        if (u < acc) {
          tok = v;
          break;
        }
      }
      lp = w.lg[tok] - lse;
      w.prefix[pos] = tok;
      const int64_t k = rec * L.P + pos;
      a.out.tokens[k] = tok;
      a.out.old_logprob[k] = (float)lp;
      a.out.old_logprob_f64[k] = lp;
    }
    __syncwarp();
  }
  if (lane == 0) a.st.samp[e] = rng;
  // value heads on the chunk's observation (trunk at position 0, no prefix)
  const double* f = trunk(a, p, obs, 0, w, lane);
  double* vs = w.u2 + L.Hv;  // scalar, then C vector entries
  value_head(a, p, f, true, w, lane, vs);
  if (lane == 0) {
    a.out.value_scalar[rec] = (float)vs[0];
    a.out.value_scalar_f64[rec] = vs[0];
  }
  __syncwarp();
  value_head(a, p, f, false, w, lane, vs);  // same feature: value() recomputes it identically
  for (int c = lane; c < L.C; c += 32) {
    a.out.value_vector[rec * L.C + c] = (float)vs[c];
    a.out.value_vector_f64[rec * L.C + c] = vs[c];
  }
}

// bootstrap values V(post_obs[slot]) for both heads (assembler.cpp:114-118, 148-152)
__global__ void boot_kernel(PipeArgs a, int64_t nslots) {
  extern __shared__ __align__(16) unsigned char smem[];
  const PolicyLayout& L = a.pl;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sl = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  const int per_warp = 2 * L.H + L.V + 2 * L.Hv + L.C + 1;
  WarpScratch w;
  double* base = reinterpret_cast<double*>(smem) + (int64_t)warp * (per_warp + (L.P + 1) / 2 + 1);
  w.x = base;
  w.h = w.x + L.H;
  w.lg = w.h + L.H;
  w.u1 = w.lg + L.V;
  w.u2 = w.u1 + L.Hv;
  w.prefix = reinterpret_cast<int32_t*>(w.u2 + L.Hv + L.C + 1);
  if (sl >= nslots) return;
  const double* obs = a.post_obs + sl * L.D;
  double* vs = w.u2 + L.Hv;
  const double* f = trunk(a, a.params, obs, 0, w, lane);
  value_head(a, a.params, f, true, w, lane, vs);
  if (lane == 0) {
    a.out.boot_scalar[sl] = (float)vs[0];
    a.out.boot_scalar_f64[sl] = vs[0];
  }
  __syncwarp();
  value_head(a, a.params, f, false, w, lane, vs);
  if (lane == 0) {
    a.out.boot_vector0[sl] = (float)vs[0];
    a.out.boot_vector0_f64[sl] = vs[0];
  }
}

// episode_table + merge_stages (rollout.cpp:85-109): closed episodes then the open one per
// env, concatenated in env order (= sorted by (env, start)).
__global__ void episodes_kernel(PipeArgs a) {
  __shared__ int32_t s_off[1025];
  const int E = a.env.num_envs;
  EnvState& s = a.st;
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (!s.awaiting[e] && s.ep_index[e] >= 0) close_episode(a, e, false);  // still running
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t acc = 0;
    for (int e = 0; e < E; ++e) {
      if (e < 1024) s_off[e] = acc;
      acc += s.ep_count[e];
    }
    a.out.episode_count[0] = acc;
    s_off[E < 1024 ? E : 1024] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t o = 0;
    if (e < 1024) {
      o = s_off[e];
    } else {
      for (int q = 0; q < e; ++q) o += s.ep_count[q];
    }
    for (int i = 0; i < s.ep_count[e]; ++i) {
      const int64_t src = (int64_t)e * a.cap_ep + i;
      a.out.ep_env_id[o + i] = e;
      a.out.ep_episode_id[o + i] = s.ep_idx[src];
      a.out.ep_start[o + i] = (int32_t)s.ep_start[src];
      a.out.ep_length[o + i] = s.ep_len[src];
      a.out.ep_total_reward[o + i] = s.ep_rew[src];
      a.out.ep_first_success[o + i] = s.ep_fs[src];
      a.out.ep_complete[o + i] = s.ep_complete[src];
      a.out.ep_task[o + i] = 0;
      a.out.ep_reset_id[o + i] = s.ep_rid[src];
    }
  }
}

// ---- workspace ------------------------------------------------------------------------
size_t pipeline_ws_layout(const ckrl_pipeline_spec& sp, EnvState* st, double** post_obs, char* base) {
  const int E = sp.env.num_envs;
  const int64_t cap = (int64_t)sp.num_chunks * sp.env.chunk_len + 1;
  const int D = sp.policy.obs_dim;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t at = off;
    off = align256(off + bytes);
    return base ? base + at : nullptr;
  };
  EnvState s;
  s.ax = (int32_t*)take(4 * E);
  s.ay = (int32_t*)take(4 * E);
  s.tx = (int32_t*)take(4 * E);
  s.ty = (int32_t*)take(4 * E);
  s.episode_step = (int64_t*)take(8 * E);
  s.global_step = (int64_t*)take(8 * E);
  s.episode_start = (int64_t*)take(8 * E);
  s.ep_index = (int64_t*)take(8 * E);
  s.first_success = (int32_t*)take(4 * E);
  s.term = (uint8_t*)take(E);
  s.trunc = (uint8_t*)take(E);
  s.awaiting = (uint8_t*)take(E);
  s.reset_id = (int32_t*)take(4 * E);
  s.episode_reward = (double*)take(8 * E);
  s.rng = (uint64_t*)take(8 * E);
  s.samp = (uint64_t*)take(8 * E);
  s.obs = (double*)take(8 * (size_t)E * D);
  s.ep_count = (int32_t*)take(4 * E);
  s.ep_idx = (int32_t*)take(4 * E * cap);
  s.ep_len = (int32_t*)take(4 * E * cap);
  s.ep_fs = (int32_t*)take(4 * E * cap);
  s.ep_start = (int64_t*)take(8 * E * cap);
  s.ep_rew = (double*)take(8 * E * cap);
  s.ep_rid = (int32_t*)take(4 * E * cap);
  s.ep_complete = (uint8_t*)take(E * cap);
  double* po = (double*)take(8 * (size_t)E * sp.num_chunks * sp.env.chunk_len * D);
  if (st) *st = s;
  if (post_obs) *post_obs = po;
  return off;
}

size_t pipeline_ws_bytes(const ckrl_pipeline_spec& sp) { return pipeline_ws_layout(sp, nullptr, nullptr, nullptr); }
int64_t policy_num_params(const ckrl_policy_desc& d) { return make_layout(d).total; }

struct PipeStreams {
  cudaStream_t gen = nullptr, sim = nullptr;
  std::vector<cudaEvent_t> obs_ev, act_ev;
  cudaEvent_t fork = nullptr, join_gen = nullptr, join_sim = nullptr;
};

PipeStreams& pipe_streams(int k) {
  static std::mutex mu;
  static PipeStreams ps;
  std::lock_guard<std::mutex> g(mu);
  if (!ps.gen) {
    cudaStreamCreateWithFlags(&ps.gen, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&ps.sim, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&ps.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ps.join_gen, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ps.join_sim, cudaEventDisableTiming);
  }
  while ((int)ps.obs_ev.size() < k) {
    cudaEvent_t a, b;
    cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
    ps.obs_ev.push_back(a);
    ps.act_ev.push_back(b);
  }
  return ps;
}

cudaError_t pipeline_run(const ckrl_pipeline_spec& sp, const double* params, ckrl_pipeline_outputs& out,
                         char* ws, cudaStream_t stream) {
  PipeArgs a;
  std::memset(&a, 0, sizeof(a));
  a.env = sp.env;
  a.pl = make_layout(sp.policy);
  a.params = params;
  a.T = sp.num_chunks;
  a.cap_ep = sp.num_chunks * sp.env.chunk_len + 1;
  a.sample_seed = sp.sample_seed;
  a.reset_ids = sp.reset_state_ids;
  a.out = out;
  pipeline_ws_layout(sp, &a.st, &a.post_obs, ws);
  const int E = sp.env.num_envs, k = sp.stages, per = E / k, T = sp.num_chunks;
  const int gen_warps = 4;
  const size_t gen_smem =
      (size_t)gen_warps * 8 * (2 * a.pl.H + a.pl.V + 2 * a.pl.Hv + a.pl.C + 1 + (a.pl.P + 1) / 2 + 1);
  cudaError_t err = cudaFuncSetAttribute(gen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gen_smem);
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(boot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gen_smem);
  if (err != cudaSuccess) return err;
  PipeStreams& ps = pipe_streams(k);
  cudaEventRecord(ps.fork, stream);
  cudaStreamWaitEvent(ps.gen, ps.fork, 0);
  cudaStreamWaitEvent(ps.sim, ps.fork, 0);
  cudaMemsetAsync(out.status, 0, sizeof(int32_t), ps.sim);
  // Reset (sim side), then per chunk: gen(s,t) after sim(s,t-1); sim(s,t) after gen(s,t).
  for (int s = 0; s < k; ++s) {
    env_reset_kernel<<<(per + 127) / 128, 128, 0, ps.sim>>>(a, s * per, per);
    cudaEventRecord(ps.obs_ev[s], ps.sim);
  }
  for (int t = 0; t < T; ++t)
    for (int s = 0; s < k; ++s) {
      cudaStreamWaitEvent(ps.gen, ps.obs_ev[s], 0);
      gen_kernel<<<(per + gen_warps - 1) / gen_warps, 32 * gen_warps, gen_smem, ps.gen>>>(a, s * per, per, t);
      cudaEventRecord(ps.act_ev[s], ps.gen);
      cudaStreamWaitEvent(ps.sim, ps.act_ev[s], 0);
      env_chunk_kernel<<<(per + 127) / 128, 128, 0, ps.sim>>>(a, s * per, per, t);
      cudaEventRecord(ps.obs_ev[s], ps.sim);
    }
  const int64_t nslots = (int64_t)E * T * sp.env.chunk_len;
  boot_kernel<<<(unsigned)((nslots + gen_warps - 1) / gen_warps), 32 * gen_warps, gen_smem, ps.sim>>>(a, nslots);
  episodes_kernel<<<1, 256, 0, ps.sim>>>(a);
  cudaEventRecord(ps.join_gen, ps.gen);
  cudaEventRecord(ps.join_sim, ps.sim);
  cudaStreamWaitEvent(stream, ps.join_gen, 0);
  cudaStreamWaitEvent(stream, ps.join_sim, 0);
  return cudaGetLastError();
}

}  // namespace ckrl
