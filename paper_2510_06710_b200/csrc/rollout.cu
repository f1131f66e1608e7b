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

// Where generation writes a chunk's action batch: the slab itself (colocated, record
// e * T + t) or the generation side's staging rows (placed, row e, T = 1, t ignored).
struct GenOut {
  int32_t* tokens;
  float* lp;
  double* lp64;
  float* vs;
  double* vs64;
  float* vv;
  double* vv64;
  float* logits;
  int T;       // records per env in this view
  int staged;  // 1: one record per env (the chunk index is not part of the row)
};
__host__ __device__ inline int64_t gen_rec(const GenOut& g, int e, int t) {
  return (int64_t)e * g.T + (g.staged ? 0 : t);
}

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
  const double* packed;  // transposed weight copies (packed_layout)
  struct {
    int64_t win, trunk, wpol, v1, v2, c1, c2, c3;
  } pk;
  int sampler;          // CKRL_SAMPLER_*
  const double* gobs;   // generation's view of the observations [E][D]
  uint64_t* gsamp;      // generation's per-env sampling streams [E]
  GenOut gout;          // generation's action-batch destination
  int gen_split;        // parallel sampler: bit 0 split trunk matvecs, bit 1 split logits matvec
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

// ---- policy (policy_net.cpp:197-403) ------------------------------------------------------
// Products and sums are rounded separately (no FMA contraction), as the reference's x86-64
// build computes them; only exp / log / tanh can differ from glibc (<= 1 ulp).
__device__ __forceinline__ double madd(double s, double a, double b) { return __dadd_rn(s, __dmul_rn(a, b)); }

// out[r] = act(sum_c W[r][c] in[c] (+ bias[r])) from the transposed copy WT[c][r]: row r is
// summed in column order (the reference's order) by one thread; consecutive threads read
// consecutive rows, so every weight load is coalesced.
__device__ void matvec_t(const double* WT, const double* bias, int rows, int cols, const double* in,
                         double* out, bool tanh_act, int tid, int nth) {
  if (cols == 32) {  // the common width: every load issued before the (unchanged) sum chain
    for (int r = tid; r < rows; r += nth) {
      double wv[32], iv[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        wv[c] = __ldg(WT + (int64_t)c * rows + r);
        iv[c] = in[c];
      }
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 32; ++c) s = madd(s, wv[c], iv[c]);
      const double v = bias ? __dadd_rn(s, __ldg(bias + r)) : s;
      out[r] = tanh_act ? tanh(v) : v;
    }
    return;
  }
  for (int r = tid; r < rows; r += nth) {
    double s = 0.0;
#pragma unroll 8
    for (int c = 0; c < cols; ++c) s = madd(s, __ldg(WT + (int64_t)c * rows + r), in[c]);
    const double v = bias ? __dadd_rn(s, __ldg(bias + r)) : s;
    out[r] = tanh_act ? tanh(v) : v;
  }
}

// CKRL_SAMPLER_PARALLEL's matvec: four consecutive threads share a row, each summing a quarter
// of the columns in order, combined as (p0 + p1) + (p2 + p3) by xor shuffles — a fixed order
// (identical for every k and placement) with a dependency chain a quarter as long. nth must be
// a multiple of 32 and every thread must call it (the shuffles span the warp).
__device__ void matvec_split(const double* WT, const double* bias, int rows, int cols, const double* in,
                             double* out, bool tanh_act, int tid, int nth) {
  constexpr int G = 4;
  const int g = tid & (G - 1), per = (cols + G - 1) / G;
  const int c0 = g * per, c1 = min(cols, c0 + per);
  for (int rb = 0; rb < rows; rb += nth / G) {
    const int r = rb + tid / G;
    double s = 0.0;
    if (r < rows) {
      if (c1 - c0 == 8) {  // H = 32: the quarter's loads issued before its sum chain
        double wv[8], iv[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          wv[c] = __ldg(WT + (int64_t)(c0 + c) * rows + r);
          iv[c] = in[c0 + c];
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) s = madd(s, wv[c], iv[c]);
      } else {
#pragma unroll 4
        for (int c = c0; c < c1; ++c) s = madd(s, __ldg(WT + (int64_t)c * rows + r), in[c]);
      }
    }
    s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
    s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
    if (g == 0 && r < rows) {
      const double v = bias ? __dadd_rn(s, __ldg(bias + r)) : s;
      out[r] = tanh_act ? tanh(v) : v;
    }
  }
}

// Transposed copies of every weight matrix (W[rows][cols] -> WT[cols][rows]), built once per
// run into the workspace; biases and embeddings are read in place.
struct PackSeg {
  int64_t src, dst;
  int rows, cols;
};
constexpr int kMaxPackSegs = 8 + 64;

struct PackTable {
  PackSeg seg[kMaxPackSegs];
  int n;
  int64_t total;
};

__global__ void pack_kernel(const double* params, double* packed, PackTable tab) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tab.total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int q = 0;
    int64_t base = 0;
    while (q + 1 < tab.n && i >= base + (int64_t)tab.seg[q].rows * tab.seg[q].cols) {
      base += (int64_t)tab.seg[q].rows * tab.seg[q].cols;
      ++q;
    }
    const PackSeg& g = tab.seg[q];
    const int64_t j = i - base;  // index in W (row-major)
    const int64_t r = j / g.cols, c = j % g.cols;
    packed[g.dst + c * g.rows + r] = params[g.src + j];
  }
}

struct Packed {
  int64_t win, trunk, wpol, v1, v2, c1, c2, c3, total;
};

Packed packed_layout(const PolicyLayout& L, PackTable* tab) {
  Packed k;
  int64_t off = 0;
  int n = 0;
  auto add = [&](int64_t src, int rows, int cols) {
    const int64_t at = off;
    if (tab) tab->seg[n] = PackSeg{src, at, rows, cols};
    ++n;
    off += (int64_t)rows * cols;
    return at;
  };
  k.win = add(L.w_in, L.H, L.D);
  k.trunk = off;
  for (int l = 0; l < L.L; ++l) add(L.trunk + (int64_t)l * ((int64_t)L.H * L.H + L.H), L.H, L.H);
  k.wpol = add(L.w_pol, L.V, L.H);
  k.v1 = add(L.v1_w, L.Hv, L.H);
  k.v2 = add(L.v2_w, L.Hv, L.Hv);
  k.c1 = add(L.c1_w, L.Hv, L.H);
  k.c2 = add(L.c2_w, L.Hv, L.Hv);
  k.c3 = add(L.c3_w, L.C, L.Hv);
  k.total = off;
  if (tab) {
    tab->n = n;
    tab->total = off;
  }
  return k;
}

// Shared-memory slice of one env's policy evaluation (doubles, then the token prefix).
struct PolScratch {
  double *x, *h, *lg, *ex, *u1, *u2, *vs, *f0, *red, *embc;
  int32_t* prefix;
};

__host__ __device__ inline size_t pol_scratch_doubles(const PolicyLayout& L, bool emb_cache) {
  return (size_t)2 * L.H + 2 * L.V + 2 * L.Hv + (L.C + 1) + L.H + 8 + (emb_cache ? (size_t)L.P * L.H : 0) +
         ((size_t)L.P + 1) / 2 + 1;
}

__device__ PolScratch carve(double* base, const PolicyLayout& L, bool emb_cache) {
  PolScratch w;
  w.x = base;
  w.h = w.x + L.H;
  w.lg = w.h + L.H;
  w.ex = w.lg + L.V;
  w.u1 = w.ex + L.V;
  w.u2 = w.u1 + L.Hv;
  w.vs = w.u2 + L.Hv;
  w.f0 = w.vs + L.C + 1;
  w.red = w.f0 + L.H;
  w.embc = w.red + 8;
  w.prefix = reinterpret_cast<int32_t*>(w.embc + (emb_cache ? (size_t)L.P * L.H : 0));
  return w;
}

// trunk layers (policy_net.cpp:214-226) on x -> feature pointer; block- or warp-synchronous
template <bool BLOCK>
__device__ const double* trunk_layers(const PipeArgs& a, const double* pk, const PolScratch& w, int tid,
                                      int nth, bool split = false) {
  const PolicyLayout& L = a.pl;
  const double* in = w.x;
  double* out = w.h;
  for (int l = 0; l < L.L; ++l) {
    const int64_t bias = L.trunk + (int64_t)l * ((int64_t)L.H * L.H + L.H) + (int64_t)L.H * L.H;
    if (split)
      matvec_split(pk + a.pk.trunk + (int64_t)l * L.H * L.H, a.params + bias, L.H, L.H, in, out, true, tid, nth);
    else
      matvec_t(pk + a.pk.trunk + (int64_t)l * L.H * L.H, a.params + bias, L.H, L.H, in, out, true, tid, nth);
    if (BLOCK) __syncthreads(); else __syncwarp();
    double* t = const_cast<double*>(in);
    in = out;
    out = t;
  }
  return in;
}

// value (policy_net.cpp:336-372): both heads on the feature f
template <bool BLOCK>
__device__ void value_heads(const PipeArgs& a, const double* pk, const double* f, const PolScratch& w,
                            int tid, int nth, double* scalar_out, double* vec_out) {
  const PolicyLayout& L = a.pl;
  const double* p = a.params;
  matvec_t(pk + a.pk.v1, p + L.v1_b, L.Hv, L.H, f, w.u1, true, tid, nth);
  if (BLOCK) __syncthreads(); else __syncwarp();
  matvec_t(pk + a.pk.v2, p + L.v2_b, L.Hv, L.Hv, w.u1, w.u2, true, tid, nth);
  if (BLOCK) __syncthreads(); else __syncwarp();
  if (tid == 0) {
    double s = 0.0;
    for (int c = 0; c < L.Hv; ++c) s = madd(s, p[L.v3_w + c], w.u2[c]);
    *scalar_out = __dadd_rn(s, p[L.v3_b]);
  }
  if (BLOCK) __syncthreads(); else __syncwarp();
  matvec_t(pk + a.pk.c1, p + L.c1_b, L.Hv, L.H, f, w.u1, true, tid, nth);
  if (BLOCK) __syncthreads(); else __syncwarp();
  matvec_t(pk + a.pk.c2, p + L.c2_b, L.Hv, L.Hv, w.u1, w.u2, true, tid, nth);
  if (BLOCK) __syncthreads(); else __syncwarp();
  matvec_t(pk + a.pk.c3, p + L.c3_b, L.C, L.Hv, w.u2, vec_out, false, tid, nth);
  if (BLOCK) __syncthreads(); else __syncwarp();
}

#ifndef CKRL_GEN_THREADS
#define CKRL_GEN_THREADS 256
#endif
constexpr int kGenThreads = CKRL_GEN_THREADS;  // threads per env (a multiple of 32, <= 256)
constexpr int kGenWarps = kGenThreads / 32;

// CKRL_SAMPLER_PARALLEL: log_softmax's sum of exp(l_v - max) and the inverse-CDF walk of
// sample_chunk (policy_net.cpp:90-102, 306-316) as block-wide fixed-order reductions: thread i
// owns the contiguous bins [i*q, (i+1)*q) (q = ceil(V / threads)), sums them in bin order, then a
// shuffle tree per warp and the warp totals in warp order (the LSE); the CDF is the same
// partition's inclusive scan (own bins serially, warp Kogge-Stone, warp offsets), and the
// token is the smallest v with u < cdf[v] (V - 1 if none, as the reference). Every thread
// returns the token; w.red[4] = lse. Deterministic and independent of scheduling.
__device__ int sample_parallel(const PolScratch& w, int V, double mx, double u, int tid, double& lse_out) {
  const int lane = tid & 31, warp = tid >> 5;
  const int q = (V + kGenThreads - 1) / kGenThreads;
  const int v0 = tid * q, v1 = min(V, v0 + q);
  // block scratch in w.ex (unused by this sampler): warp sums, warp scan totals, warp minima —
  // distinct slots, so only the three hand-off barriers below are needed
  double* s_sum = w.ex;
  double* s_scan = w.ex + kGenWarps;
  int* s_min = reinterpret_cast<int*>(w.ex + 2 * kGenWarps);
  constexpr int kQ = 8;
  double ex[kQ];  // exp(l_v - max) of this thread's bins (up to 8 kept in registers)
  double part = 0.0;
  for (int v = v0; v < v1; ++v) {
    const double e = exp(__dsub_rn(w.lg[v], mx));
    if (v - v0 < kQ) ex[v - v0] = e;
    part = __dadd_rn(part, e);
  }
  double tot = part;
#pragma unroll
  for (int o = 16; o; o >>= 1) tot = __dadd_rn(tot, __shfl_xor_sync(0xffffffffu, tot, o));
  if (lane == 0) s_sum[warp] = tot;
  __syncthreads();
  double sum = s_sum[0];
#pragma unroll
  for (int q2 = 1; q2 < kGenWarps; ++q2) sum = __dadd_rn(sum, s_sum[q2]);
  const double lse = __dadd_rn(mx, log(sum));
  // probabilities exp(l - max) / sum (one division, no second exp) and this thread's inclusive
  // sum; bins beyond the register block (V > 1024) recompute exp(l - lse)
  const double inv = 1.0 / sum;
  double pv[kQ];
  double acc = 0.0;
  for (int v = v0; v < v1; ++v) {
    const double p = v - v0 < kQ ? ex[v - v0] * inv : exp(__dsub_rn(w.lg[v], lse));
    if (v - v0 < kQ) pv[v - v0] = p;
    acc = __dadd_rn(acc, p);
  }
  // exclusive prefix of the thread totals: warp inclusive scan + preceding warps' totals
  double inc = acc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc = __dadd_rn(inc, y);
  }
  if (lane == 31) s_scan[warp] = inc;
  __syncthreads();
  double base = __shfl_up_sync(0xffffffffu, inc, 1);  // the previous lane's inclusive value
  if (lane == 0) base = 0.0;
  double woff = 0.0;
  for (int q2 = 0; q2 < warp; ++q2) woff = __dadd_rn(woff, s_scan[q2]);
  double c = __dadd_rn(woff, base);
  int hit = V;
  for (int v = v0; v < v1; ++v) {
    c = __dadd_rn(c, v - v0 < kQ ? pv[v - v0] : exp(__dsub_rn(w.lg[v], lse)));
    if (u < c && hit == V) hit = v;
  }
  int m = hit;
#pragma unroll
  for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) s_min[warp] = m;
  __syncthreads();
  m = s_min[0];
#pragma unroll
  for (int q2 = 1; q2 < kGenWarps; ++q2) m = min(m, s_min[q2]);
  lse_out = lse;
  return m < V ? m : V - 1;
}

// StageGen::generate (rollout.cpp:68-83) for one env per CTA: sample_chunk
// (policy_net.cpp:286-331) token by token, then the scalar and vector values of the obs.
__global__ void __launch_bounds__(kGenThreads) gen_kernel(PipeArgs a, int first, int count, int t) {
  extern __shared__ __align__(16) unsigned char smem[];
  const PolicyLayout& L = a.pl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int e = first + blockIdx.x;
  if (e >= first + count) return;
  const PolScratch w = carve(reinterpret_cast<double*>(smem), L, true);
  const double* p = a.params;
  const double* pk = a.packed;
  const double* obs = a.gobs + (int64_t)e * L.D;
  const GenOut& go = a.gout;
  const int64_t rec = gen_rec(go, e, t);
  const bool par = a.sampler == CKRL_SAMPLER_PARALLEL;
  uint64_t rng = (tid == 0 || par) ? a.gsamp[e] : 0;  // parallel: every thread draws the same u
  // H <= threads (one hidden unit per thread): the embedding row of the token just drawn is
  // loaded into a register and consumed only in the next position's trunk input, after the
  // token-independent part (W_in obs + b_in + pos_bias), so its latency overlaps that work;
  // the additions keep the reference's order
  const bool reg_emb = L.H <= kGenThreads;
  double e_new = 0.0, e_run = 0.0;  // (reg_emb, thread hh = tid) latest row / parallel running sum
  // (reg_emb) the chunk's W_in obs (the observation is fixed for the whole chunk), b_in and the
  // next position's pos_bias in registers: the same sums, off the per-position critical path
  double win_obs = 0.0, b_in = 0.0, pb_next = 0.0;
  if (reg_emb && tid < L.H) {
    for (int c = 0; c < L.D; ++c) win_obs = madd(win_obs, __ldg(pk + a.pk.win + (int64_t)c * L.H + tid), obs[c]);
    b_in = __ldg(p + L.b_in + tid);
    pb_next = __ldg(p + L.pos_bias + tid);
  }
  for (int pos = 0; pos < L.P; ++pos) {
    // trunk input (policy_net.cpp:197-212): W_in obs + (b_in + pos_bias) + sum_k emb[k][tok_k]
    for (int hh = tid; hh < L.H; hh += kGenThreads) {
      double s;
      if (reg_emb) {
        s = __dadd_rn(win_obs, __dadd_rn(b_in, pb_next));
        if (pos + 1 < L.P) pb_next = __ldg(p + L.pos_bias + (int64_t)(pos + 1) * L.H + hh);
      } else {
        s = 0.0;
        for (int c = 0; c < L.D; ++c) s = madd(s, __ldg(pk + a.pk.win + (int64_t)c * L.H + hh), obs[c]);
        s = __dadd_rn(s, __dadd_rn(__ldg(p + L.b_in + hh), __ldg(p + L.pos_bias + (int64_t)pos * L.H + hh)));
      }
      if (par) {  // the prefix's embeddings as one running sum
        if (reg_emb) {
          if (pos > 0) {
            e_run = pos == 1 ? e_new : __dadd_rn(e_run, e_new);
            s = __dadd_rn(s, e_run);
          }
        } else if (pos > 0) {
          s = __dadd_rn(s, w.embc[hh]);
        }
      } else if (reg_emb) {
#pragma unroll 8
        for (int k = 0; k + 1 < pos; ++k) s = __dadd_rn(s, w.embc[k * L.H + hh]);
        if (pos > 0) {
          s = __dadd_rn(s, e_new);
          w.embc[(pos - 1) * L.H + hh] = e_new;  // for the later positions' sums
        }
      } else {
#pragma unroll 8
        for (int k = 0; k < pos; ++k) s = __dadd_rn(s, w.embc[k * L.H + hh]);
      }
      w.x[hh] = s;
    }
    __syncthreads();
    const double* f = trunk_layers<true>(a, pk, w, tid, kGenThreads, par && (a.gen_split & 1));
    if (pos == 0)
      for (int hh = tid; hh < L.H; hh += kGenThreads) w.f0[hh] = f[hh];
    // logits (logits_from_feature) + block max
    double mx = -INFINITY;
    if (par && (a.gen_split & 2)) {
      matvec_split(pk + a.pk.wpol, p + L.b_pol, L.V, L.H, f, w.lg, false, tid, kGenThreads);
      __syncthreads();  // rows were written by other threads
    } else {
      matvec_t(pk + a.pk.wpol, p + L.b_pol, L.V, L.H, f, w.lg, false, tid, kGenThreads);
    }
    for (int v = tid; v < L.V; v += kGenThreads) mx = fmax(mx, w.lg[v]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) w.red[warp] = mx;
    __syncthreads();
    {
      double m2 = w.red[0];
#pragma unroll
      for (int q2 = 1; q2 < kGenWarps; ++q2) m2 = fmax(m2, w.red[q2]);
      mx = m2;
    }
    if (go.logits) {
      float* dst = go.logits + (rec * L.P + pos) * (int64_t)L.V;
      for (int v = tid; v < L.V; v += kGenThreads) dst[v] = (float)w.lg[v];
    }
    if (par) {  // fixed-order block reductions / scan (identical for every k and placement)
      double lse;
      const int tok = sample_parallel(w, L.V, mx, rng_double(rng), tid, lse);
      if (tid == 0) {
        const double lp = __dsub_rn(w.lg[tok], lse);
        const int64_t k = rec * L.P + pos;
        go.tokens[k] = tok;
        go.lp[k] = (float)lp;
        go.lp64[k] = lp;
      }
      // every thread holds the token: the running embedding sum of the prefix (a register, or
      // row 0 of the cache) is updated by the thread that reads it in the next trunk input
      if (reg_emb) {
        if (tid < L.H) e_new = __ldg(p + L.emb + ((int64_t)pos * L.V + tok) * L.H + tid);
      } else {
        for (int hh = tid; hh < L.H; hh += kGenThreads)
          w.embc[hh] = __dadd_rn(pos == 0 ? 0.0 : w.embc[hh], __ldg(p + L.emb + ((int64_t)pos * L.V + tok) * L.H + hh));
      }
      continue;
    }
    // log_softmax (policy_net.cpp:90-102): exps in parallel, the sum in v order on thread 0
    for (int v = tid; v < L.V; v += kGenThreads) w.ex[v] = exp(__dsub_rn(w.lg[v], mx));
    __syncthreads();
    if (tid == 0) {
      double sum = 0.0;
#pragma unroll 8
      for (int v = 0; v < L.V; ++v) sum = __dadd_rn(sum, w.ex[v]);
      w.red[4] = __dadd_rn(mx, log(sum));
    }
    __syncthreads();
    const double lse = w.red[4];
    for (int v = tid; v < L.V; v += kGenThreads) w.ex[v] = exp(__dsub_rn(w.lg[v], lse));
    __syncthreads();
    // inverse-CDF draw (policy_net.cpp:306-316)
    if (tid == 0) {
      const double u = rng_double(rng);
      // blocks of 8: the loads leave the dependency chain, one branch per block. The running
      // sum never decreases, so the block whose last partial sum exceeds u holds the token.
      double acc = 0.0;
      int tok = L.V - 1;
      bool found = false;
      int v = 0;
      for (; v + 8 <= L.V; v += 8) {
        double c[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) c[q] = w.ex[v + q];
        c[0] = __dadd_rn(acc, c[0]);
#pragma unroll
        for (int q = 1; q < 8; ++q) c[q] = __dadd_rn(c[q - 1], c[q]);
        if (u < c[7]) {
          int q = 7;
#pragma unroll
          for (int qq = 6; qq >= 0; --qq)
            if (u < c[qq]) q = qq;
          tok = v + q;
          found = true;
          break;
        }
        acc = c[7];
      }
      for (; !found && v < L.V; ++v) {
        acc = __dadd_rn(acc, w.ex[v]);
        if (u < acc) {
          tok = v;
          found = true;
        }
      }
      const double lp = __dsub_rn(w.lg[tok], lse);
      const int64_t k = rec * L.P + pos;
      go.tokens[k] = tok;
      go.lp[k] = (float)lp;
      go.lp64[k] = lp;
      w.prefix[pos] = tok;
    }
    __syncthreads();
    const int tok = w.prefix[pos];
    if (reg_emb) {
      if (tid < L.H) e_new = __ldg(p + L.emb + ((int64_t)pos * L.V + tok) * L.H + tid);
    } else {
      for (int hh = tid; hh < L.H; hh += kGenThreads)
        w.embc[pos * L.H + hh] = __ldg(p + L.emb + ((int64_t)pos * L.V + tok) * L.H + hh);
    }
    // the next position's trunk input reads embc[pos][hh] / e_new from the same thread
  }
  if (tid == 0) a.gsamp[e] = rng;
  __syncthreads();
  // StageGen's value calls re-run the trunk on the obs with an empty prefix: f0
  value_heads<true>(a, pk, w.f0, w, tid, kGenThreads, w.vs, w.vs + 1);
  if (tid == 0) {
    go.vs[rec] = (float)w.vs[0];
    go.vs64[rec] = w.vs[0];
  }
  for (int c = tid; c < L.C; c += kGenThreads) {
    go.vv[rec * L.C + c] = (float)w.vs[1 + c];
    go.vv64[rec * L.C + c] = w.vs[1 + c];
  }
}

// Placed generation: the sampling streams live with the generation role (StageGen owns
// them, rollout.cpp:61-66), seeded by global env id exactly as env_reset_kernel does.
__global__ void gen_init_kernel(PipeArgs a, int first, int count) {
  const int e = first + blockIdx.x * blockDim.x + threadIdx.x;
  if (e < first + count) a.gsamp[e] = rng_make(mix_seed(a.sample_seed, 0xac7100full + (uint64_t)e));
}

// The env side's receive of a stage's action batch (the act channel's recv,
// real_backend.cpp:82-84): staging row e -> slab record e * T + t, one CTA per env.
__global__ void act_scatter_kernel(PipeArgs a, GenOut src, int first, int t) {
  const int e = first + blockIdx.x;
  const PolicyLayout& L = a.pl;
  const int64_t rec = (int64_t)e * a.T + t, row = e;
  for (int i = threadIdx.x; i < L.P; i += blockDim.x) {
    a.out.tokens[rec * L.P + i] = src.tokens[row * L.P + i];
    a.out.old_logprob[rec * L.P + i] = src.lp[row * L.P + i];
    a.out.old_logprob_f64[rec * L.P + i] = src.lp64[row * L.P + i];
  }
  for (int c = threadIdx.x; c < L.C; c += blockDim.x) {
    a.out.value_vector[rec * L.C + c] = src.vv[row * L.C + c];
    a.out.value_vector_f64[rec * L.C + c] = src.vv64[row * L.C + c];
  }
  if (threadIdx.x == 0) {
    a.out.value_scalar[rec] = src.vs[row];
    a.out.value_scalar_f64[rec] = src.vs64[row];
  }
  if (a.out.logits && src.logits) {
    const int64_t n = (int64_t)L.P * L.V;
    const float4* s4 = reinterpret_cast<const float4*>(src.logits + row * n);
    float4* d4 = reinterpret_cast<float4*>(a.out.logits + rec * n);
    if ((n & 3) == 0)
      for (int64_t i = threadIdx.x; i < n / 4; i += blockDim.x) d4[i] = s4[i];
    else
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a.out.logits[rec * n + i] = src.logits[row * n + i];
  }
}

// bootstrap values V(post_obs[slot]) for both heads (assembler.cpp:114-118, 148-152), one
// warp per slot
constexpr int kBootWarps = 4;
__global__ void __launch_bounds__(32 * kBootWarps) boot_kernel(PipeArgs a, int64_t nslots) {
  extern __shared__ __align__(16) unsigned char smem[];
  const PolicyLayout& L = a.pl;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sl = (int64_t)blockIdx.x * kBootWarps + warp;
  const PolScratch w =
      carve(reinterpret_cast<double*>(smem) + (size_t)warp * pol_scratch_doubles(L, false), L, false);
  if (sl >= nslots) return;
  const double* p = a.params;
  const double* pk = a.packed;
  const double* obs = a.post_obs + sl * L.D;
  for (int hh = lane; hh < L.H; hh += 32) {
    double s = 0.0;
    for (int c = 0; c < L.D; ++c) s = madd(s, __ldg(pk + a.pk.win + (int64_t)c * L.H + hh), obs[c]);
    w.x[hh] = __dadd_rn(s, __dadd_rn(p[L.b_in + hh], p[L.pos_bias + hh]));
  }
  __syncwarp();
  const double* f = trunk_layers<false>(a, pk, w, lane, 32);
  value_heads<false>(a, pk, f, w, lane, 32, w.vs, w.vs + 1);
  if (lane == 0) {
    a.out.boot_scalar[sl] = (float)w.vs[0];
    a.out.boot_scalar_f64[sl] = w.vs[0];
    a.out.boot_vector0[sl] = (float)w.vs[1];
    a.out.boot_vector0_f64[sl] = w.vs[1];
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
size_t pipeline_ws_layout(const ckrl_pipeline_spec& sp, EnvState* st, double** post_obs, char* base,
                          double** packed = nullptr) {
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
  double* pw = (double*)take(8 * (size_t)packed_layout(make_layout(sp.policy), nullptr).total);
  if (st) *st = s;
  if (post_obs) *post_obs = po;
  if (packed) *packed = pw;
  return off;
}

size_t staging_bytes(const ckrl_pipeline_spec& sp);
size_t pipeline_ws_bytes(const ckrl_pipeline_spec& sp) {
  size_t n = pipeline_ws_layout(sp, nullptr, nullptr, nullptr);
  if (sp.placed) n += staging_bytes(sp);  // the env side's receive buffers
  return n;
}
int64_t policy_num_params(const ckrl_policy_desc& d) { return make_layout(d).total; }

// One action batch's staging rows ([E] rows: tokens, log-probs, values, optional logits),
// contiguous so a stage's rows [first, first + per) of each field move with one copy.
size_t staging_layout(const ckrl_pipeline_spec& sp, GenOut* g, char* base, bool logits) {
  const int64_t E = sp.env.num_envs, P = (int64_t)sp.policy.chunk_len * sp.policy.tokens_per_action,
                C = sp.policy.chunk_len, V = sp.policy.vocab;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t at = off;
    off = align256(off + bytes);
    return base ? base + at : nullptr;
  };
  GenOut o;
  o.tokens = (int32_t*)take(4 * E * P);
  o.lp = (float*)take(4 * E * P);
  o.lp64 = (double*)take(8 * E * P);
  o.vs = (float*)take(4 * E);
  o.vs64 = (double*)take(8 * E);
  o.vv = (float*)take(4 * E * C);
  o.vv64 = (double*)take(8 * E * C);
  o.logits = logits ? (float*)take(4 * E * P * V) : nullptr;
  o.T = 1;
  o.staged = 1;
  if (g) *g = o;
  return off;
}
size_t staging_bytes(const ckrl_pipeline_spec& sp) { return staging_layout(sp, nullptr, nullptr, true); }

// Generation side of a placed pipeline: the policy copy (+ its transposed weights), the
// sampling streams, the observation batch it receives and the action batch it sends.
struct GenWs {
  double *params, *packed, *obs;
  uint64_t* samp;
  GenOut stage;
};
size_t gen_ws_layout(const ckrl_pipeline_spec& sp, GenWs* g, char* base) {
  const PolicyLayout L = make_layout(sp.policy);
  const int64_t E = sp.env.num_envs;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t at = off;
    off = align256(off + bytes);
    return base ? base + at : nullptr;
  };
  GenWs w;
  w.params = (double*)take(8 * (size_t)L.total);
  w.packed = (double*)take(8 * (size_t)packed_layout(L, nullptr).total);
  w.obs = (double*)take(8 * (size_t)E * L.D);
  w.samp = (uint64_t*)take(8 * (size_t)E);
  char* st = (char*)take(staging_bytes(sp));
  staging_layout(sp, &w.stage, st, true);
  if (g) *g = w;
  return off;
}
size_t pipeline_gen_ws_bytes(const ckrl_pipeline_spec& sp) { return gen_ws_layout(sp, nullptr, nullptr); }

// Streams and events of one device's role (created on that device).
struct RoleStreams {
  std::vector<cudaStream_t> stage;
  std::vector<cudaEvent_t> done;  // per stage: last work of the stage on this role
  cudaEvent_t fork = nullptr;
};
RoleStreams& role_streams(int device, int k) {
  static std::vector<RoleStreams> per_dev;
  if ((int)per_dev.size() <= device) per_dev.resize(device + 1);
  RoleStreams& r = per_dev[device];
  if (!r.fork) cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming);
  while ((int)r.stage.size() < k) {
    cudaStream_t st;
    cudaEvent_t ev;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    r.stage.push_back(st);
    r.done.push_back(ev);
  }
  return r;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

static cudaError_t set_kernel_smem(size_t gen_smem, size_t boot_smem) {
  static thread_local size_t gen_set[64] = {0}, boot_set[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t err;
  if (gen_smem > gen_set[dev & 63]) {
    if ((err = cudaFuncSetAttribute(gen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gen_smem)))
      return err;
    // the transposed weights are re-read every position: leave most of the SM's 256 KB to L1
    if ((err = cudaFuncSetAttribute(gen_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    gen_smem * 3 <= 64 * 1024 ? 25 : 100)))
      return err;
    gen_set[dev & 63] = gen_smem;
  }
  if (boot_smem > boot_set[dev & 63]) {
    if ((err = cudaFuncSetAttribute(boot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)boot_smem)))
      return err;
    boot_set[dev & 63] = boot_smem;
  }
  return cudaSuccess;
}

// RealBackend::run_rollout_epoch (real_backend.cpp:59-138): stage s owns envs
// [s*E/k, (s+1)*E/k) (rollout.cpp:11-17) and runs Reset -> (Gen(t) -> Sim(t)) x T.
//   colocated: stage s on its own stream of the calling device; the k stage streams run
//     concurrently, so stage s's env step overlaps stage s'’s policy inference.
//   placed (spec.placed): the generation role on gen_device with its own policy copy and
//     sampling streams; per chunk the env stream sends the stage's obs rows (peer copy) and
//     records obs_ev[s], the gen stream waits it, samples, sends the action rows back and
//     records done(gen)[s], which the env stream waits before scattering them into the slab
//     and stepping the envs. Bootstrap values and the merged episode table follow on
//     `stream` once every stage has finished.
cudaError_t pipeline_run(const ckrl_pipeline_spec& sp, const double* params, ckrl_pipeline_outputs& out,
                         char* ws, cudaStream_t stream) {
  static std::mutex mu;
  std::lock_guard<std::mutex> guard(mu);
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
  a.sampler = sp.sampler;
  {  // CKRL_GEN_SPLIT (A/B): which matvecs the parallel sampler splits across 4 threads per row
    static int split = -1;
    if (split < 0) {
      const char* env = getenv("CKRL_GEN_SPLIT");
      split = env ? atoi(env) : 1;
    }
    a.gen_split = split;
  }
  double* packed = nullptr;
  const size_t env_ws = pipeline_ws_layout(sp, &a.st, &a.post_obs, ws, &packed);
  a.packed = packed;
  PackTable tab;
  std::memset(&tab, 0, sizeof(tab));
  if (a.pl.L + 7 > kMaxPackSegs) return cudaErrorInvalidValue;
  const Packed pk = packed_layout(a.pl, &tab);
  a.pk.win = pk.win;
  a.pk.trunk = pk.trunk;
  a.pk.wpol = pk.wpol;
  a.pk.v1 = pk.v1;
  a.pk.v2 = pk.v2;
  a.pk.c1 = pk.c1;
  a.pk.c2 = pk.c2;
  a.pk.c3 = pk.c3;
  // colocated generation reads the env state's observations and writes the slab directly
  a.gobs = a.st.obs;
  a.gsamp = a.st.samp;
  a.gout = GenOut{out.tokens, out.old_logprob, out.old_logprob_f64, out.value_scalar, out.value_scalar_f64,
                  out.value_vector, out.value_vector_f64, out.logits, a.T, 0};
  const int E = sp.env.num_envs, k = sp.stages, per = E / k, T = sp.num_chunks;
  const size_t gen_smem = 8 * pol_scratch_doubles(a.pl, true);
  const size_t boot_smem = 8 * (size_t)kBootWarps * pol_scratch_doubles(a.pl, false);
  if (gen_smem > 227 * 1024 || boot_smem > 227 * 1024) return cudaErrorInvalidValue;
  int env_dev = 0;
  cudaError_t err = cudaGetDevice(&env_dev);
  if (err) return err;
  const bool placed = sp.placed;
  const int gen_dev = placed ? sp.gen_device : env_dev;
  if ((err = set_kernel_smem(gen_smem, boot_smem))) return err;
  cudaMemsetAsync(out.status, 0, sizeof(int32_t), stream);
  pack_kernel<<<(unsigned)std::min<int64_t>((tab.total + 255) / 256, 592), 256, 0, stream>>>(params, packed, tab);
  RoleStreams& es = role_streams(env_dev, k);
  cudaEventRecord(es.fork, stream);

  if (!placed) {
    for (int s = 0; s < k; ++s) {
      cudaStream_t st = es.stage[s];
      cudaStreamWaitEvent(st, es.fork, 0);
      env_reset_kernel<<<(per + 127) / 128, 128, 0, st>>>(a, s * per, per);
      for (int t = 0; t < T; ++t) {
        gen_kernel<<<per, kGenThreads, gen_smem, st>>>(a, s * per, per, t);
        env_chunk_kernel<<<(per + 127) / 128, 128, 0, st>>>(a, s * per, per, t);
      }
      cudaEventRecord(es.done[s], st);
      cudaStreamWaitEvent(stream, es.done[s], 0);
    }
  } else {
    // the env side's receive buffers follow its workspace; the gen side's live in gen_workspace
    GenOut recv;
    staging_layout(sp, &recv, ws + env_ws, true);
    if (!out.logits) recv.logits = nullptr;
    GenWs gw;
    gen_ws_layout(sp, &gw, reinterpret_cast<char*>(sp.gen_workspace));
    if (!out.logits) gw.stage.logits = nullptr;
    PipeArgs ag = a;  // generation's view: its own policy copy, streams and staging
    ag.params = gw.params;
    ag.packed = gw.packed;
    ag.gobs = gw.obs;
    ag.gsamp = gw.samp;
    ag.gout = gw.stage;
    const int D = a.pl.D, P = a.pl.P, C = a.pl.C, V = a.pl.V;
    if (gen_dev != env_dev) {  // NVLink peer access both ways (no-op when already enabled)
      cudaDeviceEnablePeerAccess(gen_dev, 0);
      DeviceGuard g(gen_dev);
      cudaDeviceEnablePeerAccess(env_dev, 0);
      cudaGetLastError();
    }
    RoleStreams* gs;
    {
      DeviceGuard g(gen_dev);
      if ((err = set_kernel_smem(gen_smem, boot_smem))) return err;
      gs = &role_streams(gen_dev, k);
      // the policy snapshot moves to the generation role once per epoch
      cudaStream_t g0 = gs->stage[0];
      cudaStreamWaitEvent(g0, es.fork, 0);
      cudaMemcpyPeerAsync(gw.params, gen_dev, params, env_dev, sizeof(double) * (size_t)a.pl.total, g0);
      pack_kernel<<<(unsigned)std::min<int64_t>((tab.total + 255) / 256, 592), 256, 0, g0>>>(gw.params, gw.packed,
                                                                                              tab);
      cudaEventRecord(gs->fork, g0);
    }
    std::vector<cudaEvent_t>& obs_ev = es.done;  // env -> gen: "obs batch of stage s sent"
    auto send_obs = [&](int s) {
      cudaStream_t st = es.stage[s];
      cudaMemcpyPeerAsync(gw.obs + (size_t)s * per * D, gen_dev, a.st.obs + (size_t)s * per * D, env_dev,
                          sizeof(double) * (size_t)per * D, st);
      cudaEventRecord(obs_ev[s], st);
    };
    auto send_act = [&](int s, cudaStream_t st) {  // gen -> env, the stage's rows of every field
      const size_t r0 = (size_t)s * per;
      auto cp = [&](void* dst, const void* src, size_t row_bytes) {
        cudaMemcpyPeerAsync((char*)dst + r0 * row_bytes, env_dev, (const char*)src + r0 * row_bytes, gen_dev,
                            row_bytes * per, st);
      };
      cp(recv.tokens, gw.stage.tokens, 4 * (size_t)P);
      cp(recv.lp, gw.stage.lp, 4 * (size_t)P);
      cp(recv.lp64, gw.stage.lp64, 8 * (size_t)P);
      cp(recv.vs, gw.stage.vs, 4);
      cp(recv.vs64, gw.stage.vs64, 8);
      cp(recv.vv, gw.stage.vv, 4 * (size_t)C);
      cp(recv.vv64, gw.stage.vv64, 8 * (size_t)C);
      if (recv.logits) cp(recv.logits, gw.stage.logits, 4 * (size_t)P * V);
    };
    for (int s = 0; s < k; ++s) {
      cudaStream_t st = es.stage[s];
      cudaStreamWaitEvent(st, es.fork, 0);
      env_reset_kernel<<<(per + 127) / 128, 128, 0, st>>>(a, s * per, per);
      send_obs(s);
      DeviceGuard g(gen_dev);
      cudaStream_t gst = gs->stage[s];
      cudaStreamWaitEvent(gst, gs->fork, 0);
      gen_init_kernel<<<(per + 127) / 128, 128, 0, gst>>>(ag, s * per, per);
    }
    for (int t = 0; t < T; ++t) {
      for (int s = 0; s < k; ++s) {
        {
          DeviceGuard g(gen_dev);
          cudaStream_t gst = gs->stage[s];
          cudaStreamWaitEvent(gst, obs_ev[s], 0);
          gen_kernel<<<per, kGenThreads, gen_smem, gst>>>(ag, s * per, per, t);
          send_act(s, gst);
          cudaEventRecord(gs->done[s], gst);
        }
        cudaStream_t st = es.stage[s];
        cudaStreamWaitEvent(st, gs->done[s], 0);
        act_scatter_kernel<<<per, 128, 0, st>>>(a, recv, s * per, t);
        env_chunk_kernel<<<(per + 127) / 128, 128, 0, st>>>(a, s * per, per, t);
        if (t + 1 < T) send_obs(s);
      }
    }
    for (int s = 0; s < k; ++s) {
      cudaEventRecord(es.done[s], es.stage[s]);
      cudaStreamWaitEvent(stream, es.done[s], 0);
    }
  }
  const int64_t nslots = (int64_t)E * T * sp.env.chunk_len;
  boot_kernel<<<(unsigned)((nslots + kBootWarps - 1) / kBootWarps), 32 * kBootWarps, boot_smem, stream>>>(a, nslots);
  episodes_kernel<<<1, 256, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace ckrl
