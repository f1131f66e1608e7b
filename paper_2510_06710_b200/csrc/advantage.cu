// (c) advantage phase on sm_100a: GAE as a warp-segmented reverse affine scan, PPO
// batch assembly (segmentation, chunk/action units, counted masks, bootstraps) and
// GRPO group assembly (GroupKey ordering, min size, strict filter, group-relative
// advantages, valid-action masks, length-normalised weights).
//
// Reference semantics: advantage/gae.cpp:7-37, advantage/assembler.cpp:33-267,
// advantage/grpo.cpp:9-79, optim/update.cpp:14-45.
#include "common.cuh"
#include "kernels.h"

namespace ckrl {

// One advantage-level unit as the GAE recurrence sees it.
struct Unit {
  bool is_unit;  // false: transparent item (invalid slot / fully frozen chunk)
  bool term, trunc;
  int32_t uid;   // segment key (episode id); units of one segment are contiguous
  double r, v, boot;
  int counted_slots;
};

// ---------------------------------------------------------------------------------
// Warp-cooperative GAE over one env's (or one flat sequence's) item list.
//
// The reference runs, per segment, the reverse loop of gae.cpp:21-35:
//   vnext_i = 0 (terminated) | boot_i (truncated or last of segment) | V_{i+1}
//   A_i     = delta_i + (gamma*lambda) * (segment_end ? 0 : A_{i+1})
// Each unit is the affine map A_i = P_i + Q_i * A_next. Lane l owns a contiguous
// item range, composes its maps locally (reverse), the warp runs an inclusive
// suffix scan of the composed maps with shuffles, and every lane replays its range
// with the exact incoming A. Segment ends come from done flags, uid changes between
// consecutive units and the end of the list (flush_segment's open end).
// ---------------------------------------------------------------------------------
constexpr int kGaeCache = 4;  // items per lane kept in registers across the phases

template <class Acc>
__device__ void warp_gae(Acc& acc, int n_items, double gamma, double lambda, Moments& mom,
                         double& counted_slots) {
  const int lane = threadIdx.x & 31;
  const int per = (n_items + 31) / 32;
  const int lo = min(n_items, lane * per), hi = min(n_items, lo + per);
  const int cnt = hi - lo;
  const double gl = __dmul_rn(gamma, lambda);
  const bool cached = per <= kGaeCache;

  // Load once (independent loads, issued together) when the lane's range is short.
  Unit cache[kGaeCache];
  if (cached) {
#pragma unroll
    for (int q = 0; q < kGaeCache; ++q)
      if (q < cnt) cache[q] = acc.load(lo + q);
  }
  // visit(fn, reverse): apply fn(i, unit) over my range
  auto visit = [&](auto&& fn, bool reverse) {
    if (cached) {
      if (reverse) {
#pragma unroll
        for (int q = kGaeCache - 1; q >= 0; --q)
          if (q < cnt && !fn(lo + q, cache[q])) return;
      } else {
#pragma unroll
        for (int q = 0; q < kGaeCache; ++q)
          if (q < cnt && !fn(lo + q, cache[q])) return;
      }
    } else if (reverse) {
      for (int i = hi - 1; i >= lo; --i) {
        Unit u = acc.load(i);
        if (!fn(i, u)) return;
      }
    } else {
      for (int i = lo; i < hi; ++i) {
        Unit u = acc.load(i);
        if (!fn(i, u)) return;
      }
    }
  };

  // Phase 1: first unit of my range, then nearest such head to my right.
  bool h_has = false;
  int32_t h_uid = 0;
  double h_v = 0.0;
  visit([&](int, const Unit& u) {
    if (!u.is_unit) return true;
    h_has = true;
    h_uid = u.uid;
    h_v = u.v;
    return false;
  }, false);
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    bool o_has = __shfl_down_sync(0xffffffffu, h_has, off);
    int32_t o_uid = __shfl_down_sync(0xffffffffu, h_uid, off);
    double o_v = __shfl_down_sync(0xffffffffu, h_v, off);
    if (!h_has && lane + off < 32) {
      h_has = o_has;
      h_uid = o_uid;
      h_v = o_v;
    }
  }
  bool nx_has0 = __shfl_down_sync(0xffffffffu, h_has, 1);
  int32_t nx_uid0 = __shfl_down_sync(0xffffffffu, h_uid, 1);
  double nx_v0 = __shfl_down_sync(0xffffffffu, h_v, 1);
  if (lane == 31) nx_has0 = false;

  // Phase 2: compose my range's affine map (reverse order).
  double P = 0.0, Q = 1.0;
  {
    bool nx_has = nx_has0;
    int32_t nx_uid = nx_uid0;
    double nx_v = nx_v0;
    visit([&](int, const Unit& u) {
      if (!u.is_unit) return true;
      bool seg_end = u.term || u.trunc || !nx_has || nx_uid != u.uid;
      double vnext = u.term ? 0.0 : ((u.trunc || seg_end) ? u.boot : nx_v);
      double delta = __dadd_rn(__dadd_rn(u.r, __dmul_rn(gamma, vnext)), -u.v);
      double c = seg_end ? 0.0 : gl;
      P = __dadd_rn(delta, __dmul_rn(c, P));
      Q = __dmul_rn(c, Q);
      nx_has = true;
      nx_uid = u.uid;
      nx_v = u.v;
      return true;
    }, true);
  }
  // Phase 3: inclusive suffix scan of maps, G_l = F_l o G_{l+1}.
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    double oP = __shfl_down_sync(0xffffffffu, P, off);
    double oQ = __shfl_down_sync(0xffffffffu, Q, off);
    if (lane + off < 32) {
      P = __dadd_rn(P, __dmul_rn(Q, oP));
      Q = __dmul_rn(Q, oQ);
    }
  }
  double a_in = __shfl_down_sync(0xffffffffu, P, 1);
  if (lane == 31) a_in = 0.0;

  // Phase 4: replay with the exact incoming advantage; write; accumulate stats.
  bool nx_has = nx_has0;
  int32_t nx_uid = nx_uid0;
  double nx_v = nx_v0;
  double a_next = a_in;
  Moments m{0.0, 0.0, 0.0};
  double cs = 0.0;
  visit([&](int i, const Unit& u) {
    if (!u.is_unit) {
      acc.store_empty(i);
      return true;
    }
    bool seg_end = u.term || u.trunc || !nx_has || nx_uid != u.uid;
    double vnext = u.term ? 0.0 : ((u.trunc || seg_end) ? u.boot : nx_v);
    double delta = __dadd_rn(__dadd_rn(u.r, __dmul_rn(gamma, vnext)), -u.v);
    double a = __dadd_rn(delta, __dmul_rn(gl, seg_end ? 0.0 : a_next));
    acc.store(i, u, a, __dadd_rn(a, u.v));
    // Welford update (reverse item order within the lane; deterministic).
    m.n += 1.0;
    double d = a - m.mean;
    m.mean += d / m.n;
    m.m2 += d * (a - m.mean);
    cs += u.counted_slots;
    a_next = a;
    nx_has = true;
    nx_uid = u.uid;
    nx_v = u.v;
    return true;
  }, true);
  // Merge lane moments in lane order (tree over fixed partners => deterministic).
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Moments o;
    o.n = __shfl_down_sync(0xffffffffu, m.n, off);
    o.mean = __shfl_down_sync(0xffffffffu, m.mean, off);
    o.m2 = __shfl_down_sync(0xffffffffu, m.m2, off);
    double ocs = __shfl_down_sync(0xffffffffu, cs, off);
    if ((lane & (2 * off - 1)) == 0 && lane + off < 32) {
      m = merge_moments(m, o);
      cs += ocs;
    }
  }
  mom = m;  // valid in lane 0
  counted_slots = cs;
}

// ---- accessors ------------------------------------------------------------------
struct ChunkAcc {  // chunk-level units: one per record (assembler.cpp:158-190)
  const ckrl_rollout ro;
  int e;
  uint8_t* counted;
  float* adv;
  float* ret;
  __device__ Unit load(int t) const {
    // All C slots' fields are fetched with independent loads first (no data-dependent
    // load chain), then the unit is formed in registers.
    const int C = ro.chunk_len;
    const int64_t rec = (int64_t)e * ro.num_chunks + t;
    const int64_t s0 = rec * C;
    Unit u;
    u.is_unit = false;
    u.term = u.trunc = false;
    u.r = 0.0;
    u.counted_slots = 0;
    u.uid = -1;
    u.v = (double)ro.value_scalar[rec];
    u.boot = 0.0;
    constexpr int kC = 8;
    if (C <= kC) {
      uint8_t f[kC];
      int32_t id[kC];
      float rw[kC], bt[kC];
#pragma unroll
      for (int j = 0; j < kC; ++j)
        if (j < C) {
          f[j] = ro.flags[s0 + j];
          id[j] = ro.episode_id[s0 + j];
          rw[j] = ro.reward[s0 + j];
          bt[j] = ro.bootstrap[s0 + j];
        }
      int first = -1;
#pragma unroll
      for (int j = kC - 1; j >= 0; --j)
        if (j < C && (f[j] & CKRL_FLAG_VALID)) first = j;
      if (first < 0) return u;  // fully frozen chunk
      u.is_unit = true;
#pragma unroll
      for (int j = 0; j < kC; ++j)
        if (j == first) u.uid = id[j];
      bool open = true;
#pragma unroll
      for (int j = 0; j < kC; ++j) {
        if (j < first || j >= C) continue;
        open = open && (f[j] & CKRL_FLAG_VALID) && id[j] == u.uid;  // tail dropped
        if (open) {
          u.r = __dadd_rn(u.r, (double)rw[j]);
          u.term = u.term || (f[j] & CKRL_FLAG_TERMINATED);
          u.trunc = u.trunc || (f[j] & CKRL_FLAG_TRUNCATED);
          u.boot = (double)bt[j];
          ++u.counted_slots;
        }
      }
      return u;
    }
    int first = -1;
    for (int j = 0; j < C; ++j)
      if (ro.flags[s0 + j] & CKRL_FLAG_VALID) {
        first = j;
        break;
      }
    if (first < 0) return u;
    u.is_unit = true;
    u.uid = ro.episode_id[s0 + first];
    int last = first;
    for (int j = first; j < C; ++j) {
      uint8_t fl = ro.flags[s0 + j];
      if (!(fl & CKRL_FLAG_VALID) || ro.episode_id[s0 + j] != u.uid) break;
      u.r = __dadd_rn(u.r, (double)ro.reward[s0 + j]);
      u.term = u.term || (fl & CKRL_FLAG_TERMINATED);
      u.trunc = u.trunc || (fl & CKRL_FLAG_TRUNCATED);
      last = j;
      ++u.counted_slots;
    }
    u.boot = (double)ro.bootstrap[s0 + last];
    return u;
  }
  __device__ void store(int t, const Unit& u, double a, double R) const {
    const int C = ro.chunk_len;
    const int64_t rec = (int64_t)e * ro.num_chunks + t;
    adv[rec] = (float)a;
    ret[rec] = (float)R;
    // counted = the leading episode's contiguous valid prefix from the first valid slot
    int first = -1;
    for (int j = 0; j < C; ++j) {
      bool v = ro.flags[rec * C + j] & CKRL_FLAG_VALID;
      if (first < 0 && v) first = j;
      counted[rec * C + j] = (first >= 0 && j < first + u.counted_slots) ? 1 : 0;
    }
  }
  __device__ void store_empty(int t) const {
    const int C = ro.chunk_len;
    const int64_t rec = (int64_t)e * ro.num_chunks + t;
    adv[rec] = 0.0f;
    ret[rec] = 0.0f;
    for (int j = 0; j < C; ++j) counted[rec * C + j] = 0;
  }
};

struct ActionAcc {  // action-level units: one per valid slot (assembler.cpp:112-146)
  const ckrl_rollout ro;
  int e;
  uint8_t* counted;
  float* adv;
  float* ret;
  __device__ Unit load(int i) const {
    const int64_t s = (int64_t)e * ro.num_chunks * ro.chunk_len + i;
    uint8_t f = ro.flags[s];
    Unit u;
    u.is_unit = (f & CKRL_FLAG_VALID) != 0;
    u.term = f & CKRL_FLAG_TERMINATED;
    u.trunc = f & CKRL_FLAG_TRUNCATED;
    u.uid = ro.episode_id[s];
    u.r = (double)ro.reward[s];
    u.v = (double)ro.value_vector[s];
    u.boot = (double)ro.bootstrap[s];
    u.counted_slots = 1;
    return u;
  }
  __device__ void store(int i, const Unit&, double a, double R) const {
    const int64_t s = (int64_t)e * ro.num_chunks * ro.chunk_len + i;
    adv[s] = (float)a;
    ret[s] = (float)R;
    counted[s] = 1;
  }
  __device__ void store_empty(int i) const {
    const int64_t s = (int64_t)e * ro.num_chunks * ro.chunk_len + i;
    adv[s] = 0.0f;
    ret[s] = 0.0f;
    counted[s] = 0;
  }
};

struct FlatAcc {  // compute_gae over one flat sequence (gae.cpp:7-37)
  const double *r, *v, *b;
  const uint8_t* f;
  double *adv, *ret;
  int base;
  __device__ Unit load(int i) const {
    Unit u;
    u.is_unit = true;
    uint8_t fl = f[base + i];
    u.term = fl & CKRL_FLAG_TERMINATED;
    u.trunc = fl & CKRL_FLAG_TRUNCATED;
    u.uid = 0;
    u.r = r[base + i];
    u.v = v[base + i];
    u.boot = b[base + i];
    u.counted_slots = 0;
    return u;
  }
  __device__ void store(int i, const Unit&, double a, double R) const {
    adv[base + i] = a;
    ret[base + i] = R;
  }
  __device__ void store_empty(int) const {}
};

// Last-block reduction of the per-CTA assembly partials into the rank's StatsRecord.
__device__ void finish_asm_stats(AsmPartial mine, char* ws, const WsLayout L, int M) {
  __shared__ bool is_last;
  __shared__ AsmPartial wpart[kAsmWarpsPerCta];
  AsmPartial* parts = reinterpret_cast<AsmPartial*>(ws + L.asm_partials);
  uint32_t* tickets = reinterpret_cast<uint32_t*>(ws + L.tickets);
  if (threadIdx.x == 0) {
    parts[blockIdx.x] = mine;
    __threadfence();
    uint32_t t = atomicAdd(&tickets[TICKET_ASM], 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // Parallel, fixed-order merge: thread t merges partials t, t+nthr, ... (Chan), then a
  // fixed tree over lanes and warps.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Moments m{0.0, 0.0, 0.0};
  double npos = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    volatile AsmPartial* p = parts + b;
    m = merge_moments(m, Moments{p->n, p->mean, p->m2});
    npos += p->n_pos;
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Moments o;
    o.n = __shfl_down_sync(0xffffffffu, m.n, off);
    o.mean = __shfl_down_sync(0xffffffffu, m.mean, off);
    o.m2 = __shfl_down_sync(0xffffffffu, m.m2, off);
    double op = __shfl_down_sync(0xffffffffu, npos, off);
    if ((lane & (2 * off - 1)) == 0 && lane + off < 32) {
      m = merge_moments(m, o);
      npos += op;
    }
  }
  if (lane == 0) wpart[warp] = AsmPartial{m.n, m.mean, m.m2, npos};
  __syncthreads();
  if (threadIdx.x != 0) return;
  m = Moments{0.0, 0.0, 0.0};
  npos = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    m = merge_moments(m, Moments{wpart[w].n, wpart[w].mean, wpart[w].m2});
    npos += wpart[w].n_pos;
  }
  StatsRecord* st = reinterpret_cast<StatsRecord*>(ws + L.stats_local);
  st->mean = m.mean;
  st->m2 = m.m2;
  st->n_units = (int64_t)m.n;
  st->n_adv = (int64_t)m.n;
  st->n_val = (int64_t)m.n;  // value level == advantage level (assembler.cpp:82)
  st->n_pos = (int64_t)npos * M;
  st->groups_retained = 0;
  st->status = 0;
  tickets[TICKET_ASM] = 0;  // self-reset for the next launch
}

__global__ void __launch_bounds__(kAsmWarpsPerCta * 32)
ppo_assemble_kernel(ckrl_rollout ro, int action_level, double gamma, double lambda,
                    uint8_t* counted, float* adv, float* ret, char* ws, WsLayout L) {
  __shared__ Moments wm[kAsmWarpsPerCta];
  __shared__ double wc[kAsmWarpsPerCta];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * kAsmWarpsPerCta + warp;
  Moments m{0.0, 0.0, 0.0};
  double cs = 0.0;
  if (e < ro.num_envs) {
    if (action_level) {
      ActionAcc acc{ro, e, counted, adv, ret};
      warp_gae(acc, ro.num_chunks * ro.chunk_len, gamma, lambda, m, cs);
    } else {
      ChunkAcc acc{ro, e, counted, adv, ret};
      warp_gae(acc, ro.num_chunks, gamma, lambda, m, cs);
    }
  }
  if (lane == 0) {
    wm[warp] = m;
    wc[warp] = cs;
  }
  __syncthreads();
  AsmPartial p{0.0, 0.0, 0.0, 0.0};
  if (threadIdx.x == 0) {
    Moments acc{0.0, 0.0, 0.0};
    double c = 0.0;
    for (int w = 0; w < kAsmWarpsPerCta; ++w) {
      acc = merge_moments(acc, wm[w]);
      c += wc[w];
    }
    p = AsmPartial{acc.n, acc.mean, acc.m2, c};
  }
  finish_asm_stats(p, ws, L, ro.tokens_per_action);
}

__global__ void flat_gae_kernel(int num_seqs, const int32_t* offs, const double* r,
                                const double* v, const double* b, const uint8_t* f,
                                double gamma, double lambda, double* adv, double* ret) {
  const int q = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (q >= num_seqs) return;
  FlatAcc acc{r, v, b, f, adv, ret, offs[q]};
  Moments m;
  double cs;
  warp_gae(acc, offs[q + 1] - offs[q], gamma, lambda, m, cs);
}

// In-place whitening of the counted advantage units (optim/update.cpp:14-45).
__global__ void normalize_kernel(ckrl_rollout ro, int action_level, const uint8_t* counted,
                                 float* adv, const StatsRecord* recs, int world) {
  __shared__ double s_mean, s_denom;
  __shared__ int s_skip;
  if (threadIdx.x == 0) {
    Moments m{0.0, 0.0, 0.0};
    for (int r = 0; r < world; ++r) m = merge_moments(m, Moments{(double)recs[r].n_units, recs[r].mean, recs[r].m2});
    s_skip = m.n < 2.0;
    s_mean = m.mean;
    s_denom = sqrt(m.m2 / m.n) + 1e-8;
  }
  __syncthreads();
  if (s_skip) return;
  const int C = ro.chunk_len;
  const int64_t nunits = (int64_t)ro.num_envs * ro.num_chunks * (action_level ? C : 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nunits;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool is_unit;
    if (action_level) {
      is_unit = counted[i];
    } else {
      is_unit = false;
      for (int j = 0; j < C; ++j) is_unit = is_unit || counted[i * C + j];
    }
    if (is_unit) adv[i] = (float)(((double)adv[i] - s_mean) / s_denom);
  }
}

// ---------------------------------------------------------------------------------
// GRPO group assembly: one CTA. Eligible episodes (complete && start_step == 0,
// assembler.cpp:207-210) are sorted by (GroupKey, table index) — std::map order with
// members in slab.episodes order — with a shared-memory bitonic sort; groups are
// the runs of equal keys. All group statistics are fp64 in the reference's
// summation order with FMA contraction disabled, so the strict filter decision and
// the advantages are bit-identical to grpo.cpp:9-46.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t group_key(int32_t task, int32_t reset) {
  return ((uint64_t)((uint32_t)task ^ 0x80000000u) << 32) | (uint32_t)((uint32_t)reset ^ 0x80000000u);
}

template <int NT>
__device__ int block_exclusive_scan(int v, int* scratch /*NT/32+1*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int w = 0; w < NT / 32; ++w) {
      int t = scratch[w];
      scratch[w] = acc;
      acc += t;
    }
    scratch[NT / 32] = acc;
  }
  __syncthreads();
  int r = scratch[warp] + x - v;
  __syncthreads();
  return r;
}

constexpr int kGrpoThreads = 1024;

__global__ void __launch_bounds__(kGrpoThreads)
grpo_group_kernel(ckrl_episodes ep, int num_envs, ckrl_grpo_options opt, ckrl_grpo_batch gb,
                  char* ws, WsLayout L) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int scan_scratch[kGrpoThreads / 32 + 1];
  __shared__ int s_n, s_status, s_groups, s_total, s_retained;
  const int tid = threadIdx.x;
  StatsRecord* st = reinterpret_cast<StatsRecord*>(ws + L.stats_local);
  int32_t* env_len = reinterpret_cast<int32_t*>(ws + L.grpo_env);
  int32_t* env_fs = env_len + num_envs;

  for (int e = tid; e < num_envs; e += kGrpoThreads) {
    gb.env_group[e] = -1;
    gb.env_member[e] = -1;
    gb.env_episode[e] = -1;
    gb.env_advantage[e] = 0.0;
    gb.env_group_size[e] = 0;
    env_len[e] = 0;
    env_fs[e] = -1;
  }
  // 1. compact eligible episodes (table order preserved)
  int cap = 1;
  if (tid == 0) s_status = 0;
  // count first to size the sort
  int n_local = 0;
  const int per = (ep.count + kGrpoThreads - 1) / kGrpoThreads;
  const int i0 = min(ep.count, tid * per), i1 = min(ep.count, i0 + per);
  for (int i = i0; i < i1; ++i) n_local += (ep.complete[i] && ep.start_step[i] == 0) ? 1 : 0;
  int base = block_exclusive_scan<kGrpoThreads>(n_local, scan_scratch);
  if (tid == 0) s_n = scan_scratch[kGrpoThreads / 32];
  __syncthreads();
  const int n = s_n;
  if (n > kGrpoMaxEligible) {
    if (tid == 0) {
      st->status = CKRL_ERR_INVALID_ARGUMENT;
      st->groups_retained = 0;
      gb.group_counts[0] = gb.group_counts[1] = 0;
    }
    return;
  }
  while (cap < n) cap <<= 1;
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  int32_t* idx = reinterpret_cast<int32_t*>(keys + kGrpoMaxEligible);
  int32_t* gid = idx + kGrpoMaxEligible;  // reused: group id per sorted position
  for (int i = i0, k = base; i < i1; ++i)
    if (ep.complete[i] && ep.start_step[i] == 0) {
      keys[k] = group_key(ep.task_id[i], ep.reset_state_id[i]);
      idx[k] = i;
      ++k;
    }
  for (int k = n + tid; k < cap; k += kGrpoThreads) {
    keys[k] = ~0ull;
    idx[k] = 0x7fffffff;
  }
  __syncthreads();
  // 2. bitonic sort of (key, idx), skipped when already ordered (the common case:
  // envs laid out group by group, table in env order).
  int unsorted = 0;
  for (int k = tid + 1; k < n; k += kGrpoThreads)
    unsorted |= (keys[k - 1] > keys[k]) || (keys[k - 1] == keys[k] && idx[k - 1] > idx[k]);
  unsorted = __syncthreads_or(unsorted);
  if (unsorted) {
    for (int size = 2; size <= cap; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int k = tid; k < cap; k += kGrpoThreads) {
          int p = k ^ stride;
          if (p > k) {
            bool up = (k & size) == 0;
            uint64_t ka = keys[k], kb = keys[p];
            int32_t ia = idx[k], ib = idx[p];
            bool gt = ka > kb || (ka == kb && ia > ib);
            if (gt == up) {
              keys[k] = kb;
              keys[p] = ka;
              idx[k] = ib;
              idx[p] = ia;
            }
          }
        }
        __syncthreads();
      }
  }
  // 3. group ids = runs of equal keys
  const int per2 = (n + kGrpoThreads - 1) / kGrpoThreads;
  const int k0 = min(n, tid * per2), k1 = min(n, k0 + per2);
  int heads = 0;
  for (int k = k0; k < k1; ++k) heads += (k == 0 || keys[k] != keys[k - 1]);
  int gbase = block_exclusive_scan<kGrpoThreads>(heads, scan_scratch);
  if (tid == 0) s_groups = scan_scratch[kGrpoThreads / 32];
  {
    int g = gbase - 1;
    for (int k = k0; k < k1; ++k) {
      if (k == 0 || keys[k] != keys[k - 1]) ++g;
      gid[k] = g;
    }
  }
  __syncthreads();
  const int G = s_groups;
  // group start positions live in the (now free) tail of the key array
  int32_t* gstart = reinterpret_cast<int32_t*>(smem + (size_t)kGrpoMaxEligible * 16);
  for (int k = tid; k < n; k += kGrpoThreads)
    if (k == 0 || gid[k] != gid[k - 1]) gstart[gid[k]] = k;
  if (tid == 0) gstart[G] = n;
  __syncthreads();
  // 4. per group: kept (min size), mean, strict filter; ordinals by scan
  const int per3 = (G + kGrpoThreads - 1) / kGrpoThreads;
  const int g0 = min(G, tid * per3), g1 = min(G, g0 + per3);
  int kept_l = 0, ret_l = 0;
  for (int g = g0; g < g1; ++g) {
    int sz = gstart[g + 1] - gstart[g];
    if (sz < opt.min_group_size) continue;
    ++kept_l;
    double mean = 0.0;
    for (int k = gstart[g]; k < gstart[g + 1]; ++k) mean = __dadd_rn(mean, ep.total_reward[idx[k]]);
    mean = __ddiv_rn(mean, (double)sz);
    bool keep = !opt.apply_filter || (mean > opt.filter_lower && mean < opt.filter_upper);
    ret_l += keep;
  }
  int rbase = block_exclusive_scan<kGrpoThreads>(ret_l, scan_scratch);
  if (tid == 0) s_retained = scan_scratch[kGrpoThreads / 32];
  int tbase = block_exclusive_scan<kGrpoThreads>(kept_l, scan_scratch);
  if (tid == 0) s_total = scan_scratch[kGrpoThreads / 32];
  (void)tbase;
  // 5. advantages (grpo.cpp:9-28) for retained groups
  int ordinal = rbase;
  for (int g = g0; g < g1; ++g) {
    int b = gstart[g], sz = gstart[g + 1] - b;
    if (sz < opt.min_group_size) continue;
    double mean = 0.0;
    for (int k = b; k < b + sz; ++k) mean = __dadd_rn(mean, ep.total_reward[idx[k]]);
    double mean_f = __ddiv_rn(mean, (double)sz);
    bool keep = !opt.apply_filter || (mean_f > opt.filter_lower && mean_f < opt.filter_upper);
    if (!keep) continue;
    double var = 0.0;
    for (int k = b; k < b + sz; ++k) {
      double d = __dadd_rn(ep.total_reward[idx[k]], -mean_f);
      var = __dadd_rn(var, __dmul_rn(d, d));
    }
    var = __ddiv_rn(var, (double)sz);
    double sd = __dsqrt_rn(var);
    if (sz < 2 || (sd == 0.0 && opt.eps_std == 0.0)) atomicExch(&s_status, CKRL_ERR_DEGENERATE_GROUP);
    double den = __dadd_rn(sd, opt.eps_std);
    for (int k = b; k < b + sz; ++k) {
      int i = idx[k];
      int e = ep.env_id[i];
      if (e < 0 || e >= num_envs) {
        atomicExch(&s_status, CKRL_ERR_INVALID_ARGUMENT);
        continue;
      }
      gb.env_group[e] = ordinal;
      gb.env_member[e] = k - b;
      gb.env_episode[e] = ep.episode_id[i];
      gb.env_advantage[e] = __ddiv_rn(__dadd_rn(ep.total_reward[i], -mean_f), den);
      gb.env_group_size[e] = sz;
      env_len[e] = ep.length[i];
      env_fs[e] = ep.first_success[i];
    }
    ++ordinal;
  }
  __syncthreads();
  if (tid == 0) {
    gb.group_counts[0] = s_total;
    gb.group_counts[1] = s_retained;
    st->mean = 0.0;
    st->m2 = 0.0;
    st->n_units = st->n_adv = st->n_val = st->n_pos = 0;
    st->groups_retained = s_retained;
    st->status = s_status;
  }
}

// Per-slot trajectory membership and weights (assembler.cpp:247-258 with
// grpo.cpp:48-79): one warp per env walks its slots in time order; the in-episode
// index is a warp prefix count of matching slots.
__global__ void grpo_weights_kernel(ckrl_rollout ro, int length_normalized, ckrl_grpo_batch gb,
                                    const char* ws, WsLayout L) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * (blockDim.x >> 5) + warp;
  if (e >= ro.num_envs) return;
  const int32_t* env_len = reinterpret_cast<const int32_t*>(ws + L.grpo_env);
  const int32_t* env_fs = env_len + ro.num_envs;
  const int n = ro.num_chunks * ro.chunk_len;
  const int64_t s0 = (int64_t)e * n;
  const bool has = gb.env_group[e] >= 0;
  const int32_t uid = gb.env_episode[e];
  const int64_t len = has ? env_len[e] : 0;
  const int64_t fs = has ? env_fs[e] : -1;
  const bool success = fs >= 0;
  // valid_action_mask: steps after the first success are invalid (grpo.cpp:48-55)
  const int64_t t_succ = (success && fs + 1 < len) ? fs + 1 : len;
  const double u = length_normalized ? (t_succ > 0 ? 1.0 / (double)t_succ : 0.0)
                                     : (len > 0 ? 1.0 / (double)len : 0.0);
  int k_base = 0;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int i = c0 + lane;
    bool match = false;
    if (i < n && has) {
      uint8_t f = ro.flags[s0 + i];
      match = (f & CKRL_FLAG_VALID) && ro.episode_id[s0 + i] == uid;
    }
    unsigned bal = __ballot_sync(0xffffffffu, match);
    int k = k_base + __popc(bal & ((1u << lane) - 1u));
    if (i < n) {
      float w = 0.0f;
      if (match && k < len) {
        bool valid_step = !(success && k > fs);
        w = (!length_normalized || valid_step) ? (float)u : 0.0f;
      }
      gb.slot_member[s0 + i] = match ? 1 : 0;
      gb.slot_weight[s0 + i] = w;
    }
    k_base += __popc(bal);
  }
}

// ---- launchers ---------------------------------------------------------------------
cudaError_t launch_ppo_assemble(const ckrl_rollout& ro, int action_level, double gamma,
                                double lambda, ckrl_ppo_batch& b, char* ws, const WsLayout& L,
                                cudaStream_t s) {
  int grid = (ro.num_envs + kAsmWarpsPerCta - 1) / kAsmWarpsPerCta;
  ppo_assemble_kernel<<<grid, kAsmWarpsPerCta * 32, 0, s>>>(ro, action_level, gamma, lambda,
                                                             b.counted, b.advantages, b.returns,
                                                             ws, L);
  return cudaGetLastError();
}

cudaError_t launch_flat_gae(int num_seqs, const int32_t* offs, const double* r, const double* v,
                            const double* b, const uint8_t* f, double gamma, double lambda,
                            double* adv, double* ret, cudaStream_t s) {
  int grid = (num_seqs + 3) / 4;
  if (grid > 0)
    flat_gae_kernel<<<grid, 128, 0, s>>>(num_seqs, offs, r, v, b, f, gamma, lambda, adv, ret);
  return cudaGetLastError();
}

cudaError_t launch_normalize(const ckrl_rollout& ro, int action_level, const uint8_t* counted,
                             float* adv, const StatsRecord* recs, int world, cudaStream_t s) {
  int64_t nunits = (int64_t)ro.num_envs * ro.num_chunks * (action_level ? ro.chunk_len : 1);
  int grid = (int)((nunits + 255) / 256);
  if (grid > 1184) grid = 1184;
  if (grid < 1) grid = 1;
  normalize_kernel<<<grid, 256, 0, s>>>(ro, action_level, counted, adv, recs, world);
  return cudaGetLastError();
}

cudaError_t launch_grpo_assemble(const ckrl_rollout& ro, const ckrl_episodes& ep,
                                 const ckrl_grpo_options& opt, ckrl_grpo_batch& gb, char* ws,
                                 const WsLayout& L, cudaStream_t s) {
  size_t smem = (size_t)kGrpoMaxEligible * 16 + sizeof(int32_t) * (kGrpoMaxEligible + 1);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(grpo_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  grpo_group_kernel<<<1, kGrpoThreads, smem, s>>>(ep, ro.num_envs, opt, gb, ws, L);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  int grid = (ro.num_envs + 7) / 8;
  grpo_weights_kernel<<<grid, 256, 0, s>>>(ro, opt.length_normalized, gb, ws, L);
  return cudaGetLastError();
}

}  // namespace ckrl
