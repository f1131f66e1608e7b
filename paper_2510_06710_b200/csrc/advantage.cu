// (c) advantage phase on sm_100a: GAE as a warp-segmented reverse affine scan, PPO
// batch assembly (segmentation, chunk/action units, counted masks, bootstraps) and
// GRPO group assembly (GroupKey ordering, min size, strict filter, group-relative
// advantages, valid-action masks, length-normalised weights).
//
// Reference semantics: advantage/gae.cpp:7-37, advantage/assembler.cpp:33-267,
// advantage/grpo.cpp:9-79, optim/update.cpp:14-45.
#include <algorithm>
#include "common.cuh"
#include "gae.cuh"
#include "kernels.h"

#include <cstdlib>

namespace ckrl {

// Last-block reduction of the per-CTA assembly partials into the rank's StatsRecord
// (fixed order: thread t sums partials t, t+nthr, ...; then a fixed tree).
__device__ void finish_asm_stats(AsmPartial mine, char* ws, const WsLayout L, int M, const ExchangeView& ex) {
  __shared__ bool is_last;
  __shared__ AsmPartial wpart[32];  // any block size up to 1024
  AsmPartial* parts = reinterpret_cast<AsmPartial*>(ws + L.asm_partials);
  uint32_t* tickets = reinterpret_cast<uint32_t*>(ws + L.tickets);
  if (threadIdx.x == 0) {
    parts[blockIdx.x] = mine;
    // one acq_rel ticket: the release publishes this CTA's partial, the acquire (extended to
    // the CTA by the barrier below) makes every earlier CTA's visible to the last one
    uint32_t t;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(&tickets[TICKET_ASM]) : "memory");
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // thread t merges partials t, t + nthr, ... in order; then a fixed tree (deterministic)
  AsmPartial q{{0.0, 0.0, 0.0}, 0.0};
  for (unsigned b0 = 0; b0 < gridDim.x; b0 += 4 * blockDim.x) {  // 4 partials in flight per thread
    AsmPartial v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned b = b0 + threadIdx.x + j * blockDim.x;
      v[j] = b < gridDim.x ? AsmPartial{{__ldcg(&parts[b].m.n), __ldcg(&parts[b].m.mean), __ldcg(&parts[b].m.m2)},
                                        __ldcg(&parts[b].n_pos)}
                           : AsmPartial{{0.0, 0.0, 0.0}, 0.0};
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      q.m = mom_merge(q.m, v[j].m);
      q.n_pos += v[j].n_pos;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const Moments o{__shfl_down_sync(0xffffffffu, q.m.n, off), __shfl_down_sync(0xffffffffu, q.m.mean, off),
                    __shfl_down_sync(0xffffffffu, q.m.m2, off)};
    q.m = mom_merge(q.m, o);
    q.n_pos += __shfl_down_sync(0xffffffffu, q.n_pos, off);
  }
  if (lane == 0) wpart[warp] = q;
  __syncthreads();
  if (threadIdx.x != 0) return;
  AsmPartial t{{0.0, 0.0, 0.0}, 0.0};
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    t.m = mom_merge(t.m, wpart[w].m);
    t.n_pos += wpart[w].n_pos;
  }
  StatsRecord* st = reinterpret_cast<StatsRecord*>(ws + L.stats_local);
  st->mean = t.m.mean;
  st->m2 = t.m.m2;
  st->flags = 0;
  st->n_adv = (int64_t)t.m.n;
  st->n_val = (int64_t)t.m.n;  // value level == advantage level (assembler.cpp:82)
  st->n_pos = (int64_t)t.n_pos * M;
  st->groups_retained = 0;
  st->status = 0;
  tickets[TICKET_ASM] = 0;  // self-reset for the next launch
  if (ex.world > 1)  // to every rank's exchange buffer (NVLink stores)
    ex_publish_stats(ex, *st, tickets + TICKET_EPOCH);
}

// Two schedules: thread-per-env serial walk (short envs: <= kSerialItems items, the common
// case — exact reference operation order) or warp-per-env affine scan (long envs). With
// programmatic dependent launch the kernel lets the loss kernel start right away
// (griddepcontrol.launch_dependents); the loss streams logits while this runs and its unit
// phases wait for completion. The serial schedule's CTAs are small enough to co-reside
// with the loss kernel's CTAs.
template <bool SERIAL>
// 2 warps per CTA (<= 80 regs): a CTA co-resides with a loss CTA (19 warps x 96 regs), so
// the loss kernel's persistent CTAs all start at once under programmatic dependent launch.
__global__ void __launch_bounds__(32 * kAsmWarpsPerCta, 12)
ppo_assemble_kernel(ckrl_rollout ro, int action_level, double gamma, double lambda,
                    uint8_t* counted, double* adv, double* ret, char* ws, WsLayout L, ExchangeView ex) {
  asm volatile("griddepcontrol.launch_dependents;");
  __shared__ GaeSums wsum[kAsmWarpsPerCta];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = action_level ? ro.num_chunks * ro.chunk_len : ro.num_chunks;
  GaeSums g{{0.0, 0.0, 0.0}, 0.0};
  if (SERIAL) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < ro.num_envs)
      g = action_level ? serial_gae(ActionAcc{ro, e, counted, adv, ret}, n_items, gamma, lambda)
                       : serial_gae(ChunkAcc{ro, e, counted, adv, ret}, n_items, gamma, lambda);
    for (int off = 16; off > 0; off >>= 1) {
      const Moments o{__shfl_down_sync(0xffffffffu, g.m.n, off), __shfl_down_sync(0xffffffffu, g.m.mean, off),
                      __shfl_down_sync(0xffffffffu, g.m.m2, off)};
      g.m = mom_merge(g.m, o);
      g.counted_slots += __shfl_down_sync(0xffffffffu, g.counted_slots, off);
    }
  } else {
    const int e = blockIdx.x * kAsmWarpsPerCta + warp;
    if (e < ro.num_envs)
      g = action_level ? env_gae(ActionAcc{ro, e, counted, adv, ret}, n_items, gamma, lambda)
                       : env_gae(ChunkAcc{ro, e, counted, adv, ret}, n_items, gamma, lambda);
  }
  if (lane == 0) wsum[warp] = g;
  __syncthreads();
  AsmPartial p{{0.0, 0.0, 0.0}, 0.0};
  if (threadIdx.x == 0)
    for (int w = 0; w < kAsmWarpsPerCta; ++w) {
      p.m = mom_merge(p.m, wsum[w].m);
      p.n_pos += wsum[w].counted_slots;
    }
  finish_asm_stats(p, ws, L, ro.tokens_per_action, ex);
}

__global__ void flat_gae_kernel(int num_seqs, const int32_t* offs, const double* r,
                                const double* v, const double* b, const uint8_t* f,
                                double gamma, double lambda, double* adv, double* ret) {
  const int q = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (q >= num_seqs) return;
  warp_gae(FlatAcc{r, v, b, f, adv, ret, offs[q]}, offs[q + 1] - offs[q], gamma, lambda);
}

// In-place whitening of the counted advantage units (optim/update.cpp:14-45). The last CTA
// then rewrites the rank's record with the moments of the whitened values (mean 0,
// M2 / denom^2) and marks it whitened, so a following loss uses the advantages as they are
// and a second normalisation re-whitens them as the reference's recomputation would.
__global__ void normalize_kernel(ckrl_rollout ro, int action_level, const uint8_t* counted,
                                 double* adv, StatsRecord* recs, int world, uint32_t* ticket) {
  __shared__ double s_mean, s_denom;
  __shared__ int s_skip;
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    const Moments m = merge_records(recs, world);
    s_skip = m.n < 2.0;
    whitening(m, &s_mean, &s_denom);
  }
  __syncthreads();
  if (!s_skip) {
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
      if (is_unit) adv[i] = (adv[i] - s_mean) / s_denom;
    }
  }
  // every CTA has read the record (above) before the last one rewrites it
  if (threadIdx.x == 0) {
    uint32_t t;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(ticket) : "memory");
    s_last = t == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    *ticket = 0;
    for (int r = 0; r < world; ++r) {
      if (!s_skip) {
        recs[r].m2 = recs[r].m2 / (s_denom * s_denom);
        recs[r].mean = (recs[r].mean - s_mean) / s_denom;
      }
      recs[r].flags |= STATS_WHITENED;
    }
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
                  char* ws, WsLayout L, ExchangeView ex) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int scan_scratch[kGrpoThreads / 32 + 1];
  __shared__ int s_n, s_status, s_groups, s_total, s_retained;
  // the weights kernel (programmatic dependent) may launch now; it waits for this grid
  // before reading the group assignment
  asm volatile("griddepcontrol.launch_dependents;");
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
  // up to kGrpoMaxEligible eligible episodes sort in shared memory; beyond, in the workspace's
  // sort region (one eligible episode per env at most: the one starting at step 0)
  // the shared-memory arrays are sized for min(kGrpoMaxEligible, pow2 >= E) (launch_grpo_assemble):
  // small enough at a few hundred envs for the CTA to share an SM with a loss CTA
  const int scap = min(kGrpoMaxEligible, pow2_at_least(num_envs));
  const bool big = n > scap;
  if (big && n > num_envs) {
    if (tid == 0) {
      *st = StatsRecord{0.0, 0.0, 0, 0, 0, 0, 0, CKRL_ERR_INVALID_ARGUMENT};
      gb.group_counts[0] = gb.group_counts[1] = 0;
      if (ex.world > 1)  // peers must not wait for a record
        ex_publish_stats(ex, *st, reinterpret_cast<uint32_t*>(ws + L.tickets) + TICKET_EPOCH);
    }
    return;
  }
  while (cap < n) cap <<= 1;
  const int capacity = big ? pow2_at_least(num_envs) : scap;
  unsigned char* sort_base = big ? reinterpret_cast<unsigned char*>(ws + L.grpo_sort) : smem;
  uint64_t* keys = reinterpret_cast<uint64_t*>(sort_base);
  int32_t* idx = reinterpret_cast<int32_t*>(keys + capacity);
  int32_t* gid = idx + capacity;  // reused: group id per sorted position
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
  int32_t* gstart = reinterpret_cast<int32_t*>(sort_base + (size_t)capacity * 16);
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
    st->flags = 0;
    st->n_adv = st->n_val = st->n_pos = 0;
    st->groups_retained = s_retained;
    st->status = s_status;
    if (ex.world > 1)  // to every rank's exchange buffer
      ex_publish_stats(ex, *st, reinterpret_cast<uint32_t*>(ws + L.tickets) + TICKET_EPOCH);
  }
}

// Per-slot trajectory membership and weights (assembler.cpp:247-258 with
// grpo.cpp:48-79): one warp per env walks its slots in time order; the in-episode
// index is a warp prefix count of matching slots.
__global__ void grpo_weights_kernel(ckrl_rollout ro, int length_normalized, ckrl_grpo_batch gb,
                                    const char* ws, WsLayout L) {
  // the GRPO step's loss kernel may start streaming logits now (programmatic dependent
  // launch); it reads the group data only after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * (blockDim.x >> 5) + warp;
  if (e >= ro.num_envs) return;
  const int32_t* env_len = reinterpret_cast<const int32_t*>(ws + L.grpo_env);
  const int32_t* env_fs = env_len + ro.num_envs;
  const int n = ro.num_chunks * ro.chunk_len;
  const int64_t s0 = (int64_t)e * n;
  // group assignment / lengths come from grpo_group_kernel, this kernel's PDL primary
  asm volatile("griddepcontrol.wait;" ::: "memory");
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
      double w = 0.0;
      if (match && k < len) {
        bool valid_step = !(success && k > fs);
        w = (!length_normalized || valid_step) ? u : 0.0;
      }
      gb.slot_member[s0 + i] = match ? 1 : 0;
      gb.slot_weight[s0 + i] = w;
    }
    k_base += __popc(bal);
  }
}

// ---- launchers ---------------------------------------------------------------------
static bool serial_gae_enabled() {  // thread-per-env schedule (measured slower; opt-in)
  static int on = -1;
  if (on < 0) {
    const char* env = getenv("CKRL_SERIAL_GAE");
    on = (env && env[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

cudaError_t launch_ppo_assemble(const ckrl_rollout& ro, int action_level, double gamma,
                                double lambda, ckrl_ppo_batch& b, char* ws, const WsLayout& L,
                                cudaStream_t s, const ExchangeView& ex) {
  // The overlapped step's loss kernel (one ~217 KB-smem CTA per SM) starts while this runs:
  // an SM whose L1/shared split was configured for this kernel's small footprint cannot take
  // the loss CTA until it drains and reconfigures, so ask for the maximum carveout here too.
  static bool carve = false;
  if (!carve) {
    cudaFuncSetAttribute(ppo_assemble_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(ppo_assemble_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    carve = true;
  }
  const int n_items = action_level ? ro.num_chunks * ro.chunk_len : ro.num_chunks;
  if (serial_gae_enabled() && n_items <= kSerialItems) {
    const int nt = 32 * kAsmWarpsPerCta;
    const int grid = (ro.num_envs + nt - 1) / nt;
    ppo_assemble_kernel<true><<<grid > 0 ? grid : 1, nt, 0, s>>>(
        ro, action_level, gamma, lambda, b.counted, b.advantages, b.returns, ws, L, ex);
  } else {
    const int grid = (ro.num_envs + kAsmWarpsPerCta - 1) / kAsmWarpsPerCta;
    ppo_assemble_kernel<false><<<grid > 0 ? grid : 1, 32 * kAsmWarpsPerCta, 0, s>>>(
        ro, action_level, gamma, lambda, b.counted, b.advantages, b.returns, ws, L, ex);
  }
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
                             double* adv, StatsRecord* recs, int world, uint32_t* ticket, cudaStream_t s) {
  int64_t nunits = (int64_t)ro.num_envs * ro.num_chunks * (action_level ? ro.chunk_len : 1);
  int grid = (int)((nunits + 255) / 256);
  if (grid > 1184) grid = 1184;
  if (grid < 1) grid = 1;
  normalize_kernel<<<grid, 256, 0, s>>>(ro, action_level, counted, adv, recs, world, ticket);
  return cudaGetLastError();
}

cudaError_t launch_grpo_assemble(const ckrl_rollout& ro, const ckrl_episodes& ep,
                                 const ckrl_grpo_options& opt, ckrl_grpo_batch& gb, char* ws,
                                 const WsLayout& L, cudaStream_t s, const ExchangeView& ex) {
  const int scap = std::min(kGrpoMaxEligible, pow2_at_least(ro.num_envs < 1 ? 1 : ro.num_envs));
  const size_t smem = (size_t)scap * 16 + sizeof(int32_t) * (scap + 1);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(grpo_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((size_t)kGrpoMaxEligible * 16 + sizeof(int32_t) * (kGrpoMaxEligible + 1)));
    attr = (size_t)kGrpoMaxEligible * 16 + sizeof(int32_t) * (kGrpoMaxEligible + 1);
  }
  grpo_group_kernel<<<1, kGrpoThreads, smem, s>>>(ep, ro.num_envs, opt, gb, ws, L, ex);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  // programmatic dependent of the group kernel: its CTAs are resident (and trigger the loss
  // kernel's launch) while the single group CTA runs
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((ro.num_envs + 7) / 8));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, grpo_weights_kernel, ro, (int)opt.length_normalized, gb,
                            (const char*)ws, L);
}

}  // namespace ckrl

namespace ckrl {

// ---------------------------------------------------------------------------------
// Minibatch selection. optim::ppo_loss takes record_indices (losses.hpp:54-56) and
// normalises by the minibatch's own unit counts (losses.cpp:75-87); update_ppo draws
// those minibatches (update.cpp:83-99). The selected records are gathered into a compact
// [n][1] layout (16-byte copies for the logits rows) and each CTA contributes its
// subset partials to the rank's StatsRecord, so a following loss launch on the compact
// view sees exactly the minibatch's n_adv / n_val / n_pos.
// ---------------------------------------------------------------------------------
struct SelectArgs {
  ckrl_rollout src, dst;
  ckrl_ppo_batch sb, db;
  ckrl_policy_outputs sp, dp;
  int action_level, value_action;
  int64_t n;
  const int64_t* idx;
  char* ws;
  WsLayout L;
};

__device__ void copy_bytes(void* dst, const void* src, int64_t bytes) {
  if (((uintptr_t)dst | (uintptr_t)src | (uintptr_t)bytes) % 16 == 0) {
    const int4* s = reinterpret_cast<const int4*>(src);
    int4* d = reinterpret_cast<int4*>(dst);
    for (int64_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) d[i] = __ldg(s + i);
  } else {
    const uint16_t* s = reinterpret_cast<const uint16_t*>(src);
    uint16_t* d = reinterpret_cast<uint16_t*>(dst);
    for (int64_t i = threadIdx.x; i < bytes / 2; i += blockDim.x) d[i] = s[i];
  }
}

__global__ void __launch_bounds__(128) select_records_kernel(SelectArgs a) {
  const int C = a.src.chunk_len, M = a.src.tokens_per_action, V = a.src.vocab;
  const int tb = a.src.token_dtype == CKRL_DTYPE_I32 ? 4 : 1;
  // bytes per position: a V-bin logits row, or one finished token row (row N2)
  const int64_t pb = a.sp.logits_dtype == CKRL_DTYPE_TOKEN_ROWS ? (int64_t)sizeof(ckrl_token_row)
                     : (int64_t)V * (a.sp.logits_dtype == CKRL_DTYPE_BF16 ? 2 : 4);
  const int U = a.action_level ? C : 1;
  const int NV = a.value_action ? C : 1;
  AsmPartial mine{{0.0, 0.0, 0.0}, 0.0};
  MomAcc mom;
  for (int64_t i = blockIdx.x; i < a.n; i += gridDim.x) {
    const int64_t r = a.idx[i];
    const int64_t P = (int64_t)C * M;
    if (a.sp.logits)
      copy_bytes((char*)a.dp.logits + i * P * pb, (const char*)a.sp.logits + r * P * pb, P * pb);
    const int t = threadIdx.x;
    for (int k = t; k < P; k += blockDim.x) {
      if (a.src.tokens) {
        if (tb == 4)
          ((int32_t*)a.dst.tokens)[i * P + k] = ((const int32_t*)a.src.tokens)[r * P + k];
        else
          ((uint8_t*)a.dst.tokens)[i * P + k] = ((const uint8_t*)a.src.tokens)[r * P + k];
      }
      if (a.src.old_logprob) ((float*)a.dst.old_logprob)[i * P + k] = a.src.old_logprob[r * P + k];
    }
    for (int j = t; j < C; j += blockDim.x) {
      ((float*)a.dst.reward)[i * C + j] = a.src.reward[r * C + j];
      ((uint8_t*)a.dst.flags)[i * C + j] = a.src.flags[r * C + j];
      ((int32_t*)a.dst.episode_id)[i * C + j] = a.src.episode_id[r * C + j];
      if (a.src.value_vector) ((float*)a.dst.value_vector)[i * C + j] = a.src.value_vector[r * C + j];
      if (a.src.bootstrap) ((float*)a.dst.bootstrap)[i * C + j] = a.src.bootstrap[r * C + j];
      a.db.counted[i * C + j] = a.sb.counted[r * C + j];
    }
    for (int u = t; u < U; u += blockDim.x) {
      a.db.advantages[i * U + u] = a.sb.advantages[r * U + u];
      a.db.returns[i * U + u] = a.sb.returns[r * U + u];
    }
    if (a.sp.values)
      for (int u = t; u < NV; u += blockDim.x) ((float*)a.dp.values)[i * NV + u] = a.sp.values[r * NV + u];
    if (t == 0) {
      if (a.src.value_scalar) ((float*)a.dst.value_scalar)[i] = a.src.value_scalar[r];
      int cnt = 0;
      for (int j = 0; j < C; ++j) cnt += a.sb.counted[r * C + j] ? 1 : 0;
      mine.n_pos += cnt;
      if (a.action_level) {
        for (int j = 0; j < C; ++j)
          if (a.sb.counted[r * C + j]) mom.add(a.sb.advantages[r * C + j]);
      } else if (cnt) {
        mom.add(a.sb.advantages[r]);
      }
    }
    __syncthreads();
  }
  // thread 0 holds the CTA's partial; finish_asm_stats reads it from thread 0
  mine.m = mom.get();
  finish_asm_stats(mine, a.ws, a.L, M, ExchangeView{});
}

cudaError_t launch_select_records(const ckrl_rollout& src, const ckrl_ppo_batch& sb, const ckrl_policy_outputs& sp,
                                  int action_level, int value_action, int64_t n, const int64_t* idx,
                                  const ckrl_rollout& dst, const ckrl_ppo_batch& db,
                                  const ckrl_policy_outputs& dp, char* ws, cudaStream_t s) {
  SelectArgs a;
  a.src = src;
  a.dst = dst;
  a.sb = sb;
  a.db = db;
  a.sp = sp;
  a.dp = dp;
  a.action_level = action_level;
  a.value_action = value_action;
  a.n = n;
  a.idx = idx;
  a.ws = ws;
  a.L = ws_layout((int)n, 1);
  cudaMemsetAsync(ws + a.L.tickets, 0, sizeof(uint32_t), s);
  const int grid = (int)(n < 1 ? 1 : (n < kMaxLossCtas ? n : kMaxLossCtas));
  select_records_kernel<<<grid, 128, 0, s>>>(a);
  return cudaGetLastError();
}

// group_indices of optim::grpo_loss (losses.hpp:63-65): envs of unselected groups leave the
// batch (env_group = -1) and the normaliser 1/#groups counts the selected ones
// (losses.cpp:240-245).
__global__ void select_groups_kernel(int E, const int32_t* src_group, int32_t* dst_group, int n,
                                     const int32_t* sel, char* ws, WsLayout L) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int g = src_group[e];
    int out = -1;
    for (int q = 0; q < n && g >= 0; ++q)
      if (sel[q] == g) out = g;
    dst_group[e] = out;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    reinterpret_cast<StatsRecord*>(ws + L.stats_local)->groups_retained = n;
}

cudaError_t launch_select_groups(int E, const int32_t* src_group, int32_t* dst_group, int n, const int32_t* sel,
                                 char* ws, cudaStream_t s) {
  select_groups_kernel<<<(E + 255) / 256 < 1 ? 1 : (E + 255) / 256, 256, 0, s>>>(E, src_group, dst_group, n, sel,
                                                                                  ws, ws_layout(E, 1));
  return cudaGetLastError();
}

}  // namespace ckrl
