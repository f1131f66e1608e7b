// (b)+(d) the fused action-token kernel on sm_100a: one pass over the current-policy
// logits computes, per token row, the V-bin log-softmax, the sampled-token gather and
// the entropy (PolicyNet::evaluate_chunk, policy/policy_net.cpp:333-357), and — in the
// same CTA, while the tile's per-token results sit in shared memory — the PPO or GRPO
// unit terms (optim/losses.cpp:62-331): importance ratio at token/action/chunk
// granularity, clipped surrogate, clip/kl counters, value and entropy terms and every
// per-position gradient coefficient. Sums are fp64 per thread, reduced in a fixed order
// (per CTA, then a last-CTA pass over the partials), so results are run-to-run identical.
//
// Row mapping (V == 256 fast path): 8 lanes per row, 4 rows per warp instruction,
// 128-bit loads (f32: 8 x float4 per lane; bf16: 4 x uint4 per lane) so every load
// instruction moves 4 full 128-byte lines; the row stays in registers, reductions are
// 3 xor-shuffles. exp is ex2.approx on a log2-scaled argument whose shift c is carried
// into the log-prob exactly (lp = x_tok - c*ln2 - log s, s = sum 2^(x*log2e - c)).
#include "common.cuh"
#include "gae.cuh"
#include "kernels.h"

#include <cstdlib>

namespace ckrl {

// On-device probes (%globaltimer, ns), compiled in only with -DCKRL_PROBES
// (`make EXTRA=-DCKRL_PROBES`, for profiles/tools/tl_probe.py and tail_probe.py): the timeline
// of CTA 0 and the last CTA (ckrl_debug_timeline) and per-CTA start / roles-done / exit stamps
// of the last TMA loss launch (ckrl_debug_cta_times). Without it both read back zeros.
__device__ uint64_t g_timeline[32];
__device__ uint64_t g_cta_times[3][1184];
// probe build: CTA 0's per-tile trace: [0] row phase start (stage full), [1] row phase done,
// [2] unit phase start (buffer rows full), [3] unit phase done; local tile index < 64
__device__ uint64_t g_tile_times[7][64];  // [4]: unit metadata in shared memory, [5] token pass, [6] slot pass
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#ifdef CKRL_PROBES
#define CKRL_PROBE(stmt) stmt
#else
#define CKRL_PROBE(stmt) \
  do {                   \
  } while (0)
#endif
__device__ __forceinline__ void tl_mark(int slot) { CKRL_PROBE(if (blockIdx.x == 0) g_timeline[slot] = gtimer()); }

constexpr float kL2E = 1.4426950408889634f;
constexpr double kLN2 = 0.6931471805599453;
constexpr double kInvLN2 = 1.4426950408889634;
// relative error of the fp32 log2(e) the row sums are taken with, and its reciprocal
constexpr double kL2EDelta = (double)kL2E / 1.4426950408889634 - 1.0;
constexpr double kInvL2EF = 1.0 / (double)kL2E;

__device__ __forceinline__ float ex2(float y) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(y));
  return r;
}

__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ldg_stream_u4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <typename LT>
__device__ __forceinline__ float load_elem(const LT* p, int64_t i);
template <>
__device__ __forceinline__ float load_elem<float>(const float* p, int64_t i) {
  return __ldg(p + i);
}
template <>
__device__ __forceinline__ float load_elem<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}

// Per-row partial results kept in shared memory between the row and unit phases.
struct RowSmem {
  float* s;    // sum 2^(y)
  float* t2;   // sum 2^(y) * y
  float* c;    // log2-domain shift
  float* xt;   // logit of the sampled token
  float* old;  // old log-prob
  double* lp;  // new log-prob (unit phase)
  float* ent;  // entropy (unit phase)
};

__device__ __forceinline__ float grp8_max(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
  return v;
}
__device__ __forceinline__ float grp8_sum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  return v;
}

// Row phase for V == 256: every lane of the warp participates (shuffles are warp-wide);
// `need` gates the loads of this lane's row group.
template <typename LT>
__device__ __forceinline__ void row_fast(const LT* row, bool need, int l8, float& s_out,
                                         float& t_out, float& c_out) {
  float x[32];
  if constexpr (sizeof(LT) == 4) {
    const float4* p = reinterpret_cast<const float4*>(row);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 v = need ? ldg_stream(p + l8 + 8 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
      x[4 * i + 0] = v.x;
      x[4 * i + 1] = v.y;
      x[4 * i + 2] = v.z;
      x[4 * i + 3] = v.w;
    }
  } else {
    const uint4* p = reinterpret_cast<const uint4*>(row);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint4 v = need ? ldg_stream_u4(p + l8 + 8 * i) : make_uint4(0u, 0u, 0u, 0u);
      x[8 * i + 0] = bf16_lo(v.x);
      x[8 * i + 1] = bf16_hi(v.x);
      x[8 * i + 2] = bf16_lo(v.y);
      x[8 * i + 3] = bf16_hi(v.y);
      x[8 * i + 4] = bf16_lo(v.z);
      x[8 * i + 5] = bf16_hi(v.z);
      x[8 * i + 6] = bf16_lo(v.w);
      x[8 * i + 7] = bf16_hi(v.w);
    }
  }
  float m = x[0];
#pragma unroll
  for (int i = 1; i < 32; ++i) m = fmaxf(m, x[i]);
  m = grp8_max(m);
  const float c = m * kL2E;
  float s0 = 0.f, s1 = 0.f, t0 = 0.f, t1 = 0.f;
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    float y0 = fmaf(x[i], kL2E, -c), y1 = fmaf(x[i + 1], kL2E, -c);
    float e0 = ex2(y0), e1 = ex2(y1);
    s0 += e0;
    s1 += e1;
    t0 = fmaf(e0, y0, t0);
    t1 = fmaf(e1, y1, t1);
  }
  s_out = grp8_sum(s0 + s1);
  t_out = grp8_sum(t0 + t1);
  c_out = c;
}

// Generic V: three strided passes over the row (max, then sums); L1/L2 absorb re-reads.
template <typename LT>
__device__ __forceinline__ void row_generic(const LT* row, bool need, int V, int l8, float& s_out,
                                            float& t_out, float& c_out) {
  float m = -INFINITY;
  if (need)
    for (int v = l8; v < V; v += 8) m = fmaxf(m, load_elem(row, v));
  m = grp8_max(m);
  const float c = need ? m * kL2E : 0.f;
  float s = 0.f, t = 0.f;
  if (need)
    for (int v = l8; v < V; v += 8) {
      float y = fmaf(load_elem(row, v), kL2E, -c);
      float e = ex2(y);
      s += e;
      t = fmaf(e, y, t);
    }
  s_out = grp8_sum(s);
  t_out = grp8_sum(t);
  c_out = c;
}

__device__ __forceinline__ int load_token(const void* tokens, int tok_i32, int64_t k) {
  return tok_i32 ? __ldg(reinterpret_cast<const int32_t*>(tokens) + k)
                 : (int)__ldg(reinterpret_cast<const uint8_t*>(tokens) + k);
}

struct Surrogate {
  double value, dlogprob;
  bool clipped;
};

// optim/losses.cpp:32-46: ties pick the unclipped branch; clip flag is |rho-1| > eps.
__device__ __forceinline__ Surrogate clipped_surrogate(double rho, double adv, double eps) {
  double unclipped = rho * adv;
  double lo = 1.0 - eps, hi = 1.0 + eps;
  double crho = rho < lo ? lo : (hi < rho ? hi : rho);
  double clipped = crho * adv;
  Surrogate s;
  s.clipped = fabs(rho - 1.0) > eps;
  if (unclipped <= clipped) {
    s.value = unclipped;
    s.dlogprob = adv * rho;
  } else {
    s.value = clipped;
    s.dlogprob = 0.0;
  }
  return s;
}

struct Acc {
  double surr, valsq, ent, kl, clipped, units;
};

// Merge the per-rank stats records (fixed rank order) into the loss constants.
struct LossConsts {
  double inv_adv, inv_val, inv_pos, mean, denom, inv_denom, inv_groups;
  int do_norm;
  int64_t n_adv, groups;
  int status;
  unsigned long long epoch;  // exchange epoch of this step (multi-rank)
};

__device__ __forceinline__ double drecip(double x) { return __drcp_rn(x); }  // == 1.0 / x (IEEE rn)

// Loss constants from the merged moments / normalisers.
__device__ LossConsts consts_from(const Moments& mom, int64_t n_adv, int64_t n_val, int64_t n_pos,
                                  int64_t groups, int status, int normalize) {
  LossConsts k;
  k.n_adv = n_adv;
  k.groups = groups;
  k.inv_adv = n_adv > 0 ? drecip((double)n_adv) : 0.0;
  k.inv_val = n_val > 0 ? drecip((double)n_val) : 0.0;
  k.inv_pos = n_pos > 0 ? drecip((double)n_pos) : 0.0;
  k.do_norm = normalize && mom.n >= 2.0;
  whitening(mom, &k.mean, &k.denom);
  k.inv_denom = drecip(k.denom);
  k.inv_groups = groups > 0 ? drecip((double)groups) : 0.0;
  k.status = status;
  k.epoch = 0;
  return k;
}

// Merge the per-rank stats records (fixed rank order) into the loss constants. Advantages
// already whitened in place (ckrl_normalize_advantages) are used as they are.
// Multi-rank (a.ex.world > 1): the records are this step's exchange slots in the rank's own
// buffer, waited for first (every rank's assembly stored its record there over NVLink).
__device__ LossConsts merge_consts(const LossArgs& a) {
  int64_t n_val = 0, n_pos = 0, groups = 0, n_adv = 0;
  int status = 0, whitened = 0;
  const StatsRecord* recs = a.recs;
  int world = a.world;
  size_t stride = sizeof(StatsRecord);
  unsigned long long e = 0;
  if (a.ex.world > 1) {
    // this batch's epoch, as its assembly noted it in the workspace (the exchange header may
    // already hold a later batch's)
    e = (unsigned long long)reinterpret_cast<const uint32_t*>(a.ws + a.L.tickets)[TICKET_EPOCH];
    ExSlot* sl = ex_slots(a.ex.local, a.ex.world, e);
    for (int q = 0; q < a.ex.world; ++q)
      if (!ex_wait(&sl[q].stats_epoch, e)) status = CKRL_ERR_NCCL;  // a peer never posted
    recs = &sl[0].rec;
    world = a.ex.world;
    stride = sizeof(ExSlot);
  }
  for (int r = 0; r < world; ++r) {
    const StatsRecord& s = rec_at(recs, stride, r);
    n_adv += s.n_adv;
    n_val += s.n_val;
    n_pos += s.n_pos;
    groups += s.groups_retained;
    whitened |= (int)(s.flags & STATS_WHITENED);
    if (s.status && !status) status = (int)s.status;
  }
  LossConsts k = consts_from(merge_records(recs, world, stride), n_adv, n_val, n_pos, groups, status,
                             a.normalize && !whitened);
  k.epoch = e;
  return k;
}

// One advantage unit: ratio, clipped surrogate (losses.cpp:32-46) and the approx-kl term
// (losses.cpp:130).
struct UnitOut {
  double value, dlogprob, kl;
  int clipped;
};
// For |d| < 0.5 (almost every unit: d is the new-minus-old log-ratio) rho - 1 and the kl term
// come from one Horner polynomial, exp(d) - 1 - d = d^2 * sum_{k>=2} d^(k-2)/k! (truncated
// at k = 17, error < 1e-20): cheaper than libdevice exp and free of the cancellation in
// (rho - 1) - d. Otherwise exp().
__device__ __forceinline__ UnitOut surrogate_unit(double d, double adv, double eps) {
  double rho, kl;
  if (fabs(d) < 0.5) {
    // sum_{k=0..15} d^k / (k+2)! by Estrin's scheme (dependency depth 4 instead of 16)
    const double d2 = d * d, d4 = d2 * d2, d8 = d4 * d4;
    const double q0 = fma(1.0 / 6.0, d, 0.5), q1 = fma(1.0 / 120.0, d, 1.0 / 24.0);
    const double q2 = fma(1.0 / 5040.0, d, 1.0 / 720.0), q3 = fma(1.0 / 362880.0, d, 1.0 / 40320.0);
    const double q4 = fma(1.0 / 39916800.0, d, 1.0 / 3628800.0);
    const double q5 = fma(1.0 / 6227020800.0, d, 1.0 / 479001600.0);
    const double q6 = fma(1.0 / 1307674368000.0, d, 1.0 / 87178291200.0);
    const double q7 = fma(1.0 / 355687428096000.0, d, 1.0 / 20922789888000.0);
    const double r0 = fma(q1, d2, q0), r1 = fma(q3, d2, q2), r2 = fma(q5, d2, q4), r3 = fma(q7, d2, q6);
    const double p = fma(fma(r3, d4, r2), d8, fma(r1, d4, r0));
    kl = d * d * p;          // exp(d) - 1 - d
    rho = 1.0 + (d + kl);
  } else {
    rho = exp(d);
    kl = (rho - 1.0) - d;
  }
  const Surrogate s = clipped_surrogate(rho, adv, eps);
  return UnitOut{s.value, s.dlogprob, kl, s.clipped ? 1 : 0};
}

__device__ void finalize_diag(const LossArgs& a, const LossConsts& k, const double* raw,
                              double* diag) {
  for (int i = 0; i < CKRL_DIAG_COUNT; ++i) diag[i] = 0.0;
  double status = k.status;
  if (a.mode == MODE_PPO) {
    if (k.n_adv > 0) {
      double surr = -raw[RAW_SURR] * k.inv_adv;
      double vl = raw[RAW_VALSQ] * k.inv_val;
      double ent = raw[RAW_ENT] * k.inv_pos;
      diag[CKRL_DIAG_LOSS] = surr + a.vcoef * vl - a.ecoef * ent;
      diag[CKRL_DIAG_SURROGATE] = surr;
      diag[CKRL_DIAG_VALUE_LOSS] = vl;
      diag[CKRL_DIAG_ENTROPY] = ent;
    }
  } else if (a.mode == MODE_GRPO) {
    if (k.groups == 0 && status == 0) status = CKRL_ERR_SKIP_UPDATE;
    diag[CKRL_DIAG_SURROGATE] = -raw[RAW_SURR];
    diag[CKRL_DIAG_LOSS] = -raw[RAW_SURR];
  }
  double units = raw[RAW_LPUNITS];
  diag[CKRL_DIAG_CLIP_FRAC] = units > 0 ? raw[RAW_CLIPPED] / units : 0.0;
  diag[CKRL_DIAG_APPROX_KL] = units > 0 ? raw[RAW_KL] / units : 0.0;
  diag[CKRL_DIAG_UNITS] = units;
  if (status == 0 && !isfinite(diag[CKRL_DIAG_LOSS])) status = CKRL_ERR_NON_FINITE;
  diag[CKRL_DIAG_STATUS] = status;
}

// ---------------------------------------------------------------------------------
// Unit phase: everything after the tile's per-row partials (s, t2, c, x_tok) sit in
// shared memory. Token pass (one thread per token row): lp, entropy, token outputs, PPO
// entropy term and token-level units. Slot pass (one thread per slot): action-level
// units and values. Record pass (one warp per record): chunk-level units as a warp
// reduction over the record's tokens. fp64 throughout.
// ---------------------------------------------------------------------------------
// Entropy at action and chunk granularity (north star (b)): per slot the canonical-order sum
// (ascending j) of its token entropies, per record the sum (ascending i) of its slots' sums —
// the order aggregate_logprob uses for log-probs (core/granularity.cpp:83-113) — over the
// slots `on(sl)` selects (counted slots for PPO, weighted trajectory slots for GRPO, the
// caller's valid mask for token stats); other slots contribute 0. Rows' entropies are in
// shared memory (`ent`, tile-local rows); `tid`/`nthr` stride the slots / records.
template <class On>
__device__ __forceinline__ void entropy_aggregates(const LossArgs& a, const float* ent, int64_t r0, int nrec,
                                                   int tid, int nthr, On on) {
  const int C = a.C, M = a.M;
  if (a.action_ent)
    for (int sl = tid; sl < nrec * C; sl += nthr) {
      double e = 0.0;
      if (on(sl))
        for (int j = 0; j < M; ++j) e += (double)ent[sl * M + j];
      a.action_ent[r0 * C + sl] = e;
    }
  if (a.chunk_ent)
    for (int r = tid; r < nrec; r += nthr) {
      double c = 0.0;
      for (int i = 0; i < C; ++i) {
        const int sl = r * C + i;
        if (!on(sl)) continue;
        double e = 0.0;
        for (int j = 0; j < M; ++j) e += (double)ent[sl * M + j];
        c += e;
      }
      a.chunk_ent[r0 + r] = c;
    }
}

template <int MODE>
__device__ __forceinline__ void unit_phase(const LossArgs& a, const LossConsts& k, Acc& acc,
                                           const RowSmem& sm, int64_t r0, int nrec, int tid,
                                           int nthr) {
  const int C = a.C, M = a.M, P = C * M;
  const int rows = nrec * P;
  const int64_t k0 = r0 * P;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nthr >> 5;
  const bool chunk_adv = a.adv_level == CKRL_LEVEL_CHUNK;

  // ---- token pass ----
  for (int row = tid; row < rows; row += nthr) {
    const int64_t kk = k0 + row;
    const int64_t slot = kk / M;
    const int64_t rec = kk / P;
    double lp;
    float ent;
    if (a.rows_in) {  // finished on the tensor cores (ckrl_project_token_stats, row N2)
      const ckrl_token_row tr = a.rows_in[kk];
      lp = tr.logprob;
      ent = tr.entropy;
    } else {
      const double s = (double)sm.s[row];
      const double ls = log(s);
      lp = ((double)sm.xt[row] - (double)sm.c[row] * kLN2) - ls;
      ent = (float)(ls - kLN2 * (double)sm.t2[row] / s);
    }
    const float old = MODE == MODE_STATS ? 0.0f : __ldg(a.old_lp + kk);
    sm.lp[row] = lp;
    sm.old[row] = old;
    sm.ent[row] = ent;
    if (a.tok_lp) a.tok_lp[kk] = (float)lp;
    if (a.tok_ent) a.tok_ent[kk] = ent;
    if (MODE == MODE_PPO) {
      const bool cnt = a.counted[slot] != 0;
      if (cnt) acc.ent += ent;
      if (a.coeff_ent) a.coeff_ent[kk] = (cnt && a.ecoef != 0.0) ? (float)(-a.ecoef * k.inv_pos) : 0.0f;
      if (a.lp_level == CKRL_LEVEL_TOKEN) {
        float coeff = 0.0f;
        if (cnt) {
          double adv = chunk_adv ? (double)a.adv[rec] : (double)a.adv[slot];
          if (k.do_norm) adv = (adv - k.mean) * k.inv_denom;
          const double d = lp - (double)old;
          const UnitOut su = surrogate_unit(d, adv, a.clip);
          acc.surr += su.value;
          acc.units += 1.0;
          acc.clipped += su.clipped;
          acc.kl += su.kl;
          coeff = (float)(-k.inv_adv * su.dlogprob);
        }
        if (a.coeff_lp) a.coeff_lp[kk] = coeff;
      }
    } else if (MODE == MODE_GRPO && a.lp_level == CKRL_LEVEL_TOKEN) {
      const int e = (int)(rec / a.Tc);
      const double w = a.slot_weight[slot];
      float coeff = 0.0f;
      if (a.env_group[e] >= 0 && a.slot_member[slot] && w != 0.0f) {
        const double inv_g = drecip((double)a.env_group_size[e]);
        const double d = lp - (double)old;
        const UnitOut su = surrogate_unit(d, a.env_adv[e], a.clip);
        acc.surr += k.inv_groups * inv_g * (double)w * su.value;
        acc.units += 1.0;
        acc.clipped += su.clipped;
        acc.kl += su.kl;
        coeff = (float)(-k.inv_groups * inv_g * (double)w * su.dlogprob);
      }
      if (a.coeff_lp) a.coeff_lp[kk] = coeff;
    }
  }
  __syncwarp();
  // the slot / record passes read other threads' token results
  if (nthr == kLossThreads)
    asm volatile("bar.sync 1, %0;" ::"n"(kLossThreads));
  else if (nthr != 32)
    __syncthreads();

  // ---- entropy aggregates (optional outputs) ----
  if (a.action_ent || a.chunk_ent)
    entropy_aggregates(a, sm.ent, r0, nrec, tid, nthr, [&](int sl) {
      const int64_t slot = r0 * C + sl;
      if (MODE == MODE_STATS) return !a.stats_mask || a.stats_mask[slot] != 0;
      if (MODE == MODE_PPO) return a.counted[slot] != 0;
      const int e = (int)((slot / C) / a.Tc);
      return a.env_group[e] >= 0 && a.slot_member[slot] && a.slot_weight[slot] != 0.0;
    });

  // ---- slot pass ----
  if (MODE == MODE_STATS) {
    if (a.action_lp)
      for (int sl = tid; sl < nrec * C; sl += nthr) {
        double s = 0.0;
        for (int j = 0; j < M; ++j) s += sm.lp[sl * M + j];
        a.action_lp[r0 * C + sl] = s;
      }
  } else {
    const bool act_lp = a.lp_level == CKRL_LEVEL_ACTION;
    const bool act_val = MODE == MODE_PPO && a.val_level == CKRL_LEVEL_ACTION;
    if (act_lp || act_val)
      for (int sl = tid; sl < nrec * C; sl += nthr) {
        const int64_t slot = r0 * C + sl;
        const int64_t rec = r0 + sl / C;
        if (act_lp) {
          bool on;
          double adv, scale = 1.0;
          int e = 0;
          if (MODE == MODE_PPO) {
            on = a.counted[slot] != 0;
            adv = chunk_adv ? (double)a.adv[rec] : (double)a.adv[slot];
            if (k.do_norm) adv = (adv - k.mean) * k.inv_denom;
          } else {
            e = (int)(rec / a.Tc);
            const double w = a.slot_weight[slot];
            on = a.env_group[e] >= 0 && a.slot_member[slot] && w != 0.0f;
            adv = on ? a.env_adv[e] : 0.0;
            scale = on ? k.inv_groups * (drecip((double)a.env_group_size[e])) * (double)w : 0.0;
          }
          float coeff = 0.0f;
          if (on) {
            double an = 0.0, ao = 0.0;
            for (int j = 0; j < M; ++j) {
              an += sm.lp[sl * M + j];
              ao += (double)sm.old[sl * M + j];
            }
            const UnitOut su = surrogate_unit(an - ao, adv, a.clip);
            acc.units += 1.0;
            acc.clipped += su.clipped;
            acc.kl += su.kl;
            if (MODE == MODE_PPO) {
              acc.surr += su.value;
              coeff = (float)(-k.inv_adv * su.dlogprob);
            } else {
              acc.surr += scale * su.value;
              coeff = (float)(-scale * su.dlogprob);
            }
          }
          if (a.coeff_lp)
            for (int j = 0; j < M; ++j) a.coeff_lp[slot * M + j] = coeff;
        }
        if (act_val) {  // value loss per counted slot (losses.cpp:272-285)
          float cv = 0.0f;
          if (a.counted[slot] && a.new_values) {
            const double err = (double)a.new_values[slot] - (double)a.ret[slot];
            acc.valsq += err * err;
            cv = (float)(a.vcoef * 2.0 * err * k.inv_val);
          }
          if (a.coeff_val) a.coeff_val[slot] = cv;
        }
      }
  }

  // ---- record pass (one warp per record) ----
  const bool chunk_lp = MODE != MODE_STATS && a.lp_level == CKRL_LEVEL_CHUNK;
  const bool chunk_val = MODE == MODE_PPO && a.val_level == CKRL_LEVEL_CHUNK;
  if (MODE == MODE_STATS && a.chunk_lp) {
    for (int r = warp; r < nrec; r += nwarps) {
      double s = 0.0;
      for (int t = lane; t < P; t += 32) s += sm.lp[r * P + t];
      s = warp_sum(s);
      if (lane == 0) a.chunk_lp[r0 + r] = s;
    }
  }
  if (chunk_lp || chunk_val) {
    for (int r = warp; r < nrec; r += nwarps) {
      const int64_t rec = r0 + r;
      const int e = (int)(rec / a.Tc);
      // per-slot inclusion (counted for PPO; member && w != 0 for GRPO)
      bool has_env = MODE == MODE_PPO || a.env_group[e] >= 0;
      double lpn = 0.0, lpo = 0.0, wsum = 0.0;
      int any = 0;
      for (int t = lane; t < P && has_env; t += 32) {
        const int64_t slot = rec * C + t / M;
        bool on;
        if (MODE == MODE_PPO) {
          on = a.counted[slot] != 0;
        } else {
          on = a.slot_member[slot] && a.slot_weight[slot] != 0.0;
          if (on && (t % M) == 0) wsum += (double)a.slot_weight[slot];
        }
        if (on) {
          lpn += sm.lp[r * P + t];
          lpo += (double)sm.old[r * P + t];
          any = 1;
        }
      }
      lpn = warp_sum(lpn);
      lpo = warp_sum(lpo);
      wsum = warp_sum(wsum);
      any = __any_sync(0xffffffffu, any);
      if (chunk_lp) {
        float coeff = 0.0f;
        if (any) {
          double adv, scale = 1.0;
          if (MODE == MODE_PPO) {
            adv = (double)a.adv[rec];
            if (k.do_norm) adv = (adv - k.mean) * k.inv_denom;
          } else {
            adv = a.env_adv[e];
            scale = k.inv_groups * (drecip((double)a.env_group_size[e])) * wsum;
          }
          const UnitOut su = surrogate_unit(lpn - lpo, adv, a.clip);
          if (lane == 0) {
            acc.units += 1.0;
            acc.clipped += su.clipped;
            acc.kl += su.kl;
            acc.surr += MODE == MODE_PPO ? su.value : scale * su.value;
          }
          coeff = (float)(MODE == MODE_PPO ? -k.inv_adv * su.dlogprob : -scale * su.dlogprob);
        }
        if (a.coeff_lp)
          for (int t = lane; t < P; t += 32) {
            const int64_t slot = rec * C + t / M;
            bool on;
            if (MODE == MODE_PPO)
              on = a.counted[slot] != 0;
            else
              on = has_env && a.slot_member[slot] && a.slot_weight[slot] != 0.0;
            a.coeff_lp[rec * P + t] = on && any ? coeff : 0.0f;
          }
      }
      if (chunk_val && lane == 0) {  // losses.cpp:264-271
        bool cnt = false;
        for (int i = 0; i < C; ++i) cnt = cnt || a.counted[rec * C + i];
        float cv = 0.0f;
        if (cnt && a.new_values) {
          const double err = (double)a.new_values[rec] - (double)a.ret[rec];
          acc.valsq += err * err;
          cv = (float)(a.vcoef * 2.0 * err * k.inv_val);
        }
        if (a.coeff_val) a.coeff_val[rec] = cv;
      }
    }
  }
}

// Deterministic reduction of the per-thread sums: warp tree -> CTA (warp order) ->
// last CTA over the per-CTA partials (CTA order) -> raw sums [-> finalised diag].
__device__ void reduce_and_finish(const LossArgs& a, const LossConsts& k, const Acc& acc,
                                  int tid, int nthr_total, double (*s_red)[RAW_COUNT], bool* s_last) {
  const int warp = tid >> 5, lane = tid & 31, nwarps = nthr_total >> 5;
  double v[RAW_COUNT] = {acc.surr, acc.valsq, acc.ent, acc.kl, acc.clipped, acc.units, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < RAW_COUNT; ++i) {
    double x = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) s_red[warp][i] = x;
  }
  __syncthreads();
  if (tid == 0) tl_mark(25);
  double* parts = reinterpret_cast<double*>(a.ws + a.L.loss_partials);
  uint32_t* tickets = reinterpret_cast<uint32_t*>(a.ws + a.L.tickets);
  // warp i < RAW_COUNT sums quantity i over the CTA's warps (a shuffle tree, not a serial loop)
  if (warp < RAW_COUNT) {
    double x = lane < nwarps ? s_red[lane][warp] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) parts[warp * kMaxLossCtas + blockIdx.x] = x;  // quantity-major: coalesced reads below
  }
  __syncthreads();
  if (tid == 0) tl_mark(26);
  if (tid == 0) {
    // one acq_rel ticket instead of fence + atomic + fence: the release publishes this CTA's
    // partials (ordered before it by the barrier), the acquire makes every earlier CTA's visible
    uint32_t t;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(&tickets[TICKET_LOSS]) : "memory");
    *s_last = t == gridDim.x - 1;
  }
  __syncthreads();
  if (tid == 0) tl_mark(27);
  if (!*s_last) return;
  CKRL_PROBE(if (tid == 0) g_timeline[28] = gtimer());  // probe: last CTA after its ticket
  // Last CTA: warp i < RAW_COUNT sums quantity i over the CTA partials — each lane a fixed
  // strided subset (its loads in flight together), then a shuffle tree: a fixed order for a
  // given grid, so the sums are deterministic. Plain L2 loads: the acquire above ordered
  // every CTA's released partials before them.
  double* raw = reinterpret_cast<double*>(a.ws + a.L.loss_raw);
  __shared__ double s_tot[RAW_COUNT];
  if (warp < RAW_COUNT) {
    const double* q = parts + warp * kMaxLossCtas;
    double x = 0.0;
    for (unsigned b0 = 0; b0 < gridDim.x; b0 += 32 * 8) {  // 8 loads in flight per lane
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const unsigned b = b0 + lane + 32 * j;
        v[j] = b < gridDim.x ? __ldcg(q + b) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) x += v[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) {
      s_tot[warp] = x;
      raw[warp] = x;
    }
  }
  CKRL_PROBE(if (tid == 0) g_timeline[29] = gtimer());  // probe: partials loaded and warp-reduced
  __syncthreads();
  if (tid == 0) {
    CKRL_PROBE(g_timeline[30] = gtimer());  // probe: raw sums written
    tickets[TICKET_LOSS] = 0;
    if (a.ex.world > 1) {  // cross-rank sum of the raw sums over peer memory (rank order)
      LossConsts kk = k;
      if (!ex_allreduce_raw(a.ex, k.epoch, s_tot) && !kk.status) kk.status = CKRL_ERR_NCCL;
      for (int i = 0; i < RAW_COUNT; ++i) raw[i] = s_tot[i];
      if (a.finalize) finalize_diag(a, kk, s_tot, a.diag);
    } else if (a.finalize) {
      finalize_diag(a, k, s_tot, a.diag);
    }
    CKRL_PROBE(g_timeline[31] = gtimer());  // probe: finalised
  }
}

__device__ __forceinline__ RowSmem carve_rows(unsigned char* base, int rows_cap) {
  RowSmem sm;
  sm.lp = reinterpret_cast<double*>(base);
  sm.s = reinterpret_cast<float*>(sm.lp + rows_cap);
  sm.t2 = sm.s + rows_cap;
  sm.c = sm.t2 + rows_cap;
  sm.xt = sm.c + rows_cap;
  sm.old = sm.xt + rows_cap;
  sm.ent = sm.old + rows_cap;
  return sm;
}
__host__ __device__ constexpr size_t rowsmem_bytes(int rows_cap) {
  return (size_t)rows_cap * (sizeof(double) + 6 * sizeof(float));
}

__device__ __forceinline__ bool row_needed(const LossArgs& a, int mode, int64_t slot) {
  if (a.all_rows) return true;
  if (mode == MODE_PPO) return a.counted[slot] != 0;
  if (mode == MODE_GRPO) return a.slot_member[slot] && a.slot_weight[slot] != 0.0;
  return true;
}

// ---------------------------------------------------------------------------------
// Direct kernel: rows loaded straight from global into registers (used for generic V,
// very long records, and as the reference point for the TMA pipeline).
// ---------------------------------------------------------------------------------
template <int MODE, typename LT, bool FAST>
__global__ void __launch_bounds__(kLossThreads, 2) tile_kernel(LossArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ LossConsts s_k;
  __shared__ double s_red[kLossThreads / 32][RAW_COUNT];
  __shared__ bool s_last;

  const int M = a.M, P = a.C * M, V = a.V;
  const RowSmem sm = carve_rows(smem_raw, a.rec_per_tile * P);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int sub = lane >> 3, l8 = lane & 7;
  if (tid == 0) s_k = merge_consts(a);
  __syncthreads();
  const LossConsts k = s_k;
  Acc acc{0, 0, 0, 0, 0, 0};
  const LT* logits = reinterpret_cast<const LT*>(a.logits);

  for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
    const int64_t r0 = tile * a.rec_per_tile;
    const int64_t rem = a.n_rec - r0;
    const int nrec = (int)(rem < a.rec_per_tile ? rem : a.rec_per_tile);
    const int rows = nrec * P;
    const int64_t k0 = r0 * P;
    for (int rg = warp * 4; rg < rows && !a.rows_in; rg += (kLossThreads / 32) * 4) {
      const int row = rg + sub;
      bool need = row < rows && row_needed(a, MODE, (k0 + row) / M);
      const int64_t kk = k0 + (row < rows ? row : 0);
      const LT* rowp = logits + kk * (int64_t)V;
      int tok = 0;
      float xt = 0.f;
      if (need) {
        tok = load_token(a.tokens, a.tok_i32, kk);
        xt = load_elem(rowp, tok);
      }
      float s, t, c;
      if constexpr (FAST)
        row_fast<LT>(rowp, need, l8, s, t, c);
      else
        row_generic<LT>(rowp, need, V, l8, s, t, c);
      if (l8 == 0 && row < rows) {
        sm.s[row] = need ? s : 1.0f;
        sm.t2[row] = t;
        sm.c[row] = c;
        sm.xt[row] = need ? xt : 0.0f;
      }
    }
    __syncthreads();
    unit_phase<MODE>(a, k, acc, sm, r0, nrec, tid, kLossThreads);
    __syncthreads();
  }
  if (MODE == MODE_STATS) return;
  reduce_and_finish(a, k, acc, tid, kLossThreads, s_red, &s_last);
}

// ---------------------------------------------------------------------------------
// TMA pipeline kernel (V == 256): persistent, one CTA per SM, warp-specialised.
//   warp 0 (one elected lane): producer. Streams each tile — whole records, contiguous
//     in the [E][Tc][C][M][V] layout — into a ring of NSTAGE shared-memory stages with
//     cp.async.bulk (the TMA bulk-copy engine), completion tracked by mbarrier tx-count.
//   warps 1..8: consumers. Row phase from shared memory (LDS.128, conflict-free: each
//     8-lane phase reads one 128-byte run of one row), release the stage, then the unit
//     phase while the producer refills it. Per-row partials are double-buffered so only
//     one consumer barrier per tile is needed.
// ---------------------------------------------------------------------------------
constexpr int kTmaConsumers = kLossThreads;      // 8 consumer warps

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_keep(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <typename LT>
__device__ __forceinline__ void row_fast_smem(const LT* row, int l8, float& s_out, float& t_out,
                                              float& c_out) {
  float x[32];
  if constexpr (sizeof(LT) == 4) {
    const float4* p = reinterpret_cast<const float4*>(row);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 v = p[l8 + 8 * i];
      x[4 * i + 0] = v.x;
      x[4 * i + 1] = v.y;
      x[4 * i + 2] = v.z;
      x[4 * i + 3] = v.w;
    }
  } else {
    const uint4* p = reinterpret_cast<const uint4*>(row);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint4 v = p[l8 + 8 * i];
      x[8 * i + 0] = bf16_lo(v.x);
      x[8 * i + 1] = bf16_hi(v.x);
      x[8 * i + 2] = bf16_lo(v.y);
      x[8 * i + 3] = bf16_hi(v.y);
      x[8 * i + 4] = bf16_lo(v.z);
      x[8 * i + 5] = bf16_hi(v.z);
      x[8 * i + 6] = bf16_lo(v.w);
      x[8 * i + 7] = bf16_hi(v.w);
    }
  }
  // max as a 5-level tree (short dependency chain), then across the 8-lane group
  float mx[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) mx[i] = fmaxf(x[i], x[i + 16]);
#pragma unroll
  for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
    for (int i = 0; i < w; ++i) mx[i] = fmaxf(mx[i], mx[i + w]);
  const float m = grp8_max(mx[0]);
  const float c = m * kL2E;
  float sa[4] = {0.f, 0.f, 0.f, 0.f}, ta[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float y = fmaf(x[i], kL2E, -c);
    const float e = ex2(y);
    sa[i & 3] += e;
    ta[i & 3] = fmaf(e, y, ta[i & 3]);
  }
  s_out = grp8_sum((sa[0] + sa[1]) + (sa[2] + sa[3]));
  t_out = grp8_sum((ta[0] + ta[1]) + (ta[2] + ta[3]));
  c_out = c;
}

// Packed f32x2 arithmetic (FFMA2 / FADD2: two lanes of fp32 per issue slot, same rounding as
// the scalar ops) and three-input max (FMNMX3); bf16 rows take their max on the packed words
// (HMNMX2: max is exact, so the result equals the fp32 max of the widened values).
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// R independent row groups per warp in flight (ILP across the shuffle / MUFU latencies).
// Per lane and row: 32 logits as 16 (even, odd) pairs; the even / odd elements accumulate
// into the low / high halves of the packed sums (two partial sums, added at the end).
template <typename LT, int R>
__device__ __forceinline__ void rows_fast_smem(const LT* const* rowp, int l8, float* s_out,
                                               float* t_out, float* c_out) {
  // f32: the row as 16 packed (even, odd) pairs; bf16: the 16 raw words (two bf16 each),
  // widened only where the exponent loop consumes them (16 live registers per row, not 32)
  uint64_t x[R][sizeof(LT) == 4 ? 16 : 1];
  uint32_t wr[R][sizeof(LT) == 2 ? 16 : 1];
  float m[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if constexpr (sizeof(LT) == 4) {
      const float4* p = reinterpret_cast<const float4*>(rowp[r]);
      float f[32];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 v = p[l8 + 8 * i];
        f[4 * i + 0] = v.x;
        f[4 * i + 1] = v.y;
        f[4 * i + 2] = v.z;
        f[4 * i + 3] = v.w;
        x[r][2 * i] = f2pack(v.x, v.y);
        x[r][2 * i + 1] = f2pack(v.z, v.w);
      }
      float mx[11];
#pragma unroll
      for (int i = 0; i < 10; ++i) mx[i] = fmax3(f[i], f[i + 10], f[i + 20]);
      mx[10] = fmaxf(f[30], f[31]);
      const float a0 = fmax3(mx[0], mx[1], mx[2]), a1 = fmax3(mx[3], mx[4], mx[5]);
      const float a2 = fmax3(mx[6], mx[7], mx[8]), a3 = fmaxf(mx[9], mx[10]);
      m[r] = fmaxf(fmax3(a0, a1, a2), a3);
    } else {
      const uint4* p = reinterpret_cast<const uint4*>(rowp[r]);
      uint32_t w[16];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 v = p[l8 + 8 * i];
        w[4 * i + 0] = v.x;
        w[4 * i + 1] = v.y;
        w[4 * i + 2] = v.z;
        w[4 * i + 3] = v.w;
      }
      uint32_t mw[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mw[i] = bmax2(w[i], w[i + 8]);
#pragma unroll
      for (int k = 4; k >= 1; k >>= 1)
#pragma unroll
        for (int i = 0; i < k; ++i) mw[i] = bmax2(mw[i], mw[i + k]);
      m[r] = fmaxf(bf16_lo(mw[0]), bf16_hi(mw[0]));
#pragma unroll
      for (int i = 0; i < 16; ++i) wr[r][i] = w[i];
    }
  }
#pragma unroll
  for (int o = 1; o <= 4; o <<= 1)
#pragma unroll
    for (int r = 0; r < R; ++r) m[r] = fmaxf(m[r], __shfl_xor_sync(0xffffffffu, m[r], o));
  const uint64_t l2e = f2pack(kL2E, kL2E);
  uint64_t sa[R], ta[R], nc[R];
  float c[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    c[r] = m[r] * kL2E;
    nc[r] = f2pack(-c[r], -c[r]);
    sa[r] = ta[r] = 0ull;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      uint64_t xi;
      if constexpr (sizeof(LT) == 4)
        xi = x[r][i];
      else
        xi = f2pack(bf16_lo(wr[r][i]), bf16_hi(wr[r][i]));
      const uint64_t y = ffma2(xi, l2e, nc[r]);
      float y0, y1;
      f2unpack(y, y0, y1);
      const uint64_t e = f2pack(ex2(y0), ex2(y1));
      sa[r] = fadd2(sa[r], e);
      ta[r] = ffma2(e, y, ta[r]);
    }
  float sv[R], tv[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float a0, a1;
    f2unpack(sa[r], a0, a1);
    sv[r] = a0 + a1;
    f2unpack(ta[r], a0, a1);
    tv[r] = a0 + a1;
  }
#pragma unroll
  for (int o = 1; o <= 4; o <<= 1)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      sv[r] += __shfl_xor_sync(0xffffffffu, sv[r], o);
      tv[r] += __shfl_xor_sync(0xffffffffu, tv[r], o);
    }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    s_out[r] = sv[r];
    t_out[r] = tv[r];
    c_out[r] = c[r];
  }
}

// log(s) for s >= 1 with ~1e-7 absolute error: exact exponent + f32 log of the mantissa.
__device__ __forceinline__ double log_f32_exact_exp(float s) {
  int e;
  const float mant = frexpf(s, &e);  // s = mant * 2^e, mant in [0.5, 1)
  return (double)e * kLN2 + (double)logf(mant);
}

constexpr int kRowBufs = 4;        // buffer warps; row buffers come in multiples of this
constexpr int kMaxRowBufs = 32;    // row-partial + metadata buffers (row warps <-> unit warps)
constexpr int kTileRowsMax = 128;  // rows (tokens) per tile

// Per-tile small inputs staged in shared memory by the metadata warp, so consumer warps
// never wait on global memory: token ids, old log-probs, per-slot activity (counted, or
// trajectory member with non-zero weight) and weight, per-unit advantage / return / new
// value, and (GRPO) the per-record env's group data.
struct MetaSmem {
  float* old;
  double* w;
  double* adv;
  double* ret;
  float* nv;
  int32_t* esz;
  double* eadv;
  uint8_t* act;   // per slot: bit1 unit active (counted / trajectory slot with weight)
};
// One row buffer of the TMA kernel: per-row results + the tile's metadata. Row arrays are
// sized by `cap` (rows per tile), slot / unit / record arrays by `scap` (slots per tile; a
// record has C slots, a unit is a record or a slot), both multiples of 8; fp64 arrays first.
//   per row:  lp (f64), ent, s / t2 / c (the fused seam's row statistics), old (f32)
//   per slot: eadv, adv, ret, w (f64), nv, esz (4 B), act (1 B)
__host__ __device__ constexpr size_t rowbuf_bytes(int cap, int scap) {
  return (size_t)cap * (8 + 5 * 4) + (size_t)scap * (4 * 8 + 4 + 4 + 1);
}
__device__ __forceinline__ void carve_buf(unsigned char* p, int cap, int scap, RowSmem& sm, MetaSmem& m) {
  sm.lp = reinterpret_cast<double*>(p);
  m.eadv = sm.lp + cap;
  m.adv = m.eadv + scap;
  m.ret = m.adv + scap;
  m.w = m.ret + scap;
  sm.ent = reinterpret_cast<float*>(m.w + scap);
  sm.s = sm.ent + cap;
  sm.t2 = sm.s + cap;
  sm.c = sm.t2 + cap;
  sm.xt = nullptr;  // (direct kernel only)
  sm.old = nullptr;
  m.old = sm.c + cap;
  m.nv = m.old + cap;
  m.esz = reinterpret_cast<int32_t*>(m.nv + scap);
  m.act = reinterpret_cast<uint8_t*>(m.esz + scap);
}

// PPO tiles whose advantage, return and new-value units (value level == advantage level for
// GAE assembly) fit one warp three times over.
__device__ __forceinline__ bool small_units(const LossArgs& a, int nrec) {
  const int U = a.val_level == CKRL_LEVEL_CHUNK ? nrec : nrec * a.C;
  return a.adv_level == a.val_level && 3 * U <= 32;
}

// Register images of a tile's metadata hold the RAW loaded values: nothing derived from a
// load is computed before the matching *_store, so a *_load only issues loads and their
// latency hides behind whatever runs in between (the current tile's unit phase).
struct UnitRegs {
  double mix;  // PPO small-unit path: this lane's advantage / return / new value (unit_meta_load)
  float old[4];
  // q == 0 only (the tile's first 32 slots / records: every tile with M >= 4); the rare
  // q >= 1 entries are loaded directly in unit_meta_store
  float nv;
  double adv, ret, w, eadv;
  int32_t esz, g;
  uint8_t act;  // raw: counted (PPO) / slot membership (GRPO)
};

// Loads that may read what other CTAs wrote earlier in the same (fused) launch go
// through L2 (ld.global.cg): the non-coherent L1 must not serve them.
template <int MODE, bool FUSED>
__device__ __forceinline__ void unit_meta_load(const LossArgs& a, int64_t r0, int nrec, int lane,
                                               UnitRegs& R) {
  const int C = a.C, M = a.M, P = C * M;
  const int rows = nrec * P, slots = nrec * C;
  const int64_t k0 = r0 * P, s0 = r0 * C;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = lane + 32 * q;
    if (i < rows) R.old[q] = MODE == MODE_STATS ? 0.0f : __ldg(a.old_lp + k0 + i);
  }
  const int i = lane;
  if (i < slots) {
    if (MODE == MODE_PPO) {
      R.act = __ldcg(a.counted + s0 + i);
    } else if (MODE == MODE_GRPO) {
      R.g = a.env_group[(int)(s0 + i) / C / a.Tc];
      R.act = a.slot_member[s0 + i];
      R.w = a.slot_weight[s0 + i];
    }
  }
  if (MODE == MODE_PPO && small_units(a, nrec)) {
    // one warp-wide load for all three per-unit arrays: lanes [0,U) advantages, [U,2U)
    // returns, [2U,3U) new values (each global load instruction a buffer warp issues waits
    // in the MIO queue behind the row warps' shared loads)
    const int U = a.val_level == CKRL_LEVEL_CHUNK ? nrec : slots;  // == advantage units
    const int64_t ub = a.val_level == CKRL_LEVEL_CHUNK ? r0 : s0;
    const double* pd = lane < U ? a.adv + ub + lane : lane < 2 * U ? a.ret + ub + (lane - U) : nullptr;
    const float* pf = (lane >= 2 * U && lane < 3 * U && a.new_values) ? a.new_values + ub + (lane - 2 * U) : nullptr;
    R.mix = pd ? __ldcg(pd) : (pf ? (double)__ldg(pf) : 0.0);
  } else if (MODE == MODE_PPO) {
    const int adv_units = a.adv_level == CKRL_LEVEL_CHUNK ? nrec : slots;
    const int val_units = a.val_level == CKRL_LEVEL_CHUNK ? nrec : slots;
    if (i < adv_units) R.adv = __ldcg(a.adv + (a.adv_level == CKRL_LEVEL_CHUNK ? r0 : s0) + i);
    if (i < val_units) {
      const int64_t vb = a.val_level == CKRL_LEVEL_CHUNK ? r0 : s0;
      R.ret = __ldcg(a.ret + vb + i);
      R.nv = a.new_values ? __ldg(a.new_values + vb + i) : 0.0f;
    }
  }
  if (MODE == MODE_GRPO && i < nrec) {
    const int e = (int)(r0 + i) / a.Tc;
    R.esz = a.env_group_size[e];
    R.eadv = a.env_adv[e];
  }
}

template <int MODE>
__device__ __forceinline__ void unit_meta_store(const LossArgs& a, int64_t r0, int nrec, int lane,
                                                const UnitRegs& R, const MetaSmem& m) {
  const int C = a.C, P = C * a.M;
  const int rows = nrec * P, slots = nrec * C;
  const int64_t s0 = r0 * C;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = lane + 32 * q;
    if (i < rows) m.old[i] = R.old[q];
    if (i < slots) {
      if (MODE == MODE_PPO) {
        const uint8_t c = q == 0 ? R.act : __ldcg(a.counted + s0 + i);
        m.act[i] = c != 0 ? 2 : 0;
        m.w[i] = 0.0;
      } else if (MODE == MODE_GRPO) {
        int32_t g;
        uint8_t mb;
        double w;
        if (q == 0) {
          g = R.g, mb = R.act, w = R.w;
        } else {
          g = a.env_group[(int)(s0 + i) / C / a.Tc], mb = a.slot_member[s0 + i], w = a.slot_weight[s0 + i];
        }
        m.act[i] = ((g >= 0) & (mb != 0) & (w != 0.0)) ? 2 : 0;
        m.w[i] = w;
      } else {
        m.act[i] = 0;
        m.w[i] = 0.0;
      }
    }
    if (MODE == MODE_PPO && small_units(a, nrec)) {
      if (q == 0) {
        const int U = a.val_level == CKRL_LEVEL_CHUNK ? nrec : slots;
        if (lane < U) m.adv[lane] = R.mix;
        else if (lane < 2 * U) m.ret[lane - U] = R.mix;
        else if (lane < 3 * U) m.nv[lane - 2 * U] = (float)R.mix;
      }
    } else if (MODE == MODE_PPO && i < slots) {  // covers both unit kinds (nrec <= slots)
      const int adv_units = a.adv_level == CKRL_LEVEL_CHUNK ? nrec : slots;
      const int val_units = a.val_level == CKRL_LEVEL_CHUNK ? nrec : slots;
      if (q == 0) {
        m.adv[i] = R.adv;
        m.ret[i] = R.ret;
        m.nv[i] = R.nv;
      } else {  // > 32 units per tile (M < 4 at action level): direct loads
        if (i < adv_units) m.adv[i] = __ldcg(a.adv + (a.adv_level == CKRL_LEVEL_CHUNK ? r0 : s0) + i);
        if (i < val_units) {
          const int64_t vb = a.val_level == CKRL_LEVEL_CHUNK ? r0 : s0;
          m.ret[i] = __ldcg(a.ret + vb + i);
          m.nv[i] = a.new_values ? __ldg(a.new_values + vb + i) : 0.0f;
        }
      }
    }
    if (MODE == MODE_GRPO && i < nrec) {
      if (q == 0) {
        m.esz[i] = R.esz;
        m.eadv[i] = R.eadv;
      } else {
        const int e = (int)(r0 + i) / a.Tc;
        m.esz[i] = a.env_group_size[e];
        m.eadv[i] = a.env_adv[e];
      }
    }
  }
}

// Warp-level unit phase over one tile, all inputs from shared memory (see unit_phase for
// the semantics; identical arithmetic).
// Where the unit phase writes its per-position / per-unit outputs: the caller's global arrays,
// or (bulk path) shared-memory staging rebased so that index k0 + row lands on staging[row].
struct Outs {
  float *tok_lp, *tok_ent, *coeff_lp, *coeff_ent, *coeff_val;
};
__device__ __forceinline__ Outs outs_of(const LossArgs& a) {
  return Outs{a.tok_lp, a.tok_ent, a.coeff_lp, a.coeff_ent, a.coeff_val};
}

template <int MODE>
__device__ __forceinline__ void unit_phase_smem(const LossArgs& a, const LossConsts& k, Acc& acc,
                                                const RowSmem& sm, const MetaSmem& m, int64_t r0,
                                                int nrec, int lane, const Outs& o,
                                                float* gklp = nullptr, float* gkent = nullptr) {
  const int C = a.C, M = a.M, P = C * M;
  const int rows = nrec * P, slots = nrec * C;
  const int64_t k0 = r0 * P;
  const bool chunk_adv = a.adv_level == CKRL_LEVEL_CHUNK;
  // small-integer quotients (rows < 2^10, M, P, C <= 2^13) by float reciprocal: exact
  const float inv_m = 1.0f / (float)M, inv_p = 1.0f / (float)P;
  auto qdiv = [](int x, float inv) { return (int)(((float)x + 0.5f) * inv); };

  for (int row = lane; row < rows; row += 32) {
    const int64_t kk = k0 + row;
    const int sl = qdiv(row, inv_m), r = qdiv(row, inv_p);
    const double lp = sm.lp[row];  // finished by the row warps (fp64 log-prob, entropy)
    const float ent = sm.ent[row];
    const double entd = (double)ent;
    if (o.tok_lp) o.tok_lp[kk] = (float)lp;
    if (o.tok_ent) o.tok_ent[kk] = ent;
    const bool on = (m.act[sl] & 2) != 0;
    if (MODE == MODE_PPO) {
      if (on) acc.ent += entd;
      const float cent = (on && a.ecoef != 0.0) ? (float)(-a.ecoef * k.inv_pos) : 0.0f;
      if (o.coeff_ent) o.coeff_ent[kk] = cent;
      if (gkent) gkent[row] = cent;
    }
    if (MODE == MODE_GRPO && gkent) gkent[row] = 0.0f;
    if (MODE != MODE_STATS && a.lp_level == CKRL_LEVEL_TOKEN) {
      float coeff = 0.0f;
      if (on) {
        double adv, scale;
        if (MODE == MODE_PPO) {
          adv = (double)m.adv[chunk_adv ? r : sl];
          if (k.do_norm) adv = (adv - k.mean) * k.inv_denom;
          scale = k.inv_adv;
        } else {
          adv = m.eadv[r];
          scale = k.inv_groups * drecip((double)m.esz[r]) * (double)m.w[sl];
        }
        const double d = lp - (double)m.old[row];
        const UnitOut su = surrogate_unit(d, adv, a.clip);
        acc.surr += MODE == MODE_PPO ? su.value : scale * su.value;
        acc.units += 1.0;
        acc.clipped += su.clipped;
        acc.kl += su.kl;
        coeff = (float)(-scale * su.dlogprob);
      }
      if (o.coeff_lp) o.coeff_lp[kk] = coeff;
      if (gklp) gklp[row] = coeff;
    }
  }
  __syncwarp();

  CKRL_PROBE(if (blockIdx.x == 0 && lane == 0 && r0 / a.rec_per_tile / gridDim.x < 64) g_tile_times[5][r0 / a.rec_per_tile / gridDim.x] = gtimer());
  if (a.action_ent || a.chunk_ent)
    entropy_aggregates(a, sm.ent, r0, nrec, lane, 32, [&](int sl) {
      if (MODE == MODE_STATS) return !a.stats_mask || a.stats_mask[r0 * C + sl] != 0;
      return (m.act[sl] & 2) != 0;
    });
  if (MODE == MODE_STATS) {
    if (a.action_lp)
      for (int sl = lane; sl < slots; sl += 32) {
        double s = 0.0;
        for (int j = 0; j < M; ++j) s += sm.lp[sl * M + j];
        a.action_lp[r0 * C + sl] = s;
      }
    if (a.chunk_lp)
      for (int r = 0; r < nrec; ++r) {
        double s = 0.0;
        for (int t = lane; t < P; t += 32) s += sm.lp[r * P + t];
        s = warp_sum(s);
        if (lane == 0) a.chunk_lp[r0 + r] = s;
      }
    return;
  }

  const bool act_lp = a.lp_level == CKRL_LEVEL_ACTION;
  const bool act_val = MODE == MODE_PPO && a.val_level == CKRL_LEVEL_ACTION;
  if (act_lp || act_val)
    for (int sl = lane; sl < slots; sl += 32) {
      const int r = sl / C;
      const bool on = (m.act[sl] & 2) != 0;
      if (act_lp) {
        float coeff = 0.0f;
        if (on) {
          double adv, scale;
          if (MODE == MODE_PPO) {
            adv = (double)m.adv[chunk_adv ? r : sl];
            if (k.do_norm) adv = (adv - k.mean) * k.inv_denom;
            scale = k.inv_adv;
          } else {
            adv = m.eadv[r];
            scale = k.inv_groups * drecip((double)m.esz[r]) * (double)m.w[sl];
          }
          // new - old log-ratio of the action: one sum of per-token differences (fp64;
          // equal to sum(new) - sum(old) up to fp64 rounding)
          double dd = 0.0;
          for (int j = 0; j < M; ++j) dd += sm.lp[sl * M + j] - (double)m.old[sl * M + j];
          const UnitOut su = surrogate_unit(dd, adv, a.clip);
          acc.surr += MODE == MODE_PPO ? su.value : scale * su.value;
          acc.units += 1.0;
          acc.clipped += su.clipped;
          acc.kl += su.kl;
          coeff = (float)(-scale * su.dlogprob);
        }
        if (o.coeff_lp)
          for (int j = 0; j < M; ++j) o.coeff_lp[(r0 * C + sl) * M + j] = coeff;
        if (gklp)
          for (int j = 0; j < M; ++j) gklp[sl * M + j] = coeff;
      }
      if (act_val) {
        float cv = 0.0f;
        if (on && a.new_values) {
          const double err = (double)m.nv[sl] - (double)m.ret[sl];
          acc.valsq += err * err;
          cv = (float)(a.vcoef * 2.0 * err * k.inv_val);
        }
        if (o.coeff_val) o.coeff_val[r0 * C + sl] = cv;
      }
    }

  CKRL_PROBE(if (blockIdx.x == 0 && lane == 0 && r0 / a.rec_per_tile / gridDim.x < 64) g_tile_times[6][r0 / a.rec_per_tile / gridDim.x] = gtimer());
  const bool chunk_lp = a.lp_level == CKRL_LEVEL_CHUNK;
  const bool chunk_val = MODE == MODE_PPO && a.val_level == CKRL_LEVEL_CHUNK;
  if (chunk_lp || chunk_val)
    for (int r = 0; r < nrec; ++r) {
      const int64_t rec = r0 + r;
      double dd = 0.0, wsum = 0.0;  // chunk log-ratio as one sum of per-token differences
      int any = 0;
      for (int t = lane; t < P; t += 32) {
        const int sl = r * C + qdiv(t, inv_m);
        if (m.act[sl] & 2) {
          dd += sm.lp[r * P + t] - (double)m.old[r * P + t];
          if (MODE == MODE_GRPO && (t % M) == 0) wsum += (double)m.w[sl];
          any = 1;
        }
      }
      any = __any_sync(0xffffffffu, any);
      if (chunk_lp) {
        dd = warp_sum(dd);
        if (MODE == MODE_GRPO) wsum = warp_sum(wsum);
        float coeff = 0.0f;
        if (any) {
          double adv, scale;
          if (MODE == MODE_PPO) {
            adv = (double)m.adv[r];
            if (k.do_norm) adv = (adv - k.mean) * k.inv_denom;
            scale = k.inv_adv;
          } else {
            adv = m.eadv[r];
            scale = k.inv_groups * drecip((double)m.esz[r]) * wsum;
          }
          const UnitOut su = surrogate_unit(dd, adv, a.clip);
          if (lane == 0) {
            acc.units += 1.0;
            acc.clipped += su.clipped;
            acc.kl += su.kl;
            acc.surr += MODE == MODE_PPO ? su.value : scale * su.value;
          }
          coeff = (float)(-scale * su.dlogprob);
        }
        if (o.coeff_lp)
          for (int t = lane; t < P; t += 32)
            o.coeff_lp[rec * P + t] = (m.act[r * C + qdiv(t, inv_m)] & 2) ? coeff : 0.0f;
        if (gklp)
          for (int t = lane; t < P; t += 32)
            gklp[r * P + t] = (m.act[r * C + qdiv(t, inv_m)] & 2) ? coeff : 0.0f;
      }
      if (chunk_val && lane == 0) {
        float cv = 0.0f;
        if (any && a.new_values) {
          const double err = (double)m.nv[r] - (double)m.ret[r];
          acc.valsq += err * err;
          cv = (float)(a.vcoef * 2.0 * err * k.inv_val);
        }
        if (o.coeff_val) o.coeff_val[rec] = cv;
      }
    }
}


// ---------------------------------------------------------------------------------
// Fused softmax-backward seam (row f1, GRAD kernels): once a tile's unit phase has produced
// its per-position coefficients, the row warps that computed its rows re-read them (from L2:
// the ring lag is kept to 4 tiles and the first read is issued evict_last) and write
//   dlogits_v = klp * ([v == tok] - p_v) - kent * p_v * (ls_v + H)
// (policy_net.cpp:444-456) from the row statistics already in shared memory (shift c,
// log2 of the shifted sum, sum e*y / sum e) — the logits are read from HBM once, not twice.
// ---------------------------------------------------------------------------------
struct GradSmem {  // per row buffer: token id and the two coefficients of each row
  int32_t* tok;
  float* klp;
  float* kent;
};
__device__ __forceinline__ GradSmem carve_grad(unsigned char* base, int cap) {
  GradSmem g;
  g.tok = reinterpret_cast<int32_t*>(base);
  g.klp = reinterpret_cast<float*>(g.tok + cap);
  g.kent = g.klp + cap;
  return g;
}
template <typename LT>
__device__ __forceinline__ void grad_row(const LossArgs& a, const RowSmem& sm, const GradSmem& gs, int row,
                                         int64_t kk, int l8) {
  constexpr int V = 256;
  const float klp = gs.klp[row], kent = gs.kent[row];
  float d[32];
  if (klp == 0.0f && kent == 0.0f) {  // the reference skips the position: zero row
#pragma unroll
    for (int k = 0; k < 32; ++k) d[k] = 0.0f;
  } else {
    float x[32];
    if (sizeof(LT) == 4) {
      const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(a.logits) + kk * V);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 v = ldg_stream(p + l8 + 8 * i);
        x[4 * i] = v.x;
        x[4 * i + 1] = v.y;
        x[4 * i + 2] = v.z;
        x[4 * i + 3] = v.w;
      }
    } else {
      const uint4* p = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.logits) + kk * V);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 v = ldg_stream_u4(p + l8 + 8 * i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          x[8 * i + 2 * j] = __uint_as_float(w[j] << 16);
          x[8 * i + 2 * j + 1] = __uint_as_float(w[j] & 0xffff0000u);
        }
      }
    }
    const float c = sm.c[row], l2s = sm.s[row];
    const float H = 0.6931471805599453f * (l2s - sm.t2[row]);  // entropy (nats)
    const int tok = gs.tok[row];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const float z = fmaf(x[k], kL2E, -c) - l2s;  // log2 p
      const float pv = ex2(z);
      const float ls = z * 0.6931471805599453f;
      const int col = sizeof(LT) == 4 ? 4 * (l8 + 8 * (k >> 2)) + (k & 3) : 8 * (l8 + 8 * (k >> 3)) + (k & 7);
      d[k] = klp * ((col == tok ? 1.0f : 0.0f) - pv) - kent * (pv * (ls + H));
    }
  }
  if (sizeof(LT) == 4) {
    float4* q = reinterpret_cast<float4*>(static_cast<float*>(a.dlogits) + kk * V);
#pragma unroll
    for (int i = 0; i < 8; ++i) __stcs(q + l8 + 8 * i, make_float4(d[4 * i], d[4 * i + 1], d[4 * i + 2], d[4 * i + 3]));
  } else {
    uint4* q = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.dlogits) + kk * V);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __nv_bfloat162 h = __floats2bfloat162_rn(d[8 * i + 2 * j], d[8 * i + 2 * j + 1]);
        w[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      __stcs(q + l8 + 8 * i, make_uint4(w[0], w[1], w[2], w[3]));
    }
  }
}

constexpr int kBufWarps = kRowBufs;  // buffer warp m owns row buffer m (tiles i = m mod 4)
template <int ROWW, int BW = kBufWarps>
constexpr int tma_threads() { return 32 * (1 + ROWW + BW); }  // producer, row, buffer warps

template <int BW = kBufWarps>
__device__ __forceinline__ void bufwarps_sync() {  // named barrier over the buffer warps
  asm volatile("bar.sync 2, %0;" ::"n"(32 * BW) : "memory");
}

// Fused PPO step, phase A (buffer warps only): GAE + counted masks for this CTA's envs,
// CTA partial of the whitening sums, grid-wide barrier, then every CTA sums all
// partials in the same fixed order (identical, deterministic constants everywhere).
__device__ __noinline__ void fused_phase_a(const LossArgs& a, int b, int lane, LossConsts* s_kf) {
  __shared__ AsmPartial bpart[kBufWarps];
  const ckrl_rollout& ro = a.ro;
  const bool action = a.adv_level == CKRL_LEVEL_ACTION;
  AsmPartial acc{{0.0, 0.0, 0.0}, 0.0};
  for (int e = blockIdx.x + b * gridDim.x; e < ro.num_envs; e += kBufWarps * gridDim.x) {
    uint8_t* cnt = const_cast<uint8_t*>(a.counted);
    double* adv = const_cast<double*>(a.adv);
    double* ret = const_cast<double*>(a.ret);
    const GaeSums g = action ? env_gae(ActionAcc{ro, e, cnt, adv, ret}, ro.num_chunks * ro.chunk_len,
                                      a.gamma, a.lambda)
                             : env_gae(ChunkAcc{ro, e, cnt, adv, ret}, ro.num_chunks, a.gamma, a.lambda);
    acc.m = mom_merge(acc.m, g.m);
    acc.n_pos += g.counted_slots;
  }
  if (lane == 0) bpart[b] = acc;
  if (b == 0 && lane == 0) tl_mark(1);
  __threadfence();  // this warp's counted / adv / ret stores before the grid arrival
  bufwarps_sync();
  AsmPartial* parts = reinterpret_cast<AsmPartial*>(a.ws + a.L.asm_partials);
  uint32_t* tickets = reinterpret_cast<uint32_t*>(a.ws + a.L.tickets);
  if (b == 0 && lane == 0) {
    AsmPartial p{{0.0, 0.0, 0.0}, 0.0};
    for (int w = 0; w < kBufWarps; ++w) {
      p.m = mom_merge(p.m, bpart[w].m);
      p.n_pos += bpart[w].n_pos;
    }
    parts[blockIdx.x] = p;
    volatile uint32_t* gen = tickets + TICKET_GEN;
    const uint32_t g = *gen;
    __threadfence();
    if (atomicAdd(&tickets[TICKET_GRID], 1u) == gridDim.x - 1) {
      tickets[TICKET_GRID] = 0;
      __threadfence();
      atomicAdd(&tickets[TICKET_GEN], 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
    tl_mark(2);
  }
  bufwarps_sync();
  if (b == 0) {  // one warp: fixed-order sum of the grid's partials
    AsmPartial q{{0.0, 0.0, 0.0}, 0.0};
    for (unsigned g = lane; g < gridDim.x; g += 32) {
      q.m = mom_merge(q.m, Moments{__ldcg(&parts[g].m.n), __ldcg(&parts[g].m.mean), __ldcg(&parts[g].m.m2)});
      q.n_pos += __ldcg(&parts[g].n_pos);
    }
    for (int off = 16; off > 0; off >>= 1) {
      const Moments o{__shfl_down_sync(0xffffffffu, q.m.n, off), __shfl_down_sync(0xffffffffu, q.m.mean, off),
                      __shfl_down_sync(0xffffffffu, q.m.m2, off)};
      q.m = mom_merge(q.m, o);
      q.n_pos += __shfl_down_sync(0xffffffffu, q.n_pos, off);
    }
    if (lane == 0) {
      const int64_t n = (int64_t)q.m.n, npos = (int64_t)q.n_pos * a.M;
      // value level == advantage level (assembler.cpp:82): n_val == n_adv
      *s_kf = consts_from(q.m, n, n, npos, 0, 0, a.normalize);
      tl_mark(3);
      if (blockIdx.x == 0) {  // the rank's stats record, as ckrl_assemble_ppo_batch leaves it
        StatsRecord* st = reinterpret_cast<StatsRecord*>(a.ws + a.L.stats_local);
        st->mean = q.m.mean;
        st->m2 = q.m.m2;
        st->flags = 0;
        st->n_adv = st->n_val = n;
        st->n_pos = npos;
        st->groups_retained = 0;
        st->status = 0;
      }
    }
  }
  bufwarps_sync();
}

// Roles (one CTA per SM, persistent over tiles of whole records):
//   warp 0 lane 0   TMA producer: streams the tile's logits into a ring of `nstage` stages
//                   with cp.async.bulk, completion by mbarrier tx-count (full[s]).
//   ROWW row warps  V-bin log-softmax / gather / entropy per row from shared memory
//                   (LDS.128); raw row partials -> row buffer (it mod 4).
//   4 buffer warps  warp m owns row buffer m: stages tile i's row metadata (token ids,
//                   evaluate flags), loads its unit metadata while the rows are computed,
//                   runs the unit phase, then stages tile i+4. In the fused PPO step they
//                   first run the GAE scan for the CTA's envs (phase A) and a grid-wide
//                   barrier, while the producer and row warps already stream logits.
// Synchronisation is mbarrier-only: full[s]/empty[s] (producer <-> row warps),
// metafull[b] (buffer warp -> row warps), rowfull[b] (row warps -> buffer warp).
template <int MODE, typename LT, int ROWW, int RIF, bool FUSED, int BW, bool GRAD = false>
// launch bounds of at least 19 warps' worth: the register cap stays <= 104 for every variant,
// so a 16-warp variant leaves room for 2-warp assembly CTAs on each SM
__global__ void __launch_bounds__(tma_threads<ROWW, BW>() > 608 ? tma_threads<ROWW, BW>() : 608, 1)
    tma_tile_kernel(LossArgs a, int nstage,
                                                                          uint32_t tile_bytes) {
  constexpr int kThreads = tma_threads<ROWW, BW>();
  static_assert(!FUSED || BW == kBufWarps, "the fused step runs with 4 buffer warps");
  constexpr int kPasses = (kTileRowsMax + ROWW * 4 - 1) / (ROWW * 4);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ LossConsts s_k, s_kf;
  __shared__ double s_red[kThreads / 32][RAW_COUNT];
  __shared__ bool s_last;
  __shared__ __align__(8) uint64_t full_bar[4], empty_bar[4], metafull_bar[kMaxRowBufs],
      rowfull_bar[kMaxRowBufs];

  constexpr int V = 256;
  constexpr int kCW = ROWW;  // row warps
  const int M = a.M, P = a.C * M;
  unsigned char* stage_base = smem_raw;
  unsigned char* buf_base = smem_raw + (size_t)nstage * tile_bytes;
  const int nbuf = a.nbuf, cap = a.rows_cap, scap = a.slots_cap;
  unsigned char* grad_base = buf_base + (size_t)nbuf * rowbuf_bytes(cap, scap);  // GRAD: GradSmem per buffer
  auto grad_of = [&](int bi) { return carve_grad(grad_base + (size_t)bi * cap * 12, cap); };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    tl_mark(0);
    // A loss launched right after this one on the stream as a programmatic dependent (the
    // pipelined step's next batch) may start now: its CTAs take SMs as these retire, stream
    // their logits and finish rows, and wait (griddepcontrol.wait) for this grid's completion
    // before their first unit phase.
    asm volatile("griddepcontrol.launch_dependents;");
    CKRL_PROBE(if (blockIdx.x < 1184) g_cta_times[0][blockIdx.x] = gtimer());
    for (int s = 0; s < nstage; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kCW * 32);
    }
    for (int b = 0; b < a.nbuf; ++b) {
      mbar_init(&metafull_bar[b], 32);
      mbar_init(&rowfull_bar[b], kCW * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  Acc acc{0, 0, 0, 0, 0, 0};
  auto tile_recs = [&](int64_t tile, int64_t& r0) {
    r0 = tile * a.rec_per_tile;
    const int64_t rem = a.n_rec - r0;
    return (int)(rem < a.rec_per_tile ? rem : a.rec_per_tile);
  };

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      uint64_t l2_keep = 0;
      if (GRAD) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(l2_keep));
      const char* src = reinterpret_cast<const char*>(a.logits);
      const size_t rec_bytes = (size_t)P * V * sizeof(LT);
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x, ++it) {
        const int s = it % nstage;
        if (it >= nstage) mbar_wait(&empty_bar[s], ((it / nstage) - 1) & 1);
        int64_t r0;
        const int nrec = tile_recs(tile, r0);
        const uint32_t bytes = (uint32_t)(nrec * rec_bytes);
        mbar_expect_tx(&full_bar[s], bytes);
        const char* g = src + (size_t)r0 * rec_bytes;
        unsigned char* d = stage_base + (size_t)s * tile_bytes;
        for (uint32_t off = 0; off < bytes; off += 32768u) {
          const uint32_t n = bytes - off < 32768u ? bytes - off : 32768u;
          if (GRAD)  // keep the tile in L2 for the gradient pass's re-read
            bulk_g2s_keep(d + off, g + off, n, &full_bar[s], l2_keep);
          else
            bulk_g2s(d + off, g + off, n, &full_bar[s]);
        }
      }
    }
  } else if (warp <= kCW) {
    // ---------------- row warps ----------------
    const int cwarp = warp - 1;
    const int sub = lane >> 3, l8 = lane & 7;
    int it = 0;
    // ring positions and phase bits kept incrementally (no integer division per tile)
    int s = 0, b = 0;
    uint32_t sph = 0, bph = 0;
    // GRAD: dlogits of an earlier tile whose coefficients the unit phase left in buffer b
    auto grad_pass = [&](int64_t gtile, const RowSmem& gsm, const GradSmem& gs) {
      int64_t gr0;
      const int grows = tile_recs(gtile, gr0) * P;
      for (int p = 0; p < kPasses; ++p) {
        const int rg0 = (p * kCW + cwarp) * 4;
        if (rg0 >= grows) break;  // warp-uniform
        const int row = rg0 + sub;
        if (row < grows) grad_row<LT>(a, gsm, gs, row, gr0 * P + row, l8);
      }
    };
    // The token ids of this lane's rows (one per pass) come straight from global memory,
    // loaded one tile ahead into registers: their latency hides behind a whole tile, and no
    // other warp stages row metadata (a serial load -> store chain per tile under a
    // saturated HBM, which held the first unit phases back by microseconds).
    int tk_next[kPasses];
    auto load_toks = [&](int64_t tl, int* tk) {
      if (tl >= a.n_tiles) return;
      int64_t tr0;
      const int trows = tile_recs(tl, tr0) * P;
#pragma unroll
      for (int p = 0; p < kPasses; ++p) {
        const int row = (p * kCW + cwarp) * 4 + sub;
        tk[p] = row < trows ? load_token(a.tokens, a.tok_i32, tr0 * P + row) : 0;
      }
    };
    load_toks(blockIdx.x, tk_next);
    constexpr bool kBatchFinish = sizeof(LT) == 2;
    auto finish_row = [&](const RowSmem& sm, int row, float fs, float ft, float fc, float fxt) {
      // The row is finished here, by the lane that holds its sums: log2 s = ex +
      // log2(mant), mant in [1, 2) (the exponent exactly, the mantissa's log2 by the
      // accurate fp32 log2f, |result| < 1: abs error <= 6e-8, so no fp32 rounding of a
      // value up to 8 reaches the log-prob), E[y] = t / s at 2 ulp (entropy only), then
      // in fp64 the first-order correction for the fp32 log2(e) constant (the sums see x
      // scaled by 1 + kL2EDelta: LSE((1+d) x) = LSE(x) + d E[x]). The unit phase then
      // reads one fp64 log-prob and one entropy per row.
      const int ebits = (__float_as_int(fs) >> 23) - 127;  // s >= 1: normal, positive
      const float mant = __int_as_float((__float_as_int(fs) & 0x007fffff) | 0x3f800000);
      const float l2m = log2f(mant);
      const float eyf = __fdividef(ft, fs);
      const double l2s = (double)ebits + (double)l2m;
      const double ls = l2s * kLN2;
      const double ey = (double)eyf, xc = (double)fc;
      sm.lp[row] = ((double)fxt - xc * kLN2) - ls + kL2EDelta * (ey + xc) * kInvL2EF;
      sm.ent[row] = (float)(ls - kLN2 * ey);
      if (GRAD) {  // the fused seam's re-read (grad_row): shift, log2 s, E[y]
        sm.s[row] = (float)l2s;
        sm.t2[row] = eyf;
        sm.c[row] = fc;
      }
    };
    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x, ++it,
                 s = (s + 1 == nstage) ? (sph ^= 1u, 0) : s + 1, b = (b + 1 == nbuf) ? (bph ^= 1u, 0) : b + 1) {
      RowSmem sm;
      MetaSmem mt;
      carve_buf(buf_base + b * rowbuf_bytes(cap, scap), cap, scap, sm, mt);
      int64_t r0;
      const int nrec = tile_recs(tile, r0);
      const int rows = nrec * P;
      int tk[kPasses];
#pragma unroll
      for (int p = 0; p < kPasses; ++p) tk[p] = tk_next[p];
      load_toks(tile + gridDim.x, tk_next);
      mbar_wait(&metafull_bar[b], bph);  // buffer b is free (its previous tile's unit phase is done)
      if (cwarp == 0 && lane == 0 && it < 3) tl_mark(11 + 3 * it);
      if (GRAD && it >= nbuf) grad_pass(tile - (int64_t)nbuf * gridDim.x, sm, grad_of(b));
      mbar_wait(&full_bar[s], sph);
      if (cwarp == 0 && lane == 0 && it < 3) tl_mark(12 + 3 * it);
      CKRL_PROBE(if (blockIdx.x == 0 && cwarp == 0 && lane == 0 && it < 64) g_tile_times[0][it] = gtimer());
      const LT* stage = reinterpret_cast<const LT*>(stage_base + (size_t)s * tile_bytes);
      static_assert(kPasses <= 8, "one captured row per lane of an 8-lane group");
      int f_row = -1;
      float f_s = 1.0f, f_t = 0.0f, f_c = 0.0f, f_xt = 0.0f;
#pragma unroll
      for (int p = 0; p < kPasses; p += RIF) {
        const int rg0 = (p * kCW + cwarp) * 4;
        if (rg0 >= rows) break;  // warp-uniform
        const LT* rp[RIF];
        int rowq[RIF];
        bool live[RIF];
#pragma unroll
        for (int q = 0; q < RIF; ++q) {
          const int rg = ((p + q) * kCW + cwarp) * 4;
          rowq[q] = rg + sub;
          live[q] = (p + q) < kPasses && rg < rows;
          rp[q] = stage + (size_t)(live[q] && rowq[q] < rows ? rowq[q] : rg0) * V;
        }
        float s_[RIF], t_[RIF], c_[RIF];
        if (RIF == 1 || live[RIF - 1])
          rows_fast_smem<LT, RIF>(rp, l8, s_, t_, c_);
        else
          rows_fast_smem<LT, 1>(rp, l8, s_, t_, c_);
        // bf16 rows: the row of pass p + q is finished by lane p + q of its 8-lane group (every
        // lane holds the group's sums) — the capture is a few selects per pass and the
        // finishing math runs once per tile on up to kPasses lanes at a time (bf16 cfg4 226 ->
        // 208 us); f32 rows, whose passes are longer, finish on lane 0 right after each pass
        // (measured 1-2 % faster for them).
#pragma unroll
        for (int q = 0; q < RIF; ++q) {
          const int row = rowq[q];
          if (!live[q] || row >= rows) continue;
          if (GRAD && l8 == 0) grad_of(b).tok[row] = tk[p + q];
          if (l8 == (kBatchFinish ? p + q : 0)) {
            // every row is finished (the unit phase masks by counted / membership); a token
            // id outside [0, V) of an unused row must not read outside the staged row
            const int tok = tk[p + q] & (V - 1);
            const float xt = sizeof(LT) == 4
                                 ? (float)reinterpret_cast<const float*>(rp[q])[tok]
                                 : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(rp[q])[tok]);
            if (kBatchFinish) {
              f_row = row;
              f_s = s_[q];
              f_t = t_[q];
              f_c = c_[q];
              f_xt = xt;
            } else {
              finish_row(sm, row, s_[q], t_[q], c_[q], xt);
            }
          }
        }
      }
      if (kBatchFinish && f_row >= 0) finish_row(sm, f_row, f_s, f_t, f_c, f_xt);
      // Every lane arrives (barrier counts are per thread): each lane's own shared-memory
      // writes are ordered before its arrival (release, CTA scope), which the consumers'
      // try_wait acquires — a per-thread happens-before that racecheck can also see.
      mbar_arrive(&empty_bar[s]);    // stage s fully read by this lane
      mbar_arrive(&rowfull_bar[b]);  // this lane's rows' results are in buffer b
      if (lane == 0) {
        if (cwarp == 0 && it < 3) tl_mark(13 + 3 * it);
        CKRL_PROBE(if (blockIdx.x == 0 && cwarp == 0 && it < 64) g_tile_times[1][it] = gtimer());
      }
    }
    if (GRAD) {  // the last nbuf tiles' gradient passes (their buffers are not reused)
      for (int li = it > nbuf ? it - nbuf : 0; li < it; ++li) {  // local tile index
        const int bi = li % nbuf;
        RowSmem gsm;
        MetaSmem gmt;
        carve_buf(buf_base + bi * rowbuf_bytes(cap, scap), cap, scap, gsm, gmt);
        mbar_wait(&metafull_bar[bi], (uint32_t)((li / nbuf + 1) & 1));  // its unit phase is done
        grad_pass(blockIdx.x + (int64_t)li * gridDim.x, gsm, grad_of(bi));
      }
    }
  } else {
    // ---------------- buffer warps ----------------
    // Warp m owns tiles it = m, m+4, ... and their buffers it % nbuf; with nbuf > 4 the
    // row warps run up to nbuf tiles ahead of the unit phases (e.g. while the overlapped
    // step's assembly kernel is still running), and the backlog drains 4 tiles at a time.
    const int m = warp - 1 - kCW;
    const int64_t stride = (int64_t)BW * gridDim.x;
    auto buf_of = [&](int itx, RowSmem& sm, MetaSmem& mt) {
      carve_buf(buf_base + (itx % nbuf) * rowbuf_bytes(cap, scap), cap, scap, sm, mt);
    };
    RowSmem sm;
    MetaSmem mt;
    // the first nbuf buffers are free: rows of the first nbuf tiles can start right away
    for (int itx = m; itx < nbuf; itx += BW) {
      if (blockIdx.x + (int64_t)itx * gridDim.x >= a.n_tiles) break;
      mbar_arrive(&metafull_bar[itx]);  // every lane (count 32)
    }
    // Software pipeline: this warp's next tile's unit metadata and the row metadata of the
    // next user of this buffer are issued (raw, into registers) before the current unit
    // phase, so their memory latency hides behind it. PPO issues the first tile's loads as
    // soon as the assembly outputs exist, alongside the constants' loads.
    int it = m;
    int64_t tile = blockIdx.x + (int64_t)m * gridDim.x;
    int64_t r0 = 0;
    int nrec = 0;
    UnitRegs ur;
    auto first_unit_meta = [&]() {
      if (tile < a.n_tiles) {
        nrec = tile_recs(tile, r0);
        unit_meta_load<MODE, FUSED>(a, r0, nrec, lane, ur);
      }
    };
    if (FUSED) {
      fused_phase_a(a, m, lane, &s_kf);
      first_unit_meta();
    } else {
      // overlapped step: the assembly kernel's outputs (stats record, counted, advantages)
      // are consumed only from here on (no-op when not launched as a PDL dependent)
      if (a.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
      if (MODE == MODE_PPO) first_unit_meta();  // (GRPO: measured slower, register pressure)
      if (m == 0 && lane == 0) s_k = merge_consts(a);  // off the producer's critical path
      bufwarps_sync<BW>();
      if (MODE != MODE_PPO) first_unit_meta();
    }
    const LossConsts k = FUSED ? s_kf : s_k;
    for (; tile < a.n_tiles; tile += stride, it += BW) {
      const int b = it % nbuf;
      buf_of(it, sm, mt);
      mbar_wait(&rowfull_bar[b], (it / nbuf) & 1);
      CKRL_PROBE(if (blockIdx.x == 0 && lane == 0 && it < 64) g_tile_times[2][it] = gtimer());
      const bool probe = lane == 0 && m == 0;
      if (lane == 0 && it == m) tl_mark(20 + m);
      if (probe && it == BW) tl_mark(3);
      unit_meta_store<MODE>(a, r0, nrec, lane, ur, mt);
      __syncwarp();
      CKRL_PROBE(if (blockIdx.x == 0 && lane == 0 && it < 64) g_tile_times[4][it] = gtimer());
      if (probe && it == 0) tl_mark(1);
      if (probe && it == BW) tl_mark(28);
      const int64_t cr0 = r0;
      const int cn = nrec;
      const int64_t ntile = tile + stride;
      if (ntile < a.n_tiles) {
        nrec = tile_recs(ntile, r0);
        unit_meta_load<MODE, FUSED>(a, r0, nrec, lane, ur);
      }
      const int64_t rtile = tile + (int64_t)nbuf * gridDim.x;  // next user of buffer b
      if (probe && it == 0) tl_mark(2);
      if (probe && it == BW) tl_mark(29);
      if constexpr (GRAD) {
        const GradSmem gs = grad_of(b);
        unit_phase_smem<MODE>(a, k, acc, sm, mt, cr0, cn, lane, outs_of(a), gs.klp, gs.kent);
      } else {
        unit_phase_smem<MODE>(a, k, acc, sm, mt, cr0, cn, lane, outs_of(a));
      }
      __syncwarp();
      CKRL_PROBE(if (blockIdx.x == 0 && lane == 0 && it < 64) g_tile_times[3][it] = gtimer());
      if (lane == 0 && it == m) tl_mark(4 + m);  // first unit phase of each buffer warp
      if (probe && it == BW) tl_mark(30);
      if (rtile < a.n_tiles || GRAD)  // buffer b free for its next tile (GRAD without a next
        mbar_arrive(&metafull_bar[b]);  // user: releases the tile's gradient pass); every lane
    }

  }
  if (warp == 1 && lane == 0) tl_mark(8);  // row warp 0 done with its last tile
  __syncthreads();
  if (tid == 0) tl_mark(9);
  CKRL_PROBE(if (tid == 0 && blockIdx.x < 1184) g_cta_times[1][blockIdx.x] = gtimer());
  if (MODE == MODE_STATS) return;
  reduce_and_finish(a, FUSED ? s_kf : s_k, acc, tid, kThreads, s_red, &s_last);
  if (tid == 0) tl_mark(10);
  CKRL_PROBE(if (tid == 0 && blockIdx.x < 1184) g_cta_times[2][blockIdx.x] = gtimer());
}

static int device_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <int MODE, typename LT, bool FAST>
static cudaError_t launch_direct(LossArgs& a, cudaStream_t s, int* grid_out) {
  auto kern = tile_kernel<MODE, LT, FAST>;
  const int P = a.C * a.M;
  a.rec_per_tile = P >= 256 ? 1 : 256 / P;
  a.n_tiles = (a.n_rec + a.rec_per_tile - 1) / a.rec_per_tile;
  const size_t smem = rowsmem_bytes(a.rec_per_tile * P);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kLossThreads, smem);
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)device_sms() * occ;
  if (grid > a.n_tiles) grid = a.n_tiles;
  if (grid > kMaxLossCtas) grid = kMaxLossCtas;
  if (a.max_ctas > 0 && grid > a.max_ctas) grid = a.max_ctas;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = (int)grid;
  kern<<<(unsigned)grid, kLossThreads, smem, s>>>(a);
  return cudaGetLastError();
}

constexpr size_t kSmemBudget = 220 * 1024;
constexpr size_t kStageTarget = 56 * 1024;

// TMA pipeline plan: whole records per tile (~56 KB), 2-4 stages. Returns false when a
// single record does not fit twice (then the direct kernel runs).
static int max_row_bufs() {  // CKRL_NBUF caps the row-buffer count (A/B experiments)
  static int n = -1;
  if (n < 0) {
    const char* env = getenv("CKRL_NBUF");
    n = env ? atoi(env) : kMaxRowBufs;
    if (n > kMaxRowBufs) n = kMaxRowBufs;
  }
  return n;
}

static size_t stage_target() {  // CKRL_STAGE_KB overrides the tile size (A/B experiments)
  static size_t t = 0;
  if (t == 0) {
    const char* env = getenv("CKRL_STAGE_KB");
    t = env ? (size_t)atoi(env) * 1024 : kStageTarget;
    if (t == 0) t = kStageTarget;
  }
  return t;
}

static bool tma_plan(LossArgs& a, int dbytes, int& rec_per_tile, int& nstage, uint32_t& tile_bytes) {
  const size_t rec = (size_t)a.C * a.M * 256 * dbytes;
  rec_per_tile = (int)(stage_target() / rec);
  if (rec_per_tile < 1) rec_per_tile = 1;
  const int max_rows = kTileRowsMax;
  if (a.C * a.M > max_rows) return false;
  if (rec_per_tile * a.C * a.M > max_rows) rec_per_tile = max_rows / (a.C * a.M);
  tile_bytes = (uint32_t)(rec_per_tile * rec);
  const int cap = (rec_per_tile * a.C * a.M + 7) & ~7;
  const int scap = (rec_per_tile * a.C + 7) & ~7;
  const bool grad = a.dlogits != nullptr;
  const size_t buf = rowbuf_bytes(cap, scap) + (grad ? (size_t)cap * 12 : 0);  // + GradSmem
  // up to 3 stages in flight, then as many row buffers (multiples of 4) as fit; the fused
  // gradient keeps the ring at 4 so a tile's re-read (4 tiles later) still hits L2
  static int max_stage = -1;  // CKRL_NSTAGE: stage-count ceiling (A/B experiments; barriers for 4)
  if (max_stage < 0) {
    const char* env = getenv("CKRL_NSTAGE");
    max_stage = env ? atoi(env) : 3;
    if (max_stage > 4) max_stage = 4;
    if (max_stage < 2) max_stage = 2;
  }
  for (nstage = max_stage; nstage >= 2; --nstage) {
    const size_t used = (size_t)nstage * tile_bytes + 1024;
    if (used >= kSmemBudget) continue;
    int nb = (int)((kSmemBudget - used) / buf) & ~3;
    if (nb > max_row_bufs()) nb = max_row_bufs();
    if (grad && nb > kRowBufs) nb = kRowBufs;
    if (nb >= kRowBufs) {
      a.nbuf = nb;
      a.rows_cap = cap;
      a.slots_cap = scap;
      return true;
    }
  }
  return false;
}

template <int MODE, typename LT, int ROWW, int RIF, bool FUSED, int BW = kBufWarps, bool GRAD = false>
static cudaError_t launch_tma_v(LossArgs& a, cudaStream_t s, int* grid_out, int nstage, uint32_t tile_bytes) {
  auto kern = tma_tile_kernel<MODE, LT, ROWW, RIF, FUSED, BW, GRAD>;
  if (a.nbuf % BW) a.nbuf -= a.nbuf % BW;
  a.n_tiles = (a.n_rec + a.rec_per_tile - 1) / a.rec_per_tile;
  const size_t smem = (size_t)nstage * tile_bytes + (size_t)a.nbuf * rowbuf_bytes(a.rows_cap, a.slots_cap) +
                      (GRAD ? (size_t)a.nbuf * a.rows_cap * 12 : 0);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int64_t grid = device_sms();
  if (grid > a.n_tiles) grid = a.n_tiles;
  if (a.max_ctas > 0 && grid > a.max_ctas) grid = a.max_ctas;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = (int)grid;
  if (!FUSED && a.pdl) {  // programmatic dependent of the assembly kernel
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(tma_threads<ROWW, BW>());
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a, nstage, tile_bytes);
  }
  if (!FUSED) {
    kern<<<(unsigned)grid, tma_threads<ROWW, BW>(), smem, s>>>(a, nstage, tile_bytes);
    return cudaGetLastError();
  }
  // The fused step has a grid-wide barrier: co-residency of every CTA is required, so the
  // launch is cooperative (one CTA per SM by construction).
  void* args[] = {&a, &nstage, &tile_bytes};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)grid), dim3(tma_threads<ROWW, BW>()),
                                     args, smem, s);
}

static int g_tma_variant = -1;
static int device_sms_cached() {
  static int n = 0;
  if (n == 0) n = device_sms();
  return n;
}

template <int MODE, typename LT, bool FUSED>
static cudaError_t launch_tma(LossArgs& a, cudaStream_t s, int* grid_out, int nstage, uint32_t tile_bytes) {
  if (g_tma_variant < 0) {
    const char* env = getenv("CKRL_TMA_VARIANT");
    g_tma_variant = env ? atoi(env) : 99;  // 99: by shape (below)
  }
  if constexpr (!FUSED && MODE != MODE_STATS)
    if (a.dlogits)  // fused softmax-backward seam (row f1)
      return launch_tma_v<MODE, LT, 14, 1, FUSED, kBufWarps, true>(a, s, grid_out, nstage, tile_bytes);
  int variant = g_tma_variant;
  if (variant == 99) {
    // PPO launches of a few tiles per SM (cfg1 / cfg3): 16-warp CTAs, so the 2-warp assembly
    // CTAs (the previous or next step's, on another stream, or this step's under PDL) share
    // the SMs instead of waiting for loss CTAs to retire (cfg3 40.4 -> 38.4 us, cfg3 bf16
    // 35.2 -> 32.8, cfg1 bf16 21.2 -> 19.4); long launches (cfg4: 221 tiles per SM) and GRPO
    // keep 14 row warps, which the steady-state row throughput needs (cfg4 f32 308 vs 372 us)
    const int64_t per_sm = (a.n_rec + a.rec_per_tile - 1) / a.rec_per_tile / device_sms_cached();
    // a capped grid (the pipelined halves' launch policy) leaves SMs free for the assembly, so
    // the 14-row-warp CTA wins there (cfg3 29.7 -> 26.5 us, cfg1 12.3 -> 10.6 us per step)
    const bool capped = a.max_ctas > 0 && a.max_ctas < device_sms_cached();
    // the 16-warp CTA only where an assembly CTA must share its SM: a programmatic dependent
    // of its own assembly (ckrl_ppo_step) on a full grid
    variant = (MODE == MODE_PPO && !FUSED && per_sm <= 32 && !capped && a.pdl) ? 5 : 4;
  }
  switch (variant) {
    // measured on B200 (cfg4 f32): 16x1 reaches the HBM roofline; 8x2 is latency-bound
    case 3: return launch_tma_v<MODE, LT, 8, 2, FUSED>(a, s, grid_out, nstage, tile_bytes);
    // 11 row warps: 16-warp CTAs that an assembly CTA can share an SM with
    case 5: return launch_tma_v<MODE, LT, 11, 1, FUSED>(a, s, grid_out, nstage, tile_bytes);
    case 0: return launch_tma_v<MODE, LT, 16, 1, FUSED>(a, s, grid_out, nstage, tile_bytes);
    // default: 14 row warps (a 56-row tile is 14 x 4 rows) -> 19 warps, 96 registers, no spills
    default: return launch_tma_v<MODE, LT, 14, 1, FUSED>(a, s, grid_out, nstage, tile_bytes);
  }
}

static int g_force_direct = -1;

template <int MODE>
static cudaError_t launch_mode(LossArgs& a, cudaStream_t s, int* g) {
  if (g_force_direct < 0) {
    const char* env = getenv("CKRL_LOSS_KERNEL");
    g_force_direct = (env && env[0] == 'd') ? 1 : 0;
  }
  if (a.rows_in) {  // per-position rows already finished: only the unit phase is left
    if (a.dlogits) return cudaErrorInvalidValue;
    return launch_direct<MODE, float, true>(a, s, g);
  }
  const bool fast = a.V == 256;
  const int dbytes = a.logits_bf16 ? 2 : 4;
  int rpt, nstage;
  uint32_t tile_bytes;
  const uintptr_t align = reinterpret_cast<uintptr_t>(a.logits) & 15;
  const uintptr_t galign = reinterpret_cast<uintptr_t>(a.dlogits) & 15;
  if (fast && !g_force_direct && align == 0 && galign == 0 && tma_plan(a, dbytes, rpt, nstage, tile_bytes)) {
    a.rec_per_tile = rpt;
    return a.logits_bf16 ? launch_tma<MODE, __nv_bfloat16, false>(a, s, g, nstage, tile_bytes)
                         : launch_tma<MODE, float, false>(a, s, g, nstage, tile_bytes);
  }
  cudaError_t e = a.logits_bf16 ? (fast ? launch_direct<MODE, __nv_bfloat16, true>(a, s, g)
                                        : launch_direct<MODE, __nv_bfloat16, false>(a, s, g))
                                : (fast ? launch_direct<MODE, float, true>(a, s, g)
                                        : launch_direct<MODE, float, false>(a, s, g));
  if (e != cudaSuccess || !a.dlogits || MODE == MODE_STATS) return e;
  // no fused path for this shape: the standalone seam kernel over the loss's coefficients
  if (!a.coeff_lp) return cudaErrorInvalidValue;
  return launch_logits_grad(a.logits, a.logits_bf16, a.tokens, a.tok_i32, a.coeff_lp, a.coeff_ent,
                            a.n_rec * a.C * a.M, a.V, a.dlogits, a.logits_bf16, nullptr, s);
}

// The fused single-GPU PPO step (assembly + loss in one persistent launch). Returns
// cudaErrorNotSupported when the shape has no TMA plan (caller uses the 2-kernel path).
cudaError_t launch_ppo_fused(LossArgs& a, cudaStream_t s, int* g) {
  if (g_force_direct < 0) {
    const char* env = getenv("CKRL_LOSS_KERNEL");
    g_force_direct = (env && env[0] == 'd') ? 1 : 0;
  }
  const int dbytes = a.logits_bf16 ? 2 : 4;
  int rpt, nstage;
  uint32_t tile_bytes;
  const uintptr_t align = reinterpret_cast<uintptr_t>(a.logits) & 15;
  if (a.rows_in || a.V != 256 || g_force_direct || align != 0 || !tma_plan(a, dbytes, rpt, nstage, tile_bytes))
    return cudaErrorNotSupported;
  a.rec_per_tile = rpt;
  return a.logits_bf16 ? launch_tma<MODE_PPO, __nv_bfloat16, true>(a, s, g, nstage, tile_bytes)
                       : launch_tma<MODE_PPO, float, true>(a, s, g, nstage, tile_bytes);
}

cudaError_t launch_tile(LossArgs& a, cudaStream_t s, int* grid_out) {
  switch (a.mode) {
    case MODE_STATS: return launch_mode<MODE_STATS>(a, s, grid_out);
    case MODE_PPO: return launch_mode<MODE_PPO>(a, s, grid_out);
    default: return launch_mode<MODE_GRPO>(a, s, grid_out);
  }
}

cudaError_t read_timeline(uint64_t* out, int n) {
  return cudaMemcpyFromSymbol(out, g_timeline, sizeof(uint64_t) * (n < 32 ? n : 32));
}

cudaError_t debug_cta_times(uint64_t* out, int n) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_cta_times, sizeof(uint64_t) * (n < 3 * 1184 ? n : 3 * 1184));
  if (e != cudaSuccess || n < 3 * 1184 + 7 * 64) return e;
  return cudaMemcpyFromSymbol(out + 3 * 1184, g_tile_times, sizeof(uint64_t) * 7 * 64);
}

}  // namespace ckrl
