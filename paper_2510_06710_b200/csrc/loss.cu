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
#include "kernels.h"

namespace ckrl {

constexpr float kL2E = 1.4426950408889634f;
constexpr double kLN2 = 0.6931471805599453;

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
  double inv_adv, inv_val, inv_pos, mean, denom, inv_groups;
  int do_norm;
  int64_t n_adv, groups;
  int status;
};

__device__ LossConsts merge_consts(const LossArgs& a) {
  LossConsts k;
  Moments m{0.0, 0.0, 0.0};
  int64_t n_adv = 0, n_val = 0, n_pos = 0, groups = 0;
  int status = 0;
  for (int r = 0; r < a.world; ++r) {
    const StatsRecord& s = a.recs[r];
    m = merge_moments(m, Moments{(double)s.n_units, s.mean, s.m2});
    n_adv += s.n_adv;
    n_val += s.n_val;
    n_pos += s.n_pos;
    groups += s.groups_retained;
    if (s.status && !status) status = (int)s.status;
  }
  k.n_adv = n_adv;
  k.groups = groups;
  k.inv_adv = n_adv > 0 ? 1.0 / (double)n_adv : 0.0;
  k.inv_val = n_val > 0 ? 1.0 / (double)n_val : 0.0;
  k.inv_pos = n_pos > 0 ? 1.0 / (double)n_pos : 0.0;
  k.do_norm = a.normalize && m.n >= 2.0;
  k.mean = m.mean;
  k.denom = m.n > 0 ? sqrt(m.m2 / m.n) + 1e-8 : 1.0;
  k.inv_groups = groups > 0 ? 1.0 / (double)groups : 0.0;
  k.status = status;
  return k;
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

template <int MODE, typename LT, bool FAST>
__global__ void __launch_bounds__(kLossThreads, 2) tile_kernel(LossArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ LossConsts s_k;
  __shared__ double s_red[kLossThreads / 32][RAW_COUNT];
  __shared__ bool s_last;

  const int C = a.C, M = a.M, P = C * M, V = a.V;
  const int rows_cap = a.rec_per_tile * P;
  RowSmem sm;
  sm.lp = reinterpret_cast<double*>(smem_raw);
  sm.s = reinterpret_cast<float*>(sm.lp + rows_cap);
  sm.t2 = sm.s + rows_cap;
  sm.c = sm.t2 + rows_cap;
  sm.xt = sm.c + rows_cap;
  sm.old = sm.xt + rows_cap;
  sm.ent = sm.old + rows_cap;

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
    const int64_t k0 = r0 * P;  // first token of the tile
    // ---------------- row phase ----------------
    for (int rg = warp * 4; rg < rows; rg += (kLossThreads / 32) * 4) {
      const int row = rg + sub;
      bool need = row < rows;
      if (need && !a.all_rows) {
        const int64_t slot = (k0 + row) / M;
        if (MODE == MODE_PPO) need = a.counted[slot] != 0;
        if (MODE == MODE_GRPO) need = a.slot_member[slot] && a.slot_weight[slot] != 0.0f;
      }
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
    // ---------------- token pass: lp, entropy (+ PPO entropy / token-level units) ----
    for (int row = tid; row < rows; row += kLossThreads) {
      const int64_t kk = k0 + row;
      const int64_t slot = kk / M;
      const int64_t rec = kk / P;
      const double s = (double)sm.s[row];
      const double ls = log(s);
      const double lp = ((double)sm.xt[row] - (double)sm.c[row] * kLN2) - ls;
      const float ent = (float)(ls - kLN2 * (double)sm.t2[row] / s);
      const float old = MODE == MODE_STATS ? 0.0f : __ldg(a.old_lp + kk);
      sm.lp[row] = lp;
      sm.ent[row] = ent;
      sm.old[row] = old;
      if (a.tok_lp) a.tok_lp[kk] = (float)lp;
      if (a.tok_ent) a.tok_ent[kk] = ent;
      if (MODE == MODE_PPO) {
        const bool cnt = a.counted[slot] != 0;
        if (cnt) acc.ent += ent;
        if (a.coeff_ent) a.coeff_ent[kk] = (cnt && a.ecoef != 0.0) ? (float)(-a.ecoef * k.inv_pos) : 0.0f;
        if (a.lp_level == CKRL_LEVEL_TOKEN) {
          float coeff = 0.0f;
          if (cnt) {
            double adv = a.adv_level == CKRL_LEVEL_CHUNK ? (double)a.adv[rec] : (double)a.adv[slot];
            if (k.do_norm) adv = (adv - k.mean) / k.denom;
            const double d = lp - (double)old;
            const double rho = exp(d);
            Surrogate su = clipped_surrogate(rho, adv, a.clip);
            acc.surr += su.value;
            acc.units += 1.0;
            acc.clipped += su.clipped;
            acc.kl += (rho - 1.0) - d;
            coeff = (float)(-k.inv_adv * su.dlogprob);
          }
          if (a.coeff_lp) a.coeff_lp[kk] = coeff;
        }
      } else if (MODE == MODE_GRPO && a.lp_level == CKRL_LEVEL_TOKEN) {
        const int e = (int)(rec / a.Tc);
        const float w = a.slot_weight[slot];
        float coeff = 0.0f;
        if (a.env_group[e] >= 0 && a.slot_member[slot] && w != 0.0f) {
          const double inv_g = 1.0 / (double)a.env_group_size[e];
          const double d = lp - (double)old;
          const double rho = exp(d);
          Surrogate su = clipped_surrogate(rho, a.env_adv[e], a.clip);
          acc.surr += k.inv_groups * inv_g * (double)w * su.value;
          acc.units += 1.0;
          acc.clipped += su.clipped;
          acc.kl += (rho - 1.0) - d;
          coeff = (float)(-k.inv_groups * inv_g * (double)w * su.dlogprob);
        }
        if (a.coeff_lp) a.coeff_lp[kk] = coeff;
      }
    }
    __syncthreads();
    // ---------------- slot / record units ----------------
    if (MODE == MODE_STATS) {
      if (a.action_lp)
        for (int sl = tid; sl < nrec * C; sl += kLossThreads) {
          double s = 0.0;
          for (int j = 0; j < M; ++j) s += sm.lp[sl * M + j];
          a.action_lp[r0 * C + sl] = s;
        }
      if (a.chunk_lp)
        for (int r = tid; r < nrec; r += kLossThreads) {
          double s = 0.0;
          for (int i = 0; i < C; ++i) {
            double ai = 0.0;
            for (int j = 0; j < M; ++j) ai += sm.lp[(r * C + i) * M + j];
            s += ai;
          }
          a.chunk_lp[r0 + r] = s;
        }
    } else if (MODE == MODE_PPO) {
      const bool chunk_adv = a.adv_level == CKRL_LEVEL_CHUNK;
      if (a.lp_level == CKRL_LEVEL_ACTION) {
        for (int sl = tid; sl < nrec * C; sl += kLossThreads) {
          const int64_t slot = r0 * C + sl;
          float coeff = 0.0f;
          if (a.counted[slot]) {
            double an = 0.0, ao = 0.0;
            for (int j = 0; j < M; ++j) {
              an += sm.lp[sl * M + j];
              ao += (double)sm.old[sl * M + j];
            }
            double adv = chunk_adv ? (double)a.adv[r0 + sl / C] : (double)a.adv[slot];
            if (k.do_norm) adv = (adv - k.mean) / k.denom;
            const double rho = exp(an - ao);
            Surrogate su = clipped_surrogate(rho, adv, a.clip);
            acc.surr += su.value;
            acc.units += 1.0;
            acc.clipped += su.clipped;
            acc.kl += (rho - 1.0) - (an - ao);
            coeff = (float)(-k.inv_adv * su.dlogprob);
          }
          if (a.coeff_lp)
            for (int j = 0; j < M; ++j) a.coeff_lp[slot * M + j] = coeff;
        }
      } else if (a.lp_level == CKRL_LEVEL_CHUNK) {  // chunk advantage (validated)
        for (int r = tid; r < nrec; r += kLossThreads) {
          const int64_t rec = r0 + r;
          double lpn = 0.0, lpo = 0.0;
          bool any = false;
          for (int i = 0; i < C; ++i) {
            if (!a.counted[rec * C + i]) continue;
            any = true;
            double an = 0.0, ao = 0.0;
            for (int j = 0; j < M; ++j) {
              an += sm.lp[(r * C + i) * M + j];
              ao += (double)sm.old[(r * C + i) * M + j];
            }
            lpn += an;
            lpo += ao;
          }
          float coeff = 0.0f;
          if (any) {
            double adv = (double)a.adv[rec];
            if (k.do_norm) adv = (adv - k.mean) / k.denom;
            const double rho = exp(lpn - lpo);
            Surrogate su = clipped_surrogate(rho, adv, a.clip);
            acc.surr += su.value;
            acc.units += 1.0;
            acc.clipped += su.clipped;
            acc.kl += (rho - 1.0) - (lpn - lpo);
            coeff = (float)(-k.inv_adv * su.dlogprob);
          }
          if (a.coeff_lp)
            for (int i = 0; i < C; ++i) {
              const float ci = a.counted[rec * C + i] ? coeff : 0.0f;
              for (int j = 0; j < M; ++j) a.coeff_lp[(rec * C + i) * M + j] = ci;
            }
        }
      }
      // value loss at the value level (losses.cpp:262-285)
      if (a.val_level == CKRL_LEVEL_CHUNK) {
        for (int r = tid; r < nrec; r += kLossThreads) {
          const int64_t rec = r0 + r;
          bool any = false;
          for (int i = 0; i < C; ++i) any = any || a.counted[rec * C + i];
          float cv = 0.0f;
          if (any && a.new_values) {
            const double err = (double)a.new_values[rec] - (double)a.ret[rec];
            acc.valsq += err * err;
            cv = (float)(a.vcoef * 2.0 * err * k.inv_val);
          }
          if (a.coeff_val) a.coeff_val[rec] = cv;
        }
      } else {
        for (int sl = tid; sl < nrec * C; sl += kLossThreads) {
          const int64_t slot = r0 * C + sl;
          float cv = 0.0f;
          if (a.counted[slot] && a.new_values) {
            const double err = (double)a.new_values[slot] - (double)a.ret[slot];
            acc.valsq += err * err;
            cv = (float)(a.vcoef * 2.0 * err * k.inv_val);
          }
          if (a.coeff_val) a.coeff_val[slot] = cv;
        }
      }
    } else {  // MODE_GRPO, action / chunk log-prob units (losses.cpp:347-380)
      if (a.lp_level == CKRL_LEVEL_ACTION) {
        for (int sl = tid; sl < nrec * C; sl += kLossThreads) {
          const int64_t slot = r0 * C + sl;
          const int e = (int)((r0 + sl / C) / a.Tc);
          const float w = a.slot_weight[slot];
          float coeff = 0.0f;
          if (a.env_group[e] >= 0 && a.slot_member[slot] && w != 0.0f) {
            const double inv_g = 1.0 / (double)a.env_group_size[e];
            double an = 0.0, ao = 0.0;
            for (int j = 0; j < M; ++j) {
              an += sm.lp[sl * M + j];
              ao += (double)sm.old[sl * M + j];
            }
            const double rho = exp(an - ao);
            Surrogate su = clipped_surrogate(rho, a.env_adv[e], a.clip);
            acc.surr += k.inv_groups * inv_g * (double)w * su.value;
            acc.units += 1.0;
            acc.clipped += su.clipped;
            acc.kl += (rho - 1.0) - (an - ao);
            coeff = (float)(-k.inv_groups * inv_g * (double)w * su.dlogprob);
          }
          if (a.coeff_lp)
            for (int j = 0; j < M; ++j) a.coeff_lp[slot * M + j] = coeff;
        }
      } else if (a.lp_level == CKRL_LEVEL_CHUNK) {
        for (int r = tid; r < nrec; r += kLossThreads) {
          const int64_t rec = r0 + r;
          const int e = (int)(rec / a.Tc);
          double lpn = 0.0, lpo = 0.0, wsum = 0.0;
          bool any = false;
          const bool has = a.env_group[e] >= 0;
          for (int i = 0; has && i < C; ++i) {
            const float w = a.slot_weight[rec * C + i];
            if (!a.slot_member[rec * C + i] || w == 0.0f) continue;
            any = true;
            double an = 0.0, ao = 0.0;
            for (int j = 0; j < M; ++j) {
              an += sm.lp[(r * C + i) * M + j];
              ao += (double)sm.old[(r * C + i) * M + j];
            }
            lpn += an;
            lpo += ao;
            wsum += (double)w;
          }
          float coeff = 0.0f;
          if (any) {
            const double inv_g = 1.0 / (double)a.env_group_size[e];
            const double rho = exp(lpn - lpo);
            Surrogate su = clipped_surrogate(rho, a.env_adv[e], a.clip);
            acc.surr += k.inv_groups * inv_g * wsum * su.value;
            acc.units += 1.0;
            acc.clipped += su.clipped;
            acc.kl += (rho - 1.0) - (lpn - lpo);
            coeff = (float)(-k.inv_groups * inv_g * wsum * su.dlogprob);
          }
          if (a.coeff_lp)
            for (int i = 0; i < C; ++i) {
              const bool cov = any && a.slot_member[rec * C + i] && a.slot_weight[rec * C + i] != 0.0f;
              for (int j = 0; j < M; ++j) a.coeff_lp[(rec * C + i) * M + j] = cov ? coeff : 0.0f;
            }
        }
      }
    }
    __syncthreads();
  }

  if (MODE == MODE_STATS) return;
  // ---------------- deterministic reduction: warp -> CTA -> last CTA ----------------
  double v[RAW_COUNT] = {acc.surr, acc.valsq, acc.ent, acc.kl, acc.clipped, acc.units, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < RAW_COUNT; ++i) {
    double x = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) s_red[warp][i] = x;
  }
  __syncthreads();
  double* parts = reinterpret_cast<double*>(a.ws + a.L.loss_partials);
  uint32_t* tickets = reinterpret_cast<uint32_t*>(a.ws + a.L.tickets);
  if (tid < RAW_COUNT) {
    double x = 0.0;
    for (int w = 0; w < kLossThreads / 32; ++w) x += s_red[w][tid];
    parts[blockIdx.x * RAW_COUNT + tid] = x;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&tickets[TICKET_LOSS], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid < RAW_COUNT) {
    double x = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) x += const_cast<volatile double*>(parts)[b * RAW_COUNT + tid];
    reinterpret_cast<double*>(a.ws + a.L.loss_raw)[tid] = x;
  }
  __syncthreads();
  if (tid == 0) {
    tickets[TICKET_LOSS] = 0;
    if (a.finalize) finalize_diag(a, k, reinterpret_cast<double*>(a.ws + a.L.loss_raw), a.diag);
  }
}

__global__ void finalize_kernel(LossArgs a) {
  if (threadIdx.x != 0) return;
  LossConsts k = merge_consts(a);
  finalize_diag(a, k, reinterpret_cast<double*>(a.ws + a.L.loss_raw), a.diag);
}

template <int MODE, typename LT, bool FAST>
static cudaError_t launch_tile_t(LossArgs& a, cudaStream_t s, int* grid_out) {
  auto kern = tile_kernel<MODE, LT, FAST>;
  const int rows_cap = a.rec_per_tile * a.C * a.M;
  const size_t smem = (size_t)rows_cap * (sizeof(double) + 6 * sizeof(float));
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kLossThreads, smem);
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)sms * occ;
  if (grid > a.n_tiles) grid = a.n_tiles;
  if (grid > kMaxLossCtas) grid = kMaxLossCtas;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = (int)grid;
  kern<<<(unsigned)grid, kLossThreads, smem, s>>>(a);
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_mode(LossArgs& a, cudaStream_t s, int* g) {
  const bool fast = a.V == 256;
  if (a.logits_bf16)
    return fast ? launch_tile_t<MODE, __nv_bfloat16, true>(a, s, g)
                : launch_tile_t<MODE, __nv_bfloat16, false>(a, s, g);
  return fast ? launch_tile_t<MODE, float, true>(a, s, g) : launch_tile_t<MODE, float, false>(a, s, g);
}

cudaError_t launch_tile(LossArgs& a, cudaStream_t s, int* grid_out) {
  // tile = whole records, ~256 token rows per tile
  const int P = a.C * a.M;
  a.rec_per_tile = P >= 256 ? 1 : 256 / P;
  a.n_tiles = (a.n_rec + a.rec_per_tile - 1) / a.rec_per_tile;
  if (a.n_rec == 0) {
    a.n_tiles = 0;
  }
  switch (a.mode) {
    case MODE_STATS: return launch_mode<MODE_STATS>(a, s, grid_out);
    case MODE_PPO: return launch_mode<MODE_PPO>(a, s, grid_out);
    default: return launch_mode<MODE_GRPO>(a, s, grid_out);
  }
}

cudaError_t launch_finalize(LossArgs& a, cudaStream_t s) {
  finalize_kernel<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace ckrl
