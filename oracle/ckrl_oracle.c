/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path. See
 * ckrl_oracle.h for the contract (who may call it, how it is pinned).
 *
 * Each function names the reference lines it restates (paths relative to
 * /root/reference/proj/src/chunkrl). The restatement works on the SoA slab of
 * include/ckrl.h instead of the reference's AoS TrajectorySlab, but keeps every
 * floating-point operation and its order, so identical double inputs give
 * bit-identical outputs.
 */
#include "ckrl_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Status codes: include/ckrl.h (1:1 with core/errors.hpp:9-48). */
enum {
  ST_OK = 0,
  ST_UNSUPPORTED_COMBINATION = 1,
  ST_LENGTH_MISMATCH = 3,
  ST_NON_FINITE = 6,
  ST_DEGENERATE_GROUP = 7,
  ST_SKIP_UPDATE = 8,
  ST_CONFIG = 12,
  ST_ERROR = 13
};

/* core/granularity.cpp:47-60 */
int orc_validate_granularity(int adv_level, int lp_level, int val_level) {
  if (adv_level == ORC_TOKEN) return ST_UNSUPPORTED_COMBINATION;
  if (val_level == ORC_TOKEN) return ST_UNSUPPORTED_COMBINATION;
  /* rank: chunk 0 < action 1 < token 2; reject lp coarser than advantage */
  if (lp_level < adv_level) return ST_UNSUPPORTED_COMBINATION;
  return ST_OK;
}

/* advantage/gae.cpp:7-37 */
int orc_compute_gae(int n, const double* r, const double* v, const double* boot,
                    const uint8_t* term, const uint8_t* trunc, double gamma, double lambda,
                    double* adv, double* ret) {
  double next_adv = 0.0;
  for (int i = n - 1; i >= 0; --i) {
    double vnext;
    if (term[i])
      vnext = 0.0;
    else if (trunc[i] || i + 1 == n)
      vnext = boot[i];
    else
      vnext = v[i + 1];
    double delta = r[i] + gamma * vnext - v[i];
    int done = term[i] || trunc[i];
    double a = delta + gamma * lambda * (done ? 0.0 : next_adv);
    adv[i] = a;
    ret[i] = a + v[i];
    next_adv = a;
  }
  return ST_OK;
}

/* policy/policy_net.cpp:90-102 */
void orc_log_softmax(int V, const double* x, double* out) {
  double mx = x[0];
  for (int v = 0; v < V; ++v) mx = x[v] > mx ? x[v] : mx;
  double sum = 0.0;
  for (int v = 0; v < V; ++v) sum += exp(x[v] - mx);
  double lse = mx + log(sum);
  for (int v = 0; v < V; ++v) out[v] = x[v] - lse;
}

/* PolicyNet::logits_from_feature (policy/policy_net.cpp:265-274): per position,
 * logits[v] = matvec(W_pol, h)[v] + b_pol[v] -- matvec (:13-21) sums row[c] * x[c] in ascending
 * c from 0.0, then the bias is added. W is [V][H] row-major; b may be NULL (zero bias). */
void orc_project_logits(int64_t rows, int H, int V, const double* feature, const double* W,
                        const double* b, double* logits) {
  for (int64_t k = 0; k < rows; ++k) {
    const double* h = feature + k * H;
    for (int v = 0; v < V; ++v) {
      double s = 0.0;
      const double* row = W + (int64_t)v * H;
      for (int c = 0; c < H; ++c) s += row[c] * h[c];
      logits[k * V + v] = s + (b ? b[v] : 0.0);
    }
  }
}

/* policy/policy_net.cpp:345-355 (evaluate_chunk, per position) */
void orc_token_stats(int64_t rows, int V, const double* logits, const int32_t* tokens,
                     double* lp, double* ent) {
  double* ls = (double*)malloc(sizeof(double) * (size_t)V);
  for (int64_t k = 0; k < rows; ++k) {
    orc_log_softmax(V, logits + k * V, ls);
    lp[k] = ls[tokens[k]];
    double h = 0.0;
    for (int v = 0; v < V; ++v) h -= exp(ls[v]) * ls[v];
    ent[k] = h;
  }
  free(ls);
}

/* Entropy at action and chunk granularity (north star (b); the reference has only the
 * per-token entropy, policy_net.cpp:333-357 / losses.cpp:181-190): the canonical
 * aggregation order of core/granularity.cpp:83-113 applied to per-token entropies, over the
 * slots `mask` ([chunks][C], nonzero = included; NULL = all) selects, 0 elsewhere:
 *   action[s] = sum_{j ascending} H[s][j];  chunk[r] = sum_{i ascending, mask} action[r][i]. */
void orc_entropy_aggregates(int64_t chunks, int C, int M, const double* ent, const uint8_t* mask,
                            double* action, double* chunk) {
  for (int64_t r = 0; r < chunks; ++r) {
    double c = 0.0;
    for (int i = 0; i < C; ++i) {
      const int64_t s = r * C + i;
      double a = 0.0;
      if (!mask || mask[s]) {
        for (int j = 0; j < M; ++j) a += ent[s * M + j];
        c += a;
      }
      action[s] = a;
    }
    chunk[r] = c;
  }
}

/* policy/policy_net.cpp:431-456 (accumulate_chunk_gradient, the per-position logits
 * gradient before outer_add / the trunk backward): positions with klp == 0 && kent == 0
 * are skipped (zero row here), non-finite coefficients throw NonFinite (:437-438). */
int orc_logits_grad(int64_t rows, int V, const double* logits, const int32_t* tokens,
                    const double* coeff_lp, const double* coeff_ent, double* dlogits) {
  double* ls = (double*)malloc(sizeof(double) * (size_t)V);
  int st = ST_OK;
  for (int64_t k = 0; k < rows; ++k) {
    double* d = dlogits + k * V;
    const double klp = coeff_lp[k], kent = coeff_ent[k];
    if (klp == 0.0 && kent == 0.0) {
      for (int v = 0; v < V; ++v) d[v] = 0.0;
      continue;
    }
    if (!isfinite(klp) || !isfinite(kent)) {
      st = ST_NON_FINITE;
      break;
    }
    orc_log_softmax(V, logits + k * V, ls);
    double H = 0.0;
    if (kent != 0.0)
      for (int v = 0; v < V; ++v) H -= exp(ls[v]) * ls[v];
    for (int v = 0; v < V; ++v) {
      double pv = exp(ls[v]);
      double dv = klp * ((v == tokens[k] ? 1.0 : 0.0) - pv);
      if (kent != 0.0) dv += kent * (-pv * (ls[v] + H));
      d[v] = dv;
    }
  }
  free(ls);
  return st;
}

/* optim/adam.cpp:15-41 (Adam::step). `t` is the step count after this step (the reference's
 * ++t_); m, v are the moment buffers. Returns NonFinite without modifying anything when the
 * gradient norm is not finite. */
int orc_adam_step(int64_t n, double* params, double* grad, double* m, double* v, double lr,
                  double max_grad_norm, double beta1, double beta2, double eps, int64_t t,
                  double* norm_out) {
  double norm_sq = 0.0;
  for (int64_t i = 0; i < n; ++i) norm_sq += grad[i] * grad[i];
  double norm = sqrt(norm_sq);
  *norm_out = norm;
  if (!isfinite(norm)) return ST_NON_FINITE;
  if (max_grad_norm > 0.0 && norm > max_grad_norm) {
    double scale = max_grad_norm / norm;
    for (int64_t i = 0; i < n; ++i) grad[i] *= scale;
  }
  double bc1 = 1.0 - pow(beta1, (double)t);
  double bc2 = 1.0 - pow(beta2, (double)t);
  for (int64_t i = 0; i < n; ++i) {
    m[i] = beta1 * m[i] + (1.0 - beta1) * grad[i];
    v[i] = beta2 * v[i] + (1.0 - beta2) * grad[i] * grad[i];
    double mhat = m[i] / bc1;
    double vhat = v[i] / bc2;
    params[i] -= lr * mhat / (sqrt(vhat) + eps);
  }
  return ST_OK;
}

/* ---------------------------------------------------------------- PPO assembly */

typedef struct {
  int64_t* slot;   /* action level: slot index; chunk level: record index */
  int64_t* boot_slot;
  double *r, *v, *boot, *a, *R;
  uint8_t *term, *trunc;
  int n;
} segbuf;

/* advantage/assembler.cpp:33-56 (flush_segment) */
static void flush(segbuf* sg, int open_end, const orc_rollout* ro, double gamma, double lambda,
                  double* adv, double* ret, int action_level) {
  int n = sg->n;
  if (n == 0) return;
  for (int i = 0; i < n; ++i) sg->boot[i] = sg->trunc[i] ? ro->bootstrap[sg->boot_slot[i]] : 0.0;
  if (open_end && !sg->term[n - 1] && !sg->trunc[n - 1])
    sg->boot[n - 1] = ro->bootstrap[sg->boot_slot[n - 1]];
  orc_compute_gae(n, sg->r, sg->v, sg->boot, sg->term, sg->trunc, gamma, lambda, sg->a, sg->R);
  for (int i = 0; i < n; ++i) {
    adv[sg->slot[i]] = sg->a[i];
    ret[sg->slot[i]] = sg->R[i];
  }
  (void)action_level;
  sg->n = 0;
}

/* advantage/assembler.cpp:78-195 (assemble_ppo_batch) */
int orc_assemble_ppo(const orc_rollout* ro, int adv_level, int lp_level, int val_level,
                     double gamma, double lambda, uint8_t* counted, double* adv, double* ret) {
  int st = orc_validate_granularity(adv_level, lp_level, val_level);
  if (st) return st;
  if (val_level != adv_level) return ST_CONFIG;
  const int E = ro->E, Tc = ro->Tc, C = ro->C;
  const int action = adv_level == ORC_ACTION;
  const int64_t nslots = (int64_t)E * Tc * C;
  const int64_t nunits = action ? nslots : (int64_t)E * Tc;
  memset(counted, 0, (size_t)nslots);
  for (int64_t i = 0; i < nunits; ++i) adv[i] = ret[i] = 0.0;

  int cap = Tc * C;
  segbuf sg;
  sg.slot = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  sg.boot_slot = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  sg.r = (double*)malloc(sizeof(double) * (size_t)cap);
  sg.v = (double*)malloc(sizeof(double) * (size_t)cap);
  sg.boot = (double*)malloc(sizeof(double) * (size_t)cap);
  sg.a = (double*)malloc(sizeof(double) * (size_t)cap);
  sg.R = (double*)malloc(sizeof(double) * (size_t)cap);
  sg.term = (uint8_t*)malloc((size_t)cap);
  sg.trunc = (uint8_t*)malloc((size_t)cap);

  for (int e = 0; e < E; ++e) {
    sg.n = 0;
    int32_t seg_uid = -1;
    for (int t = 0; t < Tc; ++t) {
      int64_t rec = (int64_t)e * Tc + t;
      if (action) {
        for (int j = 0; j < C; ++j) {
          int64_t s = rec * C + j;
          uint8_t f = ro->flags[s];
          if (!(f & ORC_VALID)) continue;
          int32_t uid = ro->episode_id[s];
          if (sg.n > 0 && uid != seg_uid) flush(&sg, 1, ro, gamma, lambda, adv, ret, 1);
          seg_uid = uid;
          int k = sg.n++;
          sg.slot[k] = s;
          sg.boot_slot[k] = s;
          sg.r[k] = ro->reward[s];
          sg.v[k] = ro->value_vector[s];
          sg.term[k] = (f & ORC_TERMINATED) != 0;
          sg.trunc[k] = (f & ORC_TRUNCATED) != 0;
          counted[s] = 1; /* scatter marks every unit's slot counted */
          if (sg.term[k] || sg.trunc[k]) flush(&sg, 0, ro, gamma, lambda, adv, ret, 1);
        }
      } else {
        int first_valid = -1;
        for (int j = 0; j < C; ++j)
          if (ro->flags[rec * C + j] & ORC_VALID) {
            first_valid = j;
            break;
          }
        if (first_valid < 0) continue; /* fully frozen chunk */
        int32_t lead = ro->episode_id[rec * C + first_valid];
        if (sg.n > 0 && lead != seg_uid) flush(&sg, 1, ro, gamma, lambda, adv, ret, 0);
        seg_uid = lead;
        double reward = 0.0;
        int term = 0, trunc = 0, last_slot = 0;
        for (int j = first_valid; j < C; ++j) {
          int64_t s = rec * C + j;
          uint8_t f = ro->flags[s];
          if (!(f & ORC_VALID) || ro->episode_id[s] != lead) break; /* post-reset tail dropped */
          counted[s] = 1;
          reward += ro->reward[s];
          term = term || (f & ORC_TERMINATED);
          trunc = trunc || (f & ORC_TRUNCATED);
          last_slot = j;
        }
        int k = sg.n++;
        sg.slot[k] = rec;
        sg.boot_slot[k] = rec * C + last_slot;
        sg.r[k] = reward;
        sg.v[k] = ro->value_scalar[rec];
        sg.term[k] = (uint8_t)(term != 0);
        sg.trunc[k] = (uint8_t)(trunc != 0);
        if (term || trunc) flush(&sg, 0, ro, gamma, lambda, adv, ret, 0);
      }
    }
    flush(&sg, 1, ro, gamma, lambda, adv, ret, action);
  }
  free(sg.slot); free(sg.boot_slot); free(sg.r); free(sg.v); free(sg.boot);
  free(sg.a); free(sg.R); free(sg.term); free(sg.trunc);
  return ST_OK;
}

/* optim/update.cpp:14-45 (normalize_advantages): two passes over the counted
 * advantage units (one per record at chunk level, one per counted slot at action
 * level), population std + 1e-8, no-op when fewer than two units. */
static double* unit_at(int chunk, int64_t r, int C, int j, double* adv) {
  return chunk ? &adv[r] : &adv[r * C + j];
}

int orc_normalize_advantages(int E, int Tc, int C, int adv_level, const uint8_t* counted,
                             double* adv) {
  const int64_t R = (int64_t)E * Tc;
  const int chunk = adv_level == ORC_CHUNK;
  double sum = 0.0;
  int64_t n = 0;
  for (int64_t r = 0; r < R; ++r)
    for (int j = 0; j < C; ++j)
      if (counted[r * C + j]) {
        sum += *unit_at(chunk, r, C, j, adv);
        ++n;
        if (chunk) break;
      }
  if (n < 2) return ST_OK;
  double mean = sum / (double)n;
  double var = 0.0;
  for (int64_t r = 0; r < R; ++r)
    for (int j = 0; j < C; ++j)
      if (counted[r * C + j]) {
        double a = *unit_at(chunk, r, C, j, adv);
        var += (a - mean) * (a - mean);
        if (chunk) break;
      }
  var /= (double)n;
  double denom = sqrt(var) + 1e-8;
  for (int64_t r = 0; r < R; ++r)
    for (int j = 0; j < C; ++j)
      if (counted[r * C + j]) {
        double* a = unit_at(chunk, r, C, j, adv);
        *a = (*a - mean) / denom;
        if (chunk) break;
      }
  return ST_OK;
}

/* ---------------------------------------------------------------- losses */

typedef struct {
  double value;
  double dlogprob;
  int clipped;
} surrogate;

/* optim/losses.cpp:32-46 (clipped_surrogate) */
static surrogate clipped_surrogate(double rho, double a, double eps) {
  double unclipped = rho * a;
  double lo = 1.0 - eps, hi = 1.0 + eps;
  double crho = rho < lo ? lo : (hi < rho ? hi : rho); /* std::clamp */
  double clipped = crho * a;
  surrogate s;
  s.clipped = fabs(rho - 1.0) > eps;
  if (unclipped <= clipped) {
    s.value = unclipped;
    s.dlogprob = a * rho;
  } else {
    s.value = clipped;
    s.dlogprob = 0.0;
  }
  return s;
}

/* optim/losses.cpp:62-232 (ppo_loss over every record, grad_out != nullptr) */
int orc_ppo_loss(const orc_rollout* ro, int adv_level, int lp_level, int val_level,
                 const uint8_t* counted, const double* adv, const double* ret,
                 const double* logits, const double* new_values, double clip_eps, double vcoef,
                 double ecoef, double* coeff_lp, double* coeff_ent, double* coeff_val,
                 double* diag) {
  const int E = ro->E, Tc = ro->Tc, C = ro->C, M = ro->M, V = ro->V, P = C * M;
  const int chunk_adv = adv_level == ORC_CHUNK;
  const int64_t R = (int64_t)E * Tc;
  for (int i = 0; i < 7; ++i) diag[i] = 0.0;
  memset(coeff_lp, 0, sizeof(double) * (size_t)(R * P));
  memset(coeff_ent, 0, sizeof(double) * (size_t)(R * P));
  memset(coeff_val, 0, sizeof(double) * (size_t)(val_level == ORC_CHUNK ? R : R * C));

  int64_t n_adv = 0, n_val = 0, n_pos = 0;
  for (int64_t r = 0; r < R; ++r) {
    int cnt = 0;
    for (int j = 0; j < C; ++j) cnt += counted[r * C + j] != 0;
    if (cnt == 0) continue;
    n_adv += chunk_adv ? 1 : cnt;
    n_val += val_level == ORC_CHUNK ? 1 : cnt;
    n_pos += (int64_t)cnt * M;
  }
  if (n_adv == 0) return ST_OK;

  double surrogate_sum = 0.0, value_sq_sum = 0.0, entropy_sum = 0.0, kl_sum = 0.0;
  int64_t clipped_units = 0, lp_units = 0;
  const double inv_adv = 1.0 / (double)n_adv;
  const double inv_val = n_val > 0 ? 1.0 / (double)n_val : 0.0;
  const double inv_pos = n_pos > 0 ? 1.0 / (double)n_pos : 0.0;
  double* lp = (double*)malloc(sizeof(double) * (size_t)P);
  double* H = (double*)malloc(sizeof(double) * (size_t)P);

  for (int64_t r = 0; r < R; ++r) {
    const uint8_t* cnt = counted + r * C;
    int any = 0;
    for (int j = 0; j < C; ++j) any = any || cnt[j];
    if (!any) continue;
    orc_token_stats(P, V, logits + r * P * V, ro->tokens + r * P, lp, H);
    const double* old = ro->old_logprob + r * P;
    double* klp = coeff_lp + r * P;

#define ADD_UNIT(LPN, LPO, ADV, I0, I1, J0, J1)                                      \
  do {                                                                               \
    double rho_ = exp((LPN) - (LPO));                                                \
    surrogate s_ = clipped_surrogate(rho_, (ADV), clip_eps);                         \
    surrogate_sum += s_.value;                                                       \
    ++lp_units;                                                                      \
    if (s_.clipped) ++clipped_units;                                                 \
    kl_sum += (rho_ - 1.0) - ((LPN) - (LPO));                                        \
    double k_ = -inv_adv * s_.dlogprob;                                              \
    for (int i_ = (I0); i_ < (I1); ++i_)                                             \
      for (int j_ = (J0); j_ < (J1); ++j_) klp[i_ * M + j_] += k_;                   \
  } while (0)

    if (chunk_adv && lp_level == ORC_CHUNK) {
      double lpn = 0.0, lpo = 0.0;
      for (int i = 0; i < C; ++i) {
        if (!cnt[i]) continue;
        double an = 0.0, ao = 0.0;
        for (int j = 0; j < M; ++j) {
          an += lp[i * M + j];
          ao += old[i * M + j];
        }
        lpn += an;
        lpo += ao;
      }
      double rho = exp(lpn - lpo);
      surrogate s = clipped_surrogate(rho, adv[r], clip_eps);
      surrogate_sum += s.value;
      ++lp_units;
      if (s.clipped) ++clipped_units;
      kl_sum += (rho - 1.0) - (lpn - lpo);
      double k = -inv_adv * s.dlogprob;
      for (int i = 0; i < C; ++i)
        if (cnt[i])
          for (int j = 0; j < M; ++j) klp[i * M + j] += k;
    } else {
      for (int i = 0; i < C; ++i) {
        if (!cnt[i]) continue;
        double a = chunk_adv ? adv[r] : adv[r * C + i];
        if (lp_level == ORC_ACTION) {
          double an = 0.0, ao = 0.0;
          for (int j = 0; j < M; ++j) {
            an += lp[i * M + j];
            ao += old[i * M + j];
          }
          ADD_UNIT(an, ao, a, i, i + 1, 0, M);
        } else {
          for (int j = 0; j < M; ++j) ADD_UNIT(lp[i * M + j], old[i * M + j], a, i, i + 1, j, j + 1);
        }
      }
    }
#undef ADD_UNIT

    for (int i = 0; i < C; ++i) {
      if (!cnt[i]) continue;
      for (int j = 0; j < M; ++j) {
        entropy_sum += H[i * M + j];
        if (ecoef != 0.0) coeff_ent[r * P + i * M + j] = -ecoef * inv_pos;
      }
    }

    if (val_level == ORC_CHUNK) {
      double err = new_values[r] - ret[r];
      value_sq_sum += err * err;
      coeff_val[r] = vcoef * 2.0 * err * inv_val;
    } else {
      for (int j = 0; j < C; ++j) {
        if (!cnt[j]) continue;
        double err = new_values[r * C + j] - ret[r * C + j];
        value_sq_sum += err * err;
        coeff_val[r * C + j] = vcoef * 2.0 * err * inv_val;
      }
    }
  }
  free(lp);
  free(H);

  double surr = -surrogate_sum * inv_adv;
  double vl = value_sq_sum * inv_val;
  double ent = entropy_sum * inv_pos;
  diag[0] = surr + vcoef * vl - ecoef * ent;
  diag[1] = surr;
  diag[2] = vl;
  diag[3] = ent;
  diag[4] = lp_units > 0 ? (double)clipped_units / (double)lp_units : 0.0;
  diag[5] = lp_units > 0 ? kl_sum / (double)lp_units : 0.0;
  diag[6] = (double)lp_units;
  if (!isfinite(diag[0])) return ST_NON_FINITE;
  return ST_OK;
}

/* ---------------------------------------------------------------- GRPO */

/* advantage/grpo.cpp:9-28 */
int orc_grpo_group_advantage(int g, const double* R, double eps_std, double* adv) {
  if (g < 2) return ST_DEGENERATE_GROUP;
  double mean = 0.0;
  for (int i = 0; i < g; ++i) mean += R[i];
  mean /= (double)g;
  double var = 0.0;
  for (int i = 0; i < g; ++i) var += (R[i] - mean) * (R[i] - mean);
  var /= (double)g;
  double sd = sqrt(var);
  if (sd == 0.0 && eps_std == 0.0) return ST_DEGENERATE_GROUP;
  for (int i = 0; i < g; ++i) adv[i] = (R[i] - mean) / (sd + eps_std);
  return ST_OK;
}

/* advantage/grpo.cpp:30-46 (group_mean_return + the strict filter) */
int orc_success_rate_filter(int g, const double* R, double lower, double upper) {
  double mean = 0.0;
  for (int i = 0; i < g; ++i) mean += R[i];
  mean = g ? mean / (double)g : 0.0;
  return mean > lower && mean < upper;
}

/* advantage/grpo.cpp:48-55 */
void orc_valid_action_mask(int64_t length, int success, int64_t fs, uint8_t* mask) {
  for (int64_t t = 0; t < length; ++t) mask[t] = 1;
  if (success && fs >= 0)
    for (int64_t t = fs + 1; t < length; ++t) mask[t] = 0;
}

/* advantage/grpo.cpp:57-79 */
void orc_length_norm_weights(int64_t length, int success, int64_t fs, int normalized, double* w) {
  if (length <= 0) return;
  for (int64_t t = 0; t < length; ++t) w[t] = 0.0;
  if (!normalized) {
    double u = 1.0 / (double)length;
    for (int64_t t = 0; t < length; ++t) w[t] = u;
    return;
  }
  uint8_t* mask = (uint8_t*)malloc((size_t)length);
  orc_valid_action_mask(length, success, fs, mask);
  int64_t t_succ = 0;
  for (int64_t t = 0; t < length; ++t) t_succ += mask[t] != 0;
  double u = 1.0 / (double)t_succ;
  for (int64_t t = 0; t < length; ++t)
    if (mask[t]) w[t] = u;
  free(mask);
}

static const orc_episodes* g_sort_eps;
static int cmp_key(const void* pa, const void* pb) {
  int a = *(const int*)pa, b = *(const int*)pb;
  const orc_episodes* ep = g_sort_eps;
  if (ep->task_id[a] != ep->task_id[b]) return ep->task_id[a] < ep->task_id[b] ? -1 : 1;
  if (ep->reset_state_id[a] != ep->reset_state_id[b])
    return ep->reset_state_id[a] < ep->reset_state_id[b] ? -1 : 1;
  return a < b ? -1 : (a > b); /* members keep slab.episodes order */
}

/* advantage/assembler.cpp:197-267 (assemble_grpo_batch). Output is per env: the
 * retained trajectory each env owns (group ordinal among retained groups, member
 * index, episode, advantage, group size) plus per-slot membership and weights. */
int orc_assemble_grpo(const orc_rollout* ro, const orc_episodes* eps, int adv_level,
                      int lp_level, int val_level, double eps_std, int apply_filter,
                      double lower, double upper, int length_normalized, int min_group_size,
                      int* groups_total, int* groups_retained, int32_t* env_group,
                      int32_t* env_member, int32_t* env_episode, double* env_adv,
                      int32_t* env_group_size, double* slot_weight, uint8_t* slot_member) {
  int st = orc_validate_granularity(adv_level, lp_level, val_level);
  if (st) return st;
  const int E = ro->E, Tc = ro->Tc, C = ro->C;
  for (int e = 0; e < E; ++e) {
    env_group[e] = env_member[e] = env_episode[e] = -1;
    env_adv[e] = 0.0;
    env_group_size[e] = 0;
  }
  int64_t nslots = (int64_t)E * Tc * C;
  for (int64_t s = 0; s < nslots; ++s) {
    slot_weight[s] = 0.0;
    slot_member[s] = 0;
  }
  int n = 0;
  int* idx = (int*)malloc(sizeof(int) * (size_t)(eps->count + 1));
  for (int i = 0; i < eps->count; ++i)
    if (eps->complete[i] && eps->start_step[i] == 0) idx[n++] = i;
  g_sort_eps = eps;
  qsort(idx, (size_t)n, sizeof(int), cmp_key);

  double* R = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* A = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  int total = 0, retained = 0;
  st = ST_OK;
  for (int b = 0; b < n && st == ST_OK;) {
    int e_ = b;
    while (e_ < n && eps->task_id[idx[e_]] == eps->task_id[idx[b]] &&
           eps->reset_state_id[idx[e_]] == eps->reset_state_id[idx[b]])
      ++e_;
    int g = e_ - b;
    if (g >= min_group_size) {
      ++total;
      for (int i = 0; i < g; ++i) R[i] = eps->total_reward[idx[b + i]];
      if (!apply_filter || orc_success_rate_filter(g, R, lower, upper)) {
        st = orc_grpo_group_advantage(g, R, eps_std, A);
        if (st == ST_OK) {
          for (int i = 0; i < g; ++i) {
            int ep = idx[b + i];
            int env = eps->env_id[ep];
            if (env_group[env] >= 0) { st = ST_ERROR; break; }
            env_group[env] = retained;
            env_member[env] = i;
            env_episode[env] = eps->episode_id[ep];
            env_adv[env] = A[i];
            env_group_size[env] = g;
            int64_t len = eps->length[ep] > 0 ? eps->length[ep] : 0;
            int64_t fs = eps->first_success[ep];
            double* w = (double*)malloc(sizeof(double) * (size_t)(len + 1));
            orc_length_norm_weights(len, fs >= 0, fs, length_normalized, w);
            int64_t k = 0;
            for (int t = 0; t < Tc; ++t)
              for (int j = 0; j < C; ++j) {
                int64_t s = ((int64_t)env * Tc + t) * C + j;
                if (!(ro->flags[s] & ORC_VALID) || ro->episode_id[s] != eps->episode_id[ep]) continue;
                slot_member[s] = 1;
                slot_weight[s] = k < len ? w[k] : 0.0;
                ++k;
              }
            free(w);
          }
          ++retained;
        }
      }
    }
    b = e_;
  }
  *groups_total = total;
  *groups_retained = retained;
  free(idx);
  free(R);
  free(A);
  return st;
}

/* optim/losses.cpp:234-331 (grpo_loss over every retained group, grad_out != nullptr) */
int orc_grpo_loss(const orc_rollout* ro, int lp_level, int groups_retained,
                  const int32_t* env_group, const int32_t* env_member, const double* env_adv,
                  const int32_t* env_group_size, const double* slot_weight,
                  const uint8_t* slot_member, const double* logits, double clip_eps,
                  double* coeff_lp, double* diag) {
  const int E = ro->E, Tc = ro->Tc, C = ro->C, M = ro->M, V = ro->V, P = C * M;
  for (int i = 0; i < 7; ++i) diag[i] = 0.0;
  memset(coeff_lp, 0, sizeof(double) * (size_t)((int64_t)E * Tc * P));
  if (groups_retained == 0) return ST_SKIP_UPDATE;

  /* traversal order: group -> member -> record */
  int* order = (int*)malloc(sizeof(int) * (size_t)(E + 1));
  int no = 0;
  for (int g = 0; g < groups_retained; ++g)
    for (int m = 0;; ++m) {
      int found = -1;
      for (int e = 0; e < E; ++e)
        if (env_group[e] == g && env_member[e] == m) found = e;
      if (found < 0) break;
      order[no++] = found;
    }

  double total = 0.0, kl_sum = 0.0;
  int64_t lp_units = 0, clipped_units = 0;
  const double inv_groups = 1.0 / (double)groups_retained;
  double* lp = (double*)malloc(sizeof(double) * (size_t)P);
  double* H = (double*)malloc(sizeof(double) * (size_t)P);
  for (int oi = 0; oi < no; ++oi) {
    int e = order[oi];
    const double inv_g = 1.0 / (double)env_group_size[e];
    const double a = env_adv[e];
    for (int t = 0; t < Tc; ++t) {
      int64_t r = (int64_t)e * Tc + t;
      int has = 0;
      for (int j = 0; j < C; ++j) has = has || slot_member[r * C + j];
      if (!has) continue; /* not a TrajChunk */
      orc_token_stats(P, V, logits + r * P * V, ro->tokens + r * P, lp, H);
      const double* old = ro->old_logprob + r * P;
      double* klp = coeff_lp + r * P;
      const double* w = slot_weight + r * C;
      const uint8_t* mem = slot_member + r * C;

#define ADD_UNIT(LPN, LPO, W, SLOTS, NS, J0, J1)                                   \
  do {                                                                             \
    double rho_ = exp((LPN) - (LPO));                                              \
    surrogate s_ = clipped_surrogate(rho_, a, clip_eps);                           \
    total += inv_groups * inv_g * (W) * s_.value;                                  \
    ++lp_units;                                                                    \
    if (s_.clipped) ++clipped_units;                                               \
    kl_sum += (rho_ - 1.0) - ((LPN) - (LPO));                                      \
    double k_ = -inv_groups * inv_g * (W) * s_.dlogprob;                           \
    for (int q_ = 0; q_ < (NS); ++q_)                                              \
      for (int j_ = (J0); j_ < (J1); ++j_) klp[(SLOTS)[q_] * M + j_] += k_;        \
  } while (0)

      if (lp_level == ORC_CHUNK) {
        double lpn = 0.0, lpo = 0.0, wsum = 0.0;
        int cov[256], nc = 0;
        for (int j = 0; j < C; ++j) {
          if (!mem[j] || w[j] == 0.0) continue;
          double an = 0.0, ao = 0.0;
          for (int m = 0; m < M; ++m) {
            an += lp[j * M + m];
            ao += old[j * M + m];
          }
          lpn += an;
          lpo += ao;
          wsum += w[j];
          cov[nc++] = j;
        }
        if (nc > 0) ADD_UNIT(lpn, lpo, wsum, cov, nc, 0, M);
      } else {
        for (int j = 0; j < C; ++j) {
          if (!mem[j] || w[j] == 0.0) continue;
          int one[1] = {j};
          if (lp_level == ORC_ACTION) {
            double an = 0.0, ao = 0.0;
            for (int m = 0; m < M; ++m) {
              an += lp[j * M + m];
              ao += old[j * M + m];
            }
            ADD_UNIT(an, ao, w[j], one, 1, 0, M);
          } else {
            for (int m = 0; m < M; ++m) ADD_UNIT(lp[j * M + m], old[j * M + m], w[j], one, 1, m, m + 1);
          }
        }
      }
#undef ADD_UNIT
    }
  }
  free(lp);
  free(H);
  free(order);
  diag[1] = -total;
  diag[0] = diag[1];
  diag[4] = lp_units > 0 ? (double)clipped_units / (double)lp_units : 0.0;
  diag[5] = lp_units > 0 ? kl_sum / (double)lp_units : 0.0;
  diag[6] = (double)lp_units;
  if (!isfinite(diag[0])) return ST_NON_FINITE;
  return ST_OK;
}
