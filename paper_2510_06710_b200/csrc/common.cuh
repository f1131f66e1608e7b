// Shared device/host definitions for the ckrl sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ckrl.h"

namespace ckrl {

constexpr int kWarp = 32;
constexpr int kMaxRanks = 64;
constexpr int kLossThreads = 256;     // 8 warps per CTA in the tile kernel
constexpr int kAsmWarpsPerCta = 2;    // one warp per env in the assembly kernel
constexpr int kMaxLossCtas = 148 * 8; // persistent grid upper bound (partials slots)
constexpr int kGrpoMaxEligible = 8192;

// Advantage moments (n, mean, M2 = sum of squared deviations), merged with Chan's pairwise
// update in a fixed order: deterministic, and free of the one-pass s2/n - m^2 cancellation
// when |mean| >> std (the reference's two-pass whitening, optim/update.cpp:33-43).
struct Moments {
  double n, mean, m2;
};
__host__ __device__ inline Moments mom_merge(const Moments& a, const Moments& b) {
  if (a.n == 0.0) return b;
  if (b.n == 0.0) return a;
  const double n = a.n + b.n;
  const double d = b.mean - a.mean;
  Moments r;
  r.n = n;
  r.mean = a.mean + d * (b.n / n);
  r.m2 = (a.m2 + b.m2) + d * d * (a.n * (b.n / n));
  return r;
}
// Per-thread accumulation without divisions: sums of deviations from the thread's first
// value (exact subtraction for nearby values), converted to moments once at the end.
struct MomAcc {
  double n = 0.0, k = 0.0, s1 = 0.0, s2 = 0.0;
  __host__ __device__ inline void add(double a) {
    if (n == 0.0) k = a;
    const double d = a - k;
    n += 1.0;
    s1 += d;
    s2 += d * d;
  }
  __host__ __device__ inline Moments get() const {
    if (n == 0.0) return Moments{0.0, 0.0, 0.0};
    const double q = s1 / n;
    double m2 = s2 - s1 * q;
    if (m2 < 0.0) m2 = 0.0;
    return Moments{n, k + q, m2};
  }
};

// Per-rank record of everything the loss needs from the advantage phase before it
// can scale a single coefficient: whitening moments over the counted advantage units
// (optim/update.cpp:33-43) and the loss normalisers n_adv / n_val / n_pos
// (optim/losses.cpp:75-87) or the retained GRPO group count (losses.cpp:246).
// Fixed 64-byte layout so ranks can all-gather it with one NCCL call.
struct StatsRecord {
  double mean;          // mean of the rank's counted advantage units (fp64)
  double m2;            // sum of squared deviations from it
  int64_t flags;        // STATS_WHITENED: advantages were whitened in place (normalize_advantages)
  int64_t n_adv;        // advantage units (the moments' n)
  int64_t n_val;
  int64_t n_pos;
  int64_t groups_retained;
  int64_t status;       // device-detected error (DegenerateGroup, ...)
};
static_assert(sizeof(StatsRecord) == 64, "stats record must stay 64 bytes");
enum { STATS_WHITENED = 1 };

// Raw loss sums (reduced across CTAs, then across ranks) before normalisation.
enum { RAW_SURR = 0, RAW_VALSQ, RAW_ENT, RAW_KL, RAW_CLIPPED, RAW_LPUNITS, RAW_COUNT = 8 };

// Whitening parameters from merged moments: mean, population std + 1e-8 (update.cpp:33-43).
__host__ __device__ inline void whitening(const Moments& m, double* mean, double* denom) {
  const double var = m.n > 0.0 ? m.m2 / m.n : 0.0;
  *mean = m.n > 0.0 ? m.mean : 0.0;
  *denom = sqrt(var) + 1e-8;
}
// Fixed rank-order merge of `world` records.
__host__ __device__ inline Moments merge_records(const StatsRecord* r, int world) {
  Moments m{0.0, 0.0, 0.0};
  for (int i = 0; i < world; ++i) m = mom_merge(m, Moments{(double)r[i].n_adv, r[i].mean, r[i].m2});
  return m;
}

// Workspace carve-up (all offsets 256-byte aligned). Must match ckrl_workspace_bytes.
struct WsLayout {
  size_t stats_local;   // StatsRecord
  size_t stats_all;     // StatsRecord[world] (last: the only world-dependent region)
  size_t tickets;       // uint32[8] last-block counters (self-resetting)
  size_t loss_raw;      // double[RAW_COUNT]
  size_t asm_partials;  // AsmPartial per assembly CTA
  size_t loss_partials; // double[RAW_COUNT] per loss CTA
  size_t grpo_env;      // per-env int32 len, fs (GRPO assembly scratch)
  size_t total;
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct AsmPartial {
  Moments m;
  double n_pos;  // counted slots
};

__host__ __device__ inline WsLayout ws_layout(int E, int world) {
  WsLayout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t at = off;
    off = align256(off + bytes);
    return at;
  };
  int asm_ctas = (E + kAsmWarpsPerCta - 1) / kAsmWarpsPerCta;
  if (asm_ctas < kMaxLossCtas) asm_ctas = kMaxLossCtas;  // also the fused step's CTA partials
  // every world-independent region first (fixed offsets whatever `world` a workspace is
  // used with); the all-gathered records last
  L.stats_local = take(sizeof(StatsRecord));
  L.tickets = take(sizeof(uint32_t) * 8);
  L.loss_raw = take(sizeof(double) * RAW_COUNT);
  L.asm_partials = take(sizeof(AsmPartial) * (size_t)asm_ctas);
  L.loss_partials = take(sizeof(double) * RAW_COUNT * kMaxLossCtas);
  L.grpo_env = take(sizeof(int32_t) * 2 * (size_t)(E < 1 ? 1 : E));
  L.stats_all = take(sizeof(StatsRecord) * (size_t)(world < 1 ? 1 : world));
  L.total = off;
  return L;
}

enum { TICKET_ASM = 0, TICKET_LOSS = 1, TICKET_GRID = 2, TICKET_GEN = 3, TICKET_NORM = 4 };

// ---- warp helpers ----------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

}  // namespace ckrl
