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

// ---- cross-rank exchange over peer memory (NVLink P2P stores) ----------------------------
// Every rank owns one exchange buffer in its own HBM: a header (the rank's step epoch) and,
// per epoch parity, one slot per rank. A producer (the assembly's last CTA for the stats
// record, the loss's last CTA for the raw loss sums) stores its data into slot [p][rank] of
// EVERY rank's buffer, fences at system scope, then stores the epoch into that slot's flag;
// consumers spin (acquire, system scope) on the flags of their own buffer only, so every
// wait is a local-HBM poll and every transfer a remote store. Two parities: rank q can only
// reach epoch e+2's stores after every rank has finished reading epoch e (the loss tail of
// e+1 needs every rank's e+1 sums, posted after its e reads).
struct ExSlot {
  StatsRecord rec;                 // the producer rank's stats record
  double raw[RAW_COUNT];           // its raw loss sums (before normalisation)
  unsigned long long stats_epoch;  // == epoch once rec is visible
  unsigned long long raw_epoch;    // == epoch once raw is visible
  unsigned long long pad[14];
};
static_assert(sizeof(ExSlot) == 256, "exchange slot is 256 bytes");
constexpr size_t kExHeader = 256;  // [0]: the rank's epoch counter (u64)
__host__ __device__ inline size_t ex_buffer_bytes(int world) {
  return kExHeader + 2 * (size_t)world * sizeof(ExSlot);
}
// Kernel-side view of a rank's exchange (world == 0: single rank, no exchange).
struct ExchangeView {
  char* const* peers;          // device array [world]: every rank's exchange buffer (peer-mapped)
  char* local;                 // this rank's buffer (== peers[rank])
  int world, rank;
};
__host__ __device__ inline ExSlot* ex_slots(char* buf, int world, unsigned long long epoch) {
  return reinterpret_cast<ExSlot*>(buf + kExHeader) + (size_t)(epoch & 1ull) * world;
}

#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ex_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr unsigned long long kExTimeoutNs = 20ull * 1000 * 1000 * 1000;  // a peer that never posts
// Spin until *flag == e (own HBM, system-scope acquire); false after kExTimeoutNs.
__device__ inline bool ex_wait(const unsigned long long* flag, unsigned long long e) {
  if (ld_acquire_sys(flag) == e) return true;
  const unsigned long long t0 = ex_now();
  for (unsigned it = 1;; ++it) {
    if (ld_acquire_sys(flag) == e) return true;
    if ((it & 255u) == 0 && ex_now() - t0 > kExTimeoutNs) return false;
    __nanosleep(64);
  }
}
// Assembly side (one thread, after the rank's record is final): bump the rank's epoch, note it
// in the workspace (`ws_epoch`: the loss of this batch reads it there, so a batch's assembly
// and an earlier batch's loss may run concurrently), store the record into slot [p][rank] of
// every rank's buffer, then release the flags. Callers keep an assembly at most one batch
// ahead of the losses (it starts after the loss two batches back has completed), which is
// what two parities need.
static __device__ __noinline__ void ex_publish_stats(ExchangeView x, StatsRecord r, uint32_t* ws_epoch) {
  unsigned long long* ep = reinterpret_cast<unsigned long long*>(x.local);
  const unsigned long long e = *ep + 1;
  *ep = e;
  *ws_epoch = (uint32_t)e;
  for (int q = 0; q < x.world; ++q) ex_slots(x.peers[q], x.world, e)[x.rank].rec = r;
  __threadfence_system();
  for (int q = 0; q < x.world; ++q) st_release_sys(&ex_slots(x.peers[q], x.world, e)[x.rank].stats_epoch, e);
}
// The loss's last CTA (one thread): post the rank's raw sums, wait for every rank's, and sum
// them in rank order (identical on every rank). False on a peer timeout.
static __device__ __noinline__ bool ex_allreduce_raw(ExchangeView x, unsigned long long e, double* raw) {
  for (int q = 0; q < x.world; ++q) {
    ExSlot* s = ex_slots(x.peers[q], x.world, e) + x.rank;
    for (int i = 0; i < RAW_COUNT; ++i) s->raw[i] = raw[i];
  }
  __threadfence_system();
  for (int q = 0; q < x.world; ++q) st_release_sys(&ex_slots(x.peers[q], x.world, e)[x.rank].raw_epoch, e);
  ExSlot* mine = ex_slots(x.local, x.world, e);
  double tot[RAW_COUNT] = {0, 0, 0, 0, 0, 0, 0, 0};
  bool ok = true;
  for (int q = 0; q < x.world && ok; ++q) {
    ok = ex_wait(&mine[q].raw_epoch, e);
    for (int i = 0; i < RAW_COUNT; ++i) tot[i] += ok ? mine[q].raw[i] : 0.0;
  }
  for (int i = 0; i < RAW_COUNT; ++i) raw[i] = tot[i];
  return ok;
}
#endif

// Whitening parameters from merged moments: mean, population std + 1e-8 (update.cpp:33-43).
__host__ __device__ inline void whitening(const Moments& m, double* mean, double* denom) {
  const double var = m.n > 0.0 ? m.m2 / m.n : 0.0;
  *mean = m.n > 0.0 ? m.mean : 0.0;
  *denom = sqrt(var) + 1e-8;
}
// Fixed rank-order merge of `world` records `stride` bytes apart (contiguous records, or the
// stats records of a rank's exchange slots).
__host__ __device__ inline const StatsRecord& rec_at(const StatsRecord* r, size_t stride, int i) {
  return *reinterpret_cast<const StatsRecord*>(reinterpret_cast<const char*>(r) + stride * (size_t)i);
}
__host__ __device__ inline Moments merge_records(const StatsRecord* r, int world,
                                                 size_t stride = sizeof(StatsRecord)) {
  Moments m{0.0, 0.0, 0.0};
  for (int i = 0; i < world; ++i) {
    const StatsRecord& q = rec_at(r, stride, i);
    m = mom_merge(m, Moments{(double)q.n_adv, q.mean, q.m2});
  }
  return m;
}

// Workspace carve-up (all offsets 256-byte aligned). Must match ckrl_workspace_bytes.
struct WsLayout {
  size_t stats_local;   // StatsRecord
  size_t tickets;       // uint32[8] last-block counters (self-resetting)
  size_t loss_raw;      // double[RAW_COUNT]
  size_t asm_partials;  // AsmPartial per assembly CTA
  size_t loss_partials; // double[RAW_COUNT] per loss CTA
  size_t grpo_env;      // per-env int32 len, fs (GRPO assembly scratch)
  size_t grpo_sort;     // GroupKey sort scratch when more episodes are eligible than fit in
                        // shared memory: keys u64 / index / group id [pow2 >= E], starts [E+1]
  size_t total;
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct AsmPartial {
  Moments m;
  double n_pos;  // counted slots
};

__host__ __device__ inline int pow2_at_least(int n) {
  int c = 1;
  while (c < n) c <<= 1;
  return c;
}
__host__ __device__ inline size_t grpo_sort_bytes(int E) {
  return (size_t)pow2_at_least(E) * 16 + sizeof(int32_t) * ((size_t)E + 1);
}

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
  // no region depends on `world`: the cross-rank records live in the communicator's
  // exchange buffer, so one workspace serves any world size
  (void)world;
  L.stats_local = take(sizeof(StatsRecord));
  L.tickets = take(sizeof(uint32_t) * 8);
  L.loss_raw = take(sizeof(double) * RAW_COUNT);
  L.asm_partials = take(sizeof(AsmPartial) * (size_t)asm_ctas);
  L.loss_partials = take(sizeof(double) * RAW_COUNT * kMaxLossCtas);
  L.grpo_env = take(sizeof(int32_t) * 2 * (size_t)(E < 1 ? 1 : E));
  L.grpo_sort = take(E > kGrpoMaxEligible ? grpo_sort_bytes(E) : 0);
  L.total = off;
  return L;
}

enum { TICKET_ASM = 0, TICKET_LOSS = 1, TICKET_GRID = 2, TICKET_GEN = 3, TICKET_NORM = 4,
       TICKET_EPOCH = 6 };  // (not a ticket) the exchange epoch of the workspace's last assembly

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
