// GAE as a warp-segmented reverse affine scan + the unit accessors of PPO assembly.
// Shared by the standalone assembly kernel (advantage.cu) and the fused step kernel
// (loss.cu). Reference: advantage/gae.cpp:7-37, advantage/assembler.cpp:33-195.
#pragma once

#include "common.cuh"

namespace ckrl {

// One advantage-level unit as the GAE recurrence sees it.
struct Unit {
  bool is_unit;  // false: transparent item (invalid slot / fully frozen chunk)
  bool term, trunc;
  int32_t uid;   // segment key (episode id); units of one segment are contiguous
  double r, v, boot;
  int counted_slots;
  int first;     // chunk level: first valid slot of the record (its counted run starts here)
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
// Per-lane GAE statistics: advantage-unit moments (shifted sums per lane, merged with Chan's
// update in a fixed tree order: deterministic) and the counted-slot count.
struct GaeSums {
  Moments m;
  double counted_slots;
};
__device__ __forceinline__ GaeSums gae_sums_reduce(const MomAcc& acc, double counted_slots) {
  GaeSums st{acc.get(), counted_slots};
  for (int off = 16; off > 0; off >>= 1) {  // fixed-shape tree over lanes (deterministic)
    Moments o{__shfl_down_sync(0xffffffffu, st.m.n, off), __shfl_down_sync(0xffffffffu, st.m.mean, off),
              __shfl_down_sync(0xffffffffu, st.m.m2, off)};
    st.m = mom_merge(st.m, o);
    st.counted_slots += __shfl_down_sync(0xffffffffu, st.counted_slots, off);
  }
  return st;  // valid in lane 0
}

template <class Acc>
__device__ __noinline__ GaeSums warp_gae(const Acc& acc, int n_items, double gamma, double lambda) {
  const int lane = threadIdx.x & 31;
  const int per = (n_items + 31) / 32;
  const int lo = min(n_items, lane * per), hi = min(n_items, lo + per);
  const double gl = __dmul_rn(gamma, lambda);

  // Phase 1: first unit of my range, then the nearest such head to my right.
  bool h_has = false;
  int32_t h_uid = 0;
  double h_v = 0.0;
  for (int i = lo; i < hi; ++i) {
    const Unit u = acc.load(i);
    if (u.is_unit) {
      h_has = true;
      h_uid = u.uid;
      h_v = u.v;
      break;
    }
  }
  for (int off = 1; off < 32; off <<= 1) {
    const bool o_has = __shfl_down_sync(0xffffffffu, h_has, off);
    const int32_t o_uid = __shfl_down_sync(0xffffffffu, h_uid, off);
    const double o_v = __shfl_down_sync(0xffffffffu, h_v, off);
    if (!h_has && lane + off < 32) {
      h_has = o_has;
      h_uid = o_uid;
      h_v = o_v;
    }
  }
  bool nx_has0 = __shfl_down_sync(0xffffffffu, h_has, 1);
  const int32_t nx_uid0 = __shfl_down_sync(0xffffffffu, h_uid, 1);
  const double nx_v0 = __shfl_down_sync(0xffffffffu, h_v, 1);
  if (lane == 31) nx_has0 = false;

  // Phases 2 (compose my range's affine map) and 4 (replay with the exact incoming
  // advantage) share one reverse walk; pass 0 composes, pass 1 writes.
  double P = 0.0, Q = 1.0, a_next = 0.0;
  MomAcc mom;
  double counted_slots = 0.0;
  for (int pass = 0; pass < 2; ++pass) {
    bool nx_has = nx_has0;
    int32_t nx_uid = nx_uid0;
    double nx_v = nx_v0;
    for (int i = hi - 1; i >= lo; --i) {
      const Unit u = acc.load(i);
      if (!u.is_unit) {
        if (pass) acc.store_empty(i);
        continue;
      }
      const bool seg_end = u.term || u.trunc || !nx_has || nx_uid != u.uid;
      const double vnext = u.term ? 0.0 : ((u.trunc || seg_end) ? u.boot : nx_v);
      const double delta = __dadd_rn(__dadd_rn(u.r, __dmul_rn(gamma, vnext)), -u.v);
      if (pass == 0) {
        const double c = seg_end ? 0.0 : gl;
        P = __dadd_rn(delta, __dmul_rn(c, P));
        Q = __dmul_rn(c, Q);
      } else {
        const double a = __dadd_rn(delta, __dmul_rn(gl, seg_end ? 0.0 : a_next));
        acc.store(i, u, a, __dadd_rn(a, u.v));
        mom.add(a);
        counted_slots += u.counted_slots;
        a_next = a;
      }
      nx_has = true;
      nx_uid = u.uid;
      nx_v = u.v;
    }
    if (pass == 0) {
      // Phase 3: inclusive suffix scan of the lanes' maps, G_l = F_l o G_{l+1}.
      for (int off = 1; off < 32; off <<= 1) {
        const double oP = __shfl_down_sync(0xffffffffu, P, off);
        const double oQ = __shfl_down_sync(0xffffffffu, Q, off);
        if (lane + off < 32) {
          P = __dadd_rn(P, __dmul_rn(Q, oP));
          Q = __dmul_rn(Q, oQ);
        }
      }
      a_next = __shfl_down_sync(0xffffffffu, P, 1);
      if (lane == 31) a_next = 0.0;
    }
  }
  return gae_sums_reduce(mom, counted_slots);
}

// Register-resident variant: lane l owns items [l*K, l*K+K), all loaded once up front
// (independent loads: one memory round trip), then the same scan as warp_gae.
template <int K, class Acc>
__device__ __noinline__ GaeSums warp_gae_regs(const Acc& acc, int n_items, double gamma, double lambda) {
  const int lane = threadIdx.x & 31;
  const int lo = lane * K;
  const double gl = __dmul_rn(gamma, lambda);
  Unit u[K];
#pragma unroll
  for (int q = 0; q < K; ++q) {
    if (lo + q < n_items) {
      u[q] = acc.load(lo + q);
    } else {
      u[q].is_unit = false;
    }
  }
  bool h_has = false;
  int32_t h_uid = 0;
  double h_v = 0.0;
#pragma unroll
  for (int q = K - 1; q >= 0; --q)
    if (u[q].is_unit) {
      h_has = true;
      h_uid = u[q].uid;
      h_v = u[q].v;
    }
  for (int off = 1; off < 32; off <<= 1) {
    const bool o_has = __shfl_down_sync(0xffffffffu, h_has, off);
    const int32_t o_uid = __shfl_down_sync(0xffffffffu, h_uid, off);
    const double o_v = __shfl_down_sync(0xffffffffu, h_v, off);
    if (!h_has && lane + off < 32) {
      h_has = o_has;
      h_uid = o_uid;
      h_v = o_v;
    }
  }
  bool nx_has0 = __shfl_down_sync(0xffffffffu, h_has, 1);
  const int32_t nx_uid0 = __shfl_down_sync(0xffffffffu, h_uid, 1);
  const double nx_v0 = __shfl_down_sync(0xffffffffu, h_v, 1);
  if (lane == 31) nx_has0 = false;
  // per-item seg_end / delta (reverse, within the lane)
  double delta[K];
  bool segend[K];
  {
    bool nx_has = nx_has0;
    int32_t nx_uid = nx_uid0;
    double nx_v = nx_v0;
#pragma unroll
    for (int q = K - 1; q >= 0; --q) {
      delta[q] = 0.0;
      segend[q] = true;
      if (!u[q].is_unit) continue;
      segend[q] = u[q].term || u[q].trunc || !nx_has || nx_uid != u[q].uid;
      const double vnext = u[q].term ? 0.0 : ((u[q].trunc || segend[q]) ? u[q].boot : nx_v);
      delta[q] = __dadd_rn(__dadd_rn(u[q].r, __dmul_rn(gamma, vnext)), -u[q].v);
      nx_has = true;
      nx_uid = u[q].uid;
      nx_v = u[q].v;
    }
  }
  double P = 0.0, Q = 1.0;
#pragma unroll
  for (int q = K - 1; q >= 0; --q)
    if (u[q].is_unit) {
      const double c = segend[q] ? 0.0 : gl;
      P = __dadd_rn(delta[q], __dmul_rn(c, P));
      Q = __dmul_rn(c, Q);
    }
  for (int off = 1; off < 32; off <<= 1) {
    const double oP = __shfl_down_sync(0xffffffffu, P, off);
    const double oQ = __shfl_down_sync(0xffffffffu, Q, off);
    if (lane + off < 32) {
      P = __dadd_rn(P, __dmul_rn(Q, oP));
      Q = __dmul_rn(Q, oQ);
    }
  }
  double a_next = __shfl_down_sync(0xffffffffu, P, 1);
  if (lane == 31) a_next = 0.0;
  MomAcc mom;
  double counted_slots = 0.0;
#pragma unroll
  for (int q = K - 1; q >= 0; --q) {
    if (lo + q >= n_items) continue;
    if (!u[q].is_unit) {
      acc.store_empty(lo + q);
      continue;
    }
    const double a = __dadd_rn(delta[q], __dmul_rn(gl, segend[q] ? 0.0 : a_next));
    acc.store(lo + q, u[q], a, __dadd_rn(a, u[q].v));
    mom.add(a);
    counted_slots += u[q].counted_slots;
    a_next = a;
  }
  return gae_sums_reduce(mom, counted_slots);
}

// Dispatch on items per lane: register-resident for <= 4 items per lane, else re-reading.
template <class Acc>
__device__ __forceinline__ GaeSums env_gae(const Acc& acc, int n_items, double gamma, double lambda) {
  if (n_items <= 32) return warp_gae_regs<1>(acc, n_items, gamma, lambda);
  if (n_items <= 128) return warp_gae_regs<4>(acc, n_items, gamma, lambda);
  return warp_gae(acc, n_items, gamma, lambda);
}

// Thread-per-env GAE for short item lists: one reverse walk, the reference's exact
// operation order (gae.cpp:21-35 per segment) — bit-identical advantages — and no
// shuffles. Used when an env has at most kSerialItems items.
constexpr int kSerialItems = 256;

template <class Acc>
__device__ __forceinline__ GaeSums serial_gae(const Acc& acc, int n_items, double gamma, double lambda) {
  const double gl = __dmul_rn(gamma, lambda);
  MomAcc mom;
  double counted_slots = 0.0;
  bool nx_has = false;
  int32_t nx_uid = 0;
  double nx_v = 0.0, a_next = 0.0;
  for (int i = n_items - 1; i >= 0; --i) {
    const Unit u = acc.load(i);
    if (!u.is_unit) {
      acc.store_empty(i);
      continue;
    }
    const bool seg_end = u.term || u.trunc || !nx_has || nx_uid != u.uid;
    const double vnext = u.term ? 0.0 : ((u.trunc || seg_end) ? u.boot : nx_v);
    const double delta = __dadd_rn(__dadd_rn(u.r, __dmul_rn(gamma, vnext)), -u.v);
    const double a = __dadd_rn(delta, __dmul_rn(gl, seg_end ? 0.0 : a_next));
    acc.store(i, u, a, __dadd_rn(a, u.v));
    mom.add(a);
    counted_slots += u.counted_slots;
    a_next = a;
    nx_has = true;
    nx_uid = u.uid;
    nx_v = u.v;
  }
  return GaeSums{mom.get(), counted_slots};  // per thread (the caller merges)
}

// ---- accessors ------------------------------------------------------------------
// 8-slot records can be read with vector loads when the arrays are 16-byte aligned (the
// record offset, 8 slots, keeps every array's records 16-byte aligned).
__device__ __forceinline__ bool vec_ok(const ckrl_rollout& ro) {
  return ((reinterpret_cast<uintptr_t>(ro.flags) & 7) | (reinterpret_cast<uintptr_t>(ro.episode_id) & 15) |
          (reinterpret_cast<uintptr_t>(ro.reward) & 15) | (reinterpret_cast<uintptr_t>(ro.bootstrap) & 15)) == 0;
}
struct ChunkAcc {  // chunk-level units: one per record (assembler.cpp:158-190)
  const ckrl_rollout ro;
  int e;
  uint8_t* counted;
  double* adv;
  double* ret;
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
      if (C == kC && vec_ok(ro)) {
        // a record's 8 slots are contiguous in every array: 7 vector loads instead of 32
        const uint2 fw = __ldg(reinterpret_cast<const uint2*>(ro.flags + s0));
        const int4 i0 = __ldg(reinterpret_cast<const int4*>(ro.episode_id + s0));
        const int4 i1 = __ldg(reinterpret_cast<const int4*>(ro.episode_id + s0) + 1);
        const float4 r0 = __ldg(reinterpret_cast<const float4*>(ro.reward + s0));
        const float4 r1 = __ldg(reinterpret_cast<const float4*>(ro.reward + s0) + 1);
        const float4 b0 = __ldg(reinterpret_cast<const float4*>(ro.bootstrap + s0));
        const float4 b1 = __ldg(reinterpret_cast<const float4*>(ro.bootstrap + s0) + 1);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          f[j] = (uint8_t)(fw.x >> (8 * j));
          f[j + 4] = (uint8_t)(fw.y >> (8 * j));
        }
        id[0] = i0.x; id[1] = i0.y; id[2] = i0.z; id[3] = i0.w;
        id[4] = i1.x; id[5] = i1.y; id[6] = i1.z; id[7] = i1.w;
        rw[0] = r0.x; rw[1] = r0.y; rw[2] = r0.z; rw[3] = r0.w;
        rw[4] = r1.x; rw[5] = r1.y; rw[6] = r1.z; rw[7] = r1.w;
        bt[0] = b0.x; bt[1] = b0.y; bt[2] = b0.z; bt[3] = b0.w;
        bt[4] = b1.x; bt[5] = b1.y; bt[6] = b1.z; bt[7] = b1.w;
      } else {
#pragma unroll
        for (int j = 0; j < kC; ++j)
          if (j < C) {
            f[j] = ro.flags[s0 + j];
            id[j] = ro.episode_id[s0 + j];
            rw[j] = ro.reward[s0 + j];
            bt[j] = ro.bootstrap[s0 + j];
          }
      }
      int first = -1;
#pragma unroll
      for (int j = kC - 1; j >= 0; --j)
        if (j < C && (f[j] & CKRL_FLAG_VALID)) first = j;
      if (first < 0) return u;  // fully frozen chunk
      u.is_unit = true;
      u.first = first;
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
    u.first = first;
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
    adv[rec] = a;
    ret[rec] = R;
    // counted = the leading episode's contiguous valid prefix from the first valid slot
    if (C == 8 && (reinterpret_cast<uintptr_t>(counted) & 7) == 0) {
      uint64_t w = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        w |= (uint64_t)(j >= u.first && j < u.first + u.counted_slots ? 1 : 0) << (8 * j);
      *reinterpret_cast<uint64_t*>(counted + rec * 8) = w;
      return;
    }
    for (int j = 0; j < C; ++j) counted[rec * C + j] = (j >= u.first && j < u.first + u.counted_slots) ? 1 : 0;
  }
  __device__ void store_empty(int t) const {
    const int C = ro.chunk_len;
    const int64_t rec = (int64_t)e * ro.num_chunks + t;
    adv[rec] = 0.0;
    ret[rec] = 0.0;
    for (int j = 0; j < C; ++j) counted[rec * C + j] = 0;
  }
};

struct ActionAcc {  // action-level units: one per valid slot (assembler.cpp:112-146)
  const ckrl_rollout ro;
  int e;
  uint8_t* counted;
  double* adv;
  double* ret;
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
    adv[s] = a;
    ret[s] = R;
    counted[s] = 1;
  }
  __device__ void store_empty(int i) const {
    const int64_t s = (int64_t)e * ro.num_chunks * ro.chunk_len + i;
    adv[s] = 0.0;
    ret[s] = 0.0;
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

}  // namespace ckrl
