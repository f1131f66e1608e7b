// Row N2 — the hidden -> action-bin projection on the 5th-generation tensor cores, fused with
// the per-token statistics of the action-token kernel.
//
// The reference forms every position's logits as logits = W_pol . h + b_pol
// (PolicyNet::logits_from_feature, policy/policy_net.cpp:265-274: `matvec` over the trunk
// feature h of width H, then the bias) and reduces them with log_softmax
// (policy_net.cpp:90-102) to the sampled token's log-prob and the entropy
// (evaluate_chunk, policy_net.cpp:333-357). Here that is one persistent sm_100a kernel:
//
//   [rows x H] bf16 features  x  [256 x H] bf16 W_pol  ->  [128 x 256] f32 tiles in TMEM
//
//   warps 0 / 10       TMA producers (one lane each): 2-D tensor copies (128-byte swizzle) per
//                      64-wide K step — warp 0 the 128-row feature slabs into a 7-stage ring
//                      (the HBM stream, 112 KB in flight), warp 10 the 256-row W_pol slabs
//                      (L2-resident) into a 3-stage ring; mbarrier complete_tx.
//   warp 1 (one lane)  MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128 N=256 K=16, into
//                      one of two 256-column TMEM accumulators (512 columns: the epilogue of
//                      tile i overlaps the MMAs of tile i+1); tcgen05.commit frees the smem
//                      stage and, after the last K step, hands the accumulator to the epilogue.
//   warps 2-9          epilogue: TMEM lane = tile row; warp w reads lane quarter w % 4 and one
//                      128-bin column half (tcgen05.ld 32x32b.x32, the next load in flight);
//                      bias, max, sum of exp2, the entropy sum and the sampled token's logit in
//                      registers, the two halves combined through shared memory; log-prob and
//                      entropy finished in fp64; the row record {lp, H} (and optionally the
//                      logits) written straight to HBM.
//
// Nothing of the 256-bin row is ever written unless asked for: the loss consumes the
// 16-byte row records (CKRL_DTYPE_TOKEN_ROWS), so the step's HBM traffic is the features
// (2H bytes per position) plus 16 bytes, against 2H + 1 KB + 1 KB for projection -> logits
// in HBM -> token kernel.
#include <cuda.h>

#include "kernels.h"

namespace ckrl {
namespace {

constexpr int kPM = 128;  // positions per tile (UMMA M; TMEM lanes)
constexpr int kPN = 256;  // bins (UMMA N; TMEM columns per accumulator)
constexpr int kPK = 64;   // K per stage: one 128-byte swizzle atom of bf16
#ifndef CKRL_PROJ_L2PROMO
#define CKRL_PROJ_L2PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
#ifndef CKRL_PROJ_A_EVICT
#define CKRL_PROJ_A_EVICT "evict_first"
#endif
#ifndef CKRL_PROJ_STA
#define CKRL_PROJ_STA 7
#endif
#ifndef CKRL_PROJ_STB
#define CKRL_PROJ_STB 3
#endif
constexpr int kStA = CKRL_PROJ_STA;  // feature stages (16 KB): the HBM stream, deeper in flight
constexpr int kStB = CKRL_PROJ_STB;  // W_pol stages (32 KB): served from L2
constexpr uint32_t kABytes = kPM * kPK * 2;  // 16 KB
constexpr uint32_t kBBytes = kPN * kPK * 2;  // 32 KB
constexpr int kProjThreads = 352;            // A producer, MMA, 8 epilogue warps, B producer
constexpr uint32_t kTmemCols = 512;          // two 256-column accumulators
constexpr size_t kProjSmem = 1024 /*align slack*/ + kStA * (size_t)kABytes + kStB * (size_t)kBBytes + 1024 /*bias*/ +
                             256 /*barriers*/ + 5 * 128 * 4 /*half exchange*/;

// Instruction descriptor (kind::f16): D f32, A/B bf16, both K-major, N = 256, M = 128.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kPN >> 3) << 17) |
                            ((uint32_t)(kPM >> 4) << 24);

struct ProjArgs {
  int64_t rows;
  int64_t n_tiles;
  int n_kb;              // H / 64
  const float* b_pol;    // [256]
  const void* tokens;    // [rows] u8 / i32
  int tok_i32;
  ckrl_token_row* out;   // [rows] {lp, H} (nullable)
  double* lp;            // [rows] (nullable)
  float* ent;            // [rows] (nullable)
  void* logits;          // [rows][256] (nullable)
  int logits_bf16;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                       uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar)), "l"(policy)
      : "memory");
}
// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row core groups 1024 B apart
// (SBO), LBO unused (1), sm_100 descriptor version 1, layout SWIZZLE_128B (2).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// 32 consecutive TMEM columns of this warp's 32 lanes (one f32 per lane per column), issued
// asynchronously: the registers are valid after tmem_wait() (tcgen05.wait::ld waits for every
// load this thread has issued).
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, float (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
        "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]),
        "=f"(v[16]), "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]), "=f"(v[21]), "=f"(v[22]), "=f"(v[23]),
        "=f"(v[24]), "=f"(v[25]), "=f"(v[26]), "=f"(v[27]), "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
      : "r"(taddr));
}
// tcgen05.wait::ld with the just-loaded registers as in/out operands, so no use of them can be
// scheduled above the wait
__device__ __forceinline__ void tmem_wait(float (&v)[32]) {
  asm volatile(
      "tcgen05.wait::ld.sync.aligned;"
      : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]), "+f"(v[7]),
        "+f"(v[8]), "+f"(v[9]), "+f"(v[10]), "+f"(v[11]), "+f"(v[12]), "+f"(v[13]), "+f"(v[14]), "+f"(v[15]),
        "+f"(v[16]), "+f"(v[17]), "+f"(v[18]), "+f"(v[19]), "+f"(v[20]), "+f"(v[21]), "+f"(v[22]), "+f"(v[23]),
        "+f"(v[24]), "+f"(v[25]), "+f"(v[26]), "+f"(v[27]), "+f"(v[28]), "+f"(v[29]), "+f"(v[30]), "+f"(v[31])
      :
      : "memory");
}
__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ float fast_ex2(float y) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(y));
  return r;
}

constexpr double kLn2 = 0.6931471805599453094;
constexpr float kLog2e = 1.4426950408889634f;

__global__ void __launch_bounds__(kProjThreads, 1)
    proj_stats_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                      ProjArgs a) {
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte alignment for the 128-byte swizzle atoms
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* sa = base;                                   // kStA x 16 KB
  unsigned char* sb = base + kStA * kABytes;                  // kStB x 32 KB
  float* s_bias = reinterpret_cast<float*>(sb + kStB * kBBytes);
  uint64_t* full_a = reinterpret_cast<uint64_t*>(s_bias + kPN);
  uint64_t* empty_a = full_a + kStA;
  uint64_t* full_b = empty_a + kStA;
  uint64_t* empty_b = full_b + kStB;
  uint64_t* tfull = empty_b + kStB;  // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty + 2);
  float (*s_m)[kPM] = reinterpret_cast<float (*)[kPM]>(s_bias + kPN + 64);   // [2][128] half maxima
  float (*s_st)[kPM] = reinterpret_cast<float (*)[kPM]>(s_bias + kPN + 64 + 2 * kPM);  // [3][128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kPN; i += kProjThreads) s_bias[i] = a.b_pol ? a.b_pol[i] : 0.0f;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStA; ++s) {
      bar_init(&full_a[s], 1);
      bar_init(&empty_a[s], 1);
    }
    for (int s = 0; s < kStB; ++s) {
      bar_init(&full_b[s], 1);
      bar_init(&empty_b[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      bar_init(&tfull[i], 1);
      bar_init(&tempty[i], 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(s_tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == 0 || warp == 10) {
    if (lane == 0) {  // ---- TMA producers: warp 0 the feature slabs, warp 10 the W_pol slabs
      const bool is_a = warp == 0;
      uint64_t pol;
      if (is_a)
        asm volatile("createpolicy.fractional.L2::" CKRL_PROJ_A_EVICT ".b64 %0, 1.0;" : "=l"(pol));
      else
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      const int nst = is_a ? kStA : kStB;
      uint64_t* fullx = is_a ? full_a : full_b;
      uint64_t* emptyx = is_a ? empty_a : empty_b;
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        for (int kb = 0; kb < a.n_kb; ++kb) {
          bar_wait(&emptyx[stage], phase ^ 1);
          if (is_a) {
            bar_expect(&fullx[stage], kABytes);
            tma_2d(su32(sa + stage * kABytes), &map_a, kb * kPK, (int)(tile * kPM), &fullx[stage], pol);
          } else {
            bar_expect(&fullx[stage], kBBytes);
            tma_2d(su32(sb + stage * kBBytes), &map_b, kb * kPK, 0, &fullx[stage], pol);
          }
          if (++stage == nst) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      int sa_i = 0, sb_i = 0;
      uint32_t pa = 0, pb = 0;
      int i = 0;
      for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x, ++i) {
        const int acc = i & 1;
        const uint32_t acc_phase = (uint32_t)(i >> 1) & 1u;
        bar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * kPN);
        for (int kb = 0; kb < a.n_kb; ++kb) {
          bar_wait(&full_a[sa_i], pa);
          bar_wait(&full_b[sb_i], pb);
          tc_fence_after();
          const uint32_t a0 = su32(sa + sa_i * kABytes), b0 = su32(sb + sb_i * kBBytes);
#pragma unroll
          for (int k = 0; k < kPK / 16; ++k)  // +32 bytes per K=16 step inside the swizzle atom
            umma(d, sdesc(a0 + k * 32), sdesc(b0 + k * 32), (kb | k) != 0);
          umma_commit(&empty_a[sa_i]);  // both slots free once these MMAs have read them
          umma_commit(&empty_b[sb_i]);
          if (++sa_i == kStA) {
            sa_i = 0;
            pa ^= 1;
          }
          if (++sb_i == kStB) {
            sb_i = 0;
            pb ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 2 && warp < 10) {
    // ---- epilogue: 8 warps. Warp w (2..9) reads TMEM lane quarter q = w % 4 (the hardware
    // rule: a warp reaches lanes 32*(w%4) .. +31) and column half h = (w-2)/4, so every tile
    // row is split between two threads, 128 bins each; the halves trade their max and their
    // sums through shared memory under a 64-thread named barrier per quarter.
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int row_in_tile = q * 32 + lane;
    const uint32_t bar_id = 1 + q;
    int i = 0;
    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x, ++i) {
      const int acc = i & 1;
      const uint32_t acc_phase = (uint32_t)(i >> 1) & 1u;
      const int64_t row = tile * kPM + row_in_tile;
      const bool live = row < a.rows;
      int tok = 0;
      if (live)
        tok = a.tok_i32 ? reinterpret_cast<const int32_t*>(a.tokens)[row]
                        : (int)reinterpret_cast<const uint8_t*>(a.tokens)[row];
      tok &= kPN - 1;
      bar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int c0 = half * (kPN / 2);
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * kPN + c0);
      const float* bias = s_bias + c0;
      // pass 1: this half's max and (if it holds it) the sampled token's logit; the next
      // 32-column load is in flight while the current one is reduced
      float v[2][32];
      float m = -INFINITY, xt = 0.0f;
      tmem_ld32_issue(taddr, v[0]);
      tmem_wait(v[0]);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c < 3) tmem_ld32_issue(taddr + (c + 1) * 32, v[(c + 1) & 1]);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float x = v[c & 1][j] + bias[c * 32 + j];
          m = fmaxf(m, x);
          xt = (c0 + c * 32 + j == tok) ? x : xt;
        }
        if (c < 3) tmem_wait(v[(c + 1) & 1]);
      }
      s_m[half][row_in_tile] = m;
      named_bar(bar_id, 64);
      m = fmaxf(m, s_m[half ^ 1][row_in_tile]);
      // pass 2: s = sum 2^y, t = sum 2^y * y over this half, y = (x - m) log2 e
      const float mb = m * kLog2e;
      float s0 = 0.f, s1 = 0.f, t0 = 0.f, t1 = 0.f;
      tmem_ld32_issue(taddr, v[0]);
      tmem_wait(v[0]);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c < 3) tmem_ld32_issue(taddr + (c + 1) * 32, v[(c + 1) & 1]);
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float x0 = v[c & 1][j] + bias[c * 32 + j], x1 = v[c & 1][j + 1] + bias[c * 32 + j + 1];
          const float y0 = fmaf(x0, kLog2e, -mb), y1 = fmaf(x1, kLog2e, -mb);
          const float e0 = fast_ex2(y0), e1 = fast_ex2(y1);
          s0 += e0;
          s1 += e1;
          t0 = fmaf(e0, y0, t0);
          t1 = fmaf(e1, y1, t1);
          if (a.logits && live) {
            const int64_t at = row * kPN + c0 + c * 32 + j;
            if (a.logits_bf16)
              reinterpret_cast<__nv_bfloat162*>(a.logits)[at >> 1] = __floats2bfloat162_rn(x0, x1);
            else
              reinterpret_cast<float2*>(a.logits)[at >> 1] = make_float2(x0, x1);
          }
        }
        if (c < 3) tmem_wait(v[(c + 1) & 1]);
      }
      tc_fence_before();
      bar_arrive(&tempty[acc]);  // this half of the accumulator drained
      if (half == 1) {
        s_st[0][row_in_tile] = s0 + s1;
        s_st[1][row_in_tile] = t0 + t1;
        s_st[2][row_in_tile] = xt;
      }
      named_bar(bar_id, 64);
      if (half == 0 && live) {
        // bins 0..127 then 128..255: a fixed order, identical run to run
        const float s = (s0 + s1) + s_st[0][row_in_tile], t = (t0 + t1) + s_st[1][row_in_tile];
        if (tok >= kPN / 2) xt = s_st[2][row_in_tile];
        // y = fma(x, log2e, -mb) with mb = fl(m log2e): every y carries the same shift
        // r = m log2e - mb (exact by fma), so ln sum 2^((x-m) log2e) = ln s - r ln2; the
        // entropy ln S - ln2 E[(x-m) log2e] is shift-free
        const double r = (double)fmaf(m, kLog2e, -mb);
        const double ls = log((double)s);
        const double ey = (double)t / (double)s;  // E[y]
        const double lp = ((double)xt - (double)m) - (ls - r * kLn2);
        const double h = ls - kLn2 * ey;
        if (a.out) {
          ckrl_token_row rr;
          rr.logprob = lp;
          rr.entropy = (float)h;
          rr.reserved = 0;
          a.out[row] = rr;
        }
        if (a.lp) a.lp[row] = lp;
        if (a.ent) a.ent[row] = (float)h;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}

// [outer][H] bf16, row pitch H * 2 bytes, box {64, box_rows}, 128-byte swizzle, OOB rows zero.
bool make_map(CUtensorMap* m, const void* ptr, int64_t outer, int H, int box_rows) {
  EncodeTiled enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)H, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)H * 2};
  cuuint32_t box[2] = {(cuuint32_t)kPK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CKRL_PROJ_L2PROMO,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

size_t proj_smem_bytes() { return kProjSmem; }

cudaError_t launch_proj_stats(int64_t rows, int H, const void* feature, const void* w_pol, const float* b_pol,
                              const void* tokens, int tok_i32, ckrl_token_row* out, double* lp, float* ent,
                              void* logits, int logits_bf16, int max_ctas, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  CUtensorMap ma, mb;
  if (!make_map(&ma, feature, rows, H, kPM) || !make_map(&mb, w_pol, kPN, H, kPN)) return cudaErrorInvalidValue;
  ProjArgs a;
  a.rows = rows;
  a.n_tiles = (rows + kPM - 1) / kPM;
  a.n_kb = H / kPK;
  a.b_pol = b_pol;
  a.tokens = tokens;
  a.tok_i32 = tok_i32;
  a.out = out;
  a.lp = lp;
  a.ent = ent;
  a.logits = logits;
  a.logits_bf16 = logits_bf16;
  cudaError_t e = cudaFuncSetAttribute(proj_stats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kProjSmem);
  if (e != cudaSuccess) return e;
  int64_t grid = sm_count();
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  if (grid > a.n_tiles) grid = a.n_tiles;
  proj_stats_kernel<<<(unsigned)grid, kProjThreads, kProjSmem, s>>>(ma, mb, a);
  return cudaGetLastError();
}

}  // namespace ckrl
