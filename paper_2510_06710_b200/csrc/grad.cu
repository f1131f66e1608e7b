// (f1) the softmax-backward seam: per position, the gradient of
//   coeff_lp * log p(tok) + coeff_ent * H
// with respect to the V-bin logits row, i.e. what PolicyNet::accumulate_chunk_gradient forms
// before its outer_add / trunk backward (policy/policy_net.cpp:431-456):
//   dlogit_v = klp * ([v == tok] - p_v) + kent * (-p_v * (ls_v + H)),
//   ls = log_softmax(row), p = exp(ls), H = -sum_v p_v ls_v.
// Positions with klp == 0 && kent == 0 are skipped by the reference (no contribution): their
// row is written as zeros without reading the logits. A non-finite coefficient is the
// reference's NonFinite (:437-438): the row is zeroed and *status is set.
//
// Streaming kernel, HBM-bound: reads V*s_in bytes of logits and writes V*s_out bytes of
// dlogits per position (+ 9 B of token / coefficients). 8 lanes per row (V == 256: 32 values
// per lane in registers, 128-bit loads / stores, every warp instruction moves 4 full rows'
// 128-byte lines), 3 xor-shuffles per reduction, exp as ex2.approx on log2-scaled arguments.
#include "common.cuh"
#include "kernels.h"

#include <cuda_bf16.h>

namespace ckrl {
namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2f = 0.6931471805599453f;

__device__ __forceinline__ float ex2f(float y) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(y));
  return r;
}
__device__ __forceinline__ float4 ld_stream4(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream4(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_stream_u4(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ float g8_max(float v) {
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float g8_sum(float v) {
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// V == 256. Lane l8 of a row group owns values {8*i + l8 : i} in float4 units, i.e. the
// f32 columns 4*(l8 + 8*i) + {0..3} (bf16: uint4 units of 8 columns, i < 4).
template <typename LT, typename OT>
__global__ void __launch_bounds__(256) logits_grad_256(const LT* __restrict__ logits,
                                                       const void* __restrict__ tokens, int tok_i32,
                                                       const float* __restrict__ coeff_lp,
                                                       const float* __restrict__ coeff_ent,
                                                       int64_t rows, OT* __restrict__ out,
                                                       int32_t* status) {
  constexpr int V = 256;
  const int lane = threadIdx.x & 31, l8 = lane & 7;
  const int64_t groups = (int64_t)gridDim.x * (blockDim.x >> 3);
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 3) + (threadIdx.x >> 3); row < rows;
       row += groups) {
    const float klp = __ldg(coeff_lp + row), kent = coeff_ent ? __ldg(coeff_ent + row) : 0.0f;
    const bool skip = klp == 0.0f && kent == 0.0f;
    const bool bad = !skip && !(isfinite(klp) && isfinite(kent));
    if (bad && l8 == 0 && status) atomicExch(status, (int32_t)CKRL_ERR_NON_FINITE);
    float x[32];
    if (skip || bad) {
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = 0.0f;
    } else if (sizeof(LT) == 4) {
      const float4* p = reinterpret_cast<const float4*>(logits + row * V);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 v = ld_stream4(p + l8 + 8 * i);
        x[4 * i] = v.x;
        x[4 * i + 1] = v.y;
        x[4 * i + 2] = v.z;
        x[4 * i + 3] = v.w;
      }
    } else {
      const uint4* p = reinterpret_cast<const uint4*>(logits + row * V);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 v = ld_stream_u4(p + l8 + 8 * i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          x[8 * i + 2 * j] = __uint_as_float(w[j] << 16);
          x[8 * i + 2 * j + 1] = __uint_as_float(w[j] & 0xffff0000u);
        }
      }
    }
    // column of value x[k]: f32: 4*(l8 + 8*(k/4)) + k%4; bf16: 8*(l8 + 8*(k/8)) + k%8
    auto col = [&](int k) {
      return sizeof(LT) == 4 ? 4 * (l8 + 8 * (k >> 2)) + (k & 3) : 8 * (l8 + 8 * (k >> 3)) + (k & 7);
    };
    float d[32];
    if (skip || bad) {
#pragma unroll
      for (int k = 0; k < 32; ++k) d[k] = 0.0f;
    } else {
      float m = x[0];
#pragma unroll
      for (int k = 1; k < 32; ++k) m = fmaxf(m, x[k]);
      m = g8_max(m);
      const float ms = m * kLog2e;
      float s = 0.0f;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        d[k] = ex2f(fmaf(x[k], kLog2e, -ms));  // e_k = exp(x_k - m)
        s += d[k];
      }
      s = g8_sum(s);
      const float inv_s = 1.0f / s;
      const float lse = m + kLn2f * __log2f(s);
      float hs = 0.0f;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        d[k] *= inv_s;               // p_k
        x[k] -= lse;                 // ls_k
        hs = fmaf(d[k], x[k], hs);
      }
      const float H = -g8_sum(hs);
      const int tok = tok_i32 ? reinterpret_cast<const int32_t*>(tokens)[row]
                              : (int)reinterpret_cast<const uint8_t*>(tokens)[row];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const float p = d[k];
        d[k] = klp * ((col(k) == tok ? 1.0f : 0.0f) - p) - kent * (p * (x[k] + H));
      }
    }
    if (sizeof(OT) == 4) {
      float4* q = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + row * V);
      if (sizeof(LT) == 4) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          st_stream4(q + l8 + 8 * i, make_float4(d[4 * i], d[4 * i + 1], d[4 * i + 2], d[4 * i + 3]));
      } else {  // bf16 in, f32 out: lane owns 8-column runs -> two float4 per run
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          st_stream4(q + 2 * (l8 + 8 * i), make_float4(d[8 * i], d[8 * i + 1], d[8 * i + 2], d[8 * i + 3]));
          st_stream4(q + 2 * (l8 + 8 * i) + 1,
                     make_float4(d[8 * i + 4], d[8 * i + 5], d[8 * i + 6], d[8 * i + 7]));
        }
      }
    } else {
      uint4* q = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + row * V);
      if (sizeof(LT) == 2) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          st_stream_u4(q + l8 + 8 * i, make_uint4(pack_bf16(d[8 * i], d[8 * i + 1]), pack_bf16(d[8 * i + 2], d[8 * i + 3]),
                                                  pack_bf16(d[8 * i + 4], d[8 * i + 5]),
                                                  pack_bf16(d[8 * i + 6], d[8 * i + 7])));
      } else {  // f32 in (4-column runs), bf16 out: 8-byte stores
        uint2* q2 = reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + row * V);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          q2[l8 + 8 * i] = make_uint2(pack_bf16(d[4 * i], d[4 * i + 1]), pack_bf16(d[4 * i + 2], d[4 * i + 3]));
      }
    }
  }
}

// Any V: one warp per row, three strided passes (L1 absorbs the re-reads).
template <typename LT, typename OT>
__global__ void __launch_bounds__(256) logits_grad_generic(const LT* __restrict__ logits,
                                                           const void* __restrict__ tokens, int tok_i32,
                                                           const float* __restrict__ coeff_lp,
                                                           const float* __restrict__ coeff_ent,
                                                           int64_t rows, int V, OT* __restrict__ out,
                                                           int32_t* status) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  auto ld = [&](int64_t i) {
    if (sizeof(LT) == 4) return (float)reinterpret_cast<const float*>(logits)[i];
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(logits)[i]);
  };
  auto st = [&](int64_t i, float v) {
    if (sizeof(OT) == 4)
      reinterpret_cast<float*>(out)[i] = v;
    else
      reinterpret_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
  };
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows; row += warps) {
    const float klp = coeff_lp[row], kent = coeff_ent ? coeff_ent[row] : 0.0f;
    const bool skip = klp == 0.0f && kent == 0.0f;
    const bool bad = !skip && !(isfinite(klp) && isfinite(kent));
    if (bad && lane == 0 && status) atomicExch(status, (int32_t)CKRL_ERR_NON_FINITE);
    const int64_t base = row * V;
    if (skip || bad) {
      for (int v = lane; v < V; v += 32) st(base + v, 0.0f);
      continue;
    }
    float m = -INFINITY;
    for (int v = lane; v < V; v += 32) m = fmaxf(m, ld(base + v));
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float s = 0.0f;
    for (int v = lane; v < V; v += 32) s += ex2f((ld(base + v) - m) * kLog2e);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float inv_s = 1.0f / s, lse = m + kLn2f * __log2f(s);
    float hs = 0.0f;
    for (int v = lane; v < V; v += 32) {
      const float ls = ld(base + v) - lse;
      hs = fmaf(ex2f(ls * kLog2e), ls, hs);
    }
    for (int o = 16; o > 0; o >>= 1) hs += __shfl_xor_sync(0xffffffffu, hs, o);
    const float H = -hs;
    (void)inv_s;
    const int tok = tok_i32 ? reinterpret_cast<const int32_t*>(tokens)[row]
                            : (int)reinterpret_cast<const uint8_t*>(tokens)[row];
    for (int v = lane; v < V; v += 32) {
      const float ls = ld(base + v) - lse, p = ex2f(ls * kLog2e);
      st(base + v, klp * ((v == tok ? 1.0f : 0.0f) - p) - kent * (p * (ls + H)));
    }
  }
}

int grad_grid(int64_t rows, int rows_per_block) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t need = (rows + rows_per_block - 1) / rows_per_block;
  const int64_t cap = (int64_t)sms * 8;  // 8 resident 256-thread CTAs per SM
  return (int)(need < cap ? (need > 0 ? need : 1) : cap);
}

template <typename LT, typename OT>
cudaError_t launch_grad_t(const void* logits, const void* tokens, int tok_i32, const float* klp,
                          const float* kent, int64_t rows, int V, void* out, int32_t* status,
                          cudaStream_t s) {
  const bool fast = V == 256 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  if (fast) {
    logits_grad_256<LT, OT><<<grad_grid(rows, 32), 256, 0, s>>>(
        static_cast<const LT*>(logits), tokens, tok_i32, klp, kent, rows, static_cast<OT*>(out), status);
  } else {
    logits_grad_generic<LT, OT><<<grad_grid(rows, 8), 256, 0, s>>>(
        static_cast<const LT*>(logits), tokens, tok_i32, klp, kent, rows, V, static_cast<OT*>(out), status);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_logits_grad(const void* logits, int logits_bf16, const void* tokens, int tok_i32,
                               const float* coeff_lp, const float* coeff_ent, int64_t rows, int V,
                               void* out, int out_bf16, int32_t* status, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  if (!logits_bf16 && !out_bf16)
    return launch_grad_t<float, float>(logits, tokens, tok_i32, coeff_lp, coeff_ent, rows, V, out, status, s);
  if (!logits_bf16 && out_bf16)
    return launch_grad_t<float, __nv_bfloat16>(logits, tokens, tok_i32, coeff_lp, coeff_ent, rows, V, out, status, s);
  if (logits_bf16 && !out_bf16)
    return launch_grad_t<__nv_bfloat16, float>(logits, tokens, tok_i32, coeff_lp, coeff_ent, rows, V, out, status, s);
  return launch_grad_t<__nv_bfloat16, __nv_bfloat16>(logits, tokens, tok_i32, coeff_lp, coeff_ent, rows, V, out,
                                                     status, s);
}

}  // namespace ckrl
