// (f4) Adam with global gradient-norm clipping (optim/adam.cpp:15-41), the step after the
// backward. Two HBM-bound launches on the caller's stream:
//   1. adam_norm: ||g||^2 in fp64 — per-thread sums over a grid-stride range, a fixed-shape
//      warp / CTA tree, then the last CTA adds the CTA partials in CTA order (deterministic
//      for a given grid). With a communicator, the caller's step all-reduces the scalar
//      between the launches (sharded parameters); otherwise nothing crosses GPUs.
//   2. adam_update (programmatic dependent of 1): norm = sqrt(norm^2); non-finite -> the
//      reference's NonFinite (status word, nothing is modified, adam.cpp:21-22); clip
//      g *= max_norm / norm when max_norm > 0 && norm > max_norm (written back: the
//      reference clips grad in place, :23-27); then per element, in the reference's
//      operation order with FMA contraction disabled
//        m = b1*m + (1-b1)*g;  v = b2*v + (1-b2)*g*g;  p -= lr * (m/bc1) / (sqrt(v/bc2) + eps)
//      with bc1 = 1 - b1^t, bc2 = 1 - b2^t computed on the host (std::pow, like :29-30).
// Algorithmic bytes per parameter: read g (norm) + read p, g, m, v + write p, g, m, v
// = 9 * sizeof(T) (g is written only when clipping).
#include "common.cuh"
#include "kernels.h"

namespace ckrl {
namespace {

constexpr int kAdamThreads = 256;
constexpr int kAdamMaxCtas = 148 * 8;  // partial slots in the workspace

__device__ __forceinline__ double sq(double x) { return __dmul_rn(x, x); }

template <typename T>
__global__ void __launch_bounds__(kAdamThreads) adam_norm_kernel(const T* __restrict__ g, int64_t n,
                                                                 double* partials, double* norm_sq,
                                                                 unsigned* ticket) {
  asm volatile("griddepcontrol.launch_dependents;");
  __shared__ double wsum[kAdamThreads / 32];
  __shared__ bool last;
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sizeof(T) == 4 && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
    const int64_t n4 = n / 4;
    const float4* g4 = reinterpret_cast<const float4*>(g);
    for (int64_t k = i; k < n4; k += stride) {
      const float4 x = __ldcs(g4 + k);
      s += sq(x.x) + sq(x.y) + sq(x.z) + sq(x.w);
    }
    for (int64_t k = 4 * n4 + i; k < n; k += stride) s += sq((double)g[k]);
  } else {
    for (int64_t k = i; k < n; k += stride) s += sq((double)g[k]);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double c = 0.0;
    for (int w = 0; w < kAdamThreads / 32; ++w) c += wsum[w];
    partials[blockIdx.x] = c;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // last CTA: thread t sums partials t, t + 256, ... (loads in parallel), then the same
  // fixed-shape tree -> deterministic for a given grid
  double t = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) t += __ldcg(partials + b);
  for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double u = 0.0;
  for (int w = 0; w < kAdamThreads / 32; ++w) u += wsum[w];
  *norm_sq = u;
  *ticket = 0;  // self-reset for the next launch
}

struct AdamScalars {
  double lr, max_norm, b1, b2, eps, bc1, bc2;
};

template <typename T>
__device__ __forceinline__ void adam_elem(T& p, T& g, T& m, T& v, const AdamScalars& k, double scale,
                                          bool clip) {
  if (sizeof(T) == 8) {
    double gd = (double)g;
    if (clip) gd = __dmul_rn(gd, scale);
    const double md = __dadd_rn(__dmul_rn(k.b1, (double)m), __dmul_rn(__dadd_rn(1.0, -k.b1), gd));
    const double vd = __dadd_rn(__dmul_rn(k.b2, (double)v), __dmul_rn(__dmul_rn(__dadd_rn(1.0, -k.b2), gd), gd));
    const double mhat = __ddiv_rn(md, k.bc1), vhat = __ddiv_rn(vd, k.bc2);
    const double upd = __ddiv_rn(__dmul_rn(k.lr, mhat), __dadd_rn(__dsqrt_rn(vhat), k.eps));
    p = (T)__dadd_rn((double)p, -upd);
    g = (T)gd;
    m = (T)md;
    v = (T)vd;
  } else {  // f32 states: same order in f32; scalars (incl. 1 - beta, which cancels badly in
            // f32: 1 - 0.999f is 1.3e-5 off) formed in fp64 and rounded once
    const float b1 = (float)k.b1, b2 = (float)k.b2;
    const float omb1 = (float)(1.0 - k.b1), omb2 = (float)(1.0 - k.b2);
    float gf = (float)g;
    if (clip) gf = __fmul_rn(gf, (float)scale);
    const float mf = __fadd_rn(__fmul_rn(b1, (float)m), __fmul_rn(omb1, gf));
    const float vf = __fadd_rn(__fmul_rn(b2, (float)v), __fmul_rn(__fmul_rn(omb2, gf), gf));
    const float mhat = __fdiv_rn(mf, (float)k.bc1), vhat = __fdiv_rn(vf, (float)k.bc2);
    const float upd = __fdiv_rn(__fmul_rn((float)k.lr, mhat), __fadd_rn(__fsqrt_rn(vhat), (float)k.eps));
    p = (T)__fadd_rn((float)p, -upd);
    g = (T)gf;
    m = (T)mf;
    v = (T)vf;
  }
}

template <typename T>
__global__ void __launch_bounds__(kAdamThreads) adam_update_kernel(T* __restrict__ p, T* __restrict__ g,
                                                                   T* __restrict__ m, T* __restrict__ v,
                                                                   int64_t n, AdamScalars k,
                                                                   const double* norm_sq, double* norm_out,
                                                                   int32_t* status) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const double norm = __dsqrt_rn(__ldcg(norm_sq));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (norm_out) *norm_out = norm;
    if (!isfinite(norm) && status) atomicExch(status, (int32_t)CKRL_ERR_NON_FINITE);
  }
  if (!isfinite(norm)) return;  // adam.cpp:21-22 throws before touching anything
  const bool clip = k.max_norm > 0.0 && norm > k.max_norm;
  const double scale = clip ? __ddiv_rn(k.max_norm, norm) : 1.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool vec = sizeof(T) == 4 && ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) |
                                       reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
  int64_t tail = 0;
  if (vec) {
    const int64_t n4 = n / 4;
    float4* p4 = reinterpret_cast<float4*>(p);
    float4* g4 = reinterpret_cast<float4*>(g);
    float4* m4 = reinterpret_cast<float4*>(m);
    float4* v4 = reinterpret_cast<float4*>(v);
    for (int64_t q = i0; q < n4; q += stride) {
      float4 pp = __ldcs(p4 + q), gg = __ldcs(g4 + q), mm = __ldcs(m4 + q), vv = __ldcs(v4 + q);
      adam_elem<float>(pp.x, gg.x, mm.x, vv.x, k, scale, clip);
      adam_elem<float>(pp.y, gg.y, mm.y, vv.y, k, scale, clip);
      adam_elem<float>(pp.z, gg.z, mm.z, vv.z, k, scale, clip);
      adam_elem<float>(pp.w, gg.w, mm.w, vv.w, k, scale, clip);
      __stcs(p4 + q, pp);
      if (clip) __stcs(g4 + q, gg);
      __stcs(m4 + q, mm);
      __stcs(v4 + q, vv);
    }
    tail = 4 * n4;
  }
  for (int64_t q = tail + i0; q < n; q += stride) {
    T pp = p[q], gg = g[q], mm = m[q], vv = v[q];
    adam_elem<T>(pp, gg, mm, vv, k, scale, clip);
    p[q] = pp;
    if (clip) g[q] = gg;
    m[q] = mm;
    v[q] = vv;
  }
}

int adam_grid(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t need = (n / 4 + kAdamThreads - 1) / kAdamThreads;
  int64_t cap = (int64_t)sms * 8;  // 8 resident 256-thread CTAs per SM
  if (cap > kAdamMaxCtas) cap = kAdamMaxCtas;
  return (int)(need < 1 ? 1 : (need < cap ? need : cap));
}

}  // namespace

size_t adam_workspace_bytes() { return sizeof(double) * (kAdamMaxCtas + 2) + 64; }

cudaError_t launch_adam_norm(int f64, const void* g, int64_t n, char* ws, cudaStream_t s) {
  const int grid = adam_grid(n);
  double* partials = reinterpret_cast<double*>(ws);
  double* norm_sq = partials + kAdamMaxCtas;
  unsigned* ticket = reinterpret_cast<unsigned*>(norm_sq + 2);
  if (f64)
    adam_norm_kernel<double><<<grid, kAdamThreads, 0, s>>>(static_cast<const double*>(g), n, partials, norm_sq, ticket);
  else
    adam_norm_kernel<float><<<grid, kAdamThreads, 0, s>>>(static_cast<const float*>(g), n, partials, norm_sq, ticket);
  return cudaGetLastError();
}

double* adam_norm_sq_slot(char* ws) { return reinterpret_cast<double*>(ws) + kAdamMaxCtas; }

cudaError_t launch_adam_update(int f64, void* p, void* g, void* m, void* v, int64_t n, double lr,
                               double max_norm, double b1, double b2, double eps, double bc1, double bc2,
                               char* ws, double* norm_out, int32_t* status, int pdl, cudaStream_t s) {
  AdamScalars k{lr, max_norm, b1, b2, eps, bc1, bc2};
  const double* norm_sq = adam_norm_sq_slot(ws);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)adam_grid(n));
  cfg.blockDim = dim3(kAdamThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (f64)
    return cudaLaunchKernelEx(&cfg, adam_update_kernel<double>, static_cast<double*>(p), static_cast<double*>(g),
                              static_cast<double*>(m), static_cast<double*>(v), n, k, norm_sq, norm_out, status);
  return cudaLaunchKernelEx(&cfg, adam_update_kernel<float>, static_cast<float*>(p), static_cast<float*>(g),
                            static_cast<float*>(m), static_cast<float*>(v), n, k, norm_sq, norm_out, status);
}

}  // namespace ckrl
