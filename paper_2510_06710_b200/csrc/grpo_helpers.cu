// Per-group / per-episode GRPO helpers and the slab success rate, batched and segmented for
// the GPU. Every value is computed in the reference's operation order
// without FMA contraction, so results are bit-identical to the reference's fp64 code:
//
//   grpo_group_advantage   advantage/grpo.cpp:9-28   (population std, DegenerateGroup rules)
//   group_mean_return      advantage/grpo.cpp:30-35
//   success_rate_filter    advantage/grpo.cpp:37-46  (strict lower < mean < upper)
//   valid_action_mask      advantage/grpo.cpp:48-55
//   length_norm_weights    advantage/grpo.cpp:57-79
//   slab_success_rate      advantage/assembler.cpp:269-278
#include "common.cuh"
#include "kernels.h"

namespace ckrl {

__device__ __forceinline__ void set_status(int32_t* status, int32_t code) {
  if (status) atomicCAS(status, 0, code);
}

__device__ double group_mean(const double* R, int b, int e) {
  double m = 0.0;
  for (int i = b; i < e; ++i) m = __dadd_rn(m, R[i]);
  return e > b ? __ddiv_rn(m, (double)(e - b)) : 0.0;
}

__global__ void group_advantage_kernel(int G, const int32_t* off, const double* R, double eps, double* adv,
                                       int32_t* status) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  const int b = off[g], e = off[g + 1], n = e - b;
  if (n < 2) {
    set_status(status, CKRL_ERR_DEGENERATE_GROUP);
    return;
  }
  const double mean = group_mean(R, b, e);
  double var = 0.0;
  for (int i = b; i < e; ++i) {
    const double d = __dsub_rn(R[i], mean);
    var = __dadd_rn(var, __dmul_rn(d, d));
  }
  var = __ddiv_rn(var, (double)n);
  const double sd = __dsqrt_rn(var);
  if (sd == 0.0 && eps == 0.0) {
    set_status(status, CKRL_ERR_DEGENERATE_GROUP);
    return;
  }
  const double den = __dadd_rn(sd, eps);
  for (int i = b; i < e; ++i) adv[i] = __ddiv_rn(__dsub_rn(R[i], mean), den);
}

__global__ void success_filter_kernel(int G, const int32_t* off, const double* R, double lower, double upper,
                                      uint8_t* keep, double* mean_out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  const double m = group_mean(R, off[g], off[g + 1]);
  if (keep) keep[g] = (m > lower && m < upper) ? 1 : 0;
  if (mean_out) mean_out[g] = m;
}

// one block per episode, threads over its steps
__global__ void mask_weights_kernel(const int64_t* off, const uint8_t* success, const int64_t* first_success,
                                    int normalized, uint8_t* mask, double* w) {
  const int ep = blockIdx.x;
  const int64_t b = off[ep], len = off[ep + 1] - b;
  const int64_t fs = first_success[ep];
  const bool cut = success[ep] && fs >= 0;
  // T_succ = number of valid steps = min(fs + 1, len) on a cut episode, else len
  const int64_t t_succ = cut ? (fs + 1 < len ? fs + 1 : len) : len;
  const double u_norm = t_succ > 0 ? __ddiv_rn(1.0, (double)t_succ) : 0.0;
  const double u_base = len > 0 ? __ddiv_rn(1.0, (double)len) : 0.0;
  for (int64_t t = threadIdx.x; t < len; t += blockDim.x) {
    const bool valid = !(cut && t > fs);
    if (mask) mask[b + t] = valid ? 1 : 0;
    if (w) w[b + t] = normalized ? (valid ? u_norm : 0.0) : u_base;
  }
}

__global__ void success_rate_kernel(int n, const uint8_t* complete, const int32_t* first_success, double* out) {
  __shared__ unsigned long long s_tot[32], s_suc[32];
  unsigned long long tot = 0, suc = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (complete[i]) {
      ++tot;
      if (first_success[i] >= 0) ++suc;  // EpisodeInfo::success (vec_env.cpp:129)
    }
  for (int o = 16; o; o >>= 1) {
    tot += __shfl_xor_sync(0xffffffffu, tot, o);
    suc += __shfl_xor_sync(0xffffffffu, suc, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_tot[warp] = tot;
    s_suc[warp] = suc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long T = 0, S = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      T += s_tot[w];
      S += s_suc[w];
    }
    out[0] = T == 0 ? 0.0 : __ddiv_rn((double)S, (double)T);
  }
}

cudaError_t launch_group_advantage(int G, const int32_t* off, const double* R, double eps, double* adv,
                                   int32_t* status, cudaStream_t s) {
  if (G > 0) group_advantage_kernel<<<(G + 127) / 128, 128, 0, s>>>(G, off, R, eps, adv, status);
  return cudaGetLastError();
}

cudaError_t launch_success_filter(int G, const int32_t* off, const double* R, double lower, double upper,
                                  uint8_t* keep, double* mean_out, cudaStream_t s) {
  if (G > 0) success_filter_kernel<<<(G + 127) / 128, 128, 0, s>>>(G, off, R, lower, upper, keep, mean_out);
  return cudaGetLastError();
}

cudaError_t launch_mask_weights(int n_eps, const int64_t* off, const uint8_t* success, const int64_t* fs,
                                int normalized, uint8_t* mask, double* w, cudaStream_t s) {
  if (n_eps > 0) mask_weights_kernel<<<n_eps, 128, 0, s>>>(off, success, fs, normalized, mask, w);
  return cudaGetLastError();
}

cudaError_t launch_success_rate(int n, const uint8_t* complete, const int32_t* fs, double* out, cudaStream_t s) {
  success_rate_kernel<<<1, 512, 0, s>>>(n, complete, fs, out);
  return cudaGetLastError();
}

}  // namespace ckrl
