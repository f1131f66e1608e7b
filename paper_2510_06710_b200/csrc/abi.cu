// C-ABI layer (include/ckrl.h): argument validation with the reference's error
// taxonomy, workspace carve-up, kernel dispatch and the NCCL stats exchange.
// No entry point allocates device memory or synchronises the stream, except
// ckrl_read_diagnostics (which returns host scalars) and the communicator setup.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"

#include <cmath>

using namespace ckrl;

namespace {

thread_local std::string g_last_error;

int32_t fail(int32_t code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CKRL_CUDA(x)                                                                      \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) return fail(CKRL_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)

#define CKRL_REQUIRE(cond, code, msg) \
  do {                                \
    if (!(cond)) return fail((code), (msg)); \
  } while (0)

int32_t check_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(CKRL_ERR_CUDA, "no CUDA device: the ckrl hot path has no CPU fallback");
  return CKRL_OK;
}

int32_t check_rollout(const ckrl_rollout* ro, bool need_values) {
  CKRL_REQUIRE(ro != nullptr, CKRL_ERR_INVALID_ARGUMENT, "rollout is null");
  CKRL_REQUIRE(ro->num_envs >= 0 && ro->num_chunks >= 0 && ro->chunk_len >= 1 &&
                   ro->tokens_per_action >= 1 && ro->vocab >= 1,
               CKRL_ERR_LENGTH_MISMATCH, "rollout dimensions must be positive");
  CKRL_REQUIRE(ro->token_dtype == CKRL_DTYPE_U8 || ro->token_dtype == CKRL_DTYPE_I32,
               CKRL_ERR_INVALID_ARGUMENT, "token dtype must be u8 or i32");
  CKRL_REQUIRE(ro->token_dtype == CKRL_DTYPE_I32 || ro->vocab <= 256, CKRL_ERR_INVALID_ARGUMENT,
               "u8 tokens require vocab <= 256");
  CKRL_REQUIRE((int64_t)ro->chunk_len * ro->tokens_per_action <= 8192, CKRL_ERR_INVALID_ARGUMENT,
               "C*M must be <= 8192");
  const int64_t n = (int64_t)ro->num_envs * ro->num_chunks;
  if (n > 0) {
    CKRL_REQUIRE(ro->flags && ro->episode_id && ro->reward, CKRL_ERR_INVALID_ARGUMENT,
                 "rollout flags / episode_id / reward are required");
    if (need_values)
      CKRL_REQUIRE(ro->value_scalar && ro->value_vector && ro->bootstrap,
                   CKRL_ERR_INVALID_ARGUMENT, "rollout values / bootstrap are required");
  }
  return CKRL_OK;
}

int32_t check_ws(void* ws, size_t bytes, int E, int world) {
  CKRL_REQUIRE(ws != nullptr, CKRL_ERR_INVALID_ARGUMENT, "workspace is null");
  size_t need = ws_layout(E, world).total;
  if (bytes < need)
    return fail(CKRL_ERR_INVALID_ARGUMENT, "workspace too small: need " + std::to_string(need) +
                                               " bytes, got " + std::to_string(bytes));
  return CKRL_OK;
}

int32_t validate(const ckrl_granularity* g) {
  CKRL_REQUIRE(g != nullptr, CKRL_ERR_INVALID_ARGUMENT, "granularity is null");
  auto ok = [](int l) { return l >= CKRL_LEVEL_CHUNK && l <= CKRL_LEVEL_TOKEN; };
  CKRL_REQUIRE(ok(g->advantage_level) && ok(g->logprob_level) && ok(g->value_level),
               CKRL_ERR_CONFIG, "unknown granularity level");
  // core/granularity.cpp:47-60
  if (g->advantage_level == CKRL_LEVEL_TOKEN)
    return fail(CKRL_ERR_UNSUPPORTED_COMBINATION, "advantage level must be chunk_level or action_level");
  if (g->value_level == CKRL_LEVEL_TOKEN)
    return fail(CKRL_ERR_UNSUPPORTED_COMBINATION, "value level must be chunk_level or action_level");
  if (g->logprob_level < g->advantage_level)
    return fail(CKRL_ERR_UNSUPPORTED_COMBINATION,
                "unsupported combination: logprob level coarser than advantage level");
  return CKRL_OK;
}

LossArgs base_args(const ckrl_rollout* ro, const ckrl_policy_outputs* po, char* ws, int world) {
  LossArgs a;
  std::memset(&a, 0, sizeof(a));
  a.E = ro->num_envs;
  a.Tc = ro->num_chunks;
  a.C = ro->chunk_len;
  a.M = ro->tokens_per_action;
  a.V = ro->vocab;
  a.n_rec = (int64_t)ro->num_envs * ro->num_chunks;
  a.logits_bf16 = po->logits_dtype == CKRL_DTYPE_BF16;
  a.tok_i32 = ro->token_dtype == CKRL_DTYPE_I32;
  a.logits = po->logits;
  if (po->logits_dtype == CKRL_DTYPE_TOKEN_ROWS) a.rows_in = static_cast<const ckrl_token_row*>(po->logits);
  a.tokens = ro->tokens;
  a.old_lp = ro->old_logprob;
  a.ws = ws;
  a.L = ws_layout(ro->num_envs, world);
  a.world = world;
  return a;
}

void set_outputs(LossArgs& a, const ckrl_loss_outputs* o) {
  if (!o) return;
  a.coeff_lp = o->coeff_logprob;
  a.coeff_ent = o->coeff_entropy;
  a.coeff_val = o->coeff_value;
  a.tok_lp = o->token_logprob;
  a.tok_ent = o->token_entropy;
  a.dlogits = o->dlogits;
  a.action_ent = o->action_entropy;
  a.chunk_ent = o->chunk_entropy;
  a.all_rows = (o->token_logprob || o->token_entropy) ? 1 : 0;
}

int32_t check_policy(const ckrl_rollout* ro, const ckrl_policy_outputs* po, const ckrl_loss_outputs* out) {
  CKRL_REQUIRE(po != nullptr, CKRL_ERR_INVALID_ARGUMENT, "policy outputs are null");
  CKRL_REQUIRE(!(po->logits_dtype == CKRL_DTYPE_TOKEN_ROWS && out && out->dlogits), CKRL_ERR_INVALID_ARGUMENT,
               "dlogits need the logits (token rows carry only the finished log-prob / entropy)");
  CKRL_REQUIRE(po->logits_dtype == CKRL_DTYPE_F32 || po->logits_dtype == CKRL_DTYPE_BF16 ||
                   po->logits_dtype == CKRL_DTYPE_TOKEN_ROWS,
               CKRL_ERR_INVALID_ARGUMENT, "logits dtype must be f32, bf16 or token rows");
  if ((int64_t)ro->num_envs * ro->num_chunks > 0)
    CKRL_REQUIRE(po->logits && ro->tokens && ro->old_logprob, CKRL_ERR_INVALID_ARGUMENT,
                 "logits, tokens and old_logprob are required");
  if (ro->vocab == 256 || po->logits_dtype == CKRL_DTYPE_TOKEN_ROWS) {
    uintptr_t p = reinterpret_cast<uintptr_t>(po->logits);
    CKRL_REQUIRE((p & 15) == 0, CKRL_ERR_INVALID_ARGUMENT, "logits must be 16-byte aligned");
  }
  return CKRL_OK;
}

// ---- NCCL, resolved at communicator creation (no link-time dependency) -------------
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  const char* (*GetErrorString)(ncclResult_t);
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // Reuse the NCCL already in the process (torch's), else load the system one.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
      api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.AllGather && api.AllReduce &&
               api.CommDestroy && api.GetErrorString;
    }
  }
  return api;
}

}  // namespace

struct ckrl_comm {
  ncclComm_t nc = nullptr;          // optional (Adam's gradient-norm all-reduce)
  int world = 1, rank = 0, device = 0;
  char* xbuf = nullptr;             // this rank's exchange buffer (ex_buffer_bytes(world))
  char** peers_dev = nullptr;       // device table: every rank's exchange buffer
  std::vector<char*> ipc_opened;    // peers' buffers mapped with cudaIpcOpenMemHandle
  bool ready = false;               // peers opened
  int co_resident = 1;              // ranks of this job on this device (test / debug setups)
};

namespace {
// Several ranks on one device (a single-GPU test of the multi-rank path): every rank's loss
// kernel spins until all ranks' records arrive, so all of them must be resident at once —
// each rank's persistent loss grid takes an equal share of the SMs, minus one SM per rank
// for the assembly kernels.
int loss_cta_cap(const ckrl_comm* c) {
  if (!c || c->co_resident <= 1) return 0;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const int cap = (sms - c->co_resident) / c->co_resident;
  return cap > 1 ? cap : 1;
}

ckrl::ExchangeView exchange_view(const ckrl_comm* c) {
  ckrl::ExchangeView x{};
  if (c && c->world > 1) {
    x.peers = c->peers_dev;
    x.local = c->xbuf;
    x.world = c->world;
    x.rank = c->rank;
  }
  return x;
}
}  // namespace

#define CKRL_NCCL(x)                                                                    \
  do {                                                                                  \
    ncclResult_t r_ = (x);                                                              \
    if (r_ != ncclSuccess) return fail(CKRL_ERR_NCCL, std::string(#x ": ") + nccl().GetErrorString(r_)); \
  } while (0)

extern "C" {

const char* ckrl_version(void) { return "ckrl 0.1.0 (sm_100a)"; }

const char* ckrl_status_string(int32_t s) {
  switch (s) {
    case CKRL_OK: return "ok";
    case CKRL_ERR_UNSUPPORTED_COMBINATION: return "UnsupportedCombination";
    case CKRL_ERR_GRANULARITY_ORDER: return "GranularityOrderViolation";
    case CKRL_ERR_LENGTH_MISMATCH: return "LengthMismatch";
    case CKRL_ERR_BAD_RESET_ID: return "BadResetId";
    case CKRL_ERR_HEAD_MISMATCH: return "HeadMismatch";
    case CKRL_ERR_NON_FINITE: return "NonFinite";
    case CKRL_ERR_DEGENERATE_GROUP: return "DegenerateGroup";
    case CKRL_ERR_SKIP_UPDATE: return "SkipUpdate";
    case CKRL_ERR_INVALID_PLAN: return "InvalidPlan";
    case CKRL_ERR_MEMORY_OVERFLOW: return "MemoryOverflow";
    case CKRL_ERR_EMPTY_TRACE: return "EmptyTrace";
    case CKRL_ERR_CONFIG: return "ConfigError";
    case CKRL_ERR_GENERIC: return "Error";
    case CKRL_ERR_CUDA: return "CudaError";
    case CKRL_ERR_INVALID_ARGUMENT: return "InvalidArgument";
    case CKRL_ERR_NCCL: return "NcclError";
    default: return "unknown";
  }
}

const char* ckrl_last_error(void) { return g_last_error.c_str(); }

int32_t ckrl_validate_granularity(const ckrl_granularity* spec) { return validate(spec); }

size_t ckrl_workspace_bytes(int32_t num_envs, int32_t num_chunks, int32_t chunk_len,
                            int32_t tokens_per_action, int32_t world) {
  (void)num_chunks;
  (void)chunk_len;
  (void)tokens_per_action;
  return ws_layout(num_envs, world).total;
}

int32_t ckrl_workspace_init(void* ws, size_t bytes, ckrl_stream_t stream) {
  CKRL_REQUIRE(ws != nullptr, CKRL_ERR_INVALID_ARGUMENT, "workspace is null");
  CKRL_CUDA(cudaMemsetAsync(ws, 0, bytes, (cudaStream_t)stream));
  return CKRL_OK;
}

size_t ckrl_stats_record_bytes(void) { return sizeof(StatsRecord); }

int32_t ckrl_merge_stats_host(const void* records, int32_t world, double* out_mean,
                              double* out_denom, int64_t* out_counts) {
  CKRL_REQUIRE(records && world >= 1, CKRL_ERR_INVALID_ARGUMENT, "bad stats records");
  const StatsRecord* r = static_cast<const StatsRecord*>(records);
  int64_t c[4] = {0, 0, 0, 0};
  for (int i = 0; i < world; ++i) {
    c[0] += r[i].n_adv;
    c[1] += r[i].n_val;
    c[2] += r[i].n_pos;
    c[3] += r[i].groups_retained;
  }
  double mean, denom;
  whitening(merge_records(r, world), &mean, &denom);
  if (out_mean) *out_mean = mean;
  if (out_denom) *out_denom = denom;
  if (out_counts) std::memcpy(out_counts, c, sizeof(c));
  return CKRL_OK;
}

int32_t ckrl_compute_gae(int32_t num_seqs, const int32_t* seq_offsets, const double* rewards,
                         const double* values, const double* bootstrap, const uint8_t* flags,
                         const ckrl_gae_params* params, double* advantages, double* returns,
                         ckrl_stream_t stream) {
  int32_t st = check_device();
  if (st) return st;
  CKRL_REQUIRE(params && num_seqs >= 0, CKRL_ERR_INVALID_ARGUMENT, "bad arguments");
  if (num_seqs == 0) return CKRL_OK;
  CKRL_REQUIRE(seq_offsets && rewards && values && bootstrap && flags && advantages && returns,
               CKRL_ERR_LENGTH_MISMATCH, "compute_gae: null input");
  CKRL_CUDA(launch_flat_gae(num_seqs, seq_offsets, rewards, values, bootstrap, flags, params->gamma,
                            params->lambda, advantages, returns, (cudaStream_t)stream));
  return CKRL_OK;
}

int32_t ckrl_assemble_ppo_batch(const ckrl_rollout* ro, const ckrl_gae_params* gae,
                                const ckrl_granularity* spec, ckrl_ppo_batch* batch,
                                void* workspace, size_t ws_bytes, ckrl_stream_t stream) {
  int32_t st = validate(spec);
  if (st) return st;
  // assembler.cpp:82-83
  if (spec->value_level != spec->advantage_level)
    return fail(CKRL_ERR_CONFIG, "value_type must match reward_type for GAE assembly");
  if ((st = check_device())) return st;
  if ((st = check_rollout(ro, true))) return st;
  if ((st = check_ws(workspace, ws_bytes, ro->num_envs, 1))) return st;
  CKRL_REQUIRE(gae && batch && batch->counted && batch->advantages && batch->returns,
               CKRL_ERR_INVALID_ARGUMENT, "batch outputs are required");
  WsLayout L = ws_layout(ro->num_envs, 1);
  CKRL_CUDA(launch_ppo_assemble(*ro, spec->advantage_level == CKRL_LEVEL_ACTION, gae->gamma,
                                gae->lambda, *batch, (char*)workspace, L, (cudaStream_t)stream));
  return CKRL_OK;
}

int32_t ckrl_normalize_advantages(const ckrl_rollout* ro, const ckrl_granularity* spec,
                                  ckrl_ppo_batch* batch, void* workspace, size_t ws_bytes,
                                  ckrl_stream_t stream) {
  int32_t st = validate(spec);
  if (st) return st;
  if ((st = check_device())) return st;
  if ((st = check_rollout(ro, false))) return st;
  if ((st = check_ws(workspace, ws_bytes, ro->num_envs, 1))) return st;
  WsLayout L = ws_layout(ro->num_envs, 1);
  CKRL_REQUIRE(batch && batch->counted && batch->advantages, CKRL_ERR_INVALID_ARGUMENT,
               "batch counted / advantages required");
  CKRL_CUDA(launch_normalize(*ro, spec->advantage_level == CKRL_LEVEL_ACTION, batch->counted,
                             batch->advantages,
                             reinterpret_cast<StatsRecord*>((char*)workspace + L.stats_local), 1,
                             reinterpret_cast<uint32_t*>((char*)workspace + L.tickets) + TICKET_NORM,
                             (cudaStream_t)stream));
  return CKRL_OK;
}

int32_t ckrl_assemble_grpo_batch(const ckrl_rollout* ro, const ckrl_episodes* ep,
                                 const ckrl_granularity* spec, const ckrl_grpo_options* opt,
                                 ckrl_grpo_batch* gb, void* workspace, size_t ws_bytes,
                                 ckrl_stream_t stream) {
  int32_t st = validate(spec);
  if (st) return st;
  if ((st = check_device())) return st;
  if ((st = check_rollout(ro, false))) return st;
  if ((st = check_ws(workspace, ws_bytes, ro->num_envs, 1))) return st;
  CKRL_REQUIRE(ep && opt && gb, CKRL_ERR_INVALID_ARGUMENT, "episodes / options / batch required");
  CKRL_REQUIRE(gb->env_group && gb->env_member && gb->env_episode && gb->env_advantage &&
                   gb->env_group_size && gb->slot_weight && gb->slot_member && gb->group_counts,
               CKRL_ERR_INVALID_ARGUMENT, "grpo batch outputs are required");
  CKRL_REQUIRE(ep->count >= 0, CKRL_ERR_LENGTH_MISMATCH, "negative episode count");
  WsLayout L = ws_layout(ro->num_envs, 1);
  CKRL_CUDA(launch_grpo_assemble(*ro, *ep, *opt, *gb, (char*)workspace, L, (cudaStream_t)stream));
  return CKRL_OK;
}

int32_t ckrl_token_stats(int64_t num_chunks, int32_t C, int32_t M, int32_t V, int32_t logits_dtype,
                         const void* logits, int32_t token_dtype, const void* tokens,
                         float* token_logprob, float* token_entropy, double* action_logprob,
                         double* chunk_logprob, const uint8_t* slot_mask, double* action_entropy,
                         double* chunk_entropy, ckrl_stream_t stream) {
  int32_t st = check_device();
  if (st) return st;
  CKRL_REQUIRE(num_chunks >= 0 && C >= 1 && M >= 1 && V >= 1 && (int64_t)C * M <= 8192,
               CKRL_ERR_LENGTH_MISMATCH, "bad token_stats dimensions");
  if (num_chunks == 0) return CKRL_OK;
  CKRL_REQUIRE(logits && tokens, CKRL_ERR_INVALID_ARGUMENT, "logits / tokens required");
  LossArgs a;
  std::memset(&a, 0, sizeof(a));
  a.mode = MODE_STATS;
  a.C = C;
  a.M = M;
  a.V = V;
  a.E = 1;
  a.Tc = (int)num_chunks;
  a.n_rec = num_chunks;
  a.logits_bf16 = logits_dtype == CKRL_DTYPE_BF16;
  a.tok_i32 = token_dtype == CKRL_DTYPE_I32;
  a.logits = logits;
  a.tokens = tokens;
  a.tok_lp = token_logprob;
  a.tok_ent = token_entropy;
  a.action_lp = action_logprob;
  a.chunk_lp = chunk_logprob;
  a.action_ent = action_entropy;
  a.chunk_ent = chunk_entropy;
  a.stats_mask = slot_mask;
  a.all_rows = 1;
  a.world = 0;
  if (logits_dtype == CKRL_DTYPE_TOKEN_ROWS) {
    CKRL_REQUIRE((reinterpret_cast<uintptr_t>(logits) & 15) == 0, CKRL_ERR_INVALID_ARGUMENT,
                 "token rows must be 16-byte aligned");
    a.rows_in = static_cast<const ckrl_token_row*>(logits);
  } else {
    CKRL_REQUIRE(logits_dtype == CKRL_DTYPE_F32 || logits_dtype == CKRL_DTYPE_BF16, CKRL_ERR_INVALID_ARGUMENT,
                 "logits dtype must be f32, bf16 or token rows");
  }
  CKRL_CUDA(launch_tile(a, (cudaStream_t)stream, nullptr));
  return CKRL_OK;
}

// Row N2: policy head on the tensor cores + per-position reduction (csrc/proj.cu).
int32_t ckrl_project_token_stats(int64_t rows, const ckrl_policy_head* head, int32_t token_dtype,
                                 const void* tokens, ckrl_token_row* token_rows, double* token_logprob,
                                 float* token_entropy, int32_t logits_dtype, void* logits,
                                 ckrl_stream_t stream) {
  int32_t st = check_device();
  if (st) return st;
  CKRL_REQUIRE(head != nullptr, CKRL_ERR_INVALID_ARGUMENT, "policy head is null");
  CKRL_REQUIRE(rows >= 0 && rows <= (int64_t)INT32_MAX, CKRL_ERR_LENGTH_MISMATCH, "rows out of range");
  CKRL_REQUIRE(head->vocab == 256, CKRL_ERR_LENGTH_MISMATCH, "the projection kernel needs vocab == 256");
  CKRL_REQUIRE(head->hidden >= 64 && head->hidden <= 16384 && head->hidden % 64 == 0,
               CKRL_ERR_LENGTH_MISMATCH, "hidden must be a multiple of 64 in [64, 16384]");
  CKRL_REQUIRE(token_dtype == CKRL_DTYPE_U8 || token_dtype == CKRL_DTYPE_I32, CKRL_ERR_INVALID_ARGUMENT,
               "token dtype must be u8 or i32");
  CKRL_REQUIRE(!logits || logits_dtype == CKRL_DTYPE_F32 || logits_dtype == CKRL_DTYPE_BF16,
               CKRL_ERR_INVALID_ARGUMENT, "logits output dtype must be f32 or bf16");
  if (rows == 0) return CKRL_OK;
  CKRL_REQUIRE(head->feature && head->w_pol && tokens, CKRL_ERR_INVALID_ARGUMENT,
               "feature, w_pol and tokens are required");
  CKRL_REQUIRE(((reinterpret_cast<uintptr_t>(head->feature) | reinterpret_cast<uintptr_t>(head->w_pol)) & 15) == 0,
               CKRL_ERR_INVALID_ARGUMENT, "feature / w_pol must be 16-byte aligned");
  CKRL_REQUIRE((reinterpret_cast<uintptr_t>(token_rows) & 15) == 0, CKRL_ERR_INVALID_ARGUMENT,
               "token rows must be 16-byte aligned");
  CKRL_CUDA(launch_proj_stats(rows, head->hidden, head->feature, head->w_pol, head->b_pol, tokens,
                              token_dtype == CKRL_DTYPE_I32, token_rows, token_logprob, token_entropy, logits,
                              logits_dtype == CKRL_DTYPE_BF16, 0, (cudaStream_t)stream));
  return CKRL_OK;
}

int32_t ckrl_logits_grad(int64_t rows, int32_t V, int32_t logits_dtype, const void* logits,
                         int32_t token_dtype, const void* tokens, const float* coeff_lp,
                         const float* coeff_ent, int32_t out_dtype, void* dlogits,
                         int32_t* status_device, ckrl_stream_t stream) {
  int32_t st = check_device();
  if (st) return st;
  CKRL_REQUIRE(rows >= 0 && V >= 1, CKRL_ERR_LENGTH_MISMATCH, "bad logits_grad dimensions");
  if (rows == 0) return CKRL_OK;
  CKRL_REQUIRE(logits && tokens && coeff_lp && dlogits, CKRL_ERR_INVALID_ARGUMENT,
               "logits / tokens / coeff_lp / dlogits required");
  CKRL_REQUIRE((logits_dtype == CKRL_DTYPE_F32 || logits_dtype == CKRL_DTYPE_BF16) &&
                   (out_dtype == CKRL_DTYPE_F32 || out_dtype == CKRL_DTYPE_BF16) &&
                   (token_dtype == CKRL_DTYPE_U8 || token_dtype == CKRL_DTYPE_I32),
               CKRL_ERR_INVALID_ARGUMENT, "unsupported dtype");
  CKRL_REQUIRE(token_dtype == CKRL_DTYPE_I32 || V <= 256, CKRL_ERR_INVALID_ARGUMENT,
               "u8 tokens need vocab <= 256");
  CKRL_REQUIRE(dlogits != logits || out_dtype == logits_dtype, CKRL_ERR_INVALID_ARGUMENT,
               "in-place logits_grad needs matching dtypes");
  CKRL_CUDA(launch_logits_grad(logits, logits_dtype == CKRL_DTYPE_BF16, tokens, token_dtype == CKRL_DTYPE_I32,
                               coeff_lp, coeff_ent, rows, V, dlogits, out_dtype == CKRL_DTYPE_BF16,
                               status_device, (cudaStream_t)stream));
  return CKRL_OK;
}

int32_t ckrl_read_status(const int32_t* status_device, ckrl_stream_t stream) {
  CKRL_REQUIRE(status_device, CKRL_ERR_INVALID_ARGUMENT, "null status");
  int32_t host = 0;
  CKRL_CUDA(cudaMemcpyAsync(&host, status_device, sizeof(int32_t), cudaMemcpyDeviceToHost,
                            (cudaStream_t)stream));
  CKRL_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  if (host == CKRL_ERR_NON_FINITE) return fail(host, "non-finite gradient coefficient");
  if (host) return fail(host, "device-side error");
  return CKRL_OK;
}

size_t ckrl_adam_workspace_bytes(void) { return adam_workspace_bytes(); }

int32_t ckrl_adam_step(int32_t dtype, int64_t n, void* params, void* grad, void* exp_avg,
                       void* exp_avg_sq, const ckrl_adam_params* p, int64_t t, double* norm_device,
                       int32_t* status_device, void* workspace, size_t workspace_bytes,
                       ckrl_comm* comm, ckrl_stream_t stream) {
  int32_t st = check_device();
  if (st) return st;
  CKRL_REQUIRE(p && workspace, CKRL_ERR_INVALID_ARGUMENT, "params / workspace required");
  CKRL_REQUIRE(workspace_bytes >= adam_workspace_bytes(), CKRL_ERR_INVALID_ARGUMENT, "workspace too small");
  CKRL_REQUIRE(dtype == CKRL_DTYPE_F32 || dtype == CKRL_DTYPE_F64, CKRL_ERR_INVALID_ARGUMENT,
               "Adam state dtype must be f32 or f64");
  CKRL_REQUIRE(n >= 0 && t >= 1, CKRL_ERR_INVALID_ARGUMENT, "n >= 0 and step t >= 1 required");
  CKRL_REQUIRE(n == 0 || (params && grad && exp_avg && exp_avg_sq), CKRL_ERR_INVALID_ARGUMENT,
               "params / grad / moments required");
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  const int f64 = dtype == CKRL_DTYPE_F64;
  // adam.cpp:29-30: bias corrections with the host's pow, as the reference computes them
  const double bc1 = 1.0 - std::pow(p->beta1, (double)t), bc2 = 1.0 - std::pow(p->beta2, (double)t);
  CKRL_CUDA(launch_adam_norm(f64, grad, n, ws, s));
  const bool shard = comm && comm->world > 1;
  CKRL_REQUIRE(!shard || comm->nc, CKRL_ERR_INVALID_ARGUMENT,
               "a sharded Adam step needs an NCCL communicator (ckrl_comm_create with a unique id)");
  if (shard)
    CKRL_NCCL(nccl().AllReduce(adam_norm_sq_slot(ws), adam_norm_sq_slot(ws), 1, ncclFloat64, ncclSum,
                               comm->nc, s));
  CKRL_CUDA(launch_adam_update(f64, params, grad, exp_avg, exp_avg_sq, n, p->learning_rate, p->max_grad_norm,
                               p->beta1, p->beta2, p->eps, bc1, bc2, ws, norm_device, status_device,
                               shard ? 0 : 1, s));
  return CKRL_OK;
}

int32_t ckrl_dump_slab(int32_t E, int32_t Tc, int32_t C, int32_t M, int32_t token_dtype, const void* tokens,
                       const double* reward, const uint8_t* flags, const int32_t* episode_id,
                       int32_t first_env_id, char* out, size_t capacity, size_t* length) {
  CKRL_REQUIRE(E >= 0 && Tc >= 0 && C >= 1 && M >= 1, CKRL_ERR_LENGTH_MISMATCH, "bad slab dimensions");
  CKRL_REQUIRE(length, CKRL_ERR_INVALID_ARGUMENT, "length output required");
  CKRL_REQUIRE((int64_t)E * Tc == 0 || (tokens && reward && flags && episode_id), CKRL_ERR_INVALID_ARGUMENT,
               "slab arrays required");
  CKRL_REQUIRE(token_dtype == CKRL_DTYPE_U8 || token_dtype == CKRL_DTYPE_I32, CKRL_ERR_INVALID_ARGUMENT,
               "token dtype must be u8 or i32");
  std::string text;
  CKRL_REQUIRE(first_env_id >= 0, CKRL_ERR_INVALID_ARGUMENT, "first_env_id must be >= 0");
  format_slab(E, Tc, C, M, token_dtype, tokens, reward, flags, episode_id, first_env_id, text);
  *length = text.size();
  if (out && capacity) {
    const size_t n = text.size() < capacity ? text.size() : capacity;
    std::memcpy(out, text.data(), n);
    if (n < capacity) out[n] = '\0';
  }
  return CKRL_OK;
}

int32_t ckrl_save_checkpoint(const ckrl_policy_desc* d, const double* params, const char* path) {
  CKRL_REQUIRE(d && path, CKRL_ERR_INVALID_ARGUMENT, "descriptor / path required");
  const int64_t n = policy_num_params(*d);
  CKRL_REQUIRE(n >= 0, CKRL_ERR_CONFIG, "bad policy descriptor");
  CKRL_REQUIRE(n == 0 || params, CKRL_ERR_INVALID_ARGUMENT, "parameters required");
  std::string err;
  const int32_t st = write_checkpoint(*d, params, n, path, err);
  return st ? fail(st, err) : CKRL_OK;
}

int32_t ckrl_load_checkpoint(const char* path, ckrl_policy_desc* d, double* params, int64_t capacity,
                             int64_t* count) {
  CKRL_REQUIRE(path && d && count, CKRL_ERR_INVALID_ARGUMENT, "path / descriptor / count required");
  std::string err;
  const int32_t st = read_checkpoint(path, d, params, capacity, count, err);
  return st ? fail(st, err) : CKRL_OK;
}

static bool fused_enabled() {
  static int on = -1;
  if (on < 0) {
    // The fused single-launch step (GAE on the buffer warps + grid barrier) measured
    // slower on B200 (cfg3: 72.6 us vs 51.5 us for assemble + loss): the GAE's serial
    // chains crawl on SMs whose issue slots the row warps saturate. Opt-in only.
    const char* env = getenv("CKRL_FUSED_STEP");
    on = (env && env[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

// Overlapped (PDL) PPO step on/off (CKRL_ASM_SMS=0 disables). The assembly CTAs co-reside
// with the loss kernel's CTAs, so no SMs are reserved (reserved_sms = 0 below).
static int overlap_sms() {
  static int n = -1;
  if (n < 0) {
    const char* env = getenv("CKRL_ASM_SMS");
    n = env ? atoi(env) : 1;
  }
  return n;
}

// Pipelined steps: each batch's loss launched as a programmatic dependent of the previous
// launch on its stream (the previous batch's loss), so its logits stream while that loss's
// tail runs; the unit phase still waits for the predecessor (griddepcontrol.wait), so a
// same-stream assembly or any producer that does not trigger early stays a full dependency.
// CKRL_CHAIN=0 disables (A/B).
static int chain_enabled() {
  static int n = -1;
  if (n < 0) {
    const char* env = getenv("CKRL_CHAIN");
    n = env ? atoi(env) : 2;
  }
  return n;
}

// Launch policy of the pipelined halves' losses (ckrl_*_step_loss; the callers alternate them
// over two streams, optim.Pipelined). Measured per step on B200:
//  * grid cap: consecutive losses run side by side on disjoint SMs when each leaves SMs free.
//    PPO launches of 12..32 56-KB tiles per SM use 60 % of the SMs (cfg3 33.1 -> 26.8 us, with
//    the 14-row-warp CTA, csrc/loss.cu), 8..12 a third (cfg3 bf16 21.0 -> 19.2 us with the
//    losses over 3 streams; roughly 27-30 tiles per CTA in both bands), below 8 a quarter (cfg1
//    14.7 -> 10.8 us); GRPO losses of 8..12 tiles per SM use 3/7 of the SMs (cfg2 bf16 22.3 ->
//    20.8 us), other GRPO losses leave 6 SMs free, where the next
//    batch's single-CTA (1024-thread) group kernel runs (cfg2 32.9 -> 26.7 us, cfg4 bf16 241 -> 228 us);
//    long PPO launches keep one CTA per SM.
//  * chaining (programmatic dependent launch of the previous loss on the stream): on, except
//    uncapped launches of 8..64 tiles per SM (there the early-launched CTAs hold the SMs the
//    next assembly needs).
// CKRL_LOSS_CTAS overrides the cap (0 = one CTA per SM, N = N CTAs), CKRL_CHAIN the chaining
// (0 never, 1 always, 2 = policy, the default).
static int loss_cta_knob() {
  static int n = -2;
  if (n == -2) {
    const char* env = getenv("CKRL_LOSS_CTAS");
    n = env ? atoi(env) : -1;  // -1: policy
  }
  return n;
}
static int device_sm_count() {
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}
static double tiles_per_sm(const ckrl_rollout* ro, const ckrl_policy_outputs* po) {
  const double bytes = (double)ro->num_envs * ro->num_chunks * ro->chunk_len * ro->tokens_per_action *
                       ro->vocab * (po->logits_dtype == CKRL_DTYPE_BF16 ? 2 : 4);
  return bytes / (56.0 * 1024) / device_sm_count();
}
// cap: the communicator's cap (several ranks on one device) or 0
static int pipelined_cap(const ckrl_rollout* ro, const ckrl_policy_outputs* po, bool grpo, int cap) {
  const int k = loss_cta_knob();
  int want = 0;
  if (k >= 0) {
    want = k;
  } else if (po->logits_dtype != CKRL_DTYPE_TOKEN_ROWS) {
    const int sms = device_sm_count();
    const double t = tiles_per_sm(ro, po);
    if (grpo) want = (t >= 8.0 && t < 12.0) ? (sms * 3) / 7 : sms - 6;  // cfg2 bf16: 22.3 -> 20.8 us
    else if (t < 8.0) want = sms / 4;  // tiny launches: a quarter (cfg1 12.7 -> 12.3 us)
    else if (t < 12.0) want = sms / 3;  // cfg3 bf16 (9 tiles / SM), 3 loss streams: 21.0 -> 19.2 us
    else if (t <= 32.0) want = (sms * 3) / 5;
  }
  if (want <= 0) return cap;
  return (cap == 0 || want < cap) ? want : cap;
}
static bool chain_loss(const ckrl_rollout* ro, const ckrl_policy_outputs* po, bool capped) {
  const int mode = chain_enabled();
  if (mode == 0 || po->logits_dtype == CKRL_DTYPE_TOKEN_ROWS) return false;
  if (mode == 1 || capped) return true;
  const double per_sm = tiles_per_sm(ro, po);
  return per_sm < 8.0 || per_sm > 64.0;
}

static LossArgs ppo_args(const ckrl_rollout* ro, const ckrl_ppo_batch* b,
                         const ckrl_policy_outputs* po, const ckrl_granularity* spec,
                         const ckrl_ppo_params* p, ckrl_loss_outputs* out, double* diag, void* ws,
                         int world, const StatsRecord* recs, int finalize) {
  LossArgs a = base_args(ro, po, (char*)ws, world);
  a.mode = MODE_PPO;
  a.counted = b->counted;
  a.adv = b->advantages;
  a.ret = b->returns;
  a.new_values = po->values;
  a.adv_level = spec->advantage_level;
  a.lp_level = spec->logprob_level;
  a.val_level = spec->value_level;
  a.clip = p->clip_eps;
  a.vcoef = p->value_loss_coef;
  a.ecoef = p->entropy_coef;
  a.normalize = p->advantage_normalization;
  a.recs = recs;
  a.diag = diag;
  a.finalize = finalize;
  set_outputs(a, out);
  return a;
}

static int32_t ppo_loss_impl(const ckrl_rollout* ro, const ckrl_ppo_batch* b,
                             const ckrl_policy_outputs* po, const ckrl_granularity* spec,
                             const ckrl_ppo_params* p, ckrl_loss_outputs* out, double* diag,
                             void* ws, int world, const StatsRecord* recs, int finalize,
                             cudaStream_t s) {
  LossArgs a = base_args(ro, po, (char*)ws, world);
  a.mode = MODE_PPO;
  a.counted = b->counted;
  a.adv = b->advantages;
  a.ret = b->returns;
  a.new_values = po->values;
  a.adv_level = spec->advantage_level;
  a.lp_level = spec->logprob_level;
  a.val_level = spec->value_level;
  a.clip = p->clip_eps;
  a.vcoef = p->value_loss_coef;
  a.ecoef = p->entropy_coef;
  a.normalize = p->advantage_normalization;
  a.recs = recs;
  a.diag = diag;
  a.finalize = finalize;
  set_outputs(a, out);
  CKRL_CUDA(launch_tile(a, s, nullptr));
  return CKRL_OK;
}

int32_t ckrl_ppo_loss(const ckrl_rollout* ro, const ckrl_ppo_batch* b,
                      const ckrl_policy_outputs* po, const ckrl_granularity* spec,
                      const ckrl_ppo_params* p, ckrl_loss_outputs* out, double* diag,
                      void* ws, size_t ws_bytes, ckrl_stream_t stream) {
  int32_t st = validate(spec);
  if (st) return st;
  if ((st = check_device())) return st;
  if ((st = check_rollout(ro, false))) return st;
  if ((st = check_policy(ro, po, out))) return st;
  if ((st = check_ws(ws, ws_bytes, ro->num_envs, 1))) return st;
  CKRL_REQUIRE(b && p && diag && b->counted && b->advantages && b->returns,
               CKRL_ERR_INVALID_ARGUMENT, "batch / params / diag required");
  CKRL_REQUIRE(p->value_loss_coef == 0.0 || po->values, CKRL_ERR_INVALID_ARGUMENT,
               "new values required when value_loss_coef != 0");
  WsLayout L = ws_layout(ro->num_envs, 1);
  return ppo_loss_impl(ro, b, po, spec, p, out, diag, ws, 1,
                       reinterpret_cast<const StatsRecord*>((char*)ws + L.stats_local), 1,
                       (cudaStream_t)stream);
}

static int32_t grpo_loss_impl(const ckrl_rollout* ro, const ckrl_grpo_batch* gb,
                              const ckrl_policy_outputs* po, const ckrl_granularity* spec,
                              const ckrl_grpo_params* p, ckrl_loss_outputs* out, double* diag,
                              void* ws, int world, const StatsRecord* recs, int finalize,
                              cudaStream_t s, int pdl = 0, const ExchangeView& ex = ExchangeView{},
                              int max_ctas = 0) {
  LossArgs a = base_args(ro, po, (char*)ws, world);
  a.ex = ex;
  a.max_ctas = max_ctas;
  if (pdl) {  // programmatic dependent of the GRPO assembly (grpo_weights_kernel)
    a.pdl = 1;
    a.ro = *ro;
  }
  a.mode = MODE_GRPO;
  a.adv_level = spec->advantage_level;
  a.lp_level = spec->logprob_level;
  a.val_level = spec->value_level;
  a.clip = p->clip_eps;
  a.env_group = gb->env_group;
  a.env_adv = gb->env_advantage;
  a.env_group_size = gb->env_group_size;
  a.slot_weight = gb->slot_weight;
  a.slot_member = gb->slot_member;
  a.recs = recs;
  a.diag = diag;
  a.finalize = finalize;
  set_outputs(a, out);
  a.coeff_ent = nullptr;
  a.coeff_val = nullptr;
  CKRL_CUDA(launch_tile(a, s, nullptr));
  if (out && out->coeff_entropy)
    CKRL_CUDA(cudaMemsetAsync(out->coeff_entropy, 0,
                              sizeof(float) * (size_t)a.n_rec * a.C * a.M, s));
  return CKRL_OK;
}

int32_t ckrl_grpo_loss(const ckrl_rollout* ro, const ckrl_grpo_batch* gb,
                       const ckrl_policy_outputs* po, const ckrl_granularity* spec,
                       const ckrl_grpo_params* p, ckrl_loss_outputs* out, double* diag,
                       void* ws, size_t ws_bytes, ckrl_stream_t stream) {
  int32_t st = validate(spec);
  if (st) return st;
  if ((st = check_device())) return st;
  if ((st = check_rollout(ro, false))) return st;
  if ((st = check_policy(ro, po, out))) return st;
  if ((st = check_ws(ws, ws_bytes, ro->num_envs, 1))) return st;
  CKRL_REQUIRE(gb && p && diag, CKRL_ERR_INVALID_ARGUMENT, "batch / params / diag required");
  WsLayout L = ws_layout(ro->num_envs, 1);
  return grpo_loss_impl(ro, gb, po, spec, p, out, diag, ws, 1,
                        reinterpret_cast<const StatsRecord*>((char*)ws + L.stats_local), 1,
                        (cudaStream_t)stream);
}

static int32_t check_comm(const ckrl_comm* comm) {
  if (comm && comm->world > 1 && !comm->ready)
    return fail(CKRL_ERR_INVALID_ARGUMENT,
                "communicator peers not opened (ckrl_comm_open_peers / ckrl_comm_set_peers)");
  if (comm && comm->world > 1) {
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != comm->device) return fail(CKRL_ERR_INVALID_ARGUMENT, "communicator belongs to another device");
  }
  return CKRL_OK;
}

// The whole step. Multi-rank (comm->world > 1): the assembly kernel's last CTA stores the
// rank's stats record into every rank's exchange buffer (NVLink P2P stores) and the loss
// kernel -- still the assembly's programmatic dependent, streaming logits from the start --
// waits for all records before its first unit phase; its last CTA exchanges the raw loss
// sums the same way and finalises the diagnostics. No NCCL kernel and no extra launch.
int32_t ckrl_ppo_step(const ckrl_rollout* ro, const ckrl_policy_outputs* po,
                      const ckrl_gae_params* gae, const ckrl_granularity* spec,
                      const ckrl_ppo_params* p, ckrl_ppo_batch* b, ckrl_loss_outputs* out,
                      double* diag, void* ws, size_t ws_bytes, ckrl_comm* comm,
                      ckrl_stream_t stream) {
  int32_t st = validate(spec);
  if (st) return st;
  if (spec->value_level != spec->advantage_level)
    return fail(CKRL_ERR_CONFIG, "value_type must match reward_type for GAE assembly");
  if ((st = check_device())) return st;
  if ((st = check_rollout(ro, true))) return st;
  if ((st = check_policy(ro, po, out))) return st;
  if ((st = check_comm(comm))) return st;
  const int world = comm ? comm->world : 1;
  if ((st = check_ws(ws, ws_bytes, ro->num_envs, world))) return st;
  CKRL_REQUIRE(gae && p && b && diag && b->counted && b->advantages && b->returns,
               CKRL_ERR_INVALID_ARGUMENT, "gae / params / batch / diag required");
  CKRL_REQUIRE(p->value_loss_coef == 0.0 || po->values, CKRL_ERR_INVALID_ARGUMENT,
               "new values required when value_loss_coef != 0");
  cudaStream_t s = (cudaStream_t)stream;
  WsLayout L = ws_layout(ro->num_envs, world);
  char* w = (char*)ws;
  const ExchangeView ex = exchange_view(comm);
  const StatsRecord* local = reinterpret_cast<const StatsRecord*>(w + L.stats_local);
  if (world == 1 && fused_enabled() && !(out && out->dlogits)) {
    // one persistent launch: GAE assembly overlapped with the logits stream
    LossArgs a = ppo_args(ro, b, po, spec, p, out, diag, ws, 1, local, 1);
    a.ro = *ro;
    a.gamma = gae->gamma;
    a.lambda = gae->lambda;
    cudaError_t e = launch_ppo_fused(a, s, nullptr);
    if (e == cudaSuccess) return CKRL_OK;
    if (e != cudaErrorNotSupported) return fail(CKRL_ERR_CUDA, std::string("fused step: ") + cudaGetErrorString(e));
    cudaGetLastError();
  }
  CKRL_CUDA(launch_ppo_assemble(*ro, spec->advantage_level == CKRL_LEVEL_ACTION, gae->gamma,
                                gae->lambda, *b, w, L, s, ex));
  // the loss as the assembly's programmatic dependent: logits stream while the GAE scan
  // runs; the unit phases start once the assembly's outputs (and every rank's record) exist
  LossArgs a = ppo_args(ro, b, po, spec, p, out, diag, ws, 1, local, 1);
  a.ex = ex;
  a.max_ctas = loss_cta_cap(comm);
  if (overlap_sms() > 0 && po->logits_dtype >= 0) {
    a.pdl = 1;
    a.ro = *ro;
  }
  CKRL_CUDA(launch_tile(a, s, nullptr));
  return CKRL_OK;
}

int32_t ckrl_grpo_step(const ckrl_rollout* ro, const ckrl_episodes* ep,
                       const ckrl_policy_outputs* po, const ckrl_granularity* spec,
                       const ckrl_grpo_options* opt, const ckrl_grpo_params* p,
                       ckrl_grpo_batch* gb, ckrl_loss_outputs* out, double* diag, void* ws,
                       size_t ws_bytes, ckrl_comm* comm, ckrl_stream_t stream) {
  int32_t st = validate(spec);
  if (st) return st;
  if ((st = check_device())) return st;
  if ((st = check_rollout(ro, false))) return st;
  if ((st = check_policy(ro, po, out))) return st;
  if ((st = check_comm(comm))) return st;
  const int world = comm ? comm->world : 1;
  if ((st = check_ws(ws, ws_bytes, ro->num_envs, world))) return st;
  CKRL_REQUIRE(ep && opt && p && gb && diag, CKRL_ERR_INVALID_ARGUMENT,
               "episodes / options / params / batch / diag required");
  cudaStream_t s = (cudaStream_t)stream;
  WsLayout L = ws_layout(ro->num_envs, world);
  char* w = (char*)ws;
  const ExchangeView ex = exchange_view(comm);
  CKRL_CUDA(launch_grpo_assemble(*ro, *ep, *opt, *gb, w, L, s, ex));
  return grpo_loss_impl(ro, gb, po, spec, p, out, diag, ws, 1,
                        reinterpret_cast<const StatsRecord*>(w + L.stats_local), 1, s,
                        overlap_sms() > 0 && po->logits_dtype >= 0, ex, loss_cta_cap(comm));
}

// The two halves of a step, for callers that pipeline batches (the assembly of batch i+1 on
// one stream while batch i's loss runs on another, each batch with its own workspace): the
// same kernels as ckrl_*_step, the loss launched as a plain kernel after its assembly.
int32_t ckrl_ppo_step_assemble(const ckrl_rollout* ro, const ckrl_gae_params* gae,
                               const ckrl_granularity* spec, ckrl_ppo_batch* b, void* ws,
                               size_t ws_bytes, ckrl_comm* comm, ckrl_stream_t stream) {
  int32_t st = validate(spec);
  if (st) return st;
  if (spec->value_level != spec->advantage_level)
    return fail(CKRL_ERR_CONFIG, "value_type must match reward_type for GAE assembly");
  if ((st = check_device())) return st;
  if ((st = check_rollout(ro, true))) return st;
  if ((st = check_comm(comm))) return st;
  const int world = comm ? comm->world : 1;
  if ((st = check_ws(ws, ws_bytes, ro->num_envs, world))) return st;
  CKRL_REQUIRE(gae && b && b->counted && b->advantages && b->returns, CKRL_ERR_INVALID_ARGUMENT,
               "gae / batch required");
  CKRL_CUDA(launch_ppo_assemble(*ro, spec->advantage_level == CKRL_LEVEL_ACTION, gae->gamma, gae->lambda,
                                *b, (char*)ws, ws_layout(ro->num_envs, world), (cudaStream_t)stream,
                                exchange_view(comm)));
  return CKRL_OK;
}

int32_t ckrl_ppo_step_loss(const ckrl_rollout* ro, const ckrl_policy_outputs* po,
                           const ckrl_granularity* spec, const ckrl_ppo_params* p,
                           const ckrl_ppo_batch* b, ckrl_loss_outputs* out, double* diag, void* ws,
                           size_t ws_bytes, ckrl_comm* comm, ckrl_stream_t stream) {
  int32_t st = validate(spec);
  if (st) return st;
  if ((st = check_device())) return st;
  if ((st = check_rollout(ro, false))) return st;
  if ((st = check_policy(ro, po, out))) return st;
  if ((st = check_comm(comm))) return st;
  const int world = comm ? comm->world : 1;
  if ((st = check_ws(ws, ws_bytes, ro->num_envs, world))) return st;
  CKRL_REQUIRE(b && p && diag && b->counted && b->advantages && b->returns, CKRL_ERR_INVALID_ARGUMENT,
               "batch / params / diag required");
  CKRL_REQUIRE(p->value_loss_coef == 0.0 || po->values, CKRL_ERR_INVALID_ARGUMENT,
               "new values required when value_loss_coef != 0");
  WsLayout L = ws_layout(ro->num_envs, world);
  LossArgs a = ppo_args(ro, b, po, spec, p, out, diag, ws, 1,
                        reinterpret_cast<const StatsRecord*>((char*)ws + L.stats_local), 1);
  a.ex = exchange_view(comm);
  const int comm_cap = loss_cta_cap(comm);
  a.max_ctas = pipelined_cap(ro, po, false, comm_cap);
  if (chain_loss(ro, po, a.max_ctas != comm_cap)) {
    a.pdl = 1;
    a.ro = *ro;
  }
  CKRL_CUDA(launch_tile(a, (cudaStream_t)stream, nullptr));
  return CKRL_OK;
}

int32_t ckrl_grpo_step_assemble(const ckrl_rollout* ro, const ckrl_episodes* ep,
                                const ckrl_granularity* spec, const ckrl_grpo_options* opt,
                                ckrl_grpo_batch* gb, void* ws, size_t ws_bytes, ckrl_comm* comm,
                                ckrl_stream_t stream) {
  int32_t st = validate(spec);
  if (st) return st;
  if ((st = check_device())) return st;
  if ((st = check_rollout(ro, false))) return st;
  if ((st = check_comm(comm))) return st;
  const int world = comm ? comm->world : 1;
  if ((st = check_ws(ws, ws_bytes, ro->num_envs, world))) return st;
  CKRL_REQUIRE(ep && opt && gb, CKRL_ERR_INVALID_ARGUMENT, "episodes / options / batch required");
  CKRL_CUDA(launch_grpo_assemble(*ro, *ep, *opt, *gb, (char*)ws, ws_layout(ro->num_envs, world),
                                 (cudaStream_t)stream, exchange_view(comm)));
  return CKRL_OK;
}

int32_t ckrl_grpo_step_loss(const ckrl_rollout* ro, const ckrl_policy_outputs* po,
                            const ckrl_granularity* spec, const ckrl_grpo_params* p,
                            const ckrl_grpo_batch* gb, ckrl_loss_outputs* out, double* diag, void* ws,
                            size_t ws_bytes, ckrl_comm* comm, ckrl_stream_t stream) {
  int32_t st = validate(spec);
  if (st) return st;
  if ((st = check_device())) return st;
  if ((st = check_rollout(ro, false))) return st;
  if ((st = check_policy(ro, po, out))) return st;
  if ((st = check_comm(comm))) return st;
  const int world = comm ? comm->world : 1;
  if ((st = check_ws(ws, ws_bytes, ro->num_envs, world))) return st;
  CKRL_REQUIRE(gb && p && diag, CKRL_ERR_INVALID_ARGUMENT, "batch / params / diag required");
  WsLayout L = ws_layout(ro->num_envs, world);
  return grpo_loss_impl(ro, gb, po, spec, p, out, diag, ws, 1,
                        reinterpret_cast<const StatsRecord*>((char*)ws + L.stats_local), 1,
                        (cudaStream_t)stream,
                        chain_loss(ro, po, pipelined_cap(ro, po, true, loss_cta_cap(comm)) != loss_cta_cap(comm)),
                        exchange_view(comm), pipelined_cap(ro, po, true, loss_cta_cap(comm)));
}

int32_t ckrl_read_diagnostics(const double* diag_device, double* diag_host, ckrl_stream_t stream) {
  CKRL_REQUIRE(diag_device && diag_host, CKRL_ERR_INVALID_ARGUMENT, "null diagnostics");
  CKRL_CUDA(cudaMemcpyAsync(diag_host, diag_device, sizeof(double) * CKRL_DIAG_COUNT,
                            cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CKRL_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  int status = (int)diag_host[CKRL_DIAG_STATUS];
  if (status == CKRL_ERR_SKIP_UPDATE) return fail(status, "no GRPO groups retained");
  if (status == CKRL_ERR_DEGENERATE_GROUP)
    return fail(status, "all trajectories in the group have equal return");
  if (status == CKRL_ERR_NON_FINITE) return fail(status, "loss is not finite");
  if (status) return fail(status, "device-side error");
  return CKRL_OK;
}

int32_t ckrl_select_records(const ckrl_rollout* src, const ckrl_ppo_batch* sb, const ckrl_policy_outputs* sp,
                            const ckrl_granularity* spec, int64_t n, const int64_t* idx,
                            const ckrl_rollout* dst, const ckrl_ppo_batch* db, const ckrl_policy_outputs* dp,
                            void* ws, size_t ws_bytes, ckrl_stream_t stream) {
  int32_t st = validate(spec);
  if (st) return st;
  if ((st = check_device())) return st;
  if ((st = check_rollout(src, false))) return st;
  if ((st = check_rollout(dst, false))) return st;
  CKRL_REQUIRE(sb && db && sp && dp && dp->logits && sb->counted && db->counted &&
                   sb->advantages && db->advantages && sb->returns && db->returns,
               CKRL_ERR_INVALID_ARGUMENT, "batches / policy outputs required");
  CKRL_REQUIRE(n >= 1 && n <= INT32_MAX && idx, CKRL_ERR_INVALID_ARGUMENT, "empty record selection");
  CKRL_REQUIRE(dst->num_envs == n && dst->num_chunks == 1 && dst->chunk_len == src->chunk_len &&
                   dst->tokens_per_action == src->tokens_per_action && dst->vocab == src->vocab &&
                   dst->token_dtype == src->token_dtype && dp->logits_dtype == sp->logits_dtype,
               CKRL_ERR_LENGTH_MISMATCH, "selection view must be [n][1] with the source's C, M, V, dtypes");
  CKRL_REQUIRE(!sp->values || dp->values, CKRL_ERR_INVALID_ARGUMENT, "dst values required");
  if ((st = check_ws(ws, ws_bytes, (int)n, 1))) return st;
  CKRL_CUDA(launch_select_records(*src, *sb, *sp, spec->advantage_level == CKRL_LEVEL_ACTION,
                                  spec->value_level == CKRL_LEVEL_ACTION, n, idx, *dst, *db, *dp,
                                  (char*)ws, (cudaStream_t)stream));
  return CKRL_OK;
}

int32_t ckrl_read_stats(const void* ws, size_t ws_bytes, int32_t E, double* sums, int64_t* counts,
                        ckrl_stream_t stream) {
  int32_t st = check_device();
  if (st) return st;
  if ((st = check_ws(const_cast<void*>(ws), ws_bytes, E, 1))) return st;
  StatsRecord r;
  CKRL_CUDA(cudaMemcpyAsync(&r, (const char*)ws + ws_layout(E, 1).stats_local, sizeof(r), cudaMemcpyDeviceToHost,
                            (cudaStream_t)stream));
  CKRL_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  if (sums) {
    sums[0] = r.mean;
    sums[1] = r.m2;
  }
  if (counts) {
    counts[0] = r.n_adv;
    counts[1] = r.n_adv;
    counts[2] = r.n_val;
    counts[3] = r.n_pos;
    counts[4] = r.groups_retained;
    counts[5] = r.status;
  }
  if (r.status == CKRL_ERR_DEGENERATE_GROUP) return fail((int32_t)r.status, "all trajectories in the group have equal return");
  if (r.status) return fail((int32_t)r.status, "device-side error");
  return CKRL_OK;
}

int32_t ckrl_select_groups(int32_t E, const int32_t* src, int32_t* dst, int32_t n, const int32_t* sel,
                           void* ws, size_t ws_bytes, ckrl_stream_t stream) {
  int32_t st = check_device();
  if (st) return st;
  CKRL_REQUIRE(E >= 0 && n >= 0 && (E == 0 || (src && dst)) && (n == 0 || sel), CKRL_ERR_INVALID_ARGUMENT,
               "bad group selection");
  if ((st = check_ws(ws, ws_bytes, E, 1))) return st;
  CKRL_CUDA(launch_select_groups(E, src, dst, n, sel, (char*)ws, (cudaStream_t)stream));
  return CKRL_OK;
}

int32_t ckrl_grpo_group_advantage(int32_t G, const int32_t* off, const double* R, double eps,
                                  double* adv, int32_t* status, ckrl_stream_t stream) {
  CKRL_REQUIRE(G >= 0 && (G == 0 || (off && R && adv)), CKRL_ERR_INVALID_ARGUMENT, "bad group arguments");
  int32_t st;
  if ((st = check_device())) return st;
  CKRL_CUDA(launch_group_advantage(G, off, R, eps, adv, status, (cudaStream_t)stream));
  return CKRL_OK;
}

int32_t ckrl_success_rate_filter(int32_t G, const int32_t* off, const double* R, double lower,
                                 double upper, uint8_t* keep, double* mean, ckrl_stream_t stream) {
  CKRL_REQUIRE(G >= 0 && (G == 0 || (off && R)), CKRL_ERR_INVALID_ARGUMENT, "bad group arguments");
  int32_t st;
  if ((st = check_device())) return st;
  CKRL_CUDA(launch_success_filter(G, off, R, lower, upper, keep, mean, (cudaStream_t)stream));
  return CKRL_OK;
}

int32_t ckrl_valid_action_mask(int32_t n, const int64_t* off, const uint8_t* success,
                               const int64_t* fs, uint8_t* mask, ckrl_stream_t stream) {
  CKRL_REQUIRE(n >= 0 && (n == 0 || (off && success && fs)), CKRL_ERR_INVALID_ARGUMENT,
               "bad episode arguments");
  int32_t st;
  if ((st = check_device())) return st;
  CKRL_CUDA(launch_mask_weights(n, off, success, fs, 1, mask, nullptr, (cudaStream_t)stream));
  return CKRL_OK;
}

int32_t ckrl_length_norm_weights(int32_t n, const int64_t* off, const uint8_t* success,
                                 const int64_t* fs, int32_t normalized, double* w,
                                 ckrl_stream_t stream) {
  CKRL_REQUIRE(n >= 0 && (n == 0 || (off && success && fs)), CKRL_ERR_INVALID_ARGUMENT,
               "bad episode arguments");
  int32_t st;
  if ((st = check_device())) return st;
  CKRL_CUDA(launch_mask_weights(n, off, success, fs, normalized, nullptr, w, (cudaStream_t)stream));
  return CKRL_OK;
}

int32_t ckrl_slab_success_rate(const ckrl_episodes* eps, double* out, ckrl_stream_t stream) {
  CKRL_REQUIRE(eps && out && eps->count >= 0 && (eps->count == 0 || (eps->complete && eps->first_success)),
               CKRL_ERR_INVALID_ARGUMENT, "bad episode table");
  int32_t st;
  if ((st = check_device())) return st;
  CKRL_CUDA(launch_success_rate(eps->count, eps->complete, eps->first_success, out, (cudaStream_t)stream));
  return CKRL_OK;
}

int64_t ckrl_policy_num_params(const ckrl_policy_desc* d) { return d ? policy_num_params(*d) : -1; }

static int32_t check_pipeline(const ckrl_pipeline_spec* sp) {
  CKRL_REQUIRE(sp != nullptr, CKRL_ERR_INVALID_ARGUMENT, "pipeline spec is null");
  const ckrl_env_config& e = sp->env;
  const ckrl_policy_desc& p = sp->policy;
  CKRL_REQUIRE(e.kind == 0 || e.kind == 1, CKRL_ERR_CONFIG, "unknown env kind");
  CKRL_REQUIRE(e.num_envs >= 1, CKRL_ERR_CONFIG, "VecEnv needs at least one env");
  // vec_env.cpp:324-327, rollout.cpp:11-17
  CKRL_REQUIRE(sp->stages >= 1 && e.num_envs % sp->stages == 0, CKRL_ERR_CONFIG,
               "pipeline stage count must divide num_envs");
  CKRL_REQUIRE(p.obs_dim == (e.kind == 0 ? 6 : 2), CKRL_ERR_LENGTH_MISMATCH, "observation dimension mismatch");
  CKRL_REQUIRE(p.chunk_len == e.chunk_len, CKRL_ERR_LENGTH_MISMATCH, "chunk length mismatch");
  CKRL_REQUIRE(p.tokens_per_action >= 2 || e.kind == 1, CKRL_ERR_CONFIG, "toy_reach needs 2 tokens per action");
  CKRL_REQUIRE(p.hidden >= 1 && p.value_hidden >= 1 && p.vocab >= 1 && p.trunk_layers >= 0 &&
                   sp->num_chunks >= 1 && e.max_episode_steps >= 1 && e.grid_size >= 2,
               CKRL_ERR_CONFIG, "bad pipeline dimensions");
  CKRL_REQUIRE(!e.use_fixed_reset_state_ids || sp->reset_state_ids, CKRL_ERR_BAD_RESET_ID,
               "use_fixed_reset_state_ids requires reset_state_ids");
  CKRL_REQUIRE(sp->sampler == CKRL_SAMPLER_REFERENCE || sp->sampler == CKRL_SAMPLER_PARALLEL,
               CKRL_ERR_CONFIG, "unknown sampler");
  return CKRL_OK;
}

int32_t ckrl_placement_mode(int32_t num_slots, int32_t env_begin, int32_t env_end, int32_t rollout_begin,
                            int32_t rollout_end, int32_t actor_begin, int32_t actor_end,
                            int32_t pipeline_stage_num, int32_t* status) {
  auto bad = [&](const std::string& msg) {
    if (status) *status = CKRL_ERR_INVALID_PLAN;
    fail(CKRL_ERR_INVALID_PLAN, msg);
    return -1;
  };
  if (status) *status = CKRL_OK;
  // validate_plan (placement/plan.cpp:49-58) + SlotRange::parse's end >= begin (:27-28)
  if (num_slots < 1) return bad("cluster needs at least one slot");
  const int32_t r[3][2] = {{env_begin, env_end}, {rollout_begin, rollout_end}, {actor_begin, actor_end}};
  for (const auto& q : r) {
    if (q[1] < q[0]) return bad("bad slot range");
    if (q[0] < 0 || q[1] >= num_slots) return bad("slot range outside cluster");
  }
  if (pipeline_stage_num < 1) return bad("pipeline_stage_num must be >= 1");
  // derive_mode (:60-68)
  auto same = [](const int32_t* a, const int32_t* b) { return a[0] == b[0] && a[1] == b[1]; };
  auto overlaps = [](const int32_t* a, const int32_t* b) { return a[0] <= b[1] && b[0] <= a[1]; };
  if (same(r[0], r[1]) && same(r[1], r[2])) return CKRL_PLACEMENT_COLOCATED;
  const bool disjoint = !overlaps(r[0], r[1]) && !overlaps(r[0], r[2]) && !overlaps(r[1], r[2]);
  return disjoint ? CKRL_PLACEMENT_DISAGGREGATED : CKRL_PLACEMENT_HYBRID;
}

size_t ckrl_pipeline_gen_workspace_bytes(const ckrl_pipeline_spec* sp) {
  return check_pipeline(sp) == CKRL_OK ? pipeline_gen_ws_bytes(*sp) : 0;
}

size_t ckrl_pipeline_workspace_bytes(const ckrl_pipeline_spec* sp) {
  return check_pipeline(sp) == CKRL_OK ? pipeline_ws_bytes(*sp) : 0;
}

int32_t ckrl_pipeline_run(const ckrl_pipeline_spec* sp, const double* params,
                          ckrl_pipeline_outputs* out, void* ws, size_t ws_bytes,
                          ckrl_stream_t stream) {
  int32_t st = check_pipeline(sp);
  if (st) return st;
  if ((st = check_device())) return st;
  CKRL_REQUIRE(params && out && ws, CKRL_ERR_INVALID_ARGUMENT, "params / outputs / workspace required");
  CKRL_REQUIRE(ws_bytes >= pipeline_ws_bytes(*sp), CKRL_ERR_INVALID_ARGUMENT, "pipeline workspace too small");
  if (sp->placed) {
    int n = 0;
    cudaGetDeviceCount(&n);
    CKRL_REQUIRE(sp->gen_device >= 0 && sp->gen_device < n, CKRL_ERR_INVALID_ARGUMENT, "gen_device out of range");
    CKRL_REQUIRE(sp->gen_workspace && sp->gen_workspace_bytes >= pipeline_gen_ws_bytes(*sp),
                 CKRL_ERR_INVALID_ARGUMENT, "generation workspace missing or too small");
  }
  CKRL_CUDA(pipeline_run(*sp, params, *out, (char*)ws, (cudaStream_t)stream));
  return CKRL_OK;
}

int32_t ckrl_debug_cta_times(uint64_t* out, int32_t n) {
  CKRL_CUDA(cudaDeviceSynchronize());
  CKRL_CUDA(debug_cta_times(out, n));
  return CKRL_OK;
}

int32_t ckrl_debug_timeline(uint64_t* out, int32_t n) {
  CKRL_REQUIRE(out && n > 0, CKRL_ERR_INVALID_ARGUMENT, "bad timeline buffer");
  CKRL_CUDA(cudaDeviceSynchronize());
  CKRL_CUDA(read_timeline(out, n));
  return CKRL_OK;
}

int32_t ckrl_comm_unique_id(void* out_id) {
  CKRL_REQUIRE(out_id, CKRL_ERR_INVALID_ARGUMENT, "null id buffer");
  if (!nccl().ok) return fail(CKRL_ERR_NCCL, "NCCL library not found");
  ncclUniqueId id;
  CKRL_NCCL(nccl().GetUniqueId(&id));
  std::memcpy(out_id, &id, sizeof(id));
  return CKRL_OK;
}

int32_t ckrl_comm_create(int32_t world, int32_t rank, const void* unique_id, ckrl_comm** out) {
  CKRL_REQUIRE(out && world >= 1 && world <= kMaxRanks && rank >= 0 && rank < world,
               CKRL_ERR_INVALID_ARGUMENT, "bad communicator arguments");
  int32_t st = check_device();
  if (st) return st;
  ckrl_comm* c = new ckrl_comm;
  c->world = world;
  c->rank = rank;
  cudaGetDevice(&c->device);
  const size_t xb = ex_buffer_bytes(world);
  cudaError_t e = cudaMalloc(&c->xbuf, xb);
  if (e == cudaSuccess) e = cudaMemset(c->xbuf, 0, xb);
  if (e == cudaSuccess) e = cudaMalloc(&c->peers_dev, sizeof(char*) * (size_t)world);
  if (e != cudaSuccess) {
    ckrl_comm_destroy(c);
    return fail(CKRL_ERR_CUDA, std::string("exchange buffer: ") + cudaGetErrorString(e));
  }
  if (world == 1) c->ready = true;
  if (unique_id) {  // NCCL communicator too (Adam's sharded gradient norm)
    if (!nccl().ok) {
      ckrl_comm_destroy(c);
      return fail(CKRL_ERR_NCCL, "NCCL library not found");
    }
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    ncclResult_t r = nccl().CommInitRank(&c->nc, world, id, rank);
    if (r != ncclSuccess) {
      c->nc = nullptr;
      ckrl_comm_destroy(c);
      return fail(CKRL_ERR_NCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
    }
  }
  *out = c;
  return CKRL_OK;
}

int32_t ckrl_comm_ipc_handle(ckrl_comm* comm, void* out_handle) {
  CKRL_REQUIRE(comm && out_handle, CKRL_ERR_INVALID_ARGUMENT, "communicator / handle buffer required");
  static_assert(sizeof(cudaIpcMemHandle_t) == CKRL_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  CKRL_CUDA(cudaIpcGetMemHandle(&h, comm->xbuf));
  std::memcpy(out_handle, &h, sizeof(h));
  return CKRL_OK;
}

static int32_t install_peers(ckrl_comm* c, const std::vector<char*>& ptrs, int co_resident) {
  CKRL_CUDA(cudaMemcpy(c->peers_dev, ptrs.data(), sizeof(char*) * ptrs.size(), cudaMemcpyHostToDevice));
  c->co_resident = co_resident;
  c->ready = true;
  return CKRL_OK;
}

int32_t ckrl_comm_open_peers(ckrl_comm* comm, const void* handles) {
  CKRL_REQUIRE(comm && handles, CKRL_ERR_INVALID_ARGUMENT, "communicator / handles required");
  CKRL_REQUIRE(!comm->ready || comm->world == 1, CKRL_ERR_INVALID_ARGUMENT, "peers already opened");
  std::vector<char*> ptrs((size_t)comm->world, nullptr);
  const cudaIpcMemHandle_t* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
  int same = 1;
  for (int q = 0; q < comm->world; ++q) {
    if (q == comm->rank) {
      ptrs[q] = comm->xbuf;
      continue;
    }
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, hs[q], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return fail(CKRL_ERR_CUDA, "cudaIpcOpenMemHandle(rank " + std::to_string(q) + "): " + cudaGetErrorString(e));
    comm->ipc_opened.push_back((char*)p);
    ptrs[q] = (char*)p;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.device == comm->device) ++same;
    cudaGetLastError();
  }
  return install_peers(comm, ptrs, same);
}

int32_t ckrl_comm_set_peers(ckrl_comm* comm, ckrl_comm* const* comms) {
  CKRL_REQUIRE(comm && comms, CKRL_ERR_INVALID_ARGUMENT, "communicator / peers required");
  std::vector<char*> ptrs((size_t)comm->world, nullptr);
  int same = 0;
  for (int q = 0; q < comm->world; ++q) {
    CKRL_REQUIRE(comms[q] && comms[q]->world == comm->world && comms[q]->rank == q,
                 CKRL_ERR_INVALID_ARGUMENT, "peer communicators must be ranks 0..world-1 of one world");
    if (comms[q]->device != comm->device) {  // one process driving several GPUs: direct P2P
      int dev = 0;
      cudaGetDevice(&dev);
      cudaSetDevice(comm->device);
      cudaError_t e = cudaDeviceEnablePeerAccess(comms[q]->device, 0);
      cudaSetDevice(dev);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(CKRL_ERR_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
      cudaGetLastError();
    }
    ptrs[q] = comms[q]->xbuf;
    same += comms[q]->device == comm->device;
  }
  return install_peers(comm, ptrs, same);
}

int32_t ckrl_comm_destroy(ckrl_comm* comm) {
  if (!comm) return CKRL_OK;
  if (comm->nc && nccl().ok) nccl().CommDestroy(comm->nc);
  for (char* p : comm->ipc_opened) cudaIpcCloseMemHandle(p);
  if (comm->peers_dev) cudaFree(comm->peers_dev);
  if (comm->xbuf) cudaFree(comm->xbuf);
  delete comm;
  return CKRL_OK;
}

}  // extern "C"
