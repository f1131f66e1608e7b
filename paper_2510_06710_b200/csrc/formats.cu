// (f3) Wire and on-disk formats of the SoA slab and the policy parameters, host side:
//   * dump_slab (core/types.cpp:9-28): the reference's trajectories.txt text, one line per
//     atomic slot "env uid step tok.. reward(%.17g) terminated truncated valid", so a GPU
//     rollout (ckrl_pipeline_run, downloaded) diffs byte-for-byte against the reference's
//     own dump (proj/null/trajectories.txt and tooling);
//   * the CKRL checkpoint (policy/checkpoint.cpp:37-83): "CKRL", u32 version 1, 7 i32
//     descriptor fields, u64 count, count little-endian f64 parameters in the reference's
//     flat layout (policy_net.cpp:107-152) — the layout ckrl_pipeline_run consumes.
// Text formatting and file I/O are host work; nothing here touches the device.
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "kernels.h"

namespace ckrl {
namespace {

constexpr char kCkptMagic[4] = {'C', 'K', 'R', 'L'};
constexpr uint32_t kCkptVersion = 1;

template <typename T>
void put_le(std::string& out, T v) {
  using U = std::make_unsigned_t<T>;
  U u = static_cast<U>(v);
  for (size_t i = 0; i < sizeof(T); ++i) out.push_back(static_cast<char>((u >> (8 * i)) & 0xff));
}
template <typename T>
bool get_le(FILE* f, T& v) {
  using U = std::make_unsigned_t<T>;
  unsigned char b[sizeof(T)];
  if (std::fread(b, 1, sizeof(T), f) != sizeof(T)) return false;
  U u = 0;
  for (size_t i = 0; i < sizeof(T); ++i) u |= static_cast<U>(b[i]) << (8 * i);
  v = static_cast<T>(u);
  return true;
}

}  // namespace

// Appends the dump_slab text of the SoA slab to `out`.
int32_t format_slab(int32_t E, int32_t Tc, int32_t C, int32_t M, int32_t token_dtype, const void* tokens,
                    const double* reward, const uint8_t* flags, const int32_t* episode_id, int32_t first_env_id,
                    std::string& out) {
  char buf[64];
  out += "# env_id episode_uid step tokens[" + std::to_string(M) + "] reward terminated truncated valid\n";
  for (int32_t e = 0; e < E; ++e) {
    int64_t step = 0;
    for (int32_t t = 0; t < Tc; ++t)
      for (int32_t j = 0; j < C; ++j, ++step) {
        const int64_t sl = ((int64_t)e * Tc + t) * C + j;
        const int32_t id = episode_id[sl];
        // uid = global env id << 32 | k (envsim/vec_env.cpp:14-16, the env id is first_env_id + i
        // for a VecEnv partition, vec_env.cpp:94); -1 marks a frozen slot
        const int64_t uid =
            id < 0 ? -1 : (int64_t)(((uint64_t)(uint32_t)(first_env_id + e) << 32) | (uint32_t)id);
        int n = std::snprintf(buf, sizeof buf, "%d %" PRId64 " %" PRId64, e, uid, step);
        out.append(buf, (size_t)n);
        for (int32_t m = 0; m < M; ++m) {
          const int64_t k = sl * M + m;
          const int tok = token_dtype == CKRL_DTYPE_I32 ? static_cast<const int32_t*>(tokens)[k]
                                                        : (int)static_cast<const uint8_t*>(tokens)[k];
          n = std::snprintf(buf, sizeof buf, " %d", tok);
          out.append(buf, (size_t)n);
        }
        const uint8_t f = flags[sl];
        n = std::snprintf(buf, sizeof buf, " %.17g %d %d %d\n", reward[sl], (f & CKRL_FLAG_TERMINATED) ? 1 : 0,
                          (f & CKRL_FLAG_TRUNCATED) ? 1 : 0, (f & CKRL_FLAG_VALID) ? 1 : 0);
        out.append(buf, (size_t)n);
      }
  }
  return CKRL_OK;
}

int32_t write_checkpoint(const ckrl_policy_desc& d, const double* params, int64_t count, const char* path,
                         std::string& err) {
  std::string bytes;
  bytes.append(kCkptMagic, 4);
  put_le<uint32_t>(bytes, kCkptVersion);
  for (int32_t field : {d.obs_dim, d.hidden, d.trunk_layers, d.value_hidden, d.vocab, d.chunk_len,
                        d.tokens_per_action})
    put_le<int32_t>(bytes, field);
  put_le<uint64_t>(bytes, (uint64_t)count);
  for (int64_t i = 0; i < count; ++i) {
    uint64_t u;
    std::memcpy(&u, params + i, 8);
    put_le<uint64_t>(bytes, u);
  }
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    err = std::string("cannot open checkpoint for writing: ") + path;
    return CKRL_ERR_GENERIC;
  }
  const bool ok = std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size();
  if (std::fclose(f) != 0 || !ok) {
    err = std::string("checkpoint write failed: ") + path;
    return CKRL_ERR_GENERIC;
  }
  return CKRL_OK;
}

int32_t read_checkpoint(const char* path, ckrl_policy_desc* d, double* params, int64_t capacity,
                        int64_t* count_out, std::string& err) {
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    err = std::string("cannot open checkpoint: ") + path;
    return CKRL_ERR_GENERIC;
  }
  struct Closer {
    FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{f};
  char magic[4];
  if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, kCkptMagic, 4) != 0) {
    err = std::string("bad checkpoint magic: ") + path;
    return CKRL_ERR_GENERIC;
  }
  uint32_t version = 0;
  if (!get_le(f, version) || version != kCkptVersion) {
    err = "unsupported checkpoint version " + std::to_string(version);
    return CKRL_ERR_GENERIC;
  }
  int32_t fields[7];
  for (int32_t& x : fields)
    if (!get_le(f, x)) {
      err = std::string("truncated checkpoint: ") + path;
      return CKRL_ERR_GENERIC;
    }
  *d = ckrl_policy_desc{fields[0], fields[1], fields[2], fields[3], fields[4], fields[5], fields[6]};
  uint64_t count = 0;
  if (!get_le(f, count)) {
    err = std::string("truncated checkpoint: ") + path;
    return CKRL_ERR_GENERIC;
  }
  if ((int64_t)count != policy_num_params(*d)) {
    err = "checkpoint parameter count mismatch";
    return CKRL_ERR_GENERIC;
  }
  *count_out = (int64_t)count;
  if (!params) return CKRL_OK;  // size query
  if ((int64_t)count > capacity) {
    err = "checkpoint parameter buffer too small";
    return CKRL_ERR_INVALID_ARGUMENT;
  }
  for (uint64_t i = 0; i < count; ++i) {
    uint64_t u;
    if (!get_le(f, u)) {
      err = std::string("truncated checkpoint: ") + path;
      return CKRL_ERR_GENERIC;
    }
    std::memcpy(params + i, &u, 8);
  }
  return CKRL_OK;
}

}  // namespace ckrl
