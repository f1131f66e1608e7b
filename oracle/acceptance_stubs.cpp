// TEST INFRASTRUCTURE ONLY — the two harness/config.cpp functions the reference's acceptance
// suite links through harness/metrics.cpp (metadata for its metrics JSON: the config text and
// its hash). config.cpp itself needs yaml-cpp, which is not in this image; nothing the
// acceptance criteria check depends on these values.
#include <cstdint>
#include <string>

#include "chunkrl/harness/config.hpp"

namespace chunkrl::harness {
std::string serialize_config(const RunConfig&) { return "{}"; }
std::uint64_t config_hash(const RunConfig&) { return 0; }
}  // namespace chunkrl::harness
