// Golden vectors for paper_2510_06710_b200/synth.py's restatement of the reference generator
// (chunkrl::Rng / mix_seed, proj/src/chunkrl/core/rng.hpp). Build and run in the build
// container (needs /root/reference):
//   g++ -std=c++17 -O2 -I/root/reference/proj/src tests/golden/gen_rng.cpp -o /tmp/gen_rng
//   /tmp/gen_rng > tests/golden/rng_vectors.json
#include "chunkrl/core/rng.hpp"
#include <cstdio>
int main() {
  std::printf("{\n");
  const unsigned long long seeds[3][2] = {{4, 5}, {4, 6}, {11, 1000003}};
  for (int s = 0; s < 3; ++s) {
    const std::uint64_t seed = chunkrl::mix_seed(seeds[s][0], seeds[s][1]);
    std::printf(" \"%llu_%llu\": {\"seed\": %llu,", seeds[s][0], seeds[s][1], (unsigned long long)seed);
    chunkrl::Rng a(seed), b(seed), c(seed), d(seed);
    std::printf(" \"u64\": [");
    for (int i = 0; i < 16; ++i) std::printf("%s\"%llu\"", i ? ", " : "", (unsigned long long)a.next_u64());
    std::printf("], \"double\": [");
    for (int i = 0; i < 16; ++i) std::printf("%s%.17g", i ? ", " : "", b.next_double());
    std::printf("], \"below251\": [");
    for (int i = 0; i < 16; ++i) std::printf("%s%llu", i ? ", " : "", (unsigned long long)c.next_below(251));
    std::printf("], \"normal\": [");
    for (int i = 0; i < 64; ++i) std::printf("%s%.17g", i ? ", " : "", d.next_normal());
    std::printf("]}%s\n", s < 2 ? "," : "");
  }
  std::printf("}\n");
}
