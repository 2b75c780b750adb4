// cpp_dropin.cpp -- a C++ caller of the reference operator API switched to the
// B200 library: the body of the reference CLI's per-head `run` path
// (pbs_main.cpp:197-232 calls pbs::pbs_attention on Matrix<float>) with the
// call replaced by pbs_b200::pbs_attention_host on the same row-major buffers.
//
//   g++ -std=c++17 -O2 -Iinclude examples/cpp_dropin.cpp \
//       -Lpaper_2510_21270_b200 -lpbs_b200 -Wl,-rpath,$PWD/paper_2510_21270_b200 -o cpp_dropin
//   ./cpp_dropin [N] [d]
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "pbs_b200.hpp"

int main(int argc, char** argv) {
  const std::size_t n = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 4096;
  const int d = argc > 2 ? std::atoi(argv[2]) : 128;
  std::mt19937_64 rng(1);
  std::normal_distribution<float> nd;
  std::vector<float> q(n * d), k(n * d), v(n * d), out(n * d);
  for (auto* m : {&q, &k, &v})
    for (auto& x : *m) x = nd(rng);
  pbs_b200::PipelineConfig cfg;  // B=128, S=256, tau=0.9, key_permute (pipeline.hpp:30-38)
  cfg.block_size = 64;           // BASELINE configs[0]: B=64
  const std::size_t t = (n + cfg.block_size - 1) / cfg.block_size;
  std::vector<int32_t> sigma(n), pi(n);
  std::vector<uint8_t> mask(t * t);
  try {
    const auto rep = pbs_b200::pbs_attention_host(q.data(), k.data(), v.data(), n, d, cfg, out.data(),
                                                  sigma.data(), pi.data(), mask.data());
    std::printf("{\"block_density\": %.6f, \"causal_density_baseline\": %.6f, \"selected_blocks\": %lld, "
                "\"attention_us\": %.1f}\n",
                rep.block_density, rep.causal_density_baseline, (long long)rep.selected_blocks, rep.attention_us);
  } catch (const pbs_b200::Error& e) {
    std::fprintf(stderr, "%s\n", e.what());  // the CLI's single-line E_* format
    return e.exit_code();
  }
  return 0;
}
