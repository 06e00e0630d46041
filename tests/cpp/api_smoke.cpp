// Compiles against include/ntf_b200.hpp and links libntf_b200.so: the
// reference-shaped C++ API (validation, datagen) works without a GPU, and
// with one, her_run runs end to end (exercised by the -m gpu suite).
#include <cstdio>
#include <cstring>

#include "ntf_b200.hpp"

int main(int argc, char** argv) {
  ntfb::HerParams p;
  p.validate();
  bool threw = false;
  try {
    ntfb::HerParams bad;
    bad.beta0 = 0.0;
    bad.validate();
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  if (!threw) return 2;
  ntfb::AoConfig cfg;
  threw = false;
  try {
    cfg.validate();
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  if (!threw) return 3;
  ntfb::SyntheticSpec spec{{6, 5, 4}, 3, 0.1, false, 42};
  auto [t, truth] = ntfb::generate(spec);
  auto init = ntfb::random_init(spec.shape, 3, ntfb::stream_seed(42, 1));
  double sum = 0.0;
  for (double x : t) sum += x;
  std::printf("sum=%.17g init00=%.17g\n", sum, init.factor(0)(0, 0));
  if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) {
    ntfb::Context ctx(0);
    ntfb::GpuDenseProvider prov(ctx, t.data(), spec.shape);
    cfg.max_outer_iters = 10;
    auto [model, trace] = ntfb::her_run(prov, init, cfg, p);
    std::printf("f0=%.17g f10=%.17g restarts=%d\n", trace.f0, trace.final_f(), trace.restart_count());
  }
  return 0;
}
