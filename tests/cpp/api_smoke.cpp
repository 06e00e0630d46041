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
  // TuckerFormat with identity bases (a lossless, trivially orthonormal
  // format of t): NTFK save / load round trip on the host
  ntfb::TuckerFormat fmt;
  fmt.core_shape = spec.shape;
  fmt.core = t;
  for (int d : spec.shape) {
    ntfb::Matrix u(d, d);
    for (int i = 0; i < d; ++i) u(i, i) = 1.0;
    fmt.bases.push_back(u);
  }
  const std::string path = argc > 2 ? argv[2] : "/tmp/ntf_api_smoke.ntfk";
  fmt.save(path);
  const ntfb::TuckerFormat back = ntfb::TuckerFormat::load(path);
  if (back.core != fmt.core || back.core_shape != fmt.core_shape || back.bases.size() != 3) return 4;
  std::printf("ntfk roundtrip ok\n");
  if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) {
    ntfb::Context ctx(0);
    ntfb::GpuDenseProvider prov(ctx, t.data(), spec.shape);
    cfg.max_outer_iters = 10;
    auto [model, trace] = ntfb::her_run(prov, init, cfg, p);
    std::printf("f0=%.17g f10=%.17g restarts=%d\n", trace.f0, trace.final_f(), trace.restart_count());
    ntfb::TuckerProvider tp(ctx, back);
    auto [tmodel, ttrace] = ntfb::her_run(tp, init, cfg, p);
    std::printf("tucker f0=%.17g f10=%.17g restarts=%d\n", ttrace.f0, ttrace.final_f(), ttrace.restart_count());
  }
  return 0;
}
