// facade_demo.cpp -- the reference's call sequence (model_run.cpp:129-156,
// forward_rank) written against esgnn_b200.hpp.  `--host-only` exercises the
// parts that need no GPU (parameter store, coupling tables, error mapping).
#include <cmath>
#include <cstdio>
#include <cstring>

#include "esgnn_b200.hpp"

using namespace esgnn;

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::strcmp(argv[1], "--host-only") == 0;
  b200::ModelConfig cfg;
  cfg.l_max = 4;
  cfg.e_width = 16;
  cfg.layers = 3;
  cfg.r_cut = 12.0;
  const std::map<int, std::vector<int>> basis{{72, {0, 0, 1, 2}}, {8, {0, 1}}};
  {
    b200::Network host(nullptr, cfg, basis);
    host.init_params();
    std::printf("params %zu out_len %d hash %016llx\n", host.params().size(), host.out_len(),
                (unsigned long long)host.value_hash());
    const auto c = b200::coupling_matrix(1, 1, 2);
    double n = 0;
    for (double v : c) n += v * v;
    std::printf("coupling(1,1,2) frobenius^2 %.12f\n", n);
    try {
      b200::ModelConfig bad = cfg;
      bad.l_max = 2;
      b200::Network x(nullptr, bad, basis);
      std::printf("missing UsageError\n");
      return 1;
    } catch (const UsageError& e) {
      std::printf("usage error mapped: %s\n", e.what());
    }
  }
  {  // extxyz round trip (read_extxyz_file / write_extxyz_file, extxyz.h:17-20)
    b200::AtomicStructure a;
    a.positions = {{0.0, 0.1, 0.2}, {1.25, -0.0, 3e-9}};
    a.species = {72, 8};
    a.cell = {4, 0, 0, 0, 4.5, 0, 0.25, 0, 5};
    a.pbc = {true, false, true};
    const std::string path = "facade_demo_roundtrip.xyz";
    b200::write_extxyz_file(path, a);
    const b200::AtomicStructure b = b200::read_extxyz_file(path);
    std::remove(path.c_str());
    if (b.positions != a.positions || b.species != a.species || b.cell != a.cell || b.pbc != a.pbc) {
      std::printf("extxyz round trip differs\n");
      return 1;
    }
    std::printf("extxyz round trip exact\n");
  }
  if (host_only) return 0;
  b200::Context ctx(0);
  b200::AtomicStructure s;
  int n = 4;  // 4x4x4 jittered-free HfO2-like lattice, 2.2 A spacing
  for (int i = 0; i < n * n * n; ++i) {
    s.positions.push_back({(i / 16 + 0.5) * 2.2, (i / 4 % 4 + 0.5) * 2.2, (i % 4 + 0.5) * 2.2});
    s.species.push_back(i % 3 == 0 ? 72 : 8);
  }
  s.cell = {n * 2.2, 0, 0, 0, n * 2.2, 0, 0, 0, n * 2.2};
  s.pbc = {true, true, true};
  auto g = b200::build_graph(ctx, s, 5.0);
  cfg.r_cut = 5.0;
  b200::Network net(&ctx, cfg, basis);
  net.init_params();
  net.prepare(*g, s.species);
  std::vector<float> no, eo;
  const auto t = net.forward(&no, &eo);
  std::printf("graph %d edges; forward %.3f ms, %lld kernels; node_out[0] %.6f\n", g->n_edges(), t.forward_ms,
              (long long)t.gpu_launches, no[0]);
  return std::isfinite(no[0]) ? 0 : 1;
}
