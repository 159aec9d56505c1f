// forward_rank_b200.cpp -- INTEGRATION.md's patch, compiled: the reference's
// tools/model_run.cpp::forward_rank (model_run.cpp:129-156) for one rank with
// its Network / build_graph calls switched to libesg_b200 through the
// header-only façade (paper_2507_03840_b200/csrc/esgnn_b200.hpp), driven by
// the reference's own input types (structures::AtomicStructure from
// model::make_jittered_lattice, structures::BasisSet, model::ModelConfig,
// partition::Assignment) and error classes (core/error.h).  Built by
// oracle/ref.mk against the reference headers; run by
// tests/test_gpu_integration.py.
//
//   forward_rank_b200 <out_dir> <C1|small>
// writes blocks_coupled.txt / blocks_uncoupled.txt (the reference's output
// files, through esg_blocks_write_text) and heads.bin (node then edge head
// outputs, float32) to out_dir; exits 0 when the device graph equals the
// reference's structures::build_graph bit for bit and a usage error
// surfaces as the reference's esgnn::UsageError.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "esgnn/core/error.h"
#include "esgnn/model/network.h"
#include "esgnn/model/synthetic.h"
#include "esgnn/partition/partition.h"
#include "esgnn/structures/basis.h"
#include "esgnn/structures/graph.h"
#include "esgnn_b200.hpp"

using namespace esgnn;

struct Inputs {  // model_run.cpp's Inputs, built from the reference's own generators
  structures::AtomicStructure s;
  structures::BasisSet basis;
  structures::Graph g;
  partition::Assignment assign;
};

// ---- the patched forward_rank
template <typename T>
int forward_rank(const model::ModelConfig& mc, const Inputs& in, const std::string& out_dir) {
  b200::Context ctx(/*device=*/0);                                   // one GPU per rank
  auto g = b200::build_graph(ctx, b200::to_b200(in.s), mc.r_cut);   // replaces structures::build_graph
  const structures::Graph rg = b200::to_reference(*g);
  bool same = rg.n_nodes == in.g.n_nodes && rg.edges.size() == in.g.edges.size();
  for (size_t k = 0; same && k < rg.edges.size(); ++k) {
    const auto &a = rg.edges[k], &b = in.g.edges[k];
    same = a.src == b.src && a.dst == b.dst && a.shift == b.shift && a.distance == b.distance &&
           a.displacement(0) == b.displacement(0) && a.displacement(1) == b.displacement(1) &&
           a.displacement(2) == b.displacement(2);
  }
  std::printf("device graph: %d edges, %s the reference's build_graph\n", g->n_edges(),
              same ? "bit-identical to" : "DIFFERENT from");
  auto plan = b200::build_comm_plan(*g, in.s.species, b200::to_b200(in.assign), /*rank=*/0);
  b200::Network net(&ctx, b200::to_b200(mc), b200::to_map(in.basis));
  net.init_params();                                                  // the same ParamStore values
  net.prepare(*g, in.s.species, plan.get());
  std::vector<float> node_out, edge_out;
  const esg_timing t = net.forward(&node_out, &edge_out);             // 2*M halo exchanges when world > 1
  // model_run.cpp:148-151: the output files, byte format of write_blocks_file
  net.write_blocks_text(out_dir + "/blocks_coupled.txt", ESG_BLOCKS_COUPLED);
  net.write_blocks_text(out_dir + "/blocks_uncoupled.txt", ESG_BLOCKS_UNCOUPLED);
  std::ofstream f(out_dir + "/heads.bin", std::ios::binary);
  f.write(reinterpret_cast<const char*>(node_out.data()), node_out.size() * sizeof(float));
  f.write(reinterpret_cast<const char*>(edge_out.data()), edge_out.size() * sizeof(float));
  std::printf("forward: %d nodes, %d edges, %.3f ms, %lld kernels -> %s\n", g->n_nodes, g->n_edges(), t.forward_ms,
              (long long)t.gpu_launches, out_dir.c_str());
  return same ? 0 : 1;
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: forward_rank_b200 <out_dir> <C1|small>\n");
    return 2;
  }
  const std::string out_dir = argv[1], which = argv[2];
  Inputs in;
  model::ModelConfig mc;
  mc.l_max = 4;
  mc.e_width = 16;
  mc.n_radial = 32;
  mc.seed = 1;
  if (which == "C1") {
    in.s = model::make_jittered_lattice(512, 2.71, 0.30, {14}, 1);
    in.basis.add_species(14, {0, 0, 1, 1, 2});
    mc.layers = 1;
    mc.r_cut = 8.0;
  } else {
    in.s = model::make_jittered_lattice(40, 2.2, 0.45, {72, 8, 8}, 4);
    in.basis.add_species(72, {0, 0, 1, 2});
    in.basis.add_species(8, {0, 1});
    mc.layers = 2;
    mc.r_cut = 4.5;
  }
  in.g = structures::build_graph(in.s, mc.r_cut);
  in.assign = {1, std::vector<int>(in.g.n_nodes, 0)};  // model_run.cpp:60, world 1
  // error taxonomy: the façade raises the reference's own classes
  try {
    model::ModelConfig bad = mc;
    bad.l_max = 1;
    b200::Network x(nullptr, b200::to_b200(bad), b200::to_map(in.basis));
    std::printf("missing esgnn::UsageError\n");
    return 1;
  } catch (const esgnn::UsageError& e) {
    std::printf("esgnn::UsageError (core/error.h) from the façade: %s\n", e.what());
  }
  try {
    return forward_rank<float>(mc, in, out_dir);
  } catch (const esgnn::Error& e) {
    std::fprintf(stderr, "esgnn::Error: %s\n", e.what());
    return 1;
  }
}
