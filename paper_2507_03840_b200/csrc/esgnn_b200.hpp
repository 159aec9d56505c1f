// esgnn_b200.hpp -- header-only C++ façade over include/esg.h that re-exposes
// the reference's model/graph API (names, argument meaning and exceptions) so
// reference call sites switch by changing a namespace:
//
//   esgnn::structures::build_graph      (graph.h:37)          -> esgnn::b200::build_graph
//   esgnn::partition::lownn_partition   (partition.h:24)      -> esgnn::b200::lownn_partition
//   esgnn::runtime::build_comm_plan     (comm_plan.h:35)      -> esgnn::b200::build_comm_plan
//   esgnn::model::Network<float>        (network.h:77-228)    -> esgnn::b200::Network
//   esgnn::runtime::DistributedRunner   (distributed.h:183)   -> Network::forward on a plan
//   esgnn::harmonics::coupling_matrix   (clebsch_gordan.h:19) -> esgnn::b200::coupling_matrix
//   esgnn::structures::read_extxyz_file (extxyz.h:17)         -> esgnn::b200::read_extxyz_file
//
// Errors are rethrown as the esgnn::Error taxonomy (core/error.h:11-51) --
// the reference's own classes when its headers are on the include path.
// With the reference headers present, to_b200(...) converts its
// AtomicStructure, Assignment and ModelConfig, to_map its BasisSet, and
// to_reference returns a device graph as a structures::Graph.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/esg.h"


// The error taxonomy is the reference's own (core/error.h:11-51) whenever its
// headers are on the include path -- the drop-in case, so reference call
// sites catch the same types -- and a same-named standalone copy otherwise.
#if __has_include(<esgnn/core/error.h>)
#include <esgnn/core/error.h>
#define ESGNN_B200_REFERENCE_TYPES 1
#else
#define ESGNN_B200_REFERENCE_TYPES 0
namespace esgnn {
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
class UsageError : public Error {
 public:
  using Error::Error;
};
class DataError : public Error {
 public:
  using Error::Error;
};
class ShapeError : public DataError {
 public:
  using DataError::DataError;
};
class TransportError : public Error {
 public:
  using Error::Error;
};
class DivergenceError : public Error {
 public:
  using Error::Error;
};
}  // namespace esgnn
#endif

namespace esgnn {
namespace b200 {

inline void check(int rc) {
  if (rc == ESG_OK) return;
  const std::string m = esg_last_error();
  switch (rc) {
    case ESG_ERR_USAGE: throw UsageError(m);
    case ESG_ERR_DATA: throw DataError(m);
    case ESG_ERR_DIVERGENCE: throw DivergenceError(m);
    case ESG_ERR_NCCL: throw TransportError(m);
    default: throw Error(m);
  }
}

// structures::AtomicStructure (structure.h:12-36), Eigen-free.
struct AtomicStructure {
  std::vector<std::array<double, 3>> positions;
  std::vector<int> species;
  std::array<double, 9> cell{1, 0, 0, 0, 1, 0, 0, 0, 1};  // rows = lattice vectors
  std::array<bool, 3> pbc{false, false, false};
  int n_atoms() const { return (int)positions.size(); }
  std::array<uint8_t, 3> pbc8() const { return {uint8_t(pbc[0]), uint8_t(pbc[1]), uint8_t(pbc[2])}; }
};

// structures::read_extxyz_file / write_extxyz_file (extxyz.h:17-20)
inline AtomicStructure read_extxyz_file(const std::string& path) {
  int64_t n = 0;
  check(esg_extxyz_read(path.c_str(), &n, nullptr, nullptr, nullptr, nullptr));
  std::vector<double> pos((size_t)n * 3);
  std::vector<int32_t> sp((size_t)n);
  AtomicStructure s;
  uint8_t pbc[3];
  check(esg_extxyz_read(path.c_str(), &n, pos.data(), sp.data(), s.cell.data(), pbc));
  s.positions.resize((size_t)n);
  for (int64_t i = 0; i < n; ++i) s.positions[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
  s.species.assign(sp.begin(), sp.end());
  for (int d = 0; d < 3; ++d) s.pbc[d] = pbc[d] != 0;
  return s;
}
inline void write_extxyz_file(const std::string& path, const AtomicStructure& s) {
  std::vector<double> pos;
  pos.reserve(3 * s.positions.size());
  for (const auto& p : s.positions) pos.insert(pos.end(), p.begin(), p.end());
  const std::vector<int32_t> sp(s.species.begin(), s.species.end());
  const auto pbc = s.pbc8();
  check(esg_extxyz_write(path.c_str(), (int64_t)s.n_atoms(), pos.data(), sp.data(), s.cell.data(), pbc.data()));
}

// structures::Edge (graph.h:14-20)
struct Edge {
  int src = 0, dst = 0;
  std::array<int, 3> shift{0, 0, 0};
  std::array<double, 3> displacement{0, 0, 0};
  double distance = 0.0;
};

class Context {
 public:
  explicit Context(int device = 0, int rank = 0, int world = 1, const void* nccl_id = nullptr) {
    check(esg_ctx_create(device, rank, world, nccl_id, &h_));
  }
  ~Context() { esg_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  esg_ctx* get() const { return h_; }

 private:
  esg_ctx* h_ = nullptr;
};

// structures::Graph (graph.h:22-32): device CSR, host edges on demand.
class Graph {
 public:
  Graph(Context& ctx, const AtomicStructure& s, double r_cut) {
    check(esg_build_graph(ctx.get(), s.n_atoms(), s.positions.empty() ? nullptr : s.positions[0].data(),
                          s.cell.data(), s.pbc8().data(), r_cut, &h_));
    check(esg_graph_info(h_, &n_nodes, &n_edges_));
  }
  ~Graph() { esg_graph_destroy(h_); }
  Graph(const Graph&) = delete;
  Graph& operator=(const Graph&) = delete;
  int n_nodes = 0;
  int n_edges() const { return (int)n_edges_; }
  std::vector<Edge> edges() const {
    std::vector<int32_t> src(n_edges_), dst(n_edges_), sh(3 * n_edges_);
    std::vector<double> disp(3 * n_edges_), dist(n_edges_);
    check(esg_graph_export(h_, src.data(), dst.data(), sh.data(), disp.data(), dist.data()));
    std::vector<Edge> out(n_edges_);
    for (int64_t k = 0; k < n_edges_; ++k) {
      out[k].src = src[k];
      out[k].dst = dst[k];
      out[k].shift = {sh[3 * k], sh[3 * k + 1], sh[3 * k + 2]};
      out[k].displacement = {disp[3 * k], disp[3 * k + 1], disp[3 * k + 2]};
      out[k].distance = dist[k];
    }
    return out;
  }
  std::vector<int> in_degrees() const {
    std::vector<int> d(n_nodes);
    check(esg_graph_in_degrees(h_, d.data()));
    return d;
  }
  const esg_graph* get() const { return h_; }

 private:
  esg_graph* h_ = nullptr;
  int64_t n_edges_ = 0;
};

inline std::unique_ptr<Graph> build_graph(Context& ctx, const AtomicStructure& s, double r_cut) {
  return std::make_unique<Graph>(ctx, s, r_cut);
}

// partition::Assignment / lownn_partition (partition.h:16-24)
struct Assignment {
  int n_parts = 1;
  std::vector<int> node_to_part;
};
inline Assignment lownn_partition(const AtomicStructure& s, const Graph& g, int depth, double r_cut) {
  Assignment a;
  a.n_parts = 1 << depth;
  a.node_to_part.resize(s.n_atoms());
  const auto deg = g.in_degrees();
  check(esg_lownn_partition(s.n_atoms(), s.positions[0].data(), s.cell.data(), s.pbc8().data(), deg.data(), depth,
                            r_cut, a.node_to_part.data()));
  return a;
}
// the same assignment computed on ctx's device (esg_lownn_partition_gpu)
inline Assignment lownn_partition(const Context& ctx, const AtomicStructure& s, const Graph& g, int depth,
                                  double r_cut) {
  Assignment a;
  a.n_parts = 1 << depth;
  a.node_to_part.resize(s.n_atoms());
  const auto deg = g.in_degrees();
  check(esg_lownn_partition_gpu(ctx.get(), s.n_atoms(), s.positions[0].data(), s.cell.data(), s.pbc8().data(),
                                deg.data(), depth, r_cut, a.node_to_part.data()));
  return a;
}

// runtime::CommPlan (comm_plan.h:15-35)
class CommPlan {
 public:
  CommPlan(const Graph& g, const std::vector<int>& species, const Assignment& a, int rank) : rank(rank) {
    check(esg_plan_build(g.get(), species.data(), a.node_to_part.data(), a.n_parts, rank, &h_));
    int64_t info[5];
    check(esg_plan_info(h_, info));
    n_rows = (int)info[0];
    n_owned = (int)info[1];
    n_neighbors = (int)info[3];
  }
  ~CommPlan() { esg_plan_destroy(h_); }
  CommPlan(const CommPlan&) = delete;
  CommPlan& operator=(const CommPlan&) = delete;
  int rank, n_rows = 0, n_owned = 0, n_neighbors = 0;
  const esg_plan* get() const { return h_; }

 private:
  esg_plan* h_ = nullptr;
};

inline std::unique_ptr<CommPlan> build_comm_plan(const Graph& g, const std::vector<int>& species,
                                                 const Assignment& a, int rank) {
  return std::make_unique<CommPlan>(g, species, a, rank);
}

// model::ModelConfig (network.h:16-35)
struct ModelConfig {
  int l_max = 2, e_width = 8, layers = 2, n_radial = 32;
  double r_cut = 4.0;
  uint64_t seed = 1;
  bool gate_enabled = true;
  int linear_precision = ESG_LINEAR_BF16;
};

// model::Network<float>: prepare + forward (+ halo exchanges when the
// context has world > 1), heads and uncoupled blocks.
class Network {
 public:
  Network(Context* ctx, const ModelConfig& c, const std::map<int, std::vector<int>>& basis) {
    esg_model_config cfg{c.l_max, c.e_width, c.layers, c.n_radial, c.r_cut, c.seed, c.gate_enabled ? 1 : 0,
                         c.linear_precision};
    std::vector<int> z, ns, sh;
    for (const auto& kv : basis) {
      z.push_back(kv.first);
      ns.push_back((int)kv.second.size());
      sh.insert(sh.end(), kv.second.begin(), kv.second.end());
    }
    check(esg_model_create(ctx ? ctx->get() : nullptr, &cfg, (int)z.size(), z.data(), ns.data(), sh.data(), &h_));
  }
  ~Network() { esg_model_destroy(h_); }
  Network(const Network&) = delete;
  Network& operator=(const Network&) = delete;

  void init_params() { check(esg_model_init_params(h_)); }
  std::vector<float> params() const {
    std::vector<float> p(esg_model_param_count(h_));
    check(esg_model_get_params(h_, p.data()));
    return p;
  }
  uint64_t value_hash() const { return esg_model_param_hash(h_); }
  int out_len() const { return esg_model_out_len(h_); }
  void prepare(const Graph& g, const std::vector<int>& species, const CommPlan* plan = nullptr) {
    check(esg_prepare(h_, g.get(), plan ? plan->get() : nullptr, species.data()));
    int64_t info[3];
    check(esg_prepared_info(h_, info));
    n_owned_ = info[1];
    n_edges_ = info[2];
  }
  // Heads of owned nodes (n_owned x out_len) and owned edges (n_edges x out_len).
  esg_timing forward(std::vector<float>* node_out = nullptr, std::vector<float>* edge_out = nullptr) {
    if (node_out) node_out->resize((size_t)n_owned_ * out_len());
    if (edge_out) edge_out->resize((size_t)n_edges_ * out_len());
    esg_timing t{};
    check(esg_forward(h_, node_out ? node_out->data() : nullptr, edge_out ? edge_out->data() : nullptr, &t));
    return t;
  }
  // ---- training (Network::build_targets/record_loss, DistributedRunner::train_step)
  void set_targets(const std::vector<float>& node_target, const std::vector<uint8_t>& node_mask,
                   const std::vector<float>& edge_target, const std::vector<uint8_t>& edge_mask) {
    check(esg_set_targets(h_, node_target.data(), node_mask.data(), edge_target.data(), edge_mask.data()));
  }
  double loss_grad(int64_t n_total, std::vector<float>* grads = nullptr) {
    double loss = 0, partials[3];
    if (grads) grads->resize(esg_model_param_count(h_));
    check(esg_loss_grad(h_, n_total, partials, &loss, grads ? grads->data() : nullptr));
    return loss;
  }
  double train_step(esg_adam* opt, int64_t n_total, esg_timing* t = nullptr) {
    double loss = 0;
    check(esg_train_step(h_, opt, n_total, &loss, t));
    return loss;
  }
  esg_model* get() const { return h_; }

  std::vector<double> blocks_uncoupled() {
    int64_t n = 0;
    check(esg_blocks_size(h_, &n));
    std::vector<double> out(n);
    check(esg_blocks_uncoupled(h_, out.data()));
    return out;
  }
  // ---- block export (model_run.cpp:141-153 output stage)
  void write_block_shard(const std::string& path, int basis = ESG_BLOCKS_UNCOUPLED, bool symmetrize = false,
                         int value_bytes = 8) {
    check(esg_blocks_write_shard(h_, path.c_str(), basis, symmetrize ? 1 : 0, value_bytes));
  }
  void write_blocks_text(const std::string& path, int basis = ESG_BLOCKS_UNCOUPLED, bool symmetrize = false) {
    check(esg_blocks_write_text(h_, path.c_str(), basis, symmetrize ? 1 : 0));
  }
  // ---- checkpoints (checkpoint.h:37-92, plus the optimizer state)
  void save_checkpoint(const std::string& path, const esg_adam* opt = nullptr, const std::string& config = "") const {
    check(esg_checkpoint_save(h_, opt, config.c_str(), path.c_str()));
  }
  std::string load_checkpoint(const std::string& path, esg_adam* opt = nullptr) {
    std::string cfg(1 << 16, '\0');
    check(esg_checkpoint_load(h_, opt, path.c_str(), cfg.data(), (int64_t)cfg.size()));
    cfg.resize(std::strlen(cfg.c_str()));
    return cfg;
  }

 private:
  esg_model* h_ = nullptr;
  int64_t n_owned_ = 0, n_edges_ = 0;
};

// model::Optimizer (optimizer.h): Adam, fp64 moments, reduce-on-plateau
class Adam {
 public:
  explicit Adam(const Network& net, const esg_adam_config* cfg = nullptr) { check(esg_adam_create(net.get(), cfg, &h_)); }
  ~Adam() { esg_adam_destroy(h_); }
  Adam(const Adam&) = delete;
  Adam& operator=(const Adam&) = delete;
  esg_adam* get() const { return h_; }
  double lr() const { return esg_adam_lr(h_); }

 private:
  esg_adam* h_ = nullptr;
};

// model_run.cpp:103-120 gather_blocks + write_blocks_file on rank 0, from the
// ranks' shard files (no device needed)
inline void merge_block_shards(const std::vector<std::string>& shards, const std::string& out_path) {
  std::vector<const char*> p;
  for (const auto& s : shards) p.push_back(s.c_str());
  check(esg_blocks_merge_text(p.data(), (int)p.size(), out_path.c_str()));
}

inline std::vector<double> coupling_matrix(int la, int lb, int L) {
  std::vector<double> c((size_t)(2 * L + 1) * (2 * la + 1) * (2 * lb + 1));
  check(esg_coupling_matrix(la, lb, L, c.data()));
  return c;
}

#if ESGNN_B200_REFERENCE_TYPES && __has_include(<esgnn/structures/structure.h>) && \
    __has_include(<esgnn/model/network.h>) && __has_include(<esgnn/partition/partition.h>)
// ---- converters from the reference's own types (drop-in call sites)
inline AtomicStructure to_b200(const esgnn::structures::AtomicStructure& s) {
  AtomicStructure o;
  o.positions.reserve(s.positions.size());
  for (const auto& p : s.positions) o.positions.push_back({p(0), p(1), p(2)});
  o.species = s.species;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.cell[3 * i + j] = s.cell(i, j);  // rows are lattice vectors, as the reference's
  o.pbc = {s.pbc[0], s.pbc[1], s.pbc[2]};
  return o;
}
inline Assignment to_b200(const esgnn::partition::Assignment& a) {
  Assignment o;
  o.n_parts = a.n_parts;
  o.node_to_part = a.node_to_part;
  return o;
}
inline ModelConfig to_b200(const esgnn::model::ModelConfig& c, int linear_precision = ESG_LINEAR_FP32) {
  ModelConfig o;
  o.l_max = c.l_max;
  o.e_width = c.e_width;
  o.layers = c.layers;
  o.n_radial = c.n_radial;
  o.r_cut = c.r_cut;
  o.seed = c.seed;
  o.gate_enabled = c.gate_enabled;
  o.linear_precision = linear_precision;
  return o;
}
inline std::map<int, std::vector<int>> to_map(const esgnn::structures::BasisSet& b) { return b.all(); }
// Graph::edges in the reference's value type, for call sites that keep
// using a structures::Graph (the device graph is bit-identical to it)
inline esgnn::structures::Graph to_reference(const Graph& g) {
  esgnn::structures::Graph r;
  r.n_nodes = g.n_nodes;
  for (const auto& e : g.edges()) {
    esgnn::structures::Edge x;
    x.src = e.src;
    x.dst = e.dst;
    x.shift = e.shift;
    x.displacement = Eigen::Vector3d(e.displacement[0], e.displacement[1], e.displacement[2]);
    x.distance = e.distance;
    r.edges.push_back(x);
  }
  return r;
}
#endif

}  // namespace b200
}  // namespace esgnn
