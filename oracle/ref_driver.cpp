// ref_driver.cpp -- a C ABI over the REFERENCE implementation itself
// (/root/reference/proj sources compiled unmodified against
// oracle/eigen_shim by oracle/ref.mk into oracle/_ref/libesgnn_ref.so).
//
// Test infrastructure only: the tests call it (tests/ref.py) to pin the
// CPU restatement (oracle/oracle.cpp) and the B200 path against the
// reference's own code -- structures::build_graph (graph.cpp:55-131),
// partition::lownn_partition (lownn.cpp:105-133), runtime::build_comm_plan
// (comm_plan.cpp:11-106), model::Network<T>::prepare / build_forward on the
// tape (network.h:98-164) and the forward output stage of
// tools/model_run.cpp:129-156 (assemble_blocks, blocks_to_uncoupled,
// write_blocks_file).  Every call reports errors through ref_last_error().
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "esgnn/model/block_matrix.h"
#include "esgnn/model/network.h"
#include "esgnn/model/synthetic.h"
#include "esgnn/partition/partition.h"
#include "esgnn/runtime/comm_plan.h"
#include "esgnn/structures/extxyz.h"
#include "esgnn/structures/graph.h"
#include "esgnn/structures/structure.h"

using namespace esgnn;

namespace {
thread_local std::string g_err;
structures::Graph g_graph;

structures::AtomicStructure make_structure(int n, const double* pos, const int* species, const double* cell,
                                           const uint8_t* pbc) {
  structures::AtomicStructure s;
  s.positions.resize(n);
  for (int i = 0; i < n; ++i) s.positions[i] = Eigen::Vector3d(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]);
  s.species.assign(species, species + n);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) s.cell(i, j) = cell[3 * i + j];
  for (int d = 0; d < 3; ++d) s.pbc[d] = pbc[d] != 0;
  return s;
}

structures::BasisSet make_basis(int n_species, const int* z, const int* n_shells, const int* shells) {
  structures::BasisSet b;
  int at = 0;
  for (int i = 0; i < n_species; ++i) {
    b.add_species(z[i], std::vector<int>(shells + at, shells + at + n_shells[i]));
    at += n_shells[i];
  }
  return b;
}

template <typename T>
void forward(const structures::AtomicStructure& s, const structures::BasisSet& basis, const model::ModelConfig& cfg,
             double* node_out, double* edge_out, const char* coupled_path, const char* uncoupled_path) {
  const structures::Graph g = structures::build_graph(s, cfg.r_cut);
  model::Network<T> net(cfg, basis);
  net.init_params();
  const model::Prepared<T> prep = net.prepare(g, s.species);
  model::Tape<T> tape;
  const model::ForwardVars fwd = net.build_forward(tape, prep);
  const auto& no = tape.val(fwd.node_out);
  const auto& eo = tape.val(fwd.edge_out);
  if (node_out)
    for (size_t i = 0; i < no.v.size(); ++i) node_out[i] = (double)no.v[i];
  if (edge_out)
    for (size_t i = 0; i < eo.v.size(); ++i) edge_out[i] = (double)eo.v[i];
  if (coupled_path || uncoupled_path) {  // model_run.cpp:141-151, one rank
    const model::BlockMatrix coupled = net.assemble_blocks(prep.view, no, eo);
    if (coupled_path && *coupled_path) model::write_blocks_file(coupled_path, coupled);
    if (uncoupled_path && *uncoupled_path)
      model::write_blocks_file(uncoupled_path, model::blocks_to_uncoupled(coupled, basis, s.species));
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// model::make_jittered_lattice (synthetic.cpp:17-41)
int ref_jittered_lattice(int n, double spacing, double jitter, int n_cycle, const int* cycle, uint64_t seed,
                         double* pos_out, double* cell_out, int* species_out) {
  try {
    const auto s = model::make_jittered_lattice(n, spacing, jitter, std::vector<int>(cycle, cycle + n_cycle), seed);
    for (int i = 0; i < n; ++i)
      for (int d = 0; d < 3; ++d) pos_out[3 * i + d] = s.positions[i](d);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) cell_out[3 * i + j] = s.cell(i, j);
    for (int i = 0; i < n; ++i) species_out[i] = s.species[i];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// structures::build_graph; the graph is kept for ref_graph_export / ref_lownn
int64_t ref_build_graph(int n, const double* pos, const int* species, const double* cell, const uint8_t* pbc,
                        double r_cut) {
  try {
    g_graph = structures::build_graph(make_structure(n, pos, species, cell, pbc), r_cut);
    return (int64_t)g_graph.edges.size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void ref_graph_export(int* src, int* dst, int* shift, double* disp, double* dist) {
  for (size_t k = 0; k < g_graph.edges.size(); ++k) {
    const auto& e = g_graph.edges[k];
    src[k] = e.src;
    dst[k] = e.dst;
    for (int d = 0; d < 3; ++d) {
      shift[3 * k + d] = e.shift[d];
      disp[3 * k + d] = e.displacement(d);
    }
    dist[k] = e.distance;
  }
}

// partition::lownn_partition on the structure and the last ref_build_graph
int ref_lownn(int n, const double* pos, const int* species, const double* cell, const uint8_t* pbc, int depth,
              double r_cut, int* part) {
  try {
    const auto a = partition::lownn_partition(make_structure(n, pos, species, cell, pbc), g_graph, depth, r_cut);
    for (int i = 0; i < n; ++i) part[i] = a.node_to_part[i];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// runtime::build_comm_plan on the last graph: sizes into info[0..4] (rows,
// owned, edges, neighbours, send rows); arrays may be NULL to size first
int ref_comm_plan(const int* species, int n_parts, const int* part, int rank, int64_t* info, int* row_global,
                  int* src_row, int* dst_row, int* nbr_peer, int* nbr_recv_row, int* nbr_recv_count,
                  int* send_rows) {
  try {
    partition::Assignment a;
    a.n_parts = n_parts;
    a.node_to_part.assign(part, part + g_graph.n_nodes);
    const auto p = runtime::build_comm_plan(g_graph, std::vector<int>(species, species + g_graph.n_nodes), a, rank);
    info[0] = p.view.n_rows;
    info[1] = p.view.n_owned;
    info[2] = p.view.n_edges();
    info[3] = (int64_t)p.neighbors.size();
    info[4] = 0;
    for (const auto& nb : p.neighbors) info[4] += (int64_t)nb.send_rows.size();
    if (row_global)
      for (int i = 0; i < p.view.n_rows; ++i) row_global[i] = p.view.row_global[i];
    if (src_row)
      for (int k = 0; k < p.view.n_edges(); ++k) {
        src_row[k] = p.view.edges[k].src_row;
        dst_row[k] = p.view.edges[k].dst_row;
      }
    if (nbr_peer) {
      int at = 0;
      for (size_t q = 0; q < p.neighbors.size(); ++q) {
        nbr_peer[q] = p.neighbors[q].peer;
        nbr_recv_row[q] = p.neighbors[q].recv_row;
        nbr_recv_count[q] = p.neighbors[q].recv_count;
        for (int r : p.neighbors[q].send_rows) send_rows[at++] = r;
      }
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The reference forward (Network<T>, taped) on the serial view of the
// structure's graph: head outputs (n x out_len, E x out_len, double) and
// optionally the output stage's text files.  precision 4: float, 8: double.
int ref_forward(int n, const double* pos, const int* species, const double* cell, const uint8_t* pbc, double r_cut,
                int n_species, const int* z, const int* n_shells, const int* shells, int l_max, int e_width,
                int layers, int n_radial, uint64_t seed, int gate, int precision, double* node_out,
                double* edge_out, const char* coupled_path, const char* uncoupled_path) {
  try {
    model::ModelConfig cfg;
    cfg.l_max = l_max;
    cfg.e_width = e_width;
    cfg.layers = layers;
    cfg.n_radial = n_radial;
    cfg.r_cut = r_cut;
    cfg.seed = seed;
    cfg.gate_enabled = gate != 0;
    const auto s = make_structure(n, pos, species, cell, pbc);
    const auto basis = make_basis(n_species, z, n_shells, shells);
    if (precision == 4)
      forward<float>(s, basis, cfg, node_out, edge_out, coupled_path, uncoupled_path);
    else
      forward<double>(s, basis, cfg, node_out, edge_out, coupled_path, uncoupled_path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The reference forward timed on a view (the benchmark's CPU arm): the owned
// destinations [0, n_owned) of the given view are split into n_threads
// contiguous groups of about equal edge count; each thread runs the
// reference's own Network<float>::prepare(GraphView) (network.h:98-105) and
// build_forward (network.h:115-164) on its group's view -- owned rows the
// group's destinations, halo rows every other source it reads, like one rank
// of the reference's distributed run without the exchange.  Times (max over
// threads, seconds, a barrier before each phase): secs[0] prepare, secs[1]
// build_forward.  Edges processed: all of the view's edges.
int ref_forward_view_timed(int n_rows, int n_owned, const int* row_species, int64_t n_edges, const int* src_row,
                           const int* dst_row, const double* disp, const double* dist, int n_species, const int* z,
                           const int* n_shells, const int* shells, int l_max, int e_width, int layers, int n_radial,
                           double r_cut, uint64_t seed, int n_threads, double* secs) {
  try {
    model::ModelConfig cfg;
    cfg.l_max = l_max;
    cfg.e_width = e_width;
    cfg.layers = layers;
    cfg.n_radial = n_radial;
    cfg.r_cut = r_cut;
    cfg.seed = seed;
    const auto basis = make_basis(n_species, z, n_shells, shells);
    if (n_threads < 1) n_threads = 1;
    // destination groups of about n_edges / n_threads edges (dst-sorted edges)
    std::vector<int64_t> first(n_owned + 1, 0);
    for (int64_t k = 0; k < n_edges; ++k) first[dst_row[k] + 1]++;
    for (int j = 0; j < n_owned; ++j) first[j + 1] += first[j];
    std::vector<int> cut{0};
    for (int t = 1; t < n_threads; ++t) {
      const int64_t want = n_edges * t / n_threads;
      int j = cut.back();
      while (j < n_owned && first[j] < want) ++j;
      cut.push_back(j);
    }
    cut.push_back(n_owned);
    std::vector<model::GraphView> views(n_threads);
    for (int t = 0; t < n_threads; ++t) {
      model::GraphView& v = views[t];
      const int j0 = cut[t], j1 = cut[t + 1];
      std::vector<int> row_of(n_rows, -1);
      for (int j = j0; j < j1; ++j) {
        row_of[j] = j - j0;
        v.row_global.push_back(j);
      }
      for (int64_t k = first[j0]; k < first[j1]; ++k)
        if (row_of[src_row[k]] < 0) {
          row_of[src_row[k]] = (int)v.row_global.size();
          v.row_global.push_back(src_row[k]);
        }
      v.n_owned = j1 - j0;
      v.n_rows = (int)v.row_global.size();
      for (int r : v.row_global) v.row_species.push_back(row_species[r]);
      for (int j = j0; j < j1; ++j)
        v.dst_ranges.push_back({(int)(first[j] - first[j0]), (int)(first[j + 1] - first[j0])});
      for (int64_t k = first[j0]; k < first[j1]; ++k) {
        model::ViewEdge e;
        e.src_row = row_of[src_row[k]];
        e.dst_row = row_of[dst_row[k]];
        e.src_global = src_row[k];
        e.dst_global = dst_row[k];
        e.displacement = Eigen::Vector3d(disp[3 * k], disp[3 * k + 1], disp[3 * k + 2]);
        e.distance = dist[k];
        v.edges.push_back(e);
      }
    }
    std::vector<double> t_prep(n_threads, 0.0), t_fwd(n_threads, 0.0);
    std::vector<std::string> errs(n_threads);
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0, generation = 0;
    auto barrier = [&] {
      std::unique_lock<std::mutex> lk(mu);
      const int gen = generation;
      if (++arrived == n_threads) {
        arrived = 0;
        ++generation;
        cv.notify_all();
      } else {
        cv.wait(lk, [&] { return generation != gen; });
      }
    };
    auto work = [&](int t) {
      int passed = 0;  // barriers passed: a failing thread still passes both
      try {
        model::Network<float> net(cfg, basis);
        net.init_params();
        barrier();
        ++passed;
        auto t0 = std::chrono::steady_clock::now();
        const model::Prepared<float> prep = net.prepare(views[t]);
        t_prep[t] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        barrier();
        ++passed;
        t0 = std::chrono::steady_clock::now();
        model::Tape<float> tape;
        net.build_forward(tape, prep);
        t_fwd[t] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      } catch (const std::exception& e) {
        errs[t] = e.what();
        for (; passed < 2; ++passed) barrier();
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < n_threads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
    for (const auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
    secs[0] = *std::max_element(t_prep.begin(), t_prep.end());
    secs[1] = *std::max_element(t_fwd.begin(), t_fwd.end());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// structures::read_extxyz_file (extxyz.h:17): the count first (arrays may be
// NULL), then the arrays; errors through ref_last_error
int ref_read_extxyz(const char* path, int64_t* n, double* pos, int* species, double* cell, uint8_t* pbc) {
  try {
    const auto s = structures::read_extxyz_file(path);
    *n = s.n_atoms();
    for (int i = 0; i < s.n_atoms() && pos; ++i)
      for (int d = 0; d < 3; ++d) pos[3 * i + d] = s.positions[i](d);
    for (int i = 0; i < s.n_atoms() && species; ++i) species[i] = s.species[i];
    for (int i = 0; i < 3 && cell; ++i)
      for (int j = 0; j < 3; ++j) cell[3 * i + j] = s.cell(i, j);
    for (int d = 0; d < 3 && pbc; ++d) pbc[d] = s.pbc[d] ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// structures::write_extxyz_file (extxyz.h:20)
int ref_write_extxyz(const char* path, int n, const double* pos, const int* species, const double* cell,
                     const uint8_t* pbc) {
  try {
    structures::write_extxyz_file(path, make_structure(n, pos, species, cell, pbc));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// HeadLayout::out_len of a basis (layout.h:62-94)
int ref_out_len(int n_species, const int* z, const int* n_shells, const int* shells) {
  try {
    return model::HeadLayout::build(make_basis(n_species, z, n_shells, shells)).out_len;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
