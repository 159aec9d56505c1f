// capi.cpp -- the extern "C" boundary (include/esg.h).  Every entry point
// catches and maps exceptions to ESG_* codes; the message is kept per thread
// for esg_last_error().
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <random>

#include "blocks_io.h"
#include "esg_internal.h"

namespace esg {
esg_graph* build_graph_gpu(esg_ctx* ctx, int n, const double* pos, const M3& cell, const bool pbc[3], double r_cut);
void model_device_create(esg_model* M);
void model_device_destroy(esg_model* M);
void model_upload_params(esg_model* M);
void model_prepare(esg_model* M, const esg_graph* g, const esg_plan* plan, const int32_t* species);
void model_forward(esg_model* M, esg_timing* tm);
void model_forward_to_host(esg_model* M, esg_timing* tm, float* node_out, float* edge_out, bool async);
void model_outputs_wait(esg_model* M);
void model_profile(esg_model* M, int enable, double* ms, int64_t* counts);
void model_outputs(const esg_model* M, const float** no, const float** eo, const float** nf, const float** ef);
void model_copy_outputs(const esg_model* M, float* node_out, float* edge_out);
void model_copy_features(const esg_model* M, float* nodes, float* edges);
void model_copy_output_rows(const esg_model* M, int64_t nf, int64_t nc, float* node_out, int64_t ef, int64_t ec,
                            float* edge_out);
void model_prepared_info(const esg_model* M, int64_t info[3]);
void edge_rotations(esg_ctx* ctx, int64_t n, const double* disp, int l_max, float* out);
void partition_metrics_gpu(const esg_graph* g, const int32_t* part, int P, esg_metrics* m, esg_part_stats* parts,
                           int64_t* vol);
std::string metrics_json(const esg_metrics& m, const esg_part_stats* parts);
std::string partition_dot(const int64_t* vol, const esg_part_stats* parts, int P);
void write_assignment(const std::string& path, const int32_t* part, int64_t n);
std::vector<int32_t> read_assignment(const std::string& path, int* n_parts);
void blocks_count(esg_model* M, int64_t* n_blocks, int64_t* n_values);
void blocks_export(esg_model* M, int basis, bool sym, BlockRec* keys, double* values);
void blocks_export_device(esg_model* M, int basis, bool sym, int vb, void* d_keys, void* d_values, float* kernel_ms);
void blocks_write_shard(esg_model* M, const char* path, int basis, bool sym, int vb);
void blocks_write_text(esg_model* M, const char* path, int basis, bool sym);
int64_t build_targets(esg_model* M, int64_t n_blocks, const BlockRec* keys, const double* values, float* node_t,
                      uint8_t* node_m, float* edge_t, uint8_t* edge_m);

namespace {
thread_local std::string g_last;
M3 to_m3(const double c[9]) {
  M3 m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[i][j] = c[3 * i + j];
  return m;
}
}  // namespace
void set_error(const std::string& m) { g_last = m; }
const char* last_error() { return g_last.c_str(); }
}  // namespace esg

using namespace esg;

struct esg_adam {
  esg_adam_config cfg{};
  std::vector<double> m, v;  // host moments (the host path; checkpoint mirror of the device ones)
  double *d_m = nullptr, *d_v = nullptr;  // device moments (a model with a device context)
  int device = -1;
  bool host_current = true;  // m / v hold the current moments (else d_m / d_v do)
  double lr = -1.0, best = std::numeric_limits<double>::infinity();
  long t = 0;
  int stale = 0;
};

namespace esg {
esg_plan* plan_build_gpu(const esg_graph* g, const int32_t* species, const int32_t* part, int n_parts, int rank);
void lownn_gpu(esg_ctx* ctx, int n, const double* pos, const M3& cell, const bool pbc[3], const int32_t* deg, int depth,
               double r_cut, int32_t* part);  // lownn_gpu.cu
void model_set_targets(esg_model* M, const float* node_target, const uint8_t* node_mask, const float* edge_target,
                       const uint8_t* edge_mask);
void model_loss_grad(esg_model* M, int64_t n_total, double partials[3], double* loss, float* grads_out);
void model_train_timing(const esg_model* M, double* fwd_ms, double* bwd_ms);
}  // namespace esg

namespace {
// check_param_sync (distributed.h:133-145): every rank's parameter hash,
// allgathered; any mismatch is a divergence error on every rank
void check_param_sync(esg_model* m, const char* where) {
  esg_ctx* ctx = m->ctx;
  if (!ctx || ctx->world <= 1) return;
  const uint64_t h = esg::param_hash(m->params, m->host_params);
  const double mine[2] = {double(h >> 32), double(h & 0xffffffffULL)};
  double *d_mine = nullptr, *d_all = nullptr;
  ESG_CUDA(cudaMalloc(&d_mine, sizeof(mine)));
  ESG_CUDA(cudaMalloc(&d_all, sizeof(mine) * ctx->world));
  ESG_CUDA(cudaMemcpyAsync(d_mine, mine, sizeof(mine), cudaMemcpyHostToDevice, ctx->stream));
  ESG_NCCL(ncclAllGather(d_mine, d_all, 2, ncclDouble, ctx->comm, ctx->stream));
  std::vector<double> all(2 * ctx->world);
  ESG_CUDA(cudaMemcpyAsync(all.data(), d_all, sizeof(double) * all.size(), cudaMemcpyDeviceToHost, ctx->stream));
  ESG_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(d_mine);
  cudaFree(d_all);
  for (int p = 0; p < ctx->world; ++p)
    if (all[2 * p] != mine[0] || all[2 * p + 1] != mine[1])
      throw esg::Error(ESG_ERR_DIVERGENCE, std::string("parameter state diverged between ranks (") + where + ")");
}
}  // namespace

namespace {
// checkpoint.h:20-35: little-endian u64 fields
void ckpt_u64(std::ostream& out, uint64_t v) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = (unsigned char)(v >> (8 * i));
  out.write(reinterpret_cast<const char*>(b), 8);
}
uint64_t ckpt_read_u64(std::istream& in) {
  unsigned char b[8];
  in.read(reinterpret_cast<char*>(b), 8);
  if (!in) esg::data("truncated checkpoint");
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= uint64_t(b[i]) << (8 * i);
  return v;
}
void ckpt_f64(std::ostream& out, double d) {
  uint64_t v;
  std::memcpy(&v, &d, 8);
  ckpt_u64(out, v);
}
double ckpt_read_f64(std::istream& in) {
  const uint64_t v = ckpt_read_u64(in);
  double d;
  std::memcpy(&d, &v, 8);
  return d;
}
}  // namespace

#define ESG_API_BEGIN try {
#define ESG_API_END                       \
  return ESG_OK;                          \
  }                                       \
  catch (const esg::Error& e) {           \
    esg::set_error(e.what());             \
    return e.code;                        \
  }                                       \
  catch (const std::bad_alloc& e) {       \
    esg::set_error("host out of memory"); \
    return ESG_ERR_OOM;                   \
  }                                       \
  catch (const std::exception& e) {       \
    esg::set_error(e.what());             \
    return ESG_ERR_OTHER;                 \
  }

#define NEED(p, what) \
  if (!(p)) esg::usage(std::string("null ") + what)

namespace esg {
void model_adam_device(esg_model* M, double* d_m, double* d_v, const float* grads, double b1, double b2, double lr,
                       double bc1, double bc2, double eps);  // train.cu
}

namespace {
// device moments of opt, uploaded from the host mirror when they are stale
void adam_device_moments(esg_adam* opt, esg_model* m) {
  const size_t n = opt->m.size();
  if (!opt->d_m) {
    ESG_CUDA(cudaMalloc(&opt->d_m, sizeof(double) * n));
    ESG_CUDA(cudaMalloc(&opt->d_v, sizeof(double) * n));
    opt->device = m->ctx->device;
    opt->host_current = true;
  }
  if (opt->host_current) {
    ESG_CUDA(cudaMemcpy(opt->d_m, opt->m.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    ESG_CUDA(cudaMemcpy(opt->d_v, opt->v.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    opt->host_current = false;
  }
}
// the host mirror of the moments (checkpoints)
void adam_host_moments(const esg_adam* opt) {
  esg_adam* o = const_cast<esg_adam*>(opt);
  if (o->host_current || !o->d_m) return;
  ESG_CUDA(cudaSetDevice(o->device));
  ESG_CUDA(cudaMemcpy(o->m.data(), o->d_m, sizeof(double) * o->m.size(), cudaMemcpyDeviceToHost));
  ESG_CUDA(cudaMemcpy(o->v.data(), o->d_v, sizeof(double) * o->v.size(), cudaMemcpyDeviceToHost));
  o->host_current = true;
}

void adam_update(esg_adam* opt, esg_model* m, const float* g, double loss) {
  // Optimizer::step (optimizer.h:42-59), moments in fp64: on the device when
  // the model has one (k_adam, bit-identical to the host loop below)
  if (opt->lr < 0) opt->lr = opt->cfg.lr;
  ++opt->t;
  const double bc1 = 1.0 - std::pow(opt->cfg.beta1, double(opt->t));
  const double bc2 = 1.0 - std::pow(opt->cfg.beta2, double(opt->t));
  if (m->ctx && m->dev) {
    adam_device_moments(opt, m);
    esg::model_adam_device(m, opt->d_m, opt->d_v, g, opt->cfg.beta1, opt->cfg.beta2, opt->lr, bc1, bc2,
                           opt->cfg.eps);
  } else {
    adam_host_moments(opt);
    for (size_t k = 0; k < m->host_params.size(); ++k) {
    const double gk = double(g[k]);
    opt->m[k] = opt->cfg.beta1 * opt->m[k] + (1.0 - opt->cfg.beta1) * gk;
    opt->v[k] = opt->cfg.beta2 * opt->v[k] + (1.0 - opt->cfg.beta2) * gk * gk;
    const double mh = opt->m[k] / bc1;
    const double vh = opt->v[k] / bc2;
    m->host_params[k] = static_cast<float>(double(m->host_params[k]) - opt->lr * mh / (std::sqrt(vh) + opt->cfg.eps));
    }
  }
  // reduce-on-plateau (optimizer.h:62-72), a scalar rule: on the host
  if (loss < opt->best * (1.0 - opt->cfg.threshold)) {
    opt->best = loss;
    opt->stale = 0;
  } else if (++opt->stale >= opt->cfg.patience) {
    opt->lr = std::max(opt->cfg.min_lr, opt->lr * opt->cfg.factor);
    opt->stale = 0;
  }
}
}  // namespace

extern "C" {

const char* esg_last_error(void) { return esg::last_error(); }
int esg_version(void) { return 1; }

int esg_nccl_unique_id_size(void) { return (int)sizeof(ncclUniqueId); }
int esg_nccl_get_unique_id(void* out) {
  ESG_API_BEGIN
  NEED(out, "out");
  ncclUniqueId id;
  ESG_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  ESG_API_END
}

int esg_ctx_create(int device, int rank, int world, const void* nccl_id, esg_ctx** out) {
  ESG_API_BEGIN
  NEED(out, "out");
  if (world < 1 || rank < 0 || rank >= world) usage("rank outside the world");
  int ndev = 0;
  ESG_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) usage("no CUDA device " + std::to_string(device));
  ESG_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop{};
  ESG_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) usage("libesg_b200 targets sm_100a (B200); device is sm_" + std::to_string(prop.major) +
                              std::to_string(prop.minor));
  auto* c = new esg_ctx();
  c->device = device;
  c->rank = rank;
  c->world = world;
  ESG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  if (world > 1) {
    if (!nccl_id) {
      delete c;
      usage("world > 1 needs an NCCL unique id");
    }
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ESG_NCCL(ncclCommInitRank(&c->comm, world, id, rank));
  }
  *out = c;
  ESG_API_END
}

int esg_ctx_destroy(esg_ctx* ctx) {
  ESG_API_BEGIN
  if (!ctx) return ESG_OK;
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  for (esg_graph* g : ctx->graphs) {  // detach graphs and plans that outlive their context
    for (void* p : {(void*)g->d_off, (void*)g->d_src, (void*)g->d_shift, (void*)g->d_disp, (void*)g->d_dist})
      ctx->cache.release(p);
    g->d_off = nullptr;
    g->d_src = nullptr;
    g->d_shift = nullptr;
    g->d_disp = g->d_dist = nullptr;
    g->ctx = nullptr;
  }
  for (esg_plan* p : ctx->plans) {
    for (void* q : {(void*)p->d_edge_index, (void*)p->d_src_row, (void*)p->d_dst_row, (void*)p->d_seg})
      ctx->cache.release(q);
    p->d_edge_index = p->d_src_row = p->d_dst_row = nullptr;
    p->d_seg = nullptr;
    p->ctx = nullptr;
  }
  ctx->graphs.clear();
  ctx->plans.clear();
  ctx->cache.flush();
  if (ctx->zc) cudaFreeHost(ctx->zc);
  if (ctx->up) cudaFreeHost(ctx->up);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->build_stream) cudaStreamDestroy(ctx->build_stream);
  delete ctx;
  ESG_API_END
}

int esg_ctx_synchronize(esg_ctx* ctx) {
  ESG_API_BEGIN
  NEED(ctx, "ctx");
  ESG_CUDA(cudaStreamSynchronize(ctx->stream));
  ESG_API_END
}

int esg_wrap_positions(int n, double* pos, const double cell[9], const uint8_t pbc[3]) {
  ESG_API_BEGIN
  NEED(pos, "pos");
  bool p[3] = {pbc[0] != 0, pbc[1] != 0, pbc[2] != 0};
  wrap_positions(n, pos, to_m3(cell), p);
  ESG_API_END
}

// synthetic.cpp:17-41
int esg_jittered_lattice(int n_atoms, double spacing, double jitter, int n_cycle, const int* cycle, uint64_t seed,
                         double* pos_out, double cell_out[9], int* species_out) {
  ESG_API_BEGIN
  if (n_atoms < 1) usage("need at least one atom");
  if (n_cycle < 1) usage("species cycle is empty");
  if (!(spacing > 0.0)) usage("lattice spacing must be positive");
  int n = 1;
  while (n * n * n < n_atoms) ++n;
  for (int i = 0; i < 9; ++i) cell_out[i] = (i % 4 == 0) ? 1.0 * (n * spacing) : 0.0 * (n * spacing);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(-jitter, jitter);
  int placed = 0;
  for (int ix = 0; ix < n && placed < n_atoms; ++ix)
    for (int iy = 0; iy < n && placed < n_atoms; ++iy)
      for (int iz = 0; iz < n && placed < n_atoms; ++iz) {
        double p[3] = {(ix + 0.5) * spacing, (iy + 0.5) * spacing, (iz + 0.5) * spacing};
        for (int d = 0; d < 3; ++d) p[d] += u(rng);
        for (int d = 0; d < 3; ++d) pos_out[3 * placed + d] = p[d];
        species_out[placed] = cycle[placed % n_cycle];
        ++placed;
      }
  ESG_API_END
}

// structure.cpp:40-63
int esg_tile(int n, const double* pos, const double cell[9], const uint8_t pbc[3], const int* species,
             const int reps[3], double* pos_out, double cell_out[9], int* species_out) {
  ESG_API_BEGIN
  for (int d = 0; d < 3; ++d) {
    if (reps[d] < 1) usage("tile factors must be positive");
    if (reps[d] > 1 && !pbc[d]) usage("cannot tile along aperiodic dimension");
  }
  for (int d = 0; d < 3; ++d)
    for (int k = 0; k < 3; ++k) cell_out[3 * d + k] = cell[3 * d + k] * reps[d];
  int64_t at = 0;
  for (int ix = 0; ix < reps[0]; ++ix)
    for (int iy = 0; iy < reps[1]; ++iy)
      for (int iz = 0; iz < reps[2]; ++iz) {
        double off[3];
        for (int k = 0; k < 3; ++k) off[k] = (ix * cell[k] + iy * cell[3 + k]) + iz * cell[6 + k];
        for (int a = 0; a < n; ++a, ++at) {
          for (int k = 0; k < 3; ++k) pos_out[3 * at + k] = pos[3 * a + k] + off[k];
          species_out[at] = species[a];
        }
      }
  ESG_API_END
}

int esg_build_graph(esg_ctx* ctx, int n, const double* pos, const double cell[9], const uint8_t pbc[3], double r_cut,
                    esg_graph** out) {
  ESG_API_BEGIN
  NEED(ctx, "ctx");
  NEED(out, "out");
  ESG_CUDA(cudaSetDevice(ctx->device));
  bool p[3] = {pbc[0] != 0, pbc[1] != 0, pbc[2] != 0};
  *out = build_graph_gpu(ctx, n, pos, to_m3(cell), p, r_cut);
  ESG_API_END
}

int esg_graph_destroy(esg_graph* g) {
  ESG_API_BEGIN
  if (!g) return ESG_OK;
  if (g->ctx) {
    for (void* p : {(void*)g->d_off, (void*)g->d_src, (void*)g->d_shift, (void*)g->d_disp, (void*)g->d_dist})
      g->ctx->cache.release(p);
    g->ctx->graphs.erase(g);
  }
  delete g;
  ESG_API_END
}

int esg_graph_info(const esg_graph* g, int* n_nodes, int64_t* n_edges) {
  ESG_API_BEGIN
  NEED(g, "graph");
  if (n_nodes) *n_nodes = g->n;
  if (n_edges) *n_edges = g->E;
  ESG_API_END
}

int esg_graph_export(const esg_graph* g, int32_t* src, int32_t* dst, int32_t* shift, double* disp, double* dist) {
  ESG_API_BEGIN
  NEED(g, "graph");
  ESG_CUDA(cudaSetDevice(g->ctx->device));
  const int64_t E = g->E;
  g->host_sync();
  if (src) std::copy(g->h_src.begin(), g->h_src.end(), src);
  if (dst)
    for (int j = 0; j < g->n; ++j)
      for (int64_t k = g->h_off[j]; k < g->h_off[j + 1]; ++k) dst[k] = j;
  if (shift && E) {
    std::vector<uint32_t> s(E);
    ESG_CUDA(cudaMemcpy(s.data(), g->d_shift, sizeof(uint32_t) * E, cudaMemcpyDeviceToHost));
    for (int64_t k = 0; k < E; ++k) {
      shift[3 * k] = int((s[k] >> 20) & 1023) - 512;
      shift[3 * k + 1] = int((s[k] >> 10) & 1023) - 512;
      shift[3 * k + 2] = int(s[k] & 1023) - 512;
    }
  }
  if (disp && E) ESG_CUDA(cudaMemcpy(disp, g->d_disp, sizeof(double) * 3 * E, cudaMemcpyDeviceToHost));
  if (dist && E) ESG_CUDA(cudaMemcpy(dist, g->d_dist, sizeof(double) * E, cudaMemcpyDeviceToHost));
  ESG_API_END
}

int esg_graph_in_degrees(const esg_graph* g, int32_t* deg) {
  ESG_API_BEGIN
  NEED(g, "graph");
  NEED(deg, "deg");
  g->host_sync_offsets();
  for (int j = 0; j < g->n; ++j) deg[j] = (int32_t)(g->h_off[j + 1] - g->h_off[j]);
  ESG_API_END
}

int esg_graph_offsets(const esg_graph* g, int64_t* off) {
  ESG_API_BEGIN
  NEED(g, "graph");
  NEED(off, "off");
  g->host_sync_offsets();
  std::copy(g->h_off.begin(), g->h_off.end(), off);
  ESG_API_END
}

int esg_lownn_partition(int n, const double* pos, const double cell[9], const uint8_t pbc[3], const int32_t* deg,
                        int depth, double r_cut, int32_t* part) {
  ESG_API_BEGIN
  NEED(pos, "pos");
  NEED(deg, "in_degree");
  NEED(part, "node_to_part");
  bool p[3] = {pbc[0] != 0, pbc[1] != 0, pbc[2] != 0};
  auto a = lownn(n, pos, to_m3(cell), p, deg, depth, r_cut);
  std::copy(a.begin(), a.end(), part);
  ESG_API_END
}

// lownn.cpp:23-133 on the device (lownn_gpu.cu): the same assignment as
// esg_lownn_partition, level by level with segmented radix sorts
int esg_lownn_partition_gpu(esg_ctx* ctx, int n, const double* pos, const double cell[9], const uint8_t pbc[3],
                            const int32_t* deg, int depth, double r_cut, int32_t* part) {
  ESG_API_BEGIN
  NEED(ctx, "ctx");
  NEED(pos, "pos");
  NEED(deg, "in_degree");
  NEED(part, "node_to_part");
  bool p[3] = {pbc[0] != 0, pbc[1] != 0, pbc[2] != 0};
  lownn_gpu(ctx, n, pos, to_m3(cell), p, deg, depth, r_cut, part);
  ESG_API_END
}

// comm_plan.cpp:11-106: owned rows ascending by global id, halo rows for
// remote sources of owned edges grouped by (owner, id), owned edges in the
// global (dst, src, shift) order, send lists ascending by global id.
static esg_plan* plan_from_csr(int n, const int64_t* off, const int32_t* src, const int32_t* species,
                               const int32_t* part, int n_parts, int rank) {
  if (rank < 0 || rank >= n_parts) usage("rank outside the assignment");
  for (int i = 0; i < n; ++i)
    if (part[i] < 0 || part[i] >= n_parts) data("assignment part out of range");
  auto* P = new esg_plan();
  P->rank = rank;
  P->world = n_parts;
  std::vector<int> owned_row(n, -1);
  for (int i = 0; i < n; ++i)
    if (part[i] == rank) {
      owned_row[i] = P->n_owned++;
      P->row_global.push_back(i);
    }
  std::vector<std::pair<int, int>> halo;
  for (int j = 0; j < n; ++j) {
    if (part[j] != rank) continue;
    for (int64_t k = off[j]; k < off[j + 1]; ++k) {
      const int s = src[k];
      if (part[s] != rank) halo.emplace_back(part[s], s);
    }
  }
  std::sort(halo.begin(), halo.end());
  halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
  std::vector<int> halo_row(n, -1);
  for (size_t q = 0; q < halo.size(); ++q) {
    halo_row[halo[q].second] = P->n_owned + (int)q;
    P->row_global.push_back(halo[q].second);
  }
  P->n_rows = P->n_owned + (int)halo.size();
  if (species)
    for (int r = 0; r < P->n_rows; ++r) P->row_species.push_back(species[P->row_global[r]]);
  for (int j = 0; j < n; ++j) {
    if (part[j] != rank) continue;
    for (int64_t k = off[j]; k < off[j + 1]; ++k) {
      const int s = src[k];
      P->edge_index.push_back((int32_t)k);
      P->src_row.push_back(owned_row[s] >= 0 ? owned_row[s] : halo_row[s]);
      P->dst_row.push_back(owned_row[j]);
    }
  }
  std::map<int, std::vector<int>> sends;
  for (int j = 0; j < n; ++j) {
    if (part[j] == rank) continue;
    for (int64_t k = off[j]; k < off[j + 1]; ++k) {
      const int s = src[k];
      if (part[s] == rank) sends[part[j]].push_back(s);
    }
  }
  std::map<int, Neighbor> nb;
  for (auto& kv : sends) {
    std::sort(kv.second.begin(), kv.second.end());
    kv.second.erase(std::unique(kv.second.begin(), kv.second.end()), kv.second.end());
    Neighbor& x = nb[kv.first];
    x.peer = kv.first;
    for (int id : kv.second) x.send_rows.push_back(owned_row[id]);
  }
  int at = P->n_owned;
  for (size_t q = 0; q < halo.size();) {
    size_t r = q;
    while (r < halo.size() && halo[r].first == halo[q].first) ++r;
    Neighbor& x = nb[halo[q].first];
    x.peer = halo[q].first;
    x.recv_row = at;
    x.recv_count = (int)(r - q);
    at += x.recv_count;
    q = r;
  }
  for (auto& kv : nb) P->nbrs.push_back(kv.second);
  P->n_edges = (int64_t)P->src_row.size();
  return P;
}

int esg_plan_build(const esg_graph* g, const int32_t* species, const int32_t* part, int n_parts, int rank,
                   esg_plan** out) {
  ESG_API_BEGIN
  NEED(g, "graph");
  NEED(part, "node_to_part");
  NEED(out, "out");
  ESG_CUDA(cudaSetDevice(g->ctx->device));
  *out = plan_build_gpu(g, species, part, n_parts, rank);  // the device CSR, same plan as plan_from_csr
  ESG_API_END
}

int esg_plan_build_host(int n, const int64_t* dst_off, const int32_t* src, const int32_t* species,
                        const int32_t* part, int n_parts, int rank, esg_plan** out) {
  ESG_API_BEGIN
  NEED(dst_off, "dst_off");
  NEED(src, "src");
  NEED(part, "node_to_part");
  NEED(out, "out");
  *out = plan_from_csr(n, dst_off, src, species, part, n_parts, rank);
  ESG_API_END
}

int esg_plan_destroy(esg_plan* p) {
  delete p;
  return ESG_OK;
}

int esg_plan_info(const esg_plan* p, int64_t info[5]) {
  ESG_API_BEGIN
  NEED(p, "plan");
  info[0] = p->n_rows;
  info[1] = p->n_owned;
  info[2] = p->n_edges;
  info[3] = (int64_t)p->nbrs.size();
  int64_t s = 0;
  for (const auto& nb : p->nbrs) s += (int64_t)nb.send_rows.size();
  info[4] = s;
  ESG_API_END
}

int esg_plan_export(const esg_plan* p, int32_t* row_global, int32_t* row_species, int32_t* edge_index,
                    int32_t* src_row, int32_t* dst_row, int32_t* nbr_peer, int32_t* nbr_recv_row,
                    int32_t* nbr_recv_count, int32_t* nbr_send_count, int32_t* send_rows) {
  ESG_API_BEGIN
  NEED(p, "plan");
  if (edge_index || src_row || dst_row) p->host_sync_edges();
  if (row_global) std::copy(p->row_global.begin(), p->row_global.end(), row_global);
  if (row_species) std::copy(p->row_species.begin(), p->row_species.end(), row_species);
  if (edge_index) std::copy(p->edge_index.begin(), p->edge_index.end(), edge_index);
  if (src_row) std::copy(p->src_row.begin(), p->src_row.end(), src_row);
  if (dst_row) std::copy(p->dst_row.begin(), p->dst_row.end(), dst_row);
  int at = 0;
  for (size_t q = 0; q < p->nbrs.size(); ++q) {
    if (nbr_peer) nbr_peer[q] = p->nbrs[q].peer;
    if (nbr_recv_row) nbr_recv_row[q] = p->nbrs[q].recv_row;
    if (nbr_recv_count) nbr_recv_count[q] = p->nbrs[q].recv_count;
    if (nbr_send_count) nbr_send_count[q] = (int)p->nbrs[q].send_rows.size();
    if (send_rows)
      for (int r : p->nbrs[q].send_rows) send_rows[at++] = r;
  }
  ESG_API_END
}

int esg_coupling_matrix(int la, int lb, int L, double* out) {
  ESG_API_BEGIN
  NEED(out, "out");
  if (la < 0 || lb < 0 || la > 6 || lb > 6) data("coupled degree out of supported range");
  const auto C = coupling_matrix(la, lb, L);
  std::copy(C.begin(), C.end(), out);
  ESG_API_END
}

int esg_model_create(esg_ctx* ctx, const esg_model_config* cfg, int n_species, const int* z, const int* n_shells,
                     const int* shells, esg_model** out) {
  ESG_API_BEGIN
  NEED(cfg, "cfg");
  NEED(out, "out");
  // ModelConfig::validate (network.h:29-35)
  if (cfg->l_max < 0 || cfg->l_max > 6) usage("l_max must be in 0..6");
  if (cfg->e_width < 1) usage("embedding width must be >= 1");
  if (cfg->layers < 0) usage("layer count must be >= 0");
  if (cfg->n_radial < 2) usage("radial basis needs at least 2 Gaussians");
  if (!(cfg->r_cut > 0)) usage("cutoff must be positive");
  if (n_species < 1) data("basis defines no species");
  auto* M = new esg_model();
  M->ctx = ctx;
  M->cfg = *cfg;
  int at = 0;
  for (int s = 0; s < n_species; ++s) {
    if (n_shells[s] < 1) {
      delete M;
      data("basis for " + element_symbol(z[s]) + " has no shells");
    }
    std::vector<int> ls(shells + at, shells + at + n_shells[s]);
    for (int l : ls)
      if (l < 0 || l > 6) {
        delete M;
        data("shell angular momentum out of range: " + std::to_string(l));
      }
    at += n_shells[s];
    M->basis.shells[z[s]] = ls;
  }
  M->heads = head_layout(M->basis);
  if (cfg->l_max < M->heads.max_l) {
    const int need = M->heads.max_l;
    delete M;
    usage("l_max " + std::to_string(cfg->l_max) + " cannot couple the basis shells; need at least " +
          std::to_string(need));
  }
  M->lay = m_layout(cfg->l_max);
  for (const auto& kv : M->basis.shells) M->species_list.push_back(kv.first);
  M->params = register_params(*cfg, M->basis, M->heads);
  M->host_params.assign(M->params.total, 0.0f);
  if (ctx) try {
      model_device_create(M);
    } catch (...) {
      delete M;
      throw;
    }
  *out = M;
  ESG_API_END
}

int esg_model_destroy(esg_model* m) {
  ESG_API_BEGIN
  if (!m) return ESG_OK;
  model_device_destroy(m);
  delete m;
  ESG_API_END
}

int esg_model_set_precision(esg_model* m, int prec) {
  ESG_API_BEGIN
  NEED(m, "model");
  if (prec != ESG_LINEAR_FP32 && prec != ESG_LINEAR_BF16) usage("unknown linear precision");
  m->cfg.linear_precision = prec;
  ESG_API_END
}

int esg_model_init_params(esg_model* m) {
  ESG_API_BEGIN
  NEED(m, "model");
  init_params(m->params, m->cfg.seed, m->host_params);
  if (m->ctx) {
    ESG_CUDA(cudaSetDevice(m->ctx->device));
    model_upload_params(m);
  }
  ESG_API_END
}

int64_t esg_model_param_count(const esg_model* m) { return m ? m->params.total : -1; }
int esg_model_n_entries(const esg_model* m) { return m ? (int)m->params.entries.size() : -1; }
int esg_model_entry(const esg_model* m, int i, const char** name, int* rows, int* cols, int64_t* offset) {
  ESG_API_BEGIN
  NEED(m, "model");
  if (i < 0 || i >= (int)m->params.entries.size()) usage("entry index out of range");
  const auto& e = m->params.entries[i];
  if (name) *name = e.name.c_str();
  if (rows) *rows = e.rows;
  if (cols) *cols = e.cols;
  if (offset) *offset = e.offset;
  ESG_API_END
}
int esg_model_get_params(const esg_model* m, float* out) {
  ESG_API_BEGIN
  NEED(m, "model");
  std::copy(m->host_params.begin(), m->host_params.end(), out);
  ESG_API_END
}
int esg_model_set_params(esg_model* m, const float* in) {
  ESG_API_BEGIN
  NEED(m, "model");
  std::copy(in, in + m->host_params.size(), m->host_params.begin());
  if (m->ctx) {
    ESG_CUDA(cudaSetDevice(m->ctx->device));
    model_upload_params(m);
  }
  ESG_API_END
}
uint64_t esg_model_param_hash(const esg_model* m) { return m ? param_hash(m->params, m->host_params) : 0; }
int esg_model_out_len(const esg_model* m) { return m ? m->heads.out_len : -1; }

int esg_prepare(esg_model* m, const esg_graph* g, const esg_plan* plan, const int32_t* species) {
  ESG_API_BEGIN
  NEED(m, "model");
  if (!m->ctx || !m->dev) usage("model was created without a device context");
  NEED(g, "graph");
  NEED(species, "species");
  if (plan && (plan->world != m->ctx->world || plan->rank != m->ctx->rank) && m->ctx->world > 1)
    usage("plan rank/world does not match the context");
  ESG_CUDA(cudaSetDevice(m->ctx->device));
  model_prepare(m, g, plan, species);
  ESG_API_END
}

int esg_prepared_info(const esg_model* m, int64_t info[3]) {
  ESG_API_BEGIN
  NEED(m, "model");
  model_prepared_info(m, info);
  ESG_API_END
}

int esg_forward(esg_model* m, float* node_out, float* edge_out, esg_timing* timing) {
  ESG_API_BEGIN
  NEED(m, "model");
  if (!m->ctx || !m->dev) usage("model was created without a device context");
  ESG_CUDA(cudaSetDevice(m->ctx->device));
  model_forward_to_host(m, timing, node_out, edge_out, false);
  ESG_API_END
}

int esg_forward_async(esg_model* m, float* node_out, float* edge_out, esg_timing* timing) {
  ESG_API_BEGIN
  NEED(m, "model");
  if (!m->ctx || !m->dev) usage("model was created without a device context");
  ESG_CUDA(cudaSetDevice(m->ctx->device));
  model_forward_to_host(m, timing, node_out, edge_out, true);
  ESG_API_END
}

int esg_forward_wait(esg_model* m) {
  ESG_API_BEGIN
  NEED(m, "model");
  if (!m->ctx || !m->dev) usage("model was created without a device context");
  ESG_CUDA(cudaSetDevice(m->ctx->device));
  model_outputs_wait(m);
  ESG_API_END
}

int esg_profile(esg_model* m, int enable, double* ms, int64_t* counts) {
  ESG_API_BEGIN
  NEED(m, "model");
  if (!m->dev) usage("model was created without a device context");
  model_profile(m, enable, ms, counts);
  ESG_API_END
}

int esg_forward_outputs(const esg_model* m, const float** no, const float** eo, const float** nf, const float** ef) {
  ESG_API_BEGIN
  NEED(m, "model");
  model_outputs(m, no, eo, nf, ef);
  ESG_API_END
}

int esg_edge_rotations(esg_ctx* ctx, int64_t n_edges, const double* disp, int l_max, float* blocks) {
  ESG_API_BEGIN
  NEED(ctx, "context");
  if (n_edges < 0) usage("negative edge count");
  if (n_edges && (!disp || !blocks)) usage("edge rotations: NULL array");
  ESG_CUDA(cudaSetDevice(ctx->device));
  edge_rotations(ctx, n_edges, disp, l_max, blocks);
  ESG_API_END
}

int esg_outputs_export(const esg_model* m, int64_t node_first, int64_t node_count, float* node_out,
                       int64_t edge_first, int64_t edge_count, float* edge_out) {
  ESG_API_BEGIN
  NEED(m, "model");
  if (!m->ctx || !m->dev) usage("model was created without a device context");
  ESG_CUDA(cudaSetDevice(m->ctx->device));
  model_copy_output_rows(m, node_first, node_count, node_out, edge_first, edge_count, edge_out);
  ESG_API_END
}

int esg_features_export(const esg_model* m, float* nodes, float* edges) {
  ESG_API_BEGIN
  NEED(m, "model");
  if (!m->ctx || !m->dev) usage("model was created without a device context");
  ESG_CUDA(cudaSetDevice(m->ctx->device));
  model_copy_features(m, nodes, edges);
  ESG_API_END
}

namespace {
esg_model* device_model(esg_model* m) {
  if (!m) usage("model is NULL");
  if (!m->ctx || !m->dev) usage("model was created without a device context");
  ESG_CUDA(cudaSetDevice(m->ctx->device));
  return m;
}
}  // namespace

namespace {
void put_text(const std::string& t, char* out, int64_t cap, int64_t* len) {
  if (len) *len = (int64_t)t.size();
  if (out) {
    if (cap < (int64_t)t.size() + 1) usage("output buffer too small");
    std::memcpy(out, t.c_str(), t.size() + 1);
  }
}
}  // namespace

int esg_partition_metrics(const esg_graph* g, const int32_t* node_to_part, int n_parts, esg_metrics* m,
                          esg_part_stats* parts, int64_t* volume) {
  ESG_API_BEGIN
  NEED(g, "graph");
  NEED(node_to_part, "node_to_part");
  NEED(m, "metrics");
  ESG_CUDA(cudaSetDevice(g->ctx->device));
  partition_metrics_gpu(g, node_to_part, n_parts, m, parts, volume);
  ESG_API_END
}

int esg_metrics_json(const esg_metrics* m, const esg_part_stats* parts, char* out, int64_t cap, int64_t* len) {
  ESG_API_BEGIN
  NEED(m, "metrics");
  if (m->n_parts > 0) NEED(parts, "parts");
  put_text(metrics_json(*m, parts), out, cap, len);
  ESG_API_END
}

int esg_partition_dot(const int64_t* volume, const esg_part_stats* parts, int n_parts, char* out, int64_t cap,
                      int64_t* len) {
  ESG_API_BEGIN
  NEED(volume, "volume");
  NEED(parts, "parts");
  if (n_parts < 1) usage("n_parts must be positive");
  put_text(partition_dot(volume, parts, n_parts), out, cap, len);
  ESG_API_END
}

int esg_assignment_write(const char* path, const int32_t* node_to_part, int64_t n) {
  ESG_API_BEGIN
  NEED(path, "path");
  if (n > 0) NEED(node_to_part, "node_to_part");
  write_assignment(path, node_to_part, n);
  ESG_API_END
}

int esg_assignment_read(const char* path, int32_t* node_to_part, int64_t cap, int64_t* n, int* n_parts) {
  ESG_API_BEGIN
  NEED(path, "path");
  NEED(n, "n");
  int np = 0;
  const auto a = read_assignment(path, &np);
  *n = (int64_t)a.size();
  if (n_parts) *n_parts = np;
  if (node_to_part) {
    if (cap < (int64_t)a.size()) usage("node_to_part buffer too small");
    std::copy(a.begin(), a.end(), node_to_part);
  }
  ESG_API_END
}

int esg_blocks_count(esg_model* m, int64_t* n_blocks, int64_t* n_values) {
  ESG_API_BEGIN
  blocks_count(device_model(m), n_blocks, n_values);
  ESG_API_END
}

int esg_blocks_export(esg_model* m, int basis, int symmetrize_onsite, esg_block_key* keys, double* values) {
  ESG_API_BEGIN
  static_assert(sizeof(esg_block_key) == sizeof(BlockRec), "key record layout");
  blocks_export(device_model(m), basis, symmetrize_onsite != 0, reinterpret_cast<BlockRec*>(keys), values);
  ESG_API_END
}

int esg_blocks_export_device(esg_model* m, int basis, int symmetrize_onsite, int value_bytes, void* d_keys,
                             void* d_values, float* kernel_ms) {
  ESG_API_BEGIN
  blocks_export_device(device_model(m), basis, symmetrize_onsite != 0, value_bytes, d_keys, d_values, kernel_ms);
  ESG_API_END
}

int esg_blocks_write_shard(esg_model* m, const char* path, int basis, int symmetrize_onsite, int value_bytes) {
  ESG_API_BEGIN
  NEED(path, "path");
  blocks_write_shard(device_model(m), path, basis, symmetrize_onsite != 0, value_bytes);
  ESG_API_END
}

int esg_blocks_write_text(esg_model* m, const char* path, int basis, int symmetrize_onsite) {
  ESG_API_BEGIN
  NEED(path, "path");
  blocks_write_text(device_model(m), path, basis, symmetrize_onsite != 0);
  ESG_API_END
}

int esg_build_targets(esg_model* m, int64_t n_blocks, const esg_block_key* keys, const double* values,
                      float* node_target, uint8_t* node_mask, float* edge_target, uint8_t* edge_mask,
                      int64_t* count) {
  ESG_API_BEGIN
  if (n_blocks < 0) usage("n_blocks must be non-negative");
  if (n_blocks > 0) {
    NEED(keys, "keys");
    NEED(values, "values");
  }
  const int64_t c = build_targets(device_model(m), n_blocks, reinterpret_cast<const BlockRec*>(keys), values,
                                  node_target, node_mask, edge_target, edge_mask);
  if (count) *count = c;
  ESG_API_END
}

int esg_blocks_read_text(const char* path, int64_t* n_blocks, int64_t* n_values, esg_block_key* keys,
                         double* values) {
  ESG_API_BEGIN
  NEED(path, "path");
  const BlockSet s = read_blocks_text(path);
  if (n_blocks) *n_blocks = (int64_t)s.keys.size();
  if (n_values) *n_values = (int64_t)s.values.size();
  static_assert(sizeof(esg_block_key) == sizeof(BlockRec), "key record layout");
  if (keys) std::memcpy(keys, s.keys.data(), sizeof(BlockRec) * s.keys.size());
  if (values) std::memcpy(values, s.values.data(), sizeof(double) * s.values.size());
  ESG_API_END
}

int esg_blocks_merge_text(const char* const* shard_paths, int n_shards, const char* out_path) {
  ESG_API_BEGIN
  NEED(out_path, "out_path");
  if (n_shards < 0 || (n_shards > 0 && !shard_paths)) usage("shard_paths");
  std::vector<BlockSet> sets;
  sets.reserve(n_shards);
  uint32_t basis0 = 0, flags0 = 0;
  for (int r = 0; r < n_shards; ++r) {
    NEED(shard_paths[r], "shard path");
    ShardHeader h;
    sets.push_back(read_shard(shard_paths[r], &h));
    if (r == 0) {
      basis0 = h.basis;
      flags0 = h.flags;
    } else if (h.basis != basis0 || h.flags != flags0) {
      data("shards mix block bases or on-site symmetrisation");
    }
  }
  std::vector<const BlockSet*> ptrs;
  for (const auto& s : sets) ptrs.push_back(&s);
  write_blocks_text(out_path, ptrs);
  ESG_API_END
}

int esg_blocks_size(esg_model* m, int64_t* n) {
  ESG_API_BEGIN
  NEED(n, "n_values");
  blocks_count(device_model(m), nullptr, n);
  ESG_API_END
}

int esg_blocks_uncoupled(esg_model* m, double* out) {
  ESG_API_BEGIN
  NEED(out, "out");
  blocks_export(device_model(m), ESG_BLOCKS_UNCOUPLED, false, nullptr, out);
  ESG_API_END
}

int esg_set_targets(esg_model* m, const float* node_target, const uint8_t* node_mask, const float* edge_target,
                    const uint8_t* edge_mask) {
  ESG_API_BEGIN
  NEED(m, "model");
  if (!m->ctx || !m->dev) usage("model was created without a device context");
  ESG_CUDA(cudaSetDevice(m->ctx->device));
  model_set_targets(m, node_target, node_mask, edge_target, edge_mask);
  ESG_API_END
}

int esg_loss_grad(esg_model* m, int64_t n_total, double partials[3], double* loss, float* grads) {
  ESG_API_BEGIN
  NEED(m, "model");
  NEED(loss, "loss");
  if (!m->ctx || !m->dev) usage("model was created without a device context");
  ESG_CUDA(cudaSetDevice(m->ctx->device));
  double p[3];
  model_loss_grad(m, n_total, partials ? partials : p, loss, grads);
  ESG_API_END
}

void esg_adam_default_config(esg_adam_config* c) {
  if (!c) return;
  *c = esg_adam_config{5e-3, 0.9, 0.999, 1e-8, 100, 0.5, 1e-4, 1e-6};
}

int esg_adam_create(const esg_model* m, const esg_adam_config* cfg, esg_adam** out) {
  ESG_API_BEGIN
  NEED(m, "model");
  NEED(out, "out");
  auto* a = new esg_adam();
  if (cfg)
    a->cfg = *cfg;
  else
    esg_adam_default_config(&a->cfg);
  a->m.assign(m->host_params.size(), 0.0);
  a->v.assign(m->host_params.size(), 0.0);
  *out = a;
  ESG_API_END
}
void esg_adam_destroy(esg_adam* a) {
  if (a && a->d_m) {
    cudaSetDevice(a->device);
    cudaFree(a->d_m);
    cudaFree(a->d_v);
  }
  delete a;
}
double esg_adam_lr(const esg_adam* a) { return a ? (a->lr < 0 ? a->cfg.lr : a->lr) : 0.0; }

int esg_adam_apply(esg_adam* opt, esg_model* m, const float* grads, double loss) {
  ESG_API_BEGIN
  NEED(opt, "optimizer");
  NEED(m, "model");
  NEED(grads, "grads");
  if (opt->m.size() != m->host_params.size()) usage("optimizer built for another model");
  if (m->ctx && m->dev) ESG_CUDA(cudaSetDevice(m->ctx->device));
  adam_update(opt, m, grads, loss);  // the device step repacks the weights itself
  ESG_API_END
}

int esg_train_step(esg_model* m, esg_adam* opt, int64_t n_total, double* loss, esg_timing* timing) {
  ESG_API_BEGIN
  NEED(m, "model");
  NEED(opt, "optimizer");
  NEED(loss, "loss");
  if (!m->ctx || !m->dev) usage("model was created without a device context");
  ESG_CUDA(cudaSetDevice(m->ctx->device));
  if (opt->m.size() != m->host_params.size()) usage("optimizer built for another model");
  check_param_sync(m, "before step");
  std::vector<float> g(m->host_params.size());
  double partials[3];
  model_loss_grad(m, n_total, partials, loss, g.data());
  adam_update(opt, m, g.data(), *loss);  // on the device; refreshes the host parameters
  check_param_sync(m, "after update");
  if (timing) {
    double f = 0, b = 0;
    model_train_timing(m, &f, &b);
    *timing = esg_timing{};
    timing->forward_ms = f;
    timing->message_ms = b;
  }
  ESG_API_END
}

int esg_checkpoint_save(const esg_model* m, const esg_adam* opt, const char* config_text, const char* path) {
  ESG_API_BEGIN
  NEED(m, "model");
  NEED(path, "path");
  std::ofstream out(path, std::ios::binary);
  if (!out) data(std::string("cannot open file for writing: ") + path);
  const std::string cfg = config_text ? config_text : "";
  out.write("ESGNNCK1", 8);
  ckpt_u64(out, 1);  // version
  ckpt_u64(out, cfg.size());
  out.write(cfg.data(), (std::streamsize)cfg.size());
  ckpt_u64(out, sizeof(float));
  ckpt_u64(out, m->params.entries.size());
  for (const auto& e : m->params.entries) {
    ckpt_u64(out, e.name.size());
    out.write(e.name.data(), (std::streamsize)e.name.size());
    ckpt_u64(out, (uint64_t)e.rows);
    ckpt_u64(out, (uint64_t)e.cols);
    out.write(reinterpret_cast<const char*>(m->host_params.data() + e.offset),
              (std::streamsize)((size_t)e.rows * e.cols * sizeof(float)));
  }
  if (opt) {
    if (opt->m.size() != m->host_params.size()) usage("optimizer built for another model");
    out.write("ESGADAM1", 8);
    ckpt_u64(out, (uint64_t)opt->t);
    ckpt_f64(out, opt->lr);
    ckpt_f64(out, opt->best);
    ckpt_u64(out, (uint64_t)opt->stale);
    out.write(reinterpret_cast<const char*>(&opt->cfg), sizeof(opt->cfg));
    adam_host_moments(opt);
    ckpt_u64(out, opt->m.size());
    out.write(reinterpret_cast<const char*>(opt->m.data()), (std::streamsize)(opt->m.size() * sizeof(double)));
    out.write(reinterpret_cast<const char*>(opt->v.data()), (std::streamsize)(opt->v.size() * sizeof(double)));
  }
  if (!out) data(std::string("write failed: ") + path);
  ESG_API_END
}

int esg_checkpoint_load(esg_model* m, esg_adam* opt, const char* path, char* config_out, int64_t cap) {
  ESG_API_BEGIN
  NEED(m, "model");
  NEED(path, "path");
  std::ifstream in(path, std::ios::binary);
  if (!in) data(std::string("cannot open file: ") + path);
  char magic[8];
  in.read(magic, 8);
  if (!in || std::memcmp(magic, "ESGNNCK1", 8) != 0) data(std::string("not a checkpoint file: ") + path);
  if (ckpt_read_u64(in) != 1) data("unsupported checkpoint version");
  std::string cfg(ckpt_read_u64(in), '\0');
  in.read(cfg.data(), (std::streamsize)cfg.size());
  if (ckpt_read_u64(in) != sizeof(float)) data("checkpoint precision does not match the run precision");
  if (ckpt_read_u64(in) != m->params.entries.size()) data("checkpoint entry count mismatch");
  std::vector<float> p(m->host_params.size());
  for (const auto& e : m->params.entries) {
    std::string name(ckpt_read_u64(in), '\0');
    in.read(name.data(), (std::streamsize)name.size());
    if (name != e.name) data("checkpoint entry order mismatch at " + name);
    const uint64_t rows = ckpt_read_u64(in), cols = ckpt_read_u64(in);
    if (rows != (uint64_t)e.rows || cols != (uint64_t)e.cols) data("checkpoint shape mismatch at " + name);
    in.read(reinterpret_cast<char*>(p.data() + e.offset), (std::streamsize)(rows * cols * sizeof(float)));
    if (!in) data("truncated checkpoint");
  }
  if (opt) {
    char om[8];
    in.read(om, 8);
    if (!in || std::memcmp(om, "ESGADAM1", 8) != 0) data("checkpoint has no optimizer state");
    const long t = (long)ckpt_read_u64(in);
    const double lr = ckpt_read_f64(in), best = ckpt_read_f64(in);
    const int stale = (int)ckpt_read_u64(in);
    esg_adam_config c{};
    in.read(reinterpret_cast<char*>(&c), sizeof(c));
    if (ckpt_read_u64(in) != p.size()) data("optimizer state size mismatch");
    std::vector<double> mm(p.size()), vv(p.size());
    in.read(reinterpret_cast<char*>(mm.data()), (std::streamsize)(mm.size() * sizeof(double)));
    in.read(reinterpret_cast<char*>(vv.data()), (std::streamsize)(vv.size() * sizeof(double)));
    if (!in) data("truncated optimizer state");
    opt->t = t;
    opt->lr = lr;
    opt->best = best;
    opt->stale = stale;
    opt->cfg = c;
    opt->m.swap(mm);
    opt->v.swap(vv);
    opt->host_current = true;  // uploaded before the next device step
  }
  m->host_params.swap(p);
  if (m->ctx && m->dev) {
    ESG_CUDA(cudaSetDevice(m->ctx->device));
    model_upload_params(m);
  }
  if (config_out && cap > 0) {
    const size_t n = std::min<size_t>(cfg.size(), (size_t)cap - 1);
    std::memcpy(config_out, cfg.data(), n);
    config_out[n] = '\0';
  }
  ESG_API_END
}

}  // extern "C"
