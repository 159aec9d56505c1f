// esg_internal.h -- shared internal declarations of libesg_b200.so.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <nccl.h>

#include <array>
#include <cstdint>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/esg.h"

namespace esg {

// Function attributes (dynamic SMEM caps) and SM counts belong to a device,
// not the process: these helpers keep them per device, so a
// context on a second GPU of the same process configures its own.
inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) d = 0;
  return d & 63;
}
// runs f once per device for this flag word (idempotent if two threads race)
template <typename F>
inline void once_per_device(std::atomic<uint64_t>& done, F&& f) {
  const uint64_t bit = 1ull << current_device();
  if (done.load(std::memory_order_acquire) & bit) return;
  f();
  done.fetch_or(bit, std::memory_order_release);
}
inline int sm_count() {
  static std::atomic<int> cache[64];
  const int d = current_device();
  int n = cache[d].load(std::memory_order_relaxed);
  if (!n) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || n <= 0) n = 148;
    cache[d].store(n, std::memory_order_relaxed);
  }
  return n;
}


// ---- error taxonomy (core/error.h:11-51) mapped to ESG_* codes ----------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void usage(const std::string& m) { throw Error(ESG_ERR_USAGE, m); }
[[noreturn]] inline void data(const std::string& m) { throw Error(ESG_ERR_DATA, m); }
void set_error(const std::string& m);

#define ESG_CUDA(x)                                                                     \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      throw ::esg::Error(e_ == cudaErrorMemoryAllocation ? ESG_ERR_OOM : ESG_ERR_CUDA,  \
                         std::string(#x) + ": " + cudaGetErrorString(e_));              \
  } while (0)
#define ESG_NCCL(x)                                                                     \
  do {                                                                                  \
    ncclResult_t r_ = (x);                                                              \
    if (r_ != ncclSuccess)                                                              \
      throw ::esg::Error(ESG_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// ---- host structures (structure.cpp) ------------------------------------
using M3 = std::array<std::array<double, 3>, 3>;
void wrap_positions(int n, double* pos, const M3& cell, const bool pbc[3]);
double face_spacing(const M3& cell, int d);

// ---- partition / plan ----------------------------------------------------
std::vector<int> lownn(int n, const double* pos, const M3& cell, const bool pbc[3],
                       const int32_t* deg, int depth, double r_cut);

struct Neighbor {
  int peer = -1;
  std::vector<int> send_rows;
  int recv_row = 0, recv_count = 0;
};

// ---- basis / layouts (basis.cpp, layout.h) ------------------------------
struct Basis {
  std::map<int, std::vector<int>> shells;  // Z ascending
  int n_orb(int z) const;
  int off(int z, int sh) const;
  int n_slots() const;
  int slot_l(int s) const;
};
struct HeadKey {
  int sa, sb, L;
};
struct HeadLayout {
  std::vector<HeadKey> keys;
  std::vector<int> offsets;
  int out_len = 0, max_l = 0;
  int segment(int a, int b, int L) const;
};
HeadLayout head_layout(const Basis& b);

struct MLayout {
  int l_max = 0, h = 0;
  std::vector<int> to_m, to_l, m_offset;
  int nd(int m) const { return l_max - m + 1; }
};
MLayout m_layout(int l_max);

std::string element_symbol(int z);
int atomic_number(const std::string& symbol);

struct ParamEntry {
  std::string name;
  int rows, cols, fan_in;
  int64_t offset;
};
struct ParamSet {
  std::vector<ParamEntry> entries;
  std::map<std::string, int> index;
  int64_t total = 0;
  void add(const std::string& n, int r, int c, int f);
  const ParamEntry& at(const std::string& n) const;
};
ParamSet register_params(const esg_model_config& cfg, const Basis& b, const HeadLayout& h);
void init_params(const ParamSet& p, uint64_t seed, std::vector<float>& out);
uint64_t param_hash(const ParamSet& p, const std::vector<float>& v);

// Real-basis coupling matrix C(la, lb, L): (2L+1) x ((2la+1)(2lb+1)) row-major
// (clebsch_gordan.h:19), computed by the Racah closed form.
std::vector<double> coupling_matrix(int la, int lb, int L);

}  // namespace esg

// ---- opaque handle bodies -----------------------------------------------
namespace esg {
// Device block cache of one context: freed blocks are kept (up to a byte
// budget) and handed out again by best fit, so a build -> use -> destroy
// cycle of same-sized graphs does not pay cudaMalloc/cudaFree (a first free
// of GB-sized blocks costs ~0.6 s of driver unmapping on B200).  A failed
// cudaMalloc flushes the cache and retries.
struct BlockCache {
  std::multimap<size_t, void*> free_blocks;  // capacity -> block
  std::map<void*, size_t> live;              // handed-out block -> capacity
  size_t cached = 0, budget = size_t(16) << 30;
  void* alloc(size_t bytes);
  void release(void* p);
  void flush();
};
}  // namespace esg

struct esg_graph;
struct esg_plan;

struct esg_ctx {
  int device = 0, rank = 0, world = 1;
  // live objects whose device arrays come from `cache`; a context destroyed
  // first releases their arrays and detaches them (destroy order is free)
  std::set<esg_graph*> graphs;
  std::set<esg_plan*> plans;
  cudaStream_t stream = nullptr;
  // graph builds run on their own stream (created on first use), so the next
  // structure's graph is built while an async forward still runs on `stream`
  cudaStream_t build_stream = nullptr;
  ncclComm_t comm = nullptr;
  int64_t launches = 0;  // kernels launched by this library
  esg::BlockCache cache;
  // zero-copy readback buffer (pinned, mapped): small device -> host reads
  // go through a kernel store instead of the copy engine, so they never queue
  // behind the multi-GB output copies of an async forward
  void* zc = nullptr;
  size_t zc_cap = 0;
  // pinned staging for small host -> device uploads (pageable copies are
  // synchronous and can serialise behind in-flight async copies)
  void* up = nullptr;
  size_t up_cap = 0;
};

namespace esg {
// the context's graph-side stream (graph build, Low-NN, comm plans; created on first use)
inline cudaStream_t build_stream(esg_ctx* ctx) {
  if (!ctx->build_stream) ESG_CUDA(cudaStreamCreateWithFlags(&ctx->build_stream, cudaStreamNonBlocking));
  return ctx->build_stream;
}
// graph.cu; synchronous on `st` (default: the context's stream); bytes % 4 == 0
void d2h_small(esg_ctx* ctx, void* host, const void* dev, size_t bytes, cudaStream_t st = nullptr);
void h2d_staged(esg_ctx* ctx, void* dev, const void* host, size_t bytes, cudaStream_t st = nullptr);
}

struct esg_graph {
  esg_ctx* ctx = nullptr;
  int n = 0;
  int64_t E = 0;
  int nimg[3] = {0, 0, 0};
  // device CSR (dst-major): offsets, src, packed shift, fp64 geometry
  int64_t* d_off = nullptr;
  int32_t* d_src = nullptr;
  uint32_t* d_shift = nullptr;  // (sx+512)<<20 | (sy+512)<<10 | (sz+512)
  double* d_disp = nullptr;     // E*3
  double* d_dist = nullptr;
  // host mirrors filled lazily
  mutable std::vector<int64_t> h_off;
  mutable std::vector<int32_t> h_src;
  void host_sync() const;          // offsets and sources
  void host_sync_offsets() const;  // offsets only (in-degrees, segment ranges)
};

struct esg_plan {
  int rank = 0, world = 1;
  int n_rows = 0, n_owned = 0;
  int64_t n_edges = 0;
  std::vector<int32_t> row_global, row_species;
  // per owned edge (host); a GPU-built plan keeps them on the device and
  // fills these only when exported (host_sync_edges)
  mutable std::vector<int32_t> edge_index, src_row, dst_row;
  esg_ctx* ctx = nullptr;  // owner of the device arrays (block cache)
  int32_t *d_edge_index = nullptr, *d_src_row = nullptr, *d_dst_row = nullptr;
  int64_t* d_seg = nullptr;  // n_owned + 1 destination segment offsets
  std::vector<esg::Neighbor> nbrs;
  void host_sync_edges() const;  // plan_gpu.cu
  ~esg_plan();
};

namespace esg {
struct DeviceModel;  // defined in model.cu
}

struct esg_model {
  esg_ctx* ctx = nullptr;
  esg_model_config cfg{};
  esg::Basis basis;
  esg::HeadLayout heads;
  esg::MLayout lay;
  esg::ParamSet params;
  std::vector<int> species_list;  // ascending Z
  std::vector<float> host_params;
  esg::DeviceModel* dev = nullptr;
};
