// plan_gpu.cu -- runtime::build_comm_plan (comm_plan.cpp:11-106) on the
// device from the device CSR.  Produces the same esg_plan as the host
// restatement plan_from_csr (capi.cpp), bit for bit:
//   owned rows    nodes of this rank in ascending global id        (:24-30)
//   halo rows     distinct remote sources of owned edges, sorted by
//                 (owner, id)                                        (:32-50)
//   owned edges   edges whose destination this rank owns, in global
//                 (dst-major) order, with local src / dst rows       (:53-71)
//   send rows     per peer, the owned sources of that peer's edges,
//                 ascending id                                       (:73-92)
//   recv ranges   contiguous halo rows per owner                     (:94-103)
// Every rank scans all E edges on the GPU (a few ms at C4) instead of on
// the host; only the rank-local results travel to the host.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <map>
#include <vector>

#include "esg_internal.h"

namespace esg {
namespace {

template <typename T>
T* galloc_ctx(esg_ctx* ctx, size_t n) {
  return static_cast<T*>(ctx->cache.alloc(n * sizeof(T)));
}

__global__ void k_flag_owned(const int* __restrict__ part, int n, int rank, int* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = part[i] == rank;
}
__global__ void k_owned_rows(const int* __restrict__ part, int n, int rank, const int* __restrict__ scan,
                             int* __restrict__ owned_row, int* __restrict__ row_global) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool own = part[i] == rank;
  owned_row[i] = own ? scan[i] : -1;
  if (own) row_global[scan[i]] = i;
}
// warp per destination j of this rank: remote sources need a halo row;
// owned-edge counts for the edge compaction
__global__ void k_halo_need(const int64_t* __restrict__ off, const int* __restrict__ src,
                            const int* __restrict__ part, int n, int rank, uint8_t* __restrict__ need,
                            int64_t* __restrict__ cnt) {
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (j >= n) return;
  const bool own = part[j] == rank;
  if (lane == 0) cnt[j] = own ? off[j + 1] - off[j] : 0;
  if (!own) return;
  for (int64_t k = off[j] + lane; k < off[j + 1]; k += 32) {
    const int s = src[k];
    if (part[s] != rank) need[s] = 1;
  }
}
__global__ void k_halo_keys(const int* __restrict__ ids, int m, const int* __restrict__ part,
                            uint64_t* __restrict__ keys) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < m) keys[q] = ((uint64_t)(uint32_t)part[ids[q]] << 32) | (uint32_t)ids[q];
}
__global__ void k_halo_rows(const uint64_t* __restrict__ keys, int m, int n_owned, int* __restrict__ halo_row,
                            int* __restrict__ row_global) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  const int s = (int)(keys[q] & 0xffffffffu);
  halo_row[s] = n_owned + q;
  row_global[n_owned + q] = s;
}
// warp per owned destination: its edges at base[j], in CSR order
__global__ void k_fill_edges(const int64_t* __restrict__ off, const int* __restrict__ src,
                             const int* __restrict__ part, int n, int rank, const int64_t* __restrict__ base,
                             const int* __restrict__ owned_row, const int* __restrict__ halo_row,
                             int* __restrict__ edge_index, int* __restrict__ src_row, int* __restrict__ dst_row) {
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (j >= n || part[j] != rank) return;
  const int64_t b = base[j];
  const int dr = owned_row[j];
  for (int64_t k = off[j] + lane; k < off[j + 1]; k += 32) {
    const int s = src[k];
    const int64_t t = b + (k - off[j]);
    edge_index[t] = (int)k;
    src_row[t] = owned_row[s] >= 0 ? owned_row[s] : halo_row[s];
    dst_row[t] = dr;
  }
}
// warp per destination of another rank p: owned sources are sent to p
__global__ void k_send_flags(const int64_t* __restrict__ off, const int* __restrict__ src,
                             const int* __restrict__ part, int n, int rank, int n_parts, uint8_t* __restrict__ flags) {
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (j >= n) return;
  const int p = part[j];
  if (p == rank) return;
  for (int64_t k = off[j] + lane; k < off[j + 1]; k += 32) {
    const int s = src[k];
    if (part[s] == rank) flags[(int64_t)p * n + s] = 1;
  }
}

// seg[r] = first owned edge of owned row r (rows ascend in global id and
// base is the edge offset per global node), seg[n_owned] = n_e
__global__ void k_plan_seg(const int64_t* __restrict__ base, const int* __restrict__ row_global, int n_owned,
                           int64_t n_e, int64_t* __restrict__ seg) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n_owned) seg[r] = base[row_global[r]];
  if (r == n_owned) seg[r] = n_e;
}

}  // namespace

esg_plan* plan_build_gpu(const esg_graph* g, const int32_t* species, const int32_t* part_h, int n_parts,
                         int rank) {
  if (rank < 0 || rank >= n_parts) usage("rank outside the assignment");
  const int n = g->n;
  for (int i = 0; i < n; ++i)
    if (part_h[i] < 0 || part_h[i] >= n_parts) data("assignment part out of range");
  cudaStream_t st = build_stream(g->ctx);  // graph-side work: beside an async forward
  auto* P = new esg_plan();
  P->rank = rank;
  P->world = n_parts;
  int* part = galloc_ctx<int>(g->ctx, n);
  int* flag = galloc_ctx<int>(g->ctx, n + 1);
  int* scan = galloc_ctx<int>(g->ctx, n + 1);
  int* owned_row = galloc_ctx<int>(g->ctx, n);
  int* halo_row = galloc_ctx<int>(g->ctx, n);
  int* row_global = galloc_ctx<int>(g->ctx, n);
  uint8_t* need = galloc_ctx<uint8_t>(g->ctx, n);
  int64_t* cnt = galloc_ctx<int64_t>(g->ctx, n + 1);
  int64_t* base = galloc_ctx<int64_t>(g->ctx, n + 1);
  int* ids = galloc_ctx<int>(g->ctx, n);
  int* n_sel = galloc_ctx<int>(g->ctx, 1);
  uint64_t* keys = galloc_ctx<uint64_t>(g->ctx, n);
  uint64_t* keys_sorted = galloc_ctx<uint64_t>(g->ctx, n);
  uint8_t* sflags = galloc_ctx<uint8_t>(g->ctx, (size_t)n * n_parts);
  h2d_staged(g->ctx, part, part_h, sizeof(int) * n, st);
  ESG_CUDA(cudaMemsetAsync(need, 0, n, st));
  ESG_CUDA(cudaMemsetAsync(halo_row, 0xff, sizeof(int) * n, st));
  ESG_CUDA(cudaMemsetAsync(sflags, 0, (size_t)n * n_parts, st));
  ESG_CUDA(cudaMemsetAsync(flag + n, 0, sizeof(int), st));
  ESG_CUDA(cudaMemsetAsync(cnt + n, 0, sizeof(int64_t), st));
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  auto ensure_tmp = [&](size_t b) {
    if (b > tmp_bytes) {
      if (tmp) g->ctx->cache.release(tmp);
      tmp = galloc_ctx<uint8_t>(g->ctx, b);
      tmp_bytes = b;
    }
  };
  const unsigned b1 = (unsigned)((n + 255) / 256), bw = (unsigned)(((int64_t)n * 32 + 255) / 256);
  // owned rows
  k_flag_owned<<<b1, 256, 0, st>>>(part, n, rank, flag);
  size_t need_b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need_b, flag, scan, n + 1, st);
  ensure_tmp(need_b);
  cub::DeviceScan::ExclusiveSum(tmp, need_b, flag, scan, n + 1, st);
  k_owned_rows<<<b1, 256, 0, st>>>(part, n, rank, scan, owned_row, row_global);
  int n_owned = 0;
  d2h_small(g->ctx, &n_owned, scan + n, sizeof(int), st);
  // halo rows, sorted by (owner, id)
  if (n) k_halo_need<<<bw, 256, 0, st>>>(g->d_off, g->d_src, part, n, rank, need, cnt);
  thrust::counting_iterator<int> it(0);
  need_b = 0;
  cub::DeviceSelect::Flagged(nullptr, need_b, it, need, ids, n_sel, n, st);
  ensure_tmp(need_b);
  cub::DeviceSelect::Flagged(tmp, need_b, it, need, ids, n_sel, n, st);
  int n_halo = 0;
  d2h_small(g->ctx, &n_halo, n_sel, sizeof(int), st);
  ESG_CUDA(cudaStreamSynchronize(st));
  if (n_halo) {
    k_halo_keys<<<(unsigned)((n_halo + 255) / 256), 256, 0, st>>>(ids, n_halo, part, keys);
    need_b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need_b, keys, keys_sorted, n_halo, 0, 64, st);
    ensure_tmp(need_b);
    cub::DeviceRadixSort::SortKeys(tmp, need_b, keys, keys_sorted, n_halo, 0, 64, st);
    k_halo_rows<<<(unsigned)((n_halo + 255) / 256), 256, 0, st>>>(keys_sorted, n_halo, n_owned, halo_row,
                                                                   row_global);
  }
  // owned edges in global order
  need_b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need_b, cnt, base, n + 1, st);
  ensure_tmp(need_b);
  cub::DeviceScan::ExclusiveSum(tmp, need_b, cnt, base, n + 1, st);
  int64_t n_e = 0;
  d2h_small(g->ctx, &n_e, base + n, sizeof(int64_t), st);
  ESG_CUDA(cudaStreamSynchronize(st));
  int* edge_index = galloc_ctx<int>(g->ctx, (size_t)std::max<int64_t>(n_e, 1));
  int* src_row = galloc_ctx<int>(g->ctx, (size_t)std::max<int64_t>(n_e, 1));
  int* dst_row = galloc_ctx<int>(g->ctx, (size_t)std::max<int64_t>(n_e, 1));
  if (n) {
    k_fill_edges<<<bw, 256, 0, st>>>(g->d_off, g->d_src, part, n, rank, base, owned_row, halo_row, edge_index,
                                      src_row, dst_row);
    k_send_flags<<<bw, 256, 0, st>>>(g->d_off, g->d_src, part, n, rank, n_parts, sflags);
  }
  ESG_CUDA(cudaGetLastError());
  // to the host: rows, edges, owned-row map, per-peer send lists
  P->n_owned = n_owned;
  P->n_rows = n_owned + n_halo;
  P->n_edges = n_e;
  P->row_global.resize(P->n_rows);
  std::vector<int> owned_h(n), halo_keys_owner;
  if (P->n_rows)
    d2h_small(g->ctx, P->row_global.data(), row_global, sizeof(int) * P->n_rows, st);
  // the per-edge arrays stay on the device (prepare copies them device to
  // device); the host copies are made only if the plan is exported
  P->ctx = g->ctx;
  g->ctx->plans.insert(P);
  P->d_edge_index = edge_index;
  P->d_src_row = src_row;
  P->d_dst_row = dst_row;
  P->d_seg = galloc_ctx<int64_t>(g->ctx, (size_t)n_owned + 1);
  k_plan_seg<<<(unsigned)((n_owned + 256) / 256), 256, 0, st>>>(base, row_global, n_owned, n_e, P->d_seg);
  g->ctx->launches += 1;
  if (n) d2h_small(g->ctx, owned_h.data(), owned_row, sizeof(int) * n, st);
  std::map<int, Neighbor> nb;
  for (int p = 0; p < n_parts; ++p) {
    if (p == rank) continue;
    need_b = 0;
    cub::DeviceSelect::Flagged(nullptr, need_b, it, sflags + (size_t)p * n, ids, n_sel, n, st);
    ensure_tmp(need_b);
    cub::DeviceSelect::Flagged(tmp, need_b, it, sflags + (size_t)p * n, ids, n_sel, n, st);
    int m = 0;
    d2h_small(g->ctx, &m, n_sel, sizeof(int), st);
    ESG_CUDA(cudaStreamSynchronize(st));
    if (!m) continue;
    std::vector<int> s(m);
    d2h_small(g->ctx, s.data(), ids, sizeof(int) * m, st);
    Neighbor& x = nb[p];
    x.peer = p;
    for (int id : s) x.send_rows.push_back(owned_h[id]);
  }
  ESG_CUDA(cudaStreamSynchronize(st));
  // receive ranges: contiguous halo rows per owner (the halo rows are sorted by owner)
  int at = n_owned;
  for (int q = n_owned; q < P->n_rows;) {
    const int owner = part_h[P->row_global[q]];
    int r = q;
    while (r < P->n_rows && part_h[P->row_global[r]] == owner) ++r;
    Neighbor& x = nb[owner];
    x.peer = owner;
    x.recv_row = at;
    x.recv_count = r - q;
    at += x.recv_count;
    q = r;
  }
  for (auto& kv : nb) P->nbrs.push_back(kv.second);
  if (species)
    for (int r = 0; r < P->n_rows; ++r) P->row_species.push_back(species[P->row_global[r]]);
  for (void* p : {(void*)part, (void*)flag, (void*)scan, (void*)owned_row, (void*)halo_row, (void*)row_global,
                  (void*)need, (void*)cnt, (void*)base, (void*)ids, (void*)n_sel, (void*)keys, (void*)keys_sorted,
                  (void*)sflags, tmp})
    g->ctx->cache.release(p);
  return P;
}

}  // namespace esg

void esg_plan::host_sync_edges() const {
  if (!d_src_row || (int64_t)src_row.size() == n_edges) return;
  edge_index.resize(n_edges);
  src_row.resize(n_edges);
  dst_row.resize(n_edges);
  if (n_edges) {
    esg::d2h_small(ctx, edge_index.data(), d_edge_index, sizeof(int32_t) * n_edges, esg::build_stream(ctx));
    esg::d2h_small(ctx, src_row.data(), d_src_row, sizeof(int32_t) * n_edges, esg::build_stream(ctx));
    esg::d2h_small(ctx, dst_row.data(), d_dst_row, sizeof(int32_t) * n_edges, esg::build_stream(ctx));
  }
}

esg_plan::~esg_plan() {
  if (!ctx) return;
  for (void* p : {(void*)d_edge_index, (void*)d_src_row, (void*)d_dst_row, (void*)d_seg}) ctx->cache.release(p);
  ctx->plans.erase(this);
}
