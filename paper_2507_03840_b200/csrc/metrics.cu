// metrics.cu -- partition metrics on the device:
// partition::compute_metrics (metrics.cpp:49-88) and the part-to-part volume
// matrix behind write_dot (metrics.cpp:141-166), from the graph's dst-major
// CSR and an assignment.
//
// Per destination node one warp counts its in-edges, the cut ones and
// collects the cut (receiving part, source node) keys; a cub radix sort makes
// the keys unique, and every distinct key adds one to volume[part(src)][q].
// All counts are integers (exact, order-free), so the summary equals the
// reference's bit for bit; the doubles are computed on the host with the
// reference's expressions.
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <algorithm>
#include <vector>

#include "esg_internal.h"

namespace esg {

namespace {

template <typename T>
T* dmalloc(size_t n) {
  T* p = nullptr;
  if (n) ESG_CUDA(cudaMalloc(&p, n * sizeof(T)));
  return p;
}

// counts[0..P) nodes, [P..2P) edges; counts[2P] cut edges; cut[j] = number of
// cut in-edges of node j
__global__ void k_metric_counts(const int64_t* __restrict__ off, const int32_t* __restrict__ src,
                                const int32_t* __restrict__ part, int n, int P, unsigned long long* __restrict__ counts,
                                int64_t* __restrict__ cut) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const int q = part[j];
  int c = 0;
  for (int64_t k = off[j] + lane; k < off[j + 1]; k += 32) c += part[src[k]] != q;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) {
    cut[j] = c;
    atomicAdd(&counts[q], 1ull);
    atomicAdd(&counts[P + q], (unsigned long long)(off[j + 1] - off[j]));
    if (c) atomicAdd(&counts[2 * P], (unsigned long long)c);
  }
}

__global__ void k_cut_keys(const int64_t* __restrict__ off, const int32_t* __restrict__ src,
                           const int32_t* __restrict__ part, int n, const int64_t* __restrict__ pos,
                           uint64_t* __restrict__ keys) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const int q = part[j];
  int64_t at = pos[j];
  for (int64_t k0 = off[j]; k0 < off[j + 1]; k0 += 32) {
    const int64_t k = k0 + lane;
    const bool take = k < off[j + 1] && part[src[k]] != q;
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (take) keys[at + __popc(m & ((1u << lane) - 1))] = ((uint64_t)(uint32_t)q << 32) | (uint32_t)src[k];
    at += __popc(m);
  }
}

// sorted keys: each distinct (q, src) adds one to volume[part(src) * P + q]
__global__ void k_pair_volume(const uint64_t* __restrict__ keys, int64_t n, const int32_t* __restrict__ part, int P,
                              unsigned long long* __restrict__ vol) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  if (i > 0 && keys[i - 1] == k) return;
  const int q = (int)(k >> 32), f = part[(uint32_t)k];
  atomicAdd(&vol[(size_t)f * P + q], 1ull);
}

}  // namespace

// out_parts: nodes, edges, neighbors, recv_volume per part; vol (P x P,
// from-part major) may be null
void partition_metrics_gpu(const esg_graph* g, const int32_t* part_h, int P, esg_metrics* m, esg_part_stats* parts,
                           int64_t* vol_out) {
  const int n = g->n;
  cudaStream_t st = g->ctx->stream;
  if (P < 1 || P > 4096) usage("n_parts must be in [1, 4096]");
  for (int i = 0; i < n; ++i)
    if (part_h[i] < 0 || part_h[i] >= P) data("part id out of range: " + std::to_string(part_h[i]));
  int32_t* part = dmalloc<int32_t>(n);
  unsigned long long* counts = dmalloc<unsigned long long>(2 * (size_t)P + 1);
  unsigned long long* vol = dmalloc<unsigned long long>((size_t)P * P);
  int64_t* cut = dmalloc<int64_t>((size_t)n + 1);
  int64_t* pos = dmalloc<int64_t>((size_t)n + 1);
  if (n) ESG_CUDA(cudaMemcpyAsync(part, part_h, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
  ESG_CUDA(cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * (2 * P + 1), st));
  ESG_CUDA(cudaMemsetAsync(vol, 0, sizeof(unsigned long long) * P * P, st));
  ESG_CUDA(cudaMemsetAsync(cut + n, 0, sizeof(int64_t), st));
  const unsigned grid = (unsigned)((n + 7) / 8);
  if (n) {
    k_metric_counts<<<grid, 256, 0, st>>>(g->d_off, g->d_src, part, n, P, counts, cut);
    ++g->ctx->launches;
  }
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cut, pos, n + 1, st);
  void* tmp = dmalloc<uint8_t>(tb);
  ESG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cut, pos, n + 1, st));
  auto free_ptr = [](void* q) {
    if (q) cudaFree(q);
  };
  int64_t n_keys = 0;
  ESG_CUDA(cudaMemcpyAsync(&n_keys, pos + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  ESG_CUDA(cudaStreamSynchronize(st));
  free_ptr(tmp);
  if (n_keys) {
    uint64_t* keys = dmalloc<uint64_t>(n_keys);
    uint64_t* sorted = dmalloc<uint64_t>(n_keys);
    k_cut_keys<<<grid, 256, 0, st>>>(g->d_off, g->d_src, part, n, pos, keys);
    ++g->ctx->launches;
    int hi = 32;  // key bits: src (32) + q
    while ((1 << (hi - 32)) < P) ++hi;
    tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, n_keys, 0, hi, st);
    tmp = dmalloc<uint8_t>(tb);
    ESG_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, keys, sorted, n_keys, 0, hi, st));
    k_pair_volume<<<(unsigned)((n_keys + 255) / 256), 256, 0, st>>>(sorted, n_keys, part, P, vol);
    g->ctx->launches += 2;
    ESG_CUDA(cudaStreamSynchronize(st));
    free_ptr(tmp);
    free_ptr(keys);
    free_ptr(sorted);
  }
  std::vector<unsigned long long> hc(2 * P + 1), hv((size_t)P * P);
  ESG_CUDA(cudaMemcpyAsync(hc.data(), counts, sizeof(unsigned long long) * hc.size(), cudaMemcpyDeviceToHost, st));
  ESG_CUDA(cudaMemcpyAsync(hv.data(), vol, sizeof(unsigned long long) * hv.size(), cudaMemcpyDeviceToHost, st));
  ESG_CUDA(cudaStreamSynchronize(st));
  for (void* p : {(void*)part, (void*)counts, (void*)vol, (void*)cut, (void*)pos}) free_ptr(p);

  // metrics.cpp:49-88 summary on the host (integer counts, the reference's doubles)
  *m = esg_metrics{};
  m->n_parts = P;
  m->cut_edges = (int64_t)hc[2 * P];
  long nbr_sum = 0, node_total = 0, node_top = 0, edge_total = 0, edge_top = 0;
  for (int q = 0; q < P; ++q) {
    esg_part_stats s{};
    s.nodes = (int64_t)hc[q];
    s.edges = (int64_t)hc[P + q];
    for (int f = 0; f < P; ++f) {
      const int64_t v = (int64_t)hv[(size_t)f * P + q];
      s.recv_volume += v;
      s.neighbors += v > 0;
    }
    m->total_recv += s.recv_volume;
    nbr_sum += s.neighbors;
    m->max_neighbors = std::max(m->max_neighbors, s.neighbors);
    node_total += s.nodes;
    node_top = std::max<long>(node_top, s.nodes);
    edge_total += s.edges;
    edge_top = std::max<long>(edge_top, s.edges);
    if (parts) parts[q] = s;
  }
  m->mean_neighbors = double(nbr_sum) / double(P);
  m->node_imbalance = node_total == 0 ? 1.0 : double(node_top) * double(P) / double(node_total);
  m->edge_imbalance = edge_total == 0 ? 1.0 : double(edge_top) * double(P) / double(edge_total);
  if (vol_out)
    for (size_t i = 0; i < hv.size(); ++i) vol_out[i] = (int64_t)hv[i];
}

}  // namespace esg
