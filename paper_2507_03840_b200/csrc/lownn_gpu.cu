// lownn_gpu.cu -- partition::lownn_partition (lownn.cpp:23-133) on the
// device ("GPU Low-NN via segmented sorts").  Produces the
// same assignment as the host restatement `lownn` (host.cpp:73-173) bit for
// bit.  The reference recurses depth-first; here every level of the bisection
// tree is one pass over all atoms:
//   1. per-segment min / max of each coordinate (order-preserving integer
//      images of the doubles, integer atomics: exact)           (:37-60)
//   2. the host picks each segment's cut dimension from those extents with
//      the reference's rule (first uncut dimension, else the smallest
//      ceil(2 r / extent), ties to the highest index)           (:37-60)
//   3. two stable radix sorts -- by the coordinate of the segment's cut
//      dimension, then by segment -- starting from atom order, so each
//      segment ends up sorted by (coordinate, atom id), the reference
//      comparator (:72-76); -0.0 keys as 0.0 because the comparator sees them
//      equal
//   4. an inclusive scan of the in-degree weights and one CTA per segment
//      for the first minimiser of |2 prefix - total| over the admissible
//      split points (:78-91)
//   5. relabel: segment s splits into 2s (left) and 2s + 1 (right), which
//      after the last level is the reference's left-first DFS numbering.
#include <cub/cub.cuh>

#include <array>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "esg_internal.h"

namespace esg {
namespace {

__device__ __forceinline__ uint64_t ord_key(double x) {
  if (x == 0.0) x = 0.0;  // -0.0 and 0.0 compare equal in the reference
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
double from_ord(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double x;
  std::memcpy(&x, &b, sizeof x);
  return x;
}

// per (segment, dim): min and max order keys
__global__ void k_extent(const double* __restrict__ pos, const int* __restrict__ seg, int n,
                         unsigned long long* __restrict__ mn, unsigned long long* __restrict__ mx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int s = seg[i];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const unsigned long long k = ord_key(pos[3 * (int64_t)i + d]);
    atomicMin(mn + 3 * s + d, k);
    atomicMax(mx + 3 * s + d, k);
  }
}
__global__ void k_sort_keys(const double* __restrict__ pos, const int* __restrict__ seg, const int* __restrict__ dim,
                            int n, uint64_t* __restrict__ key, int* __restrict__ id) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = ord_key(pos[3 * (int64_t)i + dim[seg[i]]]);
  id[i] = i;
}
__global__ void k_gather_seg(const int* __restrict__ seg, const int* __restrict__ id, int n, int* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) out[j] = seg[id[j]];
}
__global__ void k_gather_w(const int64_t* __restrict__ w, const int* __restrict__ id, int n, int64_t* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) out[j] = w[id[j]];
}

struct DiffAt {
  int64_t diff;
  int p;
};
struct FirstMin {
  __device__ DiffAt operator()(const DiffAt& a, const DiffAt& b) const {
    return (b.diff < a.diff || (b.diff == a.diff && b.p < a.p)) ? b : a;
  }
};

// one CTA per segment: first p in [need, m - need] (and 1 <= p < m)
// minimising |2 * prefix(p) - total| (lownn.cpp:78-91); `need` default
constexpr int SPLIT_THREADS = 512;
__global__ void __launch_bounds__(SPLIT_THREADS) k_split(const int64_t* __restrict__ pre, const int64_t* __restrict__ off,
                                                         int need, int* __restrict__ split) {
  using BR = cub::BlockReduce<DiffAt, SPLIT_THREADS>;
  __shared__ typename BR::TempStorage tmp;
  const int s = blockIdx.x;
  const int64_t o = off[s], m = off[s + 1] - o;
  const int64_t base = o ? pre[o - 1] : 0, total = pre[o + m - 1] - base;
  DiffAt best{std::numeric_limits<int64_t>::max(), need};
  const int64_t lo = need > 1 ? need : 1, hi = (m - need < m - 1) ? m - need : m - 1;
  for (int64_t p = lo + threadIdx.x; p <= hi; p += SPLIT_THREADS) {
    const int64_t v = 2 * (pre[o + p - 1] - base) - total;
    const DiffAt c{v < 0 ? -v : v, (int)p};
    best = FirstMin()(best, c);
  }
  const DiffAt r = BR(tmp).Reduce(best, FirstMin());
  if (threadIdx.x == 0) split[s] = r.diff == std::numeric_limits<int64_t>::max() ? need : r.p;
}
__global__ void k_relabel(const int* __restrict__ seg_sorted, const int* __restrict__ id, const int64_t* __restrict__ off,
                          const int* __restrict__ split, int n, int* __restrict__ seg) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int s = seg_sorted[j];
  seg[id[j]] = 2 * s + (j - off[s] >= split[s] ? 1 : 0);
}

}  // namespace

void lownn_gpu(esg_ctx* ctx, int n, const double* pos_h, const M3& cell, const bool pbc[3], const int32_t* deg,
               int depth, double r_cut, int32_t* part_h) {
  if (depth < 0) usage("partition depth must be non-negative");
  if (depth >= 31 || (1 << depth) > n)
    usage("partition depth " + std::to_string(depth) + " needs at least " + std::to_string(1L << std::min(depth, 30)) +
          " atoms, have " + std::to_string(n));
  if (!(r_cut > 0.0)) usage("cutoff must be positive");
  if (depth == 0) {
    std::fill(part_h, part_h + n, 0);
    return;
  }
  std::vector<int64_t> w(deg, deg + n);
  bool all_zero = true;
  for (int64_t v : w) all_zero = all_zero && v == 0;
  if (all_zero) std::fill(w.begin(), w.end(), 1);

  cudaStream_t st = build_stream(ctx);  // graph-side work: beside an async forward
  auto& C = ctx->cache;
  const int S_max = 1 << (depth - 1);
  auto* pos = static_cast<double*>(C.alloc(sizeof(double) * 3 * (size_t)n));
  auto* wd = static_cast<int64_t*>(C.alloc(sizeof(int64_t) * n));
  auto* wv = static_cast<int64_t*>(C.alloc(sizeof(int64_t) * n));
  auto* pre = static_cast<int64_t*>(C.alloc(sizeof(int64_t) * n));
  auto* seg = static_cast<int*>(C.alloc(sizeof(int) * n));
  auto* seg_a = static_cast<int*>(C.alloc(sizeof(int) * n));
  auto* seg_b = static_cast<int*>(C.alloc(sizeof(int) * n));
  auto* id_a = static_cast<int*>(C.alloc(sizeof(int) * n));
  auto* id_b = static_cast<int*>(C.alloc(sizeof(int) * n));
  auto* key_a = static_cast<uint64_t*>(C.alloc(sizeof(uint64_t) * n));
  auto* key_b = static_cast<uint64_t*>(C.alloc(sizeof(uint64_t) * n));
  auto* ext = static_cast<unsigned long long*>(C.alloc(sizeof(unsigned long long) * 6 * S_max));
  auto* dim_d = static_cast<int*>(C.alloc(sizeof(int) * S_max));
  auto* off_d = static_cast<int64_t*>(C.alloc(sizeof(int64_t) * (S_max + 1)));
  auto* split_d = static_cast<int*>(C.alloc(sizeof(int) * S_max));
  h2d_staged(ctx, pos, pos_h, sizeof(double) * 3 * (size_t)n, st);
  h2d_staged(ctx, wd, w.data(), sizeof(int64_t) * n, st);
  ESG_CUDA(cudaMemsetAsync(seg, 0, sizeof(int) * n, st));

  size_t tmp_bytes = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, key_a, key_b, id_a, id_b, n, 0, 64, st);
  tmp_bytes = std::max(tmp_bytes, b);
  cub::DeviceScan::InclusiveSum(nullptr, b, wv, pre, n, st);
  tmp_bytes = std::max(tmp_bytes, b);
  cub::DeviceRadixSort::SortPairs(nullptr, b, seg_a, seg_b, id_b, id_a, n, 0, 31, st);
  tmp_bytes = std::max(tmp_bytes, b);
  void* tmp = C.alloc(tmp_bytes);

  const unsigned nb = (unsigned)((n + 255) / 256);
  std::vector<int64_t> off{0, n};
  std::vector<std::array<int, 3>> cuts{{0, 0, 0}};
  std::vector<unsigned long long> ext_h;
  for (int level = depth; level >= 1; --level) {
    const int S = (int)cuts.size();
    const bool root = level == depth;
    // 1-2. cut dimension per segment (lownn.cpp:37-60, host.cpp choose_dim)
    ESG_CUDA(cudaMemsetAsync(ext, 0xff, sizeof(unsigned long long) * 3 * S, st));
    ESG_CUDA(cudaMemsetAsync(ext + 3 * S_max, 0, sizeof(unsigned long long) * 3 * S, st));
    k_extent<<<nb, 256, 0, st>>>(pos, seg, n, ext, ext + 3 * S_max);
    ext_h.resize(6 * (size_t)S_max);
    d2h_small(ctx, ext_h.data(), ext, sizeof(unsigned long long) * 6 * S_max, st);
    std::vector<int> dim(S);
    for (int s = 0; s < S; ++s) {
      const auto& c = cuts[s];
      int d0 = -1;
      for (int d = 0; d < 3 && d0 < 0; ++d)
        if (c[d] == 0) d0 = d;
      if (d0 >= 0) {
        dim[s] = d0;
        continue;
      }
      long nn[3];
      for (int d = 0; d < 3; ++d) {
        double e;
        if (root && pbc[d]) {
          e = 0.0;
          for (int j = 0; j < 3; ++j) e += std::abs(cell[j][d]);
        } else {
          e = from_ord(ext_h[3 * (size_t)S_max + 3 * s + d]) - from_ord(ext_h[3 * s + d]);
        }
        if (c[d] == 1 && pbc[d])
          nn[d] = 1;
        else if (e <= 0.0)
          nn[d] = std::numeric_limits<long>::max() / 4;
        else
          nn[d] = (long)std::ceil(2.0 * r_cut / e);
      }
      int best = 0;
      for (int d = 1; d < 3; ++d)
        if (nn[d] <= nn[best]) best = d;
      dim[s] = best;
    }
    h2d_staged(ctx, dim_d, dim.data(), sizeof(int) * S, st);
    // 3. order each segment by (coordinate, atom id) (lownn.cpp:72-76)
    k_sort_keys<<<nb, 256, 0, st>>>(pos, seg, dim_d, n, key_a, id_a);
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key_a, key_b, id_a, id_b, n, 0, 64, st);
    k_gather_seg<<<nb, 256, 0, st>>>(seg, id_b, n, seg_a);
    int seg_bits = 1;
    while ((1 << seg_bits) < S) ++seg_bits;
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, seg_a, seg_b, id_b, id_a, n, 0, seg_bits, st);
    // 4. first minimiser of |2 prefix - total| per segment (lownn.cpp:78-91)
    k_gather_w<<<nb, 256, 0, st>>>(wd, id_a, n, wv);
    cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, wv, pre, n, st);
    h2d_staged(ctx, off_d, off.data(), sizeof(int64_t) * (S + 1), st);
    const int need = 1 << (level - 1);
    k_split<<<S, SPLIT_THREADS, 0, st>>>(pre, off_d, need, split_d);
    std::vector<int> split(S);
    d2h_small(ctx, split.data(), split_d, sizeof(int) * S, st);
    // 5. children 2s (left) and 2s + 1 (right)
    k_relabel<<<nb, 256, 0, st>>>(seg_b, id_a, off_d, split_d, n, seg);
    ctx->launches += 6;
    std::vector<int64_t> off2{0};
    std::vector<std::array<int, 3>> cuts2;
    for (int s = 0; s < S; ++s) {
      auto sub = cuts[s];
      ++sub[dim[s]];
      off2.push_back(off[s] + split[s]);
      off2.push_back(off[s + 1]);
      cuts2.push_back(sub);
      cuts2.push_back(sub);
    }
    off.swap(off2);
    cuts.swap(cuts2);
  }
  d2h_small(ctx, part_h, seg, sizeof(int) * n, st);
  ESG_CUDA(cudaStreamSynchronize(st));
  for (void* p : {(void*)pos, (void*)wd, (void*)wv, (void*)pre, (void*)seg, (void*)seg_a, (void*)seg_b, (void*)id_a,
                  (void*)id_b, (void*)key_a, (void*)key_b, (void*)ext, (void*)dim_d, (void*)off_d, (void*)split_d, tmp})
    C.release(p);
}

}  // namespace esg
