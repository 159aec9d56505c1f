// graph.cu -- cell-list neighbour graph on the GPU, bit-exact with
// structures::build_graph (graph.cpp:55-131).
//
// The reference enumerates, for every real atom i, the ghost images
// (atom j, shift s) whose bin is within one bin of i's bin (bins of width
// r_cut over the ghost cloud, clamped to the grid), keeps d = ghost - r_i with
// |d|^2 <= r_cut^2 (inclusive) except (i, i, 0), and sorts by (dst, src,
// shift).  The candidate relation "bins differ by <= 1 per axis" is
// symmetric, so this kernel walks it destination-major instead: for every
// destination j and image s it scans the real atoms in the 27 bins around the
// ghost's bin.  The candidate set, every fp64 operation (__dadd_rn /
// __dsub_rn / __dmul_rn / __ddiv_rn / __dsqrt_rn in the reference's operand
// order, no FMA) and therefore every kept edge, displacement and distance
// are identical; only the discovery order differs, and a per-destination
// segmented sort on the packed (src, shift) key restores Graph::edges order.
//
// HBM layout produced (dst-major CSR, SoA):
//   d_off[N+1] i64, d_src[E] i32, d_shift[E] u32 packed, d_disp[3E] f64, d_dist[E] f64
#include <cub/cub.cuh>
#include <type_traits>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>

#include "esg_internal.h"

namespace esg {
namespace {

struct Grid {
  double lo[3];
  double width;
  int dims[3];
  double r2;
  int n_img;
  int img_dims[3];  // 2*nimg+1 per axis
  int nimg[3];
  int zero_img;
};

__device__ __forceinline__ int bin_axis(double p, double lo, double w, int dim) {
  int i = (int)floor(__ddiv_rn(__dsub_rn(p, lo), w));
  return min(max(i, 0), dim - 1);
}

__global__ void k_bin_atoms(const double* __restrict__ pos, int n, Grid g, int* __restrict__ bin,
                            int* __restrict__ counts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int bx = bin_axis(pos[3 * i + 0], g.lo[0], g.width, g.dims[0]);
  const int by = bin_axis(pos[3 * i + 1], g.lo[1], g.width, g.dims[1]);
  const int bz = bin_axis(pos[3 * i + 2], g.lo[2], g.width, g.dims[2]);
  const int b = (bx * g.dims[1] + by) * g.dims[2] + bz;
  bin[i] = b;
  atomicAdd(&counts[b], 1);
}

__global__ void k_scatter_atoms(const int* __restrict__ bin, int n, const int* __restrict__ start,
                                int* __restrict__ cursor, int* __restrict__ cell_atoms) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = bin[i];
  cell_atoms[start[b] + atomicAdd(&cursor[b], 1)] = i;
}

// One warp per destination atom j.  FILL=false counts, FILL=true writes the
// packed (src, shift) keys and the dst column in discovery order.
template <bool FILL>
__global__ void k_edges(const double* __restrict__ pos, int n, Grid g, const double* __restrict__ img_off,
                        const int* __restrict__ cell_start, const int* __restrict__ cell_atoms,
                        int64_t* __restrict__ count_or_off, uint64_t* __restrict__ keys,
                        int32_t* __restrict__ dst_col) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  const int j = warp;
  const double pj0 = pos[3 * j], pj1 = pos[3 * j + 1], pj2 = pos[3 * j + 2];
  int64_t base = FILL ? count_or_off[j] : 0;
  int64_t cnt = 0;
  for (int s = 0; s < g.n_img; ++s) {
    const double g0 = __dadd_rn(pj0, img_off[3 * s + 0]);
    const double g1 = __dadd_rn(pj1, img_off[3 * s + 1]);
    const double g2 = __dadd_rn(pj2, img_off[3 * s + 2]);
    const int b0 = bin_axis(g0, g.lo[0], g.width, g.dims[0]);
    const int b1 = bin_axis(g1, g.lo[1], g.width, g.dims[1]);
    const int b2 = bin_axis(g2, g.lo[2], g.width, g.dims[2]);
    const int sx = s / (g.img_dims[1] * g.img_dims[2]) - g.nimg[0];
    const int sy = (s / g.img_dims[2]) % g.img_dims[1] - g.nimg[1];
    const int sz = s % g.img_dims[2] - g.nimg[2];
    const uint32_t packed = (uint32_t(sx + 512) << 20) | (uint32_t(sy + 512) << 10) | uint32_t(sz + 512);
    for (int bx = max(0, b0 - 1); bx <= min(g.dims[0] - 1, b0 + 1); ++bx)
      for (int by = max(0, b1 - 1); by <= min(g.dims[1] - 1, b1 + 1); ++by)
        for (int bz = max(0, b2 - 1); bz <= min(g.dims[2] - 1, b2 + 1); ++bz) {
          const int c = (bx * g.dims[1] + by) * g.dims[2] + bz;
          const int t0 = cell_start[c], t1 = cell_start[c + 1];
          for (int t = t0; t < t1; t += 32) {
            bool keep = false;
            int i = -1;
            if (t + lane < t1) {
              i = cell_atoms[t + lane];
              if (!(i == j && s == g.zero_img)) {
                const double d0 = __dsub_rn(g0, pos[3 * i]);
                const double d1 = __dsub_rn(g1, pos[3 * i + 1]);
                const double d2 = __dsub_rn(g2, pos[3 * i + 2]);
                const double q = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
                keep = !(q > g.r2);
              }
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (FILL && keep) {
              const int64_t at = base + cnt + __popc(m & ((1u << lane) - 1u));
              keys[at] = (uint64_t(uint32_t(i)) << 32) | packed;
              dst_col[at] = j;
            }
            cnt += __popc(m);
          }
        }
  }
  if (!FILL && lane == 0) count_or_off[j] = cnt;
}

__global__ void k_finalize(const uint64_t* __restrict__ keys, const int32_t* __restrict__ dst_col, int64_t E,
                           const double* __restrict__ pos, Grid g, const double* __restrict__ img_off,
                           int32_t* __restrict__ src, uint32_t* __restrict__ shift, double* __restrict__ disp,
                           double* __restrict__ dist) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= E) return;
  const uint64_t key = keys[k];
  const int i = int(key >> 32);
  const uint32_t p = uint32_t(key & 0xffffffffu);
  const int sx = int((p >> 20) & 1023) - 512, sy = int((p >> 10) & 1023) - 512, sz = int(p & 1023) - 512;
  const int s = ((sx + g.nimg[0]) * g.img_dims[1] + (sy + g.nimg[1])) * g.img_dims[2] + (sz + g.nimg[2]);
  const int j = dst_col[k];
  const double d0 = __dsub_rn(__dadd_rn(pos[3 * j], img_off[3 * s]), pos[3 * i]);
  const double d1 = __dsub_rn(__dadd_rn(pos[3 * j + 1], img_off[3 * s + 1]), pos[3 * i + 1]);
  const double d2 = __dsub_rn(__dadd_rn(pos[3 * j + 2], img_off[3 * s + 2]), pos[3 * i + 2]);
  const double q = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
  src[k] = i;
  shift[k] = p;
  disp[3 * k] = d0;
  disp[3 * k + 1] = d1;
  disp[3 * k + 2] = d2;
  dist[k] = __dsqrt_rn(q);
}

// Per-destination sort of the (source, shift) keys: one CTA per segment
// (grid-strided), bitonic over the next power of two in SMEM, padding keys
// ~0 sort last.  Keys are unique within a segment.
constexpr int SEG_SORT_CAP = 4096;
__global__ void __launch_bounds__(256) k_segment_sort(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                      const int64_t* __restrict__ off, int n) {
  __shared__ uint64_t sk[SEG_SORT_CAP];
  for (int j = blockIdx.x; j < n; j += gridDim.x) {
    const int64_t a = off[j];
    const int len = (int)(off[j + 1] - a);
    int P = 1;
    while (P < len) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) sk[i] = i < len ? in[a + i] : ~0ull;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
      for (int h = k >> 1; h > 0; h >>= 1) {
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
          const int o = i ^ h;
          if (o > i) {
            const uint64_t x = sk[i], y = sk[o];
            if ((x > y) == ((i & k) == 0)) {
              sk[i] = y;
              sk[o] = x;
            }
          }
        }
        __syncthreads();
      }
    for (int i = threadIdx.x; i < len; i += blockDim.x) out[a + i] = sk[i];
    __syncthreads();
  }
}

__global__ void k_max_segment(const int64_t* __restrict__ off, int n, unsigned long long* __restrict__ mx) {
  unsigned long long m = 0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)(off[j + 1] - off[j]));
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}

}  // namespace

esg_graph* build_graph_gpu(esg_ctx* ctx, int n, const double* pos_in, const M3& cell, const bool pbc[3],
                           double r_cut) {
  if (!(r_cut > 0.0)) usage("cutoff must be positive");
  if (n < 1) usage("structure has no atoms");
  cudaStream_t st = build_stream(ctx);  // independent of an async forward in flight on ctx->stream
  const bool dbg = std::getenv("ESG_DEBUG_BUILD") != nullptr;
  auto tmark = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!dbg) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[esg build] %-24s %.4f s\n", what, std::chrono::duration<double>(now - tmark).count());
    tmark = now;
  };
  // every device buffer through the context's block cache (esg_internal.h)
  auto dalloc_c = [&](auto* type_tag, size_t n_el) {
    using T = std::remove_pointer_t<decltype(type_tag)>;
    return static_cast<T*>(ctx->cache.alloc(n_el * sizeof(T)));
  };
  std::vector<double> pos(pos_in, pos_in + 3 * (size_t)n);
  wrap_positions(n, pos.data(), cell, pbc);

  Grid g{};
  for (int d = 0; d < 3; ++d) {
    g.nimg[d] = pbc[d] ? (int)std::ceil(r_cut / face_spacing(cell, d)) : 0;
    if (g.nimg[d] > 500) usage("cutoff reaches too many periodic images");
    g.img_dims[d] = 2 * g.nimg[d] + 1;
  }
  g.n_img = g.img_dims[0] * g.img_dims[1] * g.img_dims[2];
  // image offsets (sx*a0 + sy*a1) + sz*a2, image order sx, sy, sz ascending
  std::vector<double> off(3 * (size_t)g.n_img);
  {
    int s = 0;
    for (int sx = -g.nimg[0]; sx <= g.nimg[0]; ++sx)
      for (int sy = -g.nimg[1]; sy <= g.nimg[1]; ++sy)
        for (int sz = -g.nimg[2]; sz <= g.nimg[2]; ++sz, ++s) {
          for (int k = 0; k < 3; ++k) off[3 * s + k] = (sx * cell[0][k] + sy * cell[1][k]) + sz * cell[2][k];
          if (sx == 0 && sy == 0 && sz == 0) g.zero_img = s;
        }
  }
  // Ghost bounding box: rounding is monotone, so min_j fl(p_j + o) = fl(min_j p_j + o).
  double pmin[3], pmax[3];
  for (int d = 0; d < 3; ++d) {
    pmin[d] = std::numeric_limits<double>::max();
    pmax[d] = std::numeric_limits<double>::lowest();
  }
  for (int i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) {
      pmin[d] = std::min(pmin[d], pos[3 * i + d]);
      pmax[d] = std::max(pmax[d], pos[3 * i + d]);
    }
  for (int d = 0; d < 3; ++d) {
    g.lo[d] = std::numeric_limits<double>::max();
    double hi = std::numeric_limits<double>::lowest();
    for (int s = 0; s < g.n_img; ++s) {
      g.lo[d] = std::min(g.lo[d], pmin[d] + off[3 * s + d]);
      hi = std::max(hi, pmax[d] + off[3 * s + d]);
    }
    g.dims[d] = std::max(1, (int)std::floor((hi - g.lo[d]) / r_cut) + 1);
  }
  g.width = r_cut;
  g.r2 = r_cut * r_cut;
  const int64_t nbins = (int64_t)g.dims[0] * g.dims[1] * g.dims[2];
  if (nbins > (int64_t(1) << 27)) usage("bin grid too large for this cutoff / extent");

  auto* G = new esg_graph();
  G->ctx = ctx;
  ctx->graphs.insert(G);
  G->n = n;
  for (int d = 0; d < 3; ++d) G->nimg[d] = g.nimg[d];

  double* d_pos = dalloc_c((double*)nullptr, 3 * (size_t)n);
  double* d_img = dalloc_c((double*)nullptr, off.size());
  int* d_bin = dalloc_c((int*)nullptr, n);
  int* d_cnt = dalloc_c((int*)nullptr, nbins + 1);
  int* d_start = dalloc_c((int*)nullptr, nbins + 1);
  int* d_cur = dalloc_c((int*)nullptr, nbins);
  int* d_atoms = dalloc_c((int*)nullptr, n);
  mark("host prologue");
  h2d_staged(ctx, d_pos, pos.data(), sizeof(double) * 3 * n, st);
  h2d_staged(ctx, d_img, off.data(), sizeof(double) * off.size(), st);
  ESG_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(int) * (nbins + 1), st));
  ESG_CUDA(cudaMemsetAsync(d_cur, 0, sizeof(int) * nbins, st));
  mark("uploads");
  k_bin_atoms<<<(n + 255) / 256, 256, 0, st>>>(d_pos, n, g, d_bin, d_cnt);
  ++ctx->launches;
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_cnt, d_start, (int)(nbins + 1), st);
  void* d_tmp = nullptr;
  d_tmp = ctx->cache.alloc(tmp_bytes);
  cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_cnt, d_start, (int)(nbins + 1), st);
  ctx->cache.release(d_tmp);
  k_scatter_atoms<<<(n + 255) / 256, 256, 0, st>>>(d_bin, n, d_start, d_cur, d_atoms);
  ++ctx->launches;

  int64_t* d_cnt_e = dalloc_c((int64_t*)nullptr, n + 1);
  G->d_off = dalloc_c((int64_t*)nullptr, n + 1);
  ESG_CUDA(cudaMemsetAsync(d_cnt_e, 0, sizeof(int64_t) * (n + 1), st));
  const int threads = 256, warps_per_block = threads / 32;
  const int blocks = (n + warps_per_block - 1) / warps_per_block;
  k_edges<false><<<blocks, threads, 0, st>>>(d_pos, n, g, d_img, d_start, d_atoms, d_cnt_e, nullptr, nullptr);
  ++ctx->launches;
  tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_cnt_e, G->d_off, n + 1, st);
  d_tmp = ctx->cache.alloc(tmp_bytes);
  cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_cnt_e, G->d_off, n + 1, st);
  ctx->cache.release(d_tmp);
  int64_t E = 0;
  mark("count pass");
  d2h_small(ctx, &E, G->d_off + n, sizeof(int64_t), st);
  mark("edge count readback");
  if (E > (int64_t)std::numeric_limits<int>::max() - 1) usage("graph exceeds 2^31 edges");
  G->E = E;

  uint64_t* d_keys = dalloc_c((uint64_t*)nullptr, E);
  uint64_t* d_keys_sorted = dalloc_c((uint64_t*)nullptr, E);
  int32_t* d_dst = dalloc_c((int32_t*)nullptr, E);
  if (E > 0) {
    k_edges<true><<<blocks, threads, 0, st>>>(d_pos, n, g, d_img, d_start, d_atoms, G->d_off, d_keys, d_dst);
    ++ctx->launches;
    tmp_bytes = 0;
    // one CTA per destination segment, no host readback (DeviceSegmentedSort
    // reads its segment-size groups back to the host, which would queue behind
    // in-flight output copies); keys are unique per segment, so the order is
    // the same as any other sort's.  Bits: packed shift (30) + source index.
    unsigned long long* d_mx = dalloc_c((unsigned long long*)nullptr, 1);
    ESG_CUDA(cudaMemsetAsync(d_mx, 0, sizeof(unsigned long long), st));
    k_max_segment<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, st>>>(G->d_off, n, d_mx);
    unsigned long long max_seg = 0;
    d2h_small(ctx, &max_seg, d_mx, sizeof(max_seg), st);
    ctx->cache.release(d_mx);
    int cap = SEG_SORT_CAP;  // ESG_SEG_SORT_CAP=0 forces the cub path (tests)
    if (const char* e = std::getenv("ESG_SEG_SORT_CAP")) cap = std::min(std::max(std::atoi(e), 0), SEG_SORT_CAP);
    if (max_seg <= (unsigned long long)cap) {
      k_segment_sort<<<(unsigned)std::min<int64_t>(n, (int64_t)sm_count() * 8), 256, 0, st>>>(d_keys, d_keys_sorted, G->d_off, n);
      ctx->launches += 2;
    } else {  // very dense graphs: cub's segmented radix sort
      int end_bit = 32;
      while ((int64_t(1) << (end_bit - 32)) < n) ++end_bit;
      cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tmp_bytes, d_keys, d_keys_sorted, (int)E, n, G->d_off,
                                              G->d_off + 1, 0, end_bit, st);
      d_tmp = ctx->cache.alloc(tmp_bytes);
      cub::DeviceSegmentedRadixSort::SortKeys(d_tmp, tmp_bytes, d_keys, d_keys_sorted, (int)E, n, G->d_off,
                                              G->d_off + 1, 0, end_bit, st);
      ctx->cache.release(d_tmp);
    }
  }
  mark("sort");
  G->d_src = dalloc_c((int32_t*)nullptr, E);
  G->d_shift = dalloc_c((uint32_t*)nullptr, E);
  G->d_disp = dalloc_c((double*)nullptr, 3 * (size_t)E);
  G->d_dist = dalloc_c((double*)nullptr, E);
  if (E > 0) {
    k_finalize<<<(unsigned)((E + 255) / 256), 256, 0, st>>>(d_keys_sorted, d_dst, E, d_pos, g, d_img, G->d_src,
                                                           G->d_shift, G->d_disp, G->d_dist);
    ++ctx->launches;
  }
  ESG_CUDA(cudaGetLastError());
  ESG_CUDA(cudaStreamSynchronize(st));
  for (void* p : {(void*)d_pos, (void*)d_img, (void*)d_bin, (void*)d_cnt, (void*)d_start, (void*)d_cur,
                  (void*)d_atoms, (void*)d_cnt_e, (void*)d_keys, (void*)d_keys_sorted, (void*)d_dst})
    ctx->cache.release(p);
  mark("finalize + release");
  return G;
}

namespace {
__global__ void k_copy_words(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
}  // namespace

void h2d_staged(esg_ctx* ctx, void* dev, const void* host, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (!st) st = ctx->stream;
  if (ctx->up_cap < bytes) {
    if (ctx->up) cudaFreeHost(ctx->up);
    ctx->up = nullptr;
    ctx->up_cap = 0;
    ESG_CUDA(cudaHostAlloc(&ctx->up, bytes, cudaHostAllocDefault));
    ctx->up_cap = bytes;
  }
  // every staged copy is synchronous, so the staging buffer is free here
  std::memcpy(ctx->up, host, bytes);
  ESG_CUDA(cudaMemcpyAsync(dev, ctx->up, bytes, cudaMemcpyHostToDevice, st));
  ESG_CUDA(cudaStreamSynchronize(st));
}

void d2h_small(esg_ctx* ctx, void* host, const void* dev, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (!st) st = ctx->stream;
  if (bytes % 4 != 0) usage("d2h_small copies whole 4-byte words");
  if (ctx->zc_cap < bytes) {
    if (ctx->zc) cudaFreeHost(ctx->zc);
    ctx->zc = nullptr;
    ctx->zc_cap = 0;
    ESG_CUDA(cudaHostAlloc(&ctx->zc, bytes, cudaHostAllocMapped));
    ctx->zc_cap = bytes;
  }
  void* dptr = nullptr;
  ESG_CUDA(cudaHostGetDevicePointer(&dptr, ctx->zc, 0));
  const size_t n = bytes / 4;
  k_copy_words<<<(unsigned)std::min<size_t>((n + 255) / 256, 1024), 256, 0, st>>>(
      static_cast<const uint32_t*>(dev), static_cast<uint32_t*>(dptr), n);
  ++ctx->launches;
  ESG_CUDA(cudaGetLastError());
  ESG_CUDA(cudaStreamSynchronize(st));
  std::memcpy(host, ctx->zc, bytes);
}

}  // namespace esg

void esg_graph::host_sync_offsets() const {
  if ((int64_t)h_off.size() == n + 1) return;
  h_off.resize(n + 1);
  esg::d2h_small(ctx, h_off.data(), d_off, sizeof(int64_t) * (n + 1), esg::build_stream(ctx));
}
void esg_graph::host_sync() const {
  host_sync_offsets();
  if ((int64_t)h_src.size() == E) return;
  h_src.resize(E);
  if (E) ESG_CUDA(cudaMemcpy(h_src.data(), d_src, sizeof(int32_t) * E, cudaMemcpyDeviceToHost));
}
