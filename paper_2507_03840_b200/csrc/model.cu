// model.cu -- the eGNN forward on the GPU (network.h:115-164 composition).
//
// Per block (layer x {node, edge}), over destination-aligned edge chunks:
//   k_rotate_in   gather [src | dst | edge] rows, Wigner-D of the edge
//                 direction (recomputed, never stored), rotate into the edge
//                 frame, scatter to the order-major A1 operand     (a8-a10)
//   SO(2) linears lin1 -> gate -> lin2 per order m                  (a11-a12)
//                 fp32 CUDA-core SGEMMs (lin_kernels.cuh) or tcgen05 bf16 (so2_tc.cu)
//   k_rotate_out_edge   rotate back (D^T) and residual-add in place (a13 edge)
//   k_node_update       segment softmax over the dst CSR segment, weighted
//                       sum of rotated-back messages, one store per node
//                       (a13 node; deterministic, partition-invariant order)
// followed by the output heads (a16) and the uncoupled block assembly (a17).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <cmath>
#include <cstring>

#include "esg_internal.h"
#include "model_kernels.cuh"
#include "msg_kernels.cuh"
#include "device_model.h"
#include "lin_kernels.cuh"

namespace esg {

void so2_tc_launch(int L, int E, const uint16_t* A1, int64_t n_e, const uint16_t* W1, const uint16_t* W2,
                   uint16_t* Y, int gate, const float* att, float* logits,
                   cudaStream_t st);  // so2_tc.cu (Y in bf16, node-block logits)
bool so2_tc_available(int L, int E);

namespace {

__device__ __forceinline__ int64_t cmin64(int64_t a, int64_t b) { return a < b ? a : b; }

template <typename T>
T* dalloc(size_t n) {
  T* p = nullptr;
  if (n) ESG_CUDA(cudaMalloc(&p, n * sizeof(T)));
  return p;
}

// Device buffer of at least n elements: the previous one when it is big
// enough (repeated prepares of same-sized views reuse their memory), else a
// fresh allocation.  cap tracks the allocated elements of p.
template <typename T>
T* grow(T* p, size_t& cap, size_t n) {
  if (p && cap >= n) return p;
  if (p) cudaFree(p);
  cap = n;
  return dalloc<T>(n);
}

__device__ __forceinline__ void store_out(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_out(uint16_t* p, float v) {
  // round-to-nearest-even fp32 -> bf16
  uint32_t u = __float_as_uint(v);
  u += 0x7fffu + ((u >> 16) & 1u);
  *p = uint16_t(u >> 16);
}

// -------------------------------------------------------------- init
// ops.h:18-36 embed_nodes, network.h:41-50 radial_features (fp64 exp, cast),
// ops.h:40-63 lift_radial (sequential fp32 sum over Gaussians).
template <int H, int E>
__global__ void k_init_nodes(const int* __restrict__ row_slot, int n_rows, const float* __restrict__ embed,
                             float* __restrict__ nodes) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n_rows * H * E) return;
  const int i = int(t / (H * E)), q = int(t % (H * E));
  nodes[t] = q < E ? embed[row_slot[i] * E + q] : 0.f;
}

// A warp owns blocks of 32 consecutive edges: lane i loads the distance of
// edge i of the block (one coalesced load), then the warp walks the block 4
// edges at a time: lane g evaluates Gaussian g (fp64 exp, cast), lane c < E
// sums lift[c][g] * rbf[g] over g in ascending order (the reference's
// sequential float sum, no FMA; four edges' chains interleave), and the warp
// writes each 1,600-byte row.
template <int H, int E, int NG>
__global__ void __launch_bounds__(256) k_init_edges(const double* __restrict__ dist, int64_t n_e,
                                                    const float* __restrict__ lift, int ng, double spacing,
                                                    float* __restrict__ edges, int full,
                                                    float* __restrict__ emax = nullptr) {
  constexpr int U = 4;
  float vmax = 0.f;
  const int lane = threadIdx.x & 31;
  float w[NG];  // lane c < E keeps lift row c in registers (zero past ng)
#pragma unroll
  for (int g = 0; g < NG; ++g) w[g] = (lane < E && g < ng) ? lift[lane * ng + g] : 0.f;
  const double inv_den = 2.0 * spacing * spacing;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < n_e; base += warps * 32) {
    const int cnt = (int)(n_e - base < 32 ? n_e - base : 32);
    const double myd = lane < cnt ? dist[base + lane] : 0.0;
    for (int e0 = 0; e0 < cnt; e0 += U) {
      float rbf[U], acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double d = __shfl_sync(0xffffffffu, myd, e0 + u) - lane * spacing;
        rbf[u] = lane < ng ? (float)exp(-d * d / inv_den) : 0.f;
        acc[u] = 0.f;
      }
#pragma unroll
      for (int g = 0; g < NG; ++g)
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = __fadd_rn(acc[u], __fmul_rn(w[g], __shfl_sync(0xffffffffu, rbf[u], g)));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (e0 + u >= cnt) break;
        const int64_t k = base + e0 + u;
        float4* row = reinterpret_cast<float4*>(edges + k * (H * E));
        if (full)  // otherwise layer 0 treats the l > 0 planes as zero without reading them
          for (int q = E / 4 + lane; q < H * E / 4; q += 32) row[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (lane < E) {
          edges[k * (H * E) + lane] = acc[u];
          vmax = fmaxf(vmax, fabsf(acc[u]));
        }
      }
    }
  }
  if (emax) {  // max |edge row| (the fp16x3 chain's scale bound of layer 0)
    vmax = warp_max(vmax);
    if (lane == 0) atomic_max_abs(emax, vmax);
  }
}

// ------------------------------------------------- SO(2) linears, fp32
// The CUDA-core path runs kernels.h:133-161 (lin1 3E->2E), :210-226 (gate)
// and lin2 2E->E as per-order SGEMMs with the expanded weight
// [[Wr, Wi], [-Wi, Wr]] (lin_kernels.cuh k_gemm_m, k_gate_fwd), so
// ym = Wr xm + Wi xp and yp = Wr xp - Wi xm come out of one product.

__global__ void k_copy_rows(const float* __restrict__ src, float* __restrict__ dst, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}

// ---------------------------------------------------------- heads
// ops.h:287-335: out[i][off_k + r] = sum_c w_k[c] x[i][L^2 + r][c].
// Persistent CTAs stream tiles of HT items (H x E rows each) into a 2-stage
// shared-memory ring with cp.async (the next tile loads while this one is
// computed); thread j (one per head output) computes output j of every item
// of the tile with its key's weight row in registers, stores coalesced along
// j.  Sequential fp32 sum over the channels without FMA, as ops.h:293-306.
constexpr int HT = 16;  // items per tile
template <int H, int E>
constexpr int heads_smem_bytes() {
  return 2 * HT * H * (E + 4) * (int)sizeof(float);
}
template <int H, int E>
__global__ void __launch_bounds__(256) k_heads(const float* __restrict__ x, int64_t n_items,
                                               const float* __restrict__ W, const int* __restrict__ key_of,
                                               const int* __restrict__ row_of, int out_len, float* __restrict__ out) {
  constexpr int PS = E + 4;        // plane stride padded: distinct rows hit distinct banks
  constexpr int STAGE = HT * H * PS;
  constexpr int U = H * E / 4;     // 16-byte units per item
  extern __shared__ __align__(16) float sx[];  // 2 x HT x H x PS
  const int j = threadIdx.x;
  float w[E];
  int row = 0;
  if (j < out_len) {
    row = row_of[j];
    const int k = key_of[j];
#pragma unroll
    for (int c = 0; c < E; ++c) w[c] = W[k * E + c];
  }
  const int64_t n_tiles = (n_items + HT - 1) / HT;
  auto issue = [&](int64_t tile, int stage) {
    if (tile < n_tiles) {
      const int64_t i0 = tile * HT;
      const int ni = (int)(n_items - i0 < HT ? n_items - i0 : HT);
      const float* src = x + i0 * (H * E);
      float* dst = sx + stage * STAGE;
      for (int u = threadIdx.x; u < ni * U; u += blockDim.x) {
        const int pl = u / (E / 4), w4 = u % (E / 4);  // plane (item, row), 16 bytes within it
        cp_async16(dst + pl * PS + 4 * w4, src + 4 * u);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  int stage = 0;
  issue(blockIdx.x, 0);
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, stage ^= 1) {
    issue(tile + gridDim.x, stage ^ 1);  // next tile streams in meanwhile
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncthreads();
    const int64_t i0 = tile * HT;
    const int ni = (int)(n_items - i0 < HT ? n_items - i0 : HT);
    if (j < out_len) {
      const float* base = sx + stage * STAGE + row * PS;
#pragma unroll 4
      for (int it = 0; it < ni; ++it) {
        const float4* plane = reinterpret_cast<const float4*>(base + it * H * PS);
        float acc = 0.f;
#pragma unroll
        for (int c4 = 0; c4 < E / 4; ++c4) {
          const float4 v = plane[c4];
          acc = __fadd_rn(acc, __fmul_rn(w[4 * c4], v.x));
          acc = __fadd_rn(acc, __fmul_rn(w[4 * c4 + 1], v.y));
          acc = __fadd_rn(acc, __fmul_rn(w[4 * c4 + 2], v.z));
          acc = __fadd_rn(acc, __fmul_rn(w[4 * c4 + 3], v.w));
        }
        out[(i0 + it) * out_len + j] = acc;
      }
    }
    __syncthreads();  // this stage is refilled two tiles later
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

__global__ void k_pack_rows(const float* __restrict__ nodes, const int* __restrict__ rows, int64_t n_rows, int row_len,
                            float* __restrict__ buf) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_rows * row_len) return;
  const int64_t r = t / row_len;
  buf[t] = nodes[(int64_t)rows[r] * row_len + (t % row_len)];
}

__global__ void k_gather_dirs(const double* __restrict__ disp, const int* __restrict__ eidx, int64_t n,
                              float* __restrict__ dir, double* __restrict__ dist_in, double* __restrict__ dist_out,
                              const uint32_t* __restrict__ shift_in, uint32_t* __restrict__ shift_out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t g = eidx ? eidx[k] : k;
  dir[3 * k] = (float)disp[3 * g];
  dir[3 * k + 1] = (float)disp[3 * g + 1];
  dir[3 * k + 2] = (float)disp[3 * g + 2];
  dist_out[k] = dist_in[g];
  shift_out[k] = shift_in[g];
}

}  // namespace

// ------------------------------------------------------- weight packing
// One order block of one SO(2) linear from the flat parameters
// (network.h:266-276 names): the expanded matrix W (N x K; m = 0: W0,
// m >= 1: [[Wr, Wi], [-Wi, Wr]]) written as
//   t  -- transposed (K x N), the CUDA-core forward operand,
//   w  -- row-major (N x K), the training dx operand (W^T g),
//   b  -- bf16 tcgen05 B image: per 64-wide K chunk N rows x 128 B, 16-byte
//         units swizzled by row % 8 (SWIZZLE_128B, K-major), K padded to 64.
__global__ void k_pack_lin(const float* __restrict__ params, int64_t off_a, int64_t off_b, int m, int R, int C,
                           float* __restrict__ t, float* __restrict__ w, uint16_t* __restrict__ b) {
  const int N = m == 0 ? R : 2 * R, K = m == 0 ? C : 2 * C, KP = (K + 63) / 64 * 64;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  auto W = [&](int n, int k) -> float {
    if (m == 0) return params[off_a + (int64_t)n * C + k];
    const bool lo_n = n < R, lo_k = k < C;
    const int nn = lo_n ? n : n - R, kk = lo_k ? k : k - C;
    const float wr = params[off_a + (int64_t)nn * C + kk], wi = params[off_b + (int64_t)nn * C + kk];
    return lo_n ? (lo_k ? wr : wi) : (lo_k ? -wi : wr);
  };
  if (i < (int64_t)N * K) {
    const int n = (int)(i / K), k = (int)(i % K);
    const float v = W(n, k);
    w[i] = v;
    t[(int64_t)k * N + n] = v;
  }
  if (i < (int64_t)KP * N) {  // bf16 image: (chunk, row, unit, lane) in storage order
    const int kc = (int)(i / (64 * N)), rem = (int)(i % (64 * N)), n = rem / 64, u = (rem % 64) / 8, tl = rem % 8;
    const int k = kc * 64 + ((u ^ (n & 7)) * 8) + tl;
    float v = k < K ? W(n, k) : 0.f;
    uint32_t bits = __float_as_uint(v);
    bits += 0x7fffu + ((bits >> 16) & 1u);
    b[i] = k < K ? uint16_t(bits >> 16) : 0;
  }
}

// =================================================================== host
void free_ptr(void* p) {
  if (p) cudaFree(p);
}


namespace {

// Brackets one kernel launch with CUDA events on the launching stream when
// profiling is on; the elapsed times are summed per category after the
// forward's final synchronisation.
struct Prof {
  DeviceModel* D;
  cudaStream_t st;
  int cat, idx = -1;
  Prof(DeviceModel* d, cudaStream_t s, int c) : D(d), st(s), cat(c) {
    if (!D->profile) return;
    const size_t need = 2 * (D->marks.size() + 1);
    while (D->pool.size() < need) {
      cudaEvent_t e;
      ESG_CUDA(cudaEventCreate(&e));
      D->pool.push_back(e);
    }
    idx = (int)(2 * D->marks.size());
    D->marks.push_back({cat, idx});
    ESG_CUDA(cudaEventRecord(D->pool[idx], st));
  }
  ~Prof() {
    if (idx >= 0) cudaEventRecord(D->pool[idx + 1], st);
  }
};

void prof_collect(DeviceModel* D) {
  if (!D->profile) return;
  for (const auto& mk : D->marks) {
    float ms = 0.f;
    ESG_CUDA(cudaEventElapsedTime(&ms, D->pool[mk.second], D->pool[mk.second + 1]));
    D->prof_ms[mk.first] += ms;
    D->prof_n[mk.first] += 1;
  }
  D->marks.clear();
}




bool supported(int L, int E) { return (L == 4 || L == 2) && (E == 16 || E == 8); }


uint16_t to_bf16(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

}  // namespace

// Expanded SO(2) weight of order m in (N x K) row-major form:
// m = 0: W0 ; m >= 1: [[Wr, Wi], [-Wi, Wr]].
std::vector<float> expanded(const esg_model* M, const std::string& base, int m, int cin, int cout) {
  const int nd = M->lay.nd(m);
  if (m == 0) {
    const auto& e = M->params.at(base + "/m0");
    return std::vector<float>(M->host_params.begin() + e.offset,
                              M->host_params.begin() + e.offset + (int64_t)e.rows * e.cols);
  }
  const auto& er = M->params.at(base + "/m" + std::to_string(m) + "r");
  const auto& ei = M->params.at(base + "/m" + std::to_string(m) + "i");
  const int R = nd * cout, C = nd * cin;
  std::vector<float> W((size_t)4 * R * C);
  const float* wr = M->host_params.data() + er.offset;
  const float* wi = M->host_params.data() + ei.offset;
  for (int o = 0; o < R; ++o)
    for (int k = 0; k < C; ++k) {
      W[(size_t)o * 2 * C + k] = wr[o * C + k];
      W[(size_t)o * 2 * C + C + k] = wi[o * C + k];
      W[(size_t)(R + o) * 2 * C + k] = -wi[o * C + k];
      W[(size_t)(R + o) * 2 * C + C + k] = wr[o * C + k];
    }
  return W;
}

namespace {
// Power-of-two scale of a split operand bounded by `bound` (host twin of
// f16s_pow2_scale): every |x| / s < 2^14.
float pow2_scale_host(double bound) {
  if (!(bound > 0.0) || !std::isfinite(bound)) return 1.f;
  int k;
  std::frexp((float)bound, &k);
  return std::ldexp(1.f, k - 14);
}
uint16_t f16_bits(float x) {
  const __half h = __float2half_rn(x);
  uint16_t u;
  std::memcpy(&u, &h, 2);
  return u;
}
// The fp16x3 split image of one expanded order block W (N x K row-major):
// per 32-wide K chunk N rows of 128 bytes, [hi(32) | lo(32)] fp16 of W / s,
// 16-byte units XOR-swizzled by row % 8 (so2_f16x3.cu).  Returns s and
// ||W||_inf (max row sum of |w|, rounded up).
void pack_f16x3_block(const std::vector<float>& W, int N, int K, std::vector<uint8_t>& img, float* scale,
                      float* inf_norm) {
  double mx = 0.0, inf = 0.0;
  for (int n = 0; n < N; ++n) {
    double rs = 0.0;
    for (int k = 0; k < K; ++k) {
      const double a = std::fabs((double)W[(size_t)n * K + k]);
      mx = std::max(mx, a);
      rs += a;
    }
    inf = std::max(inf, rs);
  }
  const float s = pow2_scale_host(mx), inv = 1.f / s;
  *scale = s;
  *inf_norm = std::nextafter((float)inf, INFINITY);
  const int KP = (K + 31) / 32 * 32;
  const size_t base = img.size();
  img.resize(base + (size_t)N * KP * 4, 0);
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) {
      const float x = W[(size_t)n * K + k] * inv;
      const uint16_t hb = f16_bits(x);
      __half hh;
      std::memcpy(&hh, &hb, 2);
      const uint16_t lb = f16_bits(x - __half2float(hh));
      const int c = k >> 5, w = k & 31, u = w >> 3;
      const size_t row = base + (size_t)c * N * 128 + (size_t)n * 128 + (w & 7) * 2;
      std::memcpy(&img[row + (((u) ^ (n & 7)) << 4)], &hb, 2);
      std::memcpy(&img[row + (((4 + u) ^ (n & 7)) << 4)], &lb, 2);
    }
}
}  // namespace

// The fp16x3 split images of every block, packed on the host from the host
// parameters; run before the first fp16x3 forward after a parameter change
// (model_upload_params marks them stale), so training steps never pay it.
void pack_f16x3_images(esg_model* M) {
  DeviceModel* D = M->dev;
  if (D->w1f.empty() || !D->f16_stale) return;
  cudaStream_t st = M->ctx->stream;
  const int L = M->cfg.l_max, E = M->cfg.e_width, nb = 2 * M->cfg.layers;
  D->f16sc.resize(nb);
  for (int b = 0; b < nb; ++b) {
    const std::string base = "layer" + std::to_string(b / 2) + (b % 2 == 0 ? "/node" : "/edge");
    F16x3Scales& sc = D->f16sc[b];
    for (int li = 0; li < 2; ++li) {
      const int cin = li == 0 ? 3 * E : 2 * E, cout = li == 0 ? 2 * E : E;
      const std::string wb = base + (li == 0 ? "/lin1" : "/lin2");
      std::vector<uint8_t> img;
      for (int m = 0; m <= L; ++m) {
        const int rows = m == 0 ? M->lay.nd(0) : 2 * M->lay.nd(m);
        float sw = 1.f, inf = 0.f;
        pack_f16x3_block(expanded(M, wb, m, cin, cout), rows * cout, rows * cin, img, &sw, &inf);
        (li == 0 ? sc.w1 : sc.w2)[m] = sw;
        if (li == 0) sc.w1inf[m] = inf;
      }
      const int64_t want = li == 0 ? so2_f16x3_w1_bytes(L, E) : so2_f16x3_w2_bytes(L, E);
      if ((int64_t)img.size() != want) usage("fp16x3 weight image size mismatch");
      ESG_CUDA(cudaMemcpyAsync(li == 0 ? D->w1f[b] : D->w2f[b], img.data(), img.size(), cudaMemcpyHostToDevice, st));
      ESG_CUDA(cudaStreamSynchronize(st));  // img is freed at scope exit
    }
  }
  D->f16_stale = false;
}

void model_repack_params(esg_model* M);

void model_upload_params(esg_model* M) {
  DeviceModel* D = M->dev;
  cudaStream_t st = M->ctx->stream;
  const int L = M->cfg.l_max, E = M->cfg.e_width;
  const int nb = 2 * M->cfg.layers;
  auto pad64 = [](int x) { return (x + 63) / 64 * 64; };
  // sizes of every block's packs (fixed per model): allocated once, reused
  auto lin_sizes = [&](int cin, int cout, size_t& dense, size_t& bf) {
    dense = bf = 0;
    for (int m = 0; m <= L; ++m) {
      const int rows = m == 0 ? M->lay.nd(0) : 2 * M->lay.nd(m), K = rows * cin, N = rows * cout;
      dense += (size_t)K * N;
      bf += (size_t)pad64(K) * N;
    }
  };
  size_t d1, bf1, d2, bf2;
  lin_sizes(3 * E, 2 * E, d1, bf1);
  lin_sizes(2 * E, E, d2, bf2);
  if (!D->weights_allocated) {
    D->params = dalloc<float>(M->host_params.size());
    for (auto* v : {&D->w1t, &D->w2t, &D->w1n, &D->w2n}) v->assign(nb, nullptr);
    D->w1b.assign(nb, nullptr);
    D->w2b.assign(nb, nullptr);
    for (int b = 0; b < nb; ++b) {
      D->w1t[b] = dalloc<float>(d1);
      D->w1n[b] = dalloc<float>(d1);
      D->w2t[b] = dalloc<float>(d2);
      D->w2n[b] = dalloc<float>(d2);
      D->w1b[b] = dalloc<uint16_t>(bf1);
      D->w2b[b] = dalloc<uint16_t>(bf2);
    }
    if (so2_f16x3_available(L, E)) {
      D->w1f.assign(nb, nullptr);
      D->w2f.assign(nb, nullptr);
      for (int b = 0; b < nb; ++b) {
        D->w1f[b] = dalloc<uint8_t>(so2_f16x3_w1_bytes(L, E));
        D->w2f[b] = dalloc<uint8_t>(so2_f16x3_w2_bytes(L, E));
      }
    }
    D->tmax = dalloc<float>(16);
    D->embed = dalloc<float>(M->species_list.size() * E);
    D->head_w[0] = dalloc<float>(M->heads.keys.size() * E);
    D->head_w[1] = dalloc<float>(M->heads.keys.size() * E);
    D->head_key = dalloc<int>(M->heads.out_len);
    D->head_row = dalloc<int>(M->heads.out_len);
    // tile lists of the CUDA-core SGEMM per linear kind (lin_kernels.cuh)
    const int cin_of[4] = {3 * E, 2 * E, E, 2 * E}, cout_of[4] = {2 * E, E, 2 * E, 3 * E};
    for (int kind = 0; kind < 4; ++kind) {
      std::vector<LinTile> v;
      int64_t off = 0;
      for (int m = 0; m <= L; ++m) {
        const int rows = m == 0 ? M->lay.nd(0) : 2 * M->lay.nd(m), K = rows * cin_of[kind],
                  N = rows * cout_of[kind];
        for (int o0 = 0; o0 < N; o0 += 64) v.push_back({m, o0, K, N, off});
        off += (int64_t)K * N;
      }
      D->lt[kind] = dalloc<LinTile>(v.size());
      ESG_CUDA(cudaMemcpy(D->lt[kind], v.data(), sizeof(LinTile) * v.size(), cudaMemcpyHostToDevice));
      D->n_lt[kind] = (int)v.size();
      std::vector<TcTile> tt;
      const int64_t img = tf32_tiles(L, E, kind, &tt);
      D->tct[kind] = dalloc<TcTile>(tt.size());
      ESG_CUDA(cudaMemcpy(D->tct[kind], tt.data(), sizeof(TcTile) * tt.size(), cudaMemcpyHostToDevice));
      D->n_tct[kind] = (int)tt.size();
      for (int b = 0; b < 2 * M->cfg.layers; ++b) D->wtc[kind].push_back(dalloc<uint8_t>(img));
    }
    D->weights_allocated = true;
  }
  ESG_CUDA(cudaMemcpyAsync(D->params, M->host_params.data(), sizeof(float) * M->host_params.size(),
                           cudaMemcpyHostToDevice, st));
  model_repack_params(M);
}

// Every packed image of the linears (tf32 / bf16 / SIMT forms) and the
// embedding / head tables from the device parameters D->params (after an
// upload or a device optimizer step); the fp16x3 images are repacked lazily.
void model_repack_params(esg_model* M) {
  DeviceModel* D = M->dev;
  cudaStream_t st = M->ctx->stream;
  const int L = M->cfg.l_max, E = M->cfg.e_width;
  auto pad64 = [](int x) { return (x + 63) / 64 * 64; };
  // every linear's three images from the device parameters
  D->att_off.clear();
  for (int layer = 0; layer < M->cfg.layers; ++layer) {
    for (int bi = 0; bi < 2; ++bi) {
      const int b = 2 * layer + bi;
      const std::string base = "layer" + std::to_string(layer) + (bi == 0 ? "/node" : "/edge");
      for (int li = 0; li < 2; ++li) {
        const int cin = li == 0 ? 3 * E : 2 * E, cout = li == 0 ? 2 * E : E;
        const std::string wb = base + (li == 0 ? "/lin1" : "/lin2");
        size_t dense = 0, bf = 0;
        for (int m = 0; m <= L; ++m) {
          const int nd = M->lay.nd(m), R = nd * cout, C = nd * cin;
          const int N = m == 0 ? R : 2 * R, K = m == 0 ? C : 2 * C;
          const int64_t oa = M->params.at(m == 0 ? wb + "/m0" : wb + "/m" + std::to_string(m) + "r").offset;
          const int64_t ob = m == 0 ? oa : M->params.at(wb + "/m" + std::to_string(m) + "i").offset;
          const int64_t work = std::max<int64_t>((int64_t)N * K, (int64_t)pad64(K) * N);
          k_pack_lin<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(
              D->params, oa, ob, m, R, C, (li == 0 ? D->w1t[b] : D->w2t[b]) + dense,
              (li == 0 ? D->w1n[b] : D->w2n[b]) + dense, (li == 0 ? D->w1b[b] : D->w2b[b]) + bf);
          dense += (size_t)N * K;
          bf += (size_t)pad64(K) * N;
        }
        // tf32 hi/lo images, forward and transposed (dx)
        std::vector<int64_t> oa(L + 1), ob(L + 1);
        for (int m = 0; m <= L; ++m) {
          oa[m] = M->params.at(m == 0 ? wb + "/m0" : wb + "/m" + std::to_string(m) + "r").offset;
          ob[m] = m == 0 ? oa[m] : M->params.at(wb + "/m" + std::to_string(m) + "i").offset;
        }
        tf32_pack(D->params, L, E, li, false, oa.data(), ob.data(), D->wtc[li == 0 ? 0 : 1][b], st);
        tf32_pack(D->params, L, E, li, true, oa.data(), ob.data(), D->wtc[li == 0 ? 3 : 2][b], st);
      }
    }
    D->att_off.push_back(M->params.at("layer" + std::to_string(layer) + "/att").offset);
  }
  ESG_CUDA(cudaGetLastError());
  // embeddings per species slot (ascending Z), lift, heads
  std::vector<float> emb;
  for (int z : M->species_list) {
    const auto& e = M->params.at("embed/" + element_symbol(z));
    emb.insert(emb.end(), M->host_params.begin() + e.offset, M->host_params.begin() + e.offset + E);
  }
  ESG_CUDA(cudaMemcpyAsync(D->embed, emb.data(), sizeof(float) * emb.size(), cudaMemcpyHostToDevice, st));
  D->lift_off = M->params.at("radial/lift").offset;
  // per head output j: its key and the harmonic row it projects (k_heads)
  std::vector<int> key_of, row_of;
  for (size_t k = 0; k < M->heads.keys.size(); ++k) {
    const int Lk = M->heads.keys[k].L;
    for (int r = 0; r < 2 * Lk + 1; ++r) {
      key_of.push_back((int)k);
      row_of.push_back(Lk * Lk + r);
    }
  }
  std::vector<float> hw[2];
  for (int s = 0; s < 2; ++s) {
    for (const auto& k : M->heads.keys) {
      const auto& e = M->params.at(std::string("head/") + (s == 0 ? "node" : "edge") + "/s" + std::to_string(k.sa) +
                                   "s" + std::to_string(k.sb) + "L" + std::to_string(k.L));
      hw[s].insert(hw[s].end(), M->host_params.begin() + e.offset, M->host_params.begin() + e.offset + E);
    }
    ESG_CUDA(cudaMemcpyAsync(D->head_w[s], hw[s].data(), sizeof(float) * hw[s].size(), cudaMemcpyHostToDevice, st));
  }
  ESG_CUDA(cudaMemcpyAsync(D->head_key, key_of.data(), sizeof(int) * key_of.size(), cudaMemcpyHostToDevice, st));
  ESG_CUDA(cudaMemcpyAsync(D->head_row, row_of.data(), sizeof(int) * row_of.size(), cudaMemcpyHostToDevice, st));
  ESG_CUDA(cudaStreamSynchronize(st));  // the host staging vectors go out of scope
  D->f16_stale = true;  // pack_f16x3_images before the next fp16x3 forward
}

void model_device_create(esg_model* M) {
  const int L = M->cfg.l_max, E = M->cfg.e_width;
  if (!supported(L, E))
    usage("the B200 kernels are instantiated for l_max in {2,4} and e_width in {8,16}; got l_max " +
          std::to_string(L) + ", e_width " + std::to_string(E));
  M->dev = new DeviceModel();
  if (const char* pf = std::getenv("ESG_PREFETCH")) M->dev->prefetch = std::atoi(pf);
  if (const char* tf = std::getenv("ESG_TF32")) M->dev->tf32 = std::atoi(tf) != 0;
  if (const char* f3 = std::getenv("ESG_F16X3")) M->dev->f16x3 = std::atoi(f3) != 0;
  M->dev->L = L;
  M->dev->E = E;
  M->dev->H = (L + 1) * (L + 1);
  M->dev->precision = M->cfg.linear_precision;
  ESG_CUDA(cudaSetDevice(M->ctx->device));
  for (auto& e : M->dev->ev) ESG_CUDA(cudaEventCreate(&e));
}

void train_free(DeviceModel* D);  // train.cu

void model_device_destroy(esg_model* M) {
  DeviceModel* D = M->dev;
  if (!D) return;
  train_free(D);
  blocks_free(D);
  for (void* p : {(void*)D->params, (void*)D->embed, (void*)D->head_w[0], (void*)D->head_w[1], (void*)D->head_key,
                  (void*)D->head_row, (void*)D->head_hptr, (void*)D->row_slot, (void*)D->src_row, (void*)D->dst_row, (void*)D->dir,
                  (void*)D->dist, (void*)D->seg, (void*)D->send_rows, (void*)D->send_buf, (void*)D->nodes,
                  (void*)D->nodes_alt, (void*)D->edges, D->A1, (void*)D->Y, (void*)D->logits, (void*)D->node_out,
                  (void*)D->edge_out, (void*)D->row_global, (void*)D->eshift})
    free_ptr(p);
  for (auto p : D->w1t) free_ptr(p);
  for (auto p : D->w2t) free_ptr(p);
  for (auto p : D->w1n) free_ptr(p);
  for (int k = 0; k < 4; ++k) {
    free_ptr(D->lt[k]);
    free_ptr(D->tct[k]);
    for (auto p : D->wtc[k]) free_ptr(p);
  }
  free_ptr(D->Hbuf);
  for (auto p : D->w2n) free_ptr(p);
  for (auto p : D->w1b) free_ptr(p);
  for (auto p : D->w2b) free_ptr(p);
  for (auto p : D->w1f) free_ptr(p);
  for (auto p : D->w2f) free_ptr(p);
  free_ptr(D->tmax);
  for (auto& e : D->ev) cudaEventDestroy(e);
  for (auto& e : D->halo_ev) cudaEventDestroy(e);
  if (D->copies_pending) cudaEventSynchronize(D->copies_done);
  if (D->copies_done) cudaEventDestroy(D->copies_done);
  for (auto& e : D->out_ev) cudaEventDestroy(e);
  if (D->copy_st) cudaStreamDestroy(D->copy_st);
  delete D;
  M->dev = nullptr;
}

// Network::prepare on a rank view (comm_plan.cpp layout; plan == nullptr is
// the serial view of the whole graph).
// k_fill_dst: dst_row[k] = j for the edges of destination segment j
__global__ void k_fill_dst(const int64_t* __restrict__ off, int n, int* __restrict__ dst_row) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= n) return;
  for (int64_t k = off[j] + (threadIdx.x & 31); k < off[j + 1]; k += 32) dst_row[k] = j;
}

void model_outputs_wait(esg_model* M);

void model_prepare(esg_model* M, const esg_graph* g, const esg_plan* plan, const int32_t* species) {
  DeviceModel* D = M->dev;
  cudaStream_t st = M->ctx->stream;
  const int E = D->E, H = D->H;
  int n_rows, n_owned;
  int64_t ne;
  std::vector<int32_t> row_global;
  std::vector<int64_t> seg;
  if (plan) {
    n_rows = plan->n_rows;
    n_owned = plan->n_owned;
    row_global = plan->row_global;
    ne = plan->n_edges;
    seg.assign(n_owned + 1, 0);
    if (plan->d_seg) {  // GPU-built plan: the segment offsets are on the device
      d2h_small(M->ctx, seg.data(), plan->d_seg, sizeof(int64_t) * (n_owned + 1));
    } else {
      for (int64_t k = 0; k < ne; ++k) seg[plan->dst_row[k] + 1]++;
      for (int j = 0; j < n_owned; ++j) seg[j + 1] += seg[j];
    }
  } else {
    // the whole graph as the view: indices stay on the device (CSR src, the
    // segment offsets are the CSR offsets); only the offsets come to the host
    n_rows = n_owned = g->n;
    ne = g->E;
    row_global.resize(g->n);
    for (int i = 0; i < g->n; ++i) row_global[i] = i;
    seg.resize(g->n + 1);
    d2h_small(M->ctx, seg.data(), g->d_off, sizeof(int64_t) * (g->n + 1));
  }
  std::vector<int> slot(n_rows);
  D->row_species.resize(n_rows);
  for (int i = 0; i < n_rows; ++i) {
    const int z = species[row_global[i]];
    D->row_species[i] = z;
    auto it = std::find(M->species_list.begin(), M->species_list.end(), z);
    if (it == M->species_list.end()) data("species " + element_symbol(z) + " missing from the model's basis");
    slot[i] = int(it - M->species_list.begin());
  }
  D->n_rows = n_rows;
  D->n_owned = n_owned;
  D->n_edges = ne;
  D->h_seg = seg;
  D->blk_ready = false;
  D->row_slot = grow(D->row_slot, D->cap_row_slot, n_rows);
  D->src_row = grow(D->src_row, D->cap_src, ne);
  D->dst_row = grow(D->dst_row, D->cap_dst, ne);
  D->dir = grow(D->dir, D->cap_dir, 3 * ne);
  D->dist = grow(D->dist, D->cap_dist, ne);
  D->seg = grow(D->seg, D->cap_seg, n_owned + 1);
  D->eshift = grow(D->eshift, D->cap_eshift, ne);
  D->row_global = grow(D->row_global, D->cap_row_global, n_rows);
  h2d_staged(M->ctx, D->row_slot, slot.data(), sizeof(int) * n_rows);
  h2d_staged(M->ctx, D->row_global, row_global.data(), sizeof(int) * n_rows);
  int* d_eidx = nullptr;
  if (plan && plan->d_src_row) {
    if (ne) {
      ESG_CUDA(cudaMemcpyAsync(D->src_row, plan->d_src_row, sizeof(int) * ne, cudaMemcpyDeviceToDevice, st));
      ESG_CUDA(cudaMemcpyAsync(D->dst_row, plan->d_dst_row, sizeof(int) * ne, cudaMemcpyDeviceToDevice, st));
    }
    ESG_CUDA(cudaMemcpyAsync(D->seg, plan->d_seg, sizeof(int64_t) * (n_owned + 1), cudaMemcpyDeviceToDevice, st));
    d_eidx = plan->d_edge_index;  // read by k_gather_dirs below, owned by the plan
  } else if (plan) {
    h2d_staged(M->ctx, D->src_row, plan->src_row.data(), sizeof(int) * ne);
    h2d_staged(M->ctx, D->dst_row, plan->dst_row.data(), sizeof(int) * ne);
    h2d_staged(M->ctx, D->seg, seg.data(), sizeof(int64_t) * (n_owned + 1));
    d_eidx = dalloc<int>(ne);
    h2d_staged(M->ctx, d_eidx, plan->edge_index.data(), sizeof(int) * ne);
  } else {
    if (ne) ESG_CUDA(cudaMemcpyAsync(D->src_row, g->d_src, sizeof(int) * ne, cudaMemcpyDeviceToDevice, st));
    ESG_CUDA(cudaMemcpyAsync(D->seg, g->d_off, sizeof(int64_t) * (n_owned + 1), cudaMemcpyDeviceToDevice, st));
    if (n_owned) {
      k_fill_dst<<<(unsigned)((n_owned + 7) / 8), 256, 0, st>>>(D->seg, n_owned, D->dst_row);
      ++M->ctx->launches;
    }
  }
  if (ne) {
    k_gather_dirs<<<(unsigned)((ne + 255) / 256), 256, 0, st>>>(g->d_disp, d_eidx, ne, D->dir, g->d_dist, D->dist,
                                                                g->d_shift, D->eshift);
    ++M->ctx->launches;
  }
  // destination-aligned chunks of about chunk_cap edges
  int64_t chunk_edges = 2 << 20;  // ESG_CHUNK_EDGES overrides (experiments)
  if (const char* ce = std::getenv("ESG_CHUNK_EDGES")) chunk_edges = std::max<int64_t>(std::atoll(ce), 1024);
  const int64_t cap = std::max<int64_t>(std::min<int64_t>(ne, chunk_edges), 1);
  int64_t maxseg = 0;
  for (int j = 0; j < n_owned; ++j) maxseg = std::max(maxseg, seg[j + 1] - seg[j]);
  D->chunk_cap = std::max(cap, maxseg);
  D->chunks.clear();
  for (int j = 0; j < n_owned;) {
    int j1 = j;
    while (j1 < n_owned && (j1 == j || seg[j1 + 1] - seg[j] <= D->chunk_cap)) ++j1;
    D->chunks.push_back({j, j1});
    j = j1;
  }
  // tables and scratch
  const int64_t row = (int64_t)H * E;
  D->nodes = grow(D->nodes, D->cap_nodes, (size_t)n_rows * row);
  D->nodes_alt = grow(D->nodes_alt, D->cap_nodes_alt, (size_t)n_rows * row);
  D->edges = grow(D->edges, D->cap_edges, (size_t)std::max<int64_t>(ne, 1) * row);
  const int K1T = [&] {
    int t = 0;
    for (int m = 0; m <= D->L; ++m) t += ((m == 0 ? D->L + 1 : 2 * (D->L - m + 1)) * 3 * E + 63) / 64 * 64;
    return t;
  }();
  // fp32 row-major (CUDA-core path) or bf16 tiles of 128 edges (tensor cores)
  const size_t a1_fp32 = (size_t)D->chunk_cap * K1T * 4;
  const size_t a1_bf16 = (size_t)((D->chunk_cap + 127) / 128) * 128 * K1T * 2;
  const size_t a1_f16s =
      so2_f16x3_available(D->L, D->E) ? (size_t)((D->chunk_cap + 127) / 128) * so2_f16x3_a1_tile_bytes(D->L, D->E) : 0;
  void* a1_prev = D->A1;
  D->A1 = (void*)grow((uint8_t*)D->A1, D->cap_a1, std::max(std::max(a1_fp32, a1_bf16), a1_f16s));
  if (D->A1 != a1_prev) D->a1_zero_mode = 0;  // zeroed before the first tensor-core use (run_block)
  // fp32 rows (CUDA-core path) or bf16 tiles of 128 edges (tcgen05 epilogue)
  D->Y = (float*)grow((uint8_t*)D->Y, D->cap_y, (size_t)((D->chunk_cap + 127) / 128) * 128 * row * 4);
  D->logits = grow(D->logits, D->cap_logits, (size_t)D->chunk_cap);
  if (D->cap_node_out < (size_t)std::max(n_owned, 1) * M->heads.out_len ||
      D->cap_edge_out < (size_t)std::max<int64_t>(ne, 1) * M->heads.out_len)
    model_outputs_wait(M);  // pending copies still read the buffers about to be replaced
  D->node_out = grow(D->node_out, D->cap_node_out, (size_t)std::max(n_owned, 1) * M->heads.out_len);
  D->edge_out = grow(D->edge_out, D->cap_edge_out, (size_t)std::max<int64_t>(ne, 1) * M->heads.out_len);
  // halo
  D->nbrs.clear();
  D->n_send = 0;
  if (plan) {
    D->nbrs = plan->nbrs;
    std::vector<int> all;
    for (const auto& nb : plan->nbrs) all.insert(all.end(), nb.send_rows.begin(), nb.send_rows.end());
    D->n_send = (int64_t)all.size();
    D->send_rows = grow(D->send_rows, D->cap_send_rows, all.size());
    D->send_buf = grow(D->send_buf, D->cap_send_buf, all.size() * row);
    if (!all.empty())
      h2d_staged(M->ctx, D->send_rows, all.data(), sizeof(int) * all.size());
  }
  ESG_CUDA(cudaStreamSynchronize(st));  // host vectors above are freed on return
  if (!(plan && plan->d_src_row)) free_ptr(d_eidx);
  D->prepared = true;
  D->train_stale = true;
}

namespace {

template <int H, int E>
void launch_heads(const float* x, int64_t n, const float* W, const int* key_of, const int* row_of, int out_len,
                  float* out, cudaStream_t st);

// Layer 0 of a plain forward: k_init_edges writes only the l = 0 plane of the
// edge rows and the layer-0 kernels read the other planes as zero (layer 0's
// rotate_out writes the full rows).  Training keeps full rows (its saved
// inputs are read whole), and so does a zero-layer model (the heads read them).
bool el0_edges(const esg_model* M) { return !M->dev->save_inputs && M->cfg.layers > 0; }

// The head tables may still be read by the copies of an earlier async
// forward: everything after this point on st waits for them.
void wait_prior_copies(DeviceModel* D, cudaStream_t st) {
  if (D->copies_pending) ESG_CUDA(cudaStreamWaitEvent(st, D->copies_done, 0));
}

// Streamed outputs: rows [i0, i0 + n) of a head table are final on st; once
// they are computed (heads) copy them to the pinned host buffer on copy_st.
void stream_rows(DeviceModel* D, cudaStream_t st, const float* dev, float* host, int64_t i0, int64_t n, int ol) {
  if (n <= 0) return;
  if (D->out_ev_used == D->out_ev.size()) {
    cudaEvent_t e;
    ESG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    D->out_ev.push_back(e);
  }
  cudaEvent_t e = D->out_ev[D->out_ev_used++];
  ESG_CUDA(cudaEventRecord(e, st));
  ESG_CUDA(cudaStreamWaitEvent(D->copy_st, e, 0));
  ESG_CUDA(cudaMemcpyAsync(host + i0 * ol, dev + i0 * ol, sizeof(float) * (size_t)n * ol, cudaMemcpyDeviceToHost,
                           D->copy_st));
}

template <int L, int E>
void run_block(esg_model* M, int layer, bool node_block) {
  DeviceModel* D = M->dev;
  esg_ctx* ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  constexpr int H = (L + 1) * (L + 1);
  // layer 0 of a plain forward: the edge table still holds only its l = 0
  // plane (1), and before the node update so do the node rows (2: k_init_nodes
  // embeds into l = 0 only)
  const int el0 = layer == 0 && el0_edges(M) ? (node_block ? 3 : 1) : 0;
  const int bidx = 2 * layer + (node_block ? 0 : 1);
  // halo exchange (distributed.h:51-130): pack, grouped send/recv straight
  // into the contiguous halo rows of each peer.  No host synchronisation: the
  // exchange's events are read after the forward's final one.  With
  // profiling on, a one-float allreduce first lines the ranks up, so the
  // exchange time (pack start -> last recv) is separated from rank skew.
  if (ctx->world > 1) {
    const int x = (int)D->halo_marks.size();
    while ((int)D->halo_ev.size() < 3 * (x + 1)) {
      cudaEvent_t e;
      ESG_CUDA(cudaEventCreate(&e));
      D->halo_ev.push_back(e);
    }
    D->halo_marks.push_back(x);
    ESG_CUDA(cudaEventRecord(D->halo_ev[3 * x], st));
    if (D->profile) {
      ESG_NCCL(ncclAllReduce(D->tmax + 15, D->tmax + 15, 1, ncclFloat, ncclMax, ctx->comm, st));
    }
    ESG_CUDA(cudaEventRecord(D->halo_ev[3 * x + 1], st));
    const int row = H * E;
    if (D->n_send) {
      Prof pr(D, st, ESG_PROF_HALO);
      k_pack_rows<<<(unsigned)((D->n_send * row + 255) / 256), 256, 0, st>>>(D->nodes, D->send_rows, D->n_send, row,
                                                                             D->send_buf);
      ++ctx->launches;
    }
    ESG_NCCL(ncclGroupStart());
    int64_t so = 0;
    for (const auto& nb : D->nbrs) {
      const int64_t cnt = (int64_t)nb.send_rows.size() * row;
      ESG_NCCL(ncclSend(D->send_buf + so * row, cnt, ncclFloat, nb.peer, ctx->comm, st));
      so += (int64_t)nb.send_rows.size();
      ESG_NCCL(ncclRecv(D->nodes + (int64_t)nb.recv_row * row, (int64_t)nb.recv_count * row, ncclFloat, nb.peer,
                        ctx->comm, st));
      D->halo_bytes += (int64_t)(nb.send_rows.size() + nb.recv_count) * row * (int64_t)sizeof(float);
    }
    ESG_NCCL(ncclGroupEnd());
    ESG_CUDA(cudaEventRecord(D->halo_ev[3 * x + 2], st));
  }
  if (D->save_inputs) {  // training: this block's input tables (after the exchange)
    const size_t row_bytes = sizeof(float) * H * E;
    ESG_CUDA(cudaMemcpyAsync(D->saved_nodes[bidx], D->nodes, row_bytes * D->n_rows, cudaMemcpyDeviceToDevice, st));
    // edge tables of layers >= 1 (layer 0's is recomputed by the backward, model_init_edges)
    if (node_block && D->n_edges && (layer >= 1 || M->cfg.layers == 1))
      ESG_CUDA(cudaMemcpyAsync(D->saved_edges[layer], D->edges, row_bytes * D->n_edges, cudaMemcpyDeviceToDevice,
                               st));
  }
  if (node_block) {  // halo rows pass through (ops.h:200 copies all rows)
    const int64_t n = (int64_t)D->n_rows * H * E;
    Prof pr(D, st, ESG_PROF_COPY);
    k_copy_rows<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(D->nodes, D->nodes_alt, n);
    ++ctx->launches;
  }
  const bool tc = D->precision == ESG_LINEAR_BF16 && so2_tc_available(L, E);
  // fp32 linears on the tensor cores through the fp16x3 split (so2_f16x3.cu),
  // the training forward included (its reverse pass recomputes the block from
  // the saved inputs with the 3xTF32 GEMMs)
  const bool f3 = !tc && D->f16x3 && !D->w1f.empty();
  const int zero_mode = tc ? 1 : (f3 ? 2 : 0);
  if (zero_mode && D->a1_zero_mode != zero_mode) {
    // the K padding slots of a tensor-core image are never written by rotate_in
    ESG_CUDA(cudaMemsetAsync(D->A1, 0, D->cap_a1, st));
    D->a1_zero_mode = zero_mode;
  } else if (!zero_mode) {
    D->a1_zero_mode = 0;  // the CUDA-core path writes fp32 rows over the whole buffer
  }
  if (f3) pack_f16x3_images(M);
  const int edge_slot = 1 + layer;  // tmax slot of the edge table entering this layer
  if (f3) {  // |node table| bound after the exchange (k_abs_max, a 1.6 KB/row read)
    Prof pr(D, st, ESG_PROF_COPY);
    ESG_CUDA(cudaMemsetAsync(D->tmax, 0, sizeof(float), st));
    const int64_t n4 = (int64_t)D->n_rows * H * E / 4;
    k_abs_max<256><<<(unsigned)std::min<int64_t>((n4 + 255) / 256, (int64_t)sm_count() * 8), 256, 0, st>>>(D->nodes, 4 * n4, D->tmax);
    ++ctx->launches;
    // P ranks: the maxima over all ranks' rows and edges are the serial run's,
    // so every rank splits with the serial scales (partitioned == serial, bit
    // for bit).  One 64-byte allreduce per block.
    if (ctx->world > 1) ESG_NCCL(ncclAllReduce(D->tmax, D->tmax, 16, ncclFloat, ncclMax, ctx->comm, st));
  }
  const float* att = D->params + D->att_off[layer];
  for (const auto& ch : D->chunks) {
    const int64_t e0 = D->h_seg[ch.first], e1 = D->h_seg[ch.second];
    const int64_t n = e1 - e0;
    if (n > 0) {
      const unsigned ri_tiles = (unsigned)((n + 31) / 32);
      constexpr int RI_THREADS = 32 * 3 * E / 4 < 128 ? 128 : 32 * 3 * E / 4;  // >= 4 warps for the Wigner groups
      if (f3) {
        {
          Prof pr(D, st, ESG_PROF_ROTATE_IN);
          k_rotate_in<L, E, 32, uint8_t><<<ri_tiles, RI_THREADS, 0, st>>>(D->nodes, D->edges, D->src_row, D->dst_row,
                                                                        D->dir, e0, n, (uint8_t*)D->A1, D->prefetch,
                                                                        el0, D->tmax, edge_slot);
        }
        ++ctx->launches;
        Prof pr(D, st, ESG_PROF_SO2);
        so2_f16x3_launch(L, E, (const uint8_t*)D->A1, n, D->w1f[bidx], D->w2f[bidx], D->f16sc[bidx], D->tmax,
                         edge_slot, D->Y, M->cfg.gate_enabled, att, node_block ? D->logits : nullptr, st);
        ++ctx->launches;
      } else if (tc) {
        {
          Prof pr(D, st, ESG_PROF_ROTATE_IN);
          k_rotate_in<L, E, 64, uint16_t><<<ri_tiles, RI_THREADS, 0, st>>>(D->nodes, D->edges, D->src_row, D->dst_row,
                                                                         D->dir, e0, n, (uint16_t*)D->A1, D->prefetch,
                                                                         el0);
        }
        ++ctx->launches;
        Prof pr(D, st, ESG_PROF_SO2);
        so2_tc_launch(L, E, (const uint16_t*)D->A1, n, D->w1b[bidx], D->w2b[bidx], (uint16_t*)D->Y,
                      M->cfg.gate_enabled, att, node_block ? D->logits : nullptr, st);
        ++ctx->launches;
      } else {
        {
          Prof pr(D, st, ESG_PROF_ROTATE_IN);
          k_rotate_in<L, E, 1, float><<<ri_tiles, RI_THREADS, 0, st>>>(D->nodes, D->edges, D->src_row, D->dst_row,
                                                                    D->dir, e0, n, (float*)D->A1, D->prefetch, el0);
        }
        Prof pr(D, st, ESG_PROF_SO2);
        // CUDA-core SGEMM per order block, gate in place, SGEMM
        D->Hbuf = grow(D->Hbuf, D->cap_hbuf, (size_t)D->chunk_cap * H * 2 * E);
        if (D->tf32) {
          tf32_gemm_launch((const float*)D->A1, (int64_t)H * 3 * E, n, D->wtc[0][bidx], D->tct[0], D->n_tct[0],
                           D->Hbuf, (int64_t)H * 2 * E, st);
        } else {
          lin_launch<L, E>(0, (const float*)D->A1, n, D->w1t[bidx], D->Hbuf, D->lt[0], D->n_lt[0], st);
        }
        if (D->tf32) {  // gate fused into lin2's operand load
          tf32_gemm_launch(D->Hbuf, (int64_t)H * 2 * E, n, D->wtc[1][bidx], D->tct[1], D->n_tct[1], D->Y,
                           (int64_t)H * E, st, M->cfg.gate_enabled ? 2 * E : 0);
        } else {
          k_gate_fwd<H><<<(unsigned)((n * 2 * E + 255) / 256), 256, 0, st>>>(D->Hbuf, 2 * E, n,
                                                                              M->cfg.gate_enabled, D->Hbuf);
          lin_launch<L, E>(1, D->Hbuf, n, D->w2t[bidx], D->Y, D->lt[1], D->n_lt[1], st);
        }
        ctx->launches += 4;
      }
      if (!node_block) {
        Prof pr(D, st, ESG_PROF_ROTATE_OUT);
        const unsigned ro_grid = (unsigned)((n + 31) / 32);
        constexpr int ro_threads = 32 * E / 4 < 128 ? 128 : 32 * E / 4;
        if (tc)
          k_rotate_out_edge<L, E, uint16_t><<<ro_grid, ro_threads, 0, st>>>((const uint16_t*)D->Y, D->dir, e0, n,
                                                                            D->edges, D->prefetch, el0);
        else if (f3)  // the chain's tiled fp32 Y (no L2 prefetch: 157 vs 165 ms per C4 forward)
          k_rotate_out_edge<L, E, F32T><<<ro_grid, ro_threads, 0, st>>>((const F32T*)D->Y, D->dir, e0, n, D->edges,
                                                                      0, el0, D->tmax + 2 + layer);
        else
          k_rotate_out_edge<L, E, float><<<ro_grid, ro_threads, 0, st>>>(D->Y, D->dir, e0, n, D->edges, D->prefetch,
                                                                       el0);
        ++ctx->launches;
      }
      if (!node_block && D->host_edge_out && layer == M->cfg.layers - 1) {
        // the chunk's edge rows are final: its heads now, the copy overlaps the next chunks
        Prof pr(D, st, ESG_PROF_HEADS);
        const int ol = M->heads.out_len;
        wait_prior_copies(D, st);
        launch_heads<H, E>(D->edges + e0 * H * E, n, D->head_w[1], D->head_key, D->head_row, ol,
                           D->edge_out + e0 * ol, st);
        ++ctx->launches;
        stream_rows(D, st, D->edge_out, D->host_edge_out, e0, n, ol);
      }
    }
    if (node_block && ch.second > ch.first) {
      Prof pr(D, st, ESG_PROF_NODE);
      constexpr int dyn = node_update_smem_floats<L, E, float>() * (int)sizeof(float);
      constexpr int dyn_bf16 = node_update_smem_floats<L, E, uint16_t>() * (int)sizeof(float);
      static std::atomic<uint64_t> attr{0};
      once_per_device(attr, [&] {
        ESG_CUDA(cudaFuncSetAttribute(k_node_update<L, E, float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      dyn));
        ESG_CUDA(cudaFuncSetAttribute(k_node_update<L, E, uint16_t, true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_bf16));
        ESG_CUDA(cudaFuncSetAttribute(k_node_update<L, E, F32T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      dyn));
      });
      if (f3)  // logits from the chain's fp32 accumulator
        k_node_update<L, E, F32T, true><<<ch.second - ch.first, 128, dyn, st>>>(
            (const F32T*)D->Y, D->dir, D->seg, ch.first, e0, att, D->nodes, D->nodes_alt, D->logits, D->prefetch);
      else if (tc)
        k_node_update<L, E, uint16_t, true><<<ch.second - ch.first, 128, dyn_bf16, st>>>(
            (const uint16_t*)D->Y, D->dir, D->seg, ch.first, e0, att, D->nodes, D->nodes_alt, D->logits, D->prefetch);
      else
        k_node_update<L, E, float, false><<<ch.second - ch.first, 128, dyn, st>>>(D->Y, D->dir, D->seg, ch.first, e0, att,
                                                                          D->nodes, D->nodes_alt, D->logits, D->prefetch);
      ++ctx->launches;
    }
  }
  ESG_CUDA(cudaGetLastError());
  if (node_block) std::swap(D->nodes, D->nodes_alt);
}

template <int H, int E>
void launch_heads(const float* x, int64_t n, const float* W, const int* key_of, const int* row_of, int out_len,
                  float* out, cudaStream_t st) {
  if (out_len > 256) usage("head layout wider than 256 outputs");
  constexpr int smem = heads_smem_bytes<H, E>();
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [&] {
    ESG_CUDA(cudaFuncSetAttribute(k_heads<H, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  });
  const int threads = ((out_len + 31) / 32) * 32;
  const unsigned blocks = (unsigned)std::min<int64_t>((n + HT - 1) / HT, sm_count() * 3);  // 3 x 64 KB per SM
  k_heads<H, E><<<blocks, threads, smem, st>>>(x, n, W, key_of, row_of, out_len, out);
}

template <int L, int E>
void forward_impl(esg_model* M, esg_timing* tm) {
  DeviceModel* D = M->dev;
  esg_ctx* ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  constexpr int H = (L + 1) * (L + 1);
  const int64_t launches0 = ctx->launches;
  ESG_CUDA(cudaEventRecord(D->ev[0], st));
  {
    const int64_t n = (int64_t)D->n_rows * H * E;
    Prof pr(D, st, ESG_PROF_INIT);
    ESG_CUDA(cudaMemsetAsync(D->tmax, 0, 16 * sizeof(float), st));  // table maxima of this forward
    k_init_nodes<H, E><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(D->row_slot, D->n_rows, D->embed, D->nodes);
    ++ctx->launches;
    if (D->n_edges) {
      Prof pr2(D, st, ESG_PROF_INIT);
      if (M->cfg.n_radial > 32) usage("the GPU radial lift supports up to 32 Gaussians");
      const int64_t blocks = std::min<int64_t>((D->n_edges + 255) / 256, (int64_t)sm_count() * 8);  // 8 warps x 32-edge blocks
      k_init_edges<H, E, 32><<<(unsigned)blocks, 256, 0, st>>>(D->dist, D->n_edges, D->params + D->lift_off,
                                                                M->cfg.n_radial,
                                                                M->cfg.r_cut / (M->cfg.n_radial - 1), D->edges,
                                                                el0_edges(M) ? 0 : 1, D->tmax + 1);
      ++ctx->launches;
    }
  }
  ESG_CUDA(cudaEventRecord(D->ev[1], st));
  int64_t exchanges = 0;
  D->halo_marks.clear();
  D->halo_bytes = 0;
  const int out_len = M->heads.out_len;
  const bool streamed = D->host_node_out || D->host_edge_out;
  D->out_ev_used = 0;
  for (int layer = 0; layer < M->cfg.layers; ++layer)
    for (bool nb : {true, false}) {
      run_block<L, E>(M, layer, nb);
      ++exchanges;
      if (streamed && nb && layer == M->cfg.layers - 1 && D->n_owned) {
        // the node table is final after the last node block: its heads and
        // their copy overlap the last edge block
        Prof pr(D, st, ESG_PROF_HEADS);
        wait_prior_copies(D, st);
        launch_heads<H, E>(D->nodes, D->n_owned, D->head_w[0], D->head_key, D->head_row, out_len, D->node_out, st);
        ++ctx->launches;
        if (D->host_node_out) stream_rows(D, st, D->node_out, D->host_node_out, 0, D->n_owned, out_len);
      }
    }
  ESG_CUDA(cudaEventRecord(D->ev[2], st));
  wait_prior_copies(D, st);
  if (D->n_owned && !streamed) {
    Prof pr(D, st, ESG_PROF_HEADS);
    launch_heads<H, E>(D->nodes, D->n_owned, D->head_w[0], D->head_key, D->head_row, out_len, D->node_out, st);
    ++ctx->launches;
  }
  if (D->n_edges && (!streamed || !D->host_edge_out)) {
    Prof pr(D, st, ESG_PROF_HEADS);
    launch_heads<H, E>(D->edges, D->n_edges, D->head_w[1], D->head_key, D->head_row, out_len, D->edge_out, st);
    ++ctx->launches;
  }
  ESG_CUDA(cudaEventRecord(D->ev[3], st));
  ESG_CUDA(cudaGetLastError());
  if (D->defer_sync) return;  // async forward without timing: the host goes on
  ESG_CUDA(cudaEventSynchronize(D->ev[3]));
  prof_collect(D);
  if (tm) {
    float a = 0, b = 0, c = 0;
    ESG_CUDA(cudaEventElapsedTime(&a, D->ev[0], D->ev[3]));
    ESG_CUDA(cudaEventElapsedTime(&b, D->ev[1], D->ev[2]));
    ESG_CUDA(cudaEventElapsedTime(&c, D->ev[2], D->ev[3]));
    tm->forward_ms = a;
    tm->message_ms = b;
    tm->heads_ms = c;
    double halo = 0, skew = 0, xch = 0;
    for (int x : D->halo_marks) {
      float t0 = 0, t1 = 0;
      ESG_CUDA(cudaEventElapsedTime(&t0, D->halo_ev[3 * x], D->halo_ev[3 * x + 1]));
      ESG_CUDA(cudaEventElapsedTime(&t1, D->halo_ev[3 * x + 1], D->halo_ev[3 * x + 2]));
      halo += t0 + t1;
      skew += t0;
      xch += t1;
    }
    tm->halo_ms = halo;
    tm->halo_skew_ms = D->profile ? skew : -1.0;  // measured only with the lining-up allreduce
    tm->halo_exchange_ms = D->profile ? xch : halo;
    tm->halo_bytes = D->halo_bytes;
    tm->exchanges = ctx->world > 1 ? exchanges : 0;
    tm->gpu_launches = ctx->launches - launches0;
  }
}

}  // namespace

// Per-edge rotation blocks (kernels.h:43-68 build_edge_rotations): the
// fp32 displacement (the prepared view's `dir`, rounded from the fp64
// Graph::disp) through align_to_y and the generated Ivanic-Ruedenberg
// recursion -- the same device code the message kernels run in-register.
// Output per edge: the stacked D_l blocks l = 0..L, (2l+1)^2 row-major each.
template <int L>
__global__ void __launch_bounds__(128) k_edge_rotations(const double* __restrict__ disp, int64_t n,
                                                        float* __restrict__ out) {
  using G = Geo<L>;
  constexpr int TE = L >= 6 ? 16 : 32, DSP = G::DS + 2;  // static SMEM <= 48 KB
  __shared__ float sD[TE * DSP];
  __shared__ float sdir[TE * 3];
  const int64_t t0 = (int64_t)blockIdx.x * TE;
  const int ne = (int)(n - t0 < TE ? n - t0 : TE);
  for (int i = threadIdx.x; i < ne * 3; i += blockDim.x) sdir[i] = (float)disp[t0 * 3 + i];
  __syncthreads();
  wigner_tile_gen<L, DSP>(sdir, ne, sD);
  for (int i = threadIdx.x; i < ne * G::DS; i += blockDim.x) out[t0 * G::DS + i] = sD[(i / G::DS) * DSP + i % G::DS];
}

void edge_rotations(esg_ctx* ctx, int64_t n, const double* disp, int l_max, float* out) {
  if (l_max < 1 || l_max > 6) usage("edge rotations: l_max must be 1..6");
  if (n <= 0) return;
  const int ds = l_max + 1 == 0 ? 0 : (l_max + 1) * (4 * (l_max + 1) * (l_max + 1) - 1) / 3;
  cudaStream_t st = ctx->stream;
  double* d_disp = nullptr;
  float* d_out = nullptr;
  ESG_CUDA(cudaMalloc(&d_disp, sizeof(double) * 3 * n));
  ESG_CUDA(cudaMalloc(&d_out, sizeof(float) * ds * n));
  ESG_CUDA(cudaMemcpyAsync(d_disp, disp, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
  const unsigned grid = (unsigned)((n + 31) / 32), grid6 = (unsigned)((n + 15) / 16);
  switch (l_max) {
    case 1: k_edge_rotations<1><<<grid, 128, 0, st>>>(d_disp, n, d_out); break;
    case 2: k_edge_rotations<2><<<grid, 128, 0, st>>>(d_disp, n, d_out); break;
    case 3: k_edge_rotations<3><<<grid, 128, 0, st>>>(d_disp, n, d_out); break;
    case 4: k_edge_rotations<4><<<grid, 128, 0, st>>>(d_disp, n, d_out); break;
    case 5: k_edge_rotations<5><<<grid, 128, 0, st>>>(d_disp, n, d_out); break;
    default: k_edge_rotations<6><<<grid6, 128, 0, st>>>(d_disp, n, d_out); break;
  }
  ++ctx->launches;
  ESG_CUDA(cudaGetLastError());
  ESG_CUDA(cudaMemcpyAsync(out, d_out, sizeof(float) * ds * n, cudaMemcpyDeviceToHost, st));
  ESG_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_disp);
  cudaFree(d_out);
}

// The initial edge table (k_init_edges) into out: the training backward
// recomputes layer 0's input instead of keeping it.
void model_init_edges(esg_model* M, float* out, cudaStream_t st) {
  DeviceModel* D = M->dev;
  const int L = D->L, E = D->E;
  if (!D->n_edges) return;
  const int64_t blocks = std::min<int64_t>((D->n_edges + 255) / 256, (int64_t)sm_count() * 8);
  const double spacing = M->cfg.r_cut / (M->cfg.n_radial - 1);
  auto go = [&](auto h, auto e) {
    constexpr int H = decltype(h)::value, EE = decltype(e)::value;
    k_init_edges<H, EE, 32><<<(unsigned)blocks, 256, 0, st>>>(D->dist, D->n_edges, D->params + D->lift_off,
                                                               M->cfg.n_radial, spacing, out, 1);
  };
  using I25 = std::integral_constant<int, 25>;
  using I9 = std::integral_constant<int, 9>;
  using I16 = std::integral_constant<int, 16>;
  using I8 = std::integral_constant<int, 8>;
  if (L == 4 && E == 16)
    go(I25{}, I16{});
  else if (L == 4 && E == 8)
    go(I25{}, I8{});
  else if (L == 2 && E == 16)
    go(I9{}, I16{});
  else
    go(I9{}, I8{});
  ESG_CUDA(cudaGetLastError());
}

void model_forward(esg_model* M, esg_timing* tm) {
  DeviceModel* D = M->dev;
  if (!D->prepared) usage("forward before prepare");
  D->precision = M->cfg.linear_precision;
  const int L = D->L, E = D->E;
  if (L == 4 && E == 16)
    forward_impl<4, 16>(M, tm);
  else if (L == 4 && E == 8)
    forward_impl<4, 8>(M, tm);
  else if (L == 2 && E == 16)
    forward_impl<2, 16>(M, tm);
  else
    forward_impl<2, 8>(M, tm);
}

void model_profile(esg_model* M, int enable, double* ms, int64_t* counts) {
  DeviceModel* D = M->dev;
  if (ms)
    for (int c = 0; c < ESG_PROF_NCAT; ++c) ms[c] = D->prof_ms[c];
  if (counts)
    for (int c = 0; c < ESG_PROF_NCAT; ++c) counts[c] = D->prof_n[c];
  if (enable >= 0) {
    D->profile = enable != 0;
    for (int c = 0; c < ESG_PROF_NCAT; ++c) {
      D->prof_ms[c] = 0;
      D->prof_n[c] = 0;
    }
  }
}

void model_outputs(const esg_model* M, const float** no, const float** eo, const float** nf, const float** ef) {
  const DeviceModel* D = M->dev;
  if (no) *no = D->node_out;
  if (eo) *eo = D->edge_out;
  if (nf) *nf = D->nodes;
  if (ef) *ef = D->edges;
}

void model_copy_outputs(const esg_model* M, float* node_out, float* edge_out);

// esg_forward with host output buffers: when both given buffers are pinned
// (page-locked or registered), the heads of each final chunk are copied while
// the rest of the last edge block computes; otherwise the copies follow the
// forward.
bool pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void model_outputs_wait(esg_model* M) {
  DeviceModel* D = M->dev;
  if (!D || !D->copies_pending) return;
  ESG_CUDA(cudaEventSynchronize(D->ev[3]));  // the forward itself (a deferred one included)
  ESG_CUDA(cudaEventSynchronize(D->copies_done));
  D->copies_pending = false;
}

// async: return once the compute is done and the output copies are queued on
// copy_st (pinned buffers only); model_outputs_wait completes them.  The next
// forward overlaps those copies until its first heads launch.
void model_forward_to_host(esg_model* M, esg_timing* tm, float* node_out, float* edge_out, bool async) {
  DeviceModel* D = M->dev;
  if ((node_out || edge_out) && pinned(node_out) && pinned(edge_out) && !D->save_inputs) {
    if (!D->copy_st) ESG_CUDA(cudaStreamCreateWithFlags(&D->copy_st, cudaStreamNonBlocking));
    if (!D->copies_done) ESG_CUDA(cudaEventCreateWithFlags(&D->copies_done, cudaEventDisableTiming));
    D->host_node_out = node_out;
    D->host_edge_out = edge_out;
    // no timing asked for: the host does not wait for the forward either
    D->defer_sync = async && !tm && !D->profile;
    try {
      model_forward(M, tm);
    } catch (...) {
      D->host_node_out = D->host_edge_out = nullptr;
      D->defer_sync = false;
      cudaStreamSynchronize(M->ctx->stream);
      cudaStreamSynchronize(D->copy_st);
      D->copies_pending = false;
      throw;
    }
    D->defer_sync = false;
    D->host_node_out = D->host_edge_out = nullptr;
    ESG_CUDA(cudaEventRecord(D->copies_done, D->copy_st));
    D->copies_pending = true;
    if (!async) model_outputs_wait(M);
    return;
  }
  model_forward(M, tm);
  if (node_out || edge_out) model_copy_outputs(M, node_out, edge_out);
}

void model_copy_outputs(const esg_model* M, float* node_out, float* edge_out) {
  const DeviceModel* D = M->dev;
  const int ol = M->heads.out_len;
  ESG_CUDA(cudaStreamSynchronize(M->ctx->stream));
  if (node_out && D->n_owned)
    ESG_CUDA(cudaMemcpy(node_out, D->node_out, sizeof(float) * (size_t)D->n_owned * ol, cudaMemcpyDeviceToHost));
  if (edge_out && D->n_edges)
    ESG_CUDA(cudaMemcpy(edge_out, D->edge_out, sizeof(float) * (size_t)D->n_edges * ol, cudaMemcpyDeviceToHost));
}

// Rows [first, first + count) of the last forward's head outputs to host.
void model_copy_output_rows(const esg_model* M, int64_t nf, int64_t nc, float* node_out, int64_t ef, int64_t ec,
                            float* edge_out) {
  const DeviceModel* D = M->dev;
  const int ol = M->heads.out_len;
  if (nc < 0 || ec < 0 || nf < 0 || ef < 0 || nf + nc > D->n_owned || ef + ec > D->n_edges)
    usage("output row range outside the prepared view");
  ESG_CUDA(cudaStreamSynchronize(M->ctx->stream));
  if (node_out && nc)
    ESG_CUDA(cudaMemcpy(node_out, D->node_out + nf * ol, sizeof(float) * (size_t)nc * ol, cudaMemcpyDeviceToHost));
  if (edge_out && ec)
    ESG_CUDA(cudaMemcpy(edge_out, D->edge_out + ef * ol, sizeof(float) * (size_t)ec * ol, cudaMemcpyDeviceToHost));
}

void model_copy_features(const esg_model* M, float* nodes, float* edges) {
  const DeviceModel* D = M->dev;
  const size_t row = (size_t)D->H * D->E;
  if (nodes) ESG_CUDA(cudaMemcpy(nodes, D->nodes, sizeof(float) * D->n_rows * row, cudaMemcpyDeviceToHost));
  if (edges && D->n_edges)
    ESG_CUDA(cudaMemcpy(edges, D->edges, sizeof(float) * D->n_edges * row, cudaMemcpyDeviceToHost));
}

void model_prepared_info(const esg_model* M, int64_t info[3]) {
  info[0] = M->dev->n_rows;
  info[1] = M->dev->n_owned;
  info[2] = M->dev->n_edges;
}

// Uncoupled blocks of the last forward, items = owned nodes then view edges.
}  // namespace esg
