// train.cu -- config 5: masked loss, backward, gradient allreduce (SURVEY §8
// row a19; distributed.h:147-235, ops.h backward closures, kernels.h:163-250).
//
// The forward runs on the fp32 CUDA-core path with save_inputs set, so every
// block's input tables are kept (node table after the block's halo exchange,
// edge table entering each layer).  The backward walks the blocks in reverse;
// per destination-aligned chunk it recomputes the block's forward
// intermediates (A1, lin1 pre-activation H, gated G, and for node blocks lin2
// output Y and the back-rotated message) and then applies the adjoints:
//   msg = D^T Y               ->  gY  = D g_msg            (k_rot1<1>)
//   Y   = W2 G (per order)    ->  gG  = W2^T gY,  dW2 += gY G^T
//   G   = gate(H)             ->  gH  (kernels.h:228-250)
//   H   = W1 A1               ->  gA1 = W1^T gH,  dW1 += gH A1^T
//   A1  = D [src | dst | edge] -> g_src, g_dst, g_edge (k_rot_in_bwd)
// Every reduction has a fixed order: weight gradients accumulate per output
// tile over the chunk's edges in edge order (fp64), destination rows reduce
// their segment in edge order, source rows their chunk-local edge list in
// edge order, chunks in chunk order.  Results are deterministic run to run.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "device_model.h"
#include "esg_internal.h"
#include "model_kernels.cuh"
#include "msg_kernels.cuh"
#include "lin_kernels.cuh"

namespace esg {

std::vector<float> expanded(const esg_model* M, const std::string& base, int m, int cin, int cout);  // model.cu

struct TrainState {
  float* adam_g = nullptr;  // device Adam: this step's gradients
  int64_t adam_g_n = 0;
  // loss targets in head space, view order (network.h:187-214)
  float* node_target = nullptr;
  uint8_t* node_mask = nullptr;
  float* edge_target = nullptr;
  uint8_t* edge_mask = nullptr;
  int64_t tgt_owned = -1, tgt_edges = -1;
  // gradient tables (n_rows / n_edges x H x E) and head-output seeds
  float* g_nodes = nullptr;
  float* g_edges = nullptr;
  float* g_nodes_out = nullptr;  // node blocks: snapshot of the output gradient (attention backward input)
  float* g_node_out = nullptr;
  float* g_edge_out = nullptr;
  // chunk scratch
  int64_t cap = 0;
  float *A1 = nullptr, *Hh = nullptr, *Gg = nullptr, *Yy = nullptr, *msg = nullptr, *gY = nullptr, *gG = nullptr,
        *gH = nullptr, *gA1 = nullptr, *gx = nullptr;
  std::vector<std::pair<int, int>> chunks;  // owned-row ranges of <= cap edges
  // per chunk: edges sorted by source row (stable) for the source reduction
  std::vector<int*> src_perm, src_off, src_row_u;
  std::vector<int> n_src;
  // fp64 gradient accumulators in the expanded layout (see gacc_layout)
  double* gacc = nullptr;
  int64_t gacc_n = 0;
  std::vector<int64_t> off_lin1, off_lin2;  // per block
  std::vector<int64_t> off_att;              // per layer
  int64_t off_head[2] = {0, 0}, off_lift = 0, off_embed = 0;
  // reduction partials
  double* part = nullptr;
  int64_t part_n = 0;
  // tiled dW: tile lists of lin1 (g 2E x A1 3E) and lin2 (g E x G 2E), split partials
  DwTile* tiles1 = nullptr;
  DwTile* tiles2 = nullptr;
  int n_tiles1 = 0, n_tiles2 = 0;
  float* opart = nullptr;  // dW partial tiles (dw_tc.cu)
  int64_t opart_n = 0;
  // per head output j: its harmonic plane, and per plane the outputs (in key order)
  int* plane_ptr = nullptr;
  int* plane_out = nullptr;
  int* out_plane = nullptr;
  int* out_key = nullptr;
  float* rbf_scratch = nullptr;
  // halo backward buffers
  float* halo_send = nullptr;
  float* halo_recv = nullptr;
  int64_t halo_cap = 0;
  cudaEvent_t ev[4];
  double last_backward_ms = 0, last_forward_ms = 0;
};

namespace {

template <typename T>
T* talloc(size_t n) {
  T* p = nullptr;
  if (n) ESG_CUDA(cudaMalloc(&p, n * sizeof(T)));
  return p;
}

// ------------------------------------------------------------------ loss
// ops.h:347-371 masked_loss: partial sums of |d| and d^2 (fp64) and the
// count; the recorded backward seeds (sign(d) + 2 d) / n_total directly.
// g_out may alias pred (the seed overwrites the prediction it came from)
__global__ void k_loss(const float* pred, const float* __restrict__ tgt, const uint8_t* __restrict__ mask, int64_t n,
                       double inv_total, float* g_out, double* __restrict__ part) {
  double sa = 0.0, sq = 0.0, cnt = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    float g = 0.f;
    if (mask[k]) {
      const double d = double(pred[k]) - double(tgt[k]);
      sa += fabs(d);
      sq += d * d;
      cnt += 1.0;
      const double s = d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0);
      g = (float)((s + 2.0 * d) * inv_total);
    }
    g_out[k] = g;
  }
  __shared__ double red[3][256];
  red[0][threadIdx.x] = sa;
  red[1][threadIdx.x] = sq;
  red[2][threadIdx.x] = cnt;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if ((int)threadIdx.x < o)
      for (int q = 0; q < 3; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int q = 0; q < 3; ++q) part[blockIdx.x * 3 + q] = red[q][0];
}

// ------------------------------------------------------------- heads bwd
// ops.h:309-333.  g_x[i][p][c] += sum over outputs j of plane p (key order)
// of g_out[i][j] w[key(j)][c].
template <int H, int E>
__global__ void k_heads_bwd_x(const float* __restrict__ g_out, int out_len, int64_t n_items,
                              const float* __restrict__ W, const int* __restrict__ plane_ptr,
                              const int* __restrict__ plane_out, const int* __restrict__ out_key,
                              float* __restrict__ g_x) {
  // thread = (item, plane, 4-channel quad); the same per-channel sum order
  constexpr int Q = E / 4;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_items * H * Q) return;
  const int64_t i = t / (H * Q);
  const int p = (int)(t % (H * Q)) / Q, q = (int)(t % Q);
  float4* gx4 = reinterpret_cast<float4*>(g_x) + t;
  float4 acc = *gx4;
  for (int r = plane_ptr[p]; r < plane_ptr[p + 1]; ++r) {
    const int j = plane_out[r];
    const float up = g_out[i * out_len + j];
    if (up != 0.f) {
      const float4 w = __ldg(reinterpret_cast<const float4*>(W + out_key[j] * E) + q);
      acc.x += up * w.x;
      acc.y += up * w.y;
      acc.z += up * w.z;
      acc.w += up * w.w;
    }
  }
  *gx4 = acc;
}
// S[j][c] = sum_i g_out[i][j] x[i][plane(j)][c]: CTA partials over item
// ranges.  Tiles of TI items go through SMEM (their head gradients and
// feature rows, coalesced), then thread u = (j, c) pairs accumulate over the
// tile in item order (fp64: the same sum and order as one item at a time).
template <int H, int E>
__global__ void __launch_bounds__(256) k_heads_bwd_w(const float* __restrict__ g_out, int out_len, int64_t n_items,
                                                     const float* __restrict__ x, const int* __restrict__ out_plane,
                                                     double* __restrict__ part) {
  constexpr int TI = 16, UMAX = 16;  // out_len * E <= 256 * UMAX
  __shared__ float s_g[TI * 256];
  __shared__ float s_x[TI * H * E];
  const int64_t per = (n_items + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = blockIdx.x * per, i1 = i0 + per < n_items ? i0 + per : n_items;
  const int nu = out_len * E;
  double acc[UMAX];
  int off_x[UMAX], off_g[UMAX];
#pragma unroll
  for (int q = 0; q < UMAX; ++q) {
    acc[q] = 0.0;
    const int u = threadIdx.x + 256 * q, j = u / E, c = u % E;
    off_g[q] = u < nu ? j : 0;
    off_x[q] = u < nu ? out_plane[j] * E + c : 0;
  }
  for (int64_t t0 = i0; t0 < i1; t0 += TI) {
    const int ni = (int)(i1 - t0 < TI ? i1 - t0 : TI);
    __syncthreads();
    for (int v = threadIdx.x; v < ni * out_len; v += blockDim.x) s_g[(v / out_len) * 256 + v % out_len] = g_out[t0 * out_len + v];
    for (int v = threadIdx.x; v < ni * H * E; v += blockDim.x) s_x[v] = x[t0 * H * E + v];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < UMAX; ++q) {
      if (threadIdx.x + 256 * q < nu) {
        for (int ii = 0; ii < ni; ++ii) {
          const float up = s_g[ii * 256 + off_g[q]];
          if (up != 0.f) acc[q] += double(up) * double(s_x[ii * H * E + off_x[q]]);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < UMAX; ++q)
    if (threadIdx.x + 256 * q < nu) part[(int64_t)blockIdx.x * nu + threadIdx.x + 256 * q] = acc[q];
}
// out[u] += sum over the parts in order
__global__ void k_reduce_parts(const double* __restrict__ part, int n_parts, int64_t n, double* __restrict__ out) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  double acc = out[u];
  for (int p = 0; p < n_parts; ++p) acc += part[(int64_t)p * n + u];
  out[u] = acc;
}

// --------------------------------------------------------- SO(2) linears
// (forward and dx products: lin_kernels.cuh k_gemm_m)


// sg[e][c] = sigmoid(h[e][row 0][c]), the gate's per-edge scalars (c < c2),
// in the forward's rounding (1 / (1 + exp(-h)))
__global__ void k_gate_scale(const float* __restrict__ h, int64_t ldh, int c2, int64_t n_e, float* __restrict__ sg) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_e * c2) return;
  sg[t] = 1.f / (1.f + expf(-h[(t / c2) * ldh + t % c2]));
}

// gate (kernels.h:210-226) and its backward (kernels.h:228-250); rows are
// the 25 order-major rows of 2E channels, row 0 the l = 0 scalar
template <int H>
__global__ void k_gate_bwd(const float* __restrict__ h, const float* __restrict__ gg, int c2, int64_t n_e,
                           int enabled, float* __restrict__ gh) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_e * c2) return;
  const int64_t e = t / c2;
  const int c = (int)(t % c2);
  const float* xr = h + e * H * c2;
  const float* gr = gg + e * H * c2;
  float* dxr = gh + e * H * c2;
  if (!enabled) {
    for (int r = 0; r < H; ++r) dxr[r * c2 + c] = gr[r * c2 + c];
    return;
  }
  const float s = 1.f / (1.f + expf(-xr[c]));
  const float ds = s * (1.f - s);
  float acc = gr[c] * (s + xr[c] * ds);
  for (int r = 1; r < H; ++r) {
    dxr[r * c2 + c] = gr[r * c2 + c] * s;
    acc += gr[r * c2 + c] * xr[r * c2 + c] * ds;
  }
  dxr[c] = acc;
}

// --------------------------------------------------------------- rotations
// MODE 0: msg = D^T y (order-major rows -> degree-major, ops.h:115-117)
// MODE 1: gy  = D g  (degree-major -> order-major rows, its adjoint)
// Thread = (edge, 4-channel quad); 32 edges per CTA; D from the tile's SMEM.
template <int L, int E, int MODE>
__global__ void __launch_bounds__(128) k_rot1(const float* __restrict__ in, const float* __restrict__ dir, int64_t e0,
                                              int64_t n_e, float* __restrict__ out) {
  using G = Geo<L>;
  constexpr int TE = 32, DSP = G::DS + 2, H = G::H, Q = E / 4;
  __shared__ float sD[TE * DSP];
  __shared__ float sdir[TE * 3];
  const int64_t t0 = (int64_t)blockIdx.x * TE;
  const int ne = (int)(n_e - t0 < TE ? n_e - t0 : TE);
  for (int i = threadIdx.x; i < ne * 3; i += blockDim.x) sdir[i] = dir[(e0 + t0) * 3 + i];
  __syncthreads();
  wigner_tile_gen<L, DSP>(sdir, ne, sD);
  for (int u = threadIdx.x; u < ne * Q; u += blockDim.x) {
    const int e = u / Q, q = u % Q;
    const float* D = sD + e * DSP;
    const float4* src = reinterpret_cast<const float4*>(in + (t0 + e) * H * E) + q;
    float4* dst = reinterpret_cast<float4*>(out + (t0 + e) * H * E) + q;
#pragma unroll
    for (int l = 0; l <= L; ++l) {
      const int dd = 2 * l + 1;
      float4 x[2 * L + 1];
#pragma unroll
      for (int b = -l; b <= l; ++b) x[b + l] = src[(MODE == 0 ? G::mrow(l, b) : l * l + l + b) * Q];
#pragma unroll
      for (int a = -l; a <= l; ++a) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int b = -l; b <= l; ++b)
          acc = fma4(MODE == 0 ? D[G::doff(l) + (b + l) * dd + (a + l)] : D[G::doff(l) + (a + l) * dd + (b + l)],
                     x[b + l], acc);
        dst[(MODE == 0 ? l * l + l + a : G::mrow(l, a)) * Q] = acc;
      }
    }
  }
}

// rotate-in adjoint (ops.h:88-105 + 115-117): g_x = D^T gA1 per part; the
// edge part is added into g_edges in place, src/dst parts go to gx for the
// ordered row reductions.  Thread = (edge, part, quad).
template <int L, int E>
__global__ void __launch_bounds__(384) k_rot_in_bwd(const float* __restrict__ gA1, const float* __restrict__ dir,
                                                    int64_t e0, int64_t n_e, float* __restrict__ g_edges,
                                                    float* __restrict__ gx) {
  using G = Geo<L>;
  using Y = Lay1<L, E, 1>;
  constexpr int TE = 32, DSP = G::DS + 2, H = G::H, C3 = 3 * E, Q = E / 4, TPE = 3 * Q;
  __shared__ float sD[TE * DSP];
  __shared__ float sdir[TE * 3];
  const int64_t t0 = (int64_t)blockIdx.x * TE;
  const int ne = (int)(n_e - t0 < TE ? n_e - t0 : TE);
  for (int i = threadIdx.x; i < ne * 3; i += blockDim.x) sdir[i] = dir[(e0 + t0) * 3 + i];
  __syncthreads();
  wigner_tile_gen<L, DSP>(sdir, ne, sD);
  for (int u = threadIdx.x; u < ne * TPE; u += blockDim.x) {
    const int e = u / TPE, r = u % TPE, p = r / Q, q = r % Q;
    const float* D = sD + e * DSP;
    const float* ga = gA1 + (t0 + e) * Y::KTOT;
    float4* dst = p == 2 ? reinterpret_cast<float4*>(g_edges + (e0 + t0 + e) * H * E) + q
                         : reinterpret_cast<float4*>(gx + ((t0 + e) * 2 + p) * H * E) + q;
#pragma unroll
    for (int l = 0; l <= L; ++l) {
      const int dd = 2 * l + 1;
      float4 g[2 * L + 1];
#pragma unroll
      for (int a = -l; a <= l; ++a) {
        const int m = a < 0 ? -a : a;
        g[a + l] = *reinterpret_cast<const float4*>(ga + Y::kofs(m) + (G::mrow(l, a) - G::moff(m)) * C3 + p * E +
                                                    q * 4);
      }
#pragma unroll
      for (int b = -l; b <= l; ++b) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int a = -l; a <= l; ++a) acc = fma4(D[G::doff(l) + (a + l) * dd + (b + l)], g[a + l], acc);
        float4* o = dst + (l * l + l + b) * Q;
        if (p == 2) {
          const float4 old = *o;
          acc = make_float4(old.x + acc.x, old.y + acc.y, old.z + acc.z, old.w + acc.w);
        }
        *o = acc;
      }
    }
  }
}

// g_nodes[dst] += its segment's dst-part rows in edge order (owned rows j0..j1)
__global__ void k_dst_reduce(const float* __restrict__ gx, int row, const int64_t* __restrict__ seg, int j0,
                             int64_t e0, float* __restrict__ g_nodes) {
  // float4 columns; the adds stay in edge order (the loads run ahead)
  const int j = j0 + blockIdx.x;
  const int64_t b = seg[j], en = seg[j + 1];
  const int r4 = row >> 2;
  for (int t = threadIdx.x; t < r4; t += blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(g_nodes + (int64_t)j * row)[t];
#pragma unroll 8
    for (int64_t k = b; k < en; ++k) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(gx + ((k - e0) * 2 + 1) * row) + t);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(g_nodes + (int64_t)j * row)[t] = acc;
  }
}
// g_nodes[src] += the src-part rows of its chunk edges in edge order
__global__ void k_src_reduce(const float* __restrict__ gx, int row, const int* __restrict__ perm,
                             const int* __restrict__ off, const int* __restrict__ rows, float* __restrict__ g_nodes) {
  const int u = blockIdx.x;
  const int i = rows[u];
  const int r4 = row >> 2;
  for (int t = threadIdx.x; t < r4; t += blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(g_nodes + (int64_t)i * row)[t];
#pragma unroll 8
    for (int q = off[u]; q < off[u + 1]; ++q) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(gx + ((int64_t)perm[q] * 2 + 0) * row) + t);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(g_nodes + (int64_t)i * row)[t] = acc;
  }
}

// ----------------------------------------------------------- attention bwd
// ops.h:227-262 for the owned destinations j0 + blockIdx.x of one chunk:
// alpha from the recomputed messages (logits att . msg row 0, max-subtracted
// softmax as the forward), dot_k = <g_j, msg_k>, mean = sum alpha dot,
// g_msg_k = alpha_k g_j (+ dl_k att on row 0), dl_k = alpha_k (dot_k - mean),
// g_att partial per destination.
template <int H, int E>
__global__ void __launch_bounds__(128) k_attn_bwd(const float* __restrict__ msg, const float* __restrict__ att,
                                                  const int64_t* __restrict__ seg, int j0, int64_t e0,
                                                  const float* __restrict__ g_nodes, float* __restrict__ g_msg,
                                                  float* __restrict__ alpha_scratch, double* __restrict__ att_part) {
  constexpr int HE = H * E;
  const int j = j0 + blockIdx.x;
  const int64_t b = seg[j], en = seg[j + 1];
  const int t = threadIdx.x;
  __shared__ float sred[4];
  __shared__ float sg[HE];
  __shared__ double satt[4][E];
  for (int u = t; u < HE; u += 128) sg[u] = g_nodes[(int64_t)j * HE + u];
  if (b == en) {
    if (t < E) att_part[(int64_t)blockIdx.x * E + t] = 0.0;
    return;
  }
  float* al = alpha_scratch + (b - e0);
  float mx = -INFINITY;
  for (int64_t k = b + t; k < en; k += 128) {
    const float* m = msg + (k - e0) * HE;
    float s = 0.f;
    for (int c = 0; c < E; ++c) s = fmaf(att[c], m[c], s);
    al[k - b] = s;
    mx = fmaxf(mx, s);
  }
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((t & 31) == 0) sred[t >> 5] = mx;
  __syncthreads();
  mx = fmaxf(fmaxf(sred[0], sred[1]), fmaxf(sred[2], sred[3]));
  __syncthreads();
  float z = 0.f;
  for (int64_t k = b + t; k < en; k += 128) {
    const float a = expf(al[k - b] - mx);
    al[k - b] = a;
    z += a;
  }
  for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  if ((t & 31) == 0) sred[t >> 5] = z;
  __syncthreads();
  z = (sred[0] + sred[1]) + (sred[2] + sred[3]);
  __syncthreads();
  // dots (one warp per edge, fixed lane order), then mean
  const int w = t >> 5, lane = t & 31;
  for (int64_t k = b + w; k < en; k += 4) {
    const float* m = msg + (k - e0) * HE;
    float d = 0.f;
    for (int u = lane; u < HE; u += 32) d = fmaf(sg[u], m[u], d);
    for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane == 0) {
      const float a = al[k - b] / z;
      al[k - b] = a;                          // alpha
      g_msg[(k - e0) * HE] = d;               // dot parked in the row-0 slot until g_msg is written below
    }
  }
  __syncthreads();
  float mean = 0.f;
  if (t == 0)
    for (int64_t k = b; k < en; ++k) mean += al[k - b] * g_msg[(k - e0) * HE];
  if (t == 0) sred[0] = mean;
  __syncthreads();
  mean = sred[0];
  double aatt[E];
#pragma unroll
  for (int c = 0; c < E; ++c) aatt[c] = 0.0;
  for (int64_t k = b + w; k < en; k += 4) {
    const float a = al[k - b];
    const float dot = g_msg[(k - e0) * HE];
    const float dl = a * (dot - mean);
    const float* m = msg + (k - e0) * HE;
    float* gm = g_msg + (k - e0) * HE;
    __syncwarp();
    for (int u = lane; u < HE; u += 32) {
      float v = a * sg[u];
      if (u < E) v += dl * att[u];
      gm[u] = v;
    }
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < E; ++c) aatt[c] += double(dl) * double(m[c]);
  }
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < E; ++c) satt[w][c] = aatt[c];
  __syncthreads();
  if (t < E) att_part[(int64_t)blockIdx.x * E + t] = ((satt[0][t] + satt[1][t]) + satt[2][t]) + satt[3][t];
}

// halo backward helpers
__global__ void k_gather_rows(const float* __restrict__ src, const int* __restrict__ rows, int64_t n, int row,
                              float* __restrict__ dst) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n * row) dst[t] = src[(int64_t)rows[t / row] * row + t % row];
}
__global__ void k_add_rows(const float* __restrict__ src, const int* __restrict__ rows, int64_t n, int row,
                           float* __restrict__ dst) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n * row) dst[(int64_t)rows[t / row] * row + t % row] += src[t];
}

// lift backward (ops.h:52-60): S[c][g] = sum_e g_edges[e][0][c] rbf[e][g],
// CTA partials over edge ranges (fp64), radial features as the forward
template <int H, int E>
__global__ void __launch_bounds__(256) k_lift_bwd(const float* __restrict__ g_edges, const double* __restrict__ dist,
                                                  int64_t n_e, int ng, double spacing, double* __restrict__ part) {
  // tiles of 64 edges: the Gaussians rbf[k][g] (fp64 exp rounded to float,
  // as the forward lift) once per tile into SMEM, then thread (c, g) pairs
  // accumulate up * rbf over the tile in edge order (fp64)
  constexpr int TK = 64;
  __shared__ float s_rbf[TK * 32];
  __shared__ float s_up[TK * E];
  const int64_t per = (n_e + gridDim.x - 1) / gridDim.x;
  const int64_t k0 = blockIdx.x * per, k1 = k0 + per < n_e ? k0 + per : n_e;
  const double inv_den = 2.0 * spacing * spacing;
  double acc[(E * 32 + 255) / 256];
#pragma unroll
  for (int i = 0; i < (E * 32 + 255) / 256; ++i) acc[i] = 0.0;
  for (int64_t t0 = k0; t0 < k1; t0 += TK) {
    const int nk = (int)(k1 - t0 < TK ? k1 - t0 : TK);
    __syncthreads();
    for (int v = threadIdx.x; v < nk * ng; v += blockDim.x) {
      const int kk = v / ng, g = v % ng;
      const double d = dist[t0 + kk] - g * spacing;
      s_rbf[kk * 32 + g] = (float)exp(-d * d / inv_den);
    }
    for (int v = threadIdx.x; v < nk * E; v += blockDim.x) s_up[v] = g_edges[(t0 + v / E) * H * E + v % E];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < (E * 32 + 255) / 256; ++i) {
      const int u = threadIdx.x + 256 * i;
      if (u < E * ng) {
        const int c = u / ng, g = u % ng;
        for (int kk = 0; kk < nk; ++kk) {
          const float up = s_up[kk * E + c];
          if (up != 0.f) acc[i] += double(up) * double(s_rbf[kk * 32 + g]);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < (E * 32 + 255) / 256; ++i) {
    const int u = threadIdx.x + 256 * i;
    if (u < E * ng) part[(int64_t)blockIdx.x * E * ng + u] = acc[i];
  }
}

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

}  // namespace

// ======================================================================== host
void train_free(DeviceModel* D) {
  TrainState* T = D->train;
  if (!T) return;
  for (void* p : {(void*)T->node_target, (void*)T->node_mask, (void*)T->edge_target, (void*)T->edge_mask,
                  (void*)T->g_nodes, (void*)T->g_edges, (void*)T->g_nodes_out, (void*)T->A1,
                  (void*)T->Hh, (void*)T->Gg, (void*)T->Yy, (void*)T->msg, (void*)T->gY, (void*)T->gG, (void*)T->gH,
                  (void*)T->gA1, (void*)T->gx, (void*)T->gacc, (void*)T->part, (void*)T->plane_ptr,
                  (void*)T->plane_out, (void*)T->out_plane, (void*)T->out_key, (void*)T->rbf_scratch,
                  (void*)T->halo_send, (void*)T->halo_recv, (void*)T->tiles1, (void*)T->tiles2, (void*)T->opart,
                  (void*)T->adam_g})
    free_ptr(p);
  for (auto* v : {&T->src_perm, &T->src_off, &T->src_row_u})
    for (int* p : *v) free_ptr(p);
  for (float* p : D->saved_nodes) free_ptr(p);
  for (size_t l = 0; l < D->saved_edges.size(); ++l)
    if (!(l == 0 && D->saved_edges.size() > 1)) free_ptr(D->saved_edges[l]);  // [0] aliases [1]
  D->saved_nodes.clear();
  D->saved_edges.clear();
  for (auto& e : T->ev) cudaEventDestroy(e);
  delete T;
  D->train = nullptr;
}

// Targets in head space (view order), 1-byte masks.
void model_set_targets(esg_model* M, const float* node_target, const uint8_t* node_mask, const float* edge_target,
                       const uint8_t* edge_mask) {
  DeviceModel* D = M->dev;
  if (!D->prepared) usage("targets before prepare");
  if (!D->train) {
    D->train = new TrainState();
    for (auto& e : D->train->ev) ESG_CUDA(cudaEventCreate(&e));
  }
  TrainState* T = D->train;
  const int ol = M->heads.out_len;
  for (void* p : {(void*)T->node_target, (void*)T->node_mask, (void*)T->edge_target, (void*)T->edge_mask}) free_ptr(p);
  T->node_target = talloc<float>((size_t)D->n_owned * ol);
  T->node_mask = talloc<uint8_t>((size_t)D->n_owned * ol);
  T->edge_target = talloc<float>((size_t)D->n_edges * ol);
  T->edge_mask = talloc<uint8_t>((size_t)D->n_edges * ol);
  cudaStream_t st = M->ctx->stream;
  if (D->n_owned) {
    ESG_CUDA(cudaMemcpyAsync(T->node_target, node_target, sizeof(float) * D->n_owned * ol, cudaMemcpyHostToDevice, st));
    ESG_CUDA(cudaMemcpyAsync(T->node_mask, node_mask, (size_t)D->n_owned * ol, cudaMemcpyHostToDevice, st));
  }
  if (D->n_edges) {
    ESG_CUDA(cudaMemcpyAsync(T->edge_target, edge_target, sizeof(float) * D->n_edges * ol, cudaMemcpyHostToDevice, st));
    ESG_CUDA(cudaMemcpyAsync(T->edge_mask, edge_mask, (size_t)D->n_edges * ol, cudaMemcpyHostToDevice, st));
  }
  ESG_CUDA(cudaStreamSynchronize(st));
  T->tgt_owned = D->n_owned;
  T->tgt_edges = D->n_edges;
}

namespace {

// Sizes and offsets of the fp64 accumulators (expanded lin layout per block)
void gacc_layout(esg_model* M, TrainState* T) {
  const int L = M->cfg.l_max, E = M->cfg.e_width, layers = M->cfg.layers;
  int64_t o = 0;
  T->off_lin1.assign(2 * layers, 0);
  T->off_lin2.assign(2 * layers, 0);
  T->off_att.assign(layers, 0);
  for (int b = 0; b < 2 * layers; ++b) {
    T->off_lin1[b] = o;
    for (int m = 0; m <= L; ++m) {
      const int rows = m == 0 ? L + 1 : 2 * (L - m + 1);
      o += (int64_t)(rows * 2 * E) * (rows * 3 * E);
    }
    T->off_lin2[b] = o;
    for (int m = 0; m <= L; ++m) {
      const int rows = m == 0 ? L + 1 : 2 * (L - m + 1);
      o += (int64_t)(rows * E) * (rows * 2 * E);
    }
  }
  for (int l = 0; l < layers; ++l) {
    T->off_att[l] = o;
    o += E;
  }
  for (int s = 0; s < 2; ++s) {
    T->off_head[s] = o;
    o += (int64_t)M->heads.out_len * E;  // per output j (folded over r into keys on the host)
  }
  T->off_lift = o;
  o += (int64_t)E * M->cfg.n_radial;
  T->off_embed = o;
  o += (int64_t)M->species_list.size() * E;
  T->gacc_n = o;
}

void outer_tiles(esg_model* M, TrainState* T);

// (Re)builds everything that depends on the prepared view and the weights.
void train_setup(esg_model* M) {
  DeviceModel* D = M->dev;
  TrainState* T = D->train;
  const int L = M->cfg.l_max, E = M->cfg.e_width, H = (L + 1) * (L + 1), row = H * E;
  const int layers = M->cfg.layers;
  // saved tables
  if ((int)D->saved_nodes.size() != 2 * layers) {
    for (float* p : D->saved_nodes) free_ptr(p);
    for (size_t l = 0; l < D->saved_edges.size(); ++l)
      if (!(l == 0 && D->saved_edges.size() > 1)) free_ptr(D->saved_edges[l]);
    D->saved_nodes.assign(2 * layers, nullptr);
    D->saved_edges.assign(layers, nullptr);
  }
  for (auto& p : D->saved_nodes) {
    free_ptr(p);
    p = talloc<float>((size_t)std::max(D->n_rows, 1) * row);
  }
  // edge tables entering layers >= 1; layer 0's input is recomputed into
  // layer 1's buffer once layer 1's backward is done (one table fewer)
  for (int l = 0; l < layers; ++l) {
    if (l == 0 && layers > 1) continue;
    free_ptr(D->saved_edges[l]);
    D->saved_edges[l] = talloc<float>((size_t)std::max<int64_t>(D->n_edges, 1) * row);
  }
  if (layers > 1) D->saved_edges[0] = D->saved_edges[1];
  // gradient tables
  for (void* p : {(void*)T->g_nodes, (void*)T->g_edges, (void*)T->g_nodes_out}) free_ptr(p);
  T->g_nodes = talloc<float>((size_t)std::max(D->n_rows, 1) * row);
  T->g_nodes_out = talloc<float>((size_t)std::max(D->n_rows, 1) * row);
  T->g_edges = talloc<float>((size_t)std::max<int64_t>(D->n_edges, 1) * row);
  T->g_node_out = D->node_out;  // the loss seed overwrites the prediction (k_loss in place)
  T->g_edge_out = D->edge_out;
  // training chunks: destination-aligned, <= 256k edges (scratch ~ 6 KB/edge fp32)
  const int64_t cap0 = 256 * 1024;
  int64_t maxseg = 0;
  for (int j = 0; j < D->n_owned; ++j) maxseg = std::max(maxseg, D->h_seg[j + 1] - D->h_seg[j]);
  T->cap = std::max<int64_t>(std::min<int64_t>(std::max<int64_t>(D->n_edges, 1), cap0), maxseg);
  T->chunks.clear();
  for (int j = 0; j < D->n_owned;) {
    int j1 = j;
    while (j1 < D->n_owned && (j1 == j || D->h_seg[j1 + 1] - D->h_seg[j] <= T->cap)) ++j1;
    T->chunks.push_back({j, j1});
    j = j1;
  }
  for (void* p : {(void*)T->A1, (void*)T->Hh, (void*)T->Gg, (void*)T->Yy, (void*)T->msg, (void*)T->gY,
                  (void*)T->gG, (void*)T->gH, (void*)T->gA1, (void*)T->gx})
    free_ptr(p);
  const int K1T = H * 3 * E;  // fp32 A1 rows (KPAD 1): 25 rows x 3E
  const size_t cap = (size_t)round_up(T->cap, 32);
  T->A1 = talloc<float>(cap * K1T);
  T->Hh = talloc<float>(cap * H * 2 * E);
  T->Gg = talloc<float>(cap * H * 2 * E);
  T->Yy = talloc<float>(cap * row);
  T->msg = talloc<float>(cap * row);
  T->gY = talloc<float>(cap * row);
  T->gG = talloc<float>(cap * H * 2 * E);
  T->gH = talloc<float>(cap * H * 2 * E);
  T->gA1 = talloc<float>(cap * K1T);
  T->gx = talloc<float>(cap * 2 * row);
  // source-row reduction lists per chunk (stable sort of the chunk's edges by src row)
  for (auto* v : {&T->src_perm, &T->src_off, &T->src_row_u})
    for (int* p : *v) free_ptr(p);
  T->src_perm.clear();
  T->src_off.clear();
  T->src_row_u.clear();
  T->n_src.clear();
  std::vector<int> src(D->n_edges);
  if (D->n_edges) ESG_CUDA(cudaMemcpy(src.data(), D->src_row, sizeof(int) * D->n_edges, cudaMemcpyDeviceToHost));
  for (const auto& ch : T->chunks) {
    const int64_t e0 = D->h_seg[ch.first], e1 = D->h_seg[ch.second];
    std::vector<int> perm((size_t)(e1 - e0));
    for (int64_t k = e0; k < e1; ++k) perm[k - e0] = (int)(k - e0);
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return src[e0 + a] < src[e0 + b]; });
    std::vector<int> off{0}, rows;
    for (size_t q = 0; q < perm.size(); ++q) {
      if (q == 0 || src[e0 + perm[q]] != src[e0 + perm[q - 1]]) {
        if (q) off.push_back((int)q);
        rows.push_back(src[e0 + perm[q]]);
      }
    }
    off.push_back((int)perm.size());
    int* dp = talloc<int>(std::max<size_t>(perm.size(), 1));
    int* doff = talloc<int>(off.size());
    int* drow = talloc<int>(std::max<size_t>(rows.size(), 1));
    if (!perm.empty()) ESG_CUDA(cudaMemcpy(dp, perm.data(), sizeof(int) * perm.size(), cudaMemcpyHostToDevice));
    ESG_CUDA(cudaMemcpy(doff, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice));
    if (!rows.empty()) ESG_CUDA(cudaMemcpy(drow, rows.data(), sizeof(int) * rows.size(), cudaMemcpyHostToDevice));
    T->src_perm.push_back(dp);
    T->src_off.push_back(doff);
    T->src_row_u.push_back(drow);
    T->n_src.push_back((int)rows.size());
  }
  // head-output plane maps
  const int ol = M->heads.out_len;
  std::vector<int> out_plane(ol), out_key(ol), plane_ptr(H + 1, 0), plane_out;
  {
    int j = 0;
    for (size_t k = 0; k < M->heads.keys.size(); ++k)
      for (int r = 0; r < 2 * M->heads.keys[k].L + 1; ++r, ++j) {
        out_plane[j] = M->heads.keys[k].L * M->heads.keys[k].L + r;
        out_key[j] = (int)k;
      }
    for (int p = 0; p < H; ++p) {
      plane_ptr[p] = (int)plane_out.size();
      for (int q = 0; q < ol; ++q)
        if (out_plane[q] == p) plane_out.push_back(q);
    }
    plane_ptr[H] = (int)plane_out.size();
  }
  for (void* p : {(void*)T->plane_ptr, (void*)T->plane_out, (void*)T->out_plane, (void*)T->out_key}) free_ptr(p);
  T->plane_ptr = talloc<int>(H + 1);
  T->plane_out = talloc<int>(std::max<size_t>(plane_out.size(), 1));
  T->out_plane = talloc<int>(ol);
  T->out_key = talloc<int>(ol);
  ESG_CUDA(cudaMemcpy(T->plane_ptr, plane_ptr.data(), sizeof(int) * (H + 1), cudaMemcpyHostToDevice));
  if (!plane_out.empty())
    ESG_CUDA(cudaMemcpy(T->plane_out, plane_out.data(), sizeof(int) * plane_out.size(), cudaMemcpyHostToDevice));
  ESG_CUDA(cudaMemcpy(T->out_plane, out_plane.data(), sizeof(int) * ol, cudaMemcpyHostToDevice));
  ESG_CUDA(cudaMemcpy(T->out_key, out_key.data(), sizeof(int) * ol, cudaMemcpyHostToDevice));
  // accumulators and partials
  gacc_layout(M, T);
  outer_tiles(M, T);
  free_ptr(T->gacc);
  T->gacc = talloc<double>(T->gacc_n);
  free_ptr(T->part);
  T->part_n = std::max<int64_t>({(int64_t)296 * ol * E, (int64_t)296 * E * M->cfg.n_radial,
                                 (int64_t)std::max(D->n_owned, 1) * E, 4096});
  T->part = talloc<double>(T->part_n);
  free_ptr(T->rbf_scratch);
  T->rbf_scratch = talloc<float>(cap);  // alpha scratch of the attention backward
  // halo backward buffers
  int64_t halo_rows = 0, send_rows = 0;
  for (const auto& nb : D->nbrs) {
    halo_rows += nb.recv_count;
    send_rows += (int64_t)nb.send_rows.size();
  }
  free_ptr(T->halo_send);
  free_ptr(T->halo_recv);
  T->halo_send = talloc<float>((size_t)std::max<int64_t>(halo_rows, 1) * row);
  T->halo_recv = talloc<float>((size_t)std::max<int64_t>(send_rows, 1) * row);
}




// kind 0: lin1 forward (3E -> 2E, P = W1^T), 1: lin2 forward (2E -> E, W2^T),
// 2: lin2 dx (E -> 2E, P = W2), 3: lin1 dx (2E -> 3E, P = W1)
template <int L, int E>
void lin(int kind, const float* in, int64_t n, const float* P, float* out, int b, DeviceModel* D, cudaStream_t st) {
  constexpr int H = (L + 1) * (L + 1), cin_of[4] = {3 * E, 2 * E, E, 2 * E}, cout_of[4] = {2 * E, E, 2 * E, 3 * E};
  if (D->tf32)
    tf32_gemm_launch(in, (int64_t)H * cin_of[kind], n, D->wtc[kind][b], D->tct[kind], D->n_tct[kind], out,
                     (int64_t)H * cout_of[kind], st);
  else
    lin_launch<L, E>(kind, in, n, P, out, D->lt[kind], D->n_lt[kind], st);
}

// edges per split of a weight-gradient tile (dw_tc.cu).  The tensor cores'
// fp32 accumulation is biased: the dW error grows linearly with the number
// of MMAs accumulated (measured on the smoke problem: gradient rel-L2 4.6e-6
// at 256 edges per split, 6.5e-6 at 512, 1.0e-5 at 1,024, 2.6e-5 at 4,096),
// so the splits stay short and are added in fp64 (ESG_DW_SPLIT overrides)
int dw_split() {
  static const int v = [] {
    const char* e = std::getenv("ESG_DW_SPLIT");
    const int x = e ? std::atoi(e) : 512;
    return x >= 16 ? x / 16 * 16 : 16;
  }();
  return v;
}

// dWexp_m += g_m^T x_m over the chunk's edges on the tensor cores (dw_tc.cu)
// (gscale: x is the pre-gate hidden h, each channel scaled by its edge's gate)
template <int L>
void outer(const float* g, int cg, const float* x, int cx, int64_t n, double* acc, bool lin1, TrainState* T,
           cudaStream_t st, const float* gscale = nullptr) {
  constexpr int H = (L + 1) * (L + 1);
  dw_tf32x3_launch(g, (int64_t)H * cg, x, (int64_t)H * cx, n, lin1 ? T->tiles1 : T->tiles2,
                   lin1 ? T->n_tiles1 : T->n_tiles2, dw_split(), T->opart, acc, st, gscale, cx);
}

// tile lists of the two dW products and their partial-tile scratch
void outer_tiles(esg_model* M, TrainState* T) {
  const int L = M->cfg.l_max, E = M->cfg.e_width;
  for (int which = 0; which < 2; ++which) {
    std::vector<DwTile> v;
    dw_tiles(L, E, which, &v);
    DwTile*& dst = which == 0 ? T->tiles1 : T->tiles2;
    free_ptr(dst);
    dst = talloc<DwTile>(v.size());
    ESG_CUDA(cudaMemcpy(dst, v.data(), sizeof(DwTile) * v.size(), cudaMemcpyHostToDevice));
    (which == 0 ? T->n_tiles1 : T->n_tiles2) = (int)v.size();
  }
  free_ptr(T->opart);
  T->opart_n = dw_part_floats(std::max(T->n_tiles1, T->n_tiles2), (int)((T->cap + dw_split() - 1) / dw_split()));
  T->opart = talloc<float>(T->opart_n);
}

// reverse of the forward's exchange: halo-row gradients go back to their
// owners, are added into the owners' send rows (ascending peer order), and
// the halo rows are zeroed (distributed.h:98-129)
void halo_backward(esg_model* M, int row) {
  DeviceModel* D = M->dev;
  TrainState* T = D->train;
  esg_ctx* ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  if (ctx->world <= 1 || D->nbrs.empty()) return;
  int64_t ho = 0;
  for (const auto& nb : D->nbrs) {
    if (nb.recv_count)
      ESG_CUDA(cudaMemcpyAsync(T->halo_send + ho * row, T->g_nodes + (int64_t)nb.recv_row * row,
                               sizeof(float) * nb.recv_count * row, cudaMemcpyDeviceToDevice, st));
    ho += nb.recv_count;
  }
  ESG_NCCL(ncclGroupStart());
  ho = 0;
  int64_t so = 0;
  for (const auto& nb : D->nbrs) {
    ESG_NCCL(ncclSend(T->halo_send + ho * row, (size_t)nb.recv_count * row, ncclFloat, nb.peer, ctx->comm, st));
    ESG_NCCL(ncclRecv(T->halo_recv + so * row, nb.send_rows.size() * row, ncclFloat, nb.peer, ctx->comm, st));
    ho += nb.recv_count;
    so += (int64_t)nb.send_rows.size();
  }
  ESG_NCCL(ncclGroupEnd());
  so = 0;
  int64_t send_base = 0;
  for (const auto& nb : D->nbrs) {  // ascending peer order (the plan's order)
    const int64_t n = (int64_t)nb.send_rows.size();
    if (n)
      k_add_rows<<<(unsigned)((n * row + 255) / 256), 256, 0, st>>>(T->halo_recv + so * row,
                                                                    D->send_rows + send_base, n, row, T->g_nodes);
    so += n;
    send_base += n;
    if (nb.recv_count)
      ESG_CUDA(cudaMemsetAsync(T->g_nodes + (int64_t)nb.recv_row * row, 0, sizeof(float) * nb.recv_count * row, st));
  }
}

template <int L, int E>
void block_backward(esg_model* M, int layer, bool node_block) {
  DeviceModel* D = M->dev;
  TrainState* T = D->train;
  cudaStream_t st = M->ctx->stream;
  using G = Geo<L>;
  constexpr int H = G::H, HE = H * E;
  const int b = 2 * layer + (node_block ? 0 : 1);
  const float* nodes = D->saved_nodes[b];
  const float* edges = D->saved_edges[layer];
  const float* att = D->params + D->att_off[layer];
  if (node_block)  // the attention backward reads the block's output gradient, untouched by this block's updates
    ESG_CUDA(cudaMemcpyAsync(T->g_nodes_out, T->g_nodes, sizeof(float) * (size_t)D->n_rows * HE,
                             cudaMemcpyDeviceToDevice, st));
  for (size_t ci = 0; ci < T->chunks.size(); ++ci) {
    const auto& ch = T->chunks[ci];
    const int64_t e0 = D->h_seg[ch.first], e1 = D->h_seg[ch.second], n = e1 - e0;
    if (n <= 0) continue;
    const unsigned t32 = (unsigned)((n + 31) / 32);
    constexpr int RI_THREADS = 32 * 3 * E / 4 < 128 ? 128 : 32 * 3 * E / 4;
    // forward recompute: A1, H, G (+ Y and msg for the attention backward)
    k_rotate_in<L, E, 1, float><<<t32, RI_THREADS, 0, st>>>(nodes, edges, D->src_row, D->dst_row, D->dir, e0, n, T->A1,
                                                            D->prefetch, 0);
    lin<L, E>(0, T->A1, n, D->w1t[b], T->Hh, b, D, st);
    // the gated hidden G: materialised only on the CUDA-core path; the tensor
    // cores gate h on the fly in lin2's and dW2's operand loads
    const bool gate_fused = D->tf32;
    const int gc2 = gate_fused && M->cfg.gate_enabled ? 2 * E : 0;
    const float* Gx = gate_fused ? T->Hh : T->Gg;
    if (!gate_fused)
      k_gate_fwd<H><<<(unsigned)((n * 2 * E + 255) / 256), 256, 0, st>>>(T->Hh, 2 * E, n, M->cfg.gate_enabled, T->Gg);
    else if (gc2)  // the gate scalars sigmoid(h[row 0]) per edge (2E floats) for dW2's operand
      k_gate_scale<<<(unsigned)((n * 2 * E + 255) / 256), 256, 0, st>>>(T->Hh, (int64_t)H * 2 * E, 2 * E, n, T->Gg);
    const float* g_msg;
    if (node_block) {
      if (gate_fused)
        tf32_gemm_launch(T->Hh, (int64_t)H * 2 * E, n, D->wtc[1][b], D->tct[1], D->n_tct[1], T->Yy, (int64_t)H * E, st,
                         gc2);
      else
        lin<L, E>(1, T->Gg, n, D->w2t[b], T->Yy, b, D, st);
      k_rot1<L, E, 0><<<t32, 128, 0, st>>>(T->Yy, D->dir, e0, n, T->msg);
      // attention backward into gY's buffer (used as g_msg scratch)
      k_attn_bwd<H, E><<<(unsigned)(ch.second - ch.first), 128, 0, st>>>(
          T->msg, att, D->seg, ch.first, e0, T->g_nodes_out, T->gG /* g_msg, n x HE fits */, T->rbf_scratch,
          T->part);
      k_reduce_parts<<<1, E, 0, st>>>(T->part, ch.second - ch.first, E, T->gacc + T->off_att[layer]);
      g_msg = T->gG;
    } else {
      g_msg = T->g_edges + e0 * HE;  // add (ops.h:273-281): the update's gradient
    }
    k_rot1<L, E, 1><<<t32, 128, 0, st>>>(g_msg, D->dir, e0, n, T->gY);
    // lin2 adjoint
    outer<L>(T->gY, E, Gx, 2 * E, n, T->gacc + T->off_lin2[b], false, T, st, gc2 ? T->Gg : nullptr);
    lin<L, E>(2, T->gY, n, D->w2n[b], T->gG, b, D, st);
    k_gate_bwd<H><<<(unsigned)((n * 2 * E + 255) / 256), 256, 0, st>>>(T->Hh, T->gG, 2 * E, n, M->cfg.gate_enabled,
                                                                       T->gH);
    // lin1 adjoint
    outer<L>(T->gH, 2 * E, T->A1, 3 * E, n, T->gacc + T->off_lin1[b], true, T, st);
    lin<L, E>(3, T->gH, n, D->w1n[b], T->gA1, b, D, st);
    // rotate-in / concat adjoint, ordered row reductions
    k_rot_in_bwd<L, E><<<t32, RI_THREADS, 0, st>>>(T->gA1, D->dir, e0, n, T->g_edges, T->gx);
    k_dst_reduce<<<(unsigned)(ch.second - ch.first), 128, 0, st>>>(T->gx, HE, D->seg, ch.first, e0, T->g_nodes);
    if (T->n_src[ci])
      k_src_reduce<<<(unsigned)T->n_src[ci], 128, 0, st>>>(T->gx, HE, T->src_perm[ci], T->src_off[ci],
                                                            T->src_row_u[ci], T->g_nodes);
  }
  ESG_CUDA(cudaGetLastError());
}

}  // namespace

void model_forward(esg_model* M, esg_timing* tm);               // model.cu
void model_init_edges(esg_model* M, float* out, cudaStream_t st);  // model.cu

// ops.h:347-371 + the reverse pass + distributed.h:147-163: loss partials of
// this rank, the global loss and the parameter gradients summed over ranks
// (rank order, fp64) in the flat parameter layout.
template <int L, int E>
void loss_grad_impl(esg_model* M, int64_t n_total, double partials[3], double* loss, float* grads_out) {
  DeviceModel* D = M->dev;
  TrainState* T = D->train;
  esg_ctx* ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  using G = Geo<L>;
  constexpr int H = G::H, HE = H * E;
  if (!T || T->tgt_owned != D->n_owned || T->tgt_edges != D->n_edges) usage("targets not set for this view");
  if (n_total <= 0) data("no target elements overlap the predictions");
  // forward on the fp32 path, block inputs saved
  const int prec = M->cfg.linear_precision;
  M->cfg.linear_precision = ESG_LINEAR_FP32;
  D->save_inputs = true;
  esg_timing tf{};
  model_forward(M, &tf);
  D->save_inputs = false;
  M->cfg.linear_precision = prec;
  T->last_forward_ms = tf.forward_ms;
  ESG_CUDA(cudaEventRecord(T->ev[0], st));
  // loss and seeds
  const int ol = M->heads.out_len;
  const double inv_total = 1.0 / double(n_total);
  double sums[3] = {0, 0, 0};
  auto loss_part = [&](const float* pred, const float* tgt, const uint8_t* mask, int64_t n, float* g_out) {
    if (n <= 0) return;
    const int blocks = sm_count() * 8;  // latency-bound: 8 CTAs per SM; partials summed on the host in block order
    k_loss<<<blocks, 256, 0, st>>>(pred, tgt, mask, n, inv_total, g_out, T->part);
    std::vector<double> h(blocks * 3);
    ESG_CUDA(cudaMemcpyAsync(h.data(), T->part, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
    ESG_CUDA(cudaStreamSynchronize(st));
    for (int q = 0; q < blocks; ++q)
      for (int t = 0; t < 3; ++t) sums[t] += h[q * 3 + t];
  };
  ESG_CUDA(cudaMemsetAsync(T->gacc, 0, sizeof(double) * T->gacc_n, st));
  ESG_CUDA(cudaMemsetAsync(T->g_nodes, 0, sizeof(float) * (size_t)D->n_rows * HE, st));
  if (D->n_edges) ESG_CUDA(cudaMemsetAsync(T->g_edges, 0, sizeof(float) * (size_t)D->n_edges * HE, st));
  loss_part(D->node_out, T->node_target, T->node_mask, (int64_t)D->n_owned * ol, T->g_node_out);
  loss_part(D->edge_out, T->edge_target, T->edge_mask, D->n_edges * ol, T->g_edge_out);
  partials[0] = sums[0];
  partials[1] = sums[1];
  partials[2] = sums[2];
  // heads backward (final tables are D->nodes / D->edges)
  auto heads_bwd = [&](int set, const float* x, int64_t n_items, const float* g_out, float* g_x) {
    if (n_items <= 0) return;
    k_heads_bwd_x<H, E><<<(unsigned)((n_items * HE / 4 + 255) / 256), 256, 0, st>>>(
        g_out, ol, n_items, D->head_w[set], T->plane_ptr, T->plane_out, T->out_key, g_x);
    const int parts = (int)std::min<int64_t>(296, n_items);
    k_heads_bwd_w<H, E><<<parts, 256, 0, st>>>(g_out, ol, n_items, x, T->out_plane, T->part);
    k_reduce_parts<<<(unsigned)((ol * E + 255) / 256), 256, 0, st>>>(T->part, parts, (int64_t)ol * E,
                                                                     T->gacc + T->off_head[set]);
  };
  heads_bwd(0, D->nodes, D->n_owned, T->g_node_out, T->g_nodes);
  heads_bwd(1, D->edges, D->n_edges, T->g_edge_out, T->g_edges);
  // blocks in reverse; each block's exchange is undone after its backward
  for (int layer = M->cfg.layers - 1; layer >= 0; --layer)
    for (bool nb : {false, true}) {
      if (layer == 0 && !nb && M->cfg.layers > 1) model_init_edges(M, D->saved_edges[0], st);  // E_0 into E_1's buffer
      if (nb)
        block_backward<L, E>(M, layer, true);
      else
        block_backward<L, E>(M, layer, false);
      halo_backward(M, HE);
    }
  // embed (ops.h:27-33) and lift (ops.h:52-60)
  if (D->n_edges) {
    const int parts = (int)std::min<int64_t>(296, D->n_edges);
    k_lift_bwd<H, E><<<parts, 256, 0, st>>>(T->g_edges, D->dist, D->n_edges, M->cfg.n_radial,
                                            M->cfg.r_cut / (M->cfg.n_radial - 1), T->part);
    k_reduce_parts<<<(unsigned)((E * M->cfg.n_radial + 255) / 256), 256, 0, st>>>(
        T->part, parts, (int64_t)E * M->cfg.n_radial, T->gacc + T->off_lift);
  }
  std::vector<float> gn0((size_t)D->n_rows * E);
  {
    std::vector<float> gn((size_t)D->n_rows * HE);
    ESG_CUDA(cudaMemcpyAsync(gn.data(), T->g_nodes, sizeof(float) * gn.size(), cudaMemcpyDeviceToHost, st));
    ESG_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < D->n_rows; ++i)
      for (int c = 0; c < E; ++c) gn0[(size_t)i * E + c] = gn[(size_t)i * HE + c];
  }
  std::vector<double> acc(T->gacc_n);
  ESG_CUDA(cudaMemcpyAsync(acc.data(), T->gacc, sizeof(double) * T->gacc_n, cudaMemcpyDeviceToHost, st));
  ESG_CUDA(cudaEventRecord(T->ev[1], st));
  ESG_CUDA(cudaStreamSynchronize(st));
  float bms = 0.f;
  ESG_CUDA(cudaEventElapsedTime(&bms, T->ev[0], T->ev[1]));
  T->last_backward_ms = bms;
  for (int i = 0; i < D->n_rows; ++i) {  // embed: rows in order
    const int slot = int(std::find(M->species_list.begin(), M->species_list.end(), D->row_species[i]) -
                         M->species_list.begin());
    for (int c = 0; c < E; ++c) acc[T->off_embed + (int64_t)slot * E + c] += gn0[(size_t)i * E + c];
  }
  // fold the expanded accumulators into the flat parameter layout (fp64)
  std::vector<double> g((size_t)M->params.total, 0.0);
  auto P = [&](const std::string& name) { return g.data() + M->params.at(name).offset; };
  for (int layer = 0; layer < M->cfg.layers; ++layer)
    for (int bi = 0; bi < 2; ++bi) {
      const int b = 2 * layer + bi;
      const std::string base = "layer" + std::to_string(layer) + (bi == 0 ? "/node" : "/edge");
      for (int lin_i = 0; lin_i < 2; ++lin_i) {
        const int cin = lin_i == 0 ? 3 * E : 2 * E, cout = lin_i == 0 ? 2 * E : E;
        const double* a = acc.data() + (lin_i == 0 ? T->off_lin1[b] : T->off_lin2[b]);
        const std::string wb = base + (lin_i == 0 ? "/lin1" : "/lin2");
        for (int m = 0; m <= L; ++m) {
          const int nd = L - m + 1;
          if (m == 0) {
            const int R = nd * cout, C = nd * cin;
            double* d0 = P(wb + "/m0");
            for (int t = 0; t < R * C; ++t) d0[t] += a[t];
            a += (int64_t)R * C;
            continue;
          }
          const int R = nd * cout, C = nd * cin;  // expanded is 2R x 2C
          double* dr = P(wb + "/m" + std::to_string(m) + "r");
          double* di = P(wb + "/m" + std::to_string(m) + "i");
          for (int o = 0; o < R; ++o)
            for (int k = 0; k < C; ++k) {
              const double a00 = a[(int64_t)o * 2 * C + k], a01 = a[(int64_t)o * 2 * C + C + k];
              const double a10 = a[(int64_t)(R + o) * 2 * C + k], a11 = a[(int64_t)(R + o) * 2 * C + C + k];
              dr[(int64_t)o * C + k] += a00 + a11;  // gm xm^T + gp xp^T
              di[(int64_t)o * C + k] += a01 - a10;  // gm xp^T - gp xm^T
            }
          a += (int64_t)4 * R * C;
        }
      }
      (void)b;
    }
  for (int layer = 0; layer < M->cfg.layers; ++layer) {
    double* d = P("layer" + std::to_string(layer) + "/att");
    for (int c = 0; c < E; ++c) d[c] += acc[T->off_att[layer] + c];
  }
  for (int s = 0; s < 2; ++s) {
    int j = 0;
    for (const auto& k : M->heads.keys) {
      double* d = P(std::string("head/") + (s == 0 ? "node" : "edge") + "/s" + std::to_string(k.sa) + "s" +
                    std::to_string(k.sb) + "L" + std::to_string(k.L));
      for (int r = 0; r < 2 * k.L + 1; ++r, ++j)
        for (int c = 0; c < E; ++c) d[c] += acc[T->off_head[s] + (int64_t)j * E + c];
    }
  }
  {
    double* d = P("radial/lift");
    for (int t = 0; t < E * M->cfg.n_radial; ++t) d[t] += acc[T->off_lift + t];
  }
  for (size_t s = 0; s < M->species_list.size(); ++s) {
    double* d = P("embed/" + element_symbol(M->species_list[s]));
    for (int c = 0; c < E; ++c) d[c] += acc[T->off_embed + (int64_t)s * E + c];
  }
  // rank sums: loss partials and gradients (allgather, rank order, fp64)
  double tot[3] = {partials[0], partials[1], partials[2]};
  if (ctx->world > 1) {
    const int W = ctx->world;
    const size_t n = g.size() + 3;
    double *d_mine = nullptr, *d_all = nullptr;
    ESG_CUDA(cudaMalloc(&d_mine, sizeof(double) * n));
    ESG_CUDA(cudaMalloc(&d_all, sizeof(double) * n * W));
    std::vector<double> mine(n);
    std::copy(g.begin(), g.end(), mine.begin());
    mine[g.size()] = partials[0];
    mine[g.size() + 1] = partials[1];
    mine[g.size() + 2] = partials[2];
    ESG_CUDA(cudaMemcpyAsync(d_mine, mine.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    ESG_NCCL(ncclAllGather(d_mine, d_all, n, ncclDouble, ctx->comm, st));
    std::vector<double> all(n * W);
    ESG_CUDA(cudaMemcpyAsync(all.data(), d_all, sizeof(double) * n * W, cudaMemcpyDeviceToHost, st));
    ESG_CUDA(cudaStreamSynchronize(st));
    free_ptr(d_mine);
    free_ptr(d_all);
    for (size_t k = 0; k < n; ++k) {
      double s = 0.0;
      for (int p = 0; p < W; ++p) s += all[(size_t)p * n + k];
      if (k < g.size())
        g[k] = s;
      else
        tot[k - g.size()] = s;
    }
  }
  if ((int64_t)tot[2] != n_total)
    data("target count mismatch: " + std::to_string((int64_t)tot[2]) + " vs " + std::to_string(n_total));
  *loss = (tot[0] + tot[1]) / double(n_total);
  if (grads_out)
    for (size_t k = 0; k < g.size(); ++k) grads_out[k] = (float)g[k];
}

void model_loss_grad(esg_model* M, int64_t n_total, double partials[3], double* loss, float* grads_out) {
  DeviceModel* D = M->dev;
  if (!D->prepared) usage("loss before prepare");
  if (!D->train) usage("targets not set");
  TrainState* T = D->train;
  const int L = D->L, E = D->E;
  if (D->train_stale) {  // a new view was prepared since the last setup
    train_setup(M);
    D->train_stale = false;
  }
  if (L == 4 && E == 16)
    loss_grad_impl<4, 16>(M, n_total, partials, loss, grads_out);
  else if (L == 4 && E == 8)
    loss_grad_impl<4, 8>(M, n_total, partials, loss, grads_out);
  else if (L == 2 && E == 16)
    loss_grad_impl<2, 16>(M, n_total, partials, loss, grads_out);
  else
    loss_grad_impl<2, 8>(M, n_total, partials, loss, grads_out);
}

void model_train_timing(const esg_model* M, double* fwd_ms, double* bwd_ms) {
  const TrainState* T = M->dev->train;
  *fwd_ms = T ? T->last_forward_ms : 0.0;
  *bwd_ms = T ? T->last_backward_ms : 0.0;
}

}  // namespace esg

namespace esg {
namespace {
// Optimizer::step (optimizer.h:42-59) per parameter, moments in fp64, the
// host expression order with explicit round-to-nearest operations (no FMA
// contraction), so the new parameters equal the host Adam's bit for bit.
__global__ void k_adam(float* __restrict__ p, const float* __restrict__ g, double* __restrict__ m,
                       double* __restrict__ v, int64_t n, double b1, double omb1, double b2, double omb2, double lr,
                       double bc1, double bc2, double eps) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double gk = (double)g[k];
  const double mk = __dadd_rn(__dmul_rn(b1, m[k]), __dmul_rn(omb1, gk));
  const double vk = __dadd_rn(__dmul_rn(b2, v[k]), __dmul_rn(__dmul_rn(omb2, gk), gk));
  m[k] = mk;
  v[k] = vk;
  const double mh = __ddiv_rn(mk, bc1), vh = __ddiv_rn(vk, bc2);
  const double step = __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), eps));
  p[k] = __double2float_rn(__dadd_rn((double)p[k], -step));
}
}  // namespace

void model_repack_params(esg_model* M);  // model.cu

// The Adam step on the device: gradients (host, float) in, moments stay in
// device memory, the parameters are updated in D->params and repacked there;
// the host copy is refreshed for the parameter hash and checkpoints.
void model_adam_device(esg_model* M, double* d_m, double* d_v, const float* grads, double b1, double b2, double lr,
                       double bc1, double bc2, double eps) {
  DeviceModel* D = M->dev;
  cudaStream_t st = M->ctx->stream;
  const int64_t n = (int64_t)M->host_params.size();
  TrainState* T = D->train;
  float* g = nullptr;
  if (T) {
    if (T->adam_g_n < n) {
      free_ptr(T->adam_g);
      T->adam_g = talloc<float>(n);
      T->adam_g_n = n;
    }
    g = T->adam_g;
  } else {
    ESG_CUDA(cudaMalloc(&g, sizeof(float) * n));
  }
  h2d_staged(M->ctx, g, grads, sizeof(float) * n);
  k_adam<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(D->params, g, d_m, d_v, n, b1, 1.0 - b1, b2, 1.0 - b2, lr, bc1,
                                                       bc2, eps);
  ++M->ctx->launches;
  ESG_CUDA(cudaGetLastError());
  // the host mirror first: the embedding and head tables are packed from it
  ESG_CUDA(cudaMemcpyAsync(M->host_params.data(), D->params, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
  ESG_CUDA(cudaStreamSynchronize(st));
  model_repack_params(M);
  if (!T) cudaFree(g);
}
}  // namespace esg
