// lin_kernels.cuh -- the per-order SO(2) linears on the CUDA cores as a
// register-blocked SGEMM (fp32 forward path and the training reverse pass)
// and the gate (kernels.h:210-226).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "model_kernels.cuh"

namespace esg {

// one 64-output tile of an order block of a per-order linear (k_gemm_m)
struct LinTile {
  int m, o0, K, N;
  int64_t p_off;  // offset of P_m
};

// The per-order linear as a register-blocked SGEMM: CTA tile of 128 edges x
// 64 outputs of one order block (tile list: (m, o0)), 16-deep K stages in
// SMEM, thread (ty, tx) owns 8 edges x 4 outputs (16-byte SMEM loads).  Each output sums its K
// terms in ascending order with fmaf.
template <int L>
__global__ void __launch_bounds__(256) k_gemm_m(const float* __restrict__ in, int cin, int64_t n_e,
                                                const float* __restrict__ P, const LinTile* __restrict__ tiles, int cout,
                                                float* __restrict__ out) {
  using G = Geo<L>;
  constexpr int TM = 128, TK = 16;
  __shared__ __align__(16) float As[TK][TM + 4];
  __shared__ __align__(16) float Bs[TK][64];
  const LinTile t = tiles[blockIdx.y];
  const int64_t e0 = (int64_t)blockIdx.x * TM;
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;  // thread: edges ty*8 .. +7, outputs tx*4 .. +3
  const int io = G::moff(t.m) * cin, oo = G::moff(t.m) * cout;
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < t.K; k0 += TK) {
    __syncthreads();
    for (int u = threadIdx.x; u < TM * TK; u += 256) {  // A: 128 edges x 16 k (edge rows contiguous in k)
      const int e = u / TK, k = u % TK;
      const int64_t ee = e0 + e;
      As[k][e] = (ee < n_e && k0 + k < t.K) ? in[ee * G::H * cin + io + k0 + k] : 0.f;
    }
    for (int u = threadIdx.x; u < TK * 64; u += 256) {  // B: 16 k x 64 outputs
      const int k = u / 64, o = u % 64;
      Bs[k][o] = (k0 + k < t.K && t.o0 + o < t.N) ? P[t.p_off + (int64_t)(k0 + k) * t.N + t.o0 + o] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < TK; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[k][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[k][ty * 8 + 4]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t ee = e0 + ty * 8 + i;
    if (ee >= n_e) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int o = t.o0 + tx * 4 + j;
      if (o < t.N) out[ee * G::H * cout + oo + o] = acc[i][j];
    }
  }
}


// gate (kernels.h:210-226): rows are the 25 order-major rows of 2E channels,
// row 0 the l = 0 scalar; in place is allowed (each thread reads its own
// channel's row 0 before writing)
template <int H>
__global__ void k_gate_fwd(const float* h, int c2, int64_t n_e, int enabled, float* g) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_e * c2) return;
  const int64_t e = t / c2;
  const int c = (int)(t % c2);
  const float* hr = h + e * H * c2;
  float* gr = g + e * H * c2;
  const float s = enabled ? 1.f / (1.f + expf(-hr[c])) : 1.f;
  for (int r = 0; r < H; ++r) gr[r * c2 + c] = hr[r * c2 + c] * s;
}


// kind 0: lin1 forward (3E -> 2E, P = W1^T), 1: lin2 forward (2E -> E, W2^T),
// 2: lin2 dx (E -> 2E, P = W2), 3: lin1 dx (2E -> 3E, P = W1); tiles from
// lin_tile_list
template <int L, int E>
void lin_launch(int kind, const float* in, int64_t n, const float* P, float* out, const LinTile* tiles, int n_tiles,
                cudaStream_t st) {
  constexpr int cin_of[4] = {3 * E, 2 * E, E, 2 * E}, cout_of[4] = {2 * E, E, 2 * E, 3 * E};
  if (n > 0)
    k_gemm_m<L><<<dim3((unsigned)((n + 127) / 128), (unsigned)n_tiles), 256, 0, st>>>(in, cin_of[kind], n, P, tiles,
                                                                                  cout_of[kind], out);
}

}  // namespace esg
