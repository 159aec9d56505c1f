// model_kernels.cuh -- device building blocks shared by the message kernels.
//
// Index conventions (all follow the reference):
//   degree-major component h = l*l + l + a, a = m in -l..l   (real_sh.h:20)
//   order-major row r' = mrow(L, l, a)                       (layout.h:28-45)
//   node / edge feature rows: H x E fp32, channel fastest     (tensor.h:14)
//   A1 (aligned, order-major message) per edge: K1TOT values, m-block m at
//   kofs(m), inside it the -m rows then the +m rows (l = m..L), 3E channels
//   each ([src | dst | edge], ops.h:74-85), m-blocks padded to KPAD.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace esg {

template <int L>
struct Geo {
  static constexpr int H = (L + 1) * (L + 1);
  // stacked Wigner blocks: block l at doff(l), (2l+1)^2 row-major
  __host__ __device__ static constexpr int doff(int l) { return l * (4 * l * l - 1) / 3; }
  static constexpr int DS = doff(L + 1);
  __host__ __device__ static constexpr int nd(int m) { return L - m + 1; }
  __host__ __device__ static constexpr int rows(int m) { return m == 0 ? nd(0) : 2 * nd(m); }
  // order-major start row of order m (MMajorLayout::m_offset)
  __host__ __device__ static constexpr int moff(int m) { return m == 0 ? 0 : (L + 1) + (m - 1) * (2 * L + 2 - m); }
  __host__ __device__ static constexpr int mrow(int l, int a) {
    return a == 0 ? l : moff(a < 0 ? -a : a) + (a < 0 ? 0 : nd(a < 0 ? -a : a)) + (l - (a < 0 ? -a : a));
  }
};

template <int L, int E, int KPAD>
struct Lay1 {
  static constexpr int C3 = 3 * E;
  __host__ __device__ static constexpr int pad(int x) { return (x + KPAD - 1) / KPAD * KPAD; }
  __host__ __device__ static constexpr int K(int m) { return Geo<L>::rows(m) * C3; }  // lin1 K per order
  __host__ __device__ static constexpr int KP(int m) { return pad(K(m)); }
  __host__ __device__ static constexpr int kofs(int m) {
    int s = 0;
    for (int q = 0; q < m; ++q) s += KP(q);
    return s;
  }
  static constexpr int KTOT = kofs(L + 1);
  __host__ __device__ static constexpr int N1(int m) { return Geo<L>::rows(m) * 2 * E; }  // lin1 N == lin2 K
  __host__ __device__ static constexpr int N1P(int m) { return pad(N1(m)); }
  __host__ __device__ static constexpr int N2(int m) { return Geo<L>::rows(m) * E; }      // lin2 N
};


// Power-of-two scale of an fp16x3 split operand (so2_f16x3.cu) whose values
// are bounded by `bound`: every |x| / s stays below 2^14 (fp16 max 65504).
// rotate_in (the A1 image) and the chain evaluate it from the same bound.
__device__ __forceinline__ float f16s_pow2_scale(float bound) {
  if (!(bound > 0.f) || !(bound < 3.0e38f)) return 1.f;
  int k;
  frexpf(bound, &k);  // bound < 2^k
  return ldexpf(1.f, k - 14);
}

// Rotation taking the unit edge direction onto +y: R = Rx(-beta) Ry(-alpha)
// with alpha = atan2(ux, uz), beta = acos(uy) (align.cpp:32-39), written with
// cos/sin of alpha and beta taken directly from the displacement (no trig
// calls).  sin(beta) is the lateral length rho / |d|, not sqrt(1 - uy^2):
// the latter cancels for edges near the +-y axis (4.8e-4 absolute error at
// 0.1 A lateral offset against the reference's fp64 acos/sin; rho keeps every
// entry within a few ulp).
__device__ __forceinline__ void align_to_y(float x, float y, float z, float R[9]) {
  const float rxz2 = x * x + z * z;
  const float inv = rsqrtf(rxz2 + y * y);
  const float rho = sqrtf(rxz2);
  // on the axis atan2(+-0, z) is 0 for z = +0 and +-pi for z = -0
  float ca = signbit(z) ? -1.f : 1.f, sa = 0.f;
  if (rho > 0.f) {
    ca = z / rho;
    sa = x / rho;
  }
  const float cb = fminf(fmaxf(y * inv, -1.f), 1.f), sb = fminf(rho * inv, 1.f);
  R[0] = ca;
  R[1] = 0.f;
  R[2] = -sa;
  R[3] = sb * sa;
  R[4] = cb;
  R[5] = sb * ca;
  R[6] = cb * sa;
  R[7] = -sb;
  R[8] = cb * ca;
}

}  // namespace esg
#include "wigner_gen.cuh"
namespace esg {

// degrees l0..L of the recursion, one barrier per degree (compile-time l, so
// only the degrees this l_max needs are instantiated)
template <int L, int l, int NG>
__device__ __forceinline__ void wigner_levels(bool act, int warp, const float* R, float* d) {
  if constexpr (l <= L) {
    if (act) wigner_deg<l, NG>(warp, R, d + Geo<L>::doff(l - 1), d + Geo<L>::doff(l));
    __syncthreads();
    wigner_levels<L, l + 1, NG>(act, warp, R, d);
  }
}

// Wigner blocks for a tile of ne <= 32 edges with the generated straight-line
// recursion: lane = edge, warps 0..NG-1 each own 1/NG of every degree's
// entries.  Needs blockDim.x >= 32 NG; all threads must call it.  D rows use an
// odd stride DSP so the per-lane bases hit distinct banks.
template <int L, int DSP, int NG = 4>
__device__ void wigner_tile_gen(const float* dirs, int ne, float* D) {
  using G = Geo<L>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool act = warp < NG && lane < ne;
  float R[9];
  if (act) {
    align_to_y(dirs[3 * lane], dirs[3 * lane + 1], dirs[3 * lane + 2], R);
    if (warp == 0) {
      float* d = D + lane * DSP;
      d[0] = 1.f;
#pragma unroll
      for (int i = 0; i < 9; ++i) d[1 + i] = R[i];
    }
  }
  __syncthreads();
  wigner_levels<L, 2, NG>(act, warp, R, D + lane * DSP);
}

}  // namespace esg
