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

// Wigner recursion coefficients u, v, w for l = 2..L (wigner.cpp:64-76),
// indexed like the stacked blocks; filled by the host.
struct WignerCoef {
  float u[165], v[165], w[165];
};
static __constant__ WignerCoef c_wig;  // per translation unit; see upload_wigner_coef

// Rotation taking the unit edge direction onto +y: R = Rx(-beta) Ry(-alpha)
// with alpha = atan2(ux, uz), beta = acos(uy) (align.cpp:32-39), written with
// cos/sin of alpha and beta taken directly from u (no trig calls).
__device__ __forceinline__ void align_to_y(float x, float y, float z, float R[9]) {
  const float inv = rsqrtf(x * x + y * y + z * z);
  const float ux = x * inv, uy = fminf(fmaxf(y * inv, -1.f), 1.f), uz = z * inv;
  const float rho = sqrtf(ux * ux + uz * uz);
  float ca = 1.f, sa = 0.f;
  if (rho > 0.f) {
    ca = uz / rho;
    sa = ux / rho;
  }
  const float cb = uy, sb = sqrtf(fmaxf(1.f - uy * uy, 0.f));
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

// Ivanic-Ruedenberg recursion expanded on the host into flat recipes: entry
// q of degree l (stacked index doff(l) + (m+l)(2l+1) + (n+l)) is
// sum_t coef[t] * R[ri[t]] * prev[pi[t]] with R the 3x3 band-1 block and prev
// the degree l-1 block (wigner.cpp:58-81 with the u/v/w/P terms multiplied
// out; zero-coefficient terms skipped exactly as the reference skips them).
struct WigRecipe {
  const int* start;   // per stacked entry (DS + 1)
  const float* coef;  // per term
  const uint8_t* ri;  // R index 0..8
  const uint16_t* pi; // index inside the degree l-1 block
};

// Branch-free cooperative Wigner blocks for a tile of `ne` edges.
template <int L, int DSP>
__device__ void wigner_tile_recipe(const float* dirs, int ne, float* D, WigRecipe rc) {
  using G = Geo<L>;
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    float R[9];
    align_to_y(dirs[3 * e], dirs[3 * e + 1], dirs[3 * e + 2], R);
    float* d = D + e * DSP;
    d[0] = 1.f;
#pragma unroll
    for (int i = 0; i < 9; ++i) d[1 + i] = R[i];
  }
  __syncthreads();
#pragma unroll 1
  for (int l = 2; l <= L; ++l) {
    const int dd = (2 * l + 1) * (2 * l + 1);
    const int ob = G::doff(l), op = G::doff(l - 1);
    for (int t = threadIdx.x; t < ne * dd; t += blockDim.x) {
      const int e = t / dd, q = ob + t % dd;
      const float* R = D + e * DSP + 1;
      const float* pv = D + e * DSP + op;
      float acc = 0.f;
      const int t1 = __ldg(rc.start + q + 1);
      for (int k = __ldg(rc.start + q); k < t1; ++k) acc = fmaf(__ldg(rc.coef + k) * R[__ldg(rc.ri + k)], pv[__ldg(rc.pi + k)], acc);
      D[e * DSP + q] = acc;
    }
    __syncthreads();
  }
}

// Cooperative Wigner blocks for a tile of `ne` edges: D[e*DSP + doff(l) + ...].
// dirs: 3 floats per edge (displacement).  All threads of the block call it.
template <int L, int DSP>
__device__ void wigner_tile(const float* dirs, int ne, float* D) {
  using G = Geo<L>;
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    float R[9];
    align_to_y(dirs[3 * e], dirs[3 * e + 1], dirs[3 * e + 2], R);
    float* d = D + e * DSP;
    d[0] = 1.f;
    for (int i = 0; i < 9; ++i) d[1 + i] = R[i];
  }
  __syncthreads();
#pragma unroll 1
  for (int l = 2; l <= L; ++l) {
    const int dd = 2 * l + 1, dp = 2 * l - 1;
    const int cnt = ne * dd * dd;
    const int ob = G::doff(l), op = G::doff(l - 1);
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      const int e = t / (dd * dd), q = t % (dd * dd);
      const int m = q / dd - l, n = q % dd - l;
      const float* R = D + e * DSP + 1;          // band 1, indices -1..1
      const float* pv = D + e * DSP + op;        // degree l-1
      auto pm = [&](int a, int b) { return pv[(a + l - 1) * dp + (b + l - 1)]; };
      auto P = [&](int i, int a, int b) {
        const float* r = R + (i + 1) * 3;
        if (b == l) return r[2] * pm(a, l - 1) - r[0] * pm(a, -l + 1);
        if (b == -l) return r[2] * pm(a, -l + 1) + r[0] * pm(a, l - 1);
        return r[1] * pm(a, b);
      };
      const float cu = c_wig.u[ob + q], cv = c_wig.v[ob + q], cw = c_wig.w[ob + q];
      float acc = 0.f;
      if (cu != 0.f) acc += cu * P(0, m, n);
      if (cv != 0.f) {
        float vt;
        if (m == 0)
          vt = P(1, 1, n) + P(-1, -1, n);
        else if (m > 0)
          vt = P(1, m - 1, n) * (m == 1 ? 1.41421356237f : 1.f) - (m == 1 ? 0.f : P(-1, -m + 1, n));
        else
          vt = (m == -1 ? 0.f : P(1, m + 1, n)) + P(-1, -m - 1, n) * (m == -1 ? 1.41421356237f : 1.f);
        acc += cv * vt;
      }
      if (cw != 0.f) {
        const float wt = m > 0 ? P(1, m + 1, n) + P(-1, -m - 1, n) : P(1, m - 1, n) - P(-1, -m + 1, n);
        acc += cw * wt;
      }
      D[e * DSP + ob + q] = acc;
    }
    __syncthreads();
  }
}

}  // namespace esg
