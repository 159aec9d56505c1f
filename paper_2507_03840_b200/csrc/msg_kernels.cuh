// msg_kernels.cuh -- CUDA-core message kernels around the SO(2) linears:
// gather + rotate in, rotate back + residual, segment softmax + aggregation.
// Register-blocked on 4 channels per thread (float4 traffic, every Wigner
// entry read from SMEM once per 4 FMAs); Wigner blocks are recomputed per
// tile from the fp32 direction with the host-expanded recursion recipe.
#pragma once
#include "model_kernels.cuh"

namespace esg {

__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
// bf16x2 round-to-nearest-even pack, first argument in the low half
__device__ __forceinline__ uint32_t bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;\n" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void st4(uint16_t* p, float4 v) {
  *reinterpret_cast<uint2*>(p) = make_uint2(bf16x2(v.x, v.y), bf16x2(v.z, v.w));
}
// Element index of A1(edge el, K index k).  KPAD == 1: plain row-major
// (fp32 CUDA-core path).  KPAD == 64: the tensor-core image -- tiles of 128
// edges, one contiguous 16 KB block per 64-wide K chunk, 128-byte rows whose
// 16-byte units are XOR-swizzled by row % 8 (UMMA SWIZZLE_128B, K-major), so
// so2_tc.cu moves each chunk with a single bulk copy.
template <int KTOT, int KPAD>
__device__ __forceinline__ int64_t a1_index(int64_t el, int k) {
  if (KPAD == 1) return el * KTOT + k;
  const int64_t tile = el >> 7;
  const int r = (int)(el & 127), kc = k >> 6, w = k & 63;
  return (tile * (KTOT / 64) + kc) * 8192 + r * 64 + (((w >> 3) ^ (r & 7)) << 3) + (w & 7);
}

// Element index of Y(edge el, column c), columns in order-major row order.
// fp32 (CUDA-core path): plain row-major.  bf16 (tensor-core path): tiles of
// 128 edges, [tile][c / 8][el % 128][c % 8] -- the tcgen05 epilogue stores one
// 16-byte unit per edge contiguously across the warp, and the consumers'
// 4-column loads of consecutive edges fall into the same 128-byte lines.
template <int HE>
__device__ __forceinline__ int64_t y_index(const float*, int64_t el, int c) {
  return el * HE + c;
}
template <int HE>
__device__ __forceinline__ int64_t y_index(const uint16_t*, int64_t el, int c) {
  return (((el >> 7) * (HE / 8) + (c >> 3)) << 10) + ((el & 127) << 3) + (c & 7);
}

// a1_index(el, k) - a1_index(el, 0): the within-tile-row offset of K index k
template <int KPAD>
__device__ __forceinline__ int a1_offset(int64_t el, int k) {
  if (KPAD == 1) return k;
  const int r7 = (int)(el & 7), w = k & 63;
  return (k >> 6) * 8192 + (((w >> 3) ^ r7) - r7) * 8 + (w & 7);
}

// 4 consecutive Y values as float4 from fp32 or bf16 storage
__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ld4(const uint16_t* p) {
  const uint2 w = __ldg(reinterpret_cast<const uint2*>(p));
  return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u), __uint_as_float(w.y << 16),
                     __uint_as_float(w.y & 0xffff0000u));
}

__device__ __forceinline__ float4 fma4(float d, float4 x, float4 a) {
  return make_float4(fmaf(d, x.x, a.x), fmaf(d, x.y, a.y), fmaf(d, x.z, a.z), fmaf(d, x.w, a.w));
}

// ops.h:68-122: message = [src | dst | edge] per harmonic row, rotated into
// the edge frame with D_l (kernels.h:73-96), permuted to order-major rows
// (kernels.h:98-115), written as the A1 operand of the SO(2) linears.
// Thread = (edge, part in {src,dst,edge}, 4-channel quad); 32 edges per CTA
// (the Wigner warps then run full 32-lane tiles).
template <int L, int E, int KPAD, typename OutT>
__global__ void __launch_bounds__(32 * 3 * E / 4 < 128 ? 128 : 32 * 3 * E / 4, 2) k_rotate_in(const float* __restrict__ nodes,
                                                             const float* __restrict__ edges,
                                                             const int* __restrict__ src_row,
                                                             const int* __restrict__ dst_row,
                                                             const float* __restrict__ dir, int64_t e0, int64_t n_e,
                                                             OutT* __restrict__ A1, WigRecipe rc) {
  using G = Geo<L>;
  using Y = Lay1<L, E, KPAD>;
  constexpr int TE = 32, DSP = G::DS + 2, H = G::H, C3 = 3 * E, Q = E / 4, TPE = 3 * Q;
  __shared__ float sD[TE * DSP];
  __shared__ float sdir[TE * 3];
  const int64_t t0 = e0 + (int64_t)blockIdx.x * TE;
  const int ne = (int)min64(TE, e0 + n_e - t0);
  for (int i = threadIdx.x; i < ne * 3; i += blockDim.x) sdir[i] = dir[t0 * 3 + i];
  const int e = threadIdx.x / TPE, r = threadIdx.x % TPE, p = r / Q, q = r % Q;
  __syncthreads();
  wigner_tile_gen<L, DSP>(sdir, ne, sD);
  if (e < ne) {
    const int64_t k = t0 + e;
    const float4* base = reinterpret_cast<const float4*>(
                             p == 0 ? nodes + (int64_t)__ldg(src_row + k) * H * E
                                    : (p == 1 ? nodes + (int64_t)__ldg(dst_row + k) * H * E : edges + k * H * E)) +
                         q;
    const float* D = sD + e * DSP;
    const int64_t el = t0 + e - e0;
    // A1 element (el, k) with k = K0 + pq, K0 a compile-time multiple of 16
    // and pq = p * E + 4 q < 48 fixed per thread (a1_index, split once)
    const int pq = p * E + q * 4;
    OutT* a1_row = A1 + a1_index<Y::KTOT, KPAD>(el, 0);
#pragma unroll
    for (int l = 0; l <= L; ++l) {
      const int dd = 2 * l + 1;
      float4 x[2 * L + 1];
#pragma unroll
      for (int b = -l; b <= l; ++b) x[b + l] = __ldg(base + (l * l + l + b) * (E / 4));
#pragma unroll
      for (int a = -l; a <= l; ++a) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int b = -l; b <= l; ++b) acc = fma4(D[G::doff(l) + (a + l) * dd + (b + l)], x[b + l], acc);
        const int m = a < 0 ? -a : a;
        const int k = Y::kofs(m) + (G::mrow(l, a) - G::moff(m)) * C3 + pq;
        st4(a1_row + a1_offset<KPAD>(el, k), acc);
      }
    }
  }
  // K padding of each order block is never written: the A1 scratch is zeroed
  // once at prepare time and the padding positions are fixed.
}

// ops.h:115-117 rotate back with D^T then ops.h:265-283 residual add in
// place.  Thread = (edge, 4-channel quad); 32 edges per CTA.
template <int L, int E, typename YT>
__global__ void __launch_bounds__(32 * E / 4 < 128 ? 128 : 32 * E / 4, 4) k_rotate_out_edge(const YT* __restrict__ Yin,
                                                               const float* __restrict__ dir, int64_t e0, int64_t n_e,
                                                               float* __restrict__ edges, WigRecipe rc) {
  using G = Geo<L>;
  constexpr int TE = 32, DSP = G::DS + 2, H = G::H, Q = E / 4;
  __shared__ float sD[TE * DSP];
  __shared__ float sdir[TE * 3];
  const int64_t t0 = e0 + (int64_t)blockIdx.x * TE;
  const int ne = (int)min64(TE, e0 + n_e - t0);
  for (int i = threadIdx.x; i < ne * 3; i += blockDim.x) sdir[i] = dir[t0 * 3 + i];
  const int e = threadIdx.x / Q, q = threadIdx.x % Q;
  __syncthreads();
  wigner_tile_gen<L, DSP>(sdir, ne, sD);
  if (e < ne) {
    const int64_t el = t0 + e - e0;
    const float* D = sD + e * DSP;
    float4* row = reinterpret_cast<float4*>(edges + (t0 + e) * H * E) + q;
#pragma unroll
    for (int l = 0; l <= L; ++l) {
      const int dd = 2 * l + 1;
      float4 y[2 * L + 1], old[2 * L + 1];
#pragma unroll
      for (int b = -l; b <= l; ++b) {
        y[b + l] = ld4(Yin + y_index<H * E>(Yin, el, G::mrow(l, b) * E + 4 * q));  // order-major rows
        old[b + l] = row[(l * l + l + b) * Q];
      }
#pragma unroll
      for (int a = -l; a <= l; ++a) {
        float4 acc = old[a + l];
#pragma unroll
        for (int b = -l; b <= l; ++b) acc = fma4(D[G::doff(l) + (b + l) * dd + (a + l)], y[b + l], acc);
        row[(l * l + l + a) * Q] = acc;
      }
    }
  }
}

// ops.h:192-263.  One CTA per owned destination j; logits from the l = 0
// channels (msg row 0 == y row 0 since D_0 = 1), max-subtracted softmax, then
// out_j = node_j + sum_k alpha_k msg_k.  Tiles of 32 edges: thread (edge,
// 4-channel quad) rotates its message back (float4, D from SMEM), scales it
// by alpha and parks it in SMEM; thread (h, quad) then adds the tile's rows
// in edge order -- a fixed order, so the result depends only on the segment
// (partition-invariant and deterministic).  Dynamic SMEM: D + messages.
template <int L, int E, typename YT, bool LOGITS_GIVEN>
__global__ void __launch_bounds__(128, 6) k_node_update(const YT* __restrict__ Yin, const float* __restrict__ dir,
                                                     const int64_t* __restrict__ seg, int j0, int64_t e0,
                                                     const float* __restrict__ att,
                                                     const float* __restrict__ nodes_in, float* __restrict__ nodes_out,
                                                     float* __restrict__ logit_scratch, WigRecipe rc) {
  using G = Geo<L>;
  constexpr int TE = 16, DSP = G::DS + 2, H = G::H, HE = H * E, Q = E / 4, HQ = H * Q;
  extern __shared__ __align__(16) float dyn[];
  float* sM = dyn;                 // TE x HE
  float* sD = dyn + TE * HE;       // TE x DSP
  __shared__ float sdir[TE * 3];
  __shared__ float sA[TE];
  __shared__ float sred[4];
  const int j = j0 + blockIdx.x;
  const int64_t b = seg[j], en = seg[j + 1];
  const int t = threadIdx.x;
  const bool owner = t < HQ;  // thread (h, quad) owns one float4 of the output row
  float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
  if (owner) out = reinterpret_cast<const float4*>(nodes_in + (int64_t)j * HE)[t];
  if (b < en) {
    float* lg = logit_scratch + (b - e0);
    float mx = -INFINITY;
    for (int64_t k = b + t; k < en; k += 128) {
      float s;
      if (LOGITS_GIVEN) {  // written by the tensor-core epilogue
        s = lg[k - b];
      } else {
        s = 0.f;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const float4 v = ld4(Yin + y_index<HE>(Yin, k - e0, 4 * q));
          s = fmaf(att[4 * q], v.x, s);
          s = fmaf(att[4 * q + 1], v.y, s);
          s = fmaf(att[4 * q + 2], v.z, s);
          s = fmaf(att[4 * q + 3], v.w, s);
        }
        lg[k - b] = s;
      }
      mx = fmaxf(mx, s);
    }
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((t & 31) == 0) sred[t >> 5] = mx;
    __syncthreads();
    mx = fmaxf(fmaxf(sred[0], sred[1]), fmaxf(sred[2], sred[3]));
    __syncthreads();
    float z = 0.f;
    for (int64_t k = b + t; k < en; k += 128) {
      const float a = expf(lg[k - b] - mx);
      lg[k - b] = a;
      z += a;
    }
    for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    if ((t & 31) == 0) sred[t >> 5] = z;
    __syncthreads();
    z = (sred[0] + sred[1]) + (sred[2] + sred[3]);
    const int e = t / Q, q = t % Q;
    for (int64_t k0 = b; k0 < en; k0 += TE) {
      const int ne = (int)min64(TE, en - k0);
      __syncthreads();
      for (int i = t; i < ne * 3; i += 128) sdir[i] = dir[(k0 - e0) * 3 + i];
      for (int i = t; i < ne; i += 128) sA[i] = lg[k0 - b + i] / z;
      __syncthreads();
      wigner_tile_gen<L, DSP>(sdir, ne, sD);
      if (e < ne) {
        const int64_t el = k0 + e - e0;
        const float* D = sD + e * DSP;
        const float al = sA[e];
        float4* mrow = reinterpret_cast<float4*>(sM + e * HE) + q;
#pragma unroll
        for (int l = 0; l <= L; ++l) {
          const int dd = 2 * l + 1;
          float4 y[2 * L + 1];
#pragma unroll
          for (int bb = -l; bb <= l; ++bb) y[bb + l] = ld4(Yin + y_index<HE>(Yin, el, G::mrow(l, bb) * E + 4 * q));
#pragma unroll
          for (int a = -l; a <= l; ++a) {
            float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int bb = -l; bb <= l; ++bb) m = fma4(D[G::doff(l) + (bb + l) * dd + (a + l)], y[bb + l], m);
            mrow[(l * l + l + a) * Q] = make_float4(al * m.x, al * m.y, al * m.z, al * m.w);
          }
        }
      }
      __syncthreads();
      if (owner)
        for (int ee = 0; ee < ne; ++ee) {
          const float4 v = reinterpret_cast<const float4*>(sM + ee * HE)[t];
          out.x += v.x;
          out.y += v.y;
          out.z += v.z;
          out.w += v.w;
        }
    }
  }
  if (owner) reinterpret_cast<float4*>(nodes_out + (int64_t)j * HE)[t] = out;
}

}  // namespace esg
