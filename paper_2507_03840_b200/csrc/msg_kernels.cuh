// msg_kernels.cuh -- CUDA-core message kernels around the SO(2) linears:
// gather + rotate in, rotate back + residual, segment softmax + aggregation.
// Register-blocked on 4 channels per thread (float4 traffic, every Wigner
// entry read from SMEM once per 4 FMAs); Wigner blocks are recomputed per
// tile from the fp32 direction with the host-expanded recursion recipe.
#pragma once
#include <cuda_fp16.h>

#include <type_traits>

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

// fp32 Y in tiles of 128 edges, [tile][c / 4][el % 128][c % 4] (the fp16x3
// chain's drain: every 16-byte store of a warp lands next to its neighbour
// lane's, 512 contiguous bytes per instruction)
struct F32T {
  float x;
};
template <int HE>
__device__ __forceinline__ int64_t y_index(const F32T*, int64_t el, int c) {
  return (((el >> 7) * (HE / 4) + (c >> 2)) << 9) + ((el & 127) << 2) + (c & 3);
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
__device__ __forceinline__ float4 ld4(const F32T* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ld4(const uint16_t* p) {
  const uint2 w = __ldg(reinterpret_cast<const uint2*>(p));
  return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u), __uint_as_float(w.y << 16),
                     __uint_as_float(w.y & 0xffff0000u));
}

// L2 prefetches: the gathers of a tile are started before its Wigner blocks
// are computed, so their HBM latency hides behind the recursion.
// Bulk prefetch of a contiguous range; the instruction takes a uniform
// address, so only one lane per warp issues it (no per-lane loop).
__device__ __forceinline__ void prefetch_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// Prefetch the bf16 Y values of tile-local edges [el0, el0 + n) (tiled layout
// [tile][c/8][edge % 128][8]): one contiguous run per 8-channel block and
// 128-edge tile, issued by lane 0 of warps w, w + nw, ...
template <int HE>
__device__ __forceinline__ void prefetch_y(const uint16_t* Y, int64_t el0, int n, int w, int nw) {
  if (n <= 0 || (threadIdx.x & 31)) return;
  const int64_t el1 = el0 + n;  // exclusive
  const int64_t ta = el0 >> 7, tb = (el1 - 1) >> 7;
  const int runs = (int)(tb - ta + 1) * (HE / 8);
  for (int u = w; u < runs; u += nw) {
    const int64_t tile = ta + u / (HE / 8);
    const int blk = u % (HE / 8);
    const int64_t a = tile == ta ? el0 : tile << 7, b = tile == tb ? el1 : (tile + 1) << 7;
    prefetch_bulk(Y + y_index<HE>(Y, a, blk * 8), (uint32_t)(b - a) * 16u);
  }
}
template <int HE>
__device__ __forceinline__ void prefetch_y(const float*, int64_t, int, int, int) {}
// fp32 tiles [tile][c/4][edge % 128][4]: one run of (b - a) x 16 bytes per
// 4-channel block and 128-edge tile
template <int HE>
__device__ __forceinline__ void prefetch_y(const F32T* Y, int64_t el0, int n, int w, int nw) {
  if (n <= 0 || (threadIdx.x & 31)) return;
  const int64_t el1 = el0 + n;  // exclusive
  const int64_t ta = el0 >> 7, tb = (el1 - 1) >> 7;
  const int runs = (int)(tb - ta + 1) * (HE / 4);
  for (int u = w; u < runs; u += nw) {
    const int64_t tile = ta + u / (HE / 4);
    const int blk = u % (HE / 4);
    const int64_t a = tile == ta ? el0 : tile << 7, b = tile == tb ? el1 : (tile + 1) << 7;
    prefetch_bulk(Y + y_index<HE>(Y, a, blk * 4), (uint32_t)(b - a) * 16u);
  }
}

// |v| maxima of the feature tables (the fp16x3 chain's scale bounds): a
// non-negative float orders like its bit pattern, so an unsigned atomicMax
// on the bits is a float max (NaN bits sort above +inf and propagate)
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ void atomic_max_abs(float* p, float v) {
  atomicMax(reinterpret_cast<unsigned int*>(p), __float_as_uint(fabsf(v)));
}
__device__ __forceinline__ float max4(float4 v) { return fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))); }

// max |x| over n floats (n % 4 == 0, 16-byte aligned) into *out
template <int BLOCK = 256>
__global__ void __launch_bounds__(BLOCK) k_abs_max(const float* __restrict__ x, int64_t n, float* __restrict__ out) {
  float m = 0.f;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, max4(__ldg(x4 + i)));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomic_max_abs(out, m);
}

// The fp16x3 split image of A1 (so2_f16x3.cu): tiles of 128 edges, per
// 32-wide K chunk a 16 KB K-major SWIZZLE_128B tile whose 128-byte rows hold
// [hi(32) | lo(32)] fp16.  Byte offset of (edge el, K index k) in the hi
// half; the lo value sits 4 units (64 bytes) later, before the swizzle.
template <int KTOT>
__device__ __forceinline__ int64_t f16s_hi_off(int64_t el, int k, bool lo) {
  const int64_t tile = el >> 7;
  const int r = (int)(el & 127), w = k & 31;
  const int unit = (w >> 3) + (lo ? 4 : 0);
  return (tile * (KTOT / 32) + (k >> 5)) * 16384 + r * 128 + ((unit ^ (r & 7)) << 4) + (w & 7) * 2;
}
// The fp16x3 split of two fp32 values (|x| < 2^14): hi = x truncated to its
// leading 11 significant bits (mask the low 13 mantissa bits), an fp16
// number that packs exactly; lo = x - hi is exact in fp32 (< 2^-10 |x|) and
// rounds to fp16 (11 of its <= 13 bits: error <= 2^-22 |x|).  Two packed
// conversions (cvt.rn.f16x2.f32) per pair, no scalar ones.
__device__ __forceinline__ uint32_t pack_f16x2(float lo_half, float hi_half) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;\n" : "=r"(r) : "f"(hi_half), "f"(lo_half));
  return r;
}
__device__ __forceinline__ void split_f16x2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const float h0 = __uint_as_float(__float_as_uint(x0) & 0xffffe000u);
  const float h1 = __uint_as_float(__float_as_uint(x1) & 0xffffe000u);
  hi = pack_f16x2(h0, h1);
  lo = pack_f16x2(__fsub_rn(x0, h0), __fsub_rn(x1, h1));
}
__device__ __forceinline__ void st_f16s(uint8_t* base, int64_t off_hi, int64_t off_lo, float4 v, float inv_s) {
  uint32_t h0, l0, h1, l1;
  split_f16x2(v.x * inv_s, v.y * inv_s, h0, l0);
  split_f16x2(v.z * inv_s, v.w * inv_s, h1, l1);
  *reinterpret_cast<uint2*>(base + off_hi) = make_uint2(h0, h1);
  *reinterpret_cast<uint2*>(base + off_lo) = make_uint2(l0, l1);
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
__global__ void __launch_bounds__(32 * 3 * E / 4 < 128 ? 128 : 32 * 3 * E / 4, 3) k_rotate_in(const float* __restrict__ nodes,
                                                             const float* __restrict__ edges,
                                                             const int* __restrict__ src_row,
                                                             const int* __restrict__ dst_row,
                                                             const float* __restrict__ dir, int64_t e0, int64_t n_e,
                                                             OutT* __restrict__ A1, int pf, int el0,
                                                             const float* __restrict__ tmax = nullptr,
                                                             int edge_slot = 0) {
  using G = Geo<L>;
  using Y = Lay1<L, E, KPAD>;
  constexpr int TE = 32, DSP = G::DS + 2, H = G::H, C3 = 3 * E, Q = E / 4, TPE = 3 * Q;
  constexpr int NG = TE * TPE >= 384 ? 12 : 4;  // every warp takes a share of the Wigner recursion
  __shared__ float sD[TE * DSP];
  __shared__ float sdir[TE * 3];
  const int64_t t0 = e0 + (int64_t)blockIdx.x * TE;
  const int ne = (int)min64(TE, e0 + n_e - t0);
  const int e = threadIdx.x / TPE, r = threadIdx.x % TPE, p = r / Q, q = r % Q;
  const float* rowp = nullptr;
  if (e < ne) {
    const int64_t k = t0 + e;
    rowp = p == 0 ? nodes + (int64_t)__ldg(src_row + k) * H * E
                  : (p == 1 ? nodes + (int64_t)__ldg(dst_row + k) * H * E : edges + k * H * E);
    // pf 1: the tile's edge rows (contiguous) in one bulk prefetch, source
    // rows one each (destination rows repeat along the dst-sorted edges);
    // pf 2: every gathered row
    if (((pf & 3) == 2 ? q == 0 : (q == 0 && p == 0 && (pf & 3) == 1)) && !(el0 & 2)) prefetch_bulk(rowp, H * E * 4);
  }
  if ((pf & 3) == 1 && threadIdx.x == 0 && !(el0 & 1)) prefetch_bulk(edges + t0 * H * E, (uint32_t)ne * H * E * 4);
  for (int i = threadIdx.x; i < ne * 3; i += blockDim.x) sdir[i] = dir[t0 * 3 + i];
  __syncthreads();
  wigner_tile_gen<L, DSP, NG>(sdir, ne, sD);
  if (e < ne) {
    const float4* base = reinterpret_cast<const float4*>(rowp) + q;
    const float* D = sD + e * DSP;
    const int64_t el = t0 + e - e0;
    // A1 element (el, k) with k = K0 + pq, K0 a compile-time multiple of 16
    // and pq = p * E + 4 q < 48 fixed per thread (a1_index, split once)
    const int pq = p * E + q * 4;
    // KPAD == 32: the fp16x3 split image, values scaled by the message bound
    float inv_s = 1.f;
    if constexpr (KPAD == 32) inv_s = 1.f / f16s_pow2_scale(3.f * fmaxf(tmax[0], tmax[edge_slot]));
    OutT* a1_row = KPAD == 32 ? A1 : A1 + a1_index<Y::KTOT, KPAD>(el, 0);
    // el0 & 1: the edge table holds only its l = 0 plane (layer 0 of a
    // forward; k_init_edges leaves the other planes unwritten); el0 & 2: so do
    // the node rows (before layer 0's node update).  Those planes read as zero.
    const bool zero_l = p == 2 ? (el0 & 1) != 0 : (el0 & 2) != 0;
#pragma unroll
    for (int l = 0; l <= L; ++l) {
      const int dd = 2 * l + 1;
      float4 x[2 * L + 1];
#pragma unroll
      for (int b = -l; b <= l; ++b)
        x[b + l] = (l > 0 && zero_l) ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg(base + (l * l + l + b) * (E / 4));
#pragma unroll
      for (int a = -l; a <= l; ++a) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int b = -l; b <= l; ++b) acc = fma4(D[G::doff(l) + (a + l) * dd + (b + l)], x[b + l], acc);
        const int m = a < 0 ? -a : a;
        const int k = Y::kofs(m) + (G::mrow(l, a) - G::moff(m)) * C3 + pq;
        if constexpr (KPAD == 32)
          st_f16s(reinterpret_cast<uint8_t*>(A1), f16s_hi_off<Y::KTOT>(el, k, false),
                  f16s_hi_off<Y::KTOT>(el, k, true), acc, inv_s);
        else
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
                                                               float* __restrict__ edges, int pf, int el0,
                                                               float* __restrict__ emax = nullptr) {
  using G = Geo<L>;
  constexpr int TE = 32, DSP = G::DS + 2, H = G::H, Q = E / 4;
  __shared__ float sD[TE * DSP];
  __shared__ float sdir[TE * 3];
  const int64_t t0 = e0 + (int64_t)blockIdx.x * TE;
  const int ne = (int)min64(TE, e0 + n_e - t0);
  const int e = threadIdx.x / Q, q = threadIdx.x % Q;
  if (pf & 3) {  // the tile's edge rows (contiguous) and its Y runs
    if (threadIdx.x == 0 && !(el0 & 1)) prefetch_bulk(edges + t0 * H * E, (uint32_t)ne * H * E * 4);
    prefetch_y<H * E>(Yin, t0 - e0, ne, threadIdx.x >> 5, blockDim.x >> 5);
  }
  for (int i = threadIdx.x; i < ne * 3; i += blockDim.x) sdir[i] = dir[t0 * 3 + i];
  __syncthreads();
  wigner_tile_gen<L, DSP>(sdir, ne, sD);
  float vmax = 0.f;
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
        // el0: only the l = 0 plane of the residual holds data (layer 0)
        old[b + l] = (l > 0 && (el0 & 1)) ? make_float4(0.f, 0.f, 0.f, 0.f) : row[(l * l + l + b) * Q];
      }
#pragma unroll
      for (int a = -l; a <= l; ++a) {
        float4 acc = old[a + l];
#pragma unroll
        for (int b = -l; b <= l; ++b) acc = fma4(D[G::doff(l) + (b + l) * dd + (a + l)], y[b + l], acc);
        row[(l * l + l + a) * Q] = acc;
        vmax = fmaxf(vmax, max4(acc));
      }
    }
  }
  if (emax) {  // max |new edge row| (the next layer's fp16x3 scale bound)
    vmax = warp_max(vmax);
    if ((threadIdx.x & 31) == 0) atomic_max_abs(emax, vmax);
  }
}

// Row split of the back-rotation D^T y for the node update: four parts of
// about equal FMA work (l_max 4: l = 4 with a <= 0, l = 4 with a > 0, l = 3,
// l <= 2), one part per warp so every warp runs one straight-line path.
// Lower l_max: part p takes degree p.
template <int L>
struct NodeSplit {
  static_assert(L <= 4, "node update row split is laid out for l_max <= 4");
  __host__ __device__ static constexpr bool owns(int p, int l, int a) {
    return L == 4 ? (l == 4 ? (p == (a <= 0 ? 0 : 1)) : (l == 3 ? p == 2 : p == 3)) : l == p;
  }
  __host__ __device__ static constexpr int rows(int p) {
    int n = 0;
    for (int l = 0; l <= L; ++l)
      for (int a = -l; a <= l; ++a) n += owns(p, l, a) ? 1 : 0;
    return n;
  }
  static constexpr int RMAX = L == 4 ? 9 : 2 * L + 1;
};

// Y of one edge: from global memory (fp32 rows) or from the SMEM copy of the
// edge tile (bf16, [col / 8][edge in tile][col % 8], like the global tiles)
template <int HE, typename YT = float>
struct YGlobal {
  const YT* Y;
  int64_t el;
  __device__ __forceinline__ float4 operator()(int c) const { return ld4(Y + y_index<HE>(Y, el, c)); }
};
struct YTileSmem {
  const uint16_t* sY;
  int i;
  __device__ __forceinline__ float4 operator()(int c) const {
    const uint2 w = *reinterpret_cast<const uint2*>(sY + (((c >> 3) * 32 + i) << 3) + (c & 7));
    return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u), __uint_as_float(w.y << 16),
                       __uint_as_float(w.y & 0xffff0000u));
  }
};

// acc[slot of (l, a) in part P] += al * sum_b D[b][a] y_b for one edge
template <int L, int E, int P, typename YSrc>
__device__ __forceinline__ void node_part(const YSrc& ysrc, int q, const float* D, float al, float4* acc) {
  using G = Geo<L>;
  using S = NodeSplit<L>;
  int r = 0;
#pragma unroll
  for (int l = 0; l <= L; ++l) {
    bool any = false;
#pragma unroll
    for (int a = -l; a <= l; ++a) any |= S::owns(P, l, a);
    if (!any) continue;
    const int dd = 2 * l + 1;
    float4 y[2 * L + 1];
#pragma unroll
    for (int b = -l; b <= l; ++b) y[b + l] = ysrc(G::mrow(l, b) * E + 4 * q);
#pragma unroll
    for (int a = -l; a <= l; ++a) {
      if (!S::owns(P, l, a)) continue;
      float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int b = -l; b <= l; ++b) m = fma4(D[G::doff(l) + (b + l) * dd + (a + l)], y[b + l], m);
      acc[r] = make_float4(fmaf(al, m.x, acc[r].x), fmaf(al, m.y, acc[r].y), fmaf(al, m.z, acc[r].z),
                           fmaf(al, m.w, acc[r].w));
      ++r;
    }
  }
}
template <int L, int P>
__device__ __forceinline__ void node_part_park(float* red, int slot, int q, int Q, const float4* acc) {
  using G = Geo<L>;
  int r = 0;
#pragma unroll
  for (int l = 0; l <= L; ++l)
#pragma unroll
    for (int a = -l; a <= l; ++a)
      if (NodeSplit<L>::owns(P, l, a))
        reinterpret_cast<float4*>(red)[(slot * G::H + l * l + l + a) * Q + q] = acc[r++];
}

// dynamic SMEM of k_node_update: D of the edge tile (+ its bf16 Y rows when
// Y is bf16), reused for the slot partial sums
template <int L, int E, typename YT>
constexpr int node_update_smem_floats() {
  constexpr int TE = 32, DSP = Geo<L>::DS + 2, NSLOT = 32 / (E / 4);
  constexpr int tile = TE * DSP + (sizeof(YT) == 2 ? TE * Geo<L>::H * E / 2 : 0);
  return tile > NSLOT * Geo<L>::H * E ? tile : NSLOT * Geo<L>::H * E;
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(sdst)),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ops.h:192-263.  One CTA (4 warps) per owned destination j; logits from the
// l = 0 channels (msg row 0 == y row 0 since D_0 = 1), max-subtracted
// softmax, then out_j = node_j + sum_k alpha_k D_k^T y_k.  Tiles of 32
// edges: the Wigner blocks go to SMEM, then warp p (row part p of NodeSplit)
// lane (slot, quad) accumulates alpha_k D_k^T y_k of the tile's edges
// slot, slot + NSLOT, ... in registers.  The NSLOT partial sums are added in
// slot order at the end: a fixed order that depends only on the segment
// (partition-invariant and deterministic).  Dynamic SMEM: node_update_smem_floats.
template <int L, int E, typename YT, bool LOGITS_GIVEN>
__global__ void __launch_bounds__(128, 4) k_node_update(const YT* __restrict__ Yin, const float* __restrict__ dir,
                                                     const int64_t* __restrict__ seg, int j0, int64_t e0,
                                                     const float* __restrict__ att,
                                                     const float* __restrict__ nodes_in, float* __restrict__ nodes_out,
                                                     float* __restrict__ logit_scratch, int /*pf*/) {
  using G = Geo<L>;
  constexpr int TE = 32, DSP = G::DS + 2, H = G::H, HE = H * E, Q = E / 4, HQ = H * Q, NSLOT = 32 / Q;
  constexpr bool YSMEM = sizeof(YT) == 2;  // bf16 Y: stage the tile's rows in SMEM
  extern __shared__ __align__(16) float dyn[];
  float* sD = dyn;  // TE x DSP; reused for the NSLOT x H x E partial sums
  uint16_t* sY = reinterpret_cast<uint16_t*>(dyn + TE * DSP);  // [HE / 8][TE][8] bf16 (YSMEM)
  __shared__ float sdir[TE * 3];
  __shared__ float sA[TE];
  __shared__ float sred[4];
  const int j = j0 + blockIdx.x;
  const int64_t b = seg[j], en = seg[j + 1];
  const int t = threadIdx.x, part = t >> 5, slot = (t & 31) / Q, q = t % Q;
  float4 acc[NodeSplit<L>::RMAX];
#pragma unroll
  for (int r = 0; r < NodeSplit<L>::RMAX; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
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
        for (int qq = 0; qq < Q; ++qq) {
          const float4 v = ld4(Yin + y_index<HE>(Yin, k - e0, 4 * qq));
          s = fmaf(att[4 * qq], v.x, s);
          s = fmaf(att[4 * qq + 1], v.y, s);
          s = fmaf(att[4 * qq + 2], v.z, s);
          s = fmaf(att[4 * qq + 3], v.w, s);
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
    for (int64_t k0 = b; k0 < en; k0 += TE) {
      const int ne = (int)min64(TE, en - k0);
      // (no L2 prefetch of the next tile's Y: measured 215 -> 155 ms per C4
      // forward without it -- the loads of 4 warps x 6 CTAs per SM already
      // cover the latency, and the prefetched runs were evicted unused)
      __syncthreads();  // the previous tile's D is no longer read
      for (int i = t; i < ne * 3; i += 128) sdir[i] = dir[k0 * 3 + i];  // dir: global edge index
      for (int i = t; i < ne; i += 128) sA[i] = lg[k0 - b + i] / z;
      if constexpr (YSMEM) {  // the tile's Y rows arrive while the Wigner blocks are computed
        for (int u = t; u < (HE / 8) * TE; u += 128) {  // TE a power of two: no runtime division
          const int blk = u / TE, i = u % TE;
          if (i < ne) cp_async16(sY + ((blk * TE + i) << 3), Yin + y_index<HE>(Yin, k0 + i - e0, blk * 8));
        }
      }
      __syncthreads();
      wigner_tile_gen<L, DSP>(sdir, ne, sD);
      if constexpr (YSMEM) {
        cp_async_wait_all();
        __syncthreads();
      }
      for (int i = slot; i < ne; i += NSLOT) {
        const float* D = sD + i * DSP;
        const float al = sA[i];
        if constexpr (YSMEM) {
          const YTileSmem ys{sY, i};
          switch (part) {
            case 0: node_part<L, E, 0>(ys, q, D, al, acc); break;
            case 1: node_part<L, E, 1>(ys, q, D, al, acc); break;
            case 2: node_part<L, E, 2>(ys, q, D, al, acc); break;
            default: node_part<L, E, 3>(ys, q, D, al, acc); break;
          }
        } else {
          using YG = typename std::conditional<sizeof(YT) == 2, float, YT>::type;
          const YGlobal<HE, YG> ys{reinterpret_cast<const YG*>(Yin), k0 + i - e0};
          switch (part) {
            case 0: node_part<L, E, 0>(ys, q, D, al, acc); break;
            case 1: node_part<L, E, 1>(ys, q, D, al, acc); break;
            case 2: node_part<L, E, 2>(ys, q, D, al, acc); break;
            default: node_part<L, E, 3>(ys, q, D, al, acc); break;
          }
        }
      }
    }
  }
  // park the slot partial sums, then add them in slot order
  __syncthreads();
  switch (part) {
    case 0: node_part_park<L, 0>(dyn, slot, q, Q, acc); break;
    case 1: node_part_park<L, 1>(dyn, slot, q, Q, acc); break;
    case 2: node_part_park<L, 2>(dyn, slot, q, Q, acc); break;
    default: node_part_park<L, 3>(dyn, slot, q, Q, acc); break;
  }
  __syncthreads();
  for (int o = t; o < HQ; o += 128) {
    float4 out = reinterpret_cast<const float4*>(nodes_in + (int64_t)j * HE)[o];
    if (b < en) {
      float4 s = reinterpret_cast<const float4*>(dyn)[o];
      for (int sl = 1; sl < NSLOT; ++sl) {
        const float4 v = reinterpret_cast<const float4*>(dyn)[sl * HQ + o];
        s.x += v.x;
        s.y += v.y;
        s.z += v.z;
        s.w += v.w;
      }
      out.x += s.x;
      out.y += s.y;
      out.z += s.z;
      out.w += s.w;
    }
    reinterpret_cast<float4*>(nodes_out + (int64_t)j * HE)[o] = out;
  }
}

}  // namespace esg
