// so2_f16x3.cu -- the fp32-faithful SO(2) linear chain on the 5th-gen tensor
// cores (SURVEY §8 a11 "fp32 for parity"; kernels.h:133-161 lin1/lin2,
// :210-226 gate; network.h:144-146).
//
// Every fp32 operand x is held as two fp16 numbers after a power-of-two
// scale s:  x / s = hi + lo,  hi = rn(x / s),  lo = rn(x / s - hi).  fp16
// keeps 11 significant bits, so hi + lo carries 22 of fp32's 24 (the same
// as the 3xTF32 split of tf32_gemm.cu), and the product of two split
// operands is taken as hi.hi + hi.lo + lo.hi with fp32 accumulation in
// TMEM (the dropped lo.lo and the rounding of lo are ~2^-22 relative).
// tcgen05.mma kind::f16 runs at twice the rate of kind::tf32 and an fp16
// split moves half the bytes of a tf32 split, so this chain issues the same
// three products at half the cost of the tf32 one.
//
// The scales keep fp16's range: they are global per (block, order), derived
// from bounds that hold for every input --
//   rotated message  |a| <= 3 max(|node table|, |edge table|)  (D_l is
//                    orthogonal and 2l + 1 <= 9: |D x| <= ||x_l|| <= 3 max)
//   lin1 output      |h| <= ||W1_m||_inf |a|,  gate output |g| <= |h|
// so every scaled value stays below 2^14 (fp16 max 65504).  The table
// maxima are maintained on the device by the kernels that write the tables
// (model.cu); the weights are split once at pack time with their own scale.
// Values far below a scale lose nothing that matters: the split's absolute
// error floor is 2^-25 s = 2^-39 of the bound.
//
// Per tile of 128 edges (UMMA M = 128, one edge per TMEM lane) and per
// order m = 0..L:
//   lin1   H_m = A1_m . W1_m^T        A1 from HBM (rotate_in writes the split
//                                     image), 3 MMAs per K = 16 step
//   gate   s = sigmoid(h_0[:, l = 0 channels]) (order 0 first),
//          G_m = H_m * s[c % 2E] / s2_m, split -> A2 ring (32-column chunks)
//   lin2   Y_m = A2_m . W2_m^T        chunk-pipelined behind the gate
//   drain  Y_m -> fp32 order-major rows in HBM (+ attention logits)
//
// Operand images (HBM and SMEM alike): per 32-wide K chunk a K-major
// SWIZZLE_128B tile whose 128-byte rows hold [hi(32) | lo(32)] fp16, so the
// hi and lo operands of a K = 16 step are the same descriptor advanced by 0
// or 64 bytes.  One bulk copy (TMA, 1-D) per chunk, no tensor maps.
//
// Warp roles (608 threads, 1 CTA per SM, persistent over tiles):
//   warp 0      A producer (A1 chunks, 4-stage ring)
//   warp 18     B producer (weight chunks, 3-stage ring)
//   warp 1      MMA issuer (one elected lane)
//   warps 2-9   gate: warp w owns TMEM lanes 32 (w % 4)+, the two halves take
//               alternate 32-column chunks
//   warps 10-17 drain
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "device_model.h"
#include "esg_internal.h"
#include "model_kernels.cuh"
#include "tc_common.cuh"

namespace esg {

namespace {
using namespace tc;

constexpr int TILE_M = 128;
constexpr int THREADS = 608;
constexpr int NSA = 4;                 // A1 ring
constexpr int NSB = 3;                 // weight ring
constexpr int NS2 = 4;                 // gated-operand ring (>= the Y chunks of any order)
constexpr int CHUNK = TILE_M * 128;    // one 32-wide K chunk of 128 rows, hi | lo: 16 KB
constexpr int B_STAGE = 256 * 128;     // up to 256 weight rows: 32 KB
constexpr int GATE_THREADS = 256, DRAIN_THREADS = 256;
constexpr int SMEM_BYTES = 1024 + NSA * CHUNK + NSB * B_STAGE + NS2 * CHUNK + 512;

template <int L, int E>
struct S3 {
  using G = Geo<L>;
  __host__ __device__ static constexpr int K1(int m) { return G::rows(m) * 3 * E; }
  __host__ __device__ static constexpr int K1P(int m) { return (K1(m) + 31) / 32 * 32; }
  __host__ __device__ static constexpr int N1(int m) { return G::rows(m) * 2 * E; }  // lin1 N == lin2 K
  __host__ __device__ static constexpr int N2(int m) { return G::rows(m) * E; }
  __host__ __device__ static constexpr int kofs(int m) {
    int s = 0;
    for (int q = 0; q < m; ++q) s += K1P(q);
    return s;
  }
  static constexpr int KTOT = kofs(L + 1);
  static constexpr int KCH = KTOT / 32;  // A1 chunks per tile
  __host__ __device__ static int w1_off(int m) {  // bytes
    int o = 0;
    for (int q = 0; q < m; ++q) o += N1(q) * K1P(q) * 4;
    return o;
  }
  __host__ __device__ static int w2_off(int m) {
    int o = 0;
    for (int q = 0; q < m; ++q) o += N2(q) * N1(q) * 4;
    return o;
  }
  // lin2 of order m writes the head of lin1's region: the gate must have read
  // these leading chunks before lin2's first MMA
  __host__ __device__ static constexpr int ych(int m) { return (N2(m) + 31) / 32; }
};

__device__ __forceinline__ uint32_t idesc_f16(int N) {  // D f32, A/B f16, K-major, M = 128
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(TILE_M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// one 32-wide K chunk: two K = 16 steps x (hi.hi, hi.lo, lo.hi); the lo half
// of a 128-byte row starts 64 bytes in (descriptor start + 4)
__device__ __forceinline__ void mma_chunk(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, bool first) {
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    mma_f16(tmem_d, da + 2 * ks, db + 2 * ks, idesc, (first && ks == 0) ? 0u : 1u);
    mma_f16(tmem_d, da + 2 * ks, db + 4 + 2 * ks, idesc, 1u);
    mma_f16(tmem_d, da + 4 + 2 * ks, db + 2 * ks, idesc, 1u);
  }
}

// TMEM column plan (l_max 4, e_width 16; N1 = 160 256 192 128 64, N2 = N1/2):
// lin1 of order m accumulates into R_m = [R0[m], R0[m] + N1); lin2 then
// accumulates Y_m into its head [R0[m], R0[m] + N2), chunk by chunk behind the
// gate, once the gate has read those leading columns.  Consecutive orders'
// regions are disjoint (lin1 of order m + 1 runs while order m is gated).
// lin1 of unit u waits until units < u - LAG[m] are drained: the most recent
// earlier unit whose Y overlaps R_m (Y2 for m0, Y3 for m1, Y0 for m2, Y1 for
// m3, the previous tile's Y4 for m4); gate reads of earlier units are ordered
// by the MMA issue order (lin2 of u - 2 issues its last chunk only after the
// gate wrote it).
__device__ __forceinline__ int r0_col(int m) { return m == 1 || m == 3 ? 0 : (m == 4 ? 448 : 256); }
__device__ __forceinline__ int lag(int m) { return m <= 1 ? 2 : (m <= 3 ? 1 : 4); }

__device__ __forceinline__ uint32_t ld_acquire(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];\n" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t addr, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t h2(__half a, __half b) {
  return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}

template <int L, int E>
__global__ void __launch_bounds__(THREADS, 1)
    k_so2_f16x3(const uint8_t* __restrict__ A1, int64_t n_e, const uint8_t* __restrict__ W1,
                const uint8_t* __restrict__ W2, F16x3Scales sc, const float* __restrict__ tmax, int edge_slot,
                float* __restrict__ Y, int gate, const float* __restrict__ att, float* __restrict__ logits) {
  using G = Geo<L>;
  using S = S3<L, E>;
  static_assert(2 * E == 32, "gate scalars assume 2E = 32");
  static_assert(L == 4 && E == 16, "TMEM column plan is laid out for l_max 4, e_width 16");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sA = smem_u32(base);
  const uint32_t sB = sA + NSA * CHUNK;
  const uint32_t sA2 = sB + NSB * B_STAGE;
  uint64_t* bars = (uint64_t*)(base + NSA * CHUNK + NSB * B_STAGE + NS2 * CHUNK);
  auto bar = [&](int i) { return smem_u32(&bars[i]); };
  const int FA = 0, EA = NSA, FB = 2 * NSA, EB = FB + NSB;
  const int F2 = EB + NSB, E2 = F2 + NS2;  // gated-operand ring
  const int L1F = E2 + NS2;                // + (u & 1): lin1 of unit u complete
  const int L2F = L1F + 2;                 // + (u & 1): lin2 of unit u complete
  const int H1 = L2F + 2;                  // + (u & 1): the gate read the Y head of unit u
  uint32_t* drained = (uint32_t*)(bars + H1 + 2);
  uint32_t* tmem_slot = drained + 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NSA; ++s) {
      mbar_init(bar(FA + s), 1);
      mbar_init(bar(EA + s), 1);
    }
    for (int s = 0; s < NSB; ++s) {
      mbar_init(bar(FB + s), 1);
      mbar_init(bar(EB + s), 1);
    }
    for (int s = 0; s < NS2; ++s) {
      mbar_init(bar(F2 + s), GATE_THREADS / 2);  // one half of the gate writes a chunk
      mbar_init(bar(E2 + s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(L1F + b), 1);
      mbar_init(bar(L2F + b), 1);
      mbar_init(bar(H1 + b), GATE_THREADS);
    }
    *drained = 0;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t n_tiles = (n_e + TILE_M - 1) / TILE_M;

  if (warp == 0) {
    // ---------------------------------------------------------- A producer
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      const uint64_t pol = policy_evict_first();
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint8_t* a_tile = A1 + (size_t)tile * S::KCH * CHUNK;
        for (int c = 0; c < S::KCH; ++c) {
          mbar_wait(bar(EA + st), ph ^ 1);
          mbar_expect_tx(bar(FA + st), CHUNK);
          bulk_g2s(sA + st * CHUNK, a_tile + (size_t)c * CHUNK, CHUNK, bar(FA + st), pol);
          if (++st == NSA) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 18) {
    // ---------------------------------------------------------- B producer
    // weights in MMA issue order: lin1 of unit u, then lin2 of unit u - 1
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      const uint64_t pol = policy_evict_last();
      auto load = [&](const uint8_t* src, uint32_t bytes) {
        mbar_wait(bar(EB + st), ph ^ 1);
        mbar_expect_tx(bar(FB + st), bytes);
        bulk_g2s(sB + st * B_STAGE, src, bytes, bar(FB + st), pol);
        if (++st == NSB) { st = 0; ph ^= 1; }
      };
      auto load_w2 = [&](int m) {
        const uint8_t* w2 = W2 + S::w2_off(m);
        for (int j = 0; j < S::N1(m) / 32; ++j) load(w2 + (size_t)j * S::N2(m) * 128, S::N2(m) * 128);
      };
      int prev = -1;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x)
        for (int m = 0; m <= L; ++m) {
          const uint8_t* w1 = W1 + S::w1_off(m);
          for (int c = 0; c < S::K1P(m) / 32; ++c) load(w1 + (size_t)c * S::N1(m) * 128, S::N1(m) * 128);
          if (prev >= 0) load_w2(prev);
          prev = m;
        }
      if (prev >= 0) load_w2(prev);
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    int sa = 0, sb = 0;
    uint32_t pa = 0, pb = 0;
    uint32_t g2 = 0;  // gated-operand chunks consumed so far
    const uint32_t drained_addr = smem_u32(drained);
    auto wait_drained = [&](int need) {
      if (need > 0)
        while ((int)ld_acquire(drained_addr) < need) {
        }
    };
    auto lin2 = [&](int m, int u) {
      wait_drained(u - 1);  // Y of unit u - 2 drained: L2F[u & 1] cannot run ahead
      mbar_wait(bar(H1 + (u & 1)), (u >> 1) & 1);  // the gate read the columns Y_m overwrites
      tc_fence_after();
      const uint32_t id2 = idesc_f16(S::N2(m));
      const uint32_t t_y = tmem + r0_col(m);
      for (int j = 0; j < S::N1(m) / 32; ++j, ++g2) {
        const int s2 = (int)(g2 % NS2);
        mbar_wait(bar(F2 + s2), (g2 / NS2) & 1);
        mbar_wait(bar(FB + sb), pb);
        tc_fence_after();
        if (elect_one()) {
          mma_chunk(t_y, sdesc(sA2 + s2 * CHUNK), sdesc(sB + sb * B_STAGE), id2, j == 0);
          tc_commit(bar(E2 + s2));
          tc_commit(bar(EB + sb));
        }
        __syncwarp();
        if (++sb == NSB) { sb = 0; pb ^= 1; }
      }
      if (elect_one()) tc_commit(bar(L2F + (u & 1)));
      __syncwarp();
    };
    int u = 0, prev_m = -1;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x)
      for (int m = 0; m <= L; ++m, ++u) {
        wait_drained(u - lag(m));
        tc_fence_after();
        const uint32_t id1 = idesc_f16(S::N1(m)), t_r = tmem + r0_col(m);
        for (int c = 0; c < S::K1P(m) / 32; ++c) {
          mbar_wait(bar(FA + sa), pa);
          mbar_wait(bar(FB + sb), pb);
          tc_fence_after();
          if (elect_one()) {
            mma_chunk(t_r, sdesc(sA + sa * CHUNK), sdesc(sB + sb * B_STAGE), id1, c == 0);
            tc_commit(bar(EA + sa));
            tc_commit(bar(EB + sb));
          }
          __syncwarp();
          if (++sa == NSA) { sa = 0; pa ^= 1; }
          if (++sb == NSB) { sb = 0; pb ^= 1; }
        }
        if (elect_one()) tc_commit(bar(L1F + (u & 1)));
        __syncwarp();
        if (prev_m >= 0) lin2(prev_m, u - 1);
        prev_m = m;
      }
    if (prev_m >= 0) lin2(prev_m, u - 1);
  } else if (warp >= 2 && warp <= 9) {
    // ---------------------------------------------------------------- gate
    const int quad = warp & 3, half = (warp - 2) >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float bound_a = 3.f * fmaxf(tmax[0], tmax[edge_slot]);
    const float sa_scale = f16s_pow2_scale(bound_a);
    float sg[32];
    uint32_t gbase = 0;
    int u = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x)
      for (int m = 0; m <= L; ++m, ++u) {
        const uint32_t t_r = tmem + lane_off + r0_col(m);
        const int nch = S::N1(m) / 32, ych = S::ych(m);
        const float sc1 = sa_scale * sc.w1[m];  // lin1 accumulator -> fp32 units
        const float s2 = f16s_pow2_scale(sc.w1inf[m] * bound_a);
        const float inv_s2 = 1.f / s2;  // a power of two: exact
        mbar_sleep(bar(L1F + (u & 1)), (u >> 1) & 1);
        tc_fence_after();
        if (m == 0) {  // gate scalars from the l = 0 channels of order 0 (kernels.h:210-226)
          float v[32];
          tmem_ld32(t_r, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) sg[i] = gate ? 1.f / (1.f + expf(-v[i] * sc1)) : 1.f;
        }
        bool head_done = false;
        for (int q = half; q < nch; q += 2) {
          if (!head_done && q >= ych) {
            tc_fence_before();
            mbar_arrive(bar(H1 + (u & 1)));
            head_done = true;
          }
          float v[32];
          tmem_ld32(t_r + q * 32, v);
          const uint32_t gq = gbase + (uint32_t)q, s2i = gq % NS2;
          mbar_sleep(bar(E2 + s2i), ((gq / NS2) & 1) ^ 1);  // lin2 finished reading this stage
          const uint32_t cb = sA2 + s2i * CHUNK;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            __half hi[8], lo[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              const float x = v[8 * j + t] * sc1 * sg[8 * j + t] * inv_s2;
              hi[t] = __float2half_rn(x);
              lo[t] = __float2half_rn(x - __half2float(hi[t]));
            }
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(cb + sw128(row, j)), "r"(h2(hi[0], hi[1])),
                         "r"(h2(hi[2], hi[3])), "r"(h2(hi[4], hi[5])), "r"(h2(hi[6], hi[7]))
                         : "memory");
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(cb + sw128(row, 4 + j)), "r"(h2(lo[0], lo[1])),
                         "r"(h2(lo[2], lo[3])), "r"(h2(lo[4], lo[5])), "r"(h2(lo[6], lo[7]))
                         : "memory");
          }
          fence_async_smem();
          mbar_arrive(bar(F2 + s2i));
        }
        if (!head_done) {
          tc_fence_before();
          mbar_arrive(bar(H1 + (u & 1)));
        }
        gbase += (uint32_t)nch;
      }
  } else if (warp >= 10 && warp <= 17) {
    // --------------------------------------------------------------- drain
    const int quad = warp & 3, half = (warp - 10) >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float bound_a = 3.f * fmaxf(tmax[0], tmax[edge_slot]);
    int u = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const int64_t e0 = tile * TILE_M;
      const bool valid = e0 + row < n_e;
      float* yrow = Y + (e0 + row) * (int64_t)(G::H * E);
      for (int m = 0; m <= L; ++m, ++u) {
        const int N2 = S::N2(m);
        const uint32_t t_y = tmem + lane_off + r0_col(m);
        const float sy = f16s_pow2_scale(sc.w1inf[m] * bound_a) * sc.w2[m];
        mbar_sleep(bar(L2F + (u & 1)), (u >> 1) & 1);
        tc_fence_after();
        const int c0 = G::moff(m) * E;
        for (int q = half; q * 32 < N2; q += 2) {
          float v[32];
          tmem_ld32(t_y + q * 32, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] *= sy;
          if (m == 0 && q == 0 && logits != nullptr && valid) {
            // ops.h:203-209 attention logit from the l = 0 channels (msg row 0
            // == y row 0 since D_0 = 1), sequential fp32 as the reference
            float lg = 0.f;
#pragma unroll
            for (int c = 0; c < E; ++c) lg = fmaf(__ldg(att + c), v[c], lg);
            logits[e0 + row] = lg;
          }
          if (valid) {
            const int nv = (N2 - q * 32) < 32 ? (N2 - q * 32) : 32;
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              if (i < nv)
                *reinterpret_cast<float4*>(yrow + c0 + q * 32 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          }
        }
        tc_fence_before();
        asm volatile("bar.sync 1, %0;\n" ::"n"(DRAIN_THREADS) : "memory");  // all drain lanes read their Y
        if (warp == 10 && lane == 0) st_release(smem_u32(drained), (uint32_t)(u + 1));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

}  // namespace

bool so2_f16x3_available(int L, int E) { return L == 4 && E == 16; }

// bytes of the split A1 image per 128-edge tile, and of the W1 / W2 images
int64_t so2_f16x3_a1_tile_bytes(int L, int E) { return (int64_t)S3<4, 16>::KCH * CHUNK; }
int64_t so2_f16x3_w1_bytes(int L, int E) { return S3<4, 16>::w1_off(5); }
int64_t so2_f16x3_w2_bytes(int L, int E) { return S3<4, 16>::w2_off(5); }
int so2_f16x3_kofs(int m) { return S3<4, 16>::kofs(m); }
int so2_f16x3_ktot() { return S3<4, 16>::KTOT; }

void so2_f16x3_launch(int L, int E, const uint8_t* A1, int64_t n_e, const uint8_t* W1, const uint8_t* W2,
                      const F16x3Scales& sc, const float* tmax, int edge_slot, float* Y, int gate, const float* att,
                      float* logits, cudaStream_t st) {
  if (!so2_f16x3_available(L, E)) usage("fp16x3 SO(2) chain is instantiated for l_max 4, e_width 16");
  int dev = 0;
  ESG_CUDA(cudaGetDevice(&dev));
  static int n_sm[64] = {0};
  if (dev < 0 || dev >= 64) usage("device index out of range");
  if (!n_sm[dev]) {
    ESG_CUDA(cudaFuncSetAttribute(k_so2_f16x3<4, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    ESG_CUDA(cudaDeviceGetAttribute(&n_sm[dev], cudaDevAttrMultiProcessorCount, dev));
  }
  const int64_t tiles = (n_e + TILE_M - 1) / TILE_M;
  const int grid = (int)(tiles < n_sm[dev] ? tiles : n_sm[dev]);
  if (grid > 0)
    k_so2_f16x3<4, 16><<<grid, THREADS, SMEM_BYTES, st>>>(A1, n_e, W1, W2, sc, tmax, edge_slot, Y, gate, att,
                                                          logits);
  ESG_CUDA(cudaGetLastError());
}

}  // namespace esg
