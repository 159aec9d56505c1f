// so2_tc.cu -- the SO(2) linear chain on the 5th-gen tensor cores.
//
// Per tile of 128 edges (UMMA M = 128, one edge per TMEM lane) and per order
// m = 0..L (kernels.h:133-161, :210-226; network.h:144-146):
//   lin1   H_m[128 x N1] = A1_m[128 x K1] . W1_m^T   tcgen05.mma kind::f16
//          bf16 operands in SMEM (SWIZZLE_128B, K-major), fp32 accumulator
//          in TMEM columns [0, 256)
//   gate   s = sigmoid(H_0[:, l = 0 channels]) (m = 0 first), H_m * s[c % 2E]
//          -> bf16 A2 in SMEM (TMEM -> registers -> SMEM)
//   lin2   Y_m[128 x N2] = A2_m . W2_m^T, accumulator in TMEM [256, 384),
//          drained to the fp32 order-major Y rows in HBM.
// W_m are the expanded [[Wr, Wi], [-Wi, Wr]] order blocks (K padded to 64).
//
// Both operands are stored in HBM already in the SMEM image the UMMA
// descriptors expect (128-byte rows, 16-byte units XOR-swizzled by row % 8,
// one contiguous block per 64-wide K chunk), so every chunk is a single
// cp.async.bulk (TMA, 1-D) that completes on an mbarrier -- no tensor maps.
//
// Warp roles (352 threads, 1 CTA per SM, persistent over tiles):
//   warp 0     A producer: one lane streams A1 chunks through a 4-stage ring
//   warp 10    B producer: one lane streams weight chunks through a 3-stage ring
//   warp 1     MMA issuer: one lane issues tcgen05.mma, commits free stages
//   warps 2-9  epilogue: gate and Y drain; warp w owns TMEM lanes 32*(w%4)+
//              and the even (w < 6) or odd (w >= 6) 64-column chunks, and
//              hands each gated A2 chunk to lin2 through its own mbarrier so
//              lin2 runs while the rest of the gate is still being computed.
#include <cuda_runtime.h>

#include <cstdint>

#include "esg_internal.h"
#include "model_kernels.cuh"

namespace esg {
namespace {

constexpr int TILE_M = 128;
constexpr int THREADS = 352;
constexpr int NSA = 4;                  // A1 ring (streamed from HBM)
constexpr int NSB = 3;                  // weight ring (L2-resident)
constexpr int A_CHUNK = TILE_M * 128;   // 64 bf16 K x 128 rows = 16 KB
constexpr int B_CHUNK = 256 * 128;      // up to 256 rows x 64 K = 32 KB
constexpr int A2_BYTES = TILE_M * 256 * 2;
constexpr int SMEM_BYTES = 1024 + NSA * A_CHUNK + NSB * B_CHUNK + A2_BYTES + 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t sw128(int r, int c) { return uint32_t(r * 128 + ((c ^ (r & 7)) << 4)); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
// L2 policies: A1 tiles are read once (evict first), weights by every tile (evict last)
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar) : "memory");
}

// SMEM matrix descriptor: K-major, SWIZZLE_128B, SBO = 1024 B between 8-row
// groups, LBO unused for swizzled K-major (1), version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M = 128.
__device__ __forceinline__ uint32_t idesc_bf16(int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(TILE_M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
  ua += 0x7fffu + ((ua >> 16) & 1u);
  ub += 0x7fffu + ((ub >> 16) & 1u);
  return (ua >> 16) | (ub & 0xffff0000u);
}

template <int L, int E>
struct Shape {
  using Y1 = Lay1<L, E, 64>;
  static constexpr int KCH = Y1::KTOT / 64;  // A1 chunks per tile
  __device__ static int w1_off(int m) {     // byte offset of order m in packed W1
    int o = 0;
    for (int q = 0; q < m; ++q) o += Y1::N1(q) * Y1::KP(q) * 2;
    return o;
  }
  __device__ static int w2_off(int m) {
    int o = 0;
    for (int q = 0; q < m; ++q) o += Y1::N2(q) * Y1::N1P(q) * 2;
    return o;
  }
};

template <int L, int E>
__global__ void __launch_bounds__(THREADS, 1)
    k_so2_tc(const uint8_t* __restrict__ A1, int64_t n_e, const uint8_t* __restrict__ W1,
             const uint8_t* __restrict__ W2, uint16_t* __restrict__ Y, int gate, const float* __restrict__ att,
             float* __restrict__ logits) {
  using G = Geo<L>;
  using S = Shape<L, E>;
  using Y1 = typename S::Y1;
  static_assert(2 * E == 32, "gate scalars assume 2E = 32");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sA = smem_u32(base);
  const uint32_t sB = sA + NSA * A_CHUNK;
  const uint32_t sA2 = sB + NSB * B_CHUNK;
  uint64_t* bars = (uint64_t*)(base + NSA * A_CHUNK + NSB * B_CHUNK + A2_BYTES);
  auto bar = [&](int i) { return smem_u32(&bars[i]); };
  const int FA = 0, EA = NSA, FB = 2 * NSA, EB = 2 * NSA + NSB;
  const int L1F = 2 * NSA + 2 * NSB, L2F = L1F + 1, L2E = L1F + 2, A2F = L1F + 3;  // A2F + chunk (4)
  uint32_t* tmem_slot = (uint32_t*)(bars + A2F + 4);
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
    mbar_init(bar(L1F), 1);
    mbar_init(bar(A2F), 256);  // chunk 0 is gated by both epilogue halves
    for (int c = 1; c < 4; ++c) mbar_init(bar(A2F + c), 128);
    mbar_init(bar(L2F), 1);
    mbar_init(bar(L2E), 256);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot, t_h = tmem, t_y = tmem + 256;
  const int64_t n_tiles = (n_e + TILE_M - 1) / TILE_M;

  if (warp == 0) {
    // ---------------------------------------------------------- A producer
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      const uint64_t pol = policy_evict_first();
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint8_t* a_tile = A1 + (size_t)tile * S::KCH * A_CHUNK;
        for (int c = 0; c < S::KCH; ++c) {  // order-major chunks in m order
          mbar_wait(bar(EA + st), ph ^ 1);
          mbar_expect_tx(bar(FA + st), A_CHUNK);
          bulk_g2s(sA + st * A_CHUNK, a_tile + (size_t)c * A_CHUNK, A_CHUNK, bar(FA + st), pol);
          if (++st == NSA) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 10) {
    // ---------------------------------------------------------- B producer
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      const uint64_t pol = policy_evict_last();
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int m = 0; m <= L; ++m) {
          const int N1 = Y1::N1(m), N2 = Y1::N2(m);
          const uint8_t* w1 = W1 + S::w1_off(m);
          for (int j = 0; j < Y1::KP(m) / 64; ++j) {
            mbar_wait(bar(EB + st), ph ^ 1);
            mbar_expect_tx(bar(FB + st), N1 * 128);
            bulk_g2s(sB + st * B_CHUNK, w1 + (size_t)j * N1 * 128, N1 * 128, bar(FB + st), pol);
            if (++st == NSB) { st = 0; ph ^= 1; }
          }
          const uint8_t* w2 = W2 + S::w2_off(m);
          for (int j = 0; j < Y1::N1P(m) / 64; ++j) {
            mbar_wait(bar(EB + st), ph ^ 1);
            mbar_expect_tx(bar(FB + st), N2 * 128);
            bulk_g2s(sB + st * B_CHUNK, w2 + (size_t)j * N2 * 128, N2 * 128, bar(FB + st), pol);
            if (++st == NSB) { st = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0, l2e = 0, a2p[4] = {0, 0, 0, 0};
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int m = 0; m <= L; ++m) {
          const int N1 = Y1::N1(m), N2 = Y1::N2(m);
          const uint32_t id1 = idesc_bf16(N1), id2 = idesc_bf16(N2);
          for (int j = 0; j < Y1::KP(m) / 64; ++j) {
            mbar_wait(bar(FA + sa), pa);
            mbar_wait(bar(FB + sb), pb);
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_bf16(t_h, sdesc(sA + sa * A_CHUNK + k * 32), sdesc(sB + sb * B_CHUNK + k * 32), id1, (j | k) ? 1u : 0u);
            tc_commit(bar(EA + sa));
            tc_commit(bar(EB + sb));
            if (++sa == NSA) { sa = 0; pa ^= 1; }
            if (++sb == NSB) { sb = 0; pb ^= 1; }
          }
          tc_commit(bar(L1F));
          mbar_wait(bar(L2E), l2e ^ 1);  // previous lin2 accumulator drained
          l2e ^= 1;
          for (int j = 0; j < Y1::N1P(m) / 64; ++j) {
            mbar_wait(bar(A2F + j), a2p[j]);  // gated chunk j of order m is in A2
            a2p[j] ^= 1;
            mbar_wait(bar(FB + sb), pb);
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_bf16(t_y, sdesc(sA2 + j * A_CHUNK + k * 32), sdesc(sB + sb * B_CHUNK + k * 32), id2, (j | k) ? 1u : 0u);
            tc_commit(bar(EB + sb));
            if (++sb == NSB) { sb = 0; pb ^= 1; }
          }
          tc_commit(bar(L2F));
        }
      }
    }
  } else if (warp >= 2 && warp <= 9) {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3, half = (warp - 2) >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    uint32_t l1p = 0, l2p = 0;
    float s[32];
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const int64_t e0 = tile * TILE_M;
      const bool valid = e0 + row < n_e;
      for (int m = 0; m <= L; ++m) {
        const int N1 = Y1::N1(m), N1P = Y1::N1P(m), N2 = Y1::N2(m);
        mbar_wait(bar(L1F), l1p);
        l1p ^= 1;
        tc_fence_after();
        if (m == 0) {  // gate scalars from the l = 0 channels of order 0
          float v[32];
          tmem_ld32(t_h + lane_off, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) s[i] = gate ? 1.f / (1.f + __expf(-v[i])) : 1.f;
        }
        // chunk 0 (columns 0..63) is split across the halves so lin2 can start
        // as early as possible; chunks 1.. alternate between the halves
        for (int c2 = 0; c2 < N1P / 64; ++c2) {
          if (c2 > 0 && (c2 & 1) != (half ^ 1)) continue;
          const uint32_t cb = sA2 + (uint32_t)c2 * A_CHUNK;
#pragma unroll
          for (int hq = 0; hq < 2; ++hq) {
            if (c2 == 0 && hq != half) continue;
            const int q = 2 * c2 + hq;
            float v[32];
            if (q * 32 < N1) {
              tmem_ld32(t_h + lane_off + q * 32, v);
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] *= s[i];
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0.f;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int c = hq * 4 + j;
              asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(cb + sw128(row, c)),
                           "r"(pack_bf16(v[8 * j], v[8 * j + 1])), "r"(pack_bf16(v[8 * j + 2], v[8 * j + 3])),
                           "r"(pack_bf16(v[8 * j + 4], v[8 * j + 5])), "r"(pack_bf16(v[8 * j + 6], v[8 * j + 7]))
                           : "memory");
            }
          }
          fence_async_smem();
          tc_fence_before();
          mbar_arrive(bar(A2F + c2));
        }
        mbar_wait(bar(L2F), l2p);
        l2p ^= 1;
        tc_fence_after();
        uint16_t* yrow = Y + (e0 + row) * (G::H * E) + G::moff(m) * E;  // bf16 order-major rows
        for (int q = half; q * 32 < N2; q += 2) {
          float v[32];
          tmem_ld32(t_y + lane_off + q * 32, v);
          if (m == 0 && q == 0 && logits != nullptr && valid) {
            // ops.h:203-209 attention logit from the l = 0 channels (msg row 0
            // == y row 0 since D_0 = 1), taken from the fp32 accumulator
            float lg = 0.f;
#pragma unroll
            for (int c = 0; c < E; ++c) lg = fmaf(__ldg(att + c), v[c], lg);
            logits[e0 + row] = lg;
          }
          if (valid) {
            const int nv = (N2 - q * 32) < 32 ? (N2 - q * 32) : 32;
#pragma unroll
            for (int i = 0; i < 32; i += 8)
              if (i < nv)
                *(uint4*)(yrow + q * 32 + i) = make_uint4(pack_bf16(v[i], v[i + 1]), pack_bf16(v[i + 2], v[i + 3]),
                                                          pack_bf16(v[i + 4], v[i + 5]), pack_bf16(v[i + 6], v[i + 7]));
          }
        }
        tc_fence_before();
        mbar_arrive(bar(L2E));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

}  // namespace

bool so2_tc_available(int L, int E) { return L == 4 && E == 16; }

// A1: tiled, pre-swizzled bf16 operand (so2_tc_a1_bytes per chunk); W1/W2
// packed by so2_tc_pack_weights.
void so2_tc_launch(int L, int E, const uint16_t* A1, int64_t n_e, const uint16_t* W1, const uint16_t* W2,
                   uint16_t* Y, int gate, const float* att, float* logits, cudaStream_t st) {
  if (!so2_tc_available(L, E)) usage("tcgen05 SO(2) chain is instantiated for l_max 4, e_width 16");
  static int n_sm = 0;
  if (!n_sm) {
    ESG_CUDA(cudaFuncSetAttribute(k_so2_tc<4, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    int dev = 0;
    ESG_CUDA(cudaGetDevice(&dev));
    ESG_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  }
  const int64_t tiles = (n_e + TILE_M - 1) / TILE_M;
  const int grid = (int)(tiles < n_sm ? tiles : n_sm);
  if (grid > 0)
    k_so2_tc<4, 16><<<grid, THREADS, SMEM_BYTES, st>>>((const uint8_t*)A1, n_e, (const uint8_t*)W1,
                                                       (const uint8_t*)W2, Y, gate, att, logits);
  ESG_CUDA(cudaGetLastError());
}

}  // namespace esg
