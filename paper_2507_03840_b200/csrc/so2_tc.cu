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
//   warp 18    B producer: one lane streams weight chunks through a 3-stage ring
//   warp 1     MMA issuer: one elected lane issues tcgen05.mma, commits stages
//   warps 2-9  gate: warp w owns TMEM lanes 32*(w%4)+ and half of the 64-column
//              chunks; each gated A2 chunk goes to lin2 through its own
//              mbarrier, so lin2 runs while the rest of the gate is computed
//   warps 10-17 drain: lin2 accumulator -> bf16 Y rows (+ attention logits),
//              overlapping the next order's gate.
#include <cuda_runtime.h>

#include <cstdint>

#include "esg_internal.h"
#include "model_kernels.cuh"
#include "tc_common.cuh"

namespace esg {
namespace {
using namespace tc;

constexpr int TILE_M = 128;
constexpr int THREADS = 608;
constexpr int NSA = 4;                  // A1 ring (streamed from HBM)
constexpr int NSB = 3;                  // weight ring (L2-resident)
constexpr int A_CHUNK = TILE_M * 128;   // 64 bf16 K x 128 rows = 16 KB
constexpr int B_STAGE = 256 * 128;      // up to 256 weight rows x 64 K = 32 KB
constexpr int A2_BYTES = TILE_M * 256 * 2;  // gated operand of one order, 64 KB
constexpr int GATE_THREADS = 256, DRAIN_THREADS = 256;
constexpr int SMEM_BYTES = 1024 + NSA * A_CHUNK + NSB * B_STAGE + A2_BYTES + 256;

// SO2_PROBE (tools/so2_probe.cu only): per-role clock64 accounting of the
// mbarrier waits; compiled out of the library.
#ifdef SO2_PROBE
__device__ long long g_so2_probe[1024 * 32];
#define PW(slot, ...)                  \
  do {                                 \
    const long long _t = clock64();    \
    __VA_ARGS__;                       \
    prb[slot] += clock64() - _t;       \
  } while (0)
#define PROBE_DECL long long prb[32] = {}; const long long prb_t0 = clock64(); long long prb_m = 0
#define PROBE_MARK(slot) prb_m = clock64()
__device__ long long g_so2_trace[256];
#define PT(tile, idx)                                                            \
  do {                                                                           \
    if (blockIdx.x == 0 && (tile) == 2 * (int64_t)gridDim.x) g_so2_trace[idx] = clock64(); \
  } while (0)
#define PROBE_ACC(slot) prb[slot] += clock64() - prb_m
#define PROBE_END(total_slot, cond)                                                          \
  do {                                                                                       \
    if (cond) {                                                                              \
      prb[total_slot] = clock64() - prb_t0;                                                  \
      for (int _i = 0; _i < 32; ++_i)                                                        \
        if (prb[_i]) g_so2_probe[blockIdx.x * 32 + _i] = prb[_i];                            \
    }                                                                                        \
  } while (0)
#else
#define PW(slot, ...) __VA_ARGS__
#define PROBE_MARK(slot)
#define PROBE_ACC(slot)
#define PT(tile, idx)
#define PROBE_DECL
#define PROBE_END(total_slot, cond)
#endif

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
// two fp32 -> packed bf16x2 (round to nearest even), a in the low half
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;\n" : "=r"(r) : "f"(b), "f"(a));
  return r;
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

// TMEM column plan (l_max 4, e_width 16; N1 = 160 256 192 128 64, N2 = N1/2).
// lin1 of order m accumulates into R_m = [R0[m], R0[m] + N1); once the gate
// has consumed it, lin2 accumulates Y_m into its tail [R0[m] + N1 - N2, ...).
// Consecutive orders' regions are disjoint, so lin1 of order m + 1 runs while
// order m is gated; a region is reused only after every Y overlapping it has
// been drained: lin1 of unit u waits for units < u - LAG[m] to be drained.
__device__ __forceinline__ int r0_col(int m) { return m == 1 || m == 3 ? 0 : (m == 4 ? 448 : 256); }
__device__ __forceinline__ int lag(int m) { return m <= 1 ? 2 : (m == 2 ? 1 : 4); }

__device__ __forceinline__ uint32_t ld_acquire(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];\n" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t addr, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}

template <int L, int E>
__global__ void __launch_bounds__(THREADS, 1)
    k_so2_tc(const uint8_t* __restrict__ A1, int64_t n_e, const uint8_t* __restrict__ W1,
             const uint8_t* __restrict__ W2, uint16_t* __restrict__ Y, int gate, const float* __restrict__ att,
             float* __restrict__ logits) {
  using G = Geo<L>;
  using S = Shape<L, E>;
  using Y1 = typename S::Y1;
  static_assert(2 * E == 32, "gate scalars assume 2E = 32");
  static_assert(L == 4 && E == 16, "TMEM column plan is laid out for l_max 4, e_width 16");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sA = smem_u32(base);
  const uint32_t sB = sA + NSA * A_CHUNK;
  const uint32_t sA2 = sB + NSB * B_STAGE;
  uint64_t* bars = (uint64_t*)(base + NSA * A_CHUNK + NSB * B_STAGE + A2_BYTES);
  auto bar = [&](int i) { return smem_u32(&bars[i]); };
  const int FA = 0, EA = NSA, FB = 2 * NSA, EB = 2 * NSA + NSB;
  const int L1F = 2 * NSA + 2 * NSB;  // + (unit & 1): lin1 of the unit complete
  const int L2F = L1F + 2;            // + (unit & 1): lin2 of the unit complete
  const int A2F = L2F + 2;            // gated operand of the unit written to A2
  const int A2E = A2F + 1;            // lin2 of the unit finished reading A2
  uint32_t* drained = (uint32_t*)(bars + A2E + 1);  // units drained so far
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
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(L1F + b), 1);
      mbar_init(bar(L2F + b), 1);
    }
    mbar_init(bar(A2F), GATE_THREADS);
    mbar_init(bar(A2E), 1);
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
      PROBE_DECL;
      int st = 0;
      uint32_t ph = 0;
      const uint64_t pol = policy_evict_first();
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint8_t* a_tile = A1 + (size_t)tile * S::KCH * A_CHUNK;
        for (int c = 0; c < S::KCH; ++c) {  // order-major chunks in m order
          PW(6, mbar_wait(bar(EA + st), ph ^ 1));
          mbar_expect_tx(bar(FA + st), A_CHUNK);
          bulk_g2s(sA + st * A_CHUNK, a_tile + (size_t)c * A_CHUNK, A_CHUNK, bar(FA + st), pol);
          if (++st == NSA) { st = 0; ph ^= 1; }
        }
      }
      PROBE_END(7, true);
    }
  } else if (warp == 18) {
    // ---------------------------------------------------------- B producer
    // weights in MMA issue order: lin1 of unit u, then lin2 of unit u - 1
    if (lane == 0) {
      PROBE_DECL;
      int st = 0;
      uint32_t ph = 0;
      const uint64_t pol = policy_evict_last();
      auto load = [&](const uint8_t* src, uint32_t bytes) {
        PW(8, mbar_wait(bar(EB + st), ph ^ 1));
        mbar_expect_tx(bar(FB + st), bytes);
        bulk_g2s(sB + st * B_STAGE, src, bytes, bar(FB + st), pol);
        if (++st == NSB) { st = 0; ph ^= 1; }
      };
      auto load_w2 = [&](int m) {
        const uint8_t* w2 = W2 + S::w2_off(m);
        for (int j = 0; j < Y1::N1P(m) / 64; ++j) load(w2 + (size_t)j * Y1::N2(m) * 128, Y1::N2(m) * 128);
      };
      int prev = -1;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x)
        for (int m = 0; m <= L; ++m) {
          const uint8_t* w1 = W1 + S::w1_off(m);
          for (int c = 0; c < Y1::KP(m) / 64; ++c) load(w1 + (size_t)c * Y1::N1(m) * 128, Y1::N1(m) * 128);
          if (prev >= 0) load_w2(prev);
          prev = m;
        }
      if (prev >= 0) load_w2(prev);
      PROBE_END(9, true);
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    // unit u = (tile, m) in issue order: lin1(u), then lin2(u - 1). The whole
    // warp runs the loop; one elected lane issues the MMAs and commits.
    {
      PROBE_DECL;
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      const uint32_t drained_addr = smem_u32(drained);
      auto wait_drained = [&](int need) {
        if (need > 0)
          while ((int)ld_acquire(drained_addr) < need) {
          }
      };
      auto lin2 = [&](int m, int u) {
        PW(18, wait_drained(u - 1));  // Y of unit u - 2 drained: L2F[u & 1] cannot run ahead
        PW(3, mbar_wait(bar(A2F), u & 1));  // gated operand of unit u is in A2
        tc_fence_after();
        const uint32_t id2 = idesc_bf16(Y1::N2(m));
        const uint32_t t_y = tmem + r0_col(m) + Y1::N1(m) - Y1::N2(m);
        for (int j = 0; j < Y1::N1P(m) / 64; ++j) {
          PW(4, mbar_wait(bar(FB + sb), pb));
          tc_fence_after();
          PW(17, {
            if (elect_one()) {
              const uint64_t da = sdesc(sA2 + j * A_CHUNK), db = sdesc(sB + sb * B_STAGE);
#pragma unroll
              for (int k = 0; k < 4; ++k) mma_bf16(t_y, da + 2 * k, db + 2 * k, id2, (j | k) ? 1u : 0u);
              tc_commit(bar(EB + sb));
            }
            __syncwarp();
          });
          if (++sb == NSB) { sb = 0; pb ^= 1; }
        }
        if (elect_one()) {
          tc_commit(bar(A2E));
          tc_commit(bar(L2F + (u & 1)));
        }
        __syncwarp();
      };
      int u = 0, prev_m = -1;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x)
        for (int m = 0; m <= L; ++m, ++u) {
          PW(2, {
            wait_drained(u - lag(m));
            tc_fence_after();
          });
          const uint32_t id1 = idesc_bf16(Y1::N1(m)), t_r = tmem + r0_col(m);
          if (lane == 0) PT(tile, m * 8 + 0);
          for (int c = 0; c < Y1::KP(m) / 64; ++c) {
            PW(0, mbar_wait(bar(FA + sa), pa));
            PW(1, mbar_wait(bar(FB + sb), pb));
            tc_fence_after();
            PW(16, {
              if (elect_one()) {
                const uint64_t da = sdesc(sA + sa * A_CHUNK), db = sdesc(sB + sb * B_STAGE);
#pragma unroll
                for (int k = 0; k < 4; ++k) mma_bf16(t_r, da + 2 * k, db + 2 * k, id1, (c | k) ? 1u : 0u);
                tc_commit(bar(EA + sa));
                tc_commit(bar(EB + sb));
              }
              __syncwarp();
            });
            if (++sa == NSA) { sa = 0; pa ^= 1; }
            if (++sb == NSB) { sb = 0; pb ^= 1; }
          }
          if (elect_one()) tc_commit(bar(L1F + (u & 1)));
          __syncwarp();
          if (lane == 0) PT(tile, m * 8 + 1);
          if (prev_m >= 0) lin2(prev_m, u - 1);
          if (lane == 0) PT(tile, m * 8 + 2);
          prev_m = m;
        }
      if (prev_m >= 0) lin2(prev_m, u - 1);
      PROBE_END(5, lane == 0);
    }
  } else if (warp >= 2 && warp <= 9) {
    // ---------------------------------------------------------------- gate
    // warp w owns TMEM lanes 32*(w%4)+; the two halves take alternate
    // 32-column groups.
    const int quad = warp & 3, half = (warp - 2) >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    float sg[32];
    PROBE_DECL;
    int u = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x)
      for (int m = 0; m <= L; ++m, ++u) {
        const uint32_t t_r = tmem + lane_off + r0_col(m);
        const int N1 = Y1::N1(m);
        PW(10, mbar_sleep(bar(L1F + (u & 1)), (u >> 1) & 1));
        if (warp == 2 && lane == 0) PT(tile, 64 + m * 8 + 0);
        tc_fence_after();
        if (m == 0) {  // gate scalars from the l = 0 channels of order 0
          PW(20, {
            float v[32];
            tmem_ld32(t_r, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) sg[i] = gate ? __fdividef(1.f, 1.f + __expf(-v[i])) : 1.f;
          });
        }
        if (u > 0) PW(14, mbar_sleep(bar(A2E), (u - 1) & 1));  // lin2 of unit u - 1 done with A2
        if (warp == 2 && lane == 0) PT(tile, 64 + m * 8 + 1);
        for (int q = half; q < Y1::N1P(m) / 32; q += 2) {
          float v[32];
          if (q * 32 < N1) {
            tmem_ld32(t_r + q * 32, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] *= sg[i];  // column 32q + i uses scalar i
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
          const uint32_t cb = sA2 + (uint32_t)(q >> 1) * A_CHUNK;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(cb + sw128(row, (q & 1) * 4 + j)),
                         "r"(pack_bf16(v[8 * j], v[8 * j + 1])), "r"(pack_bf16(v[8 * j + 2], v[8 * j + 3])),
                         "r"(pack_bf16(v[8 * j + 4], v[8 * j + 5])), "r"(pack_bf16(v[8 * j + 6], v[8 * j + 7]))
                         : "memory");
        }
        fence_async_smem();
        tc_fence_before();
        mbar_arrive(bar(A2F));
        if (warp == 2 && lane == 0) PT(tile, 64 + m * 8 + 2);
      }
    PROBE_END(11, warp == 2 && lane == 0);
  } else if (warp >= 10 && warp <= 17) {
    // --------------------------------------------------------------- drain
    const int quad = warp & 3, half = (warp - 10) >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    PROBE_DECL;
    int u = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const int64_t e0 = tile * TILE_M;
      const bool valid = e0 + row < n_e;
      for (int m = 0; m <= L; ++m, ++u) {
        const int N2 = Y1::N2(m);
        const uint32_t t_y = tmem + lane_off + r0_col(m) + Y1::N1(m) - N2;
        PW(12, mbar_sleep(bar(L2F + (u & 1)), (u >> 1) & 1));
        if (warp == 10 && lane == 0) PT(tile, 128 + m * 4 + 0);
        tc_fence_after();
        // bf16 Y tile [c / 8][row][c % 8] (msg_kernels.cuh y_index): each
        // 16-byte store of the warp lands next to its neighbour lane's
        uint16_t* ytile = Y + tile * (int64_t)TILE_M * (G::H * E) + (int64_t)row * 8;
        const int c0 = G::moff(m) * E;
        for (int q = half; q * 32 < N2; q += 2) {
          float v[32];
          tmem_ld32(t_y + q * 32, v);
          if (m == 0 && q == 0 && logits != nullptr && valid) {
            // ops.h:203-209 attention logit from the l = 0 channels (msg row 0
            // == y row 0 since D_0 = 1), taken from the fp32 accumulator
            float lg = 0.f;
#pragma unroll
            for (int c = 0; c < E; ++c) lg = fmaf(__ldg(att + c), v[c], lg);
            logits[e0 + row] = lg;
          }
#ifdef SO2_PROBE_NOSTORE
          if (valid && v[0] == 12345.f) {
#else
          if (valid) {
#endif
            const int nv = (N2 - q * 32) < 32 ? (N2 - q * 32) : 32;
#pragma unroll
            for (int i = 0; i < 32; i += 8)
              if (i < nv)
                *(uint4*)(ytile + (int64_t)((c0 + q * 32 + i) >> 3) * (TILE_M * 8)) =
                    make_uint4(pack_bf16(v[i], v[i + 1]), pack_bf16(v[i + 2], v[i + 3]), pack_bf16(v[i + 4], v[i + 5]),
                               pack_bf16(v[i + 6], v[i + 7]));
          }
        }
        tc_fence_before();
        asm volatile("bar.sync 1, %0;\n" ::"n"(DRAIN_THREADS) : "memory");  // all drain lanes read their Y
        if (warp == 10 && lane == 0) {
          st_release(smem_u32(drained), (uint32_t)(u + 1));
          PT(tile, 128 + m * 4 + 1);
        }
      }
    }
    PROBE_END(13, warp == 10 && lane == 0);
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
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [] {
    ESG_CUDA(cudaFuncSetAttribute(k_so2_tc<4, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  });
  const int n_sm = sm_count();
  const int64_t tiles = (n_e + TILE_M - 1) / TILE_M;
  const int grid = (int)(tiles < n_sm ? tiles : n_sm);
  if (grid > 0)
    k_so2_tc<4, 16><<<grid, THREADS, SMEM_BYTES, st>>>((const uint8_t*)A1, n_e, (const uint8_t*)W1,
                                                       (const uint8_t*)W2, Y, gate, att, logits);
  ESG_CUDA(cudaGetLastError());
}

}  // namespace esg
