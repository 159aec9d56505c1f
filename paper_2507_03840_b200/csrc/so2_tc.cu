// so2_tc.cu -- the SO(2) linear chain on the 5th-gen tensor cores.
//
// Per tile of 128 edges (UMMA M = 128, one edge per TMEM lane) and per order
// m = 0..L (kernels.h:133-161, :210-226; network.h:144-146):
//   lin1   H_m[128 x N1] = A1_m[128 x K1] . W1_m^T   tcgen05.mma kind::f16
//          (bf16 operands in SMEM, SWIZZLE_128B K-major, fp32 accumulator in
//          TMEM columns [0, 256))
//   gate   s = sigmoid(H_0[:, l=0 channels]) from the m = 0 block (computed
//          first), H_m * s[c % 2E] -> bf16 A2 in SMEM (TMEM -> regs -> SMEM)
//   lin2   Y_m[128 x N2] = A2_m . W2_m^T               accumulator in TMEM
//          columns [256, 384), drained to the fp32 Y rows in HBM.
// W_m are the expanded [[Wr, Wi], [-Wi, Wr]] order blocks, K padded to 64.
// Operand chunks (64 K = 128 B rows) stream through a 2-stage cp.async ring;
// tcgen05.commit on a per-stage mbarrier releases a stage when its MMAs are
// done.  One elected thread issues every MMA; 4 warps load and run the
// epilogues (warp w owns TMEM lanes 32w..32w+31).
#include <cuda_runtime.h>

#include <cstdint>

#include "esg_internal.h"
#include "model_kernels.cuh"

namespace esg {
namespace {

constexpr int TILE_M = 128;
constexpr int THREADS = 128;
constexpr int A_STAGE = TILE_M * 128;      // 64 bf16 K x 128 rows = 16 KB
constexpr int B_STAGE = 256 * 128;         // up to 256 rows x 64 K   = 32 KB
constexpr int A2_BYTES = TILE_M * 256 * 2; // up to 256 K             = 64 KB
constexpr int S_BYTES = TILE_M * 33 * 4;   // gate scalars (2E = 32, padded row)
constexpr int SMEM_BYTES = 1024 + 2 * A_STAGE + 2 * B_STAGE + A2_BYTES + S_BYTES + 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major SWIZZLE_128B tile: row r, 16-byte chunk c -> r*128 + (c ^ (r&7))*16
__device__ __forceinline__ uint32_t sw128(int r, int c) { return uint32_t(r * 128 + ((c ^ (r & 7)) << 4)); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
  const int sz = pred ? 16 : 0;  // zero-fill rows past the end
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

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

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar) : "memory");
}

// SMEM matrix descriptor: K-major, SWIZZLE_128B, SBO = 1024 B (8-row group
// stride), LBO unused for swizzled K-major (encoded 1), version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor kind::f16: D f32, A/B bf16, both K-major, M=128.
__host__ __device__ constexpr uint32_t idesc_bf16(int N) {
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

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread.
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

struct Ring {
  uint32_t a[2], b[2], bar[2];
  uint32_t phase[2];
  bool pending[2];
};

// One GEMM pass: D[tmem_col : +N] (+)= sum_kc A_kc . B_kc^T over n_chunks
// 64-wide K chunks.  A comes from global (a_glob != nullptr, rows of `a_ld`
// bf16 starting at element a_k0) or from the SMEM A2 buffer; B rows (N of
// them, `b_ld` bf16 each) from global.
__device__ void gemm_pass(Ring& rg, const uint16_t* a_glob, int64_t a_ld, int a_k0, int rows_valid, uint32_t a2,
                          const uint16_t* b_glob, int b_ld, int N, int n_chunks, uint32_t tmem_d) {
  const int tid = threadIdx.x;
  const uint32_t idesc = idesc_bf16(N);
  auto load = [&](int kc, int s) {
    if (a_glob) {
      for (int i = tid; i < TILE_M * 8; i += THREADS) {
        const int r = i >> 3, c = i & 7;
        const bool ok = r < rows_valid;
        const uint16_t* src = a_glob + (ok ? (int64_t)r * a_ld : 0) + a_k0 + kc * 64 + c * 8;
        cp_async16(rg.a[s] + sw128(r, c), src, ok);
      }
    }
    for (int i = tid; i < N * 8; i += THREADS) {
      const int r = i >> 3, c = i & 7;
      cp_async16(rg.b[s] + sw128(r, c), b_glob + (int64_t)r * b_ld + kc * 64 + c * 8, true);
    }
  };
  load(0, 0);
  cp_async_commit();
  for (int kc = 0; kc < n_chunks; ++kc) {
    const int s = kc & 1;
    if (kc + 1 < n_chunks) {
      const int s2 = s ^ 1;
      if (rg.pending[s2]) {
        mbar_wait(rg.bar[s2], rg.phase[s2]);
        rg.phase[s2] ^= 1;
        rg.pending[s2] = false;
      }
      load(kc + 1, s2);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t abase = a_glob ? rg.a[s] : a2 + (uint32_t)kc * A_STAGE;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_bf16(tmem_d, sdesc(abase + k * 32), sdesc(rg.b[s] + k * 32), idesc, (kc | k) ? 1u : 0u);
      tc_commit(rg.bar[s]);
    }
    rg.pending[s] = true;
  }
  for (int s = 0; s < 2; ++s)
    if (rg.pending[s]) {
      mbar_wait(rg.bar[s], rg.phase[s]);
      rg.phase[s] ^= 1;
      rg.pending[s] = false;
    }
  tc_fence_after();
}

template <int L, int E>
__global__ void __launch_bounds__(THREADS, 1)
    k_so2_tc(const uint16_t* __restrict__ A1, int64_t n_e, const uint16_t* __restrict__ W1,
             const uint16_t* __restrict__ W2, float* __restrict__ Y, int gate) {
  using G = Geo<L>;
  using Y1 = Lay1<L, E, 64>;
  constexpr int C2 = 2 * E;
  static_assert(C2 == 32, "gate scalars assume 2E = 32");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  Ring rg;
  rg.a[0] = smem_u32(base);
  rg.a[1] = rg.a[0] + A_STAGE;
  rg.b[0] = rg.a[1] + A_STAGE;
  rg.b[1] = rg.b[0] + B_STAGE;
  const uint32_t a2 = rg.b[1] + B_STAGE;
  float* sS = (float*)(base + 2 * A_STAGE + 2 * B_STAGE + A2_BYTES);
  uint64_t* bars = (uint64_t*)(base + 2 * A_STAGE + 2 * B_STAGE + A2_BYTES + S_BYTES);
  uint32_t* tmem_slot = (uint32_t*)(bars + 4);
  rg.bar[0] = smem_u32(&bars[0]);
  rg.bar[1] = smem_u32(&bars[1]);
  rg.phase[0] = rg.phase[1] = 0;
  rg.pending[0] = rg.pending[1] = false;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(rg.bar[0], 1);
    mbar_init(rg.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_h = tmem, t_y = tmem + 256;
  const int row = warp * 32 + lane;                      // TMEM lane == tile row
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;  // lane field of the TMEM address

  const int64_t n_tiles = (n_e + TILE_M - 1) / TILE_M;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t e0 = tile * TILE_M;
    const int rows_valid = (int)((n_e - e0) < TILE_M ? (n_e - e0) : TILE_M);
    const uint16_t* a_tile = A1 + e0 * Y1::KTOT;
    int64_t w1 = 0, w2 = 0;
#pragma unroll 1
    for (int m = 0; m <= L; ++m) {
      const int K1 = Y1::KP(m), N1 = Y1::N1(m), N1P = Y1::N1P(m), N2 = Y1::N2(m);
      // ---- lin1 ------------------------------------------------------
      gemm_pass(rg, a_tile, Y1::KTOT, Y1::kofs(m), rows_valid, 0, W1 + w1, K1, N1, K1 / 64, t_h);
      // ---- gate epilogue: TMEM -> regs -> bf16 A2 (SWIZZLE_128B) -----
      for (int q = 0; q < N1P / 32; ++q) {
        float v[32];
        if (q * 32 < N1) {
          tmem_ld32(t_h + lane_off + q * 32, v);
          if (m == 0 && q == 0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) sS[row * 33 + i] = gate ? 1.f / (1.f + __expf(-v[i])) : 1.f;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] *= sS[row * 33 + i];
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        const uint32_t chunk_base = a2 + (uint32_t)(q >> 1) * A_STAGE;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = (q & 1) * 4 + j;
          const uint32_t w0 = pack_bf16(v[8 * j + 0], v[8 * j + 1]), w1v = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
          const uint32_t w2v = pack_bf16(v[8 * j + 4], v[8 * j + 5]), w3 = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(chunk_base + sw128(row, c)), "r"(w0), "r"(w1v),
                       "r"(w2v), "r"(w3)
                       : "memory");
        }
      }
      tc_fence_before();
      // ---- lin2 ------------------------------------------------------
      gemm_pass(rg, nullptr, 0, 0, rows_valid, a2, W2 + w2, N1P, N2, N1P / 64, t_y);
      // ---- drain Y_m -> HBM (fp32, order-major rows x E) --------------
      float* yrow = Y + (e0 + row) * (G::H * E) + G::moff(m) * E;
      for (int q = 0; q * 32 < N2; ++q) {
        float v[32];
        tmem_ld32(t_y + lane_off + q * 32, v);
        if (row < rows_valid) {
          const int nv = (N2 - q * 32) < 32 ? (N2 - q * 32) : 32;
          for (int i = 0; i < nv; i += 4)
            *(float4*)(yrow + q * 32 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        }
      }
      tc_fence_before();
      __syncthreads();
      w1 += (int64_t)N1 * K1;
      w2 += (int64_t)N2 * N1P;
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

}  // namespace

bool so2_tc_available(int L, int E) { return L == 4 && E == 16; }

void so2_tc_launch(int L, int E, const uint16_t* A1, int64_t n_e, const uint16_t* W1, const uint16_t* W2, float* Y,
                   int gate, cudaStream_t st) {
  if (!so2_tc_available(L, E)) usage("tcgen05 SO(2) chain is instantiated for l_max 4, e_width 16");
  static bool configured = false;
  static int n_sm = 148;
  if (!configured) {
    ESG_CUDA(cudaFuncSetAttribute(k_so2_tc<4, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    int dev = 0;
    ESG_CUDA(cudaGetDevice(&dev));
    ESG_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    configured = true;
  }
  const int64_t tiles = (n_e + TILE_M - 1) / TILE_M;
  const int grid = (int)(tiles < n_sm ? tiles : n_sm);
  if (grid > 0) k_so2_tc<4, 16><<<grid, THREADS, SMEM_BYTES, st>>>(A1, n_e, W1, W2, Y, gate);
  ESG_CUDA(cudaGetLastError());
}

}  // namespace esg
