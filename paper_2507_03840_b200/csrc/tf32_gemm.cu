// tf32_gemm.cu -- the fp32-accurate per-order SO(2) linears on the 5th-gen
// tensor cores (SURVEY §8 a11 "fp32 (3xTF32 split) for parity"): the fp32
// forward path and the training reverse pass (kernels.h:133-199).
//
//   C[e, o] = sum_k A[e, k] B[o, k]       per order block, 128 rows per CTA
//
// A (activations, fp32 rows) arrives by TMA (boxes of 32 columns x 128 rows,
// SWIZZLE_128B: the K-major layout the MMA reads) and is split in place by
// converter warps into tf32 hi = rna(a) and lo = rna(a - hi); B (weights)
// is split once at pack time into the same two images.  Three tcgen05.mma kind::tf32 passes hi.hi + hi.lo + lo.hi
// accumulate in one fp32 TMEM accumulator (the dropped lo.lo term and the
// rounding of lo are ~2^-22 relative), so the result tracks an fp32 SGEMM.
// Operands sit in SMEM as K-major SWIZZLE_128B tiles (32 tf32 per 128-byte
// row); B chunks arrive by one bulk copy each, A chunks by one TMA box each,
// and are converted while the previous chunk's MMAs run.  The epilogue reads
// TMEM rows (one per lane) straight into the fp32 output rows.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "device_model.h"
#include "tc_common.cuh"

namespace esg {

namespace {
using namespace tc;

constexpr int TM = 128;                  // rows per tile (UMMA M, one per TMEM lane)
constexpr int A_BYTES = TM * 128;        // one split of a 32-wide K chunk of A
constexpr int B_MAX = 256 * 128;         // one split of a K chunk of B (N <= 256)
// persistent warp-specialised GEMM: warps 0-3 epilogue, 4-19 A converters,
// warp 20 MMA issuer, warp 21 loader (A by TMA, B by bulk copy); rings of A
// (3 stages) and B (2 stages)
constexpr int EPI_WARPS = 4, PROD_WARPS = 16, MMA_WARP = EPI_WARPS + PROD_WARPS, LOAD_WARP = MMA_WARP + 1;
constexpr int PT = PROD_WARPS * 32, UPT = 1024 / PT;  // converter threads, 16-byte units each per A chunk
static_assert(UPT * PT == 1024, "A chunk units split evenly");
constexpr int THREADS = 32 * (LOAD_WARP + 1);
constexpr int NA = 3, NB = 2;
constexpr int A_STAGE = 2 * A_BYTES, B_STAGE = 2 * B_MAX;
constexpr int SMEM_BYTES = 1024 + NA * A_STAGE + NB * B_STAGE + 256;

__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ uint32_t idesc_tf32(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// C[e, c_col + o] = sum_k A[e, a_col + k] B[o, k] over work items (128-row
// tile, tile-list entry), tile-list major so all SMs stream the same B image.
__global__ void __launch_bounds__(THREADS, 1)
    k_gemm_tf32x3(const __grid_constant__ CUtensorMap tm_a, const float* __restrict__ A, int64_t lda, int64_t n_rows,
                  const uint8_t* __restrict__ Bimg, const TcTile* __restrict__ tiles, int n_tiles, float* __restrict__ C,
                  int64_t ldc, int gate_c2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sA = smem_u32(base), sB = sA + NA * A_STAGE;
  uint64_t* bars = (uint64_t*)(base + NA * A_STAGE + NB * B_STAGE);
  auto bar = [&](int i) { return smem_u32(&bars[i]); };
  // A: landed (TMA tx), converted, free; B: landed, free; accumulators
  const int AL = 0, AF = NA, AE = 2 * NA, BF = 3 * NA, BE = 3 * NA + NB, CF = 3 * NA + 2 * NB, CE = CF + 2;
  uint32_t* tmem_slot = (uint32_t*)(bars + CE + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < NA; ++i) {
      mbar_init(bar(AL + i), 1);
      mbar_init(bar(AF + i), PROD_WARPS * 32);
      mbar_init(bar(AE + i), 1);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(bar(BF + i), 1);
      mbar_init(bar(BE + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(CF + i), 1);
      mbar_init(bar(CE + i), EPI_WARPS * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t n_rt = (n_rows + TM - 1) / TM;
  const int64_t n_items = n_rt * n_tiles;

  if (warp == LOAD_WARP) {
    // ---- loader: lane 0 streams A (per K chunk one TMA box of 32 columns x
    // 128 rows; rows past n_rows arrive as zeros), lane 1 streams B (one bulk
    // copy per chunk), each at its own ring's pace
    if (lane < 2) {
      const bool is_a = lane == 0;
      const uint64_t pol = policy_evict_last();
      int s = 0;
      uint32_t k = 0;
      const int ns = is_a ? NA : NB;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        const TcTile t = tiles[it / n_rt];
        const int r0 = (int)((it % n_rt) * TM);
        const int nc = (t.K + 31) >> 5;
        const uint32_t bbytes = 2u * (uint32_t)t.N * 128u;
        for (int c = 0; c < nc; ++c) {
          if (is_a) {
            mbar_wait(bar(AE + s), ((k / NA) & 1) ^ 1);
            mbar_expect_tx(bar(AL + s), A_BYTES);
            tma_2d(sA + s * A_STAGE, &tm_a, t.a_col + 32 * c, r0, bar(AL + s));
          } else {
            mbar_wait(bar(BE + s), ((k / NB) & 1) ^ 1);
            mbar_expect_tx(bar(BF + s), bbytes);
            bulk_g2s(sB + s * B_STAGE, Bimg + t.b_off + (int64_t)c * bbytes, bbytes, bar(BF + s), pol);
          }
          if (++s == ns) s = 0;
          ++k;
        }
      }
    }
  } else if (warp >= EPI_WARPS && warp < MMA_WARP) {
    // ---- converters: the A box (raw fp32) split in place into tf32 hi and
    // the lo image at the same swizzled offsets.  Columns past the block's K
    // meet zero rows of the B image.
    const int pt = tid - EPI_WARPS * 32;  // 0..PT-1
    int sa = 0;
    uint32_t ka = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const TcTile t = tiles[it / n_rt];
      const int64_t r0 = (it % n_rt) * TM;
      const int nc = (t.K + 31) >> 5;
      // fused gate (kernels.h:210-226) of lin2's operand: column k of an order
      // block is channel k % 2E, and a thread always converts the same four
      // 16-byte units of a chunk (fixed row, fixed logical columns), so its
      // 4 x 4 scales sigmoid(A[row][c]) (the row's first 2E values: l = 0,
      // m = 0) are loaded once per item
      float4 gs[UPT];
      if (gate_c2) {
#pragma unroll
        for (int i = 0; i < UPT; ++i) {
          const int u = pt + PT * i, r = u >> 3, pos = u & 7;
          const int64_t row = r0 + r;
          const int c0 = (((pos ^ (r & 7)) * 4)) % gate_c2;
          float4 h = row < n_rows ? __ldg(reinterpret_cast<const float4*>(A + row * lda + c0))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
          gs[i] = make_float4(1.f / (1.f + expf(-h.x)), 1.f / (1.f + expf(-h.y)), 1.f / (1.f + expf(-h.z)),
                              1.f / (1.f + expf(-h.w)));
        }
      }
      for (int c = 0; c < nc; ++c) {
        mbar_wait(bar(AL + sa), (ka / NA) & 1);
        const uint32_t sh = sA + sa * A_STAGE, sl = sh + A_BYTES;
#pragma unroll
        for (int i = 0; i < UPT; ++i) {
          const uint32_t o = (uint32_t)(pt + PT * i) * 16u;
          float4 v = lds4(sh + o);
          if (gate_c2) v = make_float4(v.x * gs[i].x, v.y * gs[i].y, v.z * gs[i].z, v.w * gs[i].w);
          const float4 h = make_float4(to_tf32(v.x), to_tf32(v.y), to_tf32(v.z), to_tf32(v.w));
          sts4(sh + o, h);
          sts4(sl + o, make_float4(to_tf32(v.x - h.x), to_tf32(v.y - h.y), to_tf32(v.z - h.z), to_tf32(v.w - h.w)));
        }
        fence_async_smem();
        mbar_arrive(bar(AF + sa));
        if (++sa == NA) sa = 0;
        ++ka;
      }
    }
  } else if (warp == MMA_WARP) {
    // ---- MMA issuer: 3 passes per K step into the item's TMEM buffer
    int sa = 0, sb = 0;
    uint32_t ka = 0, kb = 0, j = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x, ++j) {
      const TcTile t = tiles[it / n_rt];
      const int nc = (t.K + 31) >> 5;
      const uint32_t idesc = idesc_tf32(t.N);
      const int ab = j & 1;
      mbar_wait(bar(CE + ab), ((j >> 1) & 1) ^ 1);  // the epilogue drained this accumulator
      tc_fence_after();
      const uint32_t acc = tmem + (uint32_t)(ab * 256);
      for (int c = 0; c < nc; ++c) {
        mbar_wait(bar(AF + sa), (ka / NA) & 1);
        mbar_wait(bar(BF + sb), (kb / NB) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t ah_a = sA + sa * A_STAGE, bh_a = sB + sb * B_STAGE;
          const uint64_t ah = sdesc(ah_a), al = sdesc(ah_a + A_BYTES), bh = sdesc(bh_a), bl = sdesc(bh_a + t.N * 128);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {  // K = 8 tf32 (32 bytes) per instruction
            mma_tf32(acc, ah + 2 * ks, bh + 2 * ks, idesc, (c | ks) ? 1u : 0u);
            mma_tf32(acc, ah + 2 * ks, bl + 2 * ks, idesc, 1u);
            mma_tf32(acc, al + 2 * ks, bh + 2 * ks, idesc, 1u);
          }
          tc_commit(bar(AE + sa));
          tc_commit(bar(BE + sb));
          if (c == nc - 1) tc_commit(bar(CF + ab));
        }
        __syncwarp();
        if (++sa == NA) sa = 0;
        ++ka;
        if (++sb == NB) sb = 0;
        ++kb;
      }
    }
  } else {
    // ---- epilogue: warp w drains TMEM lanes 32 w .. into the output rows
    uint32_t j = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x, ++j) {
      const TcTile t = tiles[it / n_rt];
      const int64_t row = (it % n_rt) * TM + warp * 32 + lane;
      const int ab = j & 1;
      mbar_wait(bar(CF + ab), (j >> 1) & 1);
      tc_fence_after();
      float* out = C + row * ldc + t.c_col;
      for (int c0 = 0; c0 < t.N; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(ab * 256 + c0), v);
        if (row < n_rows) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c0 + 4 * q < t.n_valid)
              reinterpret_cast<float4*>(out + c0)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(bar(CE + ab));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// the expanded order block W (N x K; m = 0: W0, m >= 1: [[Wr, Wi], [-Wi, Wr]])
__device__ __forceinline__ float w_expanded(const float* p, int64_t off_a, int64_t off_b, int m, int R, int C, int n,
                                            int k) {
  if (m == 0) return p[off_a + (int64_t)n * C + k];
  const bool lo_n = n < R, lo_k = k < C;
  const int nn = lo_n ? n : n - R, kk = lo_k ? k : k - C;
  const float wr = p[off_a + (int64_t)nn * C + kk], wi = p[off_b + (int64_t)nn * C + kk];
  return lo_n ? (lo_k ? wr : wi) : (lo_k ? -wi : wr);
}

// B image of one order block: rows o (forward: W's rows; dx: W's columns),
// reduction index k (forward: W's columns; dx: W's rows); tiles of <= 256
// rows, per 32-wide K chunk the hi rows then the lo rows, 128-byte rows with
// 16-byte units swizzled by row % 8.
__global__ void k_pack_tf32(const float* __restrict__ params, int64_t off_a, int64_t off_b, int m, int R, int C,
                            int dx, uint8_t* __restrict__ img) {
  const int N = m == 0 ? R : 2 * R, K = m == 0 ? C : 2 * C;
  const int rows = dx ? K : N, kr = dx ? N : K, kcn = (kr + 31) / 32;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)rows * kcn * 32) return;
  const int o = (int)(i / (kcn * 32)), k = (int)(i % (kcn * 32));
  const float v = k < kr ? (dx ? w_expanded(params, off_a, off_b, m, R, C, k, o)
                               : w_expanded(params, off_a, off_b, m, R, C, o, k))
                         : 0.f;
  const int nt = o / 256, r = o % 256, rt = (min(256, rows - nt * 256) + 15) / 16 * 16, kc = k / 32, kk = k % 32;
  const int64_t off = (int64_t)nt * 256 * kcn * 256 + (int64_t)kc * 2 * rt * 128 + r * 128 +
                      ((((kk >> 2) ^ (r & 7)) << 4) | ((kk & 3) << 2));
  const float hi = to_tf32(v);
  *reinterpret_cast<float*>(img + off) = hi;
  *reinterpret_cast<float*>(img + off + (int64_t)rt * 128) = to_tf32(v - hi);
}

}  // namespace

// Image bytes and tile list of one linear kind (0 lin1 fwd, 1 lin2 fwd,
// 2 lin2 dx, 3 lin1 dx) for l_max L, width E.
int64_t tf32_tiles(int L, int E, int kind, std::vector<TcTile>* tiles) {
  const int cin_of[4] = {3 * E, 2 * E, E, 2 * E}, cout_of[4] = {2 * E, E, 2 * E, 3 * E};
  int64_t off = 0;
  int moff = 0;
  for (int m = 0; m <= L; ++m) {
    const int nd = L - m + 1, rows_m = m == 0 ? nd : 2 * nd;
    const int K = rows_m * cin_of[kind], N = rows_m * cout_of[kind], kcn = (K + 31) / 32;
    for (int n0 = 0; n0 < N; n0 += 256) {
      const int nv = N - n0 < 256 ? N - n0 : 256, nt = (nv + 15) / 16 * 16;  // MMA N: multiple of 16
      if (tiles) tiles->push_back({moff * cin_of[kind], moff * cout_of[kind] + n0, K, nt, nv, off});
      off += (int64_t)kcn * 2 * nt * 128;
    }
    moff += rows_m;
  }
  return off;
}

// the image of one linear (li 0: lin1, 1: lin2) in one direction into img
void tf32_pack(const float* params, int L, int E, int li, bool dx, const int64_t* off_a, const int64_t* off_b,
               uint8_t* img, cudaStream_t st) {
  const int cin = li == 0 ? 3 * E : 2 * E, cout = li == 0 ? 2 * E : E;
  const int kind = li == 0 ? (dx ? 3 : 0) : (dx ? 2 : 1);
  std::vector<TcTile> t;
  const int64_t bytes = tf32_tiles(L, E, kind, &t);
  ESG_CUDA(cudaMemsetAsync(img, 0, bytes, st));  // padded rows of N tiles stay zero
  int ti = 0;
  for (int m = 0; m <= L; ++m) {
    const int nd = L - m + 1, R = nd * cout, C = nd * cin;
    const int N = m == 0 ? R : 2 * R, K = m == 0 ? C : 2 * C;
    const int rows = dx ? K : N, kr = dx ? N : K;
    const int64_t work = (int64_t)rows * ((kr + 31) / 32) * 32;
    k_pack_tf32<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(params, off_a[m], off_b[m], m, R, C, dx ? 1 : 0,
                                                                img + t[ti].b_off);
    ti += (rows + 255) / 256;
  }
  ESG_CUDA(cudaGetLastError());
}

void tf32_gemm_launch(const float* A, int64_t lda, int64_t n_rows, const uint8_t* img, const TcTile* tiles,
                      int n_tiles, float* C, int64_t ldc, cudaStream_t st, int gate_c2) {
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [] {
    ESG_CUDA(cudaFuncSetAttribute(k_gemm_tf32x3, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  });
  if (n_rows <= 0) return;
  if (gate_c2 && (32 % gate_c2 != 0 || gate_c2 % 4 != 0)) usage("fused gate needs 2E dividing 32");
  // A as TMA sees it: n_rows rows of lda floats, boxes of 32 columns x 128 rows, SWIZZLE_128B
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    ESG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !encode) usage("cuTensorMapEncodeTiled unavailable");
  }
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)lda, (cuuint64_t)n_rows};
  const cuuint64_t strides[1] = {(cuuint64_t)lda * 4};
  const cuuint32_t box[2] = {32, (cuuint32_t)TM}, es[2] = {1, 1};
  const CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)A, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) usage("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  const int n_sm = sm_count();
  const int64_t items = (n_rows + TM - 1) / TM * n_tiles;
  const int grid = (int)(items < n_sm ? items : n_sm);
  k_gemm_tf32x3<<<grid, THREADS, SMEM_BYTES, st>>>(tm, A, lda, n_rows, img, tiles, n_tiles, C, ldc, gate_c2);
  ESG_CUDA(cudaGetLastError());
}

}  // namespace esg
