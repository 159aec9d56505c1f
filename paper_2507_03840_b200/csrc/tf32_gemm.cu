// tf32_gemm.cu -- the fp32-accurate per-order SO(2) linears on the 5th-gen
// tensor cores (SURVEY §8 a11 "fp32 (3xTF32 split) for parity"): the fp32
// forward path and the training reverse pass (kernels.h:133-199).
//
//   C[e, o] = sum_k A[e, k] B[o, k]       per order block, 128 rows per CTA
//
// A (activations, fp32 rows) is split on the fly into tf32 hi = rna(a) and
// lo = rna(a - hi); B (weights) is split once at pack time into the same two
// images.  Three tcgen05.mma kind::tf32 passes hi.hi + hi.lo + lo.hi
// accumulate in one fp32 TMEM accumulator (the dropped lo.lo term and the
// rounding of lo are ~2^-22 relative), so the result tracks an fp32 SGEMM.
// Operands sit in SMEM as K-major SWIZZLE_128B tiles (32 tf32 per 128-byte
// row); B chunks arrive by one bulk copy each, A chunks are converted by the
// CTA's four warps while the previous chunk's MMAs run.  The epilogue reads
// TMEM rows (one per lane) straight into the fp32 output rows.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "device_model.h"
#include "tc_common.cuh"

namespace esg {

namespace {
using namespace tc;

constexpr int TM = 128;                  // rows per CTA (UMMA M, one per TMEM lane)
constexpr int THREADS = 256;
constexpr int A_BYTES = TM * 128;        // one split of a 32-wide K chunk of A
constexpr int B_MAX = 256 * 128;         // one split of a K chunk of B (N <= 256)
constexpr int STAGE = 2 * A_BYTES + 2 * B_MAX;
constexpr int SMEM_BYTES = 1024 + 2 * STAGE + 64;

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

__global__ void __launch_bounds__(THREADS, 1)
    k_gemm_tf32x3(const float* __restrict__ A, int64_t lda, int64_t n_rows, const uint8_t* __restrict__ Bimg,
                  const TcTile* __restrict__ tiles, float* __restrict__ C, int64_t ldc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t s0 = smem_u32(base);
  uint64_t* bars = (uint64_t*)(base + 2 * STAGE);  // full[2], done[2]
  uint32_t* tmem_slot = (uint32_t*)(bars + 4);
  auto bar = [&](int i) { return smem_u32(&bars[i]); };
  const TcTile t = tiles[blockIdx.y];
  const int64_t r0 = (int64_t)blockIdx.x * TM;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(bar(i), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nc = (t.K + 31) >> 5;
  const uint32_t bbytes = 2u * (uint32_t)t.N * 128u;
  const uint32_t idesc = idesc_tf32(t.N);
  const uint64_t pol = policy_evict_last();
  const int u = tid & 7;  // 16-byte unit of the K chunk this thread converts (rows tid / 8 + 32 i)
  auto load = [&](int c, float4* v) {
    const int k = c * 32 + u * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t row = r0 + (tid >> 3) + 32 * i;
      v[i] = (c < nc && row < n_rows && k < t.K)
                 ? __ldg(reinterpret_cast<const float4*>(A + row * lda + t.a_col + k))
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  float4 cur[4], nxt[4];
  load(0, cur);
  for (int c = 0; c < nc; ++c) {
    const int s = c & 1;
    const uint32_t sAh = s0 + s * STAGE, sAl = sAh + A_BYTES, sBh = sAh + 2 * A_BYTES, sBl = sBh + t.N * 128;
    load(c + 1, nxt);  // next chunk's rows in flight while this one is converted
    if (c >= 2) mbar_wait(bar(2 + s), ((c - 2) >> 1) & 1);  // MMAs of chunk c - 2 released stage s
    if (tid == 0) {
      mbar_expect_tx(bar(s), bbytes);
      bulk_g2s(sBh, Bimg + t.b_off + (int64_t)c * bbytes, bbytes, bar(s), pol);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = (tid >> 3) + 32 * i;
      const float4 h = make_float4(to_tf32(cur[i].x), to_tf32(cur[i].y), to_tf32(cur[i].z), to_tf32(cur[i].w));
      const float4 l = make_float4(to_tf32(cur[i].x - h.x), to_tf32(cur[i].y - h.y), to_tf32(cur[i].z - h.z),
                                   to_tf32(cur[i].w - h.w));
      const uint32_t o = sw128(r, u);
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(sAh + o), "f"(h.x), "f"(h.y), "f"(h.z),
                   "f"(h.w)
                   : "memory");
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(sAl + o), "f"(l.x), "f"(l.y), "f"(l.z),
                   "f"(l.w)
                   : "memory");
      cur[i] = nxt[i];
    }
    fence_async_smem();
    __syncthreads();
    if (warp == 0) {
      mbar_wait(bar(s), (c >> 1) & 1);  // B chunk landed
      tc_fence_after();
      if (elect_one()) {
        const uint64_t ah = sdesc(sAh), al = sdesc(sAl), bh = sdesc(sBh), bl = sdesc(sBl);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {  // K = 8 tf32 (32 bytes) per instruction
          mma_tf32(tmem, ah + 2 * ks, bh + 2 * ks, idesc, (c | ks) ? 1u : 0u);
          mma_tf32(tmem, ah + 2 * ks, bl + 2 * ks, idesc, 1u);
          mma_tf32(tmem, al + 2 * ks, bh + 2 * ks, idesc, 1u);
        }
        tc_commit(bar(2 + s));
      }
      __syncwarp();
    }
  }
  mbar_wait(bar(2 + ((nc - 1) & 1)), ((nc - 1) >> 1) & 1);
  tc_fence_after();
  // epilogue: warps w and w + 4 own TMEM lanes (rows) 32 (w % 4) ..; they
  // take alternate 16-column groups
  const int quarter = warp & 3;
  const int64_t row = r0 + quarter * 32 + lane;
  float* out = C + row * ldc + t.c_col;
  for (int j = (warp >> 2) * 16; j < t.N; j += 32) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)j, v);
    if (row < n_rows) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (j + 4 * q < t.n_valid)
          reinterpret_cast<float4*>(out + j)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
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
                      int n_tiles, float* C, int64_t ldc, cudaStream_t st) {
  static bool init = false;
  if (!init) {
    ESG_CUDA(cudaFuncSetAttribute(k_gemm_tf32x3, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    init = true;
  }
  if (n_rows <= 0) return;
  k_gemm_tf32x3<<<dim3((unsigned)((n_rows + TM - 1) / TM), (unsigned)n_tiles), THREADS, SMEM_BYTES, st>>>(
      A, lda, n_rows, img, tiles, C, ldc);
  ESG_CUDA(cudaGetLastError());
}

}  // namespace esg
