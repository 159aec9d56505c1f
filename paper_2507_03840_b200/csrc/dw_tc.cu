// dw_tc.cu -- the SO(2) linears' weight gradients on the 5th-gen tensor
// cores (the reverse pass of kernels.h:133-199; optimizer input of
// network.h:216-240):
//
//   dW_m[n][k] += sum_e g[e][goff_m + n] x[e][xoff_m + k]
//
// per order block m, summed over the edges of a chunk.  The reduction runs
// over edges, so both operands are edge-major activation rows.  TMA brings
// boxes of 32 channels x 16 edges straight into SMEM in the MN-major
// SWIZZLE_128B_BASE32B layout tcgen05 reads (the only MN-major layout it
// takes for 32-bit types; TMA's SWIZZLE_128B_ATOM_32B writes it), one box
// per 32 channels -- no transposition anywhere.  Converter warps then split
// every value in place into tf32 hi = rna(v) and lo = rna(v - hi) (applying
// the gate's per-edge scale when x is the pre-gate hidden), and three
// tcgen05.mma kind::tf32 passes (hi.hi + hi.lo + lo.hi) accumulate a
// 128 x N tile in TMEM (fp32), as tf32_gemm.cu does for the forward.
//
// Determinism: work item = (output tile, edge split); the split's sum is
// accumulated in a fixed chunk / instruction order, written to its partial
// slot, and k_dw_reduce adds the splits in a fixed order in fp64 into the
// gradient accumulator -- the same bits every run.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "device_model.h"
#include "tc_common.cuh"

namespace esg {

namespace {
using namespace tc;

constexpr int DM = 128;                 // MMA M: g channels per tile (TMEM lanes)
constexpr int CE = 16;                  // edges per chunk (2 MMA K steps of 8)
constexpr int BOX = 32 * CE * 4;        // one TMA box: 32 channels x CE edges (2 KB)
constexpr int A_IMG = 4 * BOX;          // g: up to 128 channels
constexpr int B_IMG = 8 * BOX;          // x: up to 256 channels
constexpr int S_IMG = BOX;              // the chunk's gate scalars (<= 32 per edge)
constexpr int STAGE = 2 * A_IMG + 2 * B_IMG + S_IMG;  // hi, lo images + gate scalars
constexpr int NS = 4;                   // stage ring
// warps 0-3 epilogue, 4-15 converters, 16 TMA loader, 17 MMA issuer
constexpr int EPI_WARPS = 4, CONV_WARPS = 12, LOAD_WARP = EPI_WARPS + CONV_WARPS, MMA_WARP = LOAD_WARP + 1;
constexpr int CT = CONV_WARPS * 32;     // converter threads
constexpr int THREADS = 32 * (MMA_WARP + 1);
constexpr int BAR_OFF = NS * STAGE;
constexpr int SMEM_BYTES = 1024 + BAR_OFF + 256;
constexpr int PART_STRIDE = DM * 256;   // floats per partial tile
static_assert(STAGE % 1024 == 0, "stages keep the 1 KB swizzle alignment");

__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// MN-major SWIZZLE_128B_BASE32B canonical layout ((8,n),(4,k)):((1,LBO),(4,SBO))
// in 16-byte units: 128-byte rows of 32 channels (one row per edge), atoms of
// 4 rows whose 32-byte chunks are XOR-permuted by row % 4; edge groups of 4
// rows SBO = 512 B apart, 32-channel groups (one TMA box each) LBO = 2 KB apart.
__device__ __forceinline__ uint64_t sdesc_mn(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(BOX >> 4) << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)1 << 61);
}
// kind::tf32, fp32 D, A and B MN-major, M = 128
__device__ __forceinline__ uint32_t idesc_dw(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(DM >> 4) << 24);
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
// the value v (raw fp32 from the TMA box at hi_img + off) -> hi = rna(v) in
// place and lo = rna(v - hi) beside it.  (Keeping the raw box as a truncated
// hi would save the rewrite, but its one-signed lo biases the dropped lo.lo
// term: measured 1.2e-5 gradient rel-L2 against 7.9e-6.)
__device__ __forceinline__ void split_in_place(uint32_t hi_img, uint32_t lo_img, uint32_t off, float4 v) {
  const float4 h = make_float4(to_tf32(v.x), to_tf32(v.y), to_tf32(v.z), to_tf32(v.w));
  sts4(hi_img + off, h);
  sts4(lo_img + off, make_float4(to_tf32(v.x - h.x), to_tf32(v.y - h.y), to_tf32(v.z - h.z), to_tf32(v.w - h.w)));
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// persistent warp-specialised: warps 0-3 epilogue, 4-15 converters, 16 TMA
// loader, 17 MMA issuer.  Items split-major (consecutive CTAs read the same
// edges: L2 reuse).
__global__ void __launch_bounds__(THREADS, 1)
    k_dw_tf32x3(const __grid_constant__ CUtensorMap tm_g, const __grid_constant__ CUtensorMap tm_x,
                const __grid_constant__ CUtensorMap tm_s, int64_t n_e, const DwTile* __restrict__ tiles, int n_tiles,
                int n_split, int split_e, float* __restrict__ part, int gate_c2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t s0a = smem_u32(base);
  uint64_t* bars = (uint64_t*)(base + BAR_OFF);
  auto bar = [&](int i) { return smem_u32(&bars[i]); };
  const int LF = 0, VF = NS, FE = 2 * NS, CF = 3 * NS, CEb = CF + 2;
  uint32_t* tmem_slot = (uint32_t*)(bars + CEb + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(bar(LF + i), 1);   // TMA landed (+ tx bytes)
      mbar_init(bar(VF + i), CT);  // converted
      mbar_init(bar(FE + i), 1);   // MMAs done with the stage
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(CF + i), 1);
      mbar_init(bar(CEb + i), EPI_WARPS * 32);
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
  const int64_t n_items = (int64_t)n_tiles * n_split;
  auto stage_addr = [&](int s) { return s0a + (uint32_t)(s * STAGE); };
  // per item: its tile, edge range and chunk count (every role walks the same list)
  auto item = [&](int64_t it, DwTile& t, int64_t& e_lo, int& nch) {
    t = tiles[it % n_tiles];
    e_lo = (it / n_tiles) * (int64_t)split_e;
    const int64_t e_hi = e_lo + split_e < n_e ? e_lo + split_e : n_e;
    nch = (int)((e_hi - e_lo + CE - 1) / CE);
  };

  if (warp == LOAD_WARP) {
    // ---- TMA loader: per chunk ceil(nN / 32) g boxes, ceil(nKp / 32) x boxes
    // (+ the gate scalars); edges past n_e arrive as zeros
    if (lane == 0) {
      int s = 0;
      uint32_t k = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        DwTile t;
        int64_t e_lo;
        int nch;
        item(it, t, e_lo, nch);
        const int na = (t.nN + 31) >> 5, nb = (t.nKp + 31) >> 5;
        const uint32_t bytes = (uint32_t)(na + nb) * BOX + (uint32_t)gate_c2 * CE * 4;  // gate box: gate_c2 x CE
        for (int c = 0; c < nch; ++c) {
          const int e0 = (int)(e_lo + (int64_t)c * CE);
          mbar_wait(bar(FE + s), ((k / NS) & 1) ^ 1);
          mbar_expect_tx(bar(LF + s), bytes);
          const uint32_t sa = stage_addr(s), sb = sa + 2 * A_IMG;
          for (int j = 0; j < na; ++j) tma_2d(sa + j * BOX, &tm_g, t.goff + 32 * j, e0, bar(LF + s));
          for (int j = 0; j < nb; ++j) tma_2d(sb + j * BOX, &tm_x, t.xoff + 32 * j, e0, bar(LF + s));
          if (gate_c2) tma_2d(sb + 2 * B_IMG, &tm_s, 0, e0, bar(LF + s));
          if (++s == NS) s = 0;
          ++k;
        }
      }
    }
  } else if (warp >= EPI_WARPS && warp < LOAD_WARP) {
    // ---- converters: the raw boxes -> tf32 hi (in place) / lo images.
    // Elementwise at fixed offsets: image layout and box layout coincide.
    const int ct = tid - EPI_WARPS * 32;  // 0..CT-1
    int s = 0;
    uint32_t k = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      DwTile t;
      int64_t e_lo;
      int nch;
      item(it, t, e_lo, nch);
      const int na = (t.nN + 31) >> 5, nb = (t.nKp + 31) >> 5;
      for (int c = 0; c < nch; ++c) {
        mbar_wait(bar(LF + s), (k / NS) & 1);
        const uint32_t sa = stage_addr(s), sb = sa + 2 * A_IMG, sg = sb + 2 * B_IMG;
        // g: na boxes of 128 float4 units
#pragma unroll 2
        for (int u = ct; u < na * (BOX / 16); u += CT) split_in_place(sa, sa + A_IMG, u * 16, lds4(sa + u * 16));
        // x: nb boxes; gated x (kernels.h:210-226): channel c of every row
        // scaled by sigmoid(h[row 0][c]), precomputed per edge
#pragma unroll 4
        for (int u = ct; u < nb * (BOX / 16); u += CT) {
          float4 v = lds4(sb + u * 16);
          if (gate_c2) {
            const int j = u >> 7, e = (u >> 3) & 15, pos = u & 7;  // box, row (edge), 16-byte unit
            const int ch = 32 * j + ((((pos >> 1) ^ (e & 3)) << 3) | ((pos & 1) << 2));  // swizzle undone
            const float4 f = lds4(sg + e * (gate_c2 * 4) + ((t.xoff + ch) % gate_c2) * 4);
            v = make_float4(v.x * f.x, v.y * f.y, v.z * f.z, v.w * f.w);
          }
          split_in_place(sb, sb + B_IMG, u * 16, v);
        }
        fence_async_smem();
        mbar_arrive(bar(VF + s));
        if (++s == NS) s = 0;
        ++k;
      }
    }
  } else if (warp == MMA_WARP) {
    // ---- MMA issuer: per chunk CE / 8 K steps x 3 split products
    int s = 0;
    uint32_t k = 0, j = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x, ++j) {
      DwTile t;
      int64_t e_lo;
      int nch;
      item(it, t, e_lo, nch);
      const uint32_t idesc = idesc_dw(t.nKp);
      const int ab = j & 1;
      mbar_wait(bar(CEb + ab), ((j >> 1) & 1) ^ 1);  // the epilogue drained this accumulator
      tc_fence_after();
      const uint32_t acc = tmem + (uint32_t)(ab * 256);
      for (int c = 0; c < nch; ++c) {
        mbar_wait(bar(VF + s), (k / NS) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = stage_addr(s), sb = sa + 2 * A_IMG;
#pragma unroll
          for (int ks = 0; ks < CE / 8; ++ks) {  // 8 edges (two 4-row swizzle atoms) per instruction
            const uint64_t ah = sdesc_mn(sa + ks * 1024), al = sdesc_mn(sa + A_IMG + ks * 1024);
            const uint64_t bh = sdesc_mn(sb + ks * 1024), bl = sdesc_mn(sb + B_IMG + ks * 1024);
            mma_tf32(acc, ah, bh, idesc, (c | ks) ? 1u : 0u);
            mma_tf32(acc, ah, bl, idesc, 1u);
            mma_tf32(acc, al, bh, idesc, 1u);
          }
          tc_commit(bar(FE + s));
          if (c == nch - 1) tc_commit(bar(CF + ab));
        }
        __syncwarp();
        if (++s == NS) s = 0;
        ++k;
      }
    }
  } else {
    // ---- epilogue: warp w drains TMEM lanes 32 w.. (g channels) to the partial tile
    uint32_t j = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x, ++j) {
      const DwTile t = tiles[it % n_tiles];
      const int ab = j & 1;
      const int r = warp * 32 + lane;
      mbar_wait(bar(CF + ab), (j >> 1) & 1);
      tc_fence_after();
      float* out = part + it * (int64_t)PART_STRIDE + (int64_t)r * 256;
      for (int c0 = 0; c0 < t.nKp; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(ab * 256 + c0), v);
        if (r < t.nN) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c0 + 4 * q < t.nK)
              reinterpret_cast<float4*>(out + c0)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(bar(CEb + ab));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// the splits of each tile into the accumulator, fp64, in a fixed order: a
// block takes 32 output elements of one tile; its 8 warps-worth of split
// groups (lane = element, group = warp) each sum a contiguous run of splits
// in split order, and the 8 group sums are added in group order
__global__ void __launch_bounds__(256) k_dw_reduce(const float* __restrict__ part, const DwTile* __restrict__ tiles,
                                                   int n_tiles, int n_split, double* __restrict__ acc) {
  __shared__ double red[8][32];
  const DwTile t = tiles[blockIdx.y];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int u = blockIdx.x * 32 + lane;  // element n * 256 + k of the partial tile
  const int n = u >> 8, k = u & 255;
  const bool valid = n < t.nN && k < t.nK;
  const int per = (n_split + 7) / 8, s0 = grp * per, s1 = s0 + per < n_split ? s0 + per : n_split;
  double s = 0.0;
  if (valid) {
    const float* p = part + (int64_t)blockIdx.y * PART_STRIDE + u;
    for (int sp = s0; sp < s1; ++sp) s += (double)__ldg(p + (int64_t)sp * n_tiles * PART_STRIDE);
  }
  red[grp][lane] = s;
  __syncthreads();
  if (grp == 0 && valid) {
    double tot = red[0][lane];
#pragma unroll
    for (int g = 1; g < 8; ++g) tot += red[g][lane];
    acc[t.acc_off + (int64_t)(t.n0 + n) * t.K + (t.k0 + k)] += tot;
  }
}

// a 2D fp32 tensor map over rows of `row` floats (stride ld floats), n rows;
// boxes of 32 floats x CE rows, SWIZZLE_128B_ATOM_32B (or none)
CUtensorMap tensor_map(const float* p, int64_t row, int64_t ld, int64_t n, bool swizzle) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    ESG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !encode) usage("cuTensorMapEncodeTiled unavailable");
  }
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)row, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {(cuuint32_t)(row < 32 ? row : 32), (cuuint32_t)CE};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)p, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE,
                            swizzle ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) usage("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

}  // namespace

// Tile lists of the two weight-gradient products: which 0 = lin1 (g: 2E
// channels, x: 3E), 1 = lin2 (g: E, x: 2E).  Per order block m (N = rows x
// cg outputs, K = rows x cx inputs): 128-row tiles along N, <= 256-column
// tiles along K (MMA N a multiple of 16).  acc_off: the order block in the
// expanded accumulator layout (N x K row-major per block, blocks in m order).
int dw_tiles(int L, int E, int which, std::vector<DwTile>* tiles) {
  const int cg = which == 0 ? 2 * E : E, cx = which == 0 ? 3 * E : 2 * E;
  int64_t off = 0;
  int moff = 0;
  int n = 0;
  for (int m = 0; m <= L; ++m) {
    const int rows = m == 0 ? L + 1 : 2 * (L - m + 1), N = rows * cg, K = rows * cx;
    const int kt = (K + 255) / 256, kw = ((K + kt - 1) / kt + 15) / 16 * 16;
    for (int n0 = 0; n0 < N; n0 += DM)
      for (int k0 = 0; k0 < K; k0 += kw) {
        const int nK = K - k0 < kw ? K - k0 : kw;
        if (tiles) tiles->push_back({moff * cg + n0, moff * cx + k0, n0, k0, N - n0 < DM ? N - n0 : DM, nK,
                                     (nK + 15) / 16 * 16, K, off});
        ++n;
      }
    off += (int64_t)N * K;
    moff += rows;
  }
  return n;
}

int64_t dw_part_floats(int n_tiles, int n_split) { return (int64_t)n_tiles * n_split * PART_STRIDE; }

void dw_tf32x3_launch(const float* g, int64_t ldg, const float* x, int64_t ldx, int64_t n_e, const DwTile* tiles,
                      int n_tiles, int split_e, float* part, double* acc, cudaStream_t st, const float* gscale,
                      int gate_c2) {
  if (n_e <= 0) return;
  if (split_e % CE) usage("weight-gradient split must be a multiple of 16 edges");
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [] {
    ESG_CUDA(cudaFuncSetAttribute(k_dw_tf32x3, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  });
  // rows as TMA sees them: every channel of an edge row (ld floats)
  const CUtensorMap tg = tensor_map(g, ldg, ldg, n_e, true), tx = tensor_map(x, ldx, ldx, n_e, true);
  if (gscale && (gate_c2 > 32 || gate_c2 % 4)) usage("gate width must be a multiple of 4, at most 32");
  const CUtensorMap ts = gscale ? tensor_map(gscale, gate_c2, gate_c2, n_e, false) : tg;
  const int n_split = (int)((n_e + split_e - 1) / split_e);
  const int64_t items = (int64_t)n_tiles * n_split;
  const int grid = (int)std::min<int64_t>(items, sm_count());
  k_dw_tf32x3<<<grid, THREADS, SMEM_BYTES, st>>>(tg, tx, ts, n_e, tiles, n_tiles, n_split, split_e, part,
                                                 gscale ? gate_c2 : 0);
  k_dw_reduce<<<dim3(PART_STRIDE / 32, (unsigned)n_tiles), 256, 0, st>>>(part, tiles, n_tiles, n_split, acc);
  ESG_CUDA(cudaGetLastError());
}

}  // namespace esg
