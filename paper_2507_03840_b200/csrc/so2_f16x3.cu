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
//   drain  Y_m -> fp32 order-major values in HBM, tiles of 128 edges
//          [c / 4][edge][c % 4] (+ attention logits)
//
// Operand images (HBM and SMEM alike): per 32-wide K chunk a K-major
// SWIZZLE_128B tile whose 128-byte rows hold [hi(32) | lo(32)] fp16, so the
// hi and lo operands of a K = 16 step are the same descriptor advanced by 0
// or 64 bytes.  One bulk copy (TMA, 1-D) per chunk, no tensor maps.
//
// Warp roles (544 threads, 1 CTA per SM, persistent over tiles):
//   warps 0/14  A1 / W1 producers (one lockstep 3-stage ring, L2 prefetch of A1)
//   warp 15     W2 producer (2-stage ring)
//   warps 1/16  lin1 / lin2 MMA issuers (one elected lane each): two
//               independent instruction streams into the tensor pipe
//   warps 2-9   gate: warp w owns TMEM lanes 32 (w % 4)+, the two halves take
//               alternate 32-column chunks
//   warps 10-13 drain (one per TMEM lane quarter)
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "device_model.h"
#include "msg_kernels.cuh"
#include "esg_internal.h"
#include "model_kernels.cuh"
#include "tc_common.cuh"

namespace esg {

namespace {
using namespace tc;

constexpr int TILE_M = 128;
constexpr int THREADS = 544;  // 17 warps
constexpr int GATE_PARTS = 2;  // gate warps per TMEM lane quarter (part p takes chunks q = p mod GATE_PARTS)
constexpr int NSA = 3;                 // A1 + lin1 weight ring (lockstep, one barrier pair per stage)
constexpr int PFA = 8;                 // L2 prefetch distance of the A1 stream (chunks)
constexpr int NL1 = 4;                 // lin1 may run NL1 - 1 units ahead of lin2's issue
constexpr int NB1 = NSA;
constexpr int NB2 = 2;                 // lin2 weight ring
constexpr int NS2 = 3;                 // gated-operand ring
constexpr int CHUNK = TILE_M * 128;    // one 32-wide K chunk of 128 rows, hi | lo: 16 KB
constexpr int B1_STAGE = 256 * 128;    // up to 256 lin1 weight rows: 32 KB
constexpr int B2_STAGE = 128 * 128;    // up to 128 lin2 weight rows: 16 KB
constexpr int GATE_THREADS = 128 * GATE_PARTS, DRAIN_THREADS = 128;
constexpr int SMEM_BYTES = 1024 + NSA * CHUNK + NB1 * B1_STAGE + NB2 * B2_STAGE + NS2 * CHUNK + 512;

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
__device__ __forceinline__ void mma_chunk(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, bool first,
                                          int nmma = 3) {
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    mma_f16(tmem_d, da + 2 * ks, db + 2 * ks, idesc, (first && ks == 0) ? 0u : 1u);
    if (nmma == 3) {
      mma_f16(tmem_d, da + 2 * ks, db + 4 + 2 * ks, idesc, 1u);
      mma_f16(tmem_d, da + 4 + 2 * ks, db + 2 * ks, idesc, 1u);
    }
  }
}

// TMEM column plan (l_max 4, e_width 16; N1 = 160 256 192 128 64, N2 = N1/2):
// lin1 of order m accumulates into R_m = [R0[m], R0[m] + N1)
//   R1 = [0,256)  R3 = [0,128)  R0 = [256,416)  R2 = [256,448)  R4 = [448,512);
// lin2 accumulates Y_m into its head [R0[m], R0[m] + N2), chunk by chunk
// behind the gate, once the gate has read those columns.  Consecutive
// orders' regions are disjoint (lin1 of order m + 1 runs while order m is
// gated).  lin1 of unit u waits until units < u - LAG[m] are drained: the
// most recent earlier unit whose region overlaps R_m (m2 for m0, m3 for m1,
// m0 for m2, m1 for m3, the previous tile's m4 for m4); a drained unit's gate
// has read all of its columns.  (A unit order / placement in which no Y
// overlaps the region two units later exists -- m = 0 1 4 3 2 -- but did
// not run faster: the chain is bound by its A1 stream.)
__device__ __forceinline__ int order_of(int u) { return u % 5; }
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
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t h2(__half a, __half b) {
  return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}

// F16X3_PROBE (tools/f16x3_probe.cu only): per-role clock64 accounting of
// every wait and of the MMA issuer's idle time by cause, plus experiment
// switches (g_probe_mode: 1 gate skips its arithmetic, 2 drain skips its
// stores, 4 one MMA per K step instead of three); compiled out of the library.
#ifdef F16X3_PROBE
__device__ long long g_probe[1024 * 32];
__device__ int g_probe_mode;
#define PROBE_ON 1
#else
#define PROBE_ON 0
#endif
struct Probe {
#if PROBE_ON
  long long v[24] = {};
  __device__ void add(int i, long long d) { v[i] += d; }
  __device__ void flush(bool cond) {
    if (cond)
      for (int i = 0; i < 24; ++i)
        if (v[i]) atomicAdd((unsigned long long*)&g_probe[blockIdx.x * 32 + i], (unsigned long long)v[i]);
  }
#else
  __device__ void add(int, long long) {}
  __device__ void flush(bool) {}
#endif
};
__device__ __forceinline__ long long pclock() {
#if PROBE_ON
  return clock64();
#else
  return 0;
#endif
}
__device__ __forceinline__ int probe_mode() {
#if PROBE_ON
  return g_probe_mode;
#else
  return 0;
#endif
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
  const uint32_t sB1 = sA + NSA * CHUNK;
  const uint32_t sB2 = sB1 + NB1 * B1_STAGE;
  const uint32_t sA2 = sB2 + NB2 * B2_STAGE;
  uint64_t* bars = (uint64_t*)(base + NSA * CHUNK + NB1 * B1_STAGE + NB2 * B2_STAGE + NS2 * CHUNK);
  auto bar = [&](int i) { return smem_u32(&bars[i]); };
  const int FAB = 0, EAB = NSA, FB2 = 2 * NSA, EB2 = FB2 + NB2;
  const int F2 = EB2 + NB2, E2 = F2 + NS2;  // gated-operand ring
  const int L1F = E2 + NS2;                 // + (u % NL1): lin1 of unit u complete
  const int L2F = L1F + NL1;                // + (u % NL1): lin2 of unit u complete
  const int H1 = L2F + NL1;                 // + (u % NL1): the gate read the Y head of unit u
  uint32_t* drained = (uint32_t*)(bars + H1 + NL1);  // units drained so far
  uint32_t* l2_issued = drained + 1;               // units whose lin2 is fully issued
  uint32_t* tmem_slot = drained + 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NSA; ++s) {
      mbar_init(bar(FAB + s), 2);  // the A1 and the W1 producer each arrive with their bytes
      mbar_init(bar(EAB + s), 1);
    }
    for (int s = 0; s < NB2; ++s) {
      mbar_init(bar(FB2 + s), 1);
      mbar_init(bar(EB2 + s), 1);
    }
    for (int s = 0; s < NS2; ++s) {
      mbar_init(bar(F2 + s), 128);  // one part of the gate (4 warps, 128 rows) writes a chunk
      mbar_init(bar(E2 + s), 1);
    }
    for (int b = 0; b < NL1; ++b) {
      mbar_init(bar(L1F + b), 1);
      mbar_init(bar(L2F + b), 1);
      mbar_init(bar(H1 + b), GATE_THREADS);
    }
    *drained = 0;
    *l2_issued = 0;
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
  const int64_t my_tiles = n_tiles > blockIdx.x ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int total = (int)(my_tiles * (L + 1));  // units (tile, order) of this CTA
  auto spin_until = [&](const uint32_t* ctr, int need) {
    const uint32_t a = smem_u32(ctr);
    if (need > 0)
      while ((int)ld_acquire(a) < need) {
      }
  };

  if (warp == 0 || warp == 14) {
    // ------------------------------------- A1 / W1 producers (lockstep ring)
    // A1 chunks in lin1 order, the chunk PFA steps ahead prefetched into L2
    // (the ring's bulk copies then see L2 latency); W1 chunks in the same
    // order.  Both arrive on the stage's one full barrier with their bytes.
    if (lane == 0) {
      const bool is_a = warp == 0;  // else the W1 producer (warp 14)
      int st = 0;
      uint32_t ph = 0;
      const uint64_t pol = is_a ? policy_evict_first() : policy_evict_last();
      Probe pr;
      const long long t_all = pclock();
      const int64_t total_a = my_tiles * S::KCH;
      auto a_chunk = [&](int64_t i) {  // A1 chunk i of this CTA's stream (orders in image order)
        const int64_t tile = blockIdx.x + (i / S::KCH) * gridDim.x;
        return A1 + ((size_t)tile * S::KCH + (size_t)(i % S::KCH)) * CHUNK;
      };
      if (is_a)
        for (int64_t i = 0; i < PFA && i < total_a; ++i) prefetch_l2(a_chunk(i), CHUNK);
      int64_t i = 0;
      for (int64_t t = 0; t < my_tiles; ++t)
        for (int k = 0; k <= L; ++k) {
          const int m = order_of(k);
          const uint32_t wbytes = (uint32_t)S::N1(m) * 128u;
          for (int c = 0; c < S::K1P(m) / 32; ++c, ++i) {
            if (is_a && i + PFA < total_a) prefetch_l2(a_chunk(i + PFA), CHUNK);
            const long long t0 = pclock();
            mbar_wait(bar(EAB + st), ph ^ 1);
            pr.add(is_a ? 15 : 18, pclock() - t0);
            const bool skip = (probe_mode() & (is_a ? 8 : 32)) != 0;  // probe: no traffic
            if (skip) {
              mbar_arrive(bar(FAB + st));
            } else if (is_a) {
              mbar_expect_tx(bar(FAB + st), CHUNK);
              bulk_g2s(sA + st * CHUNK, a_chunk(i), CHUNK, bar(FAB + st), pol);
            } else {
              mbar_expect_tx(bar(FAB + st), wbytes);
              bulk_g2s(sB1 + st * B1_STAGE, W1 + S::w1_off(m) + (size_t)c * wbytes, wbytes, bar(FAB + st), pol);
            }
            if (++st == NSA) { st = 0; ph ^= 1; }
          }
        }
      pr.add(is_a ? 16 : 19, pclock() - t_all);
      pr.flush(true);
    }
  } else if (warp == 15) {
    // ---------------------------------------------------------- W2 producer
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      const uint64_t pol = policy_evict_last();
      for (int64_t t = 0; t < my_tiles; ++t)
        for (int k = 0; k <= L; ++k) {
          const int m = order_of(k);
          const uint32_t bytes = (uint32_t)S::N2(m) * 128u;
          for (int c = 0; c < S::N1(m) / 32; ++c) {
            mbar_wait(bar(EB2 + st), ph ^ 1);
            if (probe_mode() & 32) {
              mbar_arrive(bar(FB2 + st));
            } else {
              mbar_expect_tx(bar(FB2 + st), bytes);
              bulk_g2s(sB2 + st * B2_STAGE, W2 + S::w2_off(m) + (size_t)c * bytes, bytes, bar(FB2 + st), pol);
            }
            if (++st == NB2) { st = 0; ph ^= 1; }
          }
        }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- lin1 issuer
    // MMA issue is close to synchronous (a shallow queue): the handshakes of
    // one stream leave bubbles that a second, independent stream fills, so
    // lin1 and lin2 have one issuing warp each (each commit tracks its own
    // thread's MMAs).  Unit u's lin1 starts once lin2 of u - 2 is issued (the
    // L1F phase it reuses has been consumed) and the TMEM plan's drain guard
    // holds.  The whole warp runs the loop; one elected lane issues.
    Probe pr;
    const long long t_all = pclock();
    const int nmma = (probe_mode() & 4) ? 1 : 3;
    int st = 0;
    uint32_t ph = 0;
    for (int u = 0; u < total; ++u) {
      const int m = order_of(u);
      long long t0 = pclock();
      spin_until(l2_issued, u - (NL1 - 1));  // the L1F / H1 phases of unit u - NL1 are consumed
      pr.add(4, pclock() - t0);
      t0 = pclock();
      spin_until(drained, u - lag(m));  // the units whose columns R_m reuses are drained
      pr.add(1, pclock() - t0);
      const uint32_t id1 = idesc_f16(S::N1(m)), t_r = tmem + r0_col(m);
      const int nch = S::K1P(m) / 32;
      for (int c = 0; c < nch; ++c) {
        t0 = pclock();
        mbar_wait(bar(FAB + st), ph);
        pr.add(2, pclock() - t0);
        tc_fence_after();
        if (elect_one()) {
          mma_chunk(t_r, sdesc(sA + st * CHUNK), sdesc(sB1 + st * B1_STAGE), id1, c == 0, nmma);
          tc_commit(bar(EAB + st));
          if (c == nch - 1) tc_commit(bar(L1F + u % NL1));
        }
        __syncwarp();
        if (++st == NSA) { st = 0; ph ^= 1; }
      }
    }
    pr.add(9, pclock() - t_all);
    pr.flush(lane == 0);
  } else if (warp == 16) {
    // ------------------------------------------------------- lin2 issuer
    // lin2 of unit u: once Y of unit u - 2 is drained (the L2F phase it
    // reuses) and the gate has read Y_m's columns (H1), one chunk per gated
    // operand chunk as the gate delivers them.
    Probe pr;
    const long long t_all = pclock();
    const int nmma = (probe_mode() & 4) ? 1 : 3;
    int sb = 0;
    uint32_t pb = 0, g2 = 0;
    for (int u = 0; u < total; ++u) {
      const int m = order_of(u);
      long long t0 = pclock();
      spin_until(drained, u - (NL1 - 1));  // the L2F phase of unit u - NL1 is consumed
      pr.add(5, pclock() - t0);
      t0 = pclock();
      mbar_wait(bar(H1 + u % NL1), (u / NL1) & 1);
      pr.add(6, pclock() - t0);
      const uint32_t id2 = idesc_f16(S::N2(m)), t_y = tmem + r0_col(m);
      const int nch = S::N1(m) / 32;
      for (int j = 0; j < nch; ++j, ++g2) {
        const int s2 = (int)(g2 % NS2);
        t0 = pclock();
        mbar_wait(bar(F2 + s2), (g2 / NS2) & 1);
        pr.add(7, pclock() - t0);
        t0 = pclock();
        mbar_wait(bar(FB2 + sb), pb);
        pr.add(8, pclock() - t0);
        tc_fence_after();
        if (elect_one()) {
          mma_chunk(t_y, sdesc(sA2 + s2 * CHUNK), sdesc(sB2 + sb * B2_STAGE), id2, j == 0, nmma);
          tc_commit(bar(E2 + s2));
          tc_commit(bar(EB2 + sb));
          if (j == nch - 1) tc_commit(bar(L2F + u % NL1));
        }
        __syncwarp();
        if (++sb == NB2) { sb = 0; pb ^= 1; }
      }
      if (lane == 0) st_release(smem_u32(l2_issued), (uint32_t)(u + 1));
      __syncwarp();
    }
    pr.add(17, pclock() - t_all);
    pr.flush(lane == 0);
  } else if (warp >= 2 && warp <= 9) {
    // ---------------------------------------------------------------- gate
    const int quad = warp & 3, half = (warp - 2) >> 2;  // the part: chunks q = half mod GATE_PARTS
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float bound_a = 3.f * fmaxf(tmax[0], tmax[edge_slot]);
    const float sa_scale = f16s_pow2_scale(bound_a);
    float sg[32];
    uint32_t gbase = 0;
    int u = 0;
    Probe pr;
    const long long t_all = pclock();
    const bool skip_math = probe_mode() & 1;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x)
      for (int k = 0; k <= L; ++k, ++u) {
        const int m = order_of(k);
        const uint32_t t_r = tmem + lane_off + r0_col(m);
        const int nch = S::N1(m) / 32, ych = S::ych(m);
        const float sc1 = sa_scale * sc.w1[m];  // lin1 accumulator -> fp32 units
        const float s2 = f16s_pow2_scale(sc.w1inf[m] * bound_a);
        const float inv_s2 = 1.f / s2;  // a power of two: exact
        long long t0 = pclock();
        mbar_wait(bar(L1F + u % NL1), (u / NL1) & 1);
        pr.add(10, pclock() - t0);
        tc_fence_after();
        if (m == 0) {  // gate scalars from the l = 0 channels of order 0 (kernels.h:210-226)
          float v[32];
          tmem_ld32(t_r, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) sg[i] = gate ? 1.f / (1.f + expf(-v[i] * sc1)) : 1.f;
        }
        // accumulator -> split operand: (v * sg) * scl with scl = sc1 / s2 a
        // power of two, bit-identical to ((v * sc1) * sg) / s2
        const float scl = sc1 * inv_s2;
        bool head_done = false;
        for (int q = half; q < nch; q += GATE_PARTS) {
          float v[32];
          tmem_ld32(t_r + q * 32, v);
          if (!head_done && q + GATE_PARTS >= ych) {  // this thread's last read of Y_m's columns
            tc_fence_before();
            mbar_arrive(bar(H1 + u % NL1));
            head_done = true;
          }
          const uint32_t gq = gbase + (uint32_t)q, s2i = gq % NS2;
          t0 = pclock();
          // lin2 finished reading this stage.  With two parts and three stages
          // the stage is at most one phase behind here (a part writes chunk g
          // only after g - 3 is consumed, which needs g - 4, the other part's,
          // written), so the parity test cannot alias.
          static_assert(GATE_PARTS == 2 && NS2 == 3, "the parity argument above is for two parts, three stages");
          mbar_wait(bar(E2 + s2i), ((gq / NS2) & 1) ^ 1);
          pr.add(11, pclock() - t0);
          const uint32_t cb = sA2 + s2i * CHUNK;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (probe_mode() & 16) continue;  // probe: no gated-operand stores
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int t = 0; t < 4; ++t)
              if (skip_math)
                hi[t] = lo[t] = __float_as_uint(v[8 * j + 2 * t]);
              else
                split_f16x2((v[8 * j + 2 * t] * sg[8 * j + 2 * t]) * scl, (v[8 * j + 2 * t + 1] * sg[8 * j + 2 * t + 1]) * scl,
                          hi[t], lo[t]);
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(cb + sw128(row, j)), "r"(hi[0]), "r"(hi[1]),
                         "r"(hi[2]), "r"(hi[3])
                         : "memory");
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(cb + sw128(row, 4 + j)), "r"(lo[0]),
                         "r"(lo[1]), "r"(lo[2]), "r"(lo[3])
                         : "memory");
          }
          fence_async_smem();
          mbar_arrive(bar(F2 + s2i));
        }
        if (!head_done) {
          tc_fence_before();
          mbar_arrive(bar(H1 + u % NL1));
        }
        gbase += (uint32_t)nch;
      }
    pr.add(12, pclock() - t_all);
    pr.flush(warp == 2 && lane == 0);
  } else if (warp >= 10 && warp <= 13) {
    // --------------------------------------------------------------- drain
    const int quad = warp & 3;  // one drain warp per TMEM lane quarter
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float bound_a = 3.f * fmaxf(tmax[0], tmax[edge_slot]);
    int u = 0;
    Probe pr;
    const long long t_all = pclock();
    const bool skip_st = probe_mode() & 2;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const int64_t e0 = tile * TILE_M;
      const bool valid = e0 + row < n_e;
      float* ytile = Y + tile * (int64_t)TILE_M * (G::H * E) + row * 4;  // [c / 4][row][4] (F32T)
      for (int k = 0; k <= L; ++k, ++u) {
        const int m = order_of(k);
        const int N2 = S::N2(m);
        const uint32_t t_y = tmem + lane_off + r0_col(m);
        const float sy = f16s_pow2_scale(sc.w1inf[m] * bound_a) * sc.w2[m];
        const long long t0 = pclock();
        mbar_sleep(bar(L2F + u % NL1), (u / NL1) & 1);
        pr.add(13, pclock() - t0);
        tc_fence_after();
        const int c0 = G::moff(m) * E;
        for (int q = 0; q * 32 < N2; ++q) {
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
          if (valid && !skip_st) {
            const int nv = (N2 - q * 32) < 32 ? (N2 - q * 32) : 32;
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              if (i < nv)
                *reinterpret_cast<float4*>(ytile + (int64_t)((c0 + q * 32 + i) >> 2) * (TILE_M * 4)) =
                    make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          }
        }
        tc_fence_before();
        asm volatile("bar.sync 1, %0;\n" ::"n"(DRAIN_THREADS) : "memory");  // all drain lanes read their Y
        if (warp == 10 && lane == 0) st_release(smem_u32(drained), (uint32_t)(u + 1));
      }
    }
    pr.add(14, pclock() - t_all);
    pr.flush(warp == 10 && lane == 0);
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
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [] {
    ESG_CUDA(cudaFuncSetAttribute(k_so2_f16x3<4, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  });
  const int n_sm = sm_count();
  const int64_t tiles = (n_e + TILE_M - 1) / TILE_M;
  const int grid = (int)(tiles < n_sm ? tiles : n_sm);
  if (grid > 0)
    k_so2_f16x3<4, 16><<<grid, THREADS, SMEM_BYTES, st>>>(A1, n_e, W1, W2, sc, tmax, edge_slot, Y, gate, att,
                                                          logits);
  ESG_CUDA(cudaGetLastError());
}

}  // namespace esg
