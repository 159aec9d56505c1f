// f16x3_probe.cu -- standalone timing probe for the fp16x3 SO(2) chain.
//
// Builds k_so2_f16x3 with F16X3_PROBE (per-role clock64 accounting of every
// wait, the MMA issuer's idle time by cause) and launches it on synthetic
// operands under each experiment mode given on the command line, printing
// the kernel time and the per-role breakdown in cycles per tile (CTA mean).
// Development tool only; not part of the library or the tests.
//
//   tools/build_f16x3_probe.sh && ./tools/bin/f16x3_probe [edges] [modes...]
#define F16X3_PROBE 1
#include "../paper_2507_03840_b200/csrc/so2_f16x3.cu"

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

using namespace esg;

// raw issue rate of kind::f16 MMAs (M = 128, given N) from one SMEM stage
// into one accumulator: `reps` chunks of mma_chunk (6 MMAs), one commit per
// chunk (commit_every > 0) or only at the end; cycles per chunk into out
__global__ void __launch_bounds__(128, 1) k_mma_rate(int N, int reps, int commit_every, int nmma, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sA = smem_u32(base), sB = sA + 16384;
  uint64_t* bars = (uint64_t*)(base + 16384 + 32768);
  uint32_t* slot = (uint32_t*)(bars + 4);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    mbar_init(smem_u32(&bars[1]), (1 << 20) - 1);  // never completes: arrivals only
    mbar_init(smem_u32(&bars[2]), 1);
    mbar_init(smem_u32(&bars[3]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x3c003c00u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0) {
    const long long t0 = clock64();
    const uint32_t id = idesc_f16(N);
    uint32_t ph = 0;
    for (int r = 0; r < reps; ++r) {
      if (commit_every < 0) {  // the chain's per-chunk extras: a phase test, a fence, two async commits
        (void)mbar_test(smem_u32(&bars[1]), 0);
        if (commit_every == -2) tc_fence_after();
        if (commit_every == -3) {  // v1 style: two blocking waits that are already satisfied
          mbar_wait(smem_u32(&bars[2]), 1);
          mbar_wait(smem_u32(&bars[3]), 1);
          tc_fence_after();
        }
        if (commit_every == -4) {  // v2 style: warp-uniform non-blocking tests
          const bool a = __shfl_sync(0xffffffffu, (int)mbar_test(smem_u32(&bars[2]), 1), 0);
          const bool b = a && __shfl_sync(0xffffffffu, (int)mbar_test(smem_u32(&bars[3]), 1), 0);
          const bool c = b && __shfl_sync(0xffffffffu, (int)mbar_test(smem_u32(&bars[2]), 1), 0);
          if (!c) __nanosleep(1000);
          tc_fence_after();
        }
      }
      if (elect_one()) {
        mma_chunk(tmem, sdesc(sA), sdesc(sB), id, r == 0, nmma);
        if (commit_every > 0 && (r % commit_every) == commit_every - 1) tc_commit(smem_u32(&bars[0]));
        if (commit_every < 0) {
          tc_commit(smem_u32(&bars[1]));
          tc_commit(smem_u32(&bars[1]) + 0);
        }
      }
      __syncwarp();
      if (commit_every > 0 && (r % commit_every) == commit_every - 1) {
        mbar_wait(smem_u32(&bars[0]), ph);
        ph ^= 1;
      }
    }
    if (commit_every <= 0) {
      if (commit_every < 0) {  // drain the extra arrivals' phases: wait for the final commit below
      }
      if (elect_one()) tc_commit(smem_u32(&bars[0]));
      __syncwarp();
      mbar_wait(smem_u32(&bars[0]), 0);
    }
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

void mma_rate_tests() {
  long long* d;
  cudaMalloc(&d, 1024 * 8);
  cudaFuncSetAttribute(k_mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  int grid = 0;
  cudaDeviceGetAttribute(&grid, cudaDevAttrMultiProcessorCount, 0);
  for (int nmma : {3, 1})
    for (int N : {32, 64, 128, 256})
      for (int ce : {0, -2, -3, -4}) {
        const int reps = 400;
        k_mma_rate<<<grid, 128, 64 * 1024>>>(N, reps, ce, nmma, d);
        cudaDeviceSynchronize();
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
        double s = 0;
        for (auto x : h) s += x;
        s /= grid;
        const double per_mma = s / reps / (2 * nmma), floor = 128.0 * N / 256;
        printf("mma N=%3d nmma=%d commit_every=%d: %.1f cycles/MMA (floor %.0f) %s\n", N, nmma, ce, per_mma, floor,
               cudaGetErrorString(cudaGetLastError()));
      }
  cudaFree(d);
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "rate") {
    mma_rate_tests();
    return 0;
  }
  const int64_t n_e = argc > 1 ? atoll(argv[1]) : 2000000;
  std::vector<int> modes;
  for (int i = 2; i < argc; ++i) modes.push_back(atoi(argv[i]));
  if (modes.empty()) modes = {0, 1, 2, 4, 7};
  const int64_t tiles = (n_e + 127) / 128;
  const size_t a1 = (size_t)tiles * so2_f16x3_a1_tile_bytes(4, 16);
  const size_t w1 = so2_f16x3_w1_bytes(4, 16), w2 = so2_f16x3_w2_bytes(4, 16);
  const size_t y = (size_t)tiles * 128 * 400 * 4;
  void *dA, *dW1, *dW2, *dY;
  float *dAtt, *dLog, *dT;
  cudaMalloc(&dA, a1);
  cudaMalloc(&dW1, w1);
  cudaMalloc(&dW2, w2);
  cudaMalloc(&dY, y);
  cudaMalloc(&dAtt, 64);
  cudaMalloc(&dLog, n_e * 4);
  cudaMalloc(&dT, 64);
  cudaMemset(dA, 0x3c, a1);  // fp16 ~1.0 everywhere
  cudaMemset(dW1, 0x1c, w1);
  cudaMemset(dW2, 0x1c, w2);
  cudaMemset(dAtt, 0, 64);
  std::vector<float> tmax(16, 1.f);
  cudaMemcpy(dT, tmax.data(), 64, cudaMemcpyHostToDevice);
  F16x3Scales sc;
  for (int m = 0; m < 8; ++m) sc.w1[m] = sc.w2[m] = sc.w1inf[m] = 1.f;
  int grid = 0;
  cudaDeviceGetAttribute(&grid, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[24] = {"",                 "lin1<-drained",    "lin1<-A1/W1",    "",
                           "lin1<-lin2 issued", "lin2<-drained",   "lin2<-H1",       "lin2<-F2 gate",
                           "lin2<-W2",         "lin1 total",       "gate wait L1F",  "gate wait E2",
                           "gate total",       "drain wait L2F",   "drain total",    "A wait EAB",
                           "A total",          "lin2 total",       "W1 wait EAB",    "W1 total",
                           "",                 "",                 "",               ""};
  for (int mode : modes) {
    cudaMemcpyToSymbol(g_probe_mode, &mode, sizeof(int));
    for (int rep = 0; rep < 2; ++rep)
      so2_f16x3_launch(4, 16, (const uint8_t*)dA, n_e, (const uint8_t*)dW1, (const uint8_t*)dW2, sc, dT, 1,
                       (float*)dY, 1, dAtt, dLog, 0);
    std::vector<long long> zero(1024 * 32, 0);
    cudaMemcpyToSymbol(g_probe, zero.data(), zero.size() * sizeof(long long));
    cudaEventRecord(e0);
    so2_f16x3_launch(4, 16, (const uint8_t*)dA, n_e, (const uint8_t*)dW1, (const uint8_t*)dW2, sc, dT, 1,
                     (float*)dY, 1, dAtt, dLog, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t err = cudaGetLastError();
    std::vector<long long> p(1024 * 32);
    cudaMemcpyFromSymbol(p.data(), g_probe, p.size() * sizeof(long long));
    const double tiles_per_cta = (double)tiles / grid;
    printf("mode %d: %.3f ms for %lld edges (%s), %.1f tiles per CTA\n", mode, ms, (long long)n_e,
           cudaGetErrorString(err), tiles_per_cta);
    for (int i = 0; i < 20; ++i) {
      if (!names[i][0]) continue;
      double s = 0;
      for (int b = 0; b < grid; ++b) s += (double)p[b * 32 + i];
      printf("  %-18s %10.0f cycles/tile\n", names[i], s / grid / tiles_per_cta);
    }
  }
  return 0;
}
