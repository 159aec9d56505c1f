// so2_probe.cu -- standalone timing probe for the tcgen05 SO(2) chain.
//
// Builds k_so2_tc with SO2_PROBE (clock64 accounting of every mbarrier wait,
// per warp role) and launches it on synthetic operands, printing the kernel
// time, the per-tile time and the per-role wait breakdown averaged over CTAs.
// Development tool only; not part of the library or the tests.
//
//   make -C tools so2_probe && ./tools/so2_probe [edges]
#define SO2_PROBE 1
#include "../paper_2507_03840_b200/csrc/so2_tc.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

using namespace esg;

int main(int argc, char** argv) {
  const int64_t n_e = argc > 1 ? atoll(argv[1]) : 2000000;
  using Y1 = Lay1<4, 16, 64>;
  const int64_t tiles = (n_e + 127) / 128;
  size_t w1 = 0, w2 = 0;
  for (int m = 0; m <= 4; ++m) {
    w1 += (size_t)Y1::N1(m) * Y1::KP(m) * 2;
    w2 += (size_t)Y1::N2(m) * Y1::N1P(m) * 2;
  }
  const size_t a1 = (size_t)tiles * (Y1::KTOT / 64) * 16384, y = (size_t)n_e * 25 * 16 * 2;
  void *dA, *dW1, *dW2, *dY;
  float *dAtt, *dLog;
  cudaMalloc(&dA, a1);
  cudaMalloc(&dW1, w1);
  cudaMalloc(&dW2, w2);
  cudaMalloc(&dY, y);
  cudaMalloc(&dAtt, 64);
  cudaMalloc(&dLog, n_e * 4);
  cudaMemset(dA, 0x3c, a1);
  cudaMemset(dW1, 0x3c, w1);
  cudaMemset(dW2, 0x3c, w2);
  cudaMemset(dAtt, 0, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep)
    so2_tc_launch(4, 16, (const uint16_t*)dA, n_e, (const uint16_t*)dW1, (const uint16_t*)dW2, (uint16_t*)dY, 1,
                  dAtt, dLog, 0);
  const int reps = 5;
  cudaEventRecord(e0);
  for (int rep = 0; rep < reps; ++rep)
    so2_tc_launch(4, 16, (const uint16_t*)dA, n_e, (const uint16_t*)dW1, (const uint16_t*)dW2, (uint16_t*)dY, 1,
                  dAtt, dLog, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const cudaError_t err = cudaGetLastError();
  std::vector<long long> p(1024 * 32);
  cudaMemcpyFromSymbol(p.data(), g_so2_probe, p.size() * sizeof(long long));
  int grid = 0;
  cudaDeviceGetAttribute(&grid, cudaDevAttrMultiProcessorCount, 0);
  if (tiles < grid) grid = (int)tiles;
  const double tiles_per_cta = (double)tiles / grid;
  const double bytes = (double)n_e * (Y1::KTOT * 2 + 400 * 2);
  printf("edges %lld tiles %lld grid %d err %s\n", (long long)n_e, (long long)tiles, grid, cudaGetErrorString(err));
  printf("kernel %.3f ms  %.1f M edges/s  %.1f GB/s (A1 + Y)  %.2f us/tile/CTA\n", ms, n_e / ms / 1e3,
         bytes / ms / 1e6, ms * 1e3 / tiles_per_cta);
  const char* names[21] = {"mma.wait_FA",  "mma.wait_FB1", "mma.wait_drain", "mma.wait_A2F", "mma.wait_FB2",
                           "mma.total",    "Aprod.wait_EA", "Aprod.total", "Bprod.wait_EB", "Bprod.total",
                           "gate.wait_L1F", "gate.total",  "drain.wait_L2F", "drain.total", "gate.wait_A2E", "gate.fence_arrive",
                           "mma.issue_lin1", "mma.issue_lin2", "mma.lin2_guard", "drain.tmem_ld", "gate.sigmoid"};
  for (int i = 0; i < 21; ++i) {
    double s = 0;
    for (int b = 0; b < grid; ++b) s += p[b * 32 + i];
    printf("  %-15s %10.0f cycles/tile\n", names[i], s / grid / tiles_per_cta);
  }
  std::vector<long long> t(256);
  cudaMemcpyFromSymbol(t.data(), g_so2_trace, 256 * sizeof(long long));
  const long long t0 = t[0];
  auto r = [&](int i) { return t[i] ? t[i] - t0 : -1; };
  printf("timeline of tile iteration 2, CTA 0 (cycles from the first lin1 issue)\n");
  for (int m = 0; m <= 4; ++m) {
    printf(" m=%d MMA: lin1 start %6lld issued %6lld lin2(m-1) issued %6lld | gate: L1F %6lld A2E %6lld arrive %6lld"
           " | drain: L2F %6lld done %6lld\n",
           m, r(m * 8), r(m * 8 + 1), r(m * 8 + 2), r(64 + m * 8), r(64 + m * 8 + 1), r(64 + m * 8 + 2),
           r(128 + m * 4), r(128 + m * 4 + 1));
  }
  return 0;
}
