// dw_probe.cu -- checks the tensor-core weight-gradient kernel (dw_tc.cu)
// against a host fp64 sum on random rows: per tile max |err| / max |ref|.
//   sh tools/build_dw_probe.sh && tools/bin/dw_probe [n_edges] [which: 0 lin1, 1 lin2] [unused] [timing only]
//   (ESG_DW_SPLIT sets the edge split, default 512)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "device_model.h"

int main(int argc, char** argv) {
  const int L = 4, E = 16, H = 25;
  const int64_t n = argc > 1 ? atoll(argv[1]) : 5000;
  const int which = argc > 2 ? atoi(argv[2]) : 0;
  const int cg = which == 0 ? 2 * E : E, cx = which == 0 ? 3 * E : 2 * E;
  std::vector<float> g(n * H * cg), x(n * H * cx);
  std::mt19937 rng(7);
  std::uniform_real_distribution<float> u(-1.f, 1.f);
  for (auto& v : g) v = u(rng);
  for (auto& v : x) v = u(rng);
  std::vector<esg::DwTile> tiles;
  esg::dw_tiles(L, E, which, &tiles);
  int64_t acc_n = 0;
  for (auto& t : tiles) acc_n = std::max<int64_t>(acc_n, t.acc_off + (int64_t)(t.n0 + t.nN) * t.K);
  float *dg, *dx, *part;
  double* dacc;
  esg::DwTile* dt;
  const int split = getenv("ESG_DW_SPLIT") ? atoi(getenv("ESG_DW_SPLIT")) : 512;
  const int ns = (int)((n + split - 1) / split);
  cudaMalloc(&dg, g.size() * 4);
  cudaMalloc(&dx, x.size() * 4);
  cudaMalloc(&dacc, acc_n * 8);
  cudaMalloc(&part, esg::dw_part_floats((int)tiles.size(), ns) * 4);
  cudaMalloc(&dt, tiles.size() * sizeof(esg::DwTile));
  cudaMemcpy(dg, g.data(), g.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dt, tiles.data(), tiles.size() * sizeof(esg::DwTile), cudaMemcpyHostToDevice);
  cudaMemset(dacc, 0, acc_n * 8);
  cudaMemset(part, 0xFF, esg::dw_part_floats((int)tiles.size(), ns) * 4);
  esg::dw_tf32x3_launch(dg, H * cg, dx, H * cx, n, dt, (int)tiles.size(), split, part, dacc, 0);
  cudaError_t err = cudaDeviceSynchronize();
  {  // timing: 5 launches (accumulating; the check below uses the first)
    std::vector<double> keep(acc_n);
    cudaMemcpy(keep.data(), dacc, acc_n * 8, cudaMemcpyDeviceToHost);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i)
      esg::dw_tf32x3_launch(dg, H * cg, dx, H * cx, n, dt, (int)tiles.size(), split, part, dacc, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("avg %.3f ms per launch (n %lld, which %d)\n", ms / 5, (long long)n, which);
    cudaMemcpy(dacc, keep.data(), acc_n * 8, cudaMemcpyHostToDevice);
  }
  printf("kernel: %s\n", cudaGetErrorString(err));
  {
    std::vector<float> pt(16);
    cudaMemcpy(pt.data(), part, 64, cudaMemcpyDeviceToHost);
    printf("part[0..7]:");
    for (int i = 0; i < 8; ++i) printf(" %.4f", pt[i]);
    printf("\n");
  }
  fflush(stdout);
  if (argc > 4 && atoi(argv[4])) return 0;  // timing only
  std::vector<double> acc(acc_n);
  cudaMemcpy(acc.data(), dacc, acc_n * 8, cudaMemcpyDeviceToHost);
  double worst = 0;
  for (size_t ti = 0; ti < tiles.size(); ++ti) {
    const auto& t = tiles[ti];
    double mx = 0, mref = 0;
    int pn = -1, pk = -1;
    for (int a = 0; a < t.nN; ++a)
      for (int b = 0; b < t.nK; ++b) {
        double s = 0;
        for (int64_t e = 0; e < n; ++e) s += (double)g[e * H * cg + t.goff + a] * x[e * H * cx + t.xoff + b];
        const double got = acc[t.acc_off + (int64_t)(t.n0 + a) * t.K + t.k0 + b];
        if (std::fabs(got - s) > mx) {
          mx = std::fabs(got - s);
          pn = a;
          pk = b;
        }
        mref = std::max(mref, std::fabs(s));
      }
    printf("tile %zu goff %d xoff %d nN %d nK %d nKp %d: max err %.3e (ref max %.3e) at (%d,%d)\n", ti, t.goff, t.xoff,
           t.nN, t.nK, t.nKp, mx, mref, pn, pk);
    worst = std::max(worst, mx / mref);
    if (ti == 0) {
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 6; ++b) {
          double s = 0;
          for (int64_t e = 0; e < n; ++e) s += (double)g[e * H * cg + t.goff + a] * x[e * H * cx + t.xoff + b];
          printf("  (%d,%d) got %.6f want %.6f\n", a, b, acc[t.acc_off + (int64_t)(t.n0 + a) * t.K + t.k0 + b], s);
        }
    }
  }
  printf("worst rel %.3e\n", worst);
  return worst < 1e-5 ? 0 : 1;
}
