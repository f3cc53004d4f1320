// Small C-ABI driver for compute-sanitizer (memcheck / racecheck / synccheck):
// runs every variant on ragged shapes that exercise TMA out-of-bounds fill,
// the cp.async zero-fill path, the stream-K split/fixup path and the paper
// kernel, through include/tbgpu.h only. Exit code 0 = all calls OK.
//   nvcc -O2 -I include -o tools/sanitize_driver tools/sanitize_driver.cu \
//        -L paper_2509_04594_b200 -ltbgpu -Xlinker -rpath,$PWD/paper_2509_04594_b200
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "tbgpu.h"

// Usage: sanitize_driver [--tma-only] [--pipeline] [--mgpu]
//   --tma-only: even shapes and TMA-fed variants only (racecheck does not
//   model mbarrier-ordered cp.async writes; see tests/test_gpu_sanitizer.py).
//   --pipeline: also one host-buffer call large enough for the copy/compute
//   pipeline (the flag-driven PIPE-mode phase-1 launch + row blocks).
//   --mgpu: also tb_dgemm_mgpu with device 0 listed three times (chain of
//   peer copies + K-panel GEMMs, a zero-row entry, 64-row panels).
// TB_BM=128 in the environment forces the 128-row tiles on these small shapes.
int main(int argc, char** argv) {
  bool tma_only = false, pipeline = false, mgpu = false;
  for (int i = 1; i < argc; ++i) {
    tma_only |= std::string(argv[i]) == "--tma-only";
    pipeline |= std::string(argv[i]) == "--pipeline";
    mgpu |= std::string(argv[i]) == "--mgpu";
  }
  struct Shape {
    long m, k, n;
  };
  const Shape shapes[] = {{33, 33, 33}, {129, 130, 131}, {256, 300, 128}, {515, 515, 515}, {130, 66, 258}};
  std::vector<int> variants = {TB_VARIANT_PAPER, TB_VARIANT_DMMA_TMA, TB_VARIANT_DFMA};
  if (!tma_only) variants.push_back(TB_VARIANT_DMMA_CPASYNC);
  int failures = 0;
  for (const Shape& s : shapes) {
    if (tma_only && (s.k % 2 || s.n % 2)) continue;
    std::vector<double> a(s.m * s.k), b(s.k * s.n), ref(s.m * s.n, 0.0), c(s.m * s.n);
    for (size_t i = 0; i < a.size(); ++i) a[i] = 2.0 + 3.0 * ((i * 2654435761u) % 1000) / 1000.0;
    for (size_t i = 0; i < b.size(); ++i) b[i] = 2.0 + 3.0 * ((i * 40503u) % 1000) / 1000.0;
    for (long i = 0; i < s.m; ++i)
      for (long p = 0; p < s.k; ++p)
        for (long j = 0; j < s.n; ++j) ref[i * s.n + j] += a[i * s.k + p] * b[p * s.n + j];
    double *dA, *dB, *dC;
    cudaMalloc(&dA, a.size() * 8);
    cudaMalloc(&dB, b.size() * 8);
    cudaMalloc(&dC, c.size() * 8);
    cudaMemcpy(dA, a.data(), a.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, b.data(), b.size() * 8, cudaMemcpyHostToDevice);
    for (int v : variants) {
      double sec = 0;
      const int st = tb_dgemm(dA, dB, dC, s.m, s.k, s.n, 32, v, 0, nullptr, &sec);
      cudaMemcpy(c.data(), dC, c.size() * 8, cudaMemcpyDeviceToHost);
      double num = 0, den = 0;
      for (size_t i = 0; i < c.size(); ++i) {
        num += (c[i] - ref[i]) * (c[i] - ref[i]);
        den += ref[i] * ref[i];
      }
      const double rel = std::sqrt(num / den);
      const bool ok = st == TB_STATUS_OK && rel <= 1e-12;
      failures += !ok;
      std::printf("%ldx%ldx%ld variant=%s status=%d normwise=%.2e %s\n", s.m, s.k, s.n, tb_variant_name(v), st, rel,
                  ok ? "ok" : tb_last_error());
    }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
  }
  if (pipeline) {
    const long m = 2560, k = 8192, n = 2560;  // 1.07e11 flops: pipelined (phase 1 + row blocks)
    std::vector<double> a(m * k), b(k * n), c(m * n);
    for (size_t i = 0; i < a.size(); ++i) a[i] = 2.0 + 3.0 * ((i * 2654435761u) % 1000) / 1000.0;
    for (size_t i = 0; i < b.size(); ++i) b[i] = 2.0 + 3.0 * ((i * 40503u) % 1000) / 1000.0;
    double sec = 0, e2e = 0;
    const int st = tb_gpu_tiled_multiply_flat_ex(0, a.data(), b.data(), m, k, n, 32, TB_VARIANT_AUTO, c.data(),
                                                 (long)c.size(), &sec, &e2e);
    // spot-check rows against a host dot product
    double num = 0, den = 0;
    for (long i = 0; i < m; i += 509)
      for (long j = 0; j < n; j += 7) {
        double r = 0;
        for (long p = 0; p < k; ++p) r += a[i * k + p] * b[p * n + j];
        num += (c[i * n + j] - r) * (c[i * n + j] - r);
        den += r * r;
      }
    const double rel = std::sqrt(num / den);
    const bool ok = st == TB_STATUS_OK && rel <= 1e-12;
    failures += !ok;
    std::printf("pipeline %ldx%ldx%ld status=%d normwise=%.2e %s\n", m, k, n, st, rel, ok ? "ok" : tb_last_error());
  }
  if (mgpu) {
    const long k = 300, n = 258;
    const long rows[3] = {70, 0, 133};
    std::vector<double> b(k * n);
    for (size_t i = 0; i < b.size(); ++i) b[i] = 2.0 + 3.0 * ((i * 40503u) % 1000) / 1000.0;
    double *dB, *dA[3] = {}, *dC[3] = {}, *dR[3] = {};
    cudaMalloc(&dB, b.size() * 8);
    cudaMemcpy(dB, b.data(), b.size() * 8, cudaMemcpyHostToDevice);
    std::vector<std::vector<double>> a(3);
    for (int d = 0; d < 3; ++d) {
      a[d].resize(rows[d] * k);
      for (size_t i = 0; i < a[d].size(); ++i) a[d][i] = 2.0 + 3.0 * (((i + 977 * d) * 2654435761u) % 1000) / 1000.0;
      if (rows[d]) {
        cudaMalloc(&dA[d], a[d].size() * 8);
        cudaMalloc(&dC[d], rows[d] * n * 8);
        cudaMemcpy(dA[d], a[d].data(), a[d].size() * 8, cudaMemcpyHostToDevice);
      }
      if (d) cudaMalloc(&dR[d], b.size() * 8);
    }
    setenv("TB_MGPU_PANEL", "64", 1);
    const int devs[3] = {0, 0, 0};
    const int64_t rws[3] = {rows[0], rows[1], rows[2]};
    double kmax = 0, total = 0;
    const int st = tb_dgemm_mgpu(3, devs, dA, dB, dR, dC, rws, k, n, TB_VARIANT_AUTO, &kmax, &total);
    unsetenv("TB_MGPU_PANEL");
    double num = 0, den = 0;
    for (int d = 0; d < 3; ++d) {
      if (!rows[d]) continue;
      std::vector<double> c(rows[d] * n);
      cudaMemcpy(c.data(), dC[d], c.size() * 8, cudaMemcpyDeviceToHost);
      for (long i = 0; i < rows[d]; ++i)
        for (long j = 0; j < n; ++j) {
          double r = 0;
          for (long p = 0; p < k; ++p) r += a[d][i * k + p] * b[p * n + j];
          num += (c[i * n + j] - r) * (c[i * n + j] - r);
          den += r * r;
        }
    }
    const double rel = std::sqrt(num / den);
    const bool ok = st == TB_STATUS_OK && rel <= 1e-12;
    failures += !ok;
    std::printf("mgpu 3 entries k=%ld n=%ld status=%d normwise=%.2e %s\n", k, n, st, rel, ok ? "ok" : tb_last_error());
    for (int d = 0; d < 3; ++d) {
      cudaFree(dA[d]);
      cudaFree(dC[d]);
      cudaFree(dR[d]);
    }
    cudaFree(dB);
  }
  tb_release();
  return failures ? 1 : 0;
}
