/*
 * tb_oracle.c — TEST INFRASTRUCTURE ONLY. CPU restatement of the reference's
 * FP64 square-GEMM path (tilebench, arXiv 2509.04594), used as the parity
 * checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs. The product path (paper_2509_04594_b200) never
 * links, loads or calls this file.
 *
 * Parity pin: tests/golden/ holds vectors produced by importing the reference
 * package itself (tests/golden/make_golden.py); tests/test_oracle.py checks
 * this restatement against them BITWISE (same op sequence, no FMA contraction:
 * the reference compiles its kernels with numba and no fastmath,
 * /root/reference/pkg/src/tilebench/kernels.py:1-9).
 *
 * Build: oracle/Makefile  (gcc -O2 -ffp-contract=off -pthread)
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define EXPORT __attribute__((visibility("default")))

/* naive_kernel — reference pkg/src/tilebench/kernels.py:19-29.
 * c[i,j] = sum_k a[i,k]*b[k,j], running sum in index order, one store. */
EXPORT void tbo_naive(const double* a, const double* b, double* out,
                      int64_t m, int64_t kk, int64_t n) {
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t k = 0; k < kk; ++k) acc += a[i * kk + k] * b[k * n + j];
      out[i * n + j] = acc;
    }
  }
}

/* tile_range_kernel — reference kernels.py:32-53.
 * Output tiles [start, stop) of the row-major (i0, j0) tile grid; per tile
 * the k0 phases run in order, each phase sums into a fresh acc and adds it to
 * out (which the caller pre-zeroes, backends.py:114,147,171). */
EXPORT void tbo_tile_range(const double* a, const double* b, double* out,
                           int64_t m, int64_t kk, int64_t n,
                           int64_t start, int64_t stop, int64_t tk) {
  const int64_t jt = (n + tk - 1) / tk;
  for (int64_t idx = start; idx < stop; ++idx) {
    const int64_t i0 = (idx / jt) * tk;
    const int64_t j0 = (idx % jt) * tk;
    const int64_t i_end = i0 + tk < m ? i0 + tk : m;
    const int64_t j_end = j0 + tk < n ? j0 + tk : n;
    for (int64_t k0 = 0; k0 < kk; k0 += tk) {
      const int64_t k_end = k0 + tk < kk ? k0 + tk : kk;
      for (int64_t i = i0; i < i_end; ++i) {
        for (int64_t j = j0; j < j_end; ++j) {
          double acc = 0.0;
          for (int64_t k = k0; k < k_end; ++k) acc += a[i * kk + k] * b[k * n + j];
          out[i * n + j] += acc;
        }
      }
    }
  }
}

/* plan_partitions — reference backends.py:119-136: contiguous chunks, the
 * first `extra` workers take one more tile. Writes up to `threads` (start,
 * stop) pairs into chunks[]; returns the number of non-empty chunks. */
EXPORT int64_t tbo_plan_partitions(int64_t num_tiles, int64_t threads, int64_t* chunks) {
  int64_t workers = threads < num_tiles ? threads : num_tiles;
  if (workers <= 0) return 0;
  const int64_t base = num_tiles / workers, extra = num_tiles % workers;
  int64_t start = 0;
  for (int64_t w = 0; w < workers; ++w) {
    const int64_t stop = start + base + (w < extra ? 1 : 0);
    chunks[2 * w] = start;
    chunks[2 * w + 1] = stop;
    start = stop;
  }
  return workers;
}

/* tiled_parallel_multiply — reference backends.py:139-160 (the paper's
 * "OpenMP collapse" row): the flattened tile grid split by
 * plan_partitions, one worker per chunk. `out` must be zeroed by the caller.
 * Output is bitwise identical to tiled_seq for every thread count
 * (backends.py:21-24) because each tile runs the same loop nest. */
struct tbo_job {
  const double *a, *b;
  double* out;
  int64_t m, kk, n, start, stop, tk;
};

static void* tbo_worker(void* p) {
  const struct tbo_job* j = (const struct tbo_job*)p;
  tbo_tile_range(j->a, j->b, j->out, j->m, j->kk, j->n, j->start, j->stop, j->tk);
  return NULL;
}

#define TBO_MAX_WORKERS 1024

EXPORT void tbo_tiled_parallel(const double* a, const double* b, double* out,
                               int64_t m, int64_t kk, int64_t n, int64_t tk, int64_t threads) {
  const int64_t it = (m + tk - 1) / tk, jt = (n + tk - 1) / tk;
  const int64_t num_tiles = it * jt;
  if (threads > TBO_MAX_WORKERS) threads = TBO_MAX_WORKERS;
  int64_t chunks[2 * TBO_MAX_WORKERS];
  const int64_t workers = tbo_plan_partitions(num_tiles, threads, chunks);
  if (workers <= 1) {
    tbo_tile_range(a, b, out, m, kk, n, 0, num_tiles, tk);
    return;
  }
  pthread_t tid[TBO_MAX_WORKERS];
  struct tbo_job jobs[TBO_MAX_WORKERS];
  for (int64_t w = 0; w < workers; ++w) {
    jobs[w] = (struct tbo_job){a, b, out, m, kk, n, chunks[2 * w], chunks[2 * w + 1], tk};
    pthread_create(&tid[w], NULL, tbo_worker, &jobs[w]);
  }
  for (int64_t w = 0; w < workers; ++w) pthread_join(tid[w], NULL);
}

/* tiledKernelThread — reference pkg/gpu/src/kernel.ts:50-78 (the paper's
 * hand-rolled CUDA kernel), restated on the CPU: one running
 * sum per output cell over all phases, zero-filled shared tiles, so padding
 * cells add exactly +0.0. Bitwise equal to tbo_naive for finite inputs. */
EXPORT void tbo_paper_kernel(const double* a, const double* b, double* c,
                             int64_t m, int64_t k, int64_t n, int64_t K) {
  const int64_t phases = (k + K - 1) / K;
  for (int64_t row = 0; row < m; ++row) {
    for (int64_t col = 0; col < n; ++col) {
      double acc = 0.0;
      for (int64_t p = 0; p < phases; ++p) {
        for (int64_t kk = 0; kk < K; ++kk) {
          const int64_t ka = p * K + kk;
          const double l = ka < k ? a[row * k + ka] : 0.0;
          const double r = ka < k ? b[ka * n + col] : 0.0;
          acc += l * r;
        }
      }
      c[row * n + col] = acc;
    }
  }
}

/* max_abs_rel_diff — reference matrices.py:73-86 (also kernel.ts:102-113):
 * max over elements of |a-b| / max(|a|, |b|, 1). */
EXPORT double tbo_max_abs_rel_diff(const double* x, const double* y, int64_t count) {
  double worst = 0.0;
  for (int64_t i = 0; i < count; ++i) {
    double d = fabs(x[i]) > fabs(y[i]) ? fabs(x[i]) : fabs(y[i]);
    if (d < 1.0) d = 1.0;
    const double r = fabs(x[i] - y[i]) / d;
    if (r > worst || r != r) worst = r;
  }
  return worst;
}

/* Normwise relative error ||x - ref||_F / ||ref||_F — the BASELINE.json
 * north-star parity metric (threshold 1e-12). Long-double accumulation. */
EXPORT double tbo_normwise_rel(const double* x, const double* ref, int64_t count) {
  long double num = 0.0L, den = 0.0L;
  for (int64_t i = 0; i < count; ++i) {
    const long double d = (long double)x[i] - (long double)ref[i];
    num += d * d;
    den += (long double)ref[i] * (long double)ref[i];
  }
  if (den == 0.0L) return num == 0.0L ? 0.0 : INFINITY;
  return (double)sqrtl(num / den);
}

EXPORT int tbo_max_threads(void) { return (int)sysconf(_SC_NPROCESSORS_ONLN); }
