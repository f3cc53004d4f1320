// dgemm_paper.cuh — the paper's hand-rolled CUDA kernel, restated for sm_100a.
//
// Faithful to the reference's per-thread program tiledKernelThread
// (/root/reference/pkg/gpu/src/kernel.ts:50-78): one
// K x K thread block per output tile, each thread owns one output cell; per
// phase every thread loads one zero-filled cell of the A tile and of the B
// tile into shared memory, barrier, K-long dot product into a register running
// sum, barrier; guarded single store at the end.
//
// The multiply and add are issued as separate round-to-nearest operations
// (__dmul_rn / __dadd_rn, so no FMA contraction) in k order, which makes the
// result bitwise equal to the reference's naive oracle (kernels.py:19-29):
// padding cells add exactly +0.0. This variant is the correctness anchor and
// the paper's "CUDA" row; the DMMA variants are the performance path.
#pragma once
#include <cstdint>

namespace tb {

__global__ void dgemm_paper_kernel(const double* __restrict__ a, int64_t lda, const double* __restrict__ b,
                                   int64_t ldb, double* __restrict__ c, int64_t ldc, int m, int k, int n,
                                   int K, int accumulate) {
  extern __shared__ double paper_smem[];
  double* left = paper_smem;       // K x K tile of A
  double* right = paper_smem + K * K;  // K x K tile of B
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int row = blockIdx.y * K + ty;
  const int col = blockIdx.x * K + tx;
  const int slot = ty * K + tx;

  double acc = 0.0;  // register running sum (kernel.ts:57)
  const int phases = (k + K - 1) / K;
  for (int phase = 0; phase < phases; ++phase) {
    const int a_col = phase * K + tx;
    left[slot] = (row < m && a_col < k) ? a[(int64_t)row * lda + a_col] : 0.0;
    const int b_row = phase * K + ty;
    right[slot] = (b_row < k && col < n) ? b[(int64_t)b_row * ldb + col] : 0.0;
    __syncthreads();  // every tile cell loaded before anyone reads (kernel.ts:65)
    const int row_base = ty * K;
    for (int kk = 0; kk < K; ++kk) acc = __dadd_rn(acc, __dmul_rn(left[row_base + kk], right[kk * K + tx]));
    __syncthreads();  // every read done before the next phase overwrites (kernel.ts:72)
  }
  if (row < m && col < n) {
    double* dst = c + (int64_t)row * ldc + col;
    *dst = accumulate ? __dadd_rn(*dst, acc) : acc;
  }
}

}  // namespace tb
