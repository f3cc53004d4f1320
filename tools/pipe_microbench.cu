// FP64 pipe microbenchmark for sm_100a: DMMA (mma.sync m8n8k4 f64) vs DFMA
// issue throughput, all operands in registers, so the number is the pipe's
// ceiling that the GEMM kernels are measured against. Not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_microbench tools/pipe_microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-9;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    int threads = warps * 32;
    int blocks = sms * 2;
    // DMMA: 8 independent chains per warp, 256 FMA per warp-instruction.
    dmma_loop<8><<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<8><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256.0 * 8.0 * iters * (double)blocks * warps;
    printf("{\"probe\":\"dmma_m8n8k4\",\"warps_per_cta\":%d,\"ctas\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n",
           warps, blocks, ms, flops / ms / 1e9);
    dfma_loop<16><<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<16><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 32.0 * 16.0 * iters * (double)blocks * warps;
    printf("{\"probe\":\"dfma\",\"warps_per_cta\":%d,\"ctas\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n",
           warps, blocks, ms, flops / ms / 1e9);
  }
  printf("{\"sms\":%d,\"clock_khz_attr\":%d}\n", sms, clk);
  return 0;
}
