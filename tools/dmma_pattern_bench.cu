// DMMA issue-pattern microbenchmark (tooling, not product): how close can a
// warp tile of MI x NI m8n8k4 accumulators get to the FP64 pipe peak when the
// A/B fragments rotate per instruction (register-resident), and when they are
// re-loaded from shared memory every k-step like the GEMM mainloop?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_pattern_bench tools/dmma_pattern_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MI, int NI, bool SMEM>
__global__ void __launch_bounds__(256, 1) pattern(double* out, int iters) {
  __shared__ double sh[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sh[i] = 1e-3 * i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double a[MI], b[NI];
#pragma unroll
  for (int i = 0; i < MI; ++i) a[i] = sh[lane + 32 * i];
#pragma unroll
  for (int j = 0; j < NI; ++j) b[j] = sh[1024 + lane + 32 * j];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (SMEM) {
#pragma unroll
        for (int i = 0; i < MI; ++i) a[i] = sh[((it * 4 + s) * 64 + lane + 32 * i) & 2047];
#pragma unroll
        for (int j = 0; j < NI; ++j) b[j] = sh[2048 + (((it * 4 + s) * 32 + lane + 32 * j) & 2047)];
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 1234.5) out[0] = s;
}

template <int MI, int NI, bool SMEM>
void run(const char* name, int sms, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  pattern<MI, NI, SMEM><<<sms, 256>>>(out, 10);
  cudaEventRecord(e0);
  pattern<MI, NI, SMEM><<<sms, 256>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256 * MI * NI * 4.0 * iters * 8.0 * sms;
  printf("{\"probe\":\"%s\",\"MI\":%d,\"NI\":%d,\"smem\":%d,\"tflops\":%.3f}\n", name, MI, NI, (int)SMEM,
         flops / ms / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  run<8, 4, false>("regs", sms, out);
  run<4, 8, false>("regs", sms, out);
  run<8, 4, true>("smem", sms, out);
  run<4, 8, true>("smem", sms, out);
  run<4, 4, false>("regs", sms, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"status\":\"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
