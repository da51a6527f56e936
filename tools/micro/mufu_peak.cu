// Measured MUFU (ex2.approx.ftz.f32) throughput of this GPU: the peak the attention and the
// tied-head log-sum-exp kernels are bound by (one exp per visible logit).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu_peak tools/micro/mufu_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ex2(float* out, int iters) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = -1e-3f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
      v[i] = y - 1.0f;  // keeps the argument in (-1, 0]; the FADD rides the FMA pipe
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 12345.f) out[0] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  float* out;
  cudaMalloc(&out, 4);
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  k_ex2<<<blocks, threads>>>(out, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_ex2<<<blocks, threads>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  const double n = double(blocks) * threads * iters * 8;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"ex2_per_s\": %.4g, \"ms\": %.3f, \"sms\": %d, \"per_sm_per_clk_at_max_clock\": %.2f}\n", n / (ms * 1e-3), ms,
         p.multiProcessorCount, n / (ms * 1e-3) / p.multiProcessorCount / (clk * 1e3));
  return 0;
}
