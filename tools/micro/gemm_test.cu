// Standalone GPU check of the tcgen05 GEMM engine (descriptor / swizzle / TMA
// layout validation) against a CPU fp32 reference. Prints one line per shape.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

#include "../../paper_2603_03988_b200/csrc/gemm.cuh"
#include "../../paper_2603_03988_b200/csrc/tma_host.hpp"

using namespace sortk;

struct StoreF32 {
  static constexpr int kChunk = 32;
  static constexpr int kMaxParts = 1 << 30;
  static constexpr int kSide = 0;
  static constexpr int kRopeFloats = 0;
  float* C;
  int ldc;
  __device__ void prologue(uint8_t*, int, int) const {}
  template <class Wait>
  __device__ void run(uint8_t*, uint8_t*, Wait&& wait, uint32_t tbase, int row, int n0, int c0, int c1, bool valid, int, int) const {
    wait();
    for (int c = c0; c < c1; c += 32) {
      float v[32];
      tmem_row_chunk<32>(tbase + c, v);
      if (valid) for (int i = 0; i < 32; ++i) C[(size_t)row * ldc + n0 + c + i] = v[i];
    }
  }
};

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

static int run(int M, int N, int K, int BN) {
  std::vector<__nv_bfloat16> hA((size_t)M * K), hB((size_t)N * K);
  std::vector<float> fA((size_t)M * K), fB((size_t)N * K);
  srand(M * 7 + N * 3 + K);
  for (size_t i = 0; i < hA.size(); ++i) { float x = bf((rand() % 2001 - 1000) / 1000.f); fA[i] = x; hA[i] = __float2bfloat16(x); }
  for (size_t i = 0; i < hB.size(); ++i) { float x = bf((rand() % 2001 - 1000) / 1000.f); fB[i] = x; hB[i] = __float2bfloat16(x); }
  __nv_bfloat16 *dA, *dB; float* dC;
  cudaMalloc(&dA, hA.size() * 2); cudaMalloc(&dB, hB.size() * 2); cudaMalloc(&dC, (size_t)M * N * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, (size_t)M * N * 4);
  CUtensorMap tA = make_tmap_2d(dA, M, K, K, 128, 64, 128);
  CUtensorMap tB = make_tmap_2d(dB, N, K, K, BN, 64, 128);
  StoreF32 epi; epi.C = dC; epi.ldc = N;
  auto kfn = k_gemm_bf16<StoreF32>;
  GemmPlan gp = gemm_plan(K, BN);
  cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gp.smem_bytes);
  int grid = gemm_grid((M + 127) / 128, N / BN, 148);
  kfn<<<grid, kGemmThreads, gp.smem_bytes>>>(tA, tB, tA, tA, M, N, K, BN, gp.a_stages, epi);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> hC((size_t)M * N);
  cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0; int bad = 0;
  for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) {
    double s = 0; for (int k = 0; k < K; ++k) s += (double)fA[(size_t)i * K + k] * fB[(size_t)j * K + k];
    double err = fabs(s - hC[(size_t)i * N + j]);
    if (err > maxerr) maxerr = err;
    if (err > 1e-2 && bad < 5) { printf("  mismatch (%d,%d): ref %f got %f\n", i, j, s, hC[(size_t)i * N + j]); ++bad; }
  }
  // timing at this shape
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 10; ++it) kfn<<<grid, kGemmThreads, gp.smem_bytes>>>(tA, tB, tA, tA, M, N, K, BN, gp.a_stages, epi);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
  printf("GEMM M=%d N=%d K=%d BN=%d maxerr=%.3g %s  %.3f ms  %.1f TFLOP/s\n", M, N, K, BN, maxerr,
         maxerr < 1e-2 ? "PASS" : "FAIL", ms, 2.0 * M * N * K / ms / 1e9);
  cudaFree(dA); cudaFree(dB); cudaFree(dC);
  return maxerr < 1e-2 ? 0 : 1;
}

int main() {
  int fails = 0;
  fails += run(128, 256, 64, 256);
  fails += run(300, 512, 256, 256);
  fails += run(128, 160, 160, 160);
  fails += run(1000, 1280, 256, 256);
  fails += run(257, 256, 640, 128);
  fails += run(513, 128, 256, 128);
  fails += run(70000, 1024, 256, 256);
  fails += run(20000, 256, 640, 128);
  printf(fails ? "SOME FAILED\n" : "ALL PASS\n");
  return fails;
}
