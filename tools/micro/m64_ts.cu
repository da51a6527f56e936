// Micro-test: the A-from-TMEM operand of an M = 64 tcgen05.mma (TS form). Each TMEM lane L
// holds A = (L, 1, 0, ...) as bf16 in columns [0, 8); B[n] = (1, n, 0, ...) in smem; so
// D[m][n] = (the lane row m was read from) + n. MMA 1: A at lane offset 16, D at lane offset 0;
// MMA 2: A at lane offset 0, D at lane offset 16 (both D at column 32).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2603_03988_b200/csrc
//        tools/micro/m64_ts.cu -o tools/micro/m64_ts
#include <cuda_bf16.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"
#include "tma_host.hpp"

using namespace sortk;

__global__ void k_ts(const __grid_constant__ CUtensorMap tmB, float* out) {
  __shared__ __align__(1024) uint8_t sB[32 * 32];
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&mbar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int L = warp * 32 + lane;
  uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  w[0] = pack_bf16x2(static_cast<float>(L), 1.f);
  tmem_st_32x32b_x8(tmem + (static_cast<uint32_t>(warp * 32) << 16), w);
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 32 * 32);
    tma_load_2d(sB, &tmB, &bar, 0, 0);
    mbar_wait(&bar, 0);
    tc_fence_after();
    const uint32_t idesc = umma_idesc_bf16(64, 32);
#if VARIANT == 0
    mma_bf16_ts(tmem + 32, tmem, umma_sdesc_kmajor(smem_u32(sB), 32), idesc, 0u);
#elif VARIANT == 1
    mma_bf16_ts(tmem + 32 + (16u << 16), tmem, umma_sdesc_kmajor(smem_u32(sB), 32), idesc, 0u);
#else
    mma_bf16_ts(tmem + 32, tmem + (16u << 16), umma_sdesc_kmajor(smem_u32(sB), 32), idesc, 0u);
#endif
    mma_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  tc_fence_after();
  uint32_t r[8];
  tmem_ld_32x32b_x8(tmem + 32 + (static_cast<uint32_t>(warp * 32) << 16), r);
  tmem_ld_wait();
  for (int i = 0; i < 4; ++i) out[L * 4 + i] = __uint_as_float(r[i]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

int main() {
  std::vector<__nv_bfloat16> B(32 * 16, __float2bfloat16(0.f));
  for (int n = 0; n < 32; ++n) {
    B[n * 16 + 0] = __float2bfloat16(1.f);
    B[n * 16 + 1] = __float2bfloat16(static_cast<float>(n));
  }
  __nv_bfloat16* dB;
  float* dO;
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dO, 128 * 4 * 4);
  cudaMemset(dO, 0, 128 * 16);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const CUtensorMap tB = make_tmap_2d(dB, 32, 16, 16, 32, 16, 32);
  k_ts<<<1, 128>>>(tB, dO);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    std::printf("error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> o(128 * 4);
  cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
  for (int lane = 0; lane < 128; ++lane) {
    if (!(lane % 16 == 0 || lane % 16 == 15)) continue;
    std::printf("lane %3d:", lane);
    for (int c = 0; c < 4; ++c) std::printf(" %7.1f", o[lane * 4 + c]);
    std::printf("\n");
  }
  return 0;
}
