// Micro-test: where an M = 64 (cta_group::1, kind::f16) tcgen05.mma accumulator lands in TMEM,
// and whether its D address may carry a lane offset of 64. A[m][0] = 64 (m % 32) + (m / 32),
// A[m][1] = 1; B[n][0] = 1, B[n][1] = n  ->  D[m][n] = A[m][0] + n. Two MMAs: D0 at lane 0,
// D1 at lane 64 (B rows offset so D1 = D0 + 1000); every lane's first 4 columns are printed.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2603_03988_b200/csrc
//        tools/micro/m64_layout.cu -o tools/micro/m64_layout
#include <cuda_fp16.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"
#include "tma_host.hpp"

using namespace sortk;
#ifndef LANE_OFF
#define LANE_OFF 16u
#endif

__global__ void k_m64(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmB2, float* out) {
  __shared__ __align__(1024) uint8_t sA[128 * 64];
  __shared__ __align__(1024) uint8_t sB[64 * 64];
  __shared__ __align__(1024) uint8_t sB2[64 * 64];
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
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 128 * 64 + 2 * 64 * 64);
    tma_load_2d(sA, &tmA, &bar, 0, 0);
    tma_load_2d(sB, &tmB, &bar, 0, 0);
    tma_load_2d(sB2, &tmB2, &bar, 0, 0);
    mbar_wait(&bar, 0);
    tc_fence_after();
    uint32_t idesc = umma_idesc_bf16(64, 64) & ~((7u << 7) | (7u << 10));  // A, B fp16, D f32
    for (int k = 0; k < 2; ++k)
      mma_bf16_ss(tmem, umma_sdesc_kmajor(smem_u32(sA) + k * 32, 64), umma_sdesc_kmajor(smem_u32(sB) + k * 32, 64),
                  idesc, k > 0 ? 1u : 0u);
    for (int k = 0; k < 2; ++k)
      mma_bf16_ss(tmem + (LANE_OFF << 16), umma_sdesc_kmajor(smem_u32(sA) + k * 32, 64),
                  umma_sdesc_kmajor(smem_u32(sB2) + k * 32, 64), idesc, k > 0 ? 1u : 0u);
    mma_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  tc_fence_after();
  uint32_t r[32];
  tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16), r);
  tmem_ld_wait();
  for (int i = 0; i < 4; ++i) out[(warp * 32 + lane) * 4 + i] = __uint_as_float(r[i]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

int main() {
  std::vector<__half> A(128 * 32, __float2half(0.f)), B(64 * 32, __float2half(0.f)), B2(64 * 32, __float2half(0.f));
  for (int m = 0; m < 128; ++m) {
    A[m * 32 + 0] = __float2half(64.f * (m % 32) + (m / 32));
    A[m * 32 + 1] = __float2half(1.f);
  }
  for (int n = 0; n < 64; ++n) {
    B[n * 32 + 0] = __float2half(1.f);
    B[n * 32 + 1] = __float2half(static_cast<float>(n));
    B2[n * 32 + 0] = __float2half(1.f);
    B2[n * 32 + 1] = __float2half(1000.f + n);
  }
  __half *dA, *dB, *dB2;
  float* dO;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dB2, B2.size() * 2);
  cudaMalloc(&dO, 128 * 4 * 4);
  cudaMemset(dO, 0, 128 * 4 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB2, B2.data(), B2.size() * 2, cudaMemcpyHostToDevice);
  const CUtensorMap tA = make_tmap_2d(dA, 128, 32, 32, 128, 32, 64);
  const CUtensorMap tB = make_tmap_2d(dB, 64, 32, 32, 64, 32, 64);
  const CUtensorMap tB2 = make_tmap_2d(dB2, 64, 32, 32, 64, 32, 64);
  k_m64<<<1, 128>>>(tA, tB, tB2, dO);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    std::printf("error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> o(128 * 4);
  cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
  // decode: value v = 64 (m % 32) + m / 32 + n (+1000): print (m, n) per lane / column
  for (int lane = 0; lane < 128; lane += (lane % 32 == 0 || lane % 32 == 15 || lane % 32 == 16) ? 1 : 1) {
    if (!(lane % 16 == 0 || lane % 16 == 15)) continue;
    std::printf("lane %3d:", lane);
    for (int c = 0; c < 4; ++c) std::printf(" %8.1f", o[lane * 4 + c]);
    std::printf("\n");
  }
  return 0;
}
