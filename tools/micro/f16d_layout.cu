// Micro-test: the TMEM layout of a 16-bit (f16) tcgen05.mma accumulator (kind::f16, M = 128,
// N = 64, fp16 A / B), read back with tcgen05.ld.32x32b.x32. D[m][n] = 64 * (m % 32) + n is
// exact in fp16; the host prints which (m, n) each 16-bit half of each 32-bit cell holds.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2603_03988_b200/csrc
//        tools/micro/f16d_layout.cu -o tools/micro/f16d_layout
#include <cuda_fp16.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"
#include "tma_host.hpp"

using namespace sortk;

__global__ void k_f16d(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       uint32_t* out, int f16_d) {
  __shared__ __align__(1024) uint8_t sA[128 * 64];
  __shared__ __align__(1024) uint8_t sB[64 * 64];
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
    mbar_arrive_expect_tx(&bar, 128 * 64 + 64 * 64);
    tma_load_2d(sA, &tmA, &bar, 0, 0);
    tma_load_2d(sB, &tmB, &bar, 0, 0);
    mbar_wait(&bar, 0);
    tc_fence_after();
    uint32_t idesc = umma_idesc_bf16(128, 64) & ~((7u << 7) | (7u << 10));  // A, B fp16
    if (f16_d) idesc &= ~(3u << 4);                                          // D fp16
    for (int k = 0; k < 2; ++k)
      mma_bf16_ss(tmem, umma_sdesc_kmajor(smem_u32(sA) + k * 32, 64), umma_sdesc_kmajor(smem_u32(sB) + k * 32, 64),
                  idesc, k > 0 ? 1u : 0u);
    mma_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  tc_fence_after();
  uint32_t r[32];
  tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16), r);
  tmem_ld_wait();
  for (int i = 0; i < 32; ++i) out[(warp * 32 + lane) * 32 + i] = r[i];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

int main() {
  std::vector<__half> A(128 * 32, __float2half(0.f)), B(64 * 32, __float2half(0.f));
  for (int m = 0; m < 128; ++m) {
    A[m * 32 + 0] = __float2half(64.f * (m % 32));
    A[m * 32 + 1] = __float2half(1.f);
  }
  for (int n = 0; n < 64; ++n) {
    B[n * 32 + 0] = __float2half(1.f);
    B[n * 32 + 1] = __float2half(static_cast<float>(n));
  }
  __half *dA, *dB;
  uint32_t* dO;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dO, 128 * 32 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const CUtensorMap tA = make_tmap_2d(dA, 128, 32, 32, 128, 32, 64);
  const CUtensorMap tB = make_tmap_2d(dB, 64, 32, 32, 64, 32, 64);
  std::vector<uint32_t> o(128 * 32);
  for (int f16 = 0; f16 < 2; ++f16) {
    k_f16d<<<1, 128>>>(tA, tB, dO, f16);
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      std::printf("f16_d=%d: %s\n", f16, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
    std::printf("== D %s: rows 0, 1, 33 (cells 0..7, and 16..17)\n", f16 ? "fp16" : "fp32");
    for (int row : {0, 1, 33}) {
      std::printf("row %3d:", row);
      for (int c : {0, 1, 2, 3, 4, 5, 6, 7, 16, 17, 31}) {
        const uint32_t v = o[row * 32 + c];
        if (f16) {
          __half lo, hi;
          const uint16_t l16 = v & 0xffff, h16 = v >> 16;
          memcpy(&lo, &l16, 2);
          memcpy(&hi, &h16, 2);
          std::printf(" [%d](%g,%g)", c, __half2float(lo), __half2float(hi));
        } else {
          float f;
          memcpy(&f, &v, 4);
          std::printf(" [%d]%g", c, f);
        }
      }
      std::printf("\n");
    }
  }
  return 0;
}
