// Standalone GPU check of the CTA-pair (tcgen05 cta_group::2) mechanics the block tail would
// use: cluster of 2 CTAs, TMEM allocated by both, A split by rows (128 per CTA), B split by
// N (N/2 rows per CTA), both CTAs' TMA completing on the leader's mbarrier, one MMA issuer in
// the leader, commit multicast to both CTAs, each CTA draining its own 128 TMEM lanes.
// C[256, N] = A[256, K] . B[N, K]^T for K = 64 * KB, compared with a CPU fp32 reference.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

#include "../../paper_2603_03988_b200/csrc/ptx.cuh"
#include "../../paper_2603_03988_b200/csrc/tma_host.hpp"

using namespace sortk;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}

template <int KB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_umma2(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, float* C, int N) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1k(smem_raw);
  const uint32_t rank = cluster_rank();
  const int half_n = N / 2;
  uint8_t* sA = smem;                         // KB x [128 rows x 128 B]
  uint8_t* sB = smem + KB * 16384;            // KB x [N/2 rows x 128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + KB * half_n * 128);
  uint64_t* full = bars;
  uint64_t* done = bars + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(full, 1);
    mbar_init(done, 1);
    mbar_fence_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(256u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t full_leader = map_to_rank(smem_u32(full), 0);
  if (threadIdx.x == 0) {
    if (rank == 0) mbar_arrive_expect_tx(full, 2u * KB * (16384u + half_n * 128u));
    for (int kb = 0; kb < KB; ++kb) {
      tma_load_2d_2sm(sA + kb * 16384, &tA, full_leader, kb * 64, rank * 128);
      tma_load_2d_2sm(sB + kb * half_n * 128, &tB, full_leader, kb * 64, rank * half_n);
    }
  }
  if (rank == 0 && threadIdx.x == 32) {
    mbar_wait(full, 0);
    tc_fence_after();
    const uint32_t idesc = umma_idesc_bf16(256, N);
    for (int kb = 0; kb < KB; ++kb)
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = umma_sdesc_kmajor(smem_u32(sA + kb * 16384) + k * 32, 128);
        const uint64_t bd = umma_sdesc_kmajor(smem_u32(sB + kb * half_n * 128) + k * 32, 128);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"((kb | k) != 0 ? 1u : 0u)
            : "memory");
      }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(done)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
  }
  mbar_wait(done, 0);
  tc_fence_after();
  const int row = rank * 128 + warp * 32 + lane;
  for (int c = 0; c < N; c += 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) C[static_cast<size_t>(row) * N + c + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u) : "memory");
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

template <int KB>
static int run(int N) {
  const int M = 256, K = 64 * KB;
  std::vector<__nv_bfloat16> hA((size_t)M * K), hB((size_t)N * K);
  std::vector<float> fA(hA.size()), fB(hB.size());
  srand(N + K);
  for (size_t i = 0; i < hA.size(); ++i) { float x = bf((rand() % 2001 - 1000) / 1000.f); fA[i] = x; hA[i] = __float2bfloat16(x); }
  for (size_t i = 0; i < hB.size(); ++i) { float x = bf((rand() % 2001 - 1000) / 1000.f); fB[i] = x; hB[i] = __float2bfloat16(x); }
  __nv_bfloat16 *dA, *dB; float* dC;
  cudaMalloc(&dA, hA.size() * 2); cudaMalloc(&dB, hB.size() * 2); cudaMalloc(&dC, (size_t)M * N * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, (size_t)M * N * 4);
  CUtensorMap tA = make_tmap_2d(dA, M, K, K, 128, 64, 128);
  CUtensorMap tB = make_tmap_2d(dB, N, K, K, N / 2, 64, 128);
  const size_t smem = 1024 + KB * 16384 + KB * (N / 2) * 128 + 64;
  cudaFuncSetAttribute(k_umma2<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_umma2<KB><<<2, 128, smem>>>(tA, tB, dC, N);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("N=%d K=%d: CUDA error %s\n", N, K, cudaGetErrorString(e)); return 1; }
  std::vector<float> hC((size_t)M * N);
  cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)fA[(size_t)i * K + k] * fB[(size_t)j * K + k];
      maxerr = std::fmax(maxerr, std::fabs(ref - hC[(size_t)i * N + j]));
    }
  printf("2-CTA umma M=256 N=%d K=%d: max abs err %.3g %s\n", N, K, maxerr, maxerr < 1e-2 ? "OK" : "FAIL");
  cudaFree(dA); cudaFree(dB); cudaFree(dC);
  return maxerr < 1e-2 ? 0 : 1;
}

int main() {
  int bad = 0;
  bad += run<1>(256);
  bad += run<4>(256);
  bad += run<4>(128);
  return bad;
}
