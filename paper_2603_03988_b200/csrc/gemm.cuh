// SPDX-License-Identifier: Apache-2.0
// Persistent, warp-specialised tcgen05 GEMM with a fused epilogue functor.
//
//   C[M, N] = A[M, K] * B[N, K]^T      (A, B bf16 K-major in HBM, fp32 accumulate in TMEM)
//
// This is the projection engine behind the SORT block stack: the fused
// Q/K/V/G projection (attention.cpp:93-95,125), the output projection with the
// residual add (attention.cpp:131 + SPEC.md:375), and both halves of the
// SwishGLU FFN. What differs between them is only the
// epilogue, a template functor that consumes 128-row x kChunk-column slices of
// the accumulator after tcgen05.ld.
//
// Roles (384 threads, 1 CTA per SM):
//   warp 0       TMA producer   (A tile 128x64, B tile BNx64 per stage, SW128)
//   warp 1       MMA issuer     (one thread; 4 x tcgen05.mma K=16 per stage)
//   warp 2       TMEM allocator (2 accumulator stages x 256 columns)
//   warps 4..11  epilogue       (thread <-> accumulator row; TMEM lane quarter = warp % 4;
//                                warps 4-7 take the first half of the tile's column chunks,
//                                warps 8-11 the second half)
// Tiles are walked m-major with every CTA cycling through all n-tiles, so
// epilogues with different per-section cost (e.g. Q/K vs V) balance across SMs.
#pragma once

#include "ptx.cuh"

namespace sortk {

constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;
constexpr int kGemmStages = 4;
constexpr int kGemmMaxBN = 256;
constexpr int kGemmEpiWarps = 8;
constexpr int kGemmThreads = 128 + 32 * kGemmEpiWarps;
constexpr uint32_t kGemmABytes = kGemmBM * kGemmBK * 2;     // 16 KB
constexpr uint32_t kGemmBBytes = kGemmMaxBN * kGemmBK * 2;  // 32 KB
constexpr uint32_t kGemmEpiSmem = 8192;                     // per-kernel epilogue scratch
constexpr size_t kGemmSmemBytes =
    1024 + kGemmStages * (kGemmABytes + kGemmBBytes) + kGemmEpiSmem + 8 * (2 * kGemmStages + 4) + 16;

// Tile t of the CTA-strided walk -> (m block, n block). Consecutive tiles of one CTA
// advance n fastest so each CTA sees every n-tile (section) in turn.
__device__ __forceinline__ void gemm_tile_coords(int tile, int num_n, int& mb, int& nb) {
  mb = tile / num_n;
  nb = tile - mb * num_n;
}

template <class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_bf16(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                int M, int N, int K, int BN, Epi epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kGemmStages * kGemmABytes;
  uint8_t* sEpi = sB + kGemmStages * kGemmBBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + kGemmEpiSmem);
  uint64_t* empty = full + kGemmStages;
  uint64_t* tfull = empty + kGemmStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int num_m = (M + kGemmBM - 1) / kGemmBM;
  const int num_n = N / BN;
  const int num_tiles = num_m * num_n;
  const int num_k = (K + kGemmBK - 1) / kGemmBK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kGemmStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * kGemmEpiWarps);
    }
    mbar_fence_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  epi.prologue(sEpi, threadIdx.x, kGemmThreads);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t stage_bytes = kGemmABytes + static_cast<uint32_t>(BN) * kGemmBK * 2;
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int mb, nb;
        gemm_tile_coords(tile, num_n, mb, nb);
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], stage_bytes);
          tma_load_2d(sA + s * kGemmABytes, &tmA, &full[s], kb * kGemmBK, mb * kGemmBM);
          tma_load_2d(sB + s * kGemmBBytes, &tmB, &full[s], kb * kGemmBK, nb * BN);
          if (++s == kGemmStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(kGemmBM, BN);
      int s = 0;
      uint32_t ph = 0;
      int t = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++t) {
        const int acc = t & 1;
        const uint32_t acc_ph = (t >> 1) & 1;
        mbar_wait(&tempty[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * 256;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * kGemmABytes);
          const uint32_t b0 = smem_u32(sB + s * kGemmBBytes);
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k) {
            mma_bf16_ss(d, umma_sdesc_kmajor(a0 + k * 32, 128), umma_sdesc_kmajor(b0 + k * 32, 128),
                        idesc, (kb | k) != 0 ? 1u : 0u);
          }
          mma_commit(&empty[s]);
          if (++s == kGemmStages) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    const int e = warp - 4;
    const int q = e & 3;     // == warp % 4: the TMEM lane quarter this warp may access
    const int half = e >> 2;
    const int n_chunks = BN / Epi::kChunk;
    const int split = (n_chunks + 1) >> 1;
    const int c_begin = half ? split : 0, c_end = half ? n_chunks : split;
    int t = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++t) {
      const int acc = t & 1;
      const uint32_t acc_ph = (t >> 1) & 1;
      int mb, nb;
      gemm_tile_coords(tile, num_n, mb, nb);
      const int row = mb * kGemmBM + q * 32 + lane;
      const uint32_t tbase = tmem + acc * 256 + (static_cast<uint32_t>(q * 32) << 16);
      auto wait = [&]() {
        mbar_wait(&tfull[acc], acc_ph);
        tc_fence_after();
      };
      epi.run(sEpi, wait, tbase, row, nb * BN, c_begin * Epi::kChunk, c_end * Epi::kChunk, row < M);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Loads kChunk accumulator columns [c, c+kChunk) of this thread's row as fp32.
template <int kChunk>
__device__ __forceinline__ void tmem_row_chunk(uint32_t taddr, float (&v)[kChunk]) {
  if constexpr (kChunk == 16) {
    uint32_t r[16];
    tmem_ld_32x32b_x16(taddr, r);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
  } else if constexpr (kChunk == 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(taddr, r);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  } else {
    static_assert(kChunk == 64, "chunk must be 16, 32 or 64");
    uint32_t r[32];
    tmem_ld_32x32b_x32(taddr, r);
    uint32_t r2[32];
    tmem_ld_32x32b_x32(taddr + 32, r2);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      v[i] = __uint_as_float(r[i]);
      v[32 + i] = __uint_as_float(r2[i]);
    }
  }
}

// Grid size for the persistent GEMM: at most one CTA per SM, and never a multiple of the
// n-tile count (so the CTA-strided tile walk rotates every CTA through all sections).
inline int gemm_grid(int tiles, int num_n, int sms) {
  int g = tiles < sms ? tiles : sms;
  if (g == sms && num_n > 1 && g % num_n == 0) --g;
  return g > 0 ? g : 1;
}

}  // namespace sortk
