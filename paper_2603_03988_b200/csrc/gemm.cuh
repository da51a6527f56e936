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
//   warp 0       TMA producer   (weight slice once, then per tile: the epilogue's per-row side
//                                data (row statistics, RoPE rows) and the A tiles 128x64, SW128)
//   warp 1       MMA issuer     (one thread; 4 x tcgen05.mma K=16 per stage)
//   warp 2       TMEM allocator (2 accumulator stages x 256 columns)
//   warps 4..11  epilogue       (thread <-> accumulator row; TMEM lane quarter = warp % 4;
//                                warps 4-7 take the first half of the tile's column chunks,
//                                warps 8-11 the second half)
// The weight slice of a CTA stays resident in shared memory (weight-stationary).
#pragma once

#include <type_traits>

#include "ptx.cuh"

namespace sortk {

// Grouped mode (MoE experts): an epilogue declaring `kGrouped = true` carries
//   const int32_t* tile_group;  // group (expert) of every listed 128-row tile
//   const int32_t* tile_mblk;   // its m-block (first row / 128)
//   const int32_t* num_tiles;   // number of listed tiles (device-side, written by the router)
//   int group_n;                // weight rows per group in the stacked B operand
// The A rows of each group are contiguous and padded to 128, so an m-block belongs to one
// group; B stacks the groups' [N, K] weights. A CTA keeps two weight slices resident and
// reloads one whenever its next m-block belongs to a new group (the next group's slice
// streams in while the MMA still works on the current one).
template <class E, class = void>
struct is_grouped : std::false_type {};
template <class E>
struct is_grouped<E, std::void_t<decltype(E::kGrouped)>> : std::bool_constant<E::kGrouped> {};

constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;
constexpr int kGemmEpiWarps = 8;
constexpr int kGemmThreads = 128 + 32 * kGemmEpiWarps;
constexpr uint32_t kGemmABytes = kGemmBM * kGemmBK * 2;  // 16 KB per A stage
constexpr uint32_t kGemmEpiSmem = 2048;                  // per-kernel epilogue scratch (QKNorm gains)
constexpr uint32_t kGemmSmemMax = 227 * 1024;

// Per-row side data streamed by the TMA producer next to each A tile (double-buffered):
//   bit 0  row statistics: float4 per row (sum-of-squares partials)     128 x 16 B
//   bit 1  RoPE rows: kRopeFloats fp16 per row (cos/sin pairs of the row's position, fp64 on
//          the host -> fp16: 2^-11 relative, finer than the bf16 Q/K they rotate)
// Epilogues declare `kSide` and `kRopeFloats`; side_bytes() is one buffer.
constexpr uint32_t kSideStatBytes = 128 * 16;
__host__ __device__ constexpr uint32_t side_bytes(int side, int rope_floats) {
  return side == 0 ? 0u
                   : (((side & 1) ? kSideStatBytes : 0u) + ((side & 2) ? 128u * rope_floats * 2u : 0u) +
                      1023u) / 1024u * 1024u;
}

// Shared-memory plan of one weight-stationary GEMM launch.
struct GemmPlan {
  int BN, num_k, a_stages;
  uint32_t b_bytes, smem_bytes;
};

__host__ __device__ inline GemmPlan gemm_plan(int K, int BN, uint32_t side_buf_bytes = 0, int ncta = 1,
                                              int b_bufs = 1) {
  GemmPlan p;
  p.BN = BN;
  p.num_k = (K + kGemmBK - 1) / kGemmBK;
  p.b_bytes = static_cast<uint32_t>(BN / ncta) * kGemmBK * 2 * p.num_k;  // this CTA's weight share
  const uint32_t fixed = 1024 + b_bufs * p.b_bytes + kGemmEpiSmem + 2 * side_buf_bytes + 256;
  int st = fixed < kGemmSmemMax ? static_cast<int>((kGemmSmemMax - fixed) / kGemmABytes) : 0;
  p.a_stages = st > 8 ? 8 : st;
  p.smem_bytes = fixed + p.a_stages * kGemmABytes;
  return p;
}

// Weight-stationary persistent GEMM. CTA c owns the BN-wide weight slice nb = c % num_n
// (loaded into smem once by TMA) and streams the A tiles of m-blocks c / num_n,
// c / num_n + G / num_n, ... through an a_stages-deep TMA ring. Only A moves per tile,
// which keeps the L2 -> SM traffic at ~32 B/clk/SM for K = 256 instead of re-reading
// the weights for every 128-row tile.
// kPair: the CTA-pair form (tcgen05 cta_group::2): a cluster of 2 CTAs owns the slice, each
// CTA holding half of its weight rows (BN/2 x K) and streaming its own 128 rows of every
// 256-row m-block; the leader issues M = 256 MMAs.
template <class Epi, bool kPair = false>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_bf16(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmR,
                int M, int N, int K, int BN, int a_stages, Epi epi) {
  constexpr int kNcta = kPair ? 2 : 1;
  constexpr bool kGroup = is_grouped<Epi>::value;
  static_assert(!(kGroup && kPair), "grouped GEMM runs as single CTAs");
  constexpr int kSide = Epi::kSide;
  constexpr uint32_t kSideBuf = side_bytes(Epi::kSide, Epi::kRopeFloats);
  constexpr int kRopeBoxFloats = Epi::kRopeFloats < 64 ? Epi::kRopeFloats : 64;  // fp16 per box row
  constexpr int kRopeBoxes = Epi::kRopeFloats / (kRopeBoxFloats > 0 ? kRopeBoxFloats : 1);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1k(smem_raw);
  const int num_k = (K + kGemmBK - 1) / kGemmBK;
  const uint32_t b_box = static_cast<uint32_t>(BN / kNcta) * kGemmBK * 2;
  const uint32_t b_slice = b_box * num_k;  // one resident weight slice
  uint8_t* sB = smem;
  uint8_t* sA = sB + b_slice * (kGroup ? 2 : 1);
  uint8_t* sEpi = sA + a_stages * kGemmABytes;
  uint8_t* sSide = sEpi + kGemmEpiSmem;  // 2 x kSideBuf (1024-aligned)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sSide + 2 * kSideBuf);
  uint64_t* full = bars;             // [a_stages <= 8]
  uint64_t* empty = bars + 8;        // [8]
  uint64_t* tfull = bars + 16;       // [2]
  uint64_t* tempty = bars + 18;      // [2]
  uint64_t* b_full = bars + 20;
  uint64_t* side_full = bars + 21;   // [2]
  uint64_t* side_empty = bars + 23;  // [2]
  uint64_t* gb_full = bars + 25;   // [2] grouped: weight slice slot s loaded
  uint64_t* gb_empty = bars + 27;  // [2] grouped: weight slice slot s released by the MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 29);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = kPair ? cluster_rank() : 0u;
  const int unit = kPair ? static_cast<int>(blockIdx.x) / 2 : static_cast<int>(blockIdx.x);
  const int units = kPair ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);
  int num_m = (M + kGemmBM * kNcta - 1) / (kGemmBM * kNcta);  // m-blocks of 128 (256 as a pair)
  if constexpr (kGroup) num_m = *epi.num_tiles;
  const int num_n = N / BN;
  const int nb = unit % num_n;
  const int m_first = unit / num_n;
  const int m_step = units / num_n;
  auto mrow0 = [&](int mb) {
    if constexpr (kGroup) {
      return epi.tile_mblk[mb] * kGemmBM;  // grouped: the listed tile's first row
    } else {
      return (mb * kNcta + static_cast<int>(rank)) * kGemmBM;
    }
  };
  // residual epilogues keep one sum-of-squares slot per (n-slice, half): at most 4
  if (num_n > 2 && threadIdx.x == 0 && blockIdx.x == 0 && Epi::kMaxParts < num_n * 2) __trap();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if constexpr (kSide & 1) tma_prefetch_desc(&tmS);
    if constexpr (kSide & 2) tma_prefetch_desc(&tmR);
    for (int s = 0; s < a_stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * kGemmEpiWarps * kNcta);
    }
    mbar_init(b_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&side_full[i], 1);
      mbar_init(&side_empty[i], 32 * kGemmEpiWarps);
      mbar_init(&gb_full[i], 1);
      mbar_init(&gb_empty[i], 1);
    }
    mbar_fence_init();
  }
  if (warp == 2) {
    if constexpr (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(512u)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc(tmem_slot, 512);
    }
  }
  epi.prologue(sEpi, threadIdx.x, kGemmThreads);
  tc_fence_before();
  if constexpr (kPair) {
    cluster_sync_all();
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMA into this CTA's smem completing on the (leader's, as a pair) barrier
  auto load_ab = [&](void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
    if constexpr (kPair) {
      tma_load_2d_2sm(dst, m, map_to_rank(smem_u32(bar), 0), c0, c1);
    } else {
      tma_load_2d(dst, m, bar, c0, c1);
    }
  };

  if (warp == 0) {
    if (lane == 0) {
      if constexpr (!kGroup) {
        if (rank == 0) mbar_arrive_expect_tx(b_full, b_box * num_k * kNcta);
        for (int kb = 0; kb < num_k; ++kb)
          load_ab(sB + kb * b_box, &tmB, b_full, kb * kGemmBK, nb * BN + static_cast<int>(rank) * (BN / kNcta));
      }
      int s = 0;
      uint32_t ph = 0;
      int t = 0;
      int cur_g = -1, n_loads = 0;
      for (int mb = m_first; mb < num_m; mb += m_step, ++t) {
        if constexpr (kGroup) {  // this m-block's group weights: reload on a group change
          const int g = epi.tile_group[mb];
          if (g != cur_g) {
            const int slot = n_loads & 1;
            if (n_loads >= 2) mbar_wait_sleep(&gb_empty[slot], ((n_loads >> 1) - 1) & 1);
            mbar_arrive_expect_tx(&gb_full[slot], b_slice);
            for (int kb = 0; kb < num_k; ++kb)
              tma_load_2d(sB + slot * b_slice + kb * b_box, &tmB, &gb_full[slot], kb * kGemmBK,
                          g * epi.group_n + nb * BN);
            cur_g = g;
            ++n_loads;
          }
        }
        if constexpr (kSide != 0) {  // this tile's per-row side data
          const int sb = t & 1;
          uint8_t* dst = sSide + sb * kSideBuf;
          mbar_wait_sleep(&side_empty[sb], ((t >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&side_full[sb], ((kSide & 1) ? kSideStatBytes : 0u) +
                                                    ((kSide & 2) ? 128u * Epi::kRopeFloats * 2u : 0u));
          if constexpr (kSide & 1) tma_load_2d(dst, &tmS, &side_full[sb], 0, mrow0(mb));
          if constexpr (kSide & 2) {
#pragma unroll
            for (int bx = 0; bx < kRopeBoxes; ++bx)
              tma_load_2d(dst + ((kSide & 1) ? kSideStatBytes : 0u) + bx * 128 * kRopeBoxFloats * 2, &tmR,
                          &side_full[sb], bx * kRopeBoxFloats, mrow0(mb));
          }
        }
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait_sleep(&empty[s], ph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[s], kGemmABytes * kNcta);
          load_ab(sA + s * kGemmABytes, &tmA, &full[s], kb * kGemmBK, mrow0(mb));
          if (++s == a_stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      const uint32_t idesc = umma_idesc_bf16(kGemmBM * kNcta, BN);
      uint32_t b0 = smem_u32(sB);
      if constexpr (!kGroup) mbar_wait_sleep(b_full, 0);
      int s = 0;
      uint32_t ph = 0;
      int t = 0;
      int cur_g = -1, n_loads = 0;
      for (int mb = m_first; mb < num_m; mb += m_step, ++t) {
        if constexpr (kGroup) {
          const int g = epi.tile_group[mb];
          if (g != cur_g) {
            if (n_loads > 0) mma_commit(&gb_empty[(n_loads - 1) & 1]);  // previous slice free once its MMAs retire
            const int slot = n_loads & 1;
            mbar_wait_sleep(&gb_full[slot], (n_loads >> 1) & 1);
            b0 = smem_u32(sB + slot * b_slice);
            cur_g = g;
            ++n_loads;
          }
        }
        const int acc = t & 1;
        const uint32_t acc_ph = (t >> 1) & 1;
        mbar_wait_sleep(&tempty[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * 256;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait_sleep(&full[s], ph);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * kGemmABytes);
          const uint32_t bk = b0 + kb * b_box;
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k) {
            if constexpr (kPair) {
              mma2_bf16_ss(d, umma_sdesc_kmajor(a0 + k * 32, 128), umma_sdesc_kmajor(bk + k * 32, 128), idesc,
                           (kb | k) != 0 ? 1u : 0u);
            } else {
              mma_bf16_ss(d, umma_sdesc_kmajor(a0 + k * 32, 128), umma_sdesc_kmajor(bk + k * 32, 128),
                          idesc, (kb | k) != 0 ? 1u : 0u);
            }
          }
          if constexpr (kPair) {
            mma2_commit_both(&empty[s]);
          } else {
            mma_commit(&empty[s]);
          }
          if (++s == a_stages) {
            s = 0;
            ph ^= 1;
          }
        }
        if constexpr (kPair) {
          mma2_commit_both(&tfull[acc]);
        } else {
          mma_commit(&tfull[acc]);
        }
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
    for (int mb = m_first; mb < num_m; mb += m_step, ++t) {
      const int acc = t & 1;
      const uint32_t acc_ph = (t >> 1) & 1;
      const int row = mrow0(mb) + q * 32 + lane;
      const uint32_t tbase = tmem + acc * 256 + (static_cast<uint32_t>(q * 32) << 16);
      uint8_t* side = sSide + acc * kSideBuf;
      auto wait = [&]() {
        if constexpr (kSide != 0) mbar_wait(&side_full[acc], acc_ph);
        mbar_wait(&tfull[acc], acc_ph);
        tc_fence_after();
      };
      epi.run(sEpi, side, wait, tbase, row, nb * BN, c_begin * Epi::kChunk, c_end * Epi::kChunk,
              row < M, nb * 2 + half, num_n * 2);
      tc_fence_before();
      if constexpr (kPair) {
        mbar_arrive_cluster(map_to_rank(smem_u32(&tempty[acc]), 0));
      } else {
        mbar_arrive(&tempty[acc]);
      }
      if constexpr (kSide != 0) mbar_arrive(&side_empty[acc]);
    }
  }
  tc_fence_before();
  if constexpr (kPair) {
    cluster_sync_all();
  } else {
    __syncthreads();
  }
  if (warp == 2) {
    tc_fence_after();
    if constexpr (kPair) {
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
    } else {
      tmem_dealloc(tmem, 512);
    }
  }
}

// Loads kChunk accumulator columns [c, c+kChunk) of this thread's row as fp32.
template <int kChunk>
__device__ __forceinline__ void tmem_row_chunk(uint32_t taddr, float (&v)[kChunk]) {
  if constexpr (kChunk == 8) {
    uint32_t r[8];
    tmem_ld_32x32b_x8(taddr, r);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
  } else if constexpr (kChunk == 16) {
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
    static_assert(kChunk == 64, "chunk must be 8, 16, 32 or 64");
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

// Grid of the weight-stationary GEMM: a multiple of the n-slice count (CTA c -> slice
// c % num_n), at most one CTA per SM and no more than the tiles available.
inline int gemm_grid(int num_m, int num_n, int sms) {
  int per_slice = sms / num_n;
  if (per_slice < 1) per_slice = 1;
  if (per_slice > num_m) per_slice = num_m;
  return per_slice * num_n;
}

}  // namespace sortk
