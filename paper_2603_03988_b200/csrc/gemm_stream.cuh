// SPDX-License-Identifier: Apache-2.0
// Streaming tcgen05 GEMM for widths whose weights do not fit in shared memory (SORT-large,
// d = 1024, m = 2560, and the training path's long-K gradient products):
//
//   C[M, N] = A[M, K] * B[N, K]^T   (A, B bf16 K-major in HBM; fp32 accumulation in TMEM)
//
// Both operands stream through a kGsStages-deep TMA ring (128 x 64 A box + 256 x 64 B box,
// 128-byte swizzle), so unlike the weight-stationary engine (gemm.cuh) K is unbounded. Tiles
// are 128 x 256 (one tcgen05.mma M = 128, N = 256 per K = 16 step), ordered n-fastest so the
// ~148 concurrent CTAs share a few A row blocks through L2 while the whole weight matrix stays
// L2-resident (<= 10 MB at SORT-large).
//
// Roles (384 threads, 1 CTA per SM, persistent over tiles):
//   warp 0       TMA producer
//   warp 1       MMA issuer (one thread)
//   warp 2       TMEM allocator (2 accumulator stages x 256 columns)
//   warps 4..11  epilogue: thread <-> accumulator row (TMEM lane quarter = warp % 4); warps
//                4-7 take columns [0, 128) of the tile, warps 8-11 columns [128, 256). The
//                accumulator of tile t drains while the MMAs of tile t + 1 run.
// The epilogue is a functor Epi with `kChunk` (32 or 64 columns per call) and
//   __device__ void apply(int row, int col, const float (&v)[kChunk]) const;
// called for rows < M and column chunks starting below N (N a multiple of kChunk).
#pragma once

#include "gemm.cuh"

namespace sortk {

constexpr int kGsBM = 128;
constexpr int kGsBN = 256;
constexpr int kGsBK = 64;
constexpr int kGsStages = 4;
constexpr int kGsThreads = 384;
constexpr uint32_t kGsABytes = kGsBM * kGsBK * 2;  // 16 KB
constexpr uint32_t kGsBBytes = kGsBN * kGsBK * 2;  // 32 KB
constexpr uint32_t kGsSmem = 1024 + kGsStages * (kGsABytes + kGsBBytes) + 256;

// epilogues that take the split-K index declare `static constexpr bool kSplit = true`
template <class E, class = void>
struct gs_split_epi : std::false_type {};
template <class E>
struct gs_split_epi<E, std::void_t<decltype(E::kSplit)>> : std::bool_constant<E::kSplit> {};
// epilogues that finish a row once both column halves of its tile are drained declare
// `static constexpr bool kRowEnd = true` and `void row_end(int row) const`, called by the
// half-0 thread of the row after a barrier over the 256 epilogue threads (their global
// writes to the tile's rows are visible to it)
template <class E, class = void>
struct gs_rowend_epi : std::false_type {};
template <class E>
struct gs_rowend_epi<E, std::void_t<decltype(E::kRowEnd)>> : std::bool_constant<E::kRowEnd> {};

// UMMA shared-memory descriptor of an MN-major SW128 operand tile (the canonical layout
// ((8,n),(8,k)):((1,LBO),(8,SBO)) in 16-byte units): 64-element (128-byte) MN atoms of 8-row K
// groups; TMA writes each {64 MN x 64 K} box as 64 rows of 128 bytes, so K groups are 1024 B
// apart (SBO) and consecutive MN atoms (separate boxes) 8 KB apart (LBO).
__device__ __forceinline__ uint64_t umma_sdesc_mnmajor_sw128(uint32_t saddr, uint32_t lbo = 8192u) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(lbo >> 4) << 16;    // LBO: next 128-byte MN atom (one TMA box)
  d |= static_cast<uint64_t>(1024u >> 4) << 32;  // SBO: next 8-row K group
  d |= static_cast<uint64_t>(1u) << 46;          // version (sm_100)
  d |= static_cast<uint64_t>(2u) << 61;          // 128-byte swizzle
  return d;
}

// MN-major TF32 operands only exist in the 128-byte / 32-byte-atom swizzle (layout type 1,
// Swizzle<2,5,2> on byte offsets: 4-row K groups of 128-byte rows, written by TMA with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): K groups are 512 B apart (SBO), MN atoms one box apart.
__device__ __forceinline__ uint64_t umma_sdesc_mnmajor_sw128_32b(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(lbo >> 4) << 16;
  d |= static_cast<uint64_t>(512u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(1u) << 61;  // SWIZZLE_128B_BASE32B
  return d;
}

// kAMN / kBMN: the operand is stored MN-major in HBM ([K, M] / [K, N] row-major, e.g. an
// activation matrix X [rows, in] as the A = X^T of a weight gradient, or a reference weight
// W [in, out] as the B of a forward product) and is loaded as 64 x 64 boxes. k_splits > 1
// splits K over CTAs (the weight-gradient products, K = rows): the epilogue then receives
// the split index and writes a partial that a fixed-order reduction sums (deterministic).
// T = __nv_bfloat16 (kind::f16, K = 64 per stage) or float (kind::tf32: fp32 operands at TF32
// precision, K = 32 per stage -- the fp32 ranking head and tokenizer products).
// a_kwrap > 0: A's K coordinate wraps every a_kwrap k blocks, so A [M, a_kwrap BK] meets a B of
// K = r a_kwrap BK as [A | A | ...] (the ranking head's split-precision weight pieces, GsHead).
// a_req_rows > 0: tmA is a 3D view {K, a_req_rows, requests} of rows strided inside a larger
// activation (the candidate rows of each request); an M block is 128 / a_req_rows requests.
template <class Epi, bool kAMN = false, bool kBMN = false, class T = __nv_bfloat16>
__global__ void __launch_bounds__(kGsThreads, 1)
    k_gemm_stream(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                  int K, int k_splits, Epi epi, int a_kwrap = 0, int a_req_rows = 0) {
  constexpr bool kTf32 = std::is_same_v<T, float>;
  constexpr int BK = 128 / sizeof(T);   // K per stage: one 128-byte swizzle row
  constexpr int MMA_K = 32 / sizeof(T); // K per instruction (32 bytes)
  constexpr int kAtom = 128 / sizeof(T);  // MN elements per 128-byte atom (MN-major boxes)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1k(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = sA + kGsStages * kGsABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kGsStages * kGsBBytes);
  uint64_t* full = bars;                // [kGsStages]
  uint64_t* empty = bars + kGsStages;   // [kGsStages]
  uint64_t* tfull = bars + 2 * kGsStages;  // [2]
  uint64_t* tempty = tfull + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id(), lane = lane_id();
  const int num_m = (M + kGsBM - 1) / kGsBM;
  const int num_n = (N + kGsBN - 1) / kGsBN;
  const int num_k = (K + BK - 1) / BK;
  const int kb_per = (num_k + k_splits - 1) / k_splits;  // k blocks per split
  const int n_tiles = num_m * num_n * k_splits;
  // tile t -> (split, m block, n block), n fastest, then m, then split
  auto decode = [&](int t, int& ks, int& mb, int& nb) {
    ks = t / (num_m * num_n);
    const int r = t - ks * num_m * num_n;
    mb = r / num_n;
    nb = r - mb * num_n;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kGsStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 256);
    }
    mbar_fence_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        int ks, mb, nb;
        decode(t, ks, mb, nb);
        const int kb0 = ks * kb_per, kb1 = min(num_k, kb0 + kb_per);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait_sleep(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], kGsABytes + kGsBBytes);
          uint8_t* a_dst = sA + s * kGsABytes;
          uint8_t* b_dst = sB + s * kGsBBytes;
          constexpr uint32_t kBox = BK * 128;  // one {atom MN x BK} MN-major box
          const int ka = a_kwrap > 0 ? kb % a_kwrap : kb;
          if constexpr (kAMN) {
#pragma unroll
            for (int i = 0; i < kGsBM / kAtom; ++i)
              tma_load_2d(a_dst + i * kBox, &tmA, &full[s], mb * kGsBM + kAtom * i, ka * BK);
          } else if (a_req_rows > 0) {
            tma_load_3d(a_dst, &tmA, &full[s], ka * BK, 0, mb * (kGsBM / a_req_rows));
          } else {
            tma_load_2d(a_dst, &tmA, &full[s], ka * BK, mb * kGsBM);
          }
          if constexpr (kBMN) {
#pragma unroll
            for (int i = 0; i < kGsBN / kAtom; ++i)
              tma_load_2d(b_dst + i * kBox, &tmB, &full[s], nb * kGsBN + kAtom * i, kb * BK);
          } else {
            tma_load_2d(b_dst, &tmB, &full[s], kb * BK, nb * kGsBN);
          }
          if (++s == kGsStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // the last n block of a narrow product (N - (num_n - 1) kGsBN < kGsBN, e.g. the N = 32
      // item-width GEMMs of the pre-training backward) runs MMAs of just its width
      const uint32_t major = (kAMN ? (1u << 15) : 0u) | (kBMN ? (1u << 16) : 0u);
      const int n_last = N - (num_n - 1) * kGsBN;  // a multiple of 32 (epilogue chunk)
      const uint32_t idesc_full = (kTf32 ? umma_idesc_tf32(kGsBM, kGsBN) : umma_idesc_bf16(kGsBM, kGsBN)) | major;
      const uint32_t idesc_last =
          (kTf32 ? umma_idesc_tf32(kGsBM, static_cast<uint32_t>(n_last)) : umma_idesc_bf16(kGsBM, static_cast<uint32_t>(n_last))) |
          major;
      constexpr uint32_t kBox = BK * 128;
      int s = 0, i = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
        int ks, mb, nb;
        decode(t, ks, mb, nb);
        const int kb0 = ks * kb_per, kb1 = min(num_k, kb0 + kb_per);
        const int acc = i & 1;
        const uint32_t idesc = nb == num_n - 1 ? idesc_last : idesc_full;
        mbar_wait_sleep(&tempty[acc], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * 256;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * kGsABytes), b0 = smem_u32(sB + s * kGsBBytes);
#pragma unroll
          for (int k = 0; k < BK / MMA_K; ++k) {
            // K-major: the next K slice is 32 bytes further in every row; MN-major: MMA_K rows
            // (of 128 bytes) further
            const uint64_t da = kAMN ? (kTf32 ? umma_sdesc_mnmajor_sw128_32b(a0 + k * MMA_K * 128, kBox)
                                              : umma_sdesc_mnmajor_sw128(a0 + k * MMA_K * 128, kBox))
                                     : umma_sdesc_kmajor(a0 + k * 32, 128);
            const uint64_t db = kBMN ? (kTf32 ? umma_sdesc_mnmajor_sw128_32b(b0 + k * MMA_K * 128, kBox)
                                              : umma_sdesc_mnmajor_sw128(b0 + k * MMA_K * 128, kBox))
                                     : umma_sdesc_kmajor(b0 + k * 32, 128);
            if constexpr (kTf32) {
              mma_tf32_ss(d, da, db, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            } else {
              mma_bf16_ss(d, da, db, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            }
          }
          mma_commit(&empty[s]);
          if (++s == kGsStages) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    constexpr int kC = Epi::kChunk;
    const int e = warp - 4, q = e & 3, half = e >> 2;
    int i = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      int ks, mb, nb;
      decode(t, ks, mb, nb);
      const bool empty_split = ks * kb_per >= num_k;  // (no k blocks: the accumulator is stale)
      const int acc = i & 1;
      const int row = mb * kGsBM + q * 32 + lane;
      const uint32_t tb = tmem + acc * 256 + (static_cast<uint32_t>(q * 32) << 16);
      mbar_wait_sleep(&tfull[acc], (i >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = half * 128; c < half * 128 + 128; c += kC) {
        const int col = nb * kGsBN + c;
        if (col >= N) break;
        float v[kC];
        tmem_row_chunk<kC>(tb + c, v);
        if (empty_split) {
#pragma unroll
          for (int j = 0; j < kC; ++j) v[j] = 0.f;
        }
        if (row < M) {
          if constexpr (gs_split_epi<Epi>::value) {
            epi.apply(row, col, v, ks);
          } else {
            epi.apply(row, col, v);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if constexpr (gs_rowend_epi<Epi>::value) {
        named_bar_sync(1, 256);
        if (half == 0 && row < M) epi.row_end(row);
        named_bar_sync(1, 256);  // the partials are rewritten by the next tile
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// fp32 C[M, N] = op(A)[M, K] op(B)[K, N] (+ beta C), op = transpose when ta / tb: the small or
// TMA-unfriendly fp32 products of the ranking head and the tokenizer (N = 3 logits, K = 3,
// widths that are not multiples of 32). 32 x 32 output tiles, 32-deep K slices in smem.
__global__ void __launch_bounds__(256) k_gemm_simt(bool ta, bool tb, int M, int N, int K, const float* __restrict__ A,
                                                   int lda, const float* __restrict__ B, int ldb, float* __restrict__ C,
                                                   int ldc, float beta) {
  __shared__ float sa[32][33], sb[32][33];
  const int m0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 4 outputs each
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k0 = 0; k0 < K; k0 += 32) {
    for (int i = ty; i < 32; i += 8) {
      const int m = m0 + i, k = k0 + tx;  // sa[i][tx] = op(A)[m][k]
      sa[i][tx] = (m < M && k < K) ? (ta ? A[static_cast<size_t>(k) * lda + m] : A[static_cast<size_t>(m) * lda + k]) : 0.f;
      const int kk = k0 + i, n = n0 + tx;  // sb[i][tx] = op(B)[kk][n]
      sb[i][tx] = (kk < K && n < N) ? (tb ? B[static_cast<size_t>(n) * ldb + kk] : B[static_cast<size_t>(kk) * ldb + n]) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const float bv = sb[k][tx];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = fmaf(sa[ty + 8 * r][k], bv, acc[r]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int m = m0 + ty + 8 * r, n = n0 + tx;
    if (m < M && n < N) {
      float* c = C + static_cast<size_t>(m) * ldc + n;
      *c = beta != 0.f ? acc[r] + beta * *c : acc[r];
    }
  }
}

// ---------------------------------------------------------------- epilogue functors
// C (bf16 or fp32, row-major, ldc) = acc
template <class T>
struct GsStore {
  static constexpr int kChunk = 32;
  T* C;
  int ldc;
  __device__ void apply(int row, int col, const float (&v)[32]) const {
    T* p = C + static_cast<size_t>(row) * ldc + col;
    if constexpr (std::is_same_v<T, float>) {
#pragma unroll
      for (int i = 0; i < 8; ++i) reinterpret_cast<float4*>(p)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    } else {
      uint32_t w[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) w[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
      stg256(p, *reinterpret_cast<const uint32_t(*)[8]>(w));
      stg256(p + 16, *reinterpret_cast<const uint32_t(*)[8]>(w + 8));
    }
  }
};

// split-K partial: P[split][row][col] = acc (fp32, [splits, M, N]); k_splitk_reduce sums them
struct GsPartialF32 {
  static constexpr int kChunk = 32;
  static constexpr bool kSplit = true;
  float* P;
  int M, N;
  __device__ void apply(int row, int col, const float (&v)[32], int ks) const {
    float4* p = reinterpret_cast<float4*>(P + (static_cast<size_t>(ks) * M + row) * N + col);
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  }
};

// C[M, N] (row pitch ldc, fp32 or bf16) = sum over splits of P (fixed order) + beta C
template <class T>
__global__ void k_splitk_reduce(const float* __restrict__ P, int splits, int M, int N, T* __restrict__ C, int ldc,
                                float beta) {
  const size_t total = static_cast<size_t>(M) * N;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += P[static_cast<size_t>(k) * total + i];
    const size_t r = i / N, c = i - r * N;
    T* dst = C + r * ldc + c;
    if constexpr (std::is_same_v<T, float>) {
      *dst = beta != 0.f ? s + beta * *dst : s;
    } else {
      *dst = __float2bfloat16_rn(beta != 0.f ? s + beta * __bfloat162float(*dst) : s);
    }
  }
}

// fp32 C += acc (the FFN down projection accumulating into the residual stream)
struct GsAccF32 {
  static constexpr int kChunk = 32;
  float* C;
  int ldc;
  __device__ void apply(int row, int col, const float (&v)[32]) const {
    float4* p = reinterpret_cast<float4*>(C + static_cast<size_t>(row) * ldc + col);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 o = p[i];
      p[i] = make_float4(o.x + v[4 * i], o.y + v[4 * i + 1], o.z + v[4 * i + 2], o.w + v[4 * i + 3]);
    }
  }
};

// fp32 out[row] = x[src(row)] + acc: the attention residual on the pruned stream P(x, L_out)
// (SPEC.md:375), src(row) = (row / R) * Rsrc + map[row % R] (map == nullptr: row).
struct GsResidF32 {
  static constexpr int kChunk = 32;
  const float* x;
  const int32_t* map;
  int R, Rsrc, d;
  float* out;
  __device__ void apply(int row, int col, const float (&v)[32]) const {
    const int b = row / R, r = row - b * R;
    const size_t src = map ? static_cast<size_t>(b) * Rsrc + map[r] : static_cast<size_t>(row);
    const float4* xs = reinterpret_cast<const float4*>(x + src * d + col);
    float4* p = reinterpret_cast<float4*>(out + static_cast<size_t>(row) * d + col);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 o = xs[i];
      p[i] = make_float4(o.x + v[4 * i], o.y + v[4 * i + 1], o.z + v[4 * i + 2], o.w + v[4 * i + 3]);
    }
  }
};

// SwishGLU on [gate_32 | up_32]-interleaved weight rows: each 64-column
// chunk holds gate and up of 32 hidden units; z[row, j] = bf16(swish(g_j) * u_j), [M, m].
struct GsSwiGLU {
  static constexpr int kChunk = 64;
  __nv_bfloat16* z;
  int m;
  __device__ void apply(int row, int col, const float (&v)[64]) const {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float g0 = v[2 * i], g1 = v[2 * i + 1], u0 = v[32 + 2 * i], u1 = v[32 + 2 * i + 1];
      w[i] = pack_bf16x2(g0 / (1.f + __expf(-g0)) * u0, g1 / (1.f + __expf(-g1)) * u1);
    }
    __nv_bfloat16* p = z + static_cast<size_t>(row) * m + (col >> 1);
    stg256(p, *reinterpret_cast<const uint32_t(*)[8]>(w));
    stg256(p + 16, *reinterpret_cast<const uint32_t(*)[8]>(w + 8));
  }
};

// Q/K/V/G preparation on the concatenated projections (attention.cpp:93-127), one 64-wide
// head per chunk (head dim 64): columns [0, d) are Q (or K): per-head RMSNorm with its gain
// row (attention.cpp:111-114), interleaved RoPE at the row's original position
// (rope.hpp:27-38, cos/sin from the fp64-built table) -> bf16 head-major [B*H, R, 64];
// columns [d, 2d) are G (sigmoid -> bf16 [rows, d]) or V (bf16 head-major).
struct GsQKVG {
  static constexpr int kChunk = 64;
  int d, H, R;
  const int32_t* pos;      // [R] original positions of the rows
  const float2* rope;      // [positions, 32] (cos, sin)
  const float* gain;       // [H, 64]
  __nv_bfloat16* lo_out;   // Q or K, head-major
  __nv_bfloat16* hi_out;   // G row-major [rows, d] (hi_gate) or V head-major
  bool hi_gate;
  __device__ void apply(int row, int col, const float (&v)[64]) const {
    const int b = row / R, r = row - b * R;
    uint32_t w[32];
    if (col < d) {
      const int h = col >> 6;
      float ss = 0.f;
#pragma unroll
      for (int i = 0; i < 64; ++i) ss = fmaf(v[i], v[i], ss);
      const float inv = rsqrtf(ss * (1.f / 64.f) + 1e-6f);
      const float* g = gain + h * 64;
      const float4* cs4 = reinterpret_cast<const float4*>(rope + static_cast<size_t>(pos[r]) * 32);
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float4 cs = cs4[j >> 1];  // pairs j, j + 1
        const float2 gg0 = *reinterpret_cast<const float2*>(g + 2 * j);
        const float2 gg1 = *reinterpret_cast<const float2*>(g + 2 * j + 2);
        const float a0 = v[2 * j] * inv * gg0.x, a1 = v[2 * j + 1] * inv * gg0.y;
        const float b0 = v[2 * j + 2] * inv * gg1.x, b1 = v[2 * j + 3] * inv * gg1.y;
        w[j] = pack_bf16x2(cs.x * a0 - cs.y * a1, cs.y * a0 + cs.x * a1);
        w[j + 1] = pack_bf16x2(cs.z * b0 - cs.w * b1, cs.w * b0 + cs.z * b1);
      }
      __nv_bfloat16* p = lo_out + ((static_cast<size_t>(b) * H + h) * R + r) * 64;
#pragma unroll
      for (int i = 0; i < 4; ++i) stg256(p + 16 * i, *reinterpret_cast<const uint32_t(*)[8]>(w + 8 * i));
    } else {
      const int c = col - d;
      if (hi_gate) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          w[i] = pack_bf16x2(1.f / (1.f + __expf(-v[2 * i])), 1.f / (1.f + __expf(-v[2 * i + 1])));
        __nv_bfloat16* p = hi_out + static_cast<size_t>(row) * d + c;
#pragma unroll
        for (int i = 0; i < 4; ++i) stg256(p + 16 * i, *reinterpret_cast<const uint32_t(*)[8]>(w + 8 * i));
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) w[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
        __nv_bfloat16* p = hi_out + ((static_cast<size_t>(b) * H + (c >> 6)) * R + r) * 64;
#pragma unroll
        for (int i = 0; i < 4; ++i) stg256(p + 16 * i, *reinterpret_cast<const uint32_t(*)[8]>(w + 8 * i));
      }
    }
  }
};

// W [K, N] fp32 row-major (a reference [in, out] weight) -> rows of a bf16 K-major B operand
// [*, ldk]: out[dest(n)][k] = W[k][n] for k < K (columns K..ldk-1 zero). dest(n) = row0 + n,
// or with il_blk > 0 the SwishGLU interleave (n / il_blk) * 2 il_blk + il_off + n % il_blk.
__global__ void k_transpose_bf16(const float* __restrict__ W, int K, int N, int ldk, int row0, int il_blk,
                                 int il_off, __nv_bfloat16* __restrict__ out) {
  __shared__ float tile[32][33];
  const int k0 = blockIdx.x * 32, n0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: 8 rows per pass
  for (int i = ty; i < 32; i += 8) {
    const int k = k0 + i, n = n0 + tx;
    tile[i][tx] = (k < K && n < N) ? W[static_cast<size_t>(k) * N + n] : 0.f;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int n = n0 + i, k = k0 + tx;
    if (n >= N || k >= ldk) continue;
    const int dest = il_blk > 0 ? (n / il_blk) * 2 * il_blk + il_off + n % il_blk : row0 + n;
    out[static_cast<size_t>(dest) * ldk + k] = __float2bfloat16_rn(tile[tx][i]);
  }
}

}  // namespace sortk
