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

template <class Epi>
__global__ void __launch_bounds__(kGsThreads, 1)
    k_gemm_stream(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                  int K, Epi epi) {
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
  const int num_k = (K + kGsBK - 1) / kGsBK;
  const int n_tiles = num_m * num_n;

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
        const int mb = t / num_n, nb = t - mb * num_n;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait_sleep(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], kGsABytes + kGsBBytes);
          tma_load_2d(sA + s * kGsABytes, &tmA, &full[s], kb * kGsBK, mb * kGsBM);
          tma_load_2d(sB + s * kGsBBytes, &tmB, &full[s], kb * kGsBK, nb * kGsBN);
          if (++s == kGsStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(kGsBM, kGsBN);
      int s = 0, i = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
        const int acc = i & 1;
        mbar_wait_sleep(&tempty[acc], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * 256;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * kGsABytes), b0 = smem_u32(sB + s * kGsBBytes);
#pragma unroll
          for (int k = 0; k < kGsBK / 16; ++k)
            mma_bf16_ss(d, umma_sdesc_kmajor(a0 + k * 32, 128), umma_sdesc_kmajor(b0 + k * 32, 128), idesc,
                        (kb | k) != 0 ? 1u : 0u);
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
      const int mb = t / num_n, nb = t - mb * num_n;
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
        if (row < M) epi.apply(row, col, v);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
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
