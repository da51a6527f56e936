// SPDX-License-Identifier: Apache-2.0
// DeepSeek-style MoE FFN on the SORT-base residual stream.
//
//   x1 [T, d] bf16 (after the attention residual)
//   -> k_moe_route    fp32 RMSNorm(x1; ffn_norm), router logits z = xf . W_r (fp32),
//                     s = sigmoid(z), top-k of s + bias (ties -> lower index), w = s / sum_sel s,
//                     per-expert token counts
//   -> k_moe_plan     expert segments padded to 128 rows, m-block -> expert list
//   -> k_moe_scatter  bf16 RMSNorm rows into their expert segments (shared expert: every row)
//   -> grouped tcgen05 GEMM [gate | up] with the SwishGLU epilogue -> h [P, m_e]
//   -> grouped tcgen05 GEMM down, epilogue scales by the combine weight -> y [P, d] bf16
//   -> k_moe_combine  x1 + y_shared + sum_j y_j (fixed order) -> bf16 residual + row statistics
// Every row's arithmetic is independent of where the scatter put it, so the output is
// deterministic even though segment order within an expert follows atomic arrival.
#pragma once

#include "block_tail.cuh"
#include "epilogues.cuh"
#include "gemm.cuh"
#include "train.cuh"

namespace sortk {

constexpr int kErrMoeNonFinite = 2;  // err[0] bit; err[1] = 1 + first offending token
constexpr int kMoeMaxExperts = 64;
constexpr int kMoeMaxK = 8;

// ---------------------------------------------------------------------------------- router
// One warp per token (grid-stride), lane owns 8 contiguous columns (d <= 256, d % 8 == 0).
// Router logits: every lane forms its 8-column partial dot for each expert and parks them in a
// per-warp smem tile; lane e (and e + 32) then sums expert e's 32 partials and applies the
// sigmoid. Top-k: k rounds of a warp max over order-preserving integer keys, the lowest lane
// (= lowest expert index) winning ties via a ballot.
__device__ __forceinline__ uint32_t float_key(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void __launch_bounds__(256) k_moe_route(const __nv_bfloat16* __restrict__ x, int T, int d,
                                                   const float* __restrict__ gain, const float* __restrict__ router,
                                                   const float* __restrict__ bias, int E, int k,
                                                   int32_t* __restrict__ sel, float* __restrict__ wgt,
                                                   float* __restrict__ inv_out, int32_t* __restrict__ counts,
                                                   int32_t* __restrict__ err) {
  extern __shared__ float smem_f[];
  float* wr = smem_f;  // router transposed [E][d]
  const int stride = E + 1;  // partial tile row pitch (conflict-free column sums)
  float* part = smem_f + static_cast<size_t>(E) * d + (threadIdx.x >> 5) * 32 * stride;
  __shared__ int hist[kMoeMaxExperts];
  for (int i = threadIdx.x; i < d * E; i += blockDim.x) {
    const int c = i / E, e = i - c * E;
    wr[e * d + c] = router[i];
  }
  for (int i = threadIdx.x; i < E; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int c0 = lane * 8;
  const bool act = c0 < d;
  float g[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) g[i] = act ? gain[c0 + i] : 0.f;
  const bool own0 = lane < E, own1 = lane + 32 < E;
  const float b0 = own0 ? bias[lane] : 0.f, b1 = own1 ? bias[lane + 32] : 0.f;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < T; t += warps) {
    float v[8];
    if (act) {
      const int4 raw = *reinterpret_cast<const int4*>(x + static_cast<size_t>(t) * d + c0);
      const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(p2[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = 0.f;
    }
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) ss = fmaf(v[i], v[i], ss);
    const float inv = rsqrtf(warp_sum(ss) / static_cast<float>(d) + 1e-6f);  // norm.hpp:23-24
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] *= inv * g[i];
    for (int e = 0; e < E; ++e) {
      float z = 0.f;
      if (act) {
        const float4 a = *reinterpret_cast<const float4*>(wr + e * d + c0);
        const float4 b = *reinterpret_cast<const float4*>(wr + e * d + c0 + 4);
        z = v[0] * a.x + v[1] * a.y + v[2] * a.z + v[3] * a.w + v[4] * b.x + v[5] * b.y + v[6] * b.z + v[7] * b.w;
      }
      part[lane * stride + e] = z;
    }
    __syncwarp();
    float z0 = 0.f, z1 = 0.f;
    if (own0)
#pragma unroll 8
      for (int l = 0; l < 32; ++l) z0 += part[l * stride + lane];
    if (own1)
#pragma unroll 8
      for (int l = 0; l < 32; ++l) z1 += part[l * stride + lane + 32];
    __syncwarp();
    // sigmoid gate scores and biased selection keys; a non-finite score
    // is flagged and never selected
    const float s0 = 1.f / (1.f + expf(-z0)), s1 = 1.f / (1.f + expf(-z1));
    const float k0f = s0 + b0, k1f = s1 + b1;
    bool bad = (own0 && !isfinite(k0f)) || (own1 && !isfinite(k1f));
    uint32_t key0 = own0 && isfinite(k0f) ? float_key(k0f) : 0u;
    uint32_t key1 = own1 && isfinite(k1f) ? float_key(k1f) : 0u;
    if (__any_sync(0xffffffffu, bad) && lane == 0) {
      atomicOr(err, kErrMoeNonFinite);
      atomicCAS(err + 1, 0, t + 1);
    }
    int my_e[kMoeMaxK];
    float my_s[kMoeMaxK];
    float tot = 0.f;
#pragma unroll
    for (int j = 0; j < kMoeMaxK; ++j) {
      if (j >= k) break;
      const uint32_t best = __reduce_max_sync(0xffffffffu, key0 > key1 ? key0 : key1);
      const uint32_t lo = __ballot_sync(0xffffffffu, key0 == best);   // experts 0..31 first
      const uint32_t hi = __ballot_sync(0xffffffffu, key1 == best);
      const int e = lo ? __ffs(lo) - 1 : (hi ? 32 + __ffs(hi) - 1 : 0);
      const float sw = __shfl_sync(0xffffffffu, e < 32 ? s0 : s1, e & 31);
      if (lane == (e & 31)) {
        if (e < 32) key0 = 0u;
        else key1 = 0u;
      }
      my_e[j] = e;
      my_s[j] = (lo | hi) ? sw : 1.f;
      tot += my_s[j];
    }
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < kMoeMaxK; ++j) {
        if (j >= k) break;
        sel[static_cast<size_t>(t) * k + j] = my_e[j];
        wgt[static_cast<size_t>(t) * k + j] = my_s[j] / tot;
        atomicAdd(&hist[my_e[j]], 1);
      }
      inv_out[t] = inv;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x)
    if (hist[i]) atomicAdd(&counts[i], hist[i]);
}

// Small-E router (E <= 8): the lane's 8 x 8 router slice lives in registers and the 8 expert
// partials are reduce-scattered across the warp with 9 shuffles; afterwards lane 4e holds
// expert e's logit. Same arithmetic contract as k_moe_route.
__global__ void __launch_bounds__(256) k_moe_route8(const __nv_bfloat16* __restrict__ x, int T, int d,
                                                    const float* __restrict__ gain,
                                                    const float* __restrict__ router, const float* __restrict__ bias,
                                                    int E, int k, int32_t* __restrict__ sel, float* __restrict__ wgt,
                                                    float* __restrict__ inv_out, int32_t* __restrict__ counts,
                                                    int32_t* __restrict__ err) {
  __shared__ int hist[8];
  if (threadIdx.x < 8) hist[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int c0 = lane * 8;
  const bool act = c0 < d;
  float g[8], w[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    g[i] = act ? gain[c0 + i] : 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) w[e][i] = act && e < E ? router[static_cast<size_t>(c0 + i) * E + e] : 0.f;
  }
  const int my_e = lane >> 2;
  const bool owner = (lane & 3) == 0 && my_e < E;
  const float my_b = owner ? bias[my_e] : 0.f;
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  const int warps = gridDim.x * (blockDim.x >> 5);
  int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int4 nxt = make_int4(0, 0, 0, 0);  // software pipeline: the next row's load is in flight
  if (act && t < T) nxt = *reinterpret_cast<const int4*>(x + static_cast<size_t>(t) * d + c0);
  for (; t < T; t += warps) {
    const int4 raw = nxt;
    if (act && t + warps < T) nxt = *reinterpret_cast<const int4*>(x + static_cast<size_t>(t + warps) * d + c0);
    float v[8];
    {
      const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(p2[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
      }
    }
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) ss = fmaf(v[i], v[i], ss);
    const float inv = rsqrtf(warp_sum(ss) / static_cast<float>(d) + 1e-6f);  // norm.hpp:23-24
    float p[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float z = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) z = fmaf(v[i] * inv * g[i], w[e][i], z);
      p[e] = z;
    }
    float q[4], r[2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      q[i] = (b4 ? p[i + 4] : p[i]) + __shfl_xor_sync(0xffffffffu, b4 ? p[i] : p[i + 4], 16);
#pragma unroll
    for (int i = 0; i < 2; ++i)
      r[i] = (b3 ? q[i + 2] : q[i]) + __shfl_xor_sync(0xffffffffu, b3 ? q[i] : q[i + 2], 8);
    float z = (b2 ? r[1] : r[0]) + __shfl_xor_sync(0xffffffffu, b2 ? r[0] : r[1], 4);
    z += __shfl_xor_sync(0xffffffffu, z, 2);
    z += __shfl_xor_sync(0xffffffffu, z, 1);
    const float sc = 1.f / (1.f + expf(-z));  // sigmoid gate
    const float kf = sc + my_b;
    const bool bad = owner && !isfinite(kf);
    uint32_t key = owner && !bad ? float_key(kf) : 0u;
    if (__any_sync(0xffffffffu, bad) && lane == 0) {
      atomicOr(err, kErrMoeNonFinite);
      atomicCAS(err + 1, 0, t + 1);
    }
    int se[kMoeMaxK];
    float sw[kMoeMaxK];
    float tot = 0.f;
#pragma unroll
    for (int j = 0; j < kMoeMaxK; ++j) {
      if (j >= k) break;
      const uint32_t best = __reduce_max_sync(0xffffffffu, key);
      const uint32_t m = __ballot_sync(0xffffffffu, key == best && owner);
      const int wl = m ? __ffs(m) - 1 : 0;  // lowest lane = lowest expert on ties
      sw[j] = m ? __shfl_sync(0xffffffffu, sc, wl) : 1.f;
      se[j] = wl >> 2;
      if (lane == wl) key = 0u;
      tot += sw[j];
    }
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < kMoeMaxK; ++j) {
        if (j >= k) break;
        sel[static_cast<size_t>(t) * k + j] = se[j];
        wgt[static_cast<size_t>(t) * k + j] = sw[j] / tot;
        atomicAdd(&hist[se[j]], 1);
      }
      inv_out[t] = inv;
    }
  }
  __syncthreads();
  if (threadIdx.x < E && hist[threadIdx.x]) atomicAdd(&counts[threadIdx.x], hist[threadIdx.x]);
}

// Routing and scatter in one pass (E <= 8, top-K with K <= 2): a warp routes 32 tokens
// (the k_moe_route8 arithmetic, results parked in lane i for token i), takes their expert-
// segment positions with one warp-aggregated atomic per (slot, expert) on the per-expert
// cursors (which end as the expert loads), then writes each token's normalised bf16 row into
// its K (+ shared) segments, re-reading the row from L2.
// The router columns sit in shared memory as [q][expert quad][lane] float4s (conflict-free
// LDS.128, 8 KB) rather than in 64 registers per lane: 4 CTAs per SM instead of 2 hide the
// per-token shuffle chains (the kernel is latency-bound on them).
// Each warp keeps the rows of its kRouteTok tokens in dynamic shared memory (lane l holds its
// own 16-byte chunk of every row, so no synchronisation is needed) and writes them out from
// there: the scatter never re-reads x (measured: the re-read missed L2, 4.9 % hit rate).
constexpr int kRouteTok = 16;
constexpr int kRouteCtasPerSm = 3;
constexpr size_t kRouteSmem = 8 * kRouteTok * 32 * sizeof(int4);  // 8 warps
template <int K>
__global__ void __launch_bounds__(256, kRouteCtasPerSm) k_moe_route_scatter8(
    const __nv_bfloat16* __restrict__ x, int T, int d, const float* __restrict__ gain,
    const float* __restrict__ router, const float* __restrict__ bias, int E, int shared, int Tcap,
    int32_t* __restrict__ sel, float* __restrict__ wgt, int32_t* __restrict__ cursor,
    __nv_bfloat16* __restrict__ xs, int32_t* __restrict__ tok_of, float* __restrict__ w_of,
    int32_t* __restrict__ slot_pos, int32_t* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int c0 = lane * 8;
  const bool act = c0 < d;
  const int S = K + shared;
  __shared__ float4 sw4[8][2][32];  // router[c0 + q][4 * quad + comp] of lane l at [q][quad][l]
  for (int i = threadIdx.x; i < 32 * 8 * 8; i += blockDim.x) {
    const int l = i >> 6, q = (i >> 3) & 7, e = i & 7;
    const int c = l * 8 + q;
    reinterpret_cast<float*>(&sw4[q][e >> 2][l])[e & 3] = c < d && e < E ? router[static_cast<size_t>(c) * E + e] : 0.f;
  }
  float g[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) g[i] = act ? gain[c0 + i] : 0.f;
  __syncthreads();
  const int my_e = lane >> 2;
  const bool owner = (lane & 3) == 0 && my_e < E;
  const float my_b = owner ? bias[my_e] : 0.f;
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  const int warps = gridDim.x * (blockDim.x >> 5);
  extern __shared__ int4 srow[];  // [warp][kRouteTok][32 lanes]
  int4* myrows = srow + (threadIdx.x >> 5) * kRouteTok * 32 + lane;
  for (int base = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kRouteTok; base < T;
       base += warps * kRouteTok) {
    const int n = min(kRouteTok, T - base);
    int te[K];
    float tw[K], tinv = 0.f;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      te[j] = 0;
      tw[j] = 0.f;
    }
    // software pipeline: token i + 2's row load is in flight while token i is routed
    int4 nx0 = make_int4(0, 0, 0, 0), nx1 = make_int4(0, 0, 0, 0);
    if (act) {
      nx0 = *reinterpret_cast<const int4*>(x + static_cast<size_t>(base) * d + c0);
      if (n > 1) nx1 = *reinterpret_cast<const int4*>(x + static_cast<size_t>(base + 1) * d + c0);
    }
    for (int i = 0; i < n; ++i) {
      const int t = base + i;
      const int4 raw = nx0;
      myrows[i * 32] = raw;
      nx0 = nx1;
      if (act && i + 2 < n) nx1 = *reinterpret_cast<const int4*>(x + static_cast<size_t>(t + 2) * d + c0);
      float v[8];
      {
        const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(p2[q]);
          v[2 * q] = f.x;
          v[2 * q + 1] = f.y;
        }
      }
      float ss = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) ss = fmaf(v[q], v[q], ss);
      const float inv = rsqrtf(warp_sum(ss) / static_cast<float>(d) + 1e-6f);  // norm.hpp:23-24
      float p[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) p[e] = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {  // same per-expert summation order as before (q ascending)
        const float xq = v[q] * inv * g[q];
        const float4 wa = sw4[q][0][lane], wb = sw4[q][1][lane];
        p[0] = fmaf(xq, wa.x, p[0]);
        p[1] = fmaf(xq, wa.y, p[1]);
        p[2] = fmaf(xq, wa.z, p[2]);
        p[3] = fmaf(xq, wa.w, p[3]);
        p[4] = fmaf(xq, wb.x, p[4]);
        p[5] = fmaf(xq, wb.y, p[5]);
        p[6] = fmaf(xq, wb.z, p[6]);
        p[7] = fmaf(xq, wb.w, p[7]);
      }
      float qq[4], rr[2];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        qq[q] = (b4 ? p[q + 4] : p[q]) + __shfl_xor_sync(0xffffffffu, b4 ? p[q] : p[q + 4], 16);
#pragma unroll
      for (int q = 0; q < 2; ++q)
        rr[q] = (b3 ? qq[q + 2] : qq[q]) + __shfl_xor_sync(0xffffffffu, b3 ? qq[q] : qq[q + 2], 8);
      float z = (b2 ? rr[1] : rr[0]) + __shfl_xor_sync(0xffffffffu, b2 ? rr[0] : rr[1], 4);
      z += __shfl_xor_sync(0xffffffffu, z, 2);
      z += __shfl_xor_sync(0xffffffffu, z, 1);
      const float sc = 1.f / (1.f + expf(-z));  // sigmoid gate
      const float kf = sc + my_b;
      const bool bad = owner && !isfinite(kf);
      uint32_t key = owner && !bad ? float_key(kf) : 0u;
      if (__any_sync(0xffffffffu, bad) && lane == 0) {
        atomicOr(err, kErrMoeNonFinite);
        atomicCAS(err + 1, 0, t + 1);
      }
      int se[K];
      float sw[K];
      float tot = 0.f;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const uint32_t best = __reduce_max_sync(0xffffffffu, key);
        const uint32_t m = __ballot_sync(0xffffffffu, key == best && owner);
        const int wl = m ? __ffs(m) - 1 : 0;  // lowest lane = lowest expert on ties
        sw[j] = m ? __shfl_sync(0xffffffffu, sc, wl) : 1.f;
        se[j] = wl >> 2;
        if (lane == wl) key = 0u;
        tot += sw[j];
      }
      if (lane == i) {
#pragma unroll
        for (int j = 0; j < K; ++j) {
          te[j] = se[j];
          tw[j] = sw[j] / tot;
        }
        tinv = inv;
      }
    }
    // expert-segment positions: one atomic per (slot, expert) group of the warp's tokens
    const bool tv = lane < n;
    const int t = base + lane;
    int pos[K + 1];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int e = tv ? te[j] : -1 - lane;  // inactive lanes never match
      const unsigned peers = __match_any_sync(0xffffffffu, e);
      const int leader = __ffs(peers) - 1;
      int b = 0;
      if (lane == leader && tv) b = atomicAdd(&cursor[e], __popc(peers));
      b = __shfl_sync(0xffffffffu, b, leader);
      pos[j] = tv ? e * Tcap + b + __popc(peers & ((1u << lane) - 1u)) : 0;
    }
    pos[K] = E * Tcap + t;  // shared expert: the token's own row of its segment
    if (tv) {
#pragma unroll
      for (int j = 0; j < K; ++j) {
        sel[static_cast<size_t>(t) * K + j] = te[j];
        wgt[static_cast<size_t>(t) * K + j] = tw[j];
      }
#pragma unroll
      for (int j = 0; j <= K; ++j) {
        if (j == K && !shared) break;
        tok_of[pos[j]] = t;
        w_of[pos[j]] = j < K ? tw[j] : 1.f;
        slot_pos[static_cast<size_t>(t) * S + j] = pos[j];
      }
    }
    // rows: the whole warp moves one normalised row per token (16 B per lane) from the
    // lane's own shared-memory chunks
    for (int i = 0; i < n; ++i) {
      int pj[K + 1];
#pragma unroll
      for (int j = 0; j <= K; ++j) pj[j] = __shfl_sync(0xffffffffu, pos[j], i);
      const float iv = __shfl_sync(0xffffffffu, tinv, i);
      if (!act) continue;
      const int4 raw = myrows[i * 32];
      const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(p2[q]);
        o[q] = pack_bf16x2(f.x * iv * g[2 * q], f.y * iv * g[2 * q + 1]);
      }
      const int4 ov = make_int4(o[0], o[1], o[2], o[3]);
#pragma unroll
      for (int j = 0; j <= K; ++j) {
        if (j == K && !shared) break;
        *reinterpret_cast<int4*>(xs + static_cast<size_t>(pj[j]) * d + c0) = ov;
      }
    }
  }
}

// ------------------------------------------------------------------------------------ plan
// Expert g owns the row segment [g * Tcap, (g + 1) * Tcap) (Tcap = T rounded up to 128; the
// shared expert's rows are its tokens in order). One block: the segment offsets, the list of
// 128-row tiles that hold rows (tile k: expert tile_group[k], first row 128 * tile_mblk[k]),
// padding rows of the last tile marked tok_of = -1, scatter cursors reset.
__global__ void k_moe_plan(const int32_t* __restrict__ counts, int E, int shared, int T, int Tcap,
                           int32_t* __restrict__ off, int32_t* __restrict__ cursor,
                           int32_t* __restrict__ tile_group, int32_t* __restrict__ tile_mblk,
                           int32_t* __restrict__ num_tiles, int32_t* __restrict__ tok_of) {
  __shared__ int s_first[kMoeMaxExperts + 2], s_cnt[kMoeMaxExperts + 1];
  const int G = E + shared;
  if (threadIdx.x == 0) {
    int k = 0;
    for (int g = 0; g < G; ++g) {
      const int c = g < E ? counts[g] : T;
      s_cnt[g] = c;
      s_first[g] = k;
      k += (c + 127) / 128;
    }
    s_first[G] = k;
    *num_tiles = k;
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    off[g] = g * Tcap;
    cursor[g] = 0;
  }
  for (int g = 0; g < G; ++g) {
    const int k0 = s_first[g], nk = s_first[g + 1] - k0;
    for (int i = threadIdx.x; i < nk; i += blockDim.x) {
      tile_group[k0 + i] = g;
      tile_mblk[k0 + i] = g * (Tcap / 128) + i;
    }
    const int r0 = g * Tcap + s_cnt[g], r1 = g * Tcap + nk * 128;
    for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) tok_of[r] = -1;
  }
}

// --------------------------------------------------------------------------------- scatter
// A warp takes 32 tokens: positions come from one warp-aggregated atomic per (slot, expert),
// then the warp writes each token's normalised bf16 row into its k (+ shared) segments.
__global__ void __launch_bounds__(256) k_moe_scatter(const __nv_bfloat16* __restrict__ x, int T, int d,
                                                     const float* __restrict__ gain, const float* __restrict__ inv,
                                                     const int32_t* __restrict__ sel, const float* __restrict__ wgt,
                                                     int E, int k, int shared, const int32_t* __restrict__ off,
                                                     int32_t* __restrict__ cursor, __nv_bfloat16* __restrict__ xs,
                                                     int32_t* __restrict__ tok_of, float* __restrict__ w_of,
                                                     int32_t* __restrict__ slot_pos) {
  const int lane = threadIdx.x & 31;
  const int S = k + shared;
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int c0 = lane * 8;
  const bool act = c0 < d;
  float g[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) g[i] = act ? gain[c0 + i] : 0.f;
  for (int base = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < T; base += warps * 32) {
    const int t = base + lane;
    const bool tv = t < T;
    int pos[kMoeMaxK + 1];
    for (int j = 0; j < k; ++j) {
      const int e = tv ? sel[static_cast<size_t>(t) * k + j] : -1 - lane;  // invalid lanes never match
      const unsigned peers = __match_any_sync(0xffffffffu, e);
      const int leader = __ffs(peers) - 1;
      int b = 0;
      if (lane == leader && tv) b = atomicAdd(&cursor[e], __popc(peers));
      b = __shfl_sync(0xffffffffu, b, leader);
      pos[j] = tv ? off[e] + b + __popc(peers & ((1u << lane) - 1u)) : 0;
    }
    if (shared) pos[k] = off[E] + t;
    if (tv) {
      for (int j = 0; j < S; ++j) {
        tok_of[pos[j]] = t;
        w_of[pos[j]] = j < k ? wgt[static_cast<size_t>(t) * k + j] : 1.f;
        slot_pos[static_cast<size_t>(t) * S + j] = pos[j];
      }
    }
    // rows: token by token, the whole warp moves one d-wide row (16 B per lane)
    const int n = min(32, T - base);
    for (int i = 0; i < n; ++i) {
      const int tt = base + i;
      int pj[kMoeMaxK + 1];
      for (int j = 0; j < S; ++j) pj[j] = __shfl_sync(0xffffffffu, pos[j], i);
      if (!act) continue;
      const float iv = inv[tt];
      const int4 raw = *reinterpret_cast<const int4*>(x + static_cast<size_t>(tt) * d + c0);
      const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(p2[q]);
        o[q] = pack_bf16x2(f.x * iv * g[2 * q], f.y * iv * g[2 * q + 1]);
      }
      const int4 ov = make_int4(o[0], o[1], o[2], o[3]);
      for (int j = 0; j < S; ++j) *reinterpret_cast<int4*>(xs + static_cast<size_t>(pj[j]) * d + c0) = ov;
    }
  }
}

// --------------------------------------------------------------------------------- combine
// x_out = bf16(x1 + y_shared + sum_j y_j) in place, with the row's sum-of-squares partials
// per 64-column block (the EpiResid layout the next layer's GEMMs read).
__global__ void __launch_bounds__(256) k_moe_combine(__nv_bfloat16* __restrict__ x, int T, int d,
                                                     const __nv_bfloat16* __restrict__ ys, const int32_t* __restrict__ slot_pos,
                                                     int k, int shared, float4* __restrict__ ss_out) {
  const int lane = threadIdx.x & 31;
  const int S = k + shared;
  const int c0 = lane * 8;
  const bool act = c0 < d;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < T; t += warps) {
    float acc[8];
    __nv_bfloat16* xr = x + static_cast<size_t>(t) * d + c0;
    if (act) {
      const int4 raw = *reinterpret_cast<const int4*>(xr);
      const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(p2[q]);
        acc[2 * q] = f.x;
        acc[2 * q + 1] = f.y;
      }
      // shared expert first, then the routed experts in selection order
      for (int jj = 0; jj < S; ++jj) {
        const int j = shared ? (jj == 0 ? k : jj - 1) : jj;
        const int4 yv = *reinterpret_cast<const int4*>(
            ys + static_cast<size_t>(slot_pos[static_cast<size_t>(t) * S + j]) * d + c0);
        const __nv_bfloat162* y2 = reinterpret_cast<const __nv_bfloat162*>(&yv);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(y2[q]);
          acc[2 * q] += f.x;
          acc[2 * q + 1] += f.y;
        }
      }
    }
    float ss = 0.f;
    if (act) {
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        o[q] = pack_bf16x2(acc[2 * q], acc[2 * q + 1]);
        const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o[q]));
        ss = fmaf(y.x, y.x, fmaf(y.y, y.y, ss));
      }
      *reinterpret_cast<int4*>(xr) = make_int4(o[0], o[1], o[2], o[3]);
    }
    // 64-column blocks = groups of 8 lanes
    ss += __shfl_xor_sync(0xffffffffu, ss, 4);
    ss += __shfl_xor_sync(0xffffffffu, ss, 2);
    ss += __shfl_xor_sync(0xffffffffu, ss, 1);
    const float s1 = __shfl_sync(0xffffffffu, ss, 8), s2 = __shfl_sync(0xffffffffu, ss, 16),
                s3 = __shfl_sync(0xffffffffu, ss, 24);
    if (lane == 0) {
      const int nb = (d + 63) / 64;
      ss_out[t] = make_float4(ss, nb > 1 ? s1 : 0.f, nb > 2 ? s2 : 0.f, nb > 3 ? s3 : 0.f);
    }
  }
}

// update_balance (DeepSeek style): bias_e -= gamma * sign(load_e - mean load) per layer.
__global__ void k_moe_update_bias(const int32_t* __restrict__ counts, int E, float gamma, float* __restrict__ bias) {
  const int e = threadIdx.x;
  if (e >= E) return;
  float mean = 0.f;
  for (int i = 0; i < E; ++i) mean += static_cast<float>(counts[i]);
  mean /= static_cast<float>(E);
  const float dl = static_cast<float>(counts[e]) - mean;
  bias[e] -= gamma * (dl > 0.f ? 1.f : (dl < 0.f ? -1.f : 0.f));
}

// ------------------------------------------------------------------------------- epilogues
// Expert [gate | up] GEMM on normalised rows: the stacked B interleaves 32-column blocks
// [gate_j | up_j] per expert, so a 64-column chunk holds 32 hidden units: h = swish(g) * u.
struct EpiMoeGU {
  static constexpr int kChunk = 64;
  static constexpr int kMaxParts = 1 << 30;
  static constexpr int kSide = 0;
  static constexpr int kRopeFloats = 0;
  static constexpr bool kGrouped = true;
  const int32_t* tile_group;
  const int32_t* tile_mblk;
  const int32_t* num_tiles;
  int group_n;
  const int32_t* tok_of;
  __nv_bfloat16* hidden;
  int m;

  __device__ __forceinline__ void prologue(uint8_t*, int, int) const {}

  template <class Wait>
  __device__ __forceinline__ void run(uint8_t*, uint8_t*, Wait&& wait, uint32_t tbase, int row, int n0, int c0,
                                      int c1, bool valid, int, int) const {
    const bool live = valid && tok_of[row] >= 0;
    wait();
    for (int c = c0; c < c1; c += 64) {
      float v[64];
      tmem_row_chunk<64>(tbase + c, v);
      if (!live) continue;
      float h[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) h[i] = v[i] * fast_sigmoid(v[i]) * v[32 + i];  // common.hpp:37
      store_bf16_row(hidden + static_cast<size_t>(row) * m + (n0 + c) / 2, h, 32);
    }
  }
};

// Expert down GEMM: y[row] = bf16(w_row * acc), w = the row's combine weight.
struct EpiMoeDown {
  static constexpr int kChunk = 32;
  static constexpr int kMaxParts = 1 << 30;
  static constexpr int kSide = 0;
  static constexpr int kRopeFloats = 0;
  static constexpr bool kGrouped = true;
  const int32_t* tile_group;
  const int32_t* tile_mblk;
  const int32_t* num_tiles;
  int group_n;
  const int32_t* tok_of;
  const float* w_of;
  __nv_bfloat16* y;
  int d;

  __device__ __forceinline__ void prologue(uint8_t*, int, int) const {}

  template <class Wait>
  __device__ __forceinline__ void run(uint8_t*, uint8_t*, Wait&& wait, uint32_t tbase, int row, int n0, int c0,
                                      int c1, bool valid, int, int) const {
    const bool live = valid && tok_of[row] >= 0;
    const float w = live ? w_of[row] : 0.f;
    wait();
    for (int c = c0; c < c1; c += 32) {
      float v[32];
      tmem_row_chunk<32>(tbase + c, v);
      if (!live) continue;
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= w;
      store_bf16_row(y + static_cast<size_t>(row) * d + n0 + c, v, 32);
    }
  }
};


// ------------------------------------------------------------------ fused expert kernel
// One persistent kernel per MoE layer for all experts (routed and shared) on the 128-row tiles
// of the expert-sorted rows, the block-tail structure without Wo (csrc/block_tail.cuh):
//   x tile (bf16 normalised rows, TMA) -> for hidden chunk j of the tile's expert:
//     up   U[j&1] = x . [gate_j | up_j]^T   (N = 128: 64 hidden units)
//     E2   h = swish(g) * u -> bf16 pairs in place in TMEM
//     down D += h . Wdown_j^T               (A from TMEM)
//   E3  y = bf16(w_row * D) in place over the x tile -> TMA store
// so the expert hidden activation never leaves the SM (the grouped-GEMM pair writes and
// re-reads it: 2 * m_e bytes per routed row). Weights stream through the 3-stage ring from
// L2 with the tile's expert offset (stacked [G * 2 m_e, d] and [G * d, m_e] K-major).
template <int D>
__global__ void __launch_bounds__(kTailThreads, 1)
    k_moe_expert(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmWup,
                 const __grid_constant__ CUtensorMap tmWdown, const __grid_constant__ CUtensorMap tmY,
                 const int32_t* __restrict__ tile_group, const int32_t* __restrict__ tile_mblk,
                 const int32_t* __restrict__ num_tiles, const float* __restrict__ w_of, int me) {
  static_assert(D == 128 || D == 256, "moe expert: model dim 128 or 256");
  using S = TailSmem<D>;
  constexpr int kStages = kTailStages;
  constexpr uint32_t kStageBytes = kTailStageBytes;
  constexpr uint32_t kKB = D / 64;
  constexpr uint32_t kDownStage = D * 128u;  // Wdown_j^T: D rows x 64 K
  constexpr uint32_t kUpBox = 128u * 128u;   // 128 rows x 64 K of the interleaved [gate | up]
  constexpr int kCols = D / 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::oBar);
  uint64_t* w_full = bars;        // [3]
  uint64_t* w_empty = bars + 3;   // [3]
  uint64_t* x_full = bars + 6;    // [2] x tile of buffer b landed
  uint64_t* u_full = bars + 8;    // [2]
  uint64_t* h_full = bars + 10;   // [2]
  uint64_t* d_full = bars + 12;
  uint64_t* d_empty = bars + 13;
  uint64_t* y_full = bars + 14;   // [2] y over x in buffer b, ready to store (per buffer: the
                                  // epilogue cannot complete a buffer's phase twice ahead of the store)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 16);
  const int warp = warp_id(), lane = lane_id();
  const int num_m = *num_tiles;
  const int n_chunks = me / 64;
  auto xbuf = [&](int t) { return smem + S::oX + (t & 1) * S::kTileBytes; };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmWup);
    tma_prefetch_desc(&tmWdown);
    tma_prefetch_desc(&tmY);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&w_full[s], 1);
      mbar_init(&w_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&u_full[i], 1);
      mbar_init(&h_full[i], 256);
    }
    mbar_init(d_full, 1);
    mbar_init(d_empty, 256);
    mbar_init(&y_full[0], 256);
    mbar_init(&y_full[1], 256);
    mbar_fence_init();
  }
  if (warp == 2) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ---------------------------------------------------------------- weight stream
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      auto stage = [&](uint32_t bytes) -> uint8_t* {
        mbar_wait_sleep(&w_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&w_full[s], bytes);
        return smem + S::oW + s * kStageBytes;
      };
      auto advance = [&]() {
        if (++s == kStages) {
          s = 0;
          ph ^= 1;
        }
      };
      for (int mb = blockIdx.x; mb < num_m; mb += gridDim.x) {
        const int e = tile_group[mb];
        auto up = [&](int j) {
          for (int p = 0; p < static_cast<int>(kKB) / 2; ++p) {
            uint8_t* dst = stage(2 * kUpBox);
            tma_load_2d(dst, &tmWup, &w_full[s], (2 * p) * 64, e * 2 * me + j * 128);
            tma_load_2d(dst + kUpBox, &tmWup, &w_full[s], (2 * p + 1) * 64, e * 2 * me + j * 128);
            advance();
          }
        };
        up(0);
        if (n_chunks > 1) up(1);
        for (int j = 0; j < n_chunks; ++j) {
          uint8_t* dst = stage(kDownStage);
          tma_load_2d(dst, &tmWdown, &w_full[s], j * 64, e * D);
          advance();
          if (j + 2 < n_chunks) up(j + 2);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t id_d = umma_idesc_bf16(128, D);
      const uint32_t id_u = umma_idesc_bf16(128, 128);
      const uint32_t w0 = smem_u32(smem + S::oW);
      int s = 0;
      uint32_t ph = 0;
      auto wait_stage = [&]() -> uint32_t {
        mbar_wait(&w_full[s], ph);
        tc_fence_after();
        return w0 + s * kStageBytes;
      };
      auto release_stage = [&]() {
        mma_commit(&w_empty[s]);
        if (++s == kStages) {
          s = 0;
          ph ^= 1;
        }
      };
      int t = 0, c = 0;
      for (int mb = blockIdx.x; mb < num_m; mb += gridDim.x, ++t) {
        const uint32_t xb = smem_u32(xbuf(t));
        mbar_wait_sleep(&x_full[t & 1], (t >> 1) & 1);
        tc_fence_after();
        // U buffer of hidden chunk j = the global chunk counter's parity (what E2 waits on), so
        // tiles with an odd chunk count keep the MMA issuer and E2 in step
        const int cbase = c;
        auto up = [&](int j) {
          const uint32_t u = tmem + 256 + ((cbase + j) & 1) * 128;
          for (uint32_t p = 0; p < kKB / 2; ++p) {
            const uint32_t b = wait_stage();
#pragma unroll
            for (uint32_t kh = 0; kh < 2; ++kh) {
              const uint32_t kb = 2 * p + kh;
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_ss(u, umma_sdesc_kmajor(xb + kb * 16384 + k * 32, 128),
                            umma_sdesc_kmajor(b + kh * kUpBox + k * 32, 128), id_u, (kb | k) != 0 ? 1u : 0u);
            }
            release_stage();
          }
          mma_commit(&u_full[(cbase + j) & 1]);
        };
        up(0);
        if (n_chunks > 1) up(1);
        for (int j = 0; j < n_chunks; ++j, ++c) {
          const int hb = c & 1;
          mbar_wait(&h_full[hb], (c >> 1) & 1);
          if (j == 0) mbar_wait(d_empty, (t & 1) ^ 1);  // E3 of the previous tile drained D
          tc_fence_after();
          const uint32_t hbase = tmem + 256 + hb * 128;
          const uint32_t b = wait_stage();
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_bf16_ts(tmem, hbase + (k >> 1) * 64 + (k & 1) * 8, umma_sdesc_kmajor(b + k * 32, 128), id_d,
                        (j | k) != 0 ? 1u : 0u);
          release_stage();
          if (j + 2 < n_chunks) up(j + 2);
        }
        mma_commit(d_full);
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------------- tile I/O (TMA)
    if (lane == 0) {
      auto load_x = [&](int mb, int t) {
        mbar_arrive_expect_tx(&x_full[t & 1], S::kTileBytes);
        for (uint32_t kb = 0; kb < kKB; ++kb)
          tma_load_2d(xbuf(t) + kb * 16384, &tmX, &x_full[t & 1], kb * 64, tile_mblk[mb] * 128);
      };
      int t = 0;
      if (static_cast<int>(blockIdx.x) < num_m) load_x(blockIdx.x, 0);
      for (int mb = blockIdx.x; mb < num_m; mb += gridDim.x, ++t) {
        const int next = mb + gridDim.x;
        if (t > 0) {  // drain tile t-1 from the other buffer, then load x(t+1) into it
          mbar_wait_sleep(&y_full[(t - 1) & 1], ((t - 1) >> 1) & 1);
          for (uint32_t kb = 0; kb < kKB; ++kb)
            tma_store_2d(&tmY, xbuf(t - 1) + kb * 16384, kb * 64, tile_mblk[mb - static_cast<int>(gridDim.x)] * 128);
          bulk_commit();
          bulk_wait_read0();
        }
        if (next < num_m) load_x(next, t + 1);
      }
      if (t > 0) {
        mbar_wait_sleep(&y_full[(t - 1) & 1], ((t - 1) >> 1) & 1);
        const int last = static_cast<int>(blockIdx.x) + (t - 1) * static_cast<int>(gridDim.x);
        for (uint32_t kb = 0; kb < kKB; ++kb) tma_store_2d(&tmY, xbuf(t - 1) + kb * 16384, kb * 64, tile_mblk[last] * 128);
        bulk_commit();
        bulk_wait0();
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue warps
    const int ep = warp - 4;
    const int q = ep & 3, hf = ep >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t tD = tmem + lane_off + hf * kCols;
    int t = 0, c = 0;
    for (int mb = blockIdx.x; mb < num_m; mb += gridDim.x, ++t) {
      const int row = tile_mblk[mb] * 128 + r;
      const float w = w_of[row];  // combine weight (garbage on padding rows, never read back)
      const uint32_t xs = smem_u32(xbuf(t));
      // ---- E2 per hidden chunk: h = swish(g) * u (input rows are already normalised)
      for (int j = 0; j < n_chunks; ++j, ++c) {
        const int ub = c & 1;
        mbar_wait(&u_full[ub], (c >> 1) & 1);
        tc_fence_after();
        const uint32_t tu = tmem + lane_off + 256 + ub * 128 + hf * 64;
        float v[64];
        tmem_row_chunk<64>(tu, v);
        uint32_t hw[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float hh[2];
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const float gt = v[2 * i + k], up = v[32 + 2 * i + k];
            hh[k] = gt * up * fast_sigmoid(gt);  // swish(x) = x * sigmoid(x) (common.hpp:37)
          }
          hw[i] = pack_bf16x2(hh[0], hh[1]);
        }
        tmem_st_32x32b_x16(tu, hw);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&h_full[ub]);
      }
      // ---- E3: y = bf16(w * D) in place over the x tile -> TMA store
      mbar_wait(d_full, t & 1);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < kCols / 32; ++cc) {
        float v[32];
        tmem_row_chunk<32>(tD + cc * 32, v);
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
          const uint32_t adr = xs + sw128_off(r, (hf * kCols + cc * 32) / 8 + qd);
          sts_v4(adr, make_int4(pack_bf16x2(w * v[qd * 8 + 0], w * v[qd * 8 + 1]),
                                pack_bf16x2(w * v[qd * 8 + 2], w * v[qd * 8 + 3]),
                                pack_bf16x2(w * v[qd * 8 + 4], w * v[qd * 8 + 5]),
                                pack_bf16x2(w * v[qd * 8 + 6], w * v[qd * 8 + 7])));
        }
      }
      tc_fence_before();
      mbar_arrive(d_empty);
      fence_proxy_async_smem();
      mbar_arrive(&y_full[t & 1]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace sortk
