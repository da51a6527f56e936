// SPDX-License-Identifier: Apache-2.0
// Small kernels around the block stack: pruned-row gather and the fp32 ranking head.
#pragma once

#include "ptx.cuh"

namespace sortk {

// P(x, L_out) generalised to retained rows (prune_queries / retained_rows,
// mask.cpp:125-154): dst[b, i] = src[b, rows[i]] plus the row's sum of squares.
// One warp per destination row, 16-byte vector copies.
__global__ void k_gather_rows(const __nv_bfloat16* __restrict__ src, const float4* __restrict__ ss_src,
                              __nv_bfloat16* __restrict__ dst, float4* __restrict__ ss_dst,
                              const int32_t* __restrict__ rows, int B, int Rsrc, int Rdst, int d) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= B * Rdst) return;
  const int b = w / Rdst, i = w - b * Rdst;
  const size_t s = static_cast<size_t>(b) * Rsrc + rows[i];
  const int4* sp = reinterpret_cast<const int4*>(src + s * d);
  int4* dp = reinterpret_cast<int4*>(dst + static_cast<size_t>(w) * d);
  for (int c = lane; c < d / 8; c += 32) dp[c] = sp[c];
  if (lane == 0) ss_dst[w] = ss_src[s];
}

// Final RMSNorm + ranking head on candidate rows, fp32 (
// PAPER.md:243 keeps the head in fp32): h = relu(xn W1 + b1), z = h W2 + b2,
// p = sigmoid(z) for {click, cart, purchase}. 32 candidate rows per CTA.
constexpr int kHeadRows = 32;
constexpr int kHeadThreads = 256;

__global__ void __launch_bounds__(kHeadThreads)
    k_head(const __nv_bfloat16* __restrict__ x, const float4* __restrict__ ss, int R, int N, int total,
           int d, int dh, const float* __restrict__ gain, const float* __restrict__ w1,
           const float* __restrict__ b1, const float* __restrict__ w2, const float* __restrict__ b2,
           float* __restrict__ probs, float* __restrict__ logits) {
  extern __shared__ float hsm[];
  float* xs = hsm;                  // [32][d]
  float* hs = hsm + kHeadRows * d;  // [32][dh]
  const int e0 = blockIdx.x * kHeadRows;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  for (int rr = warp; rr < kHeadRows; rr += kHeadThreads / 32) {
    const int e = e0 + rr;
    if (e < total) {
      const int b = e / N, j = e - b * N;
      const size_t row = static_cast<size_t>(b) * R + (R - N) + j;
      const float4 sp = ss[row];
      const float inv = rsqrtf(((sp.x + sp.y) + (sp.z + sp.w)) / static_cast<float>(d) + 1e-6f);
      for (int c = lane; c < d; c += 32) xs[rr * d + c] = __bfloat162float(x[row * d + c]) * inv * gain[c];
    } else {
      for (int c = lane; c < d; c += 32) xs[rr * d + c] = 0.f;
    }
  }
  __syncthreads();
  for (int c = t; c < dh; c += kHeadThreads) {
    float acc[kHeadRows];
#pragma unroll
    for (int r = 0; r < kHeadRows; ++r) acc[r] = 0.f;
    for (int k = 0; k < d; ++k) {
      const float w = __ldg(w1 + static_cast<size_t>(k) * dh + c);
#pragma unroll
      for (int r = 0; r < kHeadRows; ++r) acc[r] = fmaf(xs[r * d + k], w, acc[r]);
    }
    const float bb = b1[c];
#pragma unroll
    for (int r = 0; r < kHeadRows; ++r) hs[r * dh + c] = fmaxf(acc[r] + bb, 0.f);
  }
  __syncthreads();
  for (int rr = warp; rr < kHeadRows; rr += kHeadThreads / 32) {
    const int e = e0 + rr;
    float z0 = 0.f, z1 = 0.f, z2 = 0.f;
    for (int c = lane; c < dh; c += 32) {
      const float h = hs[rr * dh + c];
      z0 = fmaf(h, w2[c * 3 + 0], z0);
      z1 = fmaf(h, w2[c * 3 + 1], z1);
      z2 = fmaf(h, w2[c * 3 + 2], z2);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      z0 += __shfl_xor_sync(0xffffffffu, z0, o);
      z1 += __shfl_xor_sync(0xffffffffu, z1, o);
      z2 += __shfl_xor_sync(0xffffffffu, z2, o);
    }
    if (lane == 0 && e < total) {
      const float z[3] = {z0 + b2[0], z1 + b2[1], z2 + b2[2]};
      for (int o = 0; o < 3; ++o) {
        if (logits) logits[e * 3 + o] = z[o];
        // rankformer::sigmoid branch structure (common.hpp:29-35) in fp32
        probs[e * 3 + o] = z[o] >= 0.f ? 1.f / (1.f + expf(-z[o])) : expf(z[o]) / (1.f + expf(z[o]));
      }
    }
  }
}

}  // namespace sortk
