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

// Local step of the row-sharded embedding lookup (embedding-heavy):
// out[i] = table[ids[i]] for the ids this rank owns (already shard-local), 16-byte vectors,
// consecutive threads on consecutive chunks of a row (coalesced 64-byte item rows).
// Out-of-range ids set *err and read row 0 (check_id, tokenizer.cpp:14-19).
__global__ void k_gather_table_rows(const int4* __restrict__ table, int64_t n_rows, int chunks,
                                    const int64_t* __restrict__ ids, int64_t n, int4* __restrict__ out,
                                    int32_t* err) {
  const int64_t total = n * chunks;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = t / chunks;
    const int c = static_cast<int>(t - i * chunks);
    int64_t id = ids[i];
    if (id < 0 || id >= n_rows) {
      atomicOr(err, 1);
      id = 0;
    }
    out[t] = __ldg(table + id * chunks + c);
  }
}

// Final RMSNorm + ranking head on candidate rows, fp32 (
// PAPER.md:243 keeps the head in fp32): h = relu(xn W1 + b1), z = h W2 + b2,
// p = sigmoid(z) for {click, cart, purchase}.
// 128 candidate rows per CTA, 512 threads: warp w owns rows [8w, 8w+8), lane l owns hidden
// columns {l, l+32, ...} (CPT = dh/32 of them), so each thread keeps an 8 x CPT register
// tile; xn is staged transposed in smem (broadcast reads) and W1 streams through shared
// memory in 16-row slices (cp.async, double-buffered) that all 16 warps share, so each CTA
// reads W1 from L2 once.
// The 3 logits are reduced across the 32 lanes with shuffles in a fixed order.
constexpr int kHeadRows = 112;  // 147 CTAs for the 16,384 SORT-base candidate rows on 148 SMs (128 left 20 SMs idle)
constexpr int kHeadPitch = kHeadRows + 4;  // xs row pitch: 4-way (not 32-way) conflicts on the transposed store
constexpr int kHeadThreads = 448;  // 14 warps x 8 rows
constexpr int kHeadKSlice = 16;  // W1 rows staged per cp.async slice (double-buffered)

template <int CPT>
__global__ void __launch_bounds__(kHeadThreads)
    k_head(const __nv_bfloat16* __restrict__ x, const float4* __restrict__ ss, int R, int N, int total,
           int d, const float* __restrict__ gain, const float* __restrict__ w1,
           const float* __restrict__ b1, const float* __restrict__ w2, const float* __restrict__ b2,
           float* __restrict__ probs, float* __restrict__ logits) {
  constexpr int dh = CPT * 32;
  extern __shared__ float xs[];  // [d][kHeadPitch] transposed normalised rows, then 2 W1 slices
  float* sw1 = xs + static_cast<size_t>(d) * kHeadPitch;  // [2][kHeadKSlice][dh]
  auto stage_w1 = [&](int slice, int buf) {
    // kHeadKSlice x dh floats = 16 B chunks, spread over the CTA
    const int chunks = kHeadKSlice * dh / 4;
    for (int i = threadIdx.x; i < chunks; i += kHeadThreads) {
      const int k = slice * kHeadKSlice + (i * 4) / dh, c = (i * 4) % dh;
      const float* src = w1 + static_cast<size_t>(k) * dh + c;
      const uint32_t dst = smem_u32(sw1 + (buf * kHeadKSlice * dh) + i * 4);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(k < d ? 16 : 0)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  stage_w1(0, 0);
  const int e0 = blockIdx.x * kHeadRows;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  for (int rr = warp; rr < kHeadRows; rr += kHeadThreads / 32) {
    const int e = e0 + rr;
    if (e < total) {
      const int b = e / N, j = e - b * N;
      const size_t row = static_cast<size_t>(b) * R + (R - N) + j;
      const float4 sp = ss[row];
      const float inv = rsqrtf(((sp.x + sp.y) + (sp.z + sp.w)) / static_cast<float>(d) + 1e-6f);
      for (int c = lane; c < d; c += 32) xs[c * kHeadPitch + rr] = __bfloat162float(x[row * d + c]) * inv * gain[c];
    } else {
      for (int c = lane; c < d; c += 32) xs[c * kHeadPitch + rr] = 0.f;
    }
  }
  __syncthreads();
  float acc[8][CPT];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[r][c] = 0.f;
  const float* xw = xs + warp * 8;
  const int n_slices = (d + kHeadKSlice - 1) / kHeadKSlice;
  for (int sl = 0; sl < n_slices; ++sl) {
    if (sl + 1 < n_slices) {
      stage_w1(sl + 1, (sl + 1) & 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const float* ws = sw1 + (sl & 1) * kHeadKSlice * dh;
#pragma unroll 4
    for (int kk = 0; kk < kHeadKSlice; ++kk) {
      const int k = sl * kHeadKSlice + kk;
      if (k >= d) break;
      const float4 xa = *reinterpret_cast<const float4*>(xw + k * kHeadPitch);
      const float4 xb = *reinterpret_cast<const float4*>(xw + k * kHeadPitch + 4);
      const float xr[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
      float wv[CPT];
#pragma unroll
      for (int c = 0; c < CPT; ++c) wv[c] = ws[kk * dh + c * 32 + lane];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[r][c] = fmaf(xr[r], wv[c], acc[r][c]);
    }
    __syncthreads();  // slice buffer (sl & 1) is restaged two slices later
  }
  float z[8][3];
#pragma unroll
  for (int r = 0; r < 8; ++r) z[r][0] = z[r][1] = z[r][2] = 0.f;
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int col = c * 32 + lane;
    const float bb = b1[col];
    const float wa = w2[col * 3 + 0], wb = w2[col * 3 + 1], wc = w2[col * 3 + 2];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const float hv = fmaxf(acc[r][c] + bb, 0.f);
      z[r][0] = fmaf(hv, wa, z[r][0]);
      z[r][1] = fmaf(hv, wb, z[r][1]);
      z[r][2] = fmaf(hv, wc, z[r][2]);
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int o = 0; o < 3; ++o)
#pragma unroll
      for (int sft = 16; sft; sft >>= 1) z[r][o] += __shfl_xor_sync(0xffffffffu, z[r][o], sft);
  if (lane < 8) {
    float zz[3];
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (r == lane)
#pragma unroll
        for (int o = 0; o < 3; ++o) zz[o] = z[r][o];
    const int e = e0 + warp * 8 + lane;
    if (e < total) {
      for (int o = 0; o < 3; ++o) {
        const float v = zz[o] + b2[o];
        if (logits) logits[e * 3 + o] = v;
        // rankformer::sigmoid branch structure (common.hpp:29-35) in fp32
        probs[e * 3 + o] = v >= 0.f ? 1.f / (1.f + expf(-v)) : expf(v) / (1.f + expf(v));
      }
    }
  }
}

}  // namespace sortk
