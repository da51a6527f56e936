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


// ---- The ranking head on the tensor cores (default; `sort_set_option("head_tc", 0)` runs
// k_head above). Same math: h = relu(x / rms(x) (g . W1) + b1), z = h W2 + b2.
//   k_gather_cand  candidate rows x[b, R - N + j] (bf16, exact) and their row statistics
//   k_head_wsplit  Wg = g . W1 (fp32) split into three bf16 pieces hi + mid + lo, which carry all
//                  24 mantissa bits; stored as B = [hi | mid | lo]^T, [dh, 3d] K-major
//   k_gemm_stream<GsHead> with A's K coordinate wrapping every d: acc = x hi + x mid + x lo
//                  = x Wg with every product exact in the fp32 TMEM accumulator -- an fp32
//                  product up to summation order (the SIMT kernel's xn rounding differs by an ulp)
//   GsHead         epilogue per 32-column chunk: h = relu(acc inv + b1), z += h W2 in column
//                  order per 128-column half; row_end: z = half 0 + half 1 + b2, sigmoid
// A is read in place through a 3D tensor map {d, N, B} (row strides d and R d) when N divides
// 128; otherwise k_gather_cand first copies the candidate rows.
__global__ void k_gather_cand(const __nv_bfloat16* __restrict__ src, const float4* __restrict__ ss_src, int R, int N,
                              int total, int d, __nv_bfloat16* __restrict__ dst, float4* __restrict__ ss_dst) {
  const int chunks = d >> 3;  // 16-byte vectors per row
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total * chunks; t += gridDim.x * blockDim.x) {
    const int e = t / chunks, c = t - e * chunks;
    const int b = e / N, j = e - b * N;
    const size_t row = static_cast<size_t>(b) * R + (R - N) + j;
    reinterpret_cast<int4*>(dst)[static_cast<size_t>(e) * chunks + c] =
        __ldg(reinterpret_cast<const int4*>(src + row * d) + c);
    if (c == 0) ss_dst[e] = ss_src[row];
  }
}

__global__ void k_head_wsplit(const float* __restrict__ w1, const float* __restrict__ gain, int d, int dh,
                              __nv_bfloat16* __restrict__ wt) {  // wt[n][p d + k] = piece p of g[k] w1[k][n]
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d * dh; i += gridDim.x * blockDim.x) {
    const int n = i / d, k = i - n * d;
    const float w = gain[k] * w1[static_cast<size_t>(k) * dh + n];
    const __nv_bfloat16 hi = __float2bfloat16_rn(w);
    const float r1 = w - __bfloat162float(hi);  // exact (Sterbenz)
    const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
    const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
    __nv_bfloat16* row = wt + static_cast<size_t>(n) * 3 * d;
    row[k] = hi;
    row[d + k] = mid;
    row[2 * d + k] = lo;
  }
}

struct GsHead {
  static constexpr int kChunk = 32;
  static constexpr bool kRowEnd = true;
  const float4* ss;  // row sum-of-squares partials: of the last layer's rows (R > 0) or gathered rows
  int R, N;          // R > 0: row e is candidate e % N of request e / N, at b R + R - N + j in ss
  float inv_d;
  const float* b1;  // [dh]
  const float* w2;  // [dh, 3]
  const float* b2;  // [3]
  float* zp;        // [2 column halves][3][M] partial logits
  float* probs;     // [M, 3]
  float* logits;    // [M, 3] or null
  int M, dh;
  __device__ void apply(int row, int col, const float (&v)[32]) const {
    size_t sr = static_cast<size_t>(row);
    if (R > 0) {
      const int b = row / N;
      sr = static_cast<size_t>(b) * R + (R - N) + (row - b * N);
    }
    const float4 sp = ss[sr];
    const float inv = rsqrtf(((sp.x + sp.y) + (sp.z + sp.w)) * inv_d + 1e-6f);  // norm.hpp:23-24
    const float4* bb = reinterpret_cast<const float4*>(b1 + col);
    const float4* ww = reinterpret_cast<const float4*>(w2 + static_cast<size_t>(col) * 3);
    // the half's chunks accumulate in order into its partial (written and re-read by this thread)
    float* dst = zp + static_cast<size_t>(col >= 128 ? 3 : 0) * M + row;
    const bool first = (col & 127) == 0;
    float z0 = first ? 0.f : dst[0], z1 = first ? 0.f : dst[M], z2 = first ? 0.f : dst[2 * M];
#pragma unroll
    for (int q = 0; q < 8; ++q) {  // columns 4q .. 4q + 3 of the chunk
      const float4 b = __ldg(bb + q);
      const float4 wa = __ldg(ww + 3 * q), wb = __ldg(ww + 3 * q + 1), wc = __ldg(ww + 3 * q + 2);
      const float h0 = fmaxf(fmaf(v[4 * q], inv, b.x), 0.f), h1 = fmaxf(fmaf(v[4 * q + 1], inv, b.y), 0.f);
      const float h2 = fmaxf(fmaf(v[4 * q + 2], inv, b.z), 0.f), h3 = fmaxf(fmaf(v[4 * q + 3], inv, b.w), 0.f);
      // w2 rows (c, o) for c = 4q .. 4q+3: wa = (c0o0 c0o1 c0o2 c1o0), wb = (c1o1 c1o2 c2o0 c2o1),
      // wc = (c2o2 c3o0 c3o1 c3o2)
      z0 = fmaf(h3, wc.y, fmaf(h2, wb.z, fmaf(h1, wa.w, fmaf(h0, wa.x, z0))));
      z1 = fmaf(h3, wc.z, fmaf(h2, wb.w, fmaf(h1, wb.x, fmaf(h0, wa.y, z1))));
      z2 = fmaf(h3, wc.w, fmaf(h2, wc.x, fmaf(h1, wb.y, fmaf(h0, wa.z, z2))));
    }
    dst[0] = z0;
    dst[M] = z1;
    dst[2 * M] = z2;
  }
  __device__ void row_end(int row) const {
#pragma unroll
    for (int o = 0; o < 3; ++o) {
      const float* z = zp + static_cast<size_t>(o) * M + row;
      const float v = (dh > 128 ? z[0] + z[3 * static_cast<size_t>(M)] : z[0]) + b2[o];
      if (logits) logits[row * 3 + o] = v;
      // rankformer::sigmoid branch structure (common.hpp:29-35) in fp32
      probs[row * 3 + o] = v >= 0.f ? 1.f / (1.f + expf(-v)) : expf(v) / (1.f + expf(v));
    }
  }
};

}  // namespace sortk
