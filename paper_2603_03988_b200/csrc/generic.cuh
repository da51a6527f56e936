// SPDX-License-Identifier: Apache-2.0
// Generic-width forward (d > 256, SORT-large: d = 1024, 16 heads of 64, m = 2560).
//
// The SORT-base kernels keep a whole weight slice resident in shared memory and the whole
// d-wide row in one TMEM tile; at d = 1024 neither fits. This path runs the projections as
// plain library GEMMs (cuBLAS, bf16 operands, fp32 accumulation and fp32 residual stream)
// around row kernels, and the attention
// core on the same tcgen05 kernel as SORT-base (head dim 64). The row kernels restate the
// reference operations: tokenizer gather/projection/RMSNorm (tokenizer.cpp:95-238), QKNorm +
// RoPE + sigmoid gate (attention.cpp:93-127), residuals and SwishGLU,
// ranking head.
#pragma once

#include "tokenizer.cuh"
#include "train.cuh"

namespace sortk {

// One token row of a group -> its bf16 concat row [K] (history: item | action | scene | time;
// candidate: item; profile: the field's table row) and its row in the sequence.
// group 0 = history (e over B*H), 1 = candidates (B*N), 2 = profile (B*P).
__global__ void k_tok_concat(const TokParams p, int group, int K, __nv_bfloat16* __restrict__ out,
                             int32_t* __restrict__ out_row) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int count = group == 0 ? p.B * p.H : (group == 1 ? p.B * p.N : p.B * p.P);
  if (w >= count) return;
  const int st = p.special_tokens || p.click_seq ? 1 : 0;  // click sequences: [BOS; clicks]
  const int off_hist = st, off_prof = st + p.H + st, off_cand = off_prof + p.P + st;
  const __nv_bfloat16* src[4] = {nullptr, nullptr, nullptr, nullptr};
  int len[4] = {0, 0, 0, 0};
  int row = 0;
  if (group == 0) {
    const int b = w / p.H, i = w - b * p.H;
    int item = p.hist_item[w], act = p.hist_action[w], sc = p.hist_scene[w];
    // click sequences: the gap to the previous click (first click: INT64_MAX / 4), as k_tokenize
    const int64_t delta = p.click_seq ? (i == 0 ? 0x1FFFFFFFFFFFFFFFll : p.hist_ts[w] - p.hist_ts[w - 1])
                                      : p.req_ts[b] - p.hist_ts[w];
    const int tb = tok_time_bucket(delta, p.n_tb);
    if (static_cast<unsigned>(item) >= static_cast<unsigned>(p.n_items) ||
        static_cast<unsigned>(act) >= static_cast<unsigned>(p.n_actions) ||
        static_cast<unsigned>(sc) >= static_cast<unsigned>(p.n_scenes)) {
      if (lane == 0) atomicOr(p.err, kErrOOV);
      item = static_cast<unsigned>(item) < static_cast<unsigned>(p.n_items) ? item : 0;
      act = static_cast<unsigned>(act) < static_cast<unsigned>(p.n_actions) ? act : 0;
      sc = static_cast<unsigned>(sc) < static_cast<unsigned>(p.n_scenes) ? sc : 0;
    }
    if (p.hist_time && lane == 0) p.hist_time[w] = tb;
    src[0] = p.item_tab + static_cast<size_t>(item) * p.item_dim;
    src[1] = p.action_tab + static_cast<size_t>(act) * p.action_dim;
    src[2] = p.scene_tab + static_cast<size_t>(sc) * p.scene_dim;
    src[3] = p.time_tab + static_cast<size_t>(tb) * p.time_dim;
    len[0] = p.item_dim;
    len[1] = p.action_dim;
    len[2] = p.scene_dim;
    len[3] = p.time_dim;
    row = b * p.L + off_hist + i;
  } else if (group == 1) {
    const int b = w / p.N, j = w - b * p.N;
    int item = p.cand_item[w];
    if (static_cast<unsigned>(item) >= static_cast<unsigned>(p.n_items)) {
      if (lane == 0) atomicOr(p.err, kErrOOV);
      item = 0;
    }
    src[0] = p.item_tab + static_cast<size_t>(item) * p.item_dim;
    len[0] = p.item_dim;
    row = b * p.L + off_cand + j;
  } else {
    const int b = w / p.P, f = w - b * p.P;
    int v = p.profile[w];
    if (static_cast<unsigned>(v) >= static_cast<unsigned>(p.prof_vocab[f])) {
      if (lane == 0) atomicOr(p.err, kErrOOV);
      v = 0;
    }
    src[0] = p.prof_tab + static_cast<size_t>(p.prof_row_off[f] + v) * p.prof_dim;
    len[0] = p.prof_dim;
    row = b * p.L + off_prof + f;
  }
  for (int k = lane; k < K; k += 32) {
    int s = 0, base = 0;
    while (s < 3 && k - base >= len[s]) base += len[s++];
    out[static_cast<size_t>(w) * K + k] = src[s][k - base];
  }
  if (lane == 0) out_row[w] = row;
}

// X[out_row[r]] = RMSNorm(y[r] + bias; gain) (emit_group, tokenizer.cpp:220-229), fp32.
__global__ void k_tok_finish(const float* __restrict__ y, const float* __restrict__ bias,
                             const float* __restrict__ gain, const int32_t* __restrict__ out_row, int rows,
                             int d, float* __restrict__ X) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= rows) return;
  const float* yr = y + static_cast<size_t>(w) * d;
  float ss = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float v = yr[c] + bias[c];
    ss = fmaf(v, v, ss);
  }
  const float inv = rsqrtf(warp_sum(ss) / static_cast<float>(d) + 1e-6f);
  float* xr = X + static_cast<size_t>(out_row[w]) * d;
  for (int c = lane; c < d; c += 32) xr[c] = (yr[c] + bias[c]) * inv * gain[c];
}

// BOS / SEP rows: raw special-table rows (tokenizer.cpp:171-176).
__global__ void k_tok_specials(const float* __restrict__ special, int B, int L, int H, int P, int d,
                               float* __restrict__ X) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= B * 3) return;
  const int b = w / 3, k = w - b * 3;
  const int row = b * L + (k == 0 ? 0 : (k == 1 ? 1 + H : 2 + H + P));
  for (int c = lane; c < d; c += 32) X[static_cast<size_t>(row) * d + c] = special[k * d + c];
}

// Per row and head: Q/K -> per-head RMSNorm with gain (attention.cpp:111-114) -> interleaved
// RoPE at the row's position (rope.hpp:27-38) -> bf16 head-major [B*H, R, dk]; V -> bf16
// head-major; G -> sigmoid -> bf16 [rows, d]. Input: the bf16 projection (row stride ld). One warp per
// row; each lane owns 8 contiguous elements (16-byte loads/stores) of chunk c = lane + 32 i, so a
// head spans dk / 8 aligned lanes and its sum of squares is a 1-3 step shuffle reduction.
template <int kV>
__global__ void k_qkv_prep(const __nv_bfloat16* __restrict__ raw, int ld, int rows, int R, int H, int dk, int kind,
                           const int32_t* __restrict__ pos, const float2* __restrict__ rope_tab,
                           const float* __restrict__ gain, __nv_bfloat16* __restrict__ out) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int d = H * dk, d8 = d >> 3, b = row / R, r = row - b * R;
  const int e = (lane * 8) & (dk - 1);  // offset inside the head (same for every chunk: 256 % dk == 0)
  const int4* src = reinterpret_cast<const int4*>(raw + static_cast<size_t>(row) * ld);
  int4 v[kV];
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    const int c = lane + 32 * i;
    v[i] = c < d8 ? src[c] : make_int4(0, 0, 0, 0);
  }
  if (kind == 3) {  // gate: row-major [rows, d]
    int4* dst = reinterpret_cast<int4*>(out + static_cast<size_t>(row) * d);
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const int c = lane + 32 * i;
      if (c >= d8) continue;
      const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&v[i]);
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 x = __bfloat1622float2(x2[k]);
        o[k] = pack_bf16x2(1.f / (1.f + __expf(-x.x)), 1.f / (1.f + __expf(-x.y)));
      }
      dst[c] = make_int4(o[0], o[1], o[2], o[3]);
    }
    return;
  }
  const size_t head0 = static_cast<size_t>(b) * H;
  if (kind == 2) {  // V: layout change only
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const int c = lane + 32 * i;
      if (c >= d8) continue;
      const int h = (c * 8) / dk;
      *reinterpret_cast<int4*>(out + ((head0 + h) * R + r) * dk + e) = v[i];
    }
    return;
  }
  float4 cs[2];  // the lane's 4 (cos, sin) pairs
  {
    const float4* t = reinterpret_cast<const float4*>(rope_tab + static_cast<size_t>(pos[r]) * (dk / 2) + e / 2);
    cs[0] = t[0];
    cs[1] = t[1];
  }
  const float* csf = reinterpret_cast<const float*>(cs);
  float ss[kV];
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&v[i]);
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 x = __bfloat1622float2(x2[k]);
      t = fmaf(x.x, x.x, fmaf(x.y, x.y, t));
    }
    ss[i] = t;
  }
  for (int o = dk / 16; o; o >>= 1)
#pragma unroll
    for (int i = 0; i < kV; ++i) ss[i] += __shfl_xor_sync(0xffffffffu, ss[i], o);
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    const int c = lane + 32 * i;
    if (c >= d8) continue;
    const int h = (c * 8) / dk;
    const float inv = rsqrtf(ss[i] / static_cast<float>(dk) + 1e-6f);
    const float4* g4 = reinterpret_cast<const float4*>(gain + c * 8);
    const float4 ga = g4[0], gb = g4[1];
    const float g[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
    const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&v[i]);
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 x = __bfloat1622float2(x2[k]);
      const float x0 = x.x * inv * g[2 * k], x1 = x.y * inv * g[2 * k + 1];
      const float cc = csf[2 * k], sn = csf[2 * k + 1];
      o[k] = pack_bf16x2(cc * x0 - sn * x1, sn * x0 + cc * x1);
    }
    *reinterpret_cast<int4*>(out + ((head0 + h) * R + r) * dk + e) = make_int4(o[0], o[1], o[2], o[3]);
  }
}

// Row RMSNorm with gain to bf16, optionally on a residual sum first (the block's two
// pre-norms, and the attention residual on P(x, L_out)):
//   v = x[(r / R) * Rsrc + map[r % R]] (+ a[r]);  xo[r] = v (if xo);  y[r] = bf16(v * rsqrt(mean v^2 + eps) * gain)
// One warp per row, lane owns float4 j = lane + 32 v (v < kV); d % 4 == 0, d <= 128 kV.
template <int kV>
__global__ void k_resid_rmsnorm(const float* __restrict__ x, const int32_t* __restrict__ map, int R, int Rsrc,
                                const float* __restrict__ a, const float* __restrict__ gain, int rows, int d,
                                float* __restrict__ xo, __nv_bfloat16* __restrict__ y) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= rows) return;
  size_t src = w;
  if (map) src = static_cast<size_t>(w / R) * Rsrc + map[w % R];
  const int d4 = d >> 2;
  const float4* xr = reinterpret_cast<const float4*>(x + src * d);
  const float4* ar = a ? reinterpret_cast<const float4*>(a + static_cast<size_t>(w) * d) : nullptr;
  float4 v[kV];
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    const int j = lane + 32 * i;
    v[i] = j < d4 ? xr[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (ar) {
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const int j = lane + 32 * i;
      if (j < d4) {
        const float4 t = ar[j];
        v[i].x += t.x;
        v[i].y += t.y;
        v[i].z += t.z;
        v[i].w += t.w;
      }
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < kV; ++i) ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  const float inv = rsqrtf(warp_sum(ss) / static_cast<float>(d) + 1e-6f);
  float4* xor_ = xo ? reinterpret_cast<float4*>(xo + static_cast<size_t>(w) * d) : nullptr;
  uint2* yr = reinterpret_cast<uint2*>(y + static_cast<size_t>(w) * d);
  const float4* g4 = reinterpret_cast<const float4*>(gain);
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    const int j = lane + 32 * i;
    if (j >= d4) continue;
    if (xor_) xor_[j] = v[i];
    const float4 g = g4[j];
    yr[j] = make_uint2(pack_bf16x2(v[i].x * inv * g.x, v[i].y * inv * g.y),
                       pack_bf16x2(v[i].z * inv * g.z, v[i].w * inv * g.w));
  }
}

// out = x[(r / R) * Rsrc + map[r % R]] + a[r]  (residual on P(x, L_out)).
__global__ void k_residual_gather(const float* __restrict__ x, const int32_t* __restrict__ map, int R, int Rsrc,
                                  const float* __restrict__ a, int rows, int d, float* __restrict__ out) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= rows) return;
  const size_t src = static_cast<size_t>(w / R) * Rsrc + map[w % R];
  for (int c = lane; c < d; c += 32)
    out[static_cast<size_t>(w) * d + c] = x[src * d + c] + a[static_cast<size_t>(w) * d + c];
}

__global__ void k_f32_to_bf16(const float* __restrict__ x, size_t n, __nv_bfloat16* __restrict__ y) {
  const size_t t0 = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0) {
    // 8 elements per step: two 16-byte loads, one 16-byte store (same rounding per element)
    const size_t n8 = n >> 3;
    for (size_t i = t0; i < n8; i += stride) {
      const float4 a = reinterpret_cast<const float4*>(x)[2 * i], b = reinterpret_cast<const float4*>(x)[2 * i + 1];
      reinterpret_cast<uint4*>(y)[i] = make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w),
                                                  pack_bf16x2(b.x, b.y), pack_bf16x2(b.z, b.w));
    }
    for (size_t i = (n8 << 3) + t0; i < n; i += stride) y[i] = __float2bfloat16_rn(x[i]);
    return;
  }
  for (size_t i = t0; i < n; i += stride) y[i] = __float2bfloat16_rn(x[i]);
}
__global__ void k_bf16_to_f32(const __nv_bfloat16* __restrict__ x, size_t n, float* __restrict__ y) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    y[i] = __bfloat162float(x[i]);
}

// logits = lo + b2, probs = sigmoid(logits) for the 3 heads.
__global__ void k_head_out(const float* __restrict__ lo, const float* __restrict__ b2, int rows,
                           float* __restrict__ logits, float* __restrict__ probs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * 3) return;
  const float z = lo[i] + b2[i % 3];
  logits[i] = z;
  probs[i] = sigmoidf_stable(z);
}

}  // namespace sortk
