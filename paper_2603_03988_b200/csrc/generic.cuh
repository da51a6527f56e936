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
  const int st = p.special_tokens ? 1 : 0;
  const int off_hist = st, off_prof = st + p.H + st, off_cand = off_prof + p.P + st;
  const __nv_bfloat16* src[4] = {nullptr, nullptr, nullptr, nullptr};
  int len[4] = {0, 0, 0, 0};
  int row = 0;
  if (group == 0) {
    const int b = w / p.H, i = w - b * p.H;
    int item = p.hist_item[w], act = p.hist_action[w], sc = p.hist_scene[w];
    const int tb = tok_time_bucket(p.req_ts[b] - p.hist_ts[w], p.n_tb);
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
// head-major; G -> sigmoid -> bf16 [rows, d]. One warp per row; lane j owns pair j.
__global__ void k_qkv_prep(const float* __restrict__ raw, int rows, int R, int H, int dk, int kind,
                           const int32_t* __restrict__ pos, const float2* __restrict__ rope_tab,
                           const float* __restrict__ gain, __nv_bfloat16* __restrict__ out) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= rows) return;
  const int d = H * dk, b = w / R, r = w - b * R;
  const float* xr = raw + static_cast<size_t>(w) * d;
  if (kind == 3) {  // gate
    for (int c = lane; c < d; c += 32)
      out[static_cast<size_t>(w) * d + c] = __float2bfloat16_rn(1.f / (1.f + __expf(-xr[c])));
    return;
  }
  const int p = pos[r];
  const bool act = lane < dk / 2;
  for (int h = 0; h < H; ++h) {
    float x0 = 0.f, x1 = 0.f;
    if (act) {
      x0 = xr[h * dk + 2 * lane];
      x1 = xr[h * dk + 2 * lane + 1];
    }
    __nv_bfloat16* o = out + ((static_cast<size_t>(b) * H + h) * R + r) * dk;
    if (kind == 2) {  // V
      if (act) *reinterpret_cast<__nv_bfloat162*>(o + 2 * lane) = __floats2bfloat162_rn(x0, x1);
      continue;
    }
    const float inv = rsqrtf(warp_sum(x0 * x0 + x1 * x1) / static_cast<float>(dk) + 1e-6f);
    if (act) {
      x0 *= inv * gain[h * dk + 2 * lane];
      x1 *= inv * gain[h * dk + 2 * lane + 1];
      const float2 cs = rope_tab[static_cast<size_t>(p) * (dk / 2) + lane];
      *reinterpret_cast<__nv_bfloat162*>(o + 2 * lane) =
          __floats2bfloat162_rn(cs.x * x0 - cs.y * x1, cs.y * x0 + cs.x * x1);
    }
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
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
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
