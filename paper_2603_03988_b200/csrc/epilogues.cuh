// SPDX-License-Identifier: Apache-2.0
// Fused GEMM epilogues of the SORT block (thread <-> accumulator row).
//
// Pre-norm folding: RMSNorm(x; g) W = diag(1/rms(x)) x (diag(g) W). The gain is
// folded into the bf16 weight rows at load time and 1/rms is applied here from
// the row's fp32 sum of squares, written by whichever kernel produced x.
#pragma once

#include "gemm.cuh"

namespace sortk {

__device__ __forceinline__ float row_inv_rms(const float* ss, int row, float inv_d) {
  return rsqrtf(ss[row] * inv_d + 1e-6f);  // norm.hpp:23-24 (eps = kRmsEps, norm.hpp:8)
}

__device__ __forceinline__ void store_bf16_row(__nv_bfloat16* dst, const float* v, int n) {
  // n multiple of 8; dst 16-byte aligned
  for (int i = 0; i < n; i += 8) {
    int4 w = make_int4(pack_bf16x2(v[i], v[i + 1]), pack_bf16x2(v[i + 2], v[i + 3]),
                       pack_bf16x2(v[i + 4], v[i + 5]), pack_bf16x2(v[i + 6], v[i + 7]));
    *reinterpret_cast<int4*>(dst + i) = w;
  }
}

// ---------------------------------------------------------------------------
// Q/K/V/G projection epilogue (attention.cpp:93-95,109-116,124-126).
// Column chunk = one head of one section. Q,K: 1/rms -> QKNorm (per-head RMSNorm
// with gain, :111-114) -> interleaved RoPE at the row's ORIGINAL position
// (rope.hpp:27-38, cos/sin from an fp64 host table) -> bf16 [B*H, R, DK].
// V: -> bf16 V^T [B*H, DK, Rkv_pad] (the K-major B operand of PV).
// G: -> sigmoid (:125-126) -> bf16 [B*R, d].
enum : int { kSecQ = 0, kSecK = 1, kSecV = 2, kSecG = 3 };

template <int DK>
struct EpiQKVG {
  static constexpr int kChunk = DK;
  int d, H, R;  // R: rows per request of the A operand
  int sec[4];
  float inv_d;
  const float* ss;
  const float* gain_q;  // [H*DK]
  const float* gain_k;
  const float2* rope;   // [(max_pos+1) * DK/2] (cos, sin)
  const int32_t* pos;   // [R]
  __nv_bfloat16* q;
  __nv_bfloat16* k;
  __nv_bfloat16* vt;
  __nv_bfloat16* g;
  int Rq, Rkv, Rkv_pad;

  template <int C>
  __device__ __forceinline__ void run(uint32_t tbase, int row, int n0, int BN, bool valid) const {
    const int b = row / R, r = row - b * R;
    const float inv = valid ? row_inv_rms(ss, row, inv_d) : 0.f;
    for (int c = 0; c < BN; c += DK) {
      float v[DK];
      tmem_row_chunk<DK>(tbase + c, v);
      if (!valid) continue;
      const int col = n0 + c;
      const int si = col / d;
      const int s = sec[si];
      const int head = (col - si * d) / DK;
#pragma unroll
      for (int i = 0; i < DK; ++i) v[i] *= inv;
      if (s == kSecQ || s == kSecK) {
        float m = 0.f;
#pragma unroll
        for (int i = 0; i < DK; ++i) m += v[i] * v[i];
        const float qi = rsqrtf(m * (1.f / DK) + 1e-6f);
        const float* gn = (s == kSecQ ? gain_q : gain_k) + head * DK;
#pragma unroll
        for (int i = 0; i < DK; ++i) v[i] = v[i] * qi * __ldg(gn + i);
        const float2* cs = rope + static_cast<size_t>(pos[r]) * (DK / 2);
#pragma unroll
        for (int j = 0; j < DK / 2; ++j) {
          const float2 t = __ldg(cs + j);
          const float x0 = v[2 * j], x1 = v[2 * j + 1];
          v[2 * j] = t.x * x0 - t.y * x1;
          v[2 * j + 1] = t.y * x0 + t.x * x1;
        }
        __nv_bfloat16* dst =
            s == kSecQ ? q + (static_cast<size_t>(b * H + head) * Rq + r) * DK
                       : k + (static_cast<size_t>(b * H + head) * Rkv + r) * DK;
        store_bf16_row(dst, v, DK);
      } else if (s == kSecV) {
        __nv_bfloat16* dst = vt + static_cast<size_t>(b * H + head) * DK * Rkv_pad + r;
#pragma unroll
        for (int i = 0; i < DK; ++i) dst[static_cast<size_t>(i) * Rkv_pad] = __float2bfloat16_rn(v[i]);
      } else {
#pragma unroll
        for (int i = 0; i < DK; ++i) v[i] = sigmoidf_stable(v[i]);
        store_bf16_row(g + static_cast<size_t>(row) * d + head * DK, v, DK);
      }
    }
  }
};

// ---------------------------------------------------------------------------
// Residual epilogue: out = resid + acc (bf16, may alias resid -- each element is
// read and written by the same thread) and the new row's sum of squares.
// Used for x <- P(x, L_out) + Attn(...) Wo (attention.cpp:131) and
// x <- x + FFN(...).
struct EpiResid {
  static constexpr int kChunk = 32;
  const __nv_bfloat16* resid;
  __nv_bfloat16* out;
  float* ss_out;
  int d;
  int ss_atomic;

  template <int C>
  __device__ __forceinline__ void run(uint32_t tbase, int row, int n0, int BN, bool valid) const {
    float ss = 0.f;
    for (int c = 0; c < BN; c += 32) {
      float v[32];
      tmem_row_chunk<32>(tbase + c, v);
      if (!valid) continue;
      const size_t off = static_cast<size_t>(row) * d + n0 + c;
      const int4* rp = reinterpret_cast<const int4*>(resid + off);
      int4 o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int4 rv = resid ? rp[q] : make_int4(0, 0, 0, 0);
        const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&rv);
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(r2[e]);
          w[e] = pack_bf16x2(f.x + v[q * 8 + 2 * e], f.y + v[q * 8 + 2 * e + 1]);
          const float2 y = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&w[e]));
          ss += y.x * y.x + y.y * y.y;
        }
        o[q] = make_int4(w[0], w[1], w[2], w[3]);
      }
      int4* op = reinterpret_cast<int4*>(out + off);
#pragma unroll
      for (int q = 0; q < 4; ++q) op[q] = o[q];
    }
    if (valid) {
      if (ss_atomic) atomicAdd(ss_out + row, ss);
      else ss_out[row] = ss;
    }
  }
};

// ---------------------------------------------------------------------------
// SwishGLU up-projection epilogue: the B operand interleaves
// 32-column blocks [gate_j | up_j], so a 64-column chunk holds gate and up for 32
// hidden units: h = swish(g/rms) * (u/rms) -> bf16 hidden [M, m].
struct EpiSwiGLU {
  static constexpr int kChunk = 64;
  const float* ss;
  float inv_d;
  __nv_bfloat16* hidden;
  int m;

  template <int C>
  __device__ __forceinline__ void run(uint32_t tbase, int row, int n0, int BN, bool valid) const {
    const float inv = valid ? row_inv_rms(ss, row, inv_d) : 0.f;
    for (int c = 0; c < BN; c += 64) {
      float v[64];
      tmem_row_chunk<64>(tbase + c, v);
      if (!valid) continue;
      float h[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float gt = v[i] * inv, up = v[32 + i] * inv;
        h[i] = gt / (1.f + __expf(-gt)) * up;  // swish(x) = x * sigmoid(x) (common.hpp:37)
      }
      store_bf16_row(hidden + static_cast<size_t>(row) * m + (n0 + c) / 2, h, 32);
    }
  }
};

}  // namespace sortk
