// SPDX-License-Identifier: Apache-2.0
// Fused GEMM epilogues of the SORT block (thread <-> accumulator row).
//
// Interface used by k_gemm_bf16:
//   prologue(smem, tid, nthreads)  once per CTA, before the role split (fill scratch smem)
//   run(smem, side, wait, tbase, row, n0, c0, c1, valid, part, nparts)
//       issue this row's global prefetches, call wait() (accumulator + side data ready), then
//       read the tile's per-row side data from `side` (see kSide in gemm.cuh) and consume
//       accumulator columns [c0, c1) of the tile (absolute columns n0 + c). `part` numbers
//       the (n-slice, column half) this thread covers out of `nparts` per row.
//
// Pre-norm folding: RMSNorm(x; g) W = diag(1/rms(x)) x (diag(g) W). The gain is
// folded into the bf16 weight rows at load time and 1/rms is applied here from
// the row's fp32 sum of squares, written by whichever kernel produced x.
#pragma once

#include "gemm.cuh"

namespace sortk {

// Row statistics: each residual-stream row carries its sum of squares as kSSParts partial
// sums written by distinct epilogue threads; they are combined in a fixed order so the
// result (and everything downstream) is bitwise deterministic.
__device__ __forceinline__ float row_ss(const float4* ss, int row) {
  const float4 p = ss[row];
  return (p.x + p.y) + (p.z + p.w);
}
// Row statistics of tile row `lrow` from the side buffer (TMA-staged copy of the float4 row).
__device__ __forceinline__ float side_row_ss(const uint8_t* side, int lrow) {
  const float4 p = lds_f32x4(smem_u32(side + lrow * 16));
  return (p.x + p.y) + (p.z + p.w);
}
// 16-byte chunk j (8 fp16) of tile row `lrow` of a TMA-swizzled fp16 side table with
// `halfs` values per row (boxes of <= 64 fp16, swizzle span = box row bytes).
template <int halfs>
__device__ __forceinline__ uint4 side_row_chunk_h(const uint8_t* base, int lrow, int j) {
  constexpr int bh = halfs < 64 ? halfs : 64;  // fp16 per box row
  constexpr int S = bh * 2;                    // box row bytes == swizzle span
  constexpr int per = S / 16;                  // 16-byte chunks per box row
  const int box = j / per, jj = j % per;
  const int sw = ((lrow * S) >> 7) & (per - 1);
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(base + box * 128 * S + lrow * S + ((jj ^ sw) << 4))));
  return v;
}

__device__ __forceinline__ float row_inv_rms(float ss, float inv_d) {
  return rsqrtf(ss * inv_d + 1e-6f);  // norm.hpp:23-24 (eps = kRmsEps, norm.hpp:8)
}

// bf16 pair of (residual + accumulator) and its sum of squares: the residual pair r (bf16x2)
// widened, added to (a0, a1) on one fp32x2 add, rounded to bf16, and the rounded values'
// squares accumulated into ss on one fp32x2 FMA (even / odd columns in ss.x / ss.y, combined
// once per 64 columns). Every residual epilogue (fused block tail E1 / E3, EpiResid) uses it, so
// their row statistics stay bitwise equal.
__device__ __forceinline__ uint32_t resid_add_ss(uint32_t r, float a0, float a1, float2& ss) {
  const float2 y = fadd2(make_float2(__uint_as_float(r << 16), __uint_as_float(r & 0xFFFF0000u)), make_float2(a0, a1));
  const uint32_t w = pack_bf16x2(y.x, y.y);
  const float2 q = make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
  ss = ffma2(q, q, ss);
  return w;
}

__device__ __forceinline__ void store_bf16_row(__nv_bfloat16* dst, const float* v, int n) {
  // n multiple of 16 -> 32-byte sector stores (dst 32-byte aligned); else 16-byte stores
  if (n % 16 == 0) {
    for (int i = 0; i < n; i += 16) {
      uint32_t w[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) w[k] = pack_bf16x2(v[i + 2 * k], v[i + 2 * k + 1]);
      stg256(dst + i, w);
    }
    return;
  }
  for (int i = 0; i < n; i += 8) {
    int4 w = make_int4(pack_bf16x2(v[i], v[i + 1]), pack_bf16x2(v[i + 2], v[i + 3]),
                       pack_bf16x2(v[i + 4], v[i + 5]), pack_bf16x2(v[i + 6], v[i + 7]));
    *reinterpret_cast<int4*>(dst + i) = w;
  }
}

__device__ __forceinline__ float fast_sigmoid(float x) {
  // sigma(x) = (1 + tanh(x/2)) / 2: one MUFU op, saturates cleanly, no branch divergence.
  return fmaf(0.5f, tanh_approx(0.5f * x), 0.5f);
}

// ---------------------------------------------------------------------------
// Q/K/V/G projection epilogue (attention.cpp:93-95,109-116,124-126).
// Column chunk = one head of one section. Q,K: 1/rms -> QKNorm (per-head RMSNorm
// with gain, :111-114) -> interleaved RoPE at the row's ORIGINAL position
// (rope.hpp:27-38, cos/sin from an fp64 host table) -> bf16 [B*H, R, DK].
// V: -> bf16 [B*H, R, DK] like K (read MN-major as the B operand of PV).
// G: -> sigmoid (:125-126) -> bf16 [B*R, d].
enum : int { kSecQ = 0, kSecK = 1, kSecV = 2, kSecG = 3 };

template <int DK>
struct EpiQKVG {
  static constexpr int kChunk = DK;
  static constexpr int kMaxParts = 1 << 30;  // does not produce row statistics
  static constexpr int kSide = 3;            // row statistics + RoPE rows
  static constexpr int kRopeFloats = DK;     // DK/2 (cos, sin) pairs
  int d, H, R;      // R: rows per request of the A operand
  // Column chunk ci (= col / DK) of this GEMM's N dimension -> section / head. The host
  // interleaves the weight rows head by head ([Q_h V_h K_h G_h] ...) so every n-slice,
  // and each half of it, carries the same epilogue work.
  uint8_t csec[64], chead[64];
  float inv_d;
  const float* gain_q;  // [H*DK]
  const float* gain_k;
  __nv_bfloat16* q;
  __nv_bfloat16* k;
  __nv_bfloat16* v;
  __nv_bfloat16* g;
  int Rq, Rkv;

  __device__ __forceinline__ void prologue(uint8_t* smem, int tid, int nthreads) const {
    float* sg = reinterpret_cast<float*>(smem);
    for (int i = tid; i < H * DK; i += nthreads) {
      sg[i] = gain_q[i];
      sg[H * DK + i] = gain_k[i];
    }
  }

  template <class Wait>
  __device__ __forceinline__ void run(uint8_t* smem, uint8_t* side, Wait&& wait, uint32_t tbase,
                                      int row, int n0, int c0, int c1, bool valid, int, int) const {
    const uint32_t sg = smem_u32(smem);
    const int b = row / R, r = row - b * R;
    const int lrow = row & (kGemmBM - 1);
    wait();
    // Per-row side data (staged by the TMA producer): the input row's statistics -> 1/rms,
    // and the cos/sin pairs of the row's position (shared by every Q/K head of the row).
    const float ssum = side_row_ss(side, lrow);
    const float inv = row_inv_rms(ssum, inv_d);
    // QKNorm of v = inv * acc: v * rsqrt(mean(v^2) + eps) = acc * rsqrt(mean(acc^2) + eps / inv^2)
    const float eps_eff = 1e-6f * (ssum * inv_d + 1e-6f);
    float2 cs[DK / 2];
    {
      const uint8_t* rb = side + kSideStatBytes;
#pragma unroll
      for (int j = 0; j < DK / 8; ++j) {
        const uint4 t = side_row_chunk_h<DK>(rb, lrow, j);
        const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) cs[4 * j + e] = __half22float2(*reinterpret_cast<const __half2*>(&w[e]));
      }
    }
    for (int c = c0; c < c1; c += DK) {
      float v[DK];
      tmem_row_chunk<DK>(tbase + c, v);
      if (!valid) continue;
      const int ci = (n0 + c) / DK;
      const int s = csec[ci];
      const int head = chead[ci];
      if (s == kSecQ || s == kSecK) {
        float2 m2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < DK / 2; ++j) {
          const float2 x = make_float2(v[2 * j], v[2 * j + 1]);
          m2 = ffma2(x, x, m2);
        }
        const float qi = rsqrtf((m2.x + m2.y) * (1.f / DK) + eps_eff);
        const float2 qi2 = make_float2(qi, qi);
        const uint32_t gaddr = sg + ((s == kSecQ ? 0 : H * DK) + head * DK) * 4;
#pragma unroll
        for (int j4 = 0; j4 < DK / 4; ++j4) {
          const float4 g4 = lds_f32x4(gaddr + j4 * 16);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int j = 2 * j4 + u;
            const float2 x = fmul2(fmul2(make_float2(v[2 * j], v[2 * j + 1]), qi2),
                                   u ? make_float2(g4.z, g4.w) : make_float2(g4.x, g4.y));
            // (o0, o1) = (c, s) * x0 + (-s, c) * x1   (rope.hpp:35-36)
            const float2 o = ffma2(make_float2(-cs[j].y, cs[j].x), make_float2(x.y, x.y),
                                   fmul2(cs[j], make_float2(x.x, x.x)));
            v[2 * j] = o.x;
            v[2 * j + 1] = o.y;
          }
        }
        __nv_bfloat16* dst =
            s == kSecQ ? q + (static_cast<size_t>(b * H + head) * Rq + r) * DK
                       : k + (static_cast<size_t>(b * H + head) * Rkv + r) * DK;
        store_bf16_row(dst, v, DK);
      } else if (s == kSecV) {
#pragma unroll
        for (int i = 0; i < DK; ++i) v[i] *= inv;
        store_bf16_row(this->v + (static_cast<size_t>(b * H + head) * Rkv + r) * DK, v, DK);
      } else {
        const float hinv = 0.5f * inv;
#pragma unroll
        for (int i = 0; i < DK; ++i) v[i] = fmaf(0.5f, tanh_approx(hinv * v[i]), 0.5f);
        store_bf16_row(g + static_cast<size_t>(row) * d + head * DK, v, DK);
      }
    }
  }
};

// ---------------------------------------------------------------------------
// Residual epilogue: out = resid + acc (bf16, may alias resid -- each element is
// read and written by the same thread) and the new row's sum of squares.
// Used for x <- P(x, L_out) + Attn(...) Wo (attention.cpp:131) and
// x <- x + FFN(...). The residual half-row (<= 128 columns) is
// prefetched into registers before the accumulator wait.
struct EpiResid {
  static constexpr int kChunk = 32;
  static constexpr int kMaxParts = 4;
  static constexpr int kSide = 0;
  static constexpr int kRopeFloats = 0;
  const __nv_bfloat16* resid;
  __nv_bfloat16* out;
  float* ss_out;   // [rows, 4] partial sums of squares
  int d;

  __device__ __forceinline__ void prologue(uint8_t*, int, int) const {}

  template <class Wait>
  __device__ __forceinline__ void run(uint8_t*, uint8_t*, Wait&& wait, uint32_t tbase, int row,
                                      int n0, int c0, int c1, bool valid, int part, int nparts) const {
    int4 rv[16];  // up to 128 columns
    const int nq = (c1 - c0) / 8;
    if (valid && resid) {
      const int4* rp = reinterpret_cast<const int4*>(resid + static_cast<size_t>(row) * d + n0 + c0);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < nq) rv[i] = rp[i];
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) rv[i] = make_int4(0, 0, 0, 0);
    }
    wait();
    // sum of squares per 64-column block of the row (slot = block index), each summed in
    // column order; spans narrower than 64 columns (d = 64) fall back to one slot per part
    float2 ssb2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const int c = c0 + cc * 32;
      if (c >= c1) break;
      float v[32];
      tmem_row_chunk<32>(tbase + c, v);
      if (!valid) continue;
      int4 o[4];
#pragma unroll
      for (int qd = 0; qd < 4; ++qd) {
        const int4 r4 = rv[cc * 4 + qd];
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          w[e] = resid_add_ss(reinterpret_cast<const uint32_t*>(&r4)[e], v[qd * 8 + 2 * e], v[qd * 8 + 2 * e + 1],
                              ssb2[cc >> 1]);
        o[qd] = make_int4(w[0], w[1], w[2], w[3]);
      }
      uint8_t* op = reinterpret_cast<uint8_t*>(out + static_cast<size_t>(row) * d + n0 + c);
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const uint32_t w8[8] = {static_cast<uint32_t>(o[2 * h2].x), static_cast<uint32_t>(o[2 * h2].y),
                                static_cast<uint32_t>(o[2 * h2].z), static_cast<uint32_t>(o[2 * h2].w),
                                static_cast<uint32_t>(o[2 * h2 + 1].x), static_cast<uint32_t>(o[2 * h2 + 1].y),
                                static_cast<uint32_t>(o[2 * h2 + 1].z), static_cast<uint32_t>(o[2 * h2 + 1].w)};
        stg256(op + 32 * h2, w8);
      }
    }
    const float ssb[2] = {ssb2[0].x + ssb2[0].y, ssb2[1].x + ssb2[1].y};
    if (valid) {
      float* o = ss_out + static_cast<size_t>(row) * 4;
      if (c1 - c0 >= 64) {
        const int b0 = (n0 + c0) / 64;
        for (int i = 0; i < (c1 - c0) / 64; ++i) o[b0 + i] = ssb[i];
        if (b0 == 0)
          for (int k = d / 64; k < 4; ++k) o[k] = 0.f;
      } else {
        o[part] = ssb[0];
        if (part == 0)
          for (int k = nparts; k < 4; ++k) o[k] = 0.f;
      }
    }
  }
};

// ---------------------------------------------------------------------------
// SwishGLU up-projection epilogue: the B operand interleaves
// 32-column blocks [gate_j | up_j], so a 64-column chunk holds gate and up for 32
// hidden units: h = swish(g/rms) * (u/rms) -> bf16 hidden [M, m].
struct EpiSwiGLU {
  static constexpr int kChunk = 64;
  static constexpr int kMaxParts = 1 << 30;
  static constexpr int kSide = 1;  // row statistics
  static constexpr int kRopeFloats = 0;
  float inv_d;
  __nv_bfloat16* hidden;
  int m;

  __device__ __forceinline__ void prologue(uint8_t*, int, int) const {}

  template <class Wait>
  __device__ __forceinline__ void run(uint8_t*, uint8_t* side, Wait&& wait, uint32_t tbase, int row,
                                      int n0, int c0, int c1, bool valid, int, int) const {
    wait();
    const float inv = row_inv_rms(side_row_ss(side, row & (kGemmBM - 1)), inv_d);
    for (int c = c0; c < c1; c += 64) {
      float v[64];
      tmem_row_chunk<64>(tbase + c, v);
      if (!valid) continue;
      float h[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float gt = v[i] * inv, up = v[32 + i] * inv;
        h[i] = gt * up * fast_sigmoid(gt);  // swish(x) = x * sigmoid(x) (common.hpp:37)
      }
      store_bf16_row(hidden + static_cast<size_t>(row) * m + (n0 + c) / 2, h, 32);
    }
  }
};

}  // namespace sortk
