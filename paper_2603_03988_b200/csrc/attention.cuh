// SPDX-License-Identifier: Apache-2.0
// K3: structured local-window attention with query pruning, on tcgen05.
//
// One CTA computes one (request b, head h, 128-row q-tile) output block of
//   O = softmax(Q K^T / sqrt(dk) + M) V        (attention.cpp:118-121)
// followed by the sigmoid gate G (attention.cpp:124-127), visiting ONLY the
// 128-column kv tiles that hold a visible entry (the block-skip rule of
// blockwise_masked_attention, block_attention.hpp:86-99, decided analytically by
// the host plan). Inside partial tiles the mask is evaluated per element from the
// compact row form visible(r, c) = lo_r <= c <= hi_r || c == self_r
// (build_mask, mask.cpp:47-74). Masked logits are -inf before the row max, so no
// 0 * NaN can arise and candidate rows never see another candidate (exact isolation).
//
// Roles (192 threads):
//   warp 0      TMA: Q tile once; K tile (128 x dk) and V^T tile (dk x 128) per kv tile,
//               double-buffered
//   warp 1      MMA: S = Q K^T (M=128, N=128, K=dk) into TMEM; O_j = P_j V_j (M=128,
//               N=dk, K=128) into one of two TMEM O buffers
//   warps 2..5  softmax: thread <-> query row; tcgen05.ld of S, online softmax with
//               exp2 (streaming-softmax recurrence of block_attention.hpp:104-122),
//               P written bf16 into the SW128 A-operand layout in smem; the rescaled
//               accumulation of O_{j-1} is deferred one tile so PV overlaps softmax.
#pragma once

#include "gemm.cuh"

namespace sortk {

constexpr int kAttnThreads = 192;

template <int DK>
struct AttnSmem {
  static constexpr uint32_t kQBytes = 128 * DK * 2;
  static constexpr uint32_t kKBytes = 128 * DK * 2;
  static constexpr uint32_t kVBytes = DK * 128 * 2;  // two [DK x 64] SW128 boxes
  static constexpr uint32_t kPBytes = 128 * 128 * 2;
  static constexpr uint32_t oQ = 0;
  static constexpr uint32_t oK = oQ + ((kQBytes + 1023) / 1024) * 1024;
  static constexpr uint32_t oV = oK + 2 * ((kKBytes + 1023) / 1024) * 1024;
  static constexpr uint32_t oP = oV + 2 * ((kVBytes + 1023) / 1024) * 1024;
  static constexpr uint32_t oBar = oP + 2 * kPBytes;
  static constexpr uint32_t kKStride = ((kKBytes + 1023) / 1024) * 1024;
  static constexpr uint32_t kVStride = ((kVBytes + 1023) / 1024) * 1024;
  static constexpr uint32_t kTotal = oBar + 16 * 8 + 16 + 1024;
};

struct AttnArgs {
  const int4* rowmeta;        // [n_qtiles*128] {lo, hi, self, 0} in kv-index space
  const int32_t* tile_off;    // [n_qtiles+1]
  const int32_t* tile_code;   // kv_tile | partial << 16
  const int32_t* qtile_order; // heavy first
  const __nv_bfloat16* g;     // [B*Rq, d] sigmoid gate
  __nv_bfloat16* out;         // [B*Rq, d]
  int BH, H, Rq, d;
  float scale_log2;
};

template <int DK>
__global__ void __launch_bounds__(kAttnThreads, 2)
    k_attention(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  using S = AttnSmem<DK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::oBar);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* s_free = bars + 6;
  uint64_t* p_full = bars + 7;    // [2]
  uint64_t* o_full = bars + 9;    // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = warp_id(), lane = lane_id();
  const int rank = blockIdx.x / a.BH;
  const int bh = blockIdx.x - rank * a.BH;
  const int qt = a.qtile_order[rank];
  const int q0 = qt * 128;
  const int t_begin = a.tile_off[qt], n_t = a.tile_off[qt + 1] - t_begin;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_full[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 128);
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem;                 // 128 columns
  const uint32_t tO0 = tmem + 128;          // 2 x DK columns

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, S::kQBytes);
      tma_load_3d(smem + S::oQ, &tmQ, q_full, 0, q0, bh);
      for (int j = 0; j < n_t; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        const int kv0 = (a.tile_code[t_begin + j] & 0xffff) * 128;
        mbar_wait(&kv_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], S::kKBytes + S::kVBytes);
        tma_load_3d(smem + S::oK + st * S::kKStride, &tmK, &kv_full[st], 0, kv0, bh);
        uint8_t* vdst = smem + S::oV + st * S::kVStride;
        tma_load_3d(vdst, &tmV, &kv_full[st], kv0, 0, bh);
        tma_load_3d(vdst + DK * 128, &tmV, &kv_full[st], kv0 + 64, 0, bh);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = umma_idesc_bf16(128, 128);
      const uint32_t id_o = umma_idesc_bf16(128, DK);
      constexpr uint32_t qsw = DK * 2;  // Q/K rows are DK*2 bytes = the swizzle span
      mbar_wait(q_full, 0);
      const uint32_t sq = smem_u32(smem + S::oQ);
      for (int j = 0; j < n_t; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&kv_full[st], ph);
        mbar_wait(s_free, (j & 1) ^ 1);
        tc_fence_after();
        const uint32_t sk = smem_u32(smem + S::oK + st * S::kKStride);
#pragma unroll
        for (int k = 0; k < DK / 16; ++k)
          mma_bf16_ss(tS, umma_sdesc_kmajor(sq + k * 32, qsw), umma_sdesc_kmajor(sk + k * 32, qsw),
                      id_s, k > 0 ? 1u : 0u);
        mma_commit(s_full);
        const int pb = j & 1;
        mbar_wait(&p_full[pb], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t sp = smem_u32(smem + S::oP + pb * S::kPBytes);
        const uint32_t sv = smem_u32(smem + S::oV + st * S::kVStride);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t pa = sp + (kk >> 2) * 16384 + (kk & 3) * 32;
          const uint32_t va = sv + (kk >> 2) * (DK * 128) + (kk & 3) * 32;
          mma_bf16_ss(tO0 + pb * DK, umma_sdesc_kmajor(pa, 128), umma_sdesc_kmajor(va, 128), id_o,
                      kk > 0 ? 1u : 0u);
        }
        mma_commit(&o_full[pb]);
        mma_commit(&kv_empty[st]);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    // Two passes over the S row held in TMEM (max, then exp2 + P store) keep only one
    // 32-column chunk in registers, so two CTAs fit per SM. Each 32-column chunk is
    // classified warp-uniformly: fully visible for all 32 rows of the warp (no mask
    // arithmetic), fully masked (skipped: P = 0, no exp), or mixed (per-element mask).
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // row within the q-tile == TMEM lane
    const int4 meta = a.rowmeta[q0 + r];
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const float NEG_INF = -__int_as_float(0x7f800000);
    const float sl2 = a.scale_log2;
    float m = NEG_INF, l = 0.f, alpha_prev = 0.f;  // m: running max of raw logits
    float acc[DK];
#pragma unroll
    for (int i = 0; i < DK; ++i) acc[i] = 0.f;
    for (int j = 0; j < n_t; ++j) {
      const int code = a.tile_code[t_begin + j];
      const int c0 = (code & 0xffff) * 128;
      const bool partial = (code >> 16) != 0;
      // per-chunk visibility class for this warp: bit cb of full_mask / none_mask
      uint32_t full_mask = 0xF, none_mask = 0;
      if (partial) {
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) {
          const int cs = c0 + cb * 32, ce = cs + 31;
          const bool f = meta.x <= cs && meta.y >= ce;
          const bool n = (meta.y < cs || meta.x > ce) && !(meta.z >= cs && meta.z <= ce);
          if (!__all_sync(0xffffffffu, f)) full_mask &= ~(1u << cb);
          if (__all_sync(0xffffffffu, n)) none_mask |= 1u << cb;
        }
      }
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      // pass 1: masked row max of the raw logits
      float mx = NEG_INF;
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        if (none_mask & (1u << cb)) continue;
        uint32_t rr[32];
        tmem_ld_32x32b_x32(tS + lane_off + cb * 32, rr);
        tmem_ld_wait();
        if (full_mask & (1u << cb)) {
#pragma unroll
          for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(rr[i]));
        } else {
          const int cs = c0 + cb * 32;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int kv = cs + i;
            const bool vis = (kv >= meta.x && kv <= meta.y) || kv == meta.z;
            mx = fmaxf(mx, vis ? __uint_as_float(rr[i]) : NEG_INF);
          }
        }
      }
      const float m_new = fmaxf(m, mx);
      // exp2 reference point in the scaled domain; 0 while the row has seen nothing yet
      const float ms = m_new == NEG_INF ? 0.f : m_new * sl2;
      const float alpha = ex2_approx(m * sl2 - ms);  // m = -inf -> 0
      // pass 2: p = 2^(s*scale*log2e - ms), bf16 P into the SW128 A-operand layout
      float2 rs2 = make_float2(0.f, 0.f);
      const float2 sl2v = make_float2(sl2, sl2), nms = make_float2(-ms, -ms);
      uint8_t* prow = smem + S::oP + (j & 1) * S::kPBytes + r * 128;
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        uint32_t w[16];
        if (none_mask & (1u << cb)) {
#pragma unroll
          for (int i = 0; i < 16; ++i) w[i] = 0u;
        } else {
          uint32_t rr[32];
          tmem_ld_32x32b_x32(tS + lane_off + cb * 32, rr);
          tmem_ld_wait();
          const bool fullc = (full_mask & (1u << cb)) != 0;
          const int cs = c0 + cb * 32;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float2 x = ffma2(make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1])),
                             sl2v, nms);
            if (!fullc) {
              const int kv = cs + 2 * i;
              if (!((kv >= meta.x && kv <= meta.y) || kv == meta.z)) x.x = NEG_INF;
              if (!((kv + 1 >= meta.x && kv + 1 <= meta.y) || kv + 1 == meta.z)) x.y = NEG_INF;
            }
            const float p0 = ex2_approx(x.x), p1 = ex2_approx(x.y);
            rs2 = fadd2(rs2, make_float2(p0, p1));
            w[i] = pack_bf16x2(p0, p1);
          }
        }
#pragma unroll
        for (int h4 = 0; h4 < 4; ++h4) {
          const int ch = cb * 4 + h4;  // 16-byte chunk index 0..15 along the 128 kv columns
          const int atom = ch >> 3, cc = ch & 7;
          *reinterpret_cast<int4*>(prow + atom * 16384 + ((cc ^ (r & 7)) << 4)) =
              make_int4(w[4 * h4], w[4 * h4 + 1], w[4 * h4 + 2], w[4 * h4 + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(s_free);  // S fully consumed: the next QK^T may overwrite it
      l = l * alpha + (rs2.x + rs2.y);
      m = m_new;
      fence_proxy_async_smem();
      mbar_arrive(&p_full[j & 1]);
      if (j > 0) {  // deferred: acc <- acc * alpha_{j-1} + O_{j-1}
        const int pb = (j - 1) & 1;
        mbar_wait(&o_full[pb], ((j - 1) >> 1) & 1);
        tc_fence_after();
        float o[DK];
        tmem_row_chunk<DK>(tO0 + pb * DK + lane_off, o);
        const float2 av = make_float2(alpha_prev, alpha_prev);
#pragma unroll
        for (int i = 0; i < DK; i += 2) {
          const float2 rr2 = ffma2(make_float2(acc[i], acc[i + 1]), av, make_float2(o[i], o[i + 1]));
          acc[i] = rr2.x;
          acc[i + 1] = rr2.y;
        }
        tc_fence_before();
      }
      alpha_prev = alpha;
    }
    if (n_t > 0) {
      const int pb = (n_t - 1) & 1;
      mbar_wait(&o_full[pb], ((n_t - 1) >> 1) & 1);
      tc_fence_after();
      float o[DK];
      tmem_row_chunk<DK>(tO0 + pb * DK + lane_off, o);
#pragma unroll
      for (int i = 0; i < DK; ++i) acc[i] = acc[i] * alpha_prev + o[i];
    }
    const int qrow = q0 + r;
    if (qrow < a.Rq) {
      const int b = bh / a.H, h = bh - b * a.H;
      const size_t off = static_cast<size_t>(b * a.Rq + qrow) * a.d + h * DK;
      const float invl = 1.f / l;
      const __nv_bfloat16* gp = a.g + off;
      float y[DK];
#pragma unroll
      for (int i = 0; i < DK; ++i) y[i] = acc[i] * invl * __bfloat162float(gp[i]);
      for (int i = 0; i < DK; i += 8) {
        int4 w = make_int4(pack_bf16x2(y[i], y[i + 1]), pack_bf16x2(y[i + 2], y[i + 3]),
                           pack_bf16x2(y[i + 4], y[i + 5]), pack_bf16x2(y[i + 6], y[i + 7]));
        *reinterpret_cast<int4*>(a.out + off + i) = w;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

}  // namespace sortk
