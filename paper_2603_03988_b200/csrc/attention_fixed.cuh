// SPDX-License-Identifier: Apache-2.0
// K3, fixed-reference form: the attention core when QKNorm bounds every logit (kFixed in
// attention.cuh; same inputs, outputs and plan), restructured so the softmax never waits for
// the tensor core.
//
// kv tiles of the host plan (128 columns) are processed as two 64-column SUBTILES; a subtile
// whose 64 columns are invisible to all 128 rows (from the plan's chunk classes) is skipped
// by all three roles. With a fixed softmax reference (exp2(s - B), no running max) the
// P V products of an item's subtiles simply add, so O accumulates IN TMEM across the item
// (no per-tile fold into registers, no rescale):
//
//   TMEM (256 columns, 2 CTAs per SM): kSBufs S buffers of 64 columns (3 for dk <= 32, 2 for
//   dk = 64), then two O accumulators of dk columns (item parity).
//   MMA warp:   S(u) = Q K_u^T into buffer u % kSBufs (N = 64); after P(u) is written,
//               O[item] += P(u) V_u (A = P from TMEM); the buffer is reused for S(u + kSBufs)
//               once that PV has retired. So S runs up to kSBufs - 1 subtiles ahead.
//   softmax:    per subtile one 32-column chunk per warp (warp pair (w, w + 4) shares a TMEM
//               lane quarter and splits the 64 columns); P = exp2(s * log2e / sqrt(dk) - ref)
//               written as bf16 pairs in place over the chunk's first 16 columns.
//               An item's output (O / l, gate, store) is produced after the FIRST subtile of
//               the next item, so its last PV is retired by then.
// Visibility and exp work per chunk follow the plan's chunk classes exactly as in
// attention.cuh (full: every third pair on the FMA-pipe polynomial; mixed: mask bits).
//
// Measured on B200 (SORT-base, 4 layers): 1.60 ms vs 1.03 ms for k_attention<32, true>; 1.50 ms
// even without the wait for PV(u) before S(u + kSBufs). With one 32-column chunk per warp per
// subtile, the per-subtile hand-offs (S ready -> P written -> PV) are paid twice as often as
// with 128-column tiles, and that costs more than the register fold it removes. Kept as an
// A/B option (sort_set_option("attn_subtiles", 1)); k_attention stays the default.
#pragma once

#include "attention.cuh"

namespace sortk {

template <int DK>
struct AttnFLayout {
  static constexpr int kStages = DK <= 32 ? 8 : 2;  // 64-row K+V subtile ring (2 CTAs per SM)
  static constexpr int kSBufs = DK <= 32 ? 3 : 2;
  static constexpr uint32_t kOCol = kSBufs * 64;  // O[ob] at kOCol + ob * DK
  static constexpr uint32_t kCols = 256;
  static constexpr uint32_t kQBytes = 128 * DK * 2;
  static constexpr uint32_t kSubBytes = 64 * DK * 2;  // K or V subtile
  static constexpr uint32_t kQStride = ((kQBytes + 1023) / 1024) * 1024;
  static constexpr uint32_t kSubStride = ((kSubBytes + 1023) / 1024) * 1024;
  static constexpr uint32_t oQ = 0;
  static constexpr uint32_t oK = oQ + 2 * kQStride;
  static constexpr uint32_t oV = oK + kStages * kSubStride;
  static constexpr uint32_t oBar = oV + kStages * kSubStride;
  static constexpr uint32_t oRed = oBar + 64 * 8;
  static constexpr uint32_t oGate = oRed + 1024;
  static constexpr uint32_t oTiles = oGate + 2 * 128 * DK * 2;
  static constexpr uint32_t bytes(int n_tile_ints) { return oTiles + 4u * n_tile_ints + 1024; }
};

// Subtile s (0/1) of a plan tile is non-empty unless every (quarter, chunk 2s..2s+1) is "none".
__device__ __forceinline__ bool subtile_live(uint32_t cls, int s) {
  // "none" bit of (q, c) at 2 * (4q + c) + 1; chunks 2s, 2s+1 of every quarter
  const uint32_t none_bits = (s == 0 ? 0x0A0A0A0Au : 0xA0A0A0A0u);
  return ((~cls) & none_bits) != 0u;
}

template <int DK>
__global__ void __launch_bounds__(kAttnThreads, 2)
    k_attention_f(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK64,
                  const __grid_constant__ CUtensorMap tmV64, const AttnArgs a) {
  static_assert(DK == 16 || DK == 32 || DK == 64, "head dim 16, 32 or 64");
  using S = AttnFLayout<DK>;
  constexpr int NB = S::kSBufs;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::oBar);
  uint64_t* q_full = bars + 0;     // [2]
  uint64_t* q_empty = bars + 2;    // [2]
  uint64_t* s_full = bars + 4;     // [NB <= 3]
  uint64_t* p_full = bars + 8;     // [NB]
  uint64_t* s_free = bars + 12;    // [NB]  PV of the buffer's subtile retired
  uint64_t* o_full = bars + 16;    // [2]   item's last PV retired
  uint64_t* o_free = bars + 18;    // [2]   item's O read out by the softmax
  uint64_t* kv_full = bars + 20;   // [kStages]
  uint64_t* kv_empty = kv_full + S::kStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kv_empty + S::kStages);
  int32_t* s_off = reinterpret_cast<int32_t*>(smem + S::oTiles);
  int32_t* s_order = s_off + (a.n_qtiles + 1);
  int2* s_code = reinterpret_cast<int2*>(s_order + a.n_qtiles + 1);

  const int warp = warp_id(), lane = lane_id();
  const int n_items = a.n_qtiles * a.BH;
  for (int i = threadIdx.x; i <= a.n_qtiles; i += kAttnThreads) s_off[i] = a.tile_off[i];
  for (int i = threadIdx.x; i < a.n_qtiles; i += kAttnThreads) s_order[i] = a.qtile_order[i];
  for (int i = threadIdx.x; i < a.n_codes; i += kAttnThreads) s_code[i] = a.tile_code[i];
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK64);
    tma_prefetch_desc(&tmV64);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_free[i], 256);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 256);
      mbar_init(&s_free[i], 1);
    }
    for (int i = 0; i < S::kStages; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tslot, S::kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  // Subtile cursor shared by the three roles: item it (li-th of this CTA), plan tile j of
  // the item, subtile s; only live subtiles are visited.
  struct Cur {
    int it, li, t_begin, n_t, j, s;
    bool first;  // first live subtile of the item
  };
  auto item_start = [&](Cur& c) {
    if (c.it < n_items) {
      const int qt = s_order[c.it % a.n_qtiles];
      c.t_begin = s_off[qt];
      c.n_t = s_off[qt + 1] - c.t_begin;
    } else {
      c.t_begin = c.n_t = 0;
    }
    c.j = 0;
    c.s = -1;
    c.first = true;
  };
  // advance to the next live subtile (possibly of the next item); false at the end
  auto advance = [&](Cur& c) -> bool {
    while (c.it < n_items) {
      ++c.s;
      if (c.s == 2) {
        c.s = 0;
        ++c.j;
      }
      if (c.j < c.n_t) {
        if (subtile_live(static_cast<uint32_t>(s_code[c.t_begin + c.j].y), c.s)) return true;
        continue;
      }
      c.it += gridDim.x;
      ++c.li;
      item_start(c);
    }
    return false;
  };
  auto last_of_item = [&](const Cur& c) {  // no live subtile after c in its item
    int j = c.j, s = c.s;
    while (true) {
      if (++s == 2) {
        s = 0;
        ++j;
      }
      if (j >= c.n_t) return true;
      if (subtile_live(static_cast<uint32_t>(s_code[c.t_begin + j].y), s)) return false;
    }
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      Cur c{static_cast<int>(blockIdx.x), 0, 0, 0, 0, -1, true};
      item_start(c);
      int u = 0, prev_li = -1;
      while (advance(c)) {
        if (c.li != prev_li) {  // the item's Q tile
          const int qb = c.li & 1;
          const int bh = c.it / a.n_qtiles, qt = s_order[c.it % a.n_qtiles];
          mbar_wait_sleep(&q_empty[qb], ((c.li >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&q_full[qb], S::kQBytes);
          tma_load_3d(smem + S::oQ + qb * S::kQStride, &tmQ, &q_full[qb], 0, qt * 128, bh);
          prev_li = c.li;
        }
        const int bh = c.it / a.n_qtiles;
        const int kv0 = s_code[c.t_begin + c.j].x * 128 + c.s * 64;
        const int st = u % S::kStages;
        mbar_wait_sleep(&kv_empty[st], ((u / S::kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], 2 * S::kSubBytes);
        tma_load_3d(smem + S::oK + st * S::kSubStride, &tmK64, &kv_full[st], 0, kv0, bh);
        tma_load_3d(smem + S::oV + st * S::kSubStride, &tmV64, &kv_full[st], 0, kv0, bh);
        ++u;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t id_s = umma_idesc_bf16(128, 64);
      const uint32_t id_o = umma_idesc_bf16(128, DK) | (1u << 16);  // B = V, MN-major
      constexpr uint32_t sw = DK * 2;
      // S issue runs on its own cursor, up to NB - 1 subtiles ahead of PV
      Cur cs{static_cast<int>(blockIdx.x), 0, 0, 0, 0, -1, true};
      item_start(cs);
      int us = 0, s_li = -1;
      bool s_more = advance(cs);
      auto issue_s = [&]() {
        const int sb = us % NB;
        if (us >= NB) mbar_wait(&s_free[sb], ((us / NB) - 1) & 1);
        if (cs.li != s_li) {
          mbar_wait(&q_full[cs.li & 1], (cs.li >> 1) & 1);
          s_li = cs.li;
        }
        const int st = us % S::kStages;
        mbar_wait(&kv_full[st], (us / S::kStages) & 1);
        tc_fence_after();
        const uint32_t sq = smem_u32(smem + S::oQ + (cs.li & 1) * S::kQStride);
        const uint32_t sk = smem_u32(smem + S::oK + st * S::kSubStride);
#pragma unroll
        for (int k = 0; k < DK / 16; ++k)
          mma_bf16_ss(tmem + sb * 64, umma_sdesc_kmajor(sq + k * 32, sw), umma_sdesc_kmajor(sk + k * 32, sw), id_s,
                      k > 0 ? 1u : 0u);
        mma_commit(&s_full[sb]);
        if (last_of_item(cs)) mma_commit(&q_empty[cs.li & 1]);
        ++us;
        s_more = advance(cs);
      };
      for (int i = 0; i < NB && s_more; ++i) issue_s();
      Cur c{static_cast<int>(blockIdx.x), 0, 0, 0, 0, -1, true};
      item_start(c);
      int u = 0, o_li = -1;
      while (advance(c)) {
        const int sb = u % NB, st = u % S::kStages, ob = c.li & 1;
        const bool first = c.li != o_li;
        o_li = c.li;
        mbar_wait(&p_full[sb], (u / NB) & 1);
        if (first && c.li >= 2) mbar_wait(&o_free[ob], ((c.li >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t sv = smem_u32(smem + S::oV + st * S::kSubStride);
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // two 32-column halves x two K = 16 steps
          const int h2 = q >> 1, ks = q & 1;
          const uint32_t pa = tmem + sb * 64 + h2 * 32 + ks * 8;
          const uint32_t va = sv + (h2 * 32 + ks * 16) * (DK * 2);
          mma_bf16_ts(tmem + S::kOCol + ob * DK, pa, umma_sdesc_kmajor(va, sw), id_o, (first && q == 0) ? 0u : 1u);
        }
        mma_commit(&kv_empty[st]);
        mma_commit(&s_free[sb]);
        if (last_of_item(c)) mma_commit(&o_full[ob]);
        ++u;
        if (s_more) issue_s();
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    constexpr int DH = DK / 2;
    const int quarter = warp & 3;
    const int hf = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const float NEG_INF = -__int_as_float(0x7f800000);
    const float2 sl2v = make_float2(a.scale_log2, a.scale_log2);
    const float2 nref = make_float2(-a.ref_log2, -a.ref_log2);
    float* s_sum = reinterpret_cast<float*>(smem + S::oRed);  // [2 halves][128 rows]
    float2 lsum[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    // the previous item, finished after the next item's first subtile
    bool p_valid = false;
    size_t p_off = 0, p_lse = 0;
    float p_lsum = 0.f;
    int p_li = -1;
    auto finish_item = [&](int li, bool gate_pending) {
      const int ob = li & 1;
      mbar_wait_sleep(&o_full[ob], (li >> 1) & 1);
      tc_fence_after();
      float o[DH];
      tmem_row_chunk<DH>(tmem + S::kOCol + ob * DK + hf * DH + lane_off, o);
      tc_fence_before();
      mbar_arrive(&o_free[ob]);
      s_sum[hf * 128 + r] = p_lsum;
      named_bar_sync(1 + quarter, 64);
      const float l = s_sum[r] + s_sum[128 + r];
      named_bar_sync(1 + quarter, 64);
      if (gate_pending) cp_async_wait_1(); else cp_async_wait_all();
      if (!p_valid) return;
      const uint8_t* gs = smem + S::oGate + ((li & 1) * 256 + hf * 128 + r) * (DH * 2);
      const float invl = 1.f / l;
      if (a.lse) {  // training outputs: P = exp2(s * scale_log2 - lse2), pre-gate O
        if (hf == 0) a.lse[p_lse] = a.ref_log2 + log2f(l);
        uint32_t wo[DH / 2];
#pragma unroll
        for (int i = 0; i < DH / 2; ++i) wo[i] = pack_bf16x2(o[2 * i] * invl, o[2 * i + 1] * invl);
#pragma unroll
        for (int i = 0; i < DH / 8; ++i)
          reinterpret_cast<int4*>(a.o_pre + p_off)[i] = make_int4(wo[4 * i], wo[4 * i + 1], wo[4 * i + 2], wo[4 * i + 3]);
      }
      uint32_t w[DH / 2];
#pragma unroll
      for (int i = 0; i < DH / 8; ++i) {
        const int4 gv = *reinterpret_cast<const int4*>(gs + 16 * i);
        const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 gf = __bfloat1622float2(g2[e]);
          w[4 * i + e] = pack_bf16x2(o[8 * i + 2 * e] * invl * gf.x, o[8 * i + 2 * e + 1] * invl * gf.y);
        }
      }
      if constexpr (DH == 16) {
        stg256(a.out + p_off, w);
      } else {
#pragma unroll
        for (int i = 0; i < DH / 8; ++i)
          reinterpret_cast<int4*>(a.out + p_off)[i] = make_int4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
      }
    };
    Cur c{static_cast<int>(blockIdx.x), 0, 0, 0, 0, -1, true};
    item_start(c);
    int u = 0, cur_li = -1;
    int4 meta = make_int4(0, -1, -1, 0);
    size_t off = 0, lse_idx = 0;
    bool valid = false;
    while (advance(c)) {
      if (c.li != cur_li) {  // a new item: gate prefetch, row metadata
        if (cur_li >= 0) {
          p_lsum = (lsum[0].x + lsum[0].y) + (lsum[1].x + lsum[1].y);
          lsum[0] = lsum[1] = make_float2(0.f, 0.f);
          p_li = cur_li;
          p_valid = valid;
          p_off = off;
          p_lse = lse_idx;
        }
        cur_li = c.li;
        const int bh = c.it / a.n_qtiles, qt = s_order[c.it % a.n_qtiles];
        const int qrow = qt * 128 + r;
        const int b = bh / a.H, hh = bh - b * a.H;
        meta = a.rowmeta[qt * 128 + r];
        off = static_cast<size_t>(b * a.Rq + qrow) * a.d + hh * DK + hf * DH;
        valid = qrow < a.Rq;
        lse_idx = static_cast<size_t>(bh) * a.Rq + qrow;
        uint8_t* gslot = smem + S::oGate + ((c.li & 1) * 256 + hf * 128 + r) * (DH * 2);
        if (valid) {
#pragma unroll
          for (int i = 0; i < DH / 8; ++i) cp_async_16(gslot + 16 * i, a.g + off + 8 * i);
        }
        cp_async_commit();
      }
      const int sb = u % NB;
      const uint32_t tS = tmem + sb * 64 + hf * 32 + lane_off;
      const int2 code = s_code[c.t_begin + c.j];
      const int ck = 2 * c.s + hf;  // this warp's 32-column chunk of the plan tile
      const uint32_t cls = (static_cast<uint32_t>(code.y) >> (2 * (4 * quarter + ck))) & 3u;
      const int cs0 = code.x * 128 + ck * 32;
      mbar_wait_sleep(&s_full[sb], (u / NB) & 1);
      tc_fence_after();
      uint32_t w[16];
      if (cls & 2u) {  // invisible to every row of this warp
#pragma unroll
        for (int i = 0; i < 16; ++i) w[i] = 0u;
      } else {
        uint32_t rr[32];
        tmem_ld_32x32b_x32(tS, rr);
        tmem_ld_wait();
        if (cls & 1u) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 x = ffma2(make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1])), sl2v, nref);
            const float2 p = (kPolyEvery > 0 && i % kPolyEvery == kPolyEvery - 1)
                                 ? ex2_poly2(x)
                                 : make_float2(ex2_approx(x.x), ex2_approx(x.y));
            lsum[i & 1] = fadd2(lsum[i & 1], p);
            w[i] = pack_bf16x2(p.x, p.y);
          }
        } else {
          const uint32_t bits = chunk_vis_bits(cs0, meta.x, meta.y, meta.z);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float2 x = ffma2(make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1])), sl2v, nref);
            x.x = (bits >> (2 * i)) & 1u ? x.x : NEG_INF;
            x.y = (bits >> (2 * i + 1)) & 1u ? x.y : NEG_INF;
            const float2 p = make_float2(ex2_approx(x.x), ex2_approx(x.y));
            lsum[i & 1] = fadd2(lsum[i & 1], p);
            w[i] = pack_bf16x2(p.x, p.y);
          }
        }
      }
      tmem_st_32x32b_x16(tS, w);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[sb]);
      if (c.first && p_li >= 0 && p_li == c.li - 1) {
        finish_item(p_li, true);
        p_li = -2;
      }
      c.first = false;
      ++u;
    }
    if (cur_li >= 0) {
      p_lsum = (lsum[0].x + lsum[0].y) + (lsum[1].x + lsum[1].y);
      p_valid = valid;
      p_off = off;
      p_lse = lse_idx;
      finish_item(cur_li, false);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, S::kCols);
  }
}

}  // namespace sortk
