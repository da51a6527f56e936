// SPDX-License-Identifier: Apache-2.0
// K3 (fixed-reference form): structured local-window attention with query pruning on
// tcgen05, for layers whose QKNorm logit bound B is below kFixedRefMax (always, for sane
// gains; attention.cuh explains the bound and keeps the online-max kernel for the rest).
//
// One work item = one (request b, head h, 128-row q-tile) output block of
//   O = softmax(Q K^T / sqrt(dk) + M) V        (attention.cpp:118-121)
// followed by the sigmoid gate G (attention.cpp:124-127); only kv tiles with a visible entry
// are visited (block_attention.hpp:86-99, decided by the host plan) and the mask comes from
// the compact row form visible(r, c) = lo_r <= c <= hi_r || c == self_r (mask.cpp:47-74).
//
// With a fixed softmax reference there is no running max and no rescale, so O is a plain
// sum over kv tiles and lives in TMEM for the whole item: PV(g) ACCUMULATES into it, and the
// softmax warps never fold per-tile results through registers. The pipeline is decoupled so
// that no softmax warp waits for the slowest warp of the tile it just finished:
//   * S is produced as four 32-column pieces through a ring of kSlots TMEM slots; a piece's
//     slot is handed back (s_free) as soon as the owning warps have LOADED it, so the next
//     pieces are computed while the softmax does the exponentials from registers;
//   * P is double-buffered in its own TMEM columns: P(g) waits only for PV(g-2);
//   * an item's O is read out (normalised, gated, stored) at the end of the next item's first
//     tile, before that tile's P is released to the MMA warp, whose first PV overwrites O.
//
// TMEM columns per CTA: S ring [0, 32 kSlots) fp32 | P[2] 64 columns each, bf16 pairs (kv
// column k of the tile in column k/2) | O (DK fp32 columns). DK <= 32: 3 slots, 96 + 128 +
// DK <= 256 columns, 2 CTAs per SM; DK = 64: 4 slots, 512 columns, 1 CTA per SM.
//
// Roles (320 threads, persistent): warp 0 TMA (Q per item double-buffered, K/V ring),
// warp 1 MMA (one elected thread), warps 2..9 softmax: warp pair (w, w+4) shares TMEM lane
// quarter w % 4 (32 query rows) and splits every tile by S half (64 kv columns = 2 pieces);
// the half-h warp owns output columns [h DK/2, (h+1) DK/2). Row sums are combined lo + hi.
#pragma once

#include "attention.cuh"

namespace sortk {

#ifdef SORT_ATTN_DEBUG
// bounded wait: reports the stuck barrier (block, warp, tag, parity, counters) and traps
__device__ __forceinline__ void fx_wait(uint64_t* bar, uint32_t parity, int tag, int a0, int a1) {
  const uint32_t addr = smem_u32(bar);
  for (long long it = 0; !mbar_try_wait(addr, parity); ++it) {
    if (it == (1ll << 28)) {
      printf("attn_fx stuck: block %d warp %d lane %d tag %d parity %u a0 %d a1 %d\n", blockIdx.x, threadIdx.x >> 5,
             threadIdx.x & 31, tag, parity, a0, a1);
      __trap();
    }
  }
}
#define FXW(bar, par, tag, a0, a1) fx_wait(bar, par, tag, a0, a1)
#define FXS(bar, par, tag, a0, a1) fx_wait(bar, par, tag, a0, a1)
#else
// Every wait polls try_wait without a suspend-time hint: with the 1 ms hint of
// mbar_wait_sleep, waiters on barriers completed by tcgen05.commit (an async-proxy arrive)
// were observed to sleep out the hint (a B = 256 forward took minutes).
#define FXW(bar, par, tag, a0, a1) mbar_wait(bar, par)
#define FXS(bar, par, tag, a0, a1) mbar_wait(bar, par)
#endif

template <int DK>
struct FxTmem {
  static constexpr uint32_t kCols = DK <= 32 ? 256 : 512;
  static constexpr int kCtasPerSm = DK <= 32 ? 2 : 1;
  static constexpr int kSlots = DK <= 32 ? 3 : 4;  // S ring of 32-column pieces
  static constexpr uint32_t kS = 0, kP = 32 * kSlots, kO = kP + 128;
  static_assert(kO + DK <= kCols, "TMEM plan");
};

template <int DK>
__global__ void __launch_bounds__(kAttnThreads, FxTmem<DK>::kCtasPerSm)
    k_attn_fx(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  static_assert(DK == 16 || DK == 32 || DK == 64, "head dim 16, 32 or 64");
  using S = AttnSmem<DK>;
  using T = FxTmem<DK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::oBar);
  uint64_t* q_full = bars + 0;    // [2]
  uint64_t* q_empty = bars + 2;   // [2]
  uint64_t* s_full = bars + 4;    // [kSlots <= 4] S ring slots
  uint64_t* s_free = bars + 8;    // [kSlots]
  uint64_t* p_full = bars + 12;   // [1] P(g) stored (all 256 softmax threads)
  uint64_t* pv_done = bars + 13;  // [2] PV(g) retired, by P buffer g & 1
  uint64_t* kv_full = bars + 16;  // [kKvStages]
  uint64_t* kv_empty = kv_full + kKvStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kv_empty + kKvStages);
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
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&pv_done[i], 1);
    }
    for (int i = 0; i < T::kSlots; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 128);
    }
    mbar_init(p_full, 256);
    for (int i = 0; i < kKvStages; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tslot, T::kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  auto tiles_of = [&](int it) {
    const int qt = s_order[it % a.n_qtiles];
    return s_off[qt + 1] - s_off[qt];
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // Work item i -> (request*head bh = i / n_qtiles, q-tile of rank i % n_qtiles, heaviest
    // first); (b,h)-major order keeps neighbouring q-tiles' shared K/V tiles in L2.
    if (lane == 0) {
      int g = 0, li = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
        const int bh = it / a.n_qtiles, rank = it - bh * a.n_qtiles;
        const int qt = s_order[rank];
        const int t_begin = s_off[qt], n_t = s_off[qt + 1] - t_begin;
        const int qb = li & 1;
        FXW(&q_empty[qb], ((li >> 1) & 1) ^ 1, 1, li, 0);
        mbar_arrive_expect_tx(&q_full[qb], S::kTileBytes);
        tma_load_3d(smem + S::oQ + qb * S::kStride, &tmQ, &q_full[qb], 0, qt * 128, bh);
        for (int j = 0; j < n_t; ++j, ++g) {
          const int st = g % kKvStages;
          const int kv0 = s_code[t_begin + j].x * 128;
          FXW(&kv_empty[st], ((g / kKvStages) & 1) ^ 1, 2, g, li);
          mbar_arrive_expect_tx(&kv_full[st], 2 * S::kTileBytes);
          tma_load_3d(smem + S::oK + st * S::kStride, &tmK, &kv_full[st], 0, kv0, bh);
          tma_load_3d(smem + S::oV + st * S::kStride, &tmV, &kv_full[st], 0, kv0, bh);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t id_s = umma_idesc_bf16(128, 32);
      const uint32_t id_o = umma_idesc_bf16(128, DK) | (1u << 16);  // B = V, MN-major
      constexpr uint32_t sw = DK * 2;  // Q/K/V rows are DK*2 bytes = the swizzle span
      struct Cur {
        int it, li, j, n_t, g;
      };
      auto next = [&](Cur c) {
        ++c.g;
        if (++c.j == c.n_t) {
          c.j = 0;
          ++c.li;
          c.it += gridDim.x;
          c.n_t = c.it < n_items ? tiles_of(c.it) : 0;
        }
        return c;
      };
      // S(c.g) = Q K^T as four N = 32 pieces; piece n = 4g + pc goes to ring slot n % kSlots
      // once the softmax warps have loaded that slot's previous piece (n - kSlots)
      auto issue_s = [&](const Cur& c) {
        if (c.j == 0) FXS(&q_full[c.li & 1], (c.li >> 1) & 1, 3, c.li, c.g);
        const int st = c.g % kKvStages;
        FXS(&kv_full[st], (c.g / kKvStages) & 1, 4, c.g, c.li);
        const uint32_t sq = smem_u32(smem + S::oQ + (c.li & 1) * S::kStride);
        const uint32_t sk = smem_u32(smem + S::oK + st * S::kStride);
#pragma unroll
        for (int pc = 0; pc < 4; ++pc) {
          const int n = 4 * c.g + pc, slot = n % T::kSlots;
          if (n >= T::kSlots) FXS(&s_free[slot], ((n / T::kSlots) - 1) & 1, 5, n, c.li);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < DK / 16; ++k)
            mma_bf16_ss(tmem + T::kS + slot * 32, umma_sdesc_kmajor(sq + k * 32, sw),
                        umma_sdesc_kmajor(sk + pc * 32 * DK * 2 + k * 32, sw), id_s, k > 0 ? 1u : 0u);
          mma_commit(&s_full[slot]);
        }
        if (c.j == c.n_t - 1) mma_commit(&q_empty[c.li & 1]);
      };
      Cur cur{static_cast<int>(blockIdx.x), 0, 0, 0, 0};
      cur.n_t = cur.it < n_items ? tiles_of(cur.it) : 0;
      if (cur.it < n_items) issue_s(cur);
      while (cur.it < n_items) {
        const Cur nx = next(cur);
        if (nx.it < n_items) issue_s(nx);  // S(g+1) while the softmax works on tile g
        // P(g) stored; on an item's first tile the previous item's O has also been read out
        // (the softmax reads it before arriving here), so the first PV may overwrite O
        FXS(p_full, cur.g & 1, 6, cur.g, cur.li);
        tc_fence_after();
        const int st = cur.g % kKvStages;
        const uint32_t sv = smem_u32(smem + S::oV + st * S::kStride);
        const uint32_t pa = tmem + T::kP + (cur.g & 1) * 64;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t va = sv + kk * 16 * (DK * 2);  // V rows, MN-major, SBO = 8 rows
          mma_bf16_ts(tmem + T::kO, pa + kk * 8, umma_sdesc_kmajor(va, sw), id_o, (cur.j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&pv_done[cur.g & 1]);
        mma_commit(&kv_empty[st]);
        cur = nx;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    constexpr int DH = DK / 2;
    const int quarter = warp & 3;
    const int hf = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;  // row within the q-tile == TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const float NEG_INF = -__int_as_float(0x7f800000);
    const float2 sl2v = make_float2(a.scale_log2, a.scale_log2);
    const float2 nref = make_float2(-a.ref_log2, -a.ref_log2);
    float* s_red = reinterpret_cast<float*>(smem + S::oRed);  // [2 halves][128] row sums
    int g = 0, li = 0;
    float2 lsum[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    // the previous item, finished inside the next item's first tile
    size_t p_off = 0, p_lse = 0;
    bool p_valid = false;
    float p_lsum = 0.f;

    // read the finished item's O (this warp's DK/2 columns) out of TMEM, combine the half-row
    // sums, normalise, gate and store
    auto finish_item = [&](int pli, bool gate_pending) {
      float o[DH];
      tmem_row_chunk<DH>(tmem + T::kO + hf * DH + lane_off, o);
      s_red[hf * 128 + r] = p_lsum;
      named_bar_sync(1 + quarter, 64);
      const float l = s_red[r] + s_red[128 + r];
      named_bar_sync(1 + quarter, 64);  // both partners read before the next item overwrites
      if (gate_pending) cp_async_wait_1(); else cp_async_wait_all();
      if (!p_valid) return;
      const uint8_t* gs = smem + S::oGate + ((pli & 1) * 256 + hf * 128 + r) * (DH * 2);
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
        stg256(a.out + p_off, w);  // the warp half's 32-byte output sector
      } else {
#pragma unroll
        for (int i = 0; i < DH / 8; ++i)
          reinterpret_cast<int4*>(a.out + p_off)[i] = make_int4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
      }
    };

    auto meta_of = [&](int it) {  // row metadata of item it (prefetched one item ahead)
      return it < n_items ? a.rowmeta[s_order[it % a.n_qtiles] * 128 + r] : make_int4(0, -1, -1, 0);
    };
    int4 meta_nx = meta_of(blockIdx.x);
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
      const int bh = it / a.n_qtiles, rank = it - bh * a.n_qtiles;
      const int qt = s_order[rank];
      const int q0 = qt * 128;
      const int t_begin = s_off[qt], n_t = s_off[qt + 1] - t_begin;
      const int4 meta = meta_nx;
      meta_nx = meta_of(it + gridDim.x);
      const int qrow = q0 + r;
      const int b = bh / a.H, hh = bh - b * a.H;
      const size_t off = static_cast<size_t>(b * a.Rq + qrow) * a.d + hh * DK + hf * DH;
      uint8_t* gslot = smem + S::oGate + ((li & 1) * 256 + hf * 128 + r) * (DH * 2);
      if (qrow < a.Rq) {
#pragma unroll
        for (int i = 0; i < DH / 8; ++i) cp_async_16(gslot + 16 * i, a.g + off + 8 * i);
      }
      cp_async_commit();
      const bool has_prev = li > 0;
      if (has_prev) {
        p_lsum = (lsum[0].x + lsum[0].y) + (lsum[1].x + lsum[1].y);
        lsum[0] = lsum[1] = make_float2(0.f, 0.f);
      }
      for (int j = 0; j < n_t; ++j, ++g) {
        const int2 code = s_code[t_begin + j];
        const int c0 = code.x * 128 + hf * 64;  // first kv column of this warp's half
        const uint32_t cls = static_cast<uint32_t>(code.y) >> (2 * (4 * quarter + 2 * hf));
        const uint32_t full_mask = (cls & 1u) | ((cls >> 1) & 2u);
        const uint32_t none_mask = ((cls >> 1) & 1u) | ((cls >> 2) & 2u);
        const uint32_t tP = tmem + T::kP + (g & 1) * 64 + hf * 32 + lane_off;
        // per 32-column chunk: wait for its S piece, load it, hand the ring slot back to the
        // MMA warp (later pieces are computed while this warp does the exponentials), then
        // P = exp2(s * scale_log2 - ref) as bf16 pairs, row sums in fp32. Every chunk waits for
        // its piece even when fully masked, so s_free never runs a phase ahead of the MMA warp.
#pragma unroll
        for (int cb = 0; cb < 2; ++cb) {
          const int n = 4 * g + hf * 2 + cb, slot = n % T::kSlots;
          FXW(&s_full[slot], (n / T::kSlots) & 1, 7, n, li);
          tc_fence_after();
          uint32_t rr[32];
          if (!(none_mask & (1u << cb))) {
            tmem_ld_32x32b_x32(tmem + T::kS + slot * 32 + lane_off, rr);
            tmem_ld_wait();
          }
          tc_fence_before();
          mbar_arrive(&s_free[slot]);
          uint32_t w[16];
          if (none_mask & (1u << cb)) {
#pragma unroll
            for (int i = 0; i < 16; ++i) w[i] = 0u;
          } else if (full_mask & (1u << cb)) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float2 x = ffma2(make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1])),
                                     sl2v, nref);
              // every kPolyEvery-th pair on the FMA pipe, the rest on MUFU
              const float2 p = (kPolyEvery > 0 && i % kPolyEvery == kPolyEvery - 1)
                                   ? ex2_poly2(x)
                                   : make_float2(ex2_approx(x.x), ex2_approx(x.y));
              lsum[i & 1] = fadd2(lsum[i & 1], p);
              w[i] = pack_bf16x2(p.x, p.y);
            }
          } else {
            const uint32_t bits = chunk_vis_bits(c0 + cb * 32, meta.x, meta.y, meta.z);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float2 x = ffma2(make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1])),
                               sl2v, nref);
              x.x = (bits >> (2 * i)) & 1u ? x.x : NEG_INF;
              x.y = (bits >> (2 * i + 1)) & 1u ? x.y : NEG_INF;
              const float2 p = make_float2(ex2_approx(x.x), ex2_approx(x.y));
              lsum[i & 1] = fadd2(lsum[i & 1], p);
              w[i] = pack_bf16x2(p.x, p.y);
            }
          }
          // P buffer g & 1 last held P(g-2): wait until PV(g-2) has consumed it (it had all of
          // tile g-1 to retire)
          if (cb == 0 && g >= 2) {
            FXW(&pv_done[g & 1], ((g >> 1) - 1) & 1, 8, g, li);
            tc_fence_after();
          }
          tmem_st_32x32b_x16(tP + cb * 16, w);
        }
        if (j == 0 && g > 0) {
          // the previous item's last PV (tile g - 1) completes its O; read it out before
          // releasing this tile's P: the MMA warp's first PV of this item overwrites O
          FXW(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1, 9, g, li);
          tc_fence_after();
          finish_item(li - 1, true);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(p_full);
      }
      p_valid = qrow < a.Rq;
      p_off = off;
      p_lse = static_cast<size_t>(bh) * a.Rq + qrow;
    }  // item loop
    if (li > 0) {  // the last item: its final PV
      p_lsum = (lsum[0].x + lsum[0].y) + (lsum[1].x + lsum[1].y);
      FXW(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1, 9, g, li);
      tc_fence_after();
      finish_item(li - 1, false);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, T::kCols);
  }
}

}  // namespace sortk
