// SPDX-License-Identifier: Apache-2.0
// K3: structured local-window attention with query pruning, on tcgen05.
//
// One work item = one (request b, head h, 128-row q-tile) output block of
//   O = softmax(Q K^T / sqrt(dk) + M) V        (attention.cpp:118-121)
// followed by the sigmoid gate G (attention.cpp:124-127). Only the 128-column kv
// tiles holding a visible entry are visited (the block-skip rule of
// blockwise_masked_attention, block_attention.hpp:86-99, decided analytically by the
// host plan, which also pre-classifies every warp's 32-column chunks as fully visible /
// invisible / mixed). Inside mixed chunks the mask comes from the compact row form
// visible(r, c) = lo_r <= c <= hi_r || c == self_r (build_mask, mask.cpp:47-74); masked
// entries never enter the exponent, so candidate rows never see another candidate
// (exact isolation) and no 0 * NaN can arise.
//
// Softmax reference point. With QKNorm (attention.cpp:111-114) every q/k row has norm
// <= sqrt(dk) * max|gain| (RMSNorm output, then a RoPE rotation), so every logit obeys
// |s| <= B = sqrt(dk) * max|g_q| * max|g_k| ("bounded logits"). When
// B < kFixedRefMax the kernel uses the FIXED reference exp(s - B) instead of the running
// row max (softmax is shift-invariant; 2^(-2B log2 e) stays a normal fp32/bf16 number), so
// kv tiles never rescale each other. Otherwise (unbounded logits, e.g. the op-level
// sort_block_attention entry) the online max with rescaling runs (streaming-softmax
// recurrence of block_attention.hpp:104-122); the two half-row warps exchange tile maxima.
//
// TMEM (256 columns per CTA, 2 CTAs per SM): two 128-column buffers, tile g uses buffer
// g & 1. In a buffer: S (fp32, 128 cols) -> the softmax writes P (bf16 pairs) in place over
// the consumed columns [0,32) and [64,96) -> PV writes this tile's O_g (fp32, DK cols) into
// the free columns [32, 32+DK). The softmax adds O_g into registers (tile order: the result
// is deterministic) while the tensor core already computes S(g+1) in the other buffer.
//
// Roles (320 threads, persistent):
//   warp 0      TMA: Q per item (double-buffered), K and V tiles (128 x dk each) per kv tile
//               (kKvStages-deep ring); runs ahead across items
//   warp 1      MMA: S(g+1) = Q K^T as soon as O(g-1) has been read out of its buffer, then
//               O_g = P(g) V(g) (A = P from TMEM, B = V read MN-major)
//   warps 2..9  softmax: warp pair (w, w+4) shares TMEM lane quarter w % 4 (query rows) and
//               splits every tile by S half; the half-h warp owns output columns
//               [h*DK/2, (h+1)*DK/2). Row sums are combined lo + hi at item end.
#pragma once

#include "gemm.cuh"

namespace sortk {

constexpr int kAttnThreads = 320;
constexpr float kFixedRefMax = 40.f;  // 2^(-2*40*log2 e) ~ 2e-35 > FLT_MIN
constexpr int kKvStages = 4;
#ifndef SORT_ATTN_POLY_EVERY
#define SORT_ATTN_POLY_EVERY 3
#endif
#ifndef SORT_ATTN_SPIN
#define SORT_ATTN_SPIN 0
#endif
// softmax-warp waits on S / PV completion: suspend-hint try_wait (default) or a plain spin
#if SORT_ATTN_SPIN
#define SOFTMAX_WAIT mbar_wait
#else
#define SOFTMAX_WAIT mbar_wait_sleep
#endif
#ifndef SORT_ATTN_FOLD_AT
#define SORT_ATTN_FOLD_AT 1
#endif
constexpr int kFoldAt = SORT_ATTN_FOLD_AT;  // where the previous tile's O is folded (see loop)
#ifndef SORT_ATTN_MMA_ROWSUM
#define SORT_ATTN_MMA_ROWSUM 0
#endif
// Option (default off: measured equal on the same box, tools/ab_rowsum.sh): row sums of P
// on the tensor core, P * ones[128 x 16] into the tile's free TMEM columns [96, 112) (after
// P(g) is written, S columns 96..127 are consumed), so the softmax warps add no FADDs per
// element and the two half-row warps need no sum exchange.
constexpr bool kMmaRowSum = SORT_ATTN_MMA_ROWSUM != 0;
constexpr int kPolyEvery = SORT_ATTN_POLY_EVERY;  // exp2 offload ratio in fully visible chunks

template <int DK>
struct AttnSmem {
  static constexpr uint32_t kTileBytes = 128 * DK * 2;  // Q, K or V tile (rows of DK*2 bytes)
  static constexpr uint32_t kStride = ((kTileBytes + 1023) / 1024) * 1024;
  static constexpr uint32_t oQ = 0;
  static constexpr uint32_t oK = oQ + 2 * kStride;
  static constexpr uint32_t oV = oK + kKvStages * kStride;
  static constexpr uint32_t oOnes = oV + kKvStages * kStride;  // 16 x 16 bf16 ones, K-major SW32
  static constexpr uint32_t oBar = oOnes + (kMmaRowSum ? 1024 : 0);
  static constexpr uint32_t oRed = oBar + 32 * 8;      // softmax cross-warp reduction scratch
  static constexpr uint32_t oGate = oRed + 3 * 1024;   // [2 items][2 halves][128 rows][DK/2] bf16
  static constexpr uint32_t oTiles = oGate + 2 * 128 * DK * 2;  // int32 tile tables follow
  static constexpr uint32_t bytes(int n_tile_ints) { return oTiles + 4u * n_tile_ints + 1024; }
};

struct AttnArgs {
  const int4* rowmeta;        // [n_qtiles*128] {lo, hi, self, 0} in kv-index space
  const int32_t* tile_off;    // [n_qtiles+1]
  const int2* tile_code;      // {kv_tile, warp chunk classes} (plan.hpp)
  const int32_t* qtile_order; // heavy first
  const __nv_bfloat16* g;     // [B*Rq, d] sigmoid gate
  __nv_bfloat16* out;         // [B*Rq, d]
  __nv_bfloat16* o_pre;       // training: pre-gate output [B*Rq, d] (or null)
  float* lse;                 // training: log2-sum-exp per (b*H + h, row) [BH, Rq] (or null)
  int BH, H, Rq, d, n_qtiles, n_codes;
  float scale_log2;           // log2(e) / sqrt(dk)
  float ref_log2;             // fixed-reference mode: B * scale_log2
};

// Visibility of columns [cs, cs+32) for a row with compact mask (lo, hi, self), as bits.
__device__ __forceinline__ uint32_t chunk_vis_bits(int cs, int lo, int hi, int self_idx) {
  const int a = max(lo - cs, 0), b = min(hi - cs, 31);
  uint32_t bits = b >= a ? ((2u << b) - (1u << a)) : 0u;  // (2u << 31) wraps to 0: still exact
  const int so = self_idx - cs;
  if (so >= 0 && so < 32) bits |= 1u << so;
  return bits;
}

// TMEM plan: DK <= 32 keeps O_g in the free columns of its S buffer (256 columns, 2 CTAs per
// SM); DK = 64 (SORT-large) gives O_g its own 64-column buffers after the two S buffers (512
// columns, 1 CTA per SM).
template <int DK>
struct AttnTmem {
  static constexpr uint32_t kCols = DK <= 32 ? 256 : 512;
  static constexpr int kCtasPerSm = DK <= 32 ? 2 : 1;
  __device__ static constexpr uint32_t o_col(int buf) { return DK <= 32 ? buf * 128 + 32 : 256 + buf * DK; }
};

// kPre (inference, bounded logits only): Q arrives pre-multiplied by log2(e) / sqrt(dk) (folded
// into the QKNorm gain of the QKVG epilogue), so S is already the base-2 exponent and the
// reference is 0: |S| <= B log2 e < 58 keeps every 2^S a normal fp32 / bf16 number, P = 2^S
// needs no FFMA per element and the polynomial exp2 no clamp.
template <int DK, bool kFixed, bool kPre = false>
__global__ void __launch_bounds__(kAttnThreads, AttnTmem<DK>::kCtasPerSm)
    k_attention(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  static_assert(DK == 16 || DK == 32 || DK == 64, "head dim 16, 32 or 64");
  using S = AttnSmem<DK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::oBar);
  uint64_t* q_full = bars + 0;    // [2]
  uint64_t* q_empty = bars + 2;   // [2]
  uint64_t* s_full = bars + 4;    // [2 buffers][2 halves]
  uint64_t* p_full = bars + 8;    // [2 buffers]
  uint64_t* pv_done = bars + 10;  // [2 buffers]
  uint64_t* o_read = bars + 12;   // [2 buffers]
  uint64_t* kv_full = bars + 14;  // [kKvStages]
  uint64_t* kv_empty = kv_full + kKvStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kv_empty + kKvStages);
  int32_t* s_off = reinterpret_cast<int32_t*>(smem + S::oTiles);
  int32_t* s_order = s_off + (a.n_qtiles + 1);
  int2* s_code = reinterpret_cast<int2*>(s_order + a.n_qtiles + 1);  // 2n+2 ints: 8-byte aligned

  const int warp = warp_id(), lane = lane_id();
  const int n_items = a.n_qtiles * a.BH;

  for (int i = threadIdx.x; i <= a.n_qtiles; i += kAttnThreads) s_off[i] = a.tile_off[i];
  for (int i = threadIdx.x; i < a.n_qtiles; i += kAttnThreads) s_order[i] = a.qtile_order[i];
  for (int i = threadIdx.x; i < a.n_codes; i += kAttnThreads) s_code[i] = a.tile_code[i];
  if (kMmaRowSum) {
    for (int i = threadIdx.x; i < 128; i += kAttnThreads)
      reinterpret_cast<uint32_t*>(smem + S::oOnes)[i] = 0x3F803F80u;  // bf16 pair (1, 1)
    fence_proxy_async_smem();  // generic-proxy stores -> tcgen05.mma operand reads
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[2 * i], 1);
      mbar_init(&s_full[2 * i + 1], 1);
      mbar_init(&p_full[i], 256);
      mbar_init(&pv_done[i], 1);
      mbar_init(&o_read[i], 256);
    }
    for (int i = 0; i < kKvStages; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tslot, AttnTmem<DK>::kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  auto tiles_of = [&](int it) {
    const int qt = s_order[it % a.n_qtiles];
    return s_off[qt + 1] - s_off[qt];
  };

  // Work item i -> (request*head bh = i / n_qtiles, q-tile of rank i % n_qtiles, heaviest
  // first). (b,h)-major order keeps the ~2 CTAs x 148 in-flight items on a few dozen (b,h)
  // pairs, so K/V tiles shared by neighbouring q-tiles are re-read from L2, not HBM.
  if (warp == 0) {
    if (lane == 0) {
      int g = 0, li = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
        const int bh = it / a.n_qtiles, rank = it - bh * a.n_qtiles;
        const int qt = s_order[rank];
        const int t_begin = s_off[qt], n_t = s_off[qt + 1] - t_begin;
        const int qb = li & 1;
        mbar_wait_sleep(&q_empty[qb], ((li >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qb], S::kTileBytes);
        tma_load_3d(smem + S::oQ + qb * S::kStride, &tmQ, &q_full[qb], 0, qt * 128, bh);
        for (int j = 0; j < n_t; ++j, ++g) {
          const int st = g % kKvStages;
          const int kv0 = s_code[t_begin + j].x * 128;
          mbar_wait_sleep(&kv_empty[st], ((g / kKvStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&kv_full[st], 2 * S::kTileBytes);
          tma_load_3d(smem + S::oK + st * S::kStride, &tmK, &kv_full[st], 0, kv0, bh);
          tma_load_3d(smem + S::oV + st * S::kStride, &tmV, &kv_full[st], 0, kv0, bh);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = umma_idesc_bf16(128, 64);
      const uint32_t id_o = umma_idesc_bf16(128, DK) | (1u << 16);  // B = V, MN-major
      const uint32_t id_l = umma_idesc_bf16(128, 16);                  // B = ones, K-major
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
      auto issue_s = [&](const Cur& c) {  // S(c.g) into buffer c.g & 1, two N=64 halves
        const int buf = c.g & 1;
        if (c.g >= 2) {  // O of the buffer's previous tile has been read out
          mbar_wait(&o_read[buf], ((c.g >> 1) - 1) & 1);
        }
        if (c.j == 0) mbar_wait(&q_full[c.li & 1], (c.li >> 1) & 1);
        const int st = c.g % kKvStages;
        mbar_wait(&kv_full[st], (c.g / kKvStages) & 1);
        tc_fence_after();
        const uint32_t sq = smem_u32(smem + S::oQ + (c.li & 1) * S::kStride);
        const uint32_t sk = smem_u32(smem + S::oK + st * S::kStride);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
          for (int k = 0; k < DK / 16; ++k)
            mma_bf16_ss(tmem + buf * 128 + hf * 64, umma_sdesc_kmajor(sq + k * 32, sw),
                        umma_sdesc_kmajor(sk + hf * 64 * DK * 2 + k * 32, sw), id_s, k > 0 ? 1u : 0u);
          mma_commit(&s_full[buf * 2 + hf]);
        }
        if (c.j == c.n_t - 1) mma_commit(&q_empty[c.li & 1]);
      };
      Cur cur{static_cast<int>(blockIdx.x), 0, 0, 0, 0};
      cur.n_t = cur.it < n_items ? tiles_of(cur.it) : 0;
      if (cur.it < n_items) issue_s(cur);
      while (cur.it < n_items) {
        const Cur nx = next(cur);
        if (nx.it < n_items) issue_s(nx);  // S(g+1) overlaps the softmax of tile g
        const int buf = cur.g & 1;
        mbar_wait(&p_full[buf], (cur.g >> 1) & 1);  // P(g) written, S(g) consumed
        tc_fence_after();
        const uint32_t tb = tmem + buf * 128;
        const int st = cur.g % kKvStages;
        const uint32_t sv = smem_u32(smem + S::oV + st * S::kStride);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t pa = tb + (kk >> 2) * 64 + (kk & 3) * 8;  // P of half kk/4, K=16 per MMA
          const uint32_t va = sv + kk * 16 * (DK * 2);           // V rows, MN-major, SBO = 8 rows
          mma_bf16_ts(tmem + AttnTmem<DK>::o_col(buf), pa, umma_sdesc_kmajor(va, sw), id_o, kk != 0 ? 1u : 0u);
        }
        if (kMmaRowSum) {  // row sums of P(g): D[m][n] = sum_k P[m][k] for all 16 n
          const uint64_t ones = umma_sdesc_kmajor(smem_u32(smem + S::oOnes), 32);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t pa = tb + (kk >> 2) * 64 + (kk & 3) * 8;
            mma_bf16_ts(tb + 96, pa, ones, id_l, kk != 0 ? 1u : 0u);
          }
        }
        mma_commit(&pv_done[buf]);
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
    const float sl2 = a.scale_log2;
    const float2 sl2v = make_float2(sl2, sl2);
    float* s_red = reinterpret_cast<float*>(smem + S::oRed);  // [2][2][128] maxima, [2][128] sums
    int g = 0, li = 0;
    float m = NEG_INF, alpha_prev = 1.f, alpha_prev_fold = 1.f;  // online mode only
    float2 lsum[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};  // FMA-pipe row sums
    float lacc = 0.f;                                                   // MMA row sums (folded)
    float acc[DH];
#pragma unroll
    for (int i = 0; i < DH; ++i) acc[i] = 0.f;
    // the previous item, finished while the next item's first tile is in flight
    bool p_valid = false;
    size_t p_off = 0, p_lse = 0;
    float p_lsum = 0.f, p_ref = 0.f;
    // acc <- acc * alpha + O_t  (this warp's DK/2 columns of tile t's PV result)
    auto fold_o = [&](int t, float alpha) {
      const int pb = t & 1;
      SOFTMAX_WAIT(&pv_done[pb], (t >> 1) & 1);
      tc_fence_after();
      float o[DH];
      uint32_t ls = 0;
      if (kMmaRowSum)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                     : "=r"(ls) : "r"(tmem + pb * 128 + 96 + lane_off));
      tmem_row_chunk<DH>(tmem + AttnTmem<DK>::o_col(pb) + hf * DH + lane_off, o);
      tc_fence_before();
      mbar_arrive(&o_read[pb]);
#pragma unroll
      for (int i = 0; i < DH; ++i) acc[i] = kFixed ? acc[i] + o[i] : fmaf(acc[i], alpha, o[i]);
      if (kMmaRowSum) lacc = kFixed ? lacc + __uint_as_float(ls) : fmaf(lacc, alpha, __uint_as_float(ls));
    };
    // fold the item's last O (tile t), combine the half-row sums, gate, store, clear acc
    auto finish_item = [&](int t, float alpha, int pli, bool gate_pending) {
      fold_o(t, alpha);
      float l;
      if constexpr (kMmaRowSum) {
        l = lacc;  // both half-row warps fold the same full-row sums
        lacc = 0.f;
      } else {
        float* sl = s_red + 512;  // [2][128] partial row sums
        sl[hf * 128 + r] = p_lsum;
        named_bar_sync(1 + quarter, 64);
        l = sl[r] + sl[128 + r];
        named_bar_sync(1 + quarter, 64);  // both partners read before the next item overwrites
      }
      if (gate_pending) cp_async_wait_1(); else cp_async_wait_all();
      if (p_valid) {
        const uint8_t* gs = smem + S::oGate + ((pli & 1) * 256 + hf * 128 + r) * (DH * 2);
        const float invl = 1.f / l;
        if (a.lse) {  // training outputs: P = exp2(s * scale_log2 - lse2), pre-gate O
          if (hf == 0) a.lse[p_lse] = p_ref + log2f(l);
          uint32_t wo[DH / 2];
#pragma unroll
          for (int i = 0; i < DH / 2; ++i) wo[i] = pack_bf16x2(acc[2 * i] * invl, acc[2 * i + 1] * invl);
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
            w[4 * i + e] = pack_bf16x2(acc[8 * i + 2 * e] * invl * gf.x, acc[8 * i + 2 * e + 1] * invl * gf.y);
          }
        }
        if constexpr (DH == 16) {
          stg256(a.out + p_off, w);  // the warp half's 32-byte output sector
        } else {
#pragma unroll
          for (int i = 0; i < DH / 8; ++i)
            reinterpret_cast<int4*>(a.out + p_off)[i] = make_int4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        }
      }
#pragma unroll
      for (int i = 0; i < DH; ++i) acc[i] = 0.f;
    };
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
      const int bh = it / a.n_qtiles, rank = it - bh * a.n_qtiles;
      const int qt = s_order[rank];
      const int q0 = qt * 128;
      const int t_begin = s_off[qt], n_t = s_off[qt + 1] - t_begin;
      const int4 meta = a.rowmeta[q0 + r];
      const int qrow = q0 + r;
      const int b = bh / a.H, hh = bh - b * a.H;
      const size_t off = static_cast<size_t>(b * a.Rq + qrow) * a.d + hh * DK + hf * DH;
      // gate row prefetched into smem (async; slot by item parity, the previous item's
      // gate is still unread until its epilogue runs inside this item's first tile)
      uint8_t* gslot = smem + S::oGate + ((li & 1) * 256 + hf * 128 + r) * (DH * 2);
      if (qrow < a.Rq) {
#pragma unroll
        for (int i = 0; i < DH / 8; ++i) cp_async_16(gslot + 16 * i, a.g + off + 8 * i);
      }
      cp_async_commit();
      const bool has_prev = li > 0;
      if (has_prev) {  // this item's row sums start from zero; keep the previous item's
        p_lsum = (lsum[0].x + lsum[0].y) + (lsum[1].x + lsum[1].y);
        p_ref = kPre ? 0.f : (kFixed ? a.ref_log2 : (m == NEG_INF ? 0.f : m * sl2));
        lsum[0] = lsum[1] = make_float2(0.f, 0.f);
      }
      m = NEG_INF;
      for (int j = 0; j < n_t; ++j, ++g) {
        const int buf = g & 1;
        const uint32_t tSh = tmem + buf * 128 + hf * 64 + lane_off;  // this warp's S half (and P)
        const int2 code = s_code[t_begin + j];
        const int c0 = code.x * 128 + hf * 64;  // first kv column of this half
        // this warp's two 32-column chunks: classes from the host plan (full / none / mixed)
        const uint32_t cls = static_cast<uint32_t>(code.y) >> (2 * (4 * quarter + 2 * hf));
        const uint32_t full_mask = (cls & 1u) | ((cls >> 1) & 2u);
        const uint32_t none_mask = ((cls >> 1) & 1u) | ((cls >> 2) & 2u);
        SOFTMAX_WAIT(&s_full[buf * 2 + hf], (g >> 1) & 1);
        tc_fence_after();
        float ref;  // exp2 reference in the scaled domain
        if constexpr (kPre) {
          ref = 0.f;
        } else if constexpr (kFixed) {
          ref = a.ref_log2;
        } else {
          float mx4[4] = {NEG_INF, NEG_INF, NEG_INF, NEG_INF};
#pragma unroll
          for (int cb = 0; cb < 2; ++cb) {
            if (none_mask & (1u << cb)) continue;
            uint32_t rr[32];
            tmem_ld_32x32b_x32(tSh + cb * 32, rr);
            tmem_ld_wait();
            const uint32_t bits = (full_mask & (1u << cb)) ? 0xffffffffu
                                                           : chunk_vis_bits(c0 + cb * 32, meta.x, meta.y, meta.z);
#pragma unroll
            for (int i = 0; i < 32; ++i)
              mx4[i & 3] = fmaxf(mx4[i & 3], (bits >> i) & 1u ? __uint_as_float(rr[i]) : NEG_INF);
          }
          // combine the two halves' maxima (double-buffered slot by tile parity)
          float* slot = s_red + (g & 1) * 256;
          slot[hf * 128 + r] = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
          named_bar_sync(1 + quarter, 64);
          const float m_new = fmaxf(m, fmaxf(slot[r], slot[128 + r]));
          ref = m_new == NEG_INF ? 0.f : m_new * sl2;
          const float alpha = ex2_approx(m * sl2 - ref);  // m = -inf -> 0
#pragma unroll
          for (int u = 0; u < 2; ++u)
            if (!kMmaRowSum) lsum[u] = make_float2(lsum[u].x * alpha, lsum[u].y * alpha);
          alpha_prev_fold = alpha_prev;  // alpha of tile g-1, used by the fold inside this tile
          alpha_prev = alpha;  // applied to acc when O of this tile is folded in (next tile / end)
          m = m_new;
        }
        const float2 nref = make_float2(-ref, -ref);
        // Fold O of the previous tile (kFoldAt: 0 before the first chunk, 1 between the two
        // chunks, 2 after both). On an item's first tile that O is the previous item's last:
        // finish that item here.
        auto fold_prev = [&]() {
          if (j > 0) {
            fold_o(g - 1, alpha_prev_fold);
          } else if (has_prev) {
            finish_item(g - 1, alpha_prev_fold, li - 1, true);
          }
        };
        if (kFoldAt == 0) fold_prev();
#pragma unroll
        for (int cb = 0; cb < 2; ++cb) {
          uint32_t w[16];
          if (none_mask & (1u << cb)) {
#pragma unroll
            for (int i = 0; i < 16; ++i) w[i] = 0u;
          } else {
            uint32_t rr[32];
            tmem_ld_32x32b_x32(tSh + cb * 32, rr);
            tmem_ld_wait();
            if (full_mask & (1u << cb)) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float2 s2 = make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1]));
                const float2 x = kPre ? s2 : ffma2(s2, sl2v, nref);
                // every kPolyEvery-th pair on the FMA pipe, the rest on MUFU
                const float2 p = (kPolyEvery > 0 && i % kPolyEvery == kPolyEvery - 1)
                                     ? (kPre ? ex2_poly2_nc(x) : ex2_poly2(x))
                                     : make_float2(ex2_approx(x.x), ex2_approx(x.y));
                if (!kMmaRowSum) lsum[i & 1] = fadd2(lsum[i & 1], p);
                w[i] = pack_bf16x2(p.x, p.y);
              }
            } else {
              const uint32_t bits = chunk_vis_bits(c0 + cb * 32, meta.x, meta.y, meta.z);
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float2 s2 = make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1]));
                float2 x = kPre ? s2 : ffma2(s2, sl2v, nref);
                x.x = (bits >> (2 * i)) & 1u ? x.x : NEG_INF;
                x.y = (bits >> (2 * i + 1)) & 1u ? x.y : NEG_INF;
                const float2 p = make_float2(ex2_approx(x.x), ex2_approx(x.y));
                if (!kMmaRowSum) lsum[i & 1] = fadd2(lsum[i & 1], p);
                w[i] = pack_bf16x2(p.x, p.y);
              }
            }
          }
          // P of columns [cb*32, +32) of this half -> 16 bf16x2 columns, in place over S
          tmem_st_32x32b_x16(tSh + cb * 16, w);
          // Default: fold between the two chunks: its PV has had a full chunk to finish, and
          // releasing its buffer now still gives QK^T(g+1) half a tile of lead.
          if (kFoldAt == 1 && cb == 0) fold_prev();
        }
        if (kFoldAt == 2) fold_prev();
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[buf]);
      }
      p_valid = qrow < a.Rq;
      p_off = off;
      p_lse = static_cast<size_t>(bh) * a.Rq + qrow;
    }  // item loop
    if (li > 0) {  // the last item
      p_lsum = (lsum[0].x + lsum[0].y) + (lsum[1].x + lsum[1].y);
      p_ref = kPre ? 0.f : (kFixed ? a.ref_log2 : (m == NEG_INF ? 0.f : m * sl2));
      finish_item(g - 1, alpha_prev, li - 1, false);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, AttnTmem<DK>::kCols);
  }
}

}  // namespace sortk
