// SPDX-License-Identifier: Apache-2.0
// Attention-core backward on tcgen05 (AttentionLayer::backward, attention.cpp:158-183: the
// softmax backward dS = P (dP - D) with D = rowsum(dO O), then dQ = dS K, dK = dS^T Q,
// dV = P^T dO, all scaled as attention.cpp:175-176).
//
// Two deterministic passes over the same saved inputs (bf16 rotated Q/K, V, dO; per query row
// the log2-sum-exp `lse` of the forward and D), each the structure of the forward kernel --
// one work item = one 128-row block X of one (request, head), a loop over the 64-row blocks Y
// of the other side that share a visible entry with it (host lists), per step two tcgen05
// MMAs into TMEM, an elementwise pass by 8 warps, one or two accumulating TS-form MMAs:
//
//   kDQ = false (X = kv block, Y = q block):  S^T = K Q^T, dP^T = V dO^T      [128 x 64]
//       P^T = exp2(S^T log2e/sqrt(dk) - lse_q), dS^T = P^T (dP^T - D_q)
//       dV += P^T dO,  dK += dS^T Q        (A = P^T / dS^T from TMEM, B = dO / Q MN-major)
//   kDQ = true  (X = q block, Y = kv block):  S = Q K^T, dP = dO V^T
//       dS = P (dP - D),  dQ += dS K
// P is recomputed in both passes (one more exponential per visible entry than a single pass
// with fp32 atomics on dQ); in exchange no partial sums race, so gradients are bit-identical
// from run to run. The mask comes from the compact rows (lo, hi, self) of the query rows
// (mask.cpp:47-74): per 32 x 32 chunk the host classifies full / none / mixed, and mixed chunks
// test each element.
//
// TMEM (256 columns, 2 CTAs per SM): S [0, 64), dP [64, 128) fp32 -> each half's P^T / dS as
// bf16 pairs in place over the first 16 of its own 32 columns, accumulators from column 128
// (dQ; or dV then dK).
// Roles (320 threads): warp 0 TMA (the item's two X tiles double-buffered, the Y tiles
// through a ring), warp 1 MMA, warps 2..9 elementwise: warp pair (w, w+4) shares lane quarter
// w % 4 (32 X rows) and splits the 64 Y columns in halves.
#pragma once

#include "attention.cuh"

namespace sortk {

constexpr int kBwdStages = 4;

template <int DK>
struct BwdSmem {
  static constexpr uint32_t kX = 128 * DK * 2;  // one 128-row X tile
  static constexpr uint32_t kXs = ((kX + 1023) / 1024) * 1024;
  static constexpr uint32_t kY = 64 * DK * 2;   // one 64-row Y tile
  static constexpr uint32_t kYs = ((kY + 1023) / 1024) * 1024;
  static constexpr uint32_t oX = 0;                          // [2 items][2 tiles]
  static constexpr uint32_t oY = oX + 4 * kXs;               // [kBwdStages][2 tiles]
  static constexpr uint32_t oBar = oY + 2 * kBwdStages * kYs;
  static constexpr uint32_t oStat = oBar + 32 * 8;    // [8 warps][lse 32 | D 32] fp32 (pass 1)
  static constexpr uint32_t oTiles = oStat + 8 * 256;
  static constexpr uint32_t bytes(int n_tile_ints) { return oTiles + 4u * n_tile_ints + 1024; }
};

struct AttnBwdTcArgs {
  const int4* rowmeta;       // [Rq] compact mask rows of the query rows (kv index space)
  const int4* kvmeta;        // pass 1 (optional): per kv row the query rows that see it, as two
                             // intervals {lo1, hi1, lo2, hi2} (the transposed compact mask)
  const int32_t* x_off;      // [nX + 1] CSR: X block -> its Y steps
  const int2* y_code;        // {Y block (64 rows), chunk classes (2 bits per (quarter, half))}
  const float* lse;          // [BH, Rq] log2-domain
  const float* D;            // [BH, Rq]
  float* out0;               // kDQ: dq; else dk   (token-major fp32 [B*R, H*DK])
  float* out1;               // dv (kDQ: unused; may be null when only out1_16 is wanted)
  __nv_bfloat16* out1_16;    // optional bf16 copy of dv
  int BH, H, Rq, Rkv, nX;
  float scale_log2, scale;
};

template <int DK, bool kDQ>
__global__ void __launch_bounds__(kAttnThreads, 2)
    k_attn_bwd_tc(const __grid_constant__ CUtensorMap tmX0, const __grid_constant__ CUtensorMap tmX1,
                  const __grid_constant__ CUtensorMap tmY0, const __grid_constant__ CUtensorMap tmY1,
                  const AttnBwdTcArgs a) {
  static_assert(DK == 16 || DK == 32 || DK == 64, "head dim 16, 32 or 64");
  using S = BwdSmem<DK>;
  constexpr uint32_t kAcc0 = 128, kAcc1 = 128 + DK;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::oBar);
  uint64_t* x_full = bars + 0;     // [2]
  uint64_t* x_empty = bars + 2;    // [2]
  uint64_t* s_full = bars + 4;     // [1] S and dP of the step
  uint64_t* p_full = bars + 5;     // [1] P / dS written (256)
  uint64_t* acc_done = bars + 6;   // [1] the item's accumulators complete
  uint64_t* acc_free = bars + 7;   // [1] accumulators read out (256)
  uint64_t* y_full = bars + 8;     // [kBwdStages]
  uint64_t* y_empty = y_full + kBwdStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(y_empty + kBwdStages);
  int32_t* s_off = reinterpret_cast<int32_t*>(smem + S::oTiles);
  int2* s_code = reinterpret_cast<int2*>(s_off + ((a.nX + 2) & ~1));

  const int warp = warp_id(), lane = lane_id();
  const int n_items = a.nX * a.BH;
  const int n_codes = 0;
  (void)n_codes;
  for (int i = threadIdx.x; i <= a.nX; i += kAttnThreads) s_off[i] = a.x_off[i];
  __syncthreads();
  for (int i = threadIdx.x; i < s_off[a.nX]; i += kAttnThreads) s_code[i] = a.y_code[i];
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX0);
    tma_prefetch_desc(&tmX1);
    tma_prefetch_desc(&tmY0);
    tma_prefetch_desc(&tmY1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&x_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 256);
    mbar_init(acc_done, 1);
    mbar_init(acc_free, 256);
    for (int i = 0; i < kBwdStages; ++i) {
      mbar_init(&y_full[i], 1);
      mbar_init(&y_empty[i], 1);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // tensor-map coordinates of a 128-row X block / 64-row Y block of (b, h): head-major maps
  // are {dk, row, bh}; the token-major dO map is {dk, h, row, b}
  auto load_tile = [&](void* dst, const CUtensorMap* m, uint64_t* bar, bool token_major, int row0, int bh) {
    if (token_major) {
      const int b = bh / a.H, h = bh - b * a.H;
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
          "%6}], [%2];" ::"r"(smem_u32(dst)),
          "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(0), "r"(h), "r"(row0), "r"(b)
          : "memory");
    } else {
      tma_load_3d(dst, m, bar, 0, row0, bh);
    }
  };
  // which of the four maps are token-major (dO): kDQ: X1 = dO; else Y1 = dO
  constexpr bool kX1Tok = kDQ, kY1Tok = !kDQ;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int g = 0, li = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
        const int bh = it / a.nX, xb = it - bh * a.nX;
        const int xs = li & 1;
        mbar_wait(&x_empty[xs], ((li >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&x_full[xs], 2 * S::kX);
        load_tile(smem + S::oX + (2 * xs) * S::kXs, &tmX0, &x_full[xs], false, xb * 128, bh);
        load_tile(smem + S::oX + (2 * xs + 1) * S::kXs, &tmX1, &x_full[xs], kX1Tok, xb * 128, bh);
        for (int j = s_off[xb]; j < s_off[xb + 1]; ++j, ++g) {
          const int st = g % kBwdStages;
          const int y0 = s_code[j].x * 64;
          mbar_wait(&y_empty[st], ((g / kBwdStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&y_full[st], 2 * S::kY);
          load_tile(smem + S::oY + (2 * st) * S::kYs, &tmY0, &y_full[st], false, y0, bh);
          load_tile(smem + S::oY + (2 * st + 1) * S::kYs, &tmY1, &y_full[st], kY1Tok, y0, bh);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t id_s = umma_idesc_bf16(128, 64);
      const uint32_t id_a = umma_idesc_bf16(128, DK) | (1u << 16);  // B operand MN-major
      constexpr uint32_t sw = DK * 2;
      int g = 0, li = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
        const int xb = it % a.nX;
        const int xs = li & 1;
        const int j0 = s_off[xb], j1 = s_off[xb + 1];
        mbar_wait(&x_full[xs], (li >> 1) & 1);
        const uint32_t sx0 = smem_u32(smem + S::oX + (2 * xs) * S::kXs);
        const uint32_t sx1 = smem_u32(smem + S::oX + (2 * xs + 1) * S::kXs);
        for (int j = j0; j < j1; ++j, ++g) {
          const int st = g % kBwdStages;
          mbar_wait(&y_full[st], (g / kBwdStages) & 1);
          tc_fence_after();
          const uint32_t sy0 = smem_u32(smem + S::oY + (2 * st) * S::kYs);
          const uint32_t sy1 = smem_u32(smem + S::oY + (2 * st + 1) * S::kYs);
          // S = X0 Y0^T and dP = X1 Y1^T (issued behind the previous step's accumulating MMAs,
          // which read the bf16 P / dS over these columns: the tensor pipe keeps issue order)
#pragma unroll
          for (int k = 0; k < DK / 16; ++k) {
            mma_bf16_ss(tmem, umma_sdesc_kmajor(sx0 + k * 32, sw), umma_sdesc_kmajor(sy0 + k * 32, sw), id_s,
                        k > 0 ? 1u : 0u);
            mma_bf16_ss(tmem + 64, umma_sdesc_kmajor(sx1 + k * 32, sw), umma_sdesc_kmajor(sy1 + k * 32, sw), id_s,
                        k > 0 ? 1u : 0u);
          }
          mma_commit(s_full);
          if (j == j1 - 1) mma_commit(&x_empty[xs]);  // X tiles no longer needed by this item
          mbar_wait(p_full, g & 1);
          // the first accumulating MMA of an item overwrites the accumulators: the previous
          // item's must have been read out
          if (j == j0 && li > 0) mbar_wait(acc_free, (li - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // K = 64 Y rows, 16 per MMA
            const uint32_t acc = (j > j0 || kk > 0) ? 1u : 0u;
            // bf16 pairs of Y columns [16 kk, 16 kk + 16): half kk / 2 wrote them at the start of
            // its own 32 S (or dP) columns
            const uint32_t pa = (kk >> 1) * 32 + (kk & 1) * 8;
            if constexpr (kDQ) {
              // dQ += dS K_y   (A = dS from TMEM, B = K tile [64 x DK] MN-major)
              mma_bf16_ts(tmem + kAcc0, tmem + pa, umma_sdesc_kmajor(sy0 + kk * 16 * (DK * 2), sw), id_a, acc);
            } else {
              // dV += P^T dO_y, dK += dS^T Q_y
              mma_bf16_ts(tmem + kAcc0, tmem + pa, umma_sdesc_kmajor(sy1 + kk * 16 * (DK * 2), sw), id_a, acc);
              mma_bf16_ts(tmem + kAcc1, tmem + 64 + pa, umma_sdesc_kmajor(sy0 + kk * 16 * (DK * 2), sw), id_a, acc);
            }
          }
          mma_commit(&y_empty[st]);
          if (j == j1 - 1) mma_commit(acc_done);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ elementwise warps
    const int quarter = warp & 3;
    const int hf = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;  // X row within the block == TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const float NEG_INF = -__int_as_float(0x7f800000);
    const float sl2 = a.scale_log2;
    int g = 0, li = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
      const int bh = it / a.nX, xb = it - bh * a.nX;
      const int b = bh / a.H, hh = bh - b * a.H;
      const int x = xb * 128 + r;  // this thread's X row (q row in kDQ, kv row otherwise)
      int4 meta = make_int4(0, -1, -1, 0);
      float lse_r = 0.f, D_r = 0.f;
      if constexpr (kDQ) {
        if (x < a.Rq) {
          meta = a.rowmeta[x];
          lse_r = a.lse[static_cast<size_t>(bh) * a.Rq + x];
          D_r = a.D[static_cast<size_t>(bh) * a.Rq + x];
        }
      }
      int4 kvm = make_int4(0, -1, 0, -1);  // pass 1: query rows seeing this thread's kv row x
      if constexpr (!kDQ) {
        if (a.kvmeta && x < a.Rkv) kvm = a.kvmeta[x];
      }
      const float* lse_bh = a.lse + static_cast<size_t>(bh) * a.Rq;
      const float* D_bh = a.D + static_cast<size_t>(bh) * a.Rq;
      const int j0 = s_off[xb], j1 = s_off[xb + 1];
      for (int j = j0; j < j1; ++j, ++g) {
        const int2 code = s_code[j];
        const int c0 = code.x * 64 + hf * 32;  // first Y row (column of S) of this warp's half
        const uint32_t cls = (static_cast<uint32_t>(code.y) >> (2 * (2 * quarter + hf))) & 3u;
        // kDQ = false: the half's 32 columns are query rows; lane i fetches column c0 + i's lse, D
        // (and mask row for a mixed chunk) BEFORE the wait, so the loads overlap the MMAs; the
        // column loop broadcasts them with shuffles. Out-of-range columns: lse = +inf -> P = 0.
        float lse_l = __int_as_float(0x7f800000), D_l = 0.f;
        int4 m_l = make_int4(0, -1, -1, 0);
        if constexpr (!kDQ) {
          const int c = c0 + lane;
          if (cls != 2u && c < a.Rq) {
            lse_l = __ldg(lse_bh + c);
            D_l = __ldg(D_bh + c);
            if (cls != 1u && !a.kvmeta) m_l = __ldg(a.rowmeta + c);
          }
        }
        mbar_wait(s_full, g & 1);
        tc_fence_after();
        uint32_t sv[32], pv[32];
        if (cls != 2u) {
          tmem_ld_32x32b_x32(tmem + hf * 32 + lane_off, sv);
          tmem_ld_32x32b_x32(tmem + 64 + hf * 32 + lane_off, pv);
          tmem_ld_wait();
        }
        uint32_t wp[16], wd[16];  // bf16 pairs: P (or dS in kDQ) and dS^T
        if (cls == 2u) {
#pragma unroll
          for (int i = 0; i < 16; ++i) wp[i] = wd[i] = 0u;
        } else if constexpr (kDQ) {
          uint32_t bits = 0xffffffffu;
          if (cls != 1u) bits = chunk_vis_bits(c0, meta.x, meta.y, meta.z);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float p0 = ex2_approx(fmaf(__uint_as_float(sv[2 * i]), sl2, -lse_r));
            float p1 = ex2_approx(fmaf(__uint_as_float(sv[2 * i + 1]), sl2, -lse_r));
            p0 = (bits >> (2 * i)) & 1u ? p0 : 0.f;
            p1 = (bits >> (2 * i + 1)) & 1u ? p1 : 0.f;
            wp[i] = pack_bf16x2(p0 * (__uint_as_float(pv[2 * i]) - D_r), p1 * (__uint_as_float(pv[2 * i + 1]) - D_r));
          }
        } else if (a.kvmeta) {
          // column c = query row: its lse / D are warp-uniform; broadcast from this warp's shared
          // slot four columns per LDS.128, the mask from the thread's own transposed rows
          float* st = reinterpret_cast<float*>(smem + S::oStat) + (warp - 2) * 64;
          st[lane] = lse_l;
          st[32 + lane] = D_l;
          __syncwarp();
          const uint32_t bits = cls == 1u ? 0xffffffffu
                                          : (chunk_vis_bits(c0, kvm.x, kvm.y, -1) | chunk_vis_bits(c0, kvm.z, kvm.w, -1));
          const uint32_t sl_a = smem_u32(st), sd_a = sl_a + 128;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 l4 = lds_f32x4(sl_a + 4 * i), d4 = lds_f32x4(sd_a + 4 * i);
            const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dv[4] = {d4.x, d4.y, d4.z, d4.w};
            float pp[4], dd[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float p = ex2_approx(fmaf(__uint_as_float(sv[i + e]), sl2, -lv[e]));
              p = (bits >> (i + e)) & 1u ? p : 0.f;
              pp[e] = p;
              dd[e] = p * (__uint_as_float(pv[i + e]) - dv[e]);
            }
            wp[i >> 1] = pack_bf16x2(pp[0], pp[1]);
            wp[(i >> 1) + 1] = pack_bf16x2(pp[2], pp[3]);
            wd[i >> 1] = pack_bf16x2(dd[0], dd[1]);
            wd[(i >> 1) + 1] = pack_bf16x2(dd[2], dd[3]);
          }
          __syncwarp();  // the slot is rewritten at the next step
        } else {
          // column c = query row: lse, D (and for mixed chunks its mask row) are warp-uniform
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            float pp[2], dd[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const float l = __shfl_sync(0xffffffffu, lse_l, i + e);
              const float dq = __shfl_sync(0xffffffffu, D_l, i + e);
              float p = ex2_approx(fmaf(__uint_as_float(sv[i + e]), sl2, -l));
              if (cls != 1u) {
                const int mx = __shfl_sync(0xffffffffu, m_l.x, i + e), my = __shfl_sync(0xffffffffu, m_l.y, i + e),
                          mz = __shfl_sync(0xffffffffu, m_l.z, i + e);
                const bool vis = (x >= mx && x <= my) || x == mz;
                p = vis ? p : 0.f;
              }
              pp[e] = p;
              dd[e] = p * (__uint_as_float(pv[i + e]) - dq);
            }
            wp[i >> 1] = pack_bf16x2(pp[0], pp[1]);
            wd[i >> 1] = pack_bf16x2(dd[0], dd[1]);
          }
        }
        (void)NEG_INF;
        // in place over this half's own (already loaded) S / dP columns
        tmem_st_32x32b_x16(tmem + hf * 32 + lane_off, wp);
        if constexpr (!kDQ) tmem_st_32x32b_x16(tmem + 64 + hf * 32 + lane_off, wd);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(p_full);
      }
      // ---- item end: read the accumulators, scale, store
      mbar_wait(acc_done, li & 1);
      tc_fence_after();
      constexpr int DH = DK / 2;  // this warp's half of the accumulator columns
      float o0[DH];
      tmem_row_chunk<DH>(tmem + kAcc0 + hf * DH + lane_off, o0);
      float o1[DH];
      if constexpr (!kDQ) tmem_row_chunk<DH>(tmem + kAcc1 + hf * DH + lane_off, o1);
      tc_fence_before();
      mbar_arrive(acc_free);
      const int Rx = kDQ ? a.Rq : a.Rkv;
      if (x < Rx) {
        const size_t o = (static_cast<size_t>(b) * Rx + x) * a.H * DK + hh * DK + hf * DH;
        if constexpr (kDQ) {
#pragma unroll
          for (int i = 0; i < DH; i += 4)
            *reinterpret_cast<float4*>(a.out0 + o + i) =
                make_float4(o0[i] * a.scale, o0[i + 1] * a.scale, o0[i + 2] * a.scale, o0[i + 3] * a.scale);
        } else {
#pragma unroll
          for (int i = 0; i < DH; i += 4) {
            *reinterpret_cast<float4*>(a.out0 + o + i) =
                make_float4(o1[i] * a.scale, o1[i + 1] * a.scale, o1[i + 2] * a.scale, o1[i + 3] * a.scale);
            if (a.out1) *reinterpret_cast<float4*>(a.out1 + o + i) = make_float4(o0[i], o0[i + 1], o0[i + 2], o0[i + 3]);
          }
          if (a.out1_16) {
#pragma unroll
            for (int i = 0; i < DH; i += 2)
              *reinterpret_cast<uint32_t*>(a.out1_16 + o + i) = pack_bf16x2(o0[i], o0[i + 1]);
          }
        }
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
