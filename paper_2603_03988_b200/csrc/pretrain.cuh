// SPDX-License-Identifier: Apache-2.0
// Generative pre-training head: next-item logits tied to the item table.
//
//   h_t   = RMSNorm(x_t; final_norm.gain) . pretrain.proj          [T, K]  (K = item_dim)
//   z_t[v] = h_t . item_table[v]                                    over the full vocabulary
//   lse_t = log sum_v exp z_t[v],  target_t = z_t[click_t]          (CE_t = lse_t - target_t)
//
// k_pretrain_proj: one warp per token row (final norm in fp32, projection from a shared-memory
//   copy of pretrain.proj, bf16 h_t, the target logit from the bf16 h_t and the target row).
// k_ce_tied: the [T, K] x [K, V] logit GEMM never reaches HBM: each CTA holds 128 rows of h
//   as mma.sync A fragments, streams the item table through a cp.async double buffer in
//   64-item tiles and folds every logit into a per-row online log-sum-exp (exp2 domain), the
//   way attention folds QK^T without materialising it.
#pragma once

#include "attention.cuh"
#include "train.cuh"

namespace sortk {

constexpr int kPreK = 32;          // item_dim of the tied head
constexpr int kCeRows = 128;       // rows per CTA (4 warps x 32)
constexpr int kCeThreads = 128;
constexpr int kCeItems = 64;       // items per streamed tile
constexpr int kCePitch = 80;       // smem bytes per item row (64 + 16: conflict-free fragments)

// One warp per row r = b * L + t of the final residual stream.
__global__ void __launch_bounds__(256) k_pretrain_proj(const __nv_bfloat16* __restrict__ x, int T, int L, int d,
                                                       const float* __restrict__ gain, const float* __restrict__ proj,
                                                       const __nv_bfloat16* __restrict__ items,
                                                       const int32_t* __restrict__ click_item,
                                                       __nv_bfloat16* __restrict__ hp, float* __restrict__ tgt) {
  extern __shared__ float smem_f[];
  float* sW = smem_f;                                        // [d][K]
  float* sx = smem_f + d * kPreK + (threadIdx.x >> 5) * d;   // this warp's normalised row
  for (int i = threadIdx.x; i < d * kPreK; i += blockDim.x) sW[i] = proj[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int c0 = lane * 8;
  const bool act = c0 < d;
  const int n = L - 1;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < T; r += warps) {
    float v[8];
    if (act) {
      const int4 raw = *reinterpret_cast<const int4*>(x + static_cast<size_t>(r) * d + c0);
      const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(p2[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = 0.f;
    }
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) ss = fmaf(v[i], v[i], ss);
    const float inv = rsqrtf(warp_sum(ss) / static_cast<float>(d) + 1e-6f);  // norm.hpp:23-24
    if (act) {
#pragma unroll
      for (int i = 0; i < 8; ++i) sx[c0 + i] = v[i] * inv * gain[c0 + i];
    }
    __syncwarp();
    float a4[4] = {0.f, 0.f, 0.f, 0.f};  // lane j: h_j = sum_c xh[c] W[c][j], 4 independent chains
    for (int c = 0; c < d; c += 4) {
      const float4 xv = *reinterpret_cast<const float4*>(sx + c);
      a4[0] = fmaf(xv.x, sW[(c + 0) * kPreK + lane], a4[0]);
      a4[1] = fmaf(xv.y, sW[(c + 1) * kPreK + lane], a4[1]);
      a4[2] = fmaf(xv.z, sW[(c + 2) * kPreK + lane], a4[2]);
      a4[3] = fmaf(xv.w, sW[(c + 3) * kPreK + lane], a4[3]);
    }
    const float a = (a4[0] + a4[1]) + (a4[2] + a4[3]);
    __syncwarp();
    const __nv_bfloat16 hb = __float2bfloat16_rn(a);
    hp[static_cast<size_t>(r) * kPreK + lane] = hb;
    const int b = r / L, t = r - b * L;
    if (t < n) {  // position t predicts click t
      const int item = click_item[static_cast<size_t>(b) * n + t];
      float z = __bfloat162float(hb) * __bfloat162float(items[static_cast<size_t>(item) * kPreK + lane]);
      z = warp_sum(z);
      if (lane == 0) tgt[static_cast<size_t>(b) * n + t] = z;
    }
  }
}

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
  const uint32_t s = smem_u32(dst);
  const int n = pred ? 16 : 0;  // src-size 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(src), "r"(n) : "memory");
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// lse[b, t] over the full vocabulary for the rows of 128-row block blockIdx.x. 4 warps x 32 rows
// (two m16 tiles share every B fragment); B fragments by ldmatrix.x4 (one per 8-item n-tile
// covering both k16 steps); per row slot an online (max, sum) in natural-log units.
__global__ void __launch_bounds__(kCeThreads) k_ce_tied(const __nv_bfloat16* __restrict__ hp, int T, int L,
                                                        const __nv_bfloat16* __restrict__ items, int V,
                                                        float* __restrict__ lse) {
  __shared__ __align__(16) uint8_t sB[2][kCeItems * kCePitch];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int row0 = blockIdx.x * kCeRows + warp * 32;
  uint32_t a[2][2][4];  // A fragments: 2 m16 tiles x 2 k16 steps (K = 32)
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = row0 + mt * 16 + g + ((q & 1) ? 8 : 0);
        const int k = ks * 16 + 2 * tq + ((q & 2) ? 8 : 0);
        a[mt][ks][q] = r < T ? *reinterpret_cast<const uint32_t*>(hp + static_cast<size_t>(r) * kPreK + k) : 0u;
      }
  const int n_tiles = (V + kCeItems - 1) / kCeItems;
  auto stage = [&](int tile, int buf) {
    // 64 items x 64 B = 256 16-byte chunks, 2 per thread
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int ch = threadIdx.x + i * kCeThreads;
      const int it = ch >> 2, part = ch & 3;
      const int v = tile * kCeItems + it;
      cp_async16(sB[buf] + it * kCePitch + part * 16,
                 items + static_cast<size_t>(v < V ? v : 0) * kPreK + part * 8, v < V);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  constexpr float kLog2e = 1.4426950408889634f;
  float m[4], s[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    m[i] = -INFINITY;
    s[i] = 0.f;
  }
  // ldmatrix row address of this lane: matrix lane / 8 = k block, row lane % 8 = item
  const uint32_t lm_off = static_cast<uint32_t>((lane & 7) * kCePitch + (lane >> 3) * 16);
  stage(0, 0);
  for (int tile = 0; tile < n_tiles; ++tile) {
    const int buf = tile & 1;
    if (tile + 1 < n_tiles) {
      stage(tile + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    float c[2][8][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) c[mt][nt][q] = 0.f;
    const uint32_t sb = smem_u32(sB[buf]) + lm_off;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      uint32_t b[4];
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                   : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3])
                   : "r"(sb + nt * 8 * kCePitch));
      mma_bf16_16816(c[0][nt], a[0][0], b[0], b[1]);
      mma_bf16_16816(c[1][nt], a[1][0], b[0], b[1]);
      mma_bf16_16816(c[0][nt], a[0][1], b[2], b[3]);
      mma_bf16_16816(c[1][nt], a[1][1], b[2], b[3]);
    }
    __syncthreads();  // buffer `buf` is restaged two tiles later
    if (tile == n_tiles - 1) {  // vocabulary tail: columns >= V never count
      const int vbase = tile * kCeItems + 2 * tq;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (vbase + nt * 8 + (q & 1) >= V) c[mt][nt][q] = -INFINITY;
    }
#pragma unroll
    for (int slot = 0; slot < 4; ++slot) {
      const int mt = slot >> 1, hf = slot & 1;
      float z[16];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        z[2 * nt] = c[mt][nt][hf * 2];
        z[2 * nt + 1] = c[mt][nt][hf * 2 + 1];
      }
      float mx[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) mx[i] = fmax3(z[4 * i], z[4 * i + 1], fmaxf(z[4 * i + 2], z[4 * i + 3]));
      const float zmax = fmax3(mx[0], mx[1], fmaxf(mx[2], mx[3]));
      const float mn = fmaxf(m[slot], zmax);
      if (mn == -INFINITY) continue;  // no valid column seen yet (V < 64 tails)
      const float ms = mn * kLog2e;
      float2 acc0 = make_float2(m[slot] == -INFINITY ? 0.f : s[slot] * ex2_approx(fmaf(m[slot], kLog2e, -ms)), 0.f);
      float2 acc1 = make_float2(0.f, 0.f);
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const float2 arg = ffma2(make_float2(z[2 * nt], z[2 * nt + 1]), make_float2(kLog2e, kLog2e),
                                 make_float2(-ms, -ms));
        float2 e;
        if (nt == 7) {  // 1 of 8 pairs on the FMA pipe
          e = ex2_poly2(arg);
        } else {
          e.x = ex2_approx(arg.x);
          e.y = ex2_approx(arg.y);
        }
        if (nt & 1) acc1 = fadd2(acc1, e);
        else acc0 = fadd2(acc0, e);
      }
      m[slot] = mn;
      s[slot] = (acc0.x + acc1.x) + (acc0.y + acc1.y);
    }
  }
  // combine the 4 threads of a quad (same rows, different columns)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const float mo = __shfl_xor_sync(0xffffffffu, m[i], o), so = __shfl_xor_sync(0xffffffffu, s[i], o);
      const float mn = fmaxf(m[i], mo);
      if (mn == -INFINITY) continue;
      s[i] = (m[i] == -INFINITY ? 0.f : s[i] * ex2_approx((m[i] - mn) * kLog2e)) +
             (mo == -INFINITY ? 0.f : so * ex2_approx((mo - mn) * kLog2e));
      m[i] = mn;
    }
  }
  if (tq == 0) {
    const int n = L - 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = row0 + (i >> 1) * 16 + g + ((i & 1) ? 8 : 0);
      if (r >= T) continue;
      const int b = r / L, t = r - b * L;
      if (t < n) lse[static_cast<size_t>(b) * n + t] = m[i] + log2f(s[i]) * 0.6931471805599453f;
    }
  }
}

// ---------------------------------------------------------------- tcgen05 projection
// hp = RMSN(x; final_norm.gain) . proj on the streaming tcgen05 GEMM: the gain folds into the
// weight (W' = diag(g) proj, bf16 [K-major: 32 x d]) and 1/rms comes from the row statistics the
// last block tail wrote (sum of squares of the bf16 row), as everywhere else in the forward.
// The epilogue (one 32-column chunk = the whole row) writes hp in bf16 and the target logit
// from the bf16 hp and the target's item row (k_pretrain_proj's rounding points).
__global__ void k_pretrain_wfold(const float* __restrict__ proj, const float* __restrict__ gain, int d,
                                 __nv_bfloat16* __restrict__ wt) {  // wt[j][c] = g[c] proj[c][j]
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kPreK * d; i += gridDim.x * blockDim.x) {
    const int j = i / d, c = i - j * d;
    wt[i] = __float2bfloat16_rn(gain[c] * proj[static_cast<size_t>(c) * kPreK + j]);
  }
}

struct GsPretrainHead {
  static constexpr int kChunk = 32;
  const float4* ss;  // [T] row sum-of-squares partials of x
  float inv_d;
  __nv_bfloat16* hp;              // [T, 32]
  const __nv_bfloat16* items;     // [V, 32]
  const int32_t* click;           // [B, n]
  float* tgt;                     // [B, n]
  int L, n;
  __device__ void apply(int row, int col, const float (&v)[32]) const {
    (void)col;
    const float4 sp = ss[row];
    const float inv = rsqrtf(((sp.x + sp.y) + (sp.z + sp.w)) * inv_d + 1e-6f);  // norm.hpp:23-24
    uint32_t w[16];
    float hb[32];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      w[i] = pack_bf16x2(v[2 * i] * inv, v[2 * i + 1] * inv);
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
      hb[2 * i] = f.x;
      hb[2 * i + 1] = f.y;
    }
    __nv_bfloat16* dst = hp + static_cast<size_t>(row) * kPreK;
    stg256(dst, *reinterpret_cast<const uint32_t(*)[8]>(w));
    stg256(dst + 16, *reinterpret_cast<const uint32_t(*)[8]>(w + 8));
    const int b = row / L, t = row - b * L;
    if (t < n) {  // position t predicts click t
      const int item = click[static_cast<size_t>(b) * n + t];
      const int4* er = reinterpret_cast<const int4*>(items + static_cast<size_t>(item) * kPreK);
      float z = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int4 e4 = er[q];
        const __nv_bfloat162* e2 = reinterpret_cast<const __nv_bfloat162*>(&e4);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(e2[k]);
          z = fmaf(hb[8 * q + 2 * k], f.x, fmaf(hb[8 * q + 2 * k + 1], f.y, z));
        }
      }
      tgt[static_cast<size_t>(b) * n + t] = z;
    }
  }
};

// ---------------------------------------------------------------- tcgen05 log-sum-exp
// lse_t over the full vocabulary on tcgen05 (the k_attention skeleton without P V): a work item
// = (128-row block of hp, vocabulary chunk of kCeChunk items); per 128-item tile the MMA warp
// computes Z = hp_blk E_tile^T (two N = 64 halves, K = 32) into one of two TMEM buffers while
// the 8 softmax warps fold the other buffer into a per-(row, half) online (max, sum) in the
// log2 domain (no P is written back and nothing else is read from TMEM). Each (row, chunk,
// half) leaves a partial; k_ce_combine merges them in a fixed order.
constexpr int kCeChunk = 8192;
constexpr int kCeStages = 4;
struct CeTcSmem {
  static constexpr uint32_t kTile = 128 * kPreK * 2;  // 8 KB: 128 rows x 32 bf16
  static constexpr uint32_t oH = 0;                    // [2] hp tiles
  static constexpr uint32_t oE = oH + 2 * kTile;       // [kCeStages] item tiles
  static constexpr uint32_t oBar = oE + kCeStages * kTile;
  static constexpr uint32_t bytes = oBar + 32 * 8 + 1024;
};
struct CeTcArgs {
  int T, V, n_chunks, n_items;
  float2* part;  // [T][n_chunks][2] (max, sum) in the log2 domain
};

__global__ void __launch_bounds__(kAttnThreads, 2) k_ce_tc(const __grid_constant__ CUtensorMap tmH,
                                                            const __grid_constant__ CUtensorMap tmE,
                                                            const CeTcArgs a) {
  using S = CeTcSmem;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::oBar);
  uint64_t* h_full = bars + 0;   // [2]
  uint64_t* h_empty = bars + 2;  // [2]
  uint64_t* s_full = bars + 4;   // [2 buffers][2 halves]
  uint64_t* s_free = bars + 8;   // [2 buffers] (256: every softmax thread has loaded its half)
  uint64_t* e_full = bars + 10;  // [kCeStages]
  uint64_t* e_empty = e_full + kCeStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(e_empty + kCeStages);
  const int warp = warp_id(), lane = lane_id();
  const int tiles_per_chunk = kCeChunk / 128;
  auto n_tiles_of = [&](int it) {
    const int ch = it % a.n_chunks;
    const int items = min(kCeChunk, a.V - ch * kCeChunk);
    return (items + 127) / 128;
  };
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmH);
    tma_prefetch_desc(&tmE);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&h_full[i], 1);
      mbar_init(&h_empty[i], 1);
      mbar_init(&s_full[2 * i], 1);
      mbar_init(&s_full[2 * i + 1], 1);
      mbar_init(&s_free[i], 256);
    }
    for (int i = 0; i < kCeStages; ++i) {
      mbar_init(&e_full[i], 1);
      mbar_init(&e_empty[i], 1);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      int g = 0, li = 0;
      for (int it = blockIdx.x; it < a.n_items; it += gridDim.x, ++li) {
        const int rb = it / a.n_chunks, ch = it % a.n_chunks, n_t = n_tiles_of(it);
        const int hs = li & 1;
        mbar_wait_sleep(&h_empty[hs], ((li >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&h_full[hs], S::kTile);
        tma_load_2d(smem + S::oH + hs * S::kTile, &tmH, &h_full[hs], 0, rb * 128);
        for (int j = 0; j < n_t; ++j, ++g) {
          const int st = g % kCeStages;
          mbar_wait_sleep(&e_empty[st], ((g / kCeStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&e_full[st], S::kTile);
          tma_load_2d(smem + S::oE + st * S::kTile, &tmE, &e_full[st], 0, ch * kCeChunk + j * 128);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t id_s = umma_idesc_bf16(128, 64);
      constexpr uint32_t sw = kPreK * 2;  // 64-byte rows
      int g = 0, li = 0;
      for (int it = blockIdx.x; it < a.n_items; it += gridDim.x, ++li) {
        const int n_t = n_tiles_of(it), hs = li & 1;
        mbar_wait(&h_full[hs], (li >> 1) & 1);
        const uint32_t sh = smem_u32(smem + S::oH + hs * S::kTile);
        for (int j = 0; j < n_t; ++j, ++g) {
          const int buf = g & 1, st = g % kCeStages;
          if (g >= 2) mbar_wait(&s_free[buf], ((g >> 1) - 1) & 1);
          mbar_wait(&e_full[st], (g / kCeStages) & 1);
          tc_fence_after();
          const uint32_t se = smem_u32(smem + S::oE + st * S::kTile);
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
            for (int k = 0; k < kPreK / 16; ++k)
              mma_bf16_ss(tmem + buf * 128 + hf * 64, umma_sdesc_kmajor(sh + k * 32, sw),
                          umma_sdesc_kmajor(se + hf * 64 * kPreK * 2 + k * 32, sw), id_s, k > 0 ? 1u : 0u);
            mma_commit(&s_full[buf * 2 + hf]);
          }
          mma_commit(&e_empty[st]);
          if (j == n_t - 1) mma_commit(&h_empty[hs]);
        }
      }
    }
  } else {  // softmax warps: warp pair (w, w + 4) shares lane quarter w % 4, half = which pair
    const int quarter = warp & 3, hf = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    constexpr float kLog2e = 1.4426950408889634f;
    const float NEG_INF = -__int_as_float(0x7f800000);
    int g = 0;
    (void)tiles_per_chunk;
    for (int it = blockIdx.x; it < a.n_items; it += gridDim.x) {
      const int rb = it / a.n_chunks, ch = it % a.n_chunks, n_t = n_tiles_of(it);
      float m2 = NEG_INF;  // running max (log2 units) of this row's half
      float2 sacc = make_float2(0.f, 0.f);
      for (int j = 0; j < n_t; ++j, ++g) {
        const int buf = g & 1;
        const int c0 = ch * kCeChunk + j * 128 + hf * 64;  // first item of this half
        mbar_wait_sleep(&s_full[buf * 2 + hf], (g >> 1) & 1);
        tc_fence_after();
        uint32_t z[64];
        tmem_ld_32x32b_x32(tmem + buf * 128 + hf * 64 + lane_off, *reinterpret_cast<uint32_t(*)[32]>(z));
        tmem_ld_32x32b_x32(tmem + buf * 128 + hf * 64 + 32 + lane_off, *reinterpret_cast<uint32_t(*)[32]>(z + 32));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&s_free[buf]);
        if (c0 + 64 > a.V) {  // vocabulary tail
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (c0 + i >= a.V) z[i] = __float_as_uint(NEG_INF);
        }
        float mx[4] = {NEG_INF, NEG_INF, NEG_INF, NEG_INF};
#pragma unroll
        for (int i = 0; i < 64; ++i) mx[i & 3] = fmaxf(mx[i & 3], __uint_as_float(z[i]));
        const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * kLog2e;
        const float mn = fmaxf(m2, mt);
        if (mn == NEG_INF) continue;
        const float alpha = ex2_approx(m2 - mn);  // m2 = -inf -> 0
        sacc = make_float2(sacc.x * alpha, sacc.y * alpha);
        const float2 l2 = make_float2(kLog2e, kLog2e), nm = make_float2(-mn, -mn);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float2 x = ffma2(make_float2(__uint_as_float(z[2 * i]), __uint_as_float(z[2 * i + 1])), l2, nm);
          const float2 e = (i % 3 == 2) ? ex2_poly2(x) : make_float2(ex2_approx(x.x), ex2_approx(x.y));
          sacc = fadd2(sacc, e);
        }
        m2 = mn;
      }
      const int row = rb * 128 + r;
      if (row < a.T) a.part[(static_cast<size_t>(row) * a.n_chunks + ch) * 2 + hf] = make_float2(m2, sacc.x + sacc.y);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// lse[b, t] (natural log) of row r = b * L + t, t < n, from its 2 n_chunks partials (fixed order).
__global__ void k_ce_combine(const float2* __restrict__ part, int T, int L, int n_parts, float* __restrict__ lse) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= T) return;
  const int b = r / L, t = r - b * L, n = L - 1;
  if (t >= n) return;
  const float2* p = part + static_cast<size_t>(r) * n_parts;
  float m = -__int_as_float(0x7f800000);
  for (int i = 0; i < n_parts; ++i) m = fmaxf(m, p[i].x);
  float s = 0.f;
  for (int i = 0; i < n_parts; ++i)
    if (p[i].x != -__int_as_float(0x7f800000)) s += p[i].y * exp2f(p[i].x - m);
  lse[static_cast<size_t>(b) * n + t] = (m + log2f(s)) * 0.6931471805599453f;
}

// ---------------------------------------------------------------- backward
// Epilogue of the recomputed logit GEMM z = hp E^T (k_gemm_stream, 32-column chunks): the
// pre-training loss gradient dL/dz_t[v] = scale * (softmax_t[v] - [v == click_t]) with the
// forward's natural-log lse (position t < n predicts click t; the last position predicts
// nothing), as bf16 P [T, V] -- the operand of dh = P E and dE += P^T hp.
struct GsCeGrad {
  static constexpr int kChunk = 32;
  __nv_bfloat16* P;
  int ldp;
  const float* lse;       // [B, n]
  const int32_t* click;   // [B, n]
  int L, n;
  float scale;            // 1 / (B n): the loss is the mean CE over predicted positions
  __device__ void apply(int row, int col, const float (&v)[32]) const {
    const int b = row / L, t = row - b * L;
    uint32_t w[16];
    if (t >= n) {
#pragma unroll
      for (int i = 0; i < 16; ++i) w[i] = 0u;
    } else {
      const float l = lse[static_cast<size_t>(b) * n + t];
      const int tg = click[static_cast<size_t>(b) * n + t] - col;
      constexpr float kLog2e = 1.4426950408889634f;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float p0 = ex2_approx((v[2 * i] - l) * kLog2e) * scale;
        float p1 = ex2_approx((v[2 * i + 1] - l) * kLog2e) * scale;
        if (tg == 2 * i) p0 -= scale;
        if (tg == 2 * i + 1) p1 -= scale;
        w[i] = pack_bf16x2(p0, p1);
      }
    }
    __nv_bfloat16* p = P + static_cast<size_t>(row) * ldp + col;
    stg256(p, *reinterpret_cast<const uint32_t(*)[8]>(w));
    stg256(p + 16, *reinterpret_cast<const uint32_t(*)[8]>(w + 8));
  }
};

// loss = mean over the B n predicted positions of lse - target (one block, fixed order).
__global__ void __launch_bounds__(1024) k_ce_loss(const float* __restrict__ lse, const float* __restrict__ tgt, int n,
                                                  float* __restrict__ loss) {
  __shared__ float red[1024];
  float acc = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += lse[i] - tgt[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = red[0] / static_cast<float>(n);
}

}  // namespace sortk
