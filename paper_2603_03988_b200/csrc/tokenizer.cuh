// SPDX-License-Identifier: Apache-2.0
// K1: feature tokenizer -- Tokenizer::tokenize_sample (tokenizer.cpp:144-238) for a
// whole batch in one persistent kernel.
//
// Each 128-row tile belongs to one token group (history / candidate / profile):
//   1. gather: one thread per token row issues 16-byte vector loads of the
//      embedding rows (item | action | scene | time for history, tokenizer.cpp:95-112;
//      item for candidates, :114-127; profile_table[f] for profile fields, :196-205)
//      straight into the SW128 K-major A-operand layout in shared memory (K padded
//      to 64 with zeros). Ids are range-checked (check_id, :14-19): an
//      out-of-vocabulary id raises the device error flag and reads row 0 instead.
//   2. one tcgen05.mma chain (M=128, N=d, K=64) projects the tile against the
//      group's W^T (resident in smem) into TMEM.
//   3. epilogue (thread <-> row): + bias, RMSNorm with the group gain (norm.hpp:17-29,
//      emit_group :220-229), bf16 token row + its fp32 sum of squares (the
//      next pre-norm's statistic) written to the row's place in the sequence.
// BOS/SEP rows copy the special table (:171-176). Positions/roles are batch-uniform
// and live in the host plan.
#pragma once

#include "ptx.cuh"

namespace sortk {

struct TokParams {
  // tables (bf16, row-major)
  const __nv_bfloat16* item_tab;
  const __nv_bfloat16* action_tab;
  const __nv_bfloat16* scene_tab;
  const __nv_bfloat16* time_tab;
  const __nv_bfloat16* prof_tab;  // all profile tables concatenated
  const __nv_bfloat16* special;   // [3, d]
  int prof_row_off[SORT_MAX_PROFILE_FIELDS];
  int prof_vocab[SORT_MAX_PROFILE_FIELDS];
  // per-group projection W^T [d, 64] bf16 (K-major, zero padded) + bias/gain fp32 [d]
  const __nv_bfloat16* wt[3];
  const float* bias[3];
  const float* gain[3];
  // inputs (device)
  const int32_t* hist_item;
  const int32_t* hist_action;
  const int32_t* hist_scene;
  const int64_t* hist_ts;
  const int64_t* req_ts;
  const int32_t* profile;
  const int32_t* cand_item;
  // outputs
  __nv_bfloat16* x;      // [B, L, d]
  float4* ss;            // [B, L] sum of squares of the bf16 token row (slot 0 of 4)
  int32_t* hist_time;    // [B, H] or null
  int32_t* err;          // device error flags
  // geometry
  int B, H, P, N, L, d;
  int item_dim, action_dim, scene_dim, time_dim, prof_dim;
  int n_items, n_actions, n_scenes, n_tb;
  int special_tokens;
  int click_seq;  // tokenize_click_sequence (tokenizer.cpp:240-284): [BOS; clicks], gap buckets
  int tiles_hist, tiles_cand, tiles_prof;
};

enum : int { kGroupHist = 0, kGroupCand = 1, kGroupProf = 2 };
constexpr int kTokThreads = 256;  // two threads per token row (gather halves, epilogue column halves)
constexpr int kErrOOV = 1;

__device__ __forceinline__ int tok_time_bucket(int64_t delta, int nb) {
  // time_bucket (tokenizer.cpp:36-40) in exact integer form (valid for nb <= 48).
  const unsigned long long d = delta > 0 ? static_cast<unsigned long long>(delta) : 0ull;
  const int b = 63 - __clzll(static_cast<long long>(d + 1ull));
  return b < nb - 1 ? b : nb - 1;
}

// Copy `n8` 16-byte chunks from src into the swizzled A row starting at chunk c0.
__device__ __forceinline__ void tok_put(uint8_t* arow, int r, int c0, const __nv_bfloat16* src, int n8) {
  const int4* s = reinterpret_cast<const int4*>(src);
#pragma unroll 4
  for (int i = 0; i < n8; ++i) {
    const int c = c0 + i;
    *reinterpret_cast<int4*>(arow + ((c ^ (r & 7)) << 4)) = __ldg(s + i);
  }
}

__global__ void __launch_bounds__(kTokThreads) k_tokenize(const TokParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1k(smem_raw);
  const int d = p.d;
  uint8_t* sW = smem;                       // [d rows x 128 B] SW128
  uint8_t* sA = smem + d * 128;             // [128 rows x 128 B] SW128
  float* sBias = reinterpret_cast<float*>(sA + 128 * 128);
  float* sGain = sBias + d;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sGain + d);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  float* sSS = reinterpret_cast<float*>(bar + 2);  // [2 column halves][128 rows] partial sums

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int rt = t & 127, hh = t >> 7;  // token row of the tile, which half of it this thread owns
  const uint32_t tcols = d <= 32 ? 32 : (d <= 64 ? 64 : (d <= 128 ? 128 : 256));
  if (t == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(tslot, tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t idesc = umma_idesc_bf16(128, d);

  const int n_tiles = p.tiles_hist + p.tiles_cand + p.tiles_prof;
  const int st = p.special_tokens || p.click_seq ? 1 : 0;
  const int off_hist = st, off_prof = st + p.H + st, off_cand = off_prof + p.P + st;
  auto group_of = [&](int tile, int& e0, int& count) {
    if (tile < p.tiles_hist) {
      e0 = tile * 128; count = p.B * p.H;
      return static_cast<int>(kGroupHist);
    }
    if (tile < p.tiles_hist + p.tiles_cand) {
      e0 = (tile - p.tiles_hist) * 128; count = p.B * p.N;
      return static_cast<int>(kGroupCand);
    }
    e0 = (tile - p.tiles_hist - p.tiles_cand) * 128; count = p.B * p.P;
    return static_cast<int>(kGroupProf);
  };
  // ---- gather of one token row into registers: up to 8 16-byte chunks of the concatenated
  // embedding rows (K padded to 64 with zeros). Two stages so no thread waits on a load:
  // the row's ids (and timestamps) are fetched TWO tiles ahead, the embedding chunks they
  // address ONE tile ahead -- both in flight while the current tile's MMA and epilogue run.
  struct Ids {
    int a, b, c;      // hist: item, action, scene; cand: item; prof: value
    int64_t t0, t1;   // hist: event time and the request time (clicks: the previous click)
  };
  struct Row {
    int4 c[4];  // chunks [4 hh, 4 hh + 4) of the row
    int out_row;
  };
  auto fetch_ids = [&](int tile, Ids& q) {
    q.a = q.b = q.c = 0;
    q.t0 = q.t1 = 0;
    if (tile >= n_tiles) return;
    int e0, count;
    const int group = group_of(tile, e0, count);
    const int e = e0 + rt;
    if (e >= count) return;
    if (group == kGroupHist) {
      const int b = e / p.H, i = e - b * p.H;
      q.a = p.hist_item[e];
      q.b = p.hist_action[e];
      q.c = p.hist_scene[e];
      q.t0 = p.hist_ts[e];
      q.t1 = p.click_seq ? (i == 0 ? 0 : p.hist_ts[e - 1]) : p.req_ts[b];
    } else if (group == kGroupCand) {
      q.a = p.cand_item[e];
    } else {
      q.a = p.profile[e];
    }
  };
  auto gather = [&](int tile, const Ids& q, Row& g) {
    g.out_row = -1;
    const __nv_bfloat16* src[4] = {nullptr, nullptr, nullptr, nullptr};
    int n8[4] = {0, 0, 0, 0};
    if (tile < n_tiles) {
      int e0, count;
      const int group = group_of(tile, e0, count);
      const int e = e0 + rt;
      if (e < count) {
        if (group == kGroupHist) {
          const int b = e / p.H, i = e - b * p.H;
          int item = q.a, act = q.b, sc = q.c;
          // click sequences: the gap to the previous click, the first click at INT64_MAX / 4
          // (tokenizer.cpp:262-270); requests: request time - event time (:95-112)
          const int64_t delta = p.click_seq ? (i == 0 ? 0x1FFFFFFFFFFFFFFFll : q.t0 - q.t1) : q.t1 - q.t0;
          const int tb = tok_time_bucket(delta, p.n_tb);
          if (static_cast<unsigned>(item) >= static_cast<unsigned>(p.n_items) ||
              static_cast<unsigned>(act) >= static_cast<unsigned>(p.n_actions) ||
              static_cast<unsigned>(sc) >= static_cast<unsigned>(p.n_scenes)) {
            atomicOr(p.err, kErrOOV);
            item = static_cast<unsigned>(item) < static_cast<unsigned>(p.n_items) ? item : 0;
            act = static_cast<unsigned>(act) < static_cast<unsigned>(p.n_actions) ? act : 0;
            sc = static_cast<unsigned>(sc) < static_cast<unsigned>(p.n_scenes) ? sc : 0;
          }
          if (p.hist_time && hh == 0) p.hist_time[e] = tb;
          src[0] = p.item_tab + static_cast<size_t>(item) * p.item_dim;
          src[1] = p.action_tab + static_cast<size_t>(act) * p.action_dim;
          src[2] = p.scene_tab + static_cast<size_t>(sc) * p.scene_dim;
          src[3] = p.time_tab + static_cast<size_t>(tb) * p.time_dim;
          n8[0] = p.item_dim >> 3;
          n8[1] = p.action_dim >> 3;
          n8[2] = p.scene_dim >> 3;
          n8[3] = p.time_dim >> 3;
          g.out_row = b * p.L + off_hist + i;
        } else if (group == kGroupCand) {
          const int b = e / p.N, j = e - b * p.N;
          int item = q.a;
          if (static_cast<unsigned>(item) >= static_cast<unsigned>(p.n_items)) {
            atomicOr(p.err, kErrOOV);
            item = 0;
          }
          src[0] = p.item_tab + static_cast<size_t>(item) * p.item_dim;
          n8[0] = p.item_dim >> 3;
          g.out_row = b * p.L + off_cand + j;
        } else {
          const int b = e / p.P, f = e - b * p.P;
          int v = q.a;
          if (static_cast<unsigned>(v) >= static_cast<unsigned>(p.prof_vocab[f])) {
            atomicOr(p.err, kErrOOV);
            v = 0;
          }
          src[0] = p.prof_tab + static_cast<size_t>(p.prof_row_off[f] + v) * p.prof_dim;
          n8[0] = p.prof_dim >> 3;
          g.out_row = b * p.L + off_prof + f;
        }
      }
    }
    // chunk c = 4 hh + i of the concatenated row -> (segment, offset), constant-indexed selects
    const int e1 = n8[0], e2 = e1 + n8[1], e3 = e2 + n8[2], e4 = e3 + n8[3];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = hh * 4 + i;
      const __nv_bfloat16* sp = c < e1 ? src[0] : (c < e2 ? src[1] : (c < e3 ? src[2] : src[3]));
      const int o = c < e1 ? c : (c < e2 ? c - e1 : (c < e3 ? c - e2 : c - e3));
      g.c[i] = c < e4 ? __ldg(reinterpret_cast<const int4*>(sp) + o) : make_int4(0, 0, 0, 0);
    }
  };
  int cur_group = -1;
  uint32_t phase = 0;
  Row g;
  Ids ids;
  fetch_ids(blockIdx.x, ids);
  gather(blockIdx.x, ids, g);
  fetch_ids(blockIdx.x + gridDim.x, ids);
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    int e0, count;
    const int group = group_of(tile, e0, count);
    if (group != cur_group) {  // (re)load this group's W^T, bias and gain
      __syncthreads();
      const int4* w = reinterpret_cast<const int4*>(p.wt[group]);
      for (int i = t; i < d * 8; i += kTokThreads) {
        const int n = i >> 3, c = i & 7;
        *reinterpret_cast<int4*>(sW + n * 128 + ((c ^ (n & 7)) << 4)) = __ldg(w + i);
      }
      for (int i = t; i < d; i += kTokThreads) {
        sBias[i] = p.bias[group][i];
        sGain[i] = p.gain[group][i];
      }
      cur_group = group;
    }
    // ---- 1. this thread's gathered row -> the swizzled A tile
    uint8_t* arow = sA + rt * 128;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = hh * 4 + i;
      *reinterpret_cast<int4*>(arow + ((c ^ (rt & 7)) << 4)) = g.c[i];
    }
    const int out_row = g.out_row;
    const bool valid = out_row >= 0;
    fence_proxy_async_smem();
    __syncthreads();
    // ---- 2. projection on the tensor cores
    if (t == 0) {
      tc_fence_after();
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sW);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_bf16_ss(tmem, umma_sdesc_kmajor(a0 + k * 32, 128), umma_sdesc_kmajor(b0 + k * 32, 128),
                    idesc, k > 0 ? 1u : 0u);
      mma_commit(bar);
    }
    gather(tile + gridDim.x, ids, g);       // next tile's rows in flight during this tile's epilogue
    fetch_ids(tile + 2 * gridDim.x, ids);  // and the ids of the tile after
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    // ---- 3. epilogue: bias + RMSNorm(gain) -> bf16 row + sum of squares. Warp w reads TMEM
    // lane quarter w % 4 (its 32 rows) and columns [hh * d/2, (hh + 1) * d/2); the two halves
    // combine their sums of squares through shared memory. 32 accumulator columns per load.
    const int q = warp & 3, r = q * 32 + lane;
    const int cb = hh * (d / 2), ce = cb + d / 2;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t sb = smem_u32(sBias), sgn = smem_u32(sGain);
    float ss = 0.f;
    for (int c = cb; c < ce; c += 32) {
      uint32_t rv[32];
      tmem_ld_32x32b_x32(trow + c, rv);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float4 bv = lds_f32x4(sb + (c + i) * 4);
        const float2 v01 = fadd2(make_float2(__uint_as_float(rv[i]), __uint_as_float(rv[i + 1])), make_float2(bv.x, bv.y));
        const float2 v23 =
            fadd2(make_float2(__uint_as_float(rv[i + 2]), __uint_as_float(rv[i + 3])), make_float2(bv.z, bv.w));
        ss += v01.x * v01.x + v01.y * v01.y + v23.x * v23.x + v23.y * v23.y;
        rv[i] = __float_as_uint(v01.x);
        rv[i + 1] = __float_as_uint(v01.y);
        rv[i + 2] = __float_as_uint(v23.x);
        rv[i + 3] = __float_as_uint(v23.y);
      }
      // acc + b back over the accumulator: pass 2 reads it without reloading the bias
      tmem_st_32x32b_x16(trow + c, *reinterpret_cast<const uint32_t(*)[16]>(rv));
      tmem_st_32x32b_x16(trow + c + 16, *reinterpret_cast<const uint32_t(*)[16]>(rv + 16));
    }
    tmem_st_wait();
    sSS[hh * 128 + r] = ss;
    named_bar_sync(1 + q, 64);
    const float inv = rsqrtf((sSS[r] + sSS[128 + r]) / static_cast<float>(d) + 1e-6f);
    named_bar_sync(1 + q, 64);  // both halves have read before the sums are overwritten
    // (thread t gathered tile row t & 127 == q * 32 + lane: out_row / valid are this lane's row)
    const float2 inv2 = make_float2(inv, inv);
    float ss_out = 0.f;
    for (int c = cb; c < ce; c += 32) {
      uint32_t rv[32];
      tmem_ld_32x32b_x32(trow + c, rv);
      tmem_ld_wait();
#pragma unroll
      for (int q16 = 0; q16 < 2; ++q16) {
        uint32_t packed[8];
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
          const int k = q16 * 16 + i;
          const float4 gv = lds_f32x4(sgn + (c + k) * 4);
          // ((acc + b) / rms) g on packed fp32x2 ops (acc + b stored by pass 1): the same IEEE
          // operations in the same order as the scalar form, so the rows are bit-identical to it
          const float2 y01 =
              fmul2(fmul2(make_float2(__uint_as_float(rv[k]), __uint_as_float(rv[k + 1])), inv2), make_float2(gv.x, gv.y));
          const float2 y23 = fmul2(fmul2(make_float2(__uint_as_float(rv[k + 2]), __uint_as_float(rv[k + 3])), inv2),
                                   make_float2(gv.z, gv.w));
          const uint32_t w01 = pack_bf16x2(y01.x, y01.y), w23 = pack_bf16x2(y23.x, y23.y);
          packed[i / 2] = w01;
          packed[i / 2 + 1] = w23;
          const float q0x = __uint_as_float(w01 << 16), q0y = __uint_as_float(w01 & 0xFFFF0000u);
          const float q1x = __uint_as_float(w23 << 16), q1y = __uint_as_float(w23 & 0xFFFF0000u);
          ss_out += q0x * q0x + q0y * q0y + q1x * q1x + q1y * q1y;
        }
        if (valid) stg256(p.x + static_cast<size_t>(out_row) * d + c + q16 * 16, packed);
      }
    }
    sSS[hh * 128 + r] = ss_out;
    named_bar_sync(1 + q, 64);
    if (valid && hh == 0) p.ss[out_row] = make_float4(sSS[r], sSS[128 + r], 0.f, 0.f);
    named_bar_sync(1 + q, 64);
    tc_fence_before();
    __syncthreads();
  }
  // ---- BOS / SEP rows: raw special-table rows (tokenizer.cpp:171-176), one warp per row.
  if (p.special_tokens || p.click_seq) {
    const int nwarps = gridDim.x * (kTokThreads / 32);
    const int per = p.click_seq ? 1 : 3;  // click sequences carry BOS only
    for (int w = blockIdx.x * (kTokThreads / 32) + warp; w < p.B * per; w += nwarps) {
      const int b = w / per, k = w - b * per;
      const int row = b * p.L + (k == 0 ? 0 : (k == 1 ? 1 + p.H : 2 + p.H + p.P));
      float ss = 0.f;
      for (int c = lane; c < d; c += 32) {
        const __nv_bfloat16 v = p.special[k * d + c];
        p.x[static_cast<size_t>(row) * d + c] = v;
        const float f = __bfloat162float(v);
        ss += f * f;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) p.ss[row] = make_float4(ss, 0.f, 0.f, 0.f);
    }
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, tcols);
  }
}

inline size_t tok_smem_bytes(int d) { return 1024 + d * 128 + 128 * 128 + 2 * d * 4 + 16 + 2 * 128 * 4; }

}  // namespace sortk
