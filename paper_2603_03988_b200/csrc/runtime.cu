// SPDX-License-Identifier: Apache-2.0
// libsort_b200.so: handle, device weights/workspace, forward orchestration and the
// C ABI declared in include/sort_b200.h.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <numeric>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/sort_b200.h"
#include "attention.cuh"
#include "attn_bwd.cuh"
#include "block_tail.cuh"
#include "epilogues.cuh"
#include "gemm.cuh"
#include "misc.cuh"
#include "plan.hpp"
#include "tma_host.hpp"
#include "tokenizer.cuh"
#include "train.cuh"
#include "generic.cuh"
#include "gemm_stream.cuh"
#include "moe.cuh"
#include "pretrain.cuh"

namespace sortk {

thread_local std::string g_last_error;

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw RuntimeFailure(std::string(#x) + " failed: " + cudaGetErrorString(e_));        \
  } while (0)

static inline __nv_bfloat16 f2bf(float x) { return __float2bfloat16_rn(x); }

struct HostParam {
  std::vector<float> v;
  int64_t rows = 0, cols = 0;
};

struct LayerDev {
  int4* rowmeta = nullptr;
  int32_t *tile_off = nullptr, *tile_code = nullptr, *qtile_order = nullptr;
  int32_t *pos_q = nullptr, *pos_kv = nullptr, *query_rows = nullptr;
  __nv_bfloat16 *w_all = nullptr, *w_kv = nullptr, *w_qg = nullptr, *w_o = nullptr,
                *w_up = nullptr, *w_down = nullptr;
  float *gain_q = nullptr, *gain_k = nullptr;
  float* gain_q_s = nullptr;  // gain_q * log2(e) / sqrt(dk): the pre-scaled Q of inference attention
  int in_buf = 0, q_buf = 0;
  int Rq = 0, Rkv = 0;
  int bn_full = 0, bn_half = 0, bn_up = 0, bn_o = 0, bn_down = 0;
  float logit_bound = 0.f;  // QKNorm logit bound (0 = unknown -> online-max softmax)
  CUtensorMap tmA_in, tmA_q, tmB_all, tmB_qg, tmB_kv, tmA_hg, tmB_o, tmB_up, tmA_hid, tmB_down;
  CUtensorMap tmQ, tmK, tmV;
  CUtensorMap tmRopeKV, tmRopeQ;  // per-row RoPE side tables for the K/V rows and the Q rows
  CUtensorMap tmWo_t, tmWup_t, tmWdown_t;  // k_block_tail weight stages
  CUtensorMap tmWo_p, tmWup_p, tmWdown_p;  // ... as a CTA pair (each CTA loads half the rows)
  CUtensorMap tmB_all_p, tmB_kv_p, tmB_qg_p;  // QKVG weight slices as a CTA pair (BN/2 rows)
  // MoE FFN: stacked expert weights (routed experts, then the shared one), router in the
  // fp32 master buffer, this layer's routing of the last forward
  __nv_bfloat16 *w_moe_gu = nullptr, *w_moe_down = nullptr;
  CUtensorMap tmB_moe_gu, tmB_moe_down;
  CUtensorMap tmWup_moe, tmWdown_moe;  // k_moe_expert weight stages (128 x 64 and d x 64 boxes)
  int bn_moe_gu = 0, bn_moe_down = 0;
  const float* router = nullptr;
  float* router_bias = nullptr;
  int32_t* moe_sel = nullptr;
  float* moe_w = nullptr;
};

struct Handle {
  SortConfig cfg{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  Plan plan;
  int d = 0, H = 0, dk = 0, m = 0, dh = 0, L0 = 0, Bmax = 0, num_sms = 148;
  std::map<std::string, HostParam> host;
  bool finalized = false;
  bool fused_tail = true;  // sort_set_option("fused_tail")
  bool tail_pair = false;  // sort_set_option("tail_pair"): block tail as CTA pairs (cta_group::2)
  bool attn_bwd_mma = true; // sort_set_option("attn_bwd_mma"): tensor-core attention backward
  bool attn_bwd_tc = true;  // sort_set_option("attn_bwd_tc"): tcgen05 attention backward (0: mma.sync)
  bool qkvg_pair = false;   // sort_set_option("qkvg_pair"): QKVG projection as CTA pairs
  bool attn_prescale = true;  // sort_set_option("attn_prescale"): inference Q pre-scaled into the exp2 domain
  bool generic = false;    // d > 256 (SORT-large): projections through the generic path
  // ---- MoE FFN: routed + shared experts as grouped tcgen05 GEMMs
  bool moe = false;
  int moe_E = 0, moe_k = 0, moe_s = 0, moe_m = 0, moe_pmax = 0, moe_tiles_max = 0;
  __nv_bfloat16 *moe_xs = nullptr, *moe_hs = nullptr;
  __nv_bfloat16* moe_ys = nullptr;
  float *moe_inv = nullptr, *moe_wof = nullptr;
  int32_t *moe_tok = nullptr, *moe_slot = nullptr, *moe_off = nullptr, *moe_cursor = nullptr,
          *moe_tile_group = nullptr, *moe_tile_mblk = nullptr, *moe_ntiles = nullptr,
          *moe_counts = nullptr;  // counts [layers][E]
  int moe_rows[SORT_MAX_LAYERS] = {0};  // rows routed per layer in the last forward
  CUtensorMap tmA_moe_xs, tmA_moe_hs, tmY_moe;
  bool moe_fused = true;  // sort_set_option("moe_fused"): k_moe_expert instead of the grouped GEMM pair
  // ---- pre-training head
  const float* pre_proj = nullptr;  // pretrain.proj [d, item_dim] in the master buffer
  __nv_bfloat16* pre_hp = nullptr;  // projected rows [B * L, item_dim]
  bool pre_proj_tc = true;  // sort_set_option("pre_proj_tc"): pre-training projection on tcgen05
  __nv_bfloat16* pre_wt = nullptr;  // diag(final_norm.gain) . pretrain.proj, K-major bf16 [32, d]
  bool ce_tc = true;  // sort_set_option("ce_tc"): tied-head log-sum-exp on tcgen05 (0: mma.sync k_ce_tied)
  float2* ce_part = nullptr;  // k_ce_tc partials
  size_t ce_part_cap = 0;
  float *pre_lse = nullptr, *pre_tgt = nullptr;  // [B, n_hist]
  __nv_bfloat16* pre_P = nullptr;   // training: dL/dz [B * L, V] bf16 (recomputed logits' gradient)
  float *pre_dh = nullptr, *pre_loss = nullptr;  // dL/d(hp) [B * L, item_dim], the step's loss
  // row-sharded item table (sort_set_item_table): the batch's item rows, gathered from the
  // owning ranks, replace the handle's table for the following calls
  const __nv_bfloat16* item_ext = nullptr;
  int64_t item_ext_rows = 0;
  // ---- training (sort_train_step): fp32 master copies of the block/head parameters,
  // a flat fp32 gradient buffer, saved forward activations per layer, workspace
  std::map<std::string, float*> w32;
  std::map<std::string, __nv_bfloat16*> w16;  // bf16 copies for the generic path's GEMMs
  std::map<std::string, __nv_bfloat16*> wT;   // bf16 K-major (transposed) weights of the streaming GEMMs
  std::map<std::tuple<const void*, uint64_t, uint64_t, uint64_t, uint32_t>, CUtensorMap> gs_maps;
  bool stream_gemm = true;  // sort_set_option("stream_gemm"): generic path on k_gemm_stream (0: cuBLAS)
  bool train_cublas = false;  // sort_set_option("train_cublas"): training GEMMs on cuBLAS (A/B)
  float* splitk_ws = nullptr;  // split-K partials of the streaming GEMM
  size_t splitk_cap = 0;
  std::map<std::string, std::pair<__nv_bfloat16*, size_t>> tw16;  // training: bf16 weights of the FFN backward
  CastSeg* tw16_segs = nullptr;  // device list of the tw16 casts (k_cast_segs)
  int tw16_nseg = 0;
  size_t tw16_nmax = 0;
  std::map<std::string, std::pair<size_t, std::pair<int64_t, int64_t>>> grad_index;  // offset, shape
  float* grads = nullptr;
  float* master = nullptr;                 // fp32 master parameters (grad_index layout)
  float *adam_m = nullptr, *adam_v = nullptr;
  int adam_t = 0;
  unsigned long long* adam_bad = nullptr;  // first non-finite gradient index + 1
  size_t grad_count = 0;
  bool training = false;  // forward currently saving activations
  struct TrainLayer {
    __nv_bfloat16 *x_in = nullptr, *q = nullptr, *k = nullptr, *v = nullptr, *g = nullptr,
                  *o_pre = nullptr, *x1 = nullptr;
    float* lse = nullptr;
    int32_t *dq_off = nullptr, *dkv_off = nullptr;
    int2 *dq_iv = nullptr, *dkv_iv = nullptr;
    int32_t *qb_off = nullptr, *qb_list = nullptr;  // tensor-core backward: q blocks per kv block
    CUtensorMap tmQ, tmK, tmV;  // the attention core reads the saved Q / K / V directly
    // tcgen05 backward (attn_bwd.cuh): X/Y step lists of the dK/dV and dQ passes and the
    // 128-row (X) / 64-row (Y) boxes of Q, K, V and the token-major dO
    int32_t *tc_kv_off = nullptr, *tc_q_off = nullptr;
    int2 *tc_kv_code = nullptr, *tc_q_code = nullptr;
    int tc_kv_n = 0, tc_q_n = 0;
    CUtensorMap tmQ64, tmK64, tmV64, tmDO128, tmDO64;
    int4* kvmeta = nullptr;  // transposed compact mask (pass 1), null if not two-interval
  };
  std::vector<TrainLayer> tl;
  const TrainLayer* save_to = nullptr;  // training forward: QKVG writes straight into these buffers
  float *tw[16] = {nullptr};  // backward workspace
  __nv_bfloat16* dO16 = nullptr;  // bf16 copy of dL/d(attention output) for the tensor-core backward
  float* dtokens = nullptr;
  float* wpad = nullptr;  // tokenizer backward: zero-padded projection weight
  // Parameter::frozen (params.hpp:15-25): frozen tensors get no gradient and no optimizer
  // update. The item table starts frozen (SORT's transfer + freeze setting);
  // unfreezing it allocates an fp32 master / gradient / AdamW moments for it.
  std::set<std::string> frozen{"tok.item_table"};
  float *item_master = nullptr, *item_grad = nullptr, *item_m = nullptr, *item_v = nullptr;
  size_t wpad_cap = 0;
  float* dz_dev = nullptr;                 // dL/dlogits of the current step
  int32_t* t_rows = nullptr;               // tokenizer backward: token row of each group row
  // generic (d > 256) forward: fp32 residual stream and workspace
  float* gX[2] = {nullptr, nullptr};
  float* gw[10] = {nullptr};
  int32_t* g_rows = nullptr;
  int gX_final = 0;
  std::map<int, int32_t*> cand_maps;       // candidate-row maps for the head backward
  int train_B = 0;
  cublasHandle_t cublas = nullptr;
  // device weights
  __nv_bfloat16 *item = nullptr, *action = nullptr, *scene = nullptr, *time = nullptr,
                *prof = nullptr, *special = nullptr;
  __nv_bfloat16* tok_wt[3] = {nullptr, nullptr, nullptr};
  float* tok_b[3] = {nullptr, nullptr, nullptr};
  float* tok_g[3] = {nullptr, nullptr, nullptr};
  int prof_off[SORT_MAX_PROFILE_FIELDS] = {0};
  float2* rope = nullptr;
  float *head_gain = nullptr, *head_w1 = nullptr, *head_b1 = nullptr, *head_w2 = nullptr,
        *head_b2 = nullptr;
  // tensor-core head (misc.cuh GsHead): g . W1 as three bf16 pieces [dh, 3d], gathered candidate
  // rows + statistics, per-chunk partial logits
  bool head_tc = true;  // sort_set_option("head_tc"): 0 runs the SIMT k_head
  __nv_bfloat16 *head_wt = nullptr, *head_xc = nullptr;
  float4* head_ssc = nullptr;
  float* head_zp = nullptr;
  std::vector<LayerDev> layers;
  // workspace
  __nv_bfloat16* X[2] = {nullptr, nullptr};
  float4* SS[2] = {nullptr, nullptr};  // per-row sum-of-squares partials
  CUtensorMap tmSS[2];                 // the same rows as a TMA side stream (128-row boxes)
  std::map<std::pair<int, std::vector<int32_t>>, CUtensorMap> rope_tables;
  __nv_bfloat16 *Qb = nullptr, *Kb = nullptr, *Vb = nullptr, *Gb = nullptr, *Hg = nullptr,
                *hid = nullptr;
  float *probs = nullptr, *logits = nullptr;
  int32_t* err = nullptr;
  int32_t* hist_time = nullptr;
  int32_t *in_item = nullptr, *in_action = nullptr, *in_scene = nullptr, *in_prof = nullptr,
          *in_cand = nullptr;
  int64_t *in_ts = nullptr, *in_req = nullptr;
  // sort_forward_async: two input staging slots filled on a copy stream, so step i+1's
  // host->device copy overlaps step i's kernels
  struct InSlot {
    int32_t *item = nullptr, *action = nullptr, *scene = nullptr, *prof = nullptr, *cand = nullptr;
    int64_t *ts = nullptr, *req = nullptr;
  } in_slot[2];
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t slot_copied[2] = {nullptr, nullptr}, slot_free[2] = {nullptr, nullptr};
  int64_t async_steps = 0;
  // CUDA graphs of the inference forward, one per (batch, input slot, item table): a replay
  // is one launch instead of ~160 (sort_set_option("graphs")); dropped whenever weights,
  // options or logit bounds change
  bool use_graphs = true;
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
  };
  std::map<std::tuple<int, const void*, const void*, int64_t>, GraphEntry> graphs;
  void drop_graphs() {
    for (auto& kv : graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
  }
  std::vector<void*> allocs;
  // instrumentation
  bool timing = false;
  std::vector<cudaEvent_t> events;
  std::vector<std::string> stage_names;
  std::vector<float> stage_ms;
  int launches = 0;

  template <class T>
  T* dalloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    CK(cudaMalloc(&p, n * sizeof(T)));
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const std::vector<T>& h) {
    T* p = dalloc<T>(h.size());
    CK(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return p;
  }
  ~Handle() {
    if (device >= 0) cudaSetDevice(device);
    drop_graphs();
    for (void* p : allocs) cudaFree(p);
    for (auto e : events) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i) {
      if (slot_copied[i]) cudaEventDestroy(slot_copied[i]);
      if (slot_free[i]) cudaEventDestroy(slot_free[i]);
    }
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (splitk_ws) cudaFree(splitk_ws);
    if (cublas) cublasDestroy(cublas);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }
};

// ------------------------------------------------------------------ params
static const HostParam& need_param(Handle& h, const std::string& name, int64_t rows, int64_t cols) {
  auto it = h.host.find(name);
  if (it == h.host.end()) throw ConfigError("missing parameter " + name);
  if (it->second.rows != rows || it->second.cols != cols)
    throw ConfigError("parameter " + name + " has shape [" + std::to_string(it->second.rows) + ", " +
                      std::to_string(it->second.cols) + "], expected [" + std::to_string(rows) +
                      ", " + std::to_string(cols) + "]");
  return it->second;
}

static std::vector<__nv_bfloat16> to_bf16(const std::vector<float>& v) {
  std::vector<__nv_bfloat16> o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = f2bf(v[i]);
  return o;
}

// W [K, N] (reference [in, out]) -> W^T [N, Kpad] bf16, optionally scaling input row k by g[k].
static std::vector<__nv_bfloat16> transpose_bf16(const HostParam& w, int Kpad, const float* g) {
  const int K = static_cast<int>(w.rows), N = static_cast<int>(w.cols);
  std::vector<__nv_bfloat16> o(static_cast<size_t>(N) * Kpad, f2bf(0.f));
  for (int k = 0; k < K; ++k)
    for (int n = 0; n < N; ++n) o[static_cast<size_t>(n) * Kpad + k] = f2bf(w.v[static_cast<size_t>(k) * N + n] * (g ? g[k] : 1.f));
  return o;
}

// Per-row RoPE side table for a GEMM over B x R rows whose row r sits at position pos[r]:
// row b*R + r holds the (cos, sin) pairs of pos[r] (rope.hpp:23-38, fp64 -> fp32), so the
// TMA producer can stage a tile's rows next to its A tile. Shared by GEMMs with equal (R, pos).
static const CUtensorMap& rope_table(Handle& h, int R, const std::vector<int32_t>& pos) {
  auto key = std::make_pair(R, pos);
  auto it = h.rope_tables.find(key);
  if (it != h.rope_tables.end()) return it->second;
  const int dk = h.dk;
  std::vector<__half> one(static_cast<size_t>(R) * dk);
  for (int r = 0; r < R; ++r)
    for (int j = 0; j < dk / 2; ++j) {
      const double freq = std::pow(h.cfg.rope_theta, -2.0 * j / static_cast<double>(dk));
      const double ang = static_cast<double>(pos[r]) * freq;
      one[static_cast<size_t>(r) * dk + 2 * j] = __float2half_rn(static_cast<float>(std::cos(ang)));
      one[static_cast<size_t>(r) * dk + 2 * j + 1] = __float2half_rn(static_cast<float>(std::sin(ang)));
    }
  const size_t rows = static_cast<size_t>(h.Bmax) * R;
  __half* dev = h.dalloc<__half>(rows * dk);
  for (int b = 0; b < h.Bmax; ++b)
    CK(cudaMemcpy(dev + static_cast<size_t>(b) * R * dk, one.data(), one.size() * 2, cudaMemcpyHostToDevice));
  const uint32_t box = static_cast<uint32_t>(std::min(dk, 64));
  uint64_t dims[2] = {static_cast<uint64_t>(dk), rows};
  uint64_t strides[1] = {static_cast<uint64_t>(dk) * 2};
  uint32_t bx[2] = {box, 128};
  return h.rope_tables[key] = make_tmap(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, dev, 2, dims, strides, bx, box * 2);
}

// Shapes the fused block tail covers (TMEM: d accumulator + 2 x 128 hidden-chunk columns).
static bool tail_supported(const Handle& h) {
  return !h.moe && (h.d == 128 || h.d == 256) && h.m % 64 == 0 && h.m >= 64;
}

// MoE layer weights: expert g (routed 0..E-1, then the shared expert) as
//   [gate | up]: rows g*2m_e .. interleaving 32-column blocks [gate_j | up_j] (W^T, K = d)
//   down:        rows g*d ..    W_down^T [d, m_e]
// The expert input is the RMSNorm'd row itself (the router needs it in fp32 anyway), so the
// ffn_norm gain is applied by the scatter kernel instead of being folded into the weights.
static void build_moe_layer(Handle& h, int l, LayerDev& L) {
  const int d = h.d, me = h.moe_m, G = h.moe_E + h.moe_s;
  const std::string f = "ffn." + std::to_string(l) + ".";
  need_param(h, f + "router", d, h.moe_E);
  need_param(h, f + "router_bias", 1, h.moe_E);
  std::vector<__nv_bfloat16> gu(static_cast<size_t>(G) * 2 * me * d), dn(static_cast<size_t>(G) * d * me);
  for (int g = 0; g < G; ++g) {
    const std::string X = g < h.moe_E ? f + "expert." + std::to_string(g) + "." : f + "shared.";
    const HostParam& wg = need_param(h, X + "w_gate", d, me);
    const HostParam& wu = need_param(h, X + "w_up", d, me);
    const HostParam& wd = need_param(h, X + "w_down", me, d);
    __nv_bfloat16* o = gu.data() + static_cast<size_t>(g) * 2 * me * d;
    for (int j = 0; j < me / 32; ++j)
      for (int i = 0; i < 64; ++i) {
        const HostParam& src = i < 32 ? wg : wu;
        const int col = 32 * j + (i & 31);
        const size_t row = static_cast<size_t>(64 * j + i);
        for (int k = 0; k < d; ++k) o[row * d + k] = f2bf(src.v[static_cast<size_t>(k) * me + col]);
      }
    const std::vector<__nv_bfloat16> t = transpose_bf16(wd, me, nullptr);
    std::copy(t.begin(), t.end(), dn.begin() + static_cast<size_t>(g) * d * me);
  }
  L.w_moe_gu = h.upload(gu);
  L.w_moe_down = h.upload(dn);
  auto pick = [&](int N, int K, int chunk) {
    for (int bn = 256; bn >= chunk; bn /= 2)
      if (N % bn == 0 && bn % chunk == 0 && gemm_plan(K, bn, 0, 1, 2).a_stages >= 2) return bn;
    throw ConfigError("unsupported MoE GEMM shape N=" + std::to_string(N) + " K=" + std::to_string(K));
  };
  L.bn_moe_gu = pick(2 * me, d, 64);
  L.bn_moe_down = pick(d, me, 32);
  L.tmB_moe_gu = make_tmap_2d(L.w_moe_gu, static_cast<uint64_t>(G) * 2 * me, d, d, L.bn_moe_gu, 64, 128);
  L.tmB_moe_down = make_tmap_2d(L.w_moe_down, static_cast<uint64_t>(G) * d, me, me, L.bn_moe_down, 64, 128);
  L.tmWup_moe = make_tmap_2d(L.w_moe_gu, static_cast<uint64_t>(G) * 2 * me, d, d, 128, 64, 128);
  L.tmWdown_moe = make_tmap_2d(L.w_moe_down, static_cast<uint64_t>(G) * d, me, me, d, 64, 128);
  const size_t T = static_cast<size_t>(h.Bmax) * h.plan.layers[l].l_q;
  L.moe_sel = h.dalloc<int32_t>(T * h.moe_k);
  L.moe_w = h.dalloc<float>(T * h.moe_k);
}

// MoE workspace sized for the largest layer: expert g owns rows [g Tcap, (g + 1) Tcap) of the
// expert-sorted buffers (Tcap = the layer's token count rounded up to 128), so routing can
// place rows before the expert loads are known.
static void ensure_moe_buffers(Handle& h) {
  int tq = 0;
  for (const LayerPlan& lp : h.plan.layers) tq = std::max(tq, lp.l_q);
  const size_t T = static_cast<size_t>(h.Bmax) * tq;
  const size_t Tcap = (T + 127) / 128 * 128;
  const int G = h.moe_E + h.moe_s, S = h.moe_k + h.moe_s;
  h.moe_pmax = static_cast<int>(static_cast<size_t>(G) * Tcap);
  h.moe_tiles_max = static_cast<int>(T * S / 128 + G + 1);
  const size_t P = h.moe_pmax;
  h.moe_xs = h.dalloc<__nv_bfloat16>(P * h.d);
  h.moe_hs = h.dalloc<__nv_bfloat16>(P * h.moe_m);
  h.moe_ys = h.dalloc<__nv_bfloat16>(P * h.d);
  h.moe_tok = h.dalloc<int32_t>(P);
  h.moe_wof = h.dalloc<float>(P);
  h.moe_slot = h.dalloc<int32_t>(T * S);
  h.moe_inv = h.dalloc<float>(T);
  h.moe_off = h.dalloc<int32_t>(G + 1);
  h.moe_cursor = h.dalloc<int32_t>(G + 1);
  h.moe_tile_group = h.dalloc<int32_t>(h.moe_tiles_max + 1);
  h.moe_tile_mblk = h.dalloc<int32_t>(h.moe_tiles_max + 1);
  h.moe_ntiles = h.dalloc<int32_t>(1);
  h.moe_counts = h.dalloc<int32_t>(static_cast<size_t>(h.cfg.layers) * h.moe_E);
  CK(cudaMemset(h.moe_counts, 0, static_cast<size_t>(h.cfg.layers) * h.moe_E * 4));
  h.tmA_moe_xs = make_tmap_2d(h.moe_xs, P, h.d, h.d, 128, 64, 128);
  h.tmA_moe_hs = make_tmap_2d(h.moe_hs, P, h.moe_m, h.moe_m, 128, 64, 128);
  h.tmY_moe = make_tmap_2d(h.moe_ys, P, h.d, h.d, 128, 64, 128);
}

// g . W1 of the ranking head as three bf16 pieces for the tensor-core head (misc.cuh GsHead);
// rebuilt whenever the weights change (finalize, repack_weights)
static void head_wsplit(Handle& h) {
  const int n = h.d * h.dh;
  k_head_wsplit<<<std::min((n + 255) / 256, 148 * 8), 256, 0, h.stream>>>(h.head_w1, h.head_gain, h.d, h.dh, h.head_wt);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw RuntimeFailure(std::string("head weight split launch failed: ") + cudaGetErrorString(e));
}

static void finalize(Handle& h) {
  const SortConfig& c = h.cfg;
  const int d = h.d, m = h.m, H = h.H, dk = h.dk;
  // ---- tokenizer tables and projections (tokenizer.cpp:45-63)
  h.item = h.upload(to_bf16(need_param(h, "tok.item_table", c.n_items, c.item_dim).v));
  h.action = h.upload(to_bf16(need_param(h, "tok.action_table", c.n_actions, c.action_dim).v));
  h.scene = h.upload(to_bf16(need_param(h, "tok.scene_table", c.n_scenes, c.scene_dim).v));
  h.time = h.upload(to_bf16(need_param(h, "tok.time_table", c.n_time_buckets, c.time_dim).v));
  {
    std::vector<float> all;
    int off = 0;
    for (int f = 0; f < c.n_profile_fields; ++f) {
      const HostParam& t = need_param(h, "tok.profile_table." + std::to_string(f), c.profile_vocab[f], c.profile_dim);
      h.prof_off[f] = off;
      off += c.profile_vocab[f];
      all.insert(all.end(), t.v.begin(), t.v.end());
    }
    if (all.empty()) all.assign(8, 0.f);
    h.prof = h.upload(to_bf16(all));
  }
  h.special = h.upload(to_bf16(need_param(h, "tok.special", 3, d).v));
  const int hw = c.item_dim + c.action_dim + c.scene_dim + c.time_dim;
  const char* gw[3] = {"tok.w_hist", "tok.w_cand", "tok.w_prof"};
  const char* gb[3] = {"tok.b_hist", "tok.b_cand", "tok.b_prof"};
  const char* gg[3] = {"tok.g_hist", "tok.g_cand", "tok.g_prof"};
  const int gk[3] = {hw, c.item_dim, c.profile_dim};
  for (int g = 0; g < 3; ++g) {
    if (!h.generic) h.tok_wt[g] = h.upload(transpose_bf16(need_param(h, gw[g], gk[g], d), 64, nullptr));
    h.tok_b[g] = h.upload(need_param(h, gb[g], 1, d).v);
    h.tok_g[g] = h.upload(need_param(h, gg[g], 1, d).v);
  }
  // ---- RoPE table in fp64 (rope.hpp:23-38), stored fp32 (cos, sin)
  {
    std::vector<float2> tab(static_cast<size_t>(h.plan.max_pos + 1) * (dk / 2));
    for (int p = 0; p <= h.plan.max_pos; ++p)
      for (int j = 0; j < dk / 2; ++j) {
        const double freq = std::pow(c.rope_theta, -2.0 * j / static_cast<double>(dk));
        const double ang = static_cast<double>(p) * freq;
        tab[static_cast<size_t>(p) * (dk / 2) + j] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
      }
    h.rope = h.upload(tab);
  }
  // ---- workspace
  const size_t rows_max = static_cast<size_t>(h.Bmax) * h.L0;
  for (int i = 0; i < 2; ++i) {
    h.X[i] = h.dalloc<__nv_bfloat16>(rows_max * d);
    h.SS[i] = h.dalloc<float4>(rows_max);
    h.tmSS[i] = make_tmap_2d_f32(h.SS[i], rows_max, 4, 128, 4, 0);
  }
  h.Qb = h.dalloc<__nv_bfloat16>(rows_max * d);
  h.Kb = h.dalloc<__nv_bfloat16>(rows_max * d);
  h.Vb = h.dalloc<__nv_bfloat16>(rows_max * d);
  h.Gb = h.dalloc<__nv_bfloat16>(rows_max * d);
  h.Hg = h.dalloc<__nv_bfloat16>(rows_max * d);
  h.hid = h.dalloc<__nv_bfloat16>(rows_max * m);
  h.probs = h.dalloc<float>(static_cast<size_t>(h.Bmax) * c.n_cand * 3);
  h.logits = h.dalloc<float>(static_cast<size_t>(h.Bmax) * c.n_cand * 3);
  h.err = h.dalloc<int32_t>(4);
  CK(cudaMemset(h.err, 0, 4 * sizeof(int32_t)));
  h.hist_time = h.dalloc<int32_t>(static_cast<size_t>(h.Bmax) * std::max(c.n_hist, 1));
  const size_t BH_ = static_cast<size_t>(h.Bmax) * std::max(c.n_hist, 1);
  h.in_item = h.dalloc<int32_t>(BH_);
  h.in_action = h.dalloc<int32_t>(BH_);
  h.in_scene = h.dalloc<int32_t>(BH_);
  h.in_ts = h.dalloc<int64_t>(BH_);
  h.in_req = h.dalloc<int64_t>(h.Bmax);
  h.in_prof = h.dalloc<int32_t>(static_cast<size_t>(h.Bmax) * std::max(c.n_profile_fields, 1));
  h.in_cand = h.dalloc<int32_t>(static_cast<size_t>(h.Bmax) * c.n_cand);
  h.in_slot[0] = {h.in_item, h.in_action, h.in_scene, h.in_prof, h.in_cand, h.in_ts, h.in_req};

  // ---- per-layer weights, plan arrays and TMA descriptors
  int cur = 0;
  h.layers.resize(c.layers);
  for (int l = 0; l < c.layers; ++l) {
    const LayerPlan& lp = h.plan.layers[l];
    LayerDev& L = h.layers[l];
    const std::string a = "attn." + std::to_string(l) + ".";
    const std::string bk = "block." + std::to_string(l) + ".";
    const std::string f = "ffn." + std::to_string(l) + ".";
    const HostParam& ga = need_param(h, bk + "attn_norm", 1, d);
    const HostParam& gf = need_param(h, bk + "ffn_norm", 1, d);
    if (!h.generic) {  // Q/K/V/G projections: W^T rows interleaved head by head in section
                       // order `order`, attention pre-norm gain folded into the input rows.
      const std::string names[4] = {"wq", "wk", "wv", "wg"};  // kSecQ, kSecK, kSecV, kSecG
      std::vector<__nv_bfloat16> t[4];
      for (int sct = 0; sct < 4; ++sct) t[sct] = transpose_bf16(need_param(h, a + names[sct], d, d), d, ga.v.data());
      auto build = [&](const std::vector<int>& order) {
        std::vector<__nv_bfloat16> w;
        w.reserve(order.size() * static_cast<size_t>(d) * d);
        for (int hd = 0; hd < H; ++hd)
          for (int sct : order)
            w.insert(w.end(), t[sct].begin() + static_cast<size_t>(hd) * dk * d,
                     t[sct].begin() + static_cast<size_t>(hd + 1) * dk * d);
        return h.upload(w);
      };
      L.w_all = build({kSecQ, kSecV, kSecK, kSecG});
      L.w_kv = build({kSecK, kSecV});
      L.w_qg = build({kSecQ, kSecG});
    }
    if (!h.generic) L.w_o = h.upload(transpose_bf16(need_param(h, a + "wo", d, d), d, nullptr));
    if (h.moe) build_moe_layer(h, l, L);
    if (!h.generic && !h.moe) {  // SwishGLU up: interleave 32-column blocks [gate_j | up_j], ffn pre-norm gain folded
      const HostParam& wg = need_param(h, f + "w_gate", d, m);
      const HostParam& wu = need_param(h, f + "w_up", d, m);
      std::vector<__nv_bfloat16> w(static_cast<size_t>(2) * m * d);
      for (int j = 0; j < m / 32; ++j)
        for (int i = 0; i < 64; ++i) {
          const HostParam& src = i < 32 ? wg : wu;
          const int col = 32 * j + (i & 31);
          const size_t row = static_cast<size_t>(64 * j + i);
          for (int k = 0; k < d; ++k) w[row * d + k] = f2bf(src.v[static_cast<size_t>(k) * m + col] * gf.v[k]);
        }
      L.w_up = h.upload(w);
    }
    if (!h.generic && !h.moe) L.w_down = h.upload(transpose_bf16(need_param(h, f + "w_down", m, d), m, nullptr));
    {
      const HostParam& gq = need_param(h, a + "qk_gain_q", H, dk);
      const HostParam& gk = need_param(h, a + "qk_gain_k", H, dk);
      L.gain_q = h.upload(gq.v);
      L.gain_k = h.upload(gk.v);
      // |q.k| / sqrt(dk) <= sqrt(dk) * max|g_q| * max|g_k| for every head (QKNorm + RoPE
      // rotation); 2% margin for the bf16 rounding of q and k.
      float mq = 0.f, mk = 0.f;
      for (float v : gq.v) mq = std::max(mq, std::fabs(v));
      for (float v : gk.v) mk = std::max(mk, std::fabs(v));
      L.logit_bound = 1.02f * std::sqrt(static_cast<float>(dk)) * mq * mk + 1e-3f;
      std::vector<float> gs(gq.v);
      const float sl2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(dk)));
      for (float& v : gs) v *= sl2;
      L.gain_q_s = h.upload(gs);
    }
    // plan arrays
    std::vector<int4> meta(static_cast<size_t>(lp.n_qtiles) * 128, make_int4(0, -1, -1, 0));
    for (int r = 0; r < lp.l_q; ++r) meta[r] = make_int4(lp.lo[r], lp.hi[r], lp.self_idx[r], 0);
    L.rowmeta = h.upload(meta);
    L.tile_off = h.upload(lp.tile_off);
    L.tile_code = h.upload(lp.tile_code.empty() ? std::vector<int32_t>{0, 0} : lp.tile_code);
    L.qtile_order = h.upload(lp.qtile_order);
    L.pos_q = h.upload(lp.pos_q);
    L.pos_kv = h.upload(lp.pos_kv);
    L.query_rows = h.upload(lp.query_rows);
    L.Rq = lp.l_q;
    L.Rkv = lp.l_kv;
    L.in_buf = cur;
    L.q_buf = lp.q_identity ? cur : 1 - cur;
    cur = L.q_buf;
    if (!h.generic) {
    // GEMM tile widths (weight-stationary: BN x K weight slice resident in smem)
    auto pick_bn = [&](int N, int K, int chunk, uint32_t side = 0) {
      for (int bn = 256; bn >= chunk; bn /= 2)
        if (N % bn == 0 && bn % chunk == 0 && gemm_plan(K, bn, side).a_stages >= 2) return bn;
      throw ConfigError("unsupported GEMM shape N=" + std::to_string(N) + " K=" + std::to_string(K));
    };
    const uint32_t qkvg_side = side_bytes(3, dk);
    L.bn_full = pick_bn(4 * d, d, 4 * dk, qkvg_side);
    L.bn_half = pick_bn(2 * d, d, 2 * dk, qkvg_side);
    L.bn_o = pick_bn(d, d, 32);
    if (!h.moe) {
      L.bn_up = pick_bn(2 * m, d, 64, side_bytes(1, 0));
      L.bn_down = pick_bn(d, m, 32);
    }
    // TMA descriptors (sized for max_batch; launches use the call's batch)
    const uint64_t Mkv = static_cast<uint64_t>(h.Bmax) * L.Rkv, Mq = static_cast<uint64_t>(h.Bmax) * L.Rq;
    L.tmA_in = make_tmap_2d(h.X[L.in_buf], Mkv, d, d, 128, 64, 128);
    L.tmA_q = make_tmap_2d(h.X[L.q_buf], Mq, d, d, 128, 64, 128);
    L.tmB_all = make_tmap_2d(L.w_all, 4 * d, d, d, L.bn_full, 64, 128);
    L.tmB_qg = make_tmap_2d(L.w_qg, 2 * d, d, d, L.bn_half, 64, 128);
    L.tmB_kv = make_tmap_2d(L.w_kv, 2 * d, d, d, L.bn_half, 64, 128);
    L.tmB_all_p = make_tmap_2d(L.w_all, 4 * d, d, d, L.bn_full / 2, 64, 128);
    L.tmB_qg_p = make_tmap_2d(L.w_qg, 2 * d, d, d, L.bn_half / 2, 64, 128);
    L.tmB_kv_p = make_tmap_2d(L.w_kv, 2 * d, d, d, L.bn_half / 2, 64, 128);
    L.tmA_hg = make_tmap_2d(h.Hg, Mq, d, d, 128, 64, 128);
    L.tmB_o = make_tmap_2d(L.w_o, d, d, d, L.bn_o, 64, 128);
    if (!h.moe) L.tmB_up = make_tmap_2d(L.w_up, 2 * m, d, d, L.bn_up, 64, 128);
    L.tmRopeKV = rope_table(h, L.Rkv, lp.pos_kv);
    L.tmRopeQ = rope_table(h, L.Rq, lp.pos_q);
    L.tmA_hid = make_tmap_2d(h.hid, Mq, m, m, 128, 64, 128);
    if (!h.moe) L.tmB_down = make_tmap_2d(L.w_down, d, m, m, L.bn_down, 64, 128);
    if (tail_supported(h)) {
      L.tmWo_t = make_tmap_2d(L.w_o, d, d, d, d, 64, 128);
      L.tmWup_t = make_tmap_2d(L.w_up, 2 * m, d, d, 128, 64, 128);
      L.tmWdown_t = make_tmap_2d(L.w_down, d, m, m, d, 64, 128);
      L.tmWo_p = make_tmap_2d(L.w_o, d, d, d, d / 2, 64, 128);
      L.tmWup_p = make_tmap_2d(L.w_up, 2 * m, d, d, 64, 64, 128);
      L.tmWdown_p = make_tmap_2d(L.w_down, d, m, m, d / 2, 64, 128);
    }
    }  // !generic
    {
      const uint64_t BH = static_cast<uint64_t>(h.Bmax) * H;
      uint64_t dq[3] = {static_cast<uint64_t>(dk), static_cast<uint64_t>(L.Rq), BH};
      uint64_t sq[2] = {static_cast<uint64_t>(dk) * 2, static_cast<uint64_t>(L.Rq) * dk * 2};
      uint32_t bq[3] = {static_cast<uint32_t>(dk), 128, 1};
      L.tmQ = make_tmap_bf16(h.Qb, 3, dq, sq, bq, dk * 2);
      uint64_t dkd[3] = {static_cast<uint64_t>(dk), static_cast<uint64_t>(L.Rkv), BH};
      uint64_t skd[2] = {static_cast<uint64_t>(dk) * 2, static_cast<uint64_t>(L.Rkv) * dk * 2};
      L.tmK = make_tmap_bf16(h.Kb, 3, dkd, skd, bq, dk * 2);
      L.tmV = make_tmap_bf16(h.Vb, 3, dkd, skd, bq, dk * 2);
    }
  }
  // ---- head (fp32)
  need_param(h, "final_norm.gain", 1, d);
  if (c.pretrain) {
    h.frozen.clear();  // pre-training learns the item table (the tables transfer_sparse copies)
    if (c.item_dim != kPreK) throw ConfigError("pretrain: the tied head needs item_dim == 32 in this build");
    need_param(h, "pretrain.proj", d, c.item_dim);
    h.pre_hp = h.dalloc<__nv_bfloat16>(static_cast<size_t>(h.Bmax) * h.L0 * kPreK);
    h.pre_lse = h.dalloc<float>(static_cast<size_t>(h.Bmax) * c.n_hist);
    h.pre_tgt = h.dalloc<float>(static_cast<size_t>(h.Bmax) * c.n_hist);
  } else {
    need_param(h, "head.w1", d, h.dh);
    need_param(h, "head.b1", 1, h.dh);
    need_param(h, "head.w2", h.dh, 3);
    need_param(h, "head.b2", 1, 3);
  }
  // fp32 copies of the differentiated parameters (training backward), and the flat gradient
  // buffer in the same name order; W_gate | W_up also concatenated as ffn.<l>.w_gu [d, 2m]
  // Trainable parameters: every tensor except the (frozen) item table, one flat fp32 master
  // buffer in name order; the gradient buffer and the AdamW moments share its layout.
  size_t goff = 0;
  for (auto& kv : h.host) {
    if (kv.first == "tok.item_table") continue;
    goff = (goff + 3) & ~static_cast<size_t>(3);  // 16-byte aligned tensors (vector / cp.async loads)
    h.grad_index[kv.first] = {goff, {kv.second.rows, kv.second.cols}};
    goff += static_cast<size_t>(kv.second.rows) * kv.second.cols;
  }
  h.master = h.dalloc<float>(std::max<size_t>(goff, 1));
  CK(cudaMemset(h.master, 0, std::max<size_t>(goff, 1) * sizeof(float)));  // alignment gaps
  for (auto& kv : h.grad_index) {
    const HostParam& hp = h.host.at(kv.first);
    CK(cudaMemcpy(h.master + kv.second.first, hp.v.data(), hp.v.size() * 4, cudaMemcpyHostToDevice));
    h.w32[kv.first] = h.master + kv.second.first;
  }
  for (int l = 0; l < c.layers && !h.moe; ++l) {
    const std::string f = "ffn." + std::to_string(l) + ".";
    const HostParam& wg = h.host.at(f + "w_gate");
    const HostParam& wu = h.host.at(f + "w_up");
    std::vector<float> gu(static_cast<size_t>(d) * 2 * m);
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < m; ++j) {
        gu[static_cast<size_t>(i) * 2 * m + j] = wg.v[static_cast<size_t>(i) * m + j];
        gu[static_cast<size_t>(i) * 2 * m + m + j] = wu.v[static_cast<size_t>(i) * m + j];
      }
    h.w32[f + "w_gu"] = h.upload(gu);
  }
  h.grad_count = goff;
  // fp32 parameters the inference kernels read directly now live in the master buffer, so
  // an optimizer step updates them in place
  h.head_gain = h.w32["final_norm.gain"];
  if (c.pretrain) h.pre_proj = h.w32["pretrain.proj"];
  h.head_w1 = h.w32["head.w1"];
  h.head_b1 = h.w32["head.b1"];
  h.head_w2 = h.w32["head.w2"];
  h.head_b2 = h.w32["head.b2"];
  const char* gnames[3] = {"hist", "cand", "prof"};
  for (int g = 0; g < 3; ++g) {
    h.tok_b[g] = h.w32[std::string("tok.b_") + gnames[g]];
    h.tok_g[g] = h.w32[std::string("tok.g_") + gnames[g]];
  }
  for (int l = 0; l < c.layers; ++l) {
    h.layers[l].gain_q = h.w32["attn." + std::to_string(l) + ".qk_gain_q"];
    h.layers[l].gain_k = h.w32["attn." + std::to_string(l) + ".qk_gain_k"];
    if (h.moe) {  // router and balancing bias read (and updated) in the master buffer
      h.layers[l].router = h.w32["ffn." + std::to_string(l) + ".router"];
      h.layers[l].router_bias = h.w32["ffn." + std::to_string(l) + ".router_bias"];
    }
  }
  if (h.moe) ensure_moe_buffers(h);
  if (!c.pretrain && !h.generic && h.d % 64 == 0 && h.dh % 32 == 0 && h.dh <= 256) {  // the SORT-base head path
    const size_t rows = static_cast<size_t>(h.Bmax) * c.n_cand;
    h.head_wt = h.dalloc<__nv_bfloat16>(static_cast<size_t>(h.dh) * 3 * h.d);
    h.head_xc = h.dalloc<__nv_bfloat16>(rows * h.d);
    h.head_ssc = h.dalloc<float4>(rows);
    h.head_zp = h.dalloc<float>(static_cast<size_t>(6) * rows);  // [2 halves][3][rows]
    head_wsplit(h);
  }
  h.host.clear();  // device copies are authoritative from here on
  h.finalized = true;
}

// cudaFuncSetAttribute is per device: the largest dynamic shared memory set so far is
// remembered per (device, kernel), so handles on several GPUs in one process all get it.
static void ensure_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = done[{dev, fn}];
  if (bytes > cur) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    cur = bytes;
  }
}
template <class F>
static void ensure_smem(F* fn, size_t bytes) {
  ensure_smem(reinterpret_cast<const void*>(fn), bytes);
}

// ------------------------------------------------------------------ launches
// Grid of a persistent kernel that walks work items `it = blockIdx.x + k * grid` laid out
// (request, head)-major with `period` tiles of unequal cost per (request, head) (the q-tiles
// of an attention layer, heaviest first): with gcd(grid, period) > 1 a CTA would only ever
// see some of the ranks -- at a pruned layer (period 2: the 128 retained rows and the
// candidate tile) and 2 x 148 CTAs, every even CTA got only the heavy candidate tiles. The
// largest grid <= want coprime to the period makes every CTA cycle through all ranks.
static int coprime_grid(int want, int period) {
  if (period <= 1) return std::max(1, want);
  for (int g = want; g > 1; --g)
    if (std::gcd(g, period) == 1) return g;
  return 1;
}

static void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw RuntimeFailure(std::string(what) + " launch failed: " + cudaGetErrorString(e));
}

template <class Epi>
static void launch_gemm(Handle& h, const CUtensorMap& A, const CUtensorMap& B, int M, int N, int K,
                        int BN, const Epi& epi, const CUtensorMap* side_stats = nullptr,
                        const CUtensorMap* side_rope = nullptr) {
  const GemmPlan gp = gemm_plan(K, BN, side_bytes(Epi::kSide, Epi::kRopeFloats));
  if (N % BN || gp.a_stages < 2) throw RuntimeFailure("gemm: unsupported tile plan");
  if (((Epi::kSide & 1) && !side_stats) || ((Epi::kSide & 2) && !side_rope))
    throw RuntimeFailure("gemm: epilogue side data missing");
  ensure_smem(k_gemm_bf16<Epi>, gp.smem_bytes);
  const int num_m = (M + kGemmBM - 1) / kGemmBM;
  const int grid = gemm_grid(num_m, N / BN, h.num_sms);
  k_gemm_bf16<Epi><<<grid, kGemmThreads, gp.smem_bytes, h.stream>>>(
      A, B, side_stats ? *side_stats : A, side_rope ? *side_rope : A, M, N, K, BN, gp.a_stages, epi);
  check_launch("gemm");
  ++h.launches;
}

// Grouped (MoE expert) GEMM: A = expert-sorted rows padded per expert to 128, B = the stacked
// expert weights; the m-block count and each block's expert are read on the device.
template <class Epi>
static void launch_gemm_grouped(Handle& h, const CUtensorMap& A, const CUtensorMap& B, int N, int K, int BN,
                                const Epi& epi) {
  static_assert(is_grouped<Epi>::value, "grouped epilogue expected");
  const GemmPlan gp = gemm_plan(K, BN, 0, 1, 2);
  if (N % BN || gp.a_stages < 2) throw RuntimeFailure("grouped gemm: unsupported tile plan");
  ensure_smem(k_gemm_bf16<Epi>, gp.smem_bytes);
  const int grid = gemm_grid(h.moe_tiles_max, N / BN, h.num_sms);
  k_gemm_bf16<Epi><<<grid, kGemmThreads, gp.smem_bytes, h.stream>>>(A, B, A, A, h.moe_pmax, N, K, BN,
                                                                      gp.a_stages, epi);
  check_launch("grouped gemm");
  ++h.launches;
}

// The same GEMM as CTA pairs (cluster of 2, tcgen05 cta_group::2); B is the pair map whose
// box holds BN/2 weight rows.
template <class Epi>
static void launch_gemm_pair(Handle& h, const CUtensorMap& A, const CUtensorMap& B, int M, int N, int K, int BN,
                             const Epi& epi, const CUtensorMap* side_stats, const CUtensorMap* side_rope) {
  const GemmPlan gp = gemm_plan(K, BN, side_bytes(Epi::kSide, Epi::kRopeFloats), 2);
  if (N % BN || gp.a_stages < 2) throw RuntimeFailure("gemm: unsupported tile plan");
  ensure_smem(k_gemm_bf16<Epi, true>, gp.smem_bytes);
  const int num_m2 = (M + 2 * kGemmBM - 1) / (2 * kGemmBM);
  const int units = gemm_grid(num_m2, N / BN, h.num_sms / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * units);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = gp.smem_bytes;
  cfg.stream = h.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_gemm_bf16<Epi, true>, A, B, side_stats ? *side_stats : A,
                        side_rope ? *side_rope : A, M, N, K, BN, gp.a_stages, epi));
  check_launch("gemm (pair)");
  ++h.launches;
}

// Inference with bounded logits: Q leaves the QKVG epilogue multiplied by log2(e)/sqrt(dk)
// (gain_q_s) and k_attention<.., kPre> exponentiates S directly. Training keeps the unscaled Q
// (the backward recomputes S from it).
static bool attn_prescaled(const Handle& h, const LayerDev& L) {
  return h.attn_prescale && !h.training && L.gain_q_s && L.logit_bound > 0.f && L.logit_bound < kFixedRefMax;
}

template <int DK, bool kFixed, bool kPre = false>
static void launch_attention_dk(Handle& h, const LayerDev& L, const LayerPlan& lp, int B) {
  const int n_codes = static_cast<int>(lp.tile_code.size()) / 2;  // {kv_tile, classes} pairs
  AttnArgs a;
  a.rowmeta = L.rowmeta;
  a.tile_off = L.tile_off;
  a.tile_code = reinterpret_cast<const int2*>(L.tile_code);
  a.qtile_order = L.qtile_order;
  a.g = h.save_to ? h.save_to->g : h.Gb;
  a.out = h.Hg;
  a.o_pre = nullptr;
  a.lse = nullptr;
  if (h.training) {
    const int li = static_cast<int>(&L - h.layers.data());
    a.o_pre = h.tl[li].o_pre;
    a.lse = h.tl[li].lse;
  }
  a.BH = B * h.H;
  a.H = h.H;
  a.Rq = L.Rq;
  a.d = h.d;
  a.n_qtiles = lp.n_qtiles;
  a.n_codes = n_codes;
  a.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(DK)));
  // fixed softmax reference in log2 units: the exponent is s * log2e with s = S / sqrt(dk) the
  // scaled logit, |s| <= logit_bound, so the reference is logit_bound * log2e (every P <= 1)
  a.ref_log2 = L.logit_bound * 1.4426950408889634f;
  const int n_items = lp.n_qtiles * B * h.H;
  const int tile_ints = 2 * lp.n_qtiles + 2 + 2 * n_codes;
  const CUtensorMap& tq = h.save_to ? h.save_to->tmQ : L.tmQ;
  const CUtensorMap& tk = h.save_to ? h.save_to->tmK : L.tmK;
  const CUtensorMap& tv = h.save_to ? h.save_to->tmV : L.tmV;
  const size_t smem = AttnSmem<DK>::bytes(tile_ints);
  ensure_smem(k_attention<DK, kFixed, kPre>, smem);
  const int grid = coprime_grid(std::min(n_items, AttnTmem<DK>::kCtasPerSm * h.num_sms), lp.n_qtiles);
  k_attention<DK, kFixed, kPre><<<grid, kAttnThreads, smem, h.stream>>>(tq, tk, tv, a);
  check_launch("attention");
  ++h.launches;
}

static void launch_attention(Handle& h, const LayerDev& L, const LayerPlan& lp, int B) {
  const bool fixed = L.logit_bound > 0.f && L.logit_bound < kFixedRefMax;
  if (attn_prescaled(h, L)) {
    switch (h.dk) {
      case 16: launch_attention_dk<16, true, true>(h, L, lp, B); return;
      case 32: launch_attention_dk<32, true, true>(h, L, lp, B); return;
      case 64: launch_attention_dk<64, true, true>(h, L, lp, B); return;
      default: throw ConfigError("unsupported head dim");
    }
  }
  switch (h.dk * 2 + (fixed ? 1 : 0)) {
    case 32: launch_attention_dk<16, false>(h, L, lp, B); break;
    case 33: launch_attention_dk<16, true>(h, L, lp, B); break;
    case 64: launch_attention_dk<32, false>(h, L, lp, B); break;
    case 65: launch_attention_dk<32, true>(h, L, lp, B); break;
    case 128: launch_attention_dk<64, false>(h, L, lp, B); break;
    case 129: launch_attention_dk<64, true>(h, L, lp, B); break;
    default: throw ConfigError("unsupported head dim");
  }
}

template <int DK>
static void launch_qkvg_dk(Handle& h, const LayerDev& L, const CUtensorMap& A, const CUtensorMap& Bm,
                           int M, int N, int BN, int R, const std::vector<int>& order,
                           const CUtensorMap& tmS, const CUtensorMap& tmR, const CUtensorMap* Bpair) {
  EpiQKVG<DK> e;
  e.d = h.d;
  e.H = h.H;
  e.R = R;
  const int ns = static_cast<int>(order.size());
  for (int ci = 0; ci < N / DK && ci < 64; ++ci) {
    e.csec[ci] = static_cast<uint8_t>(order[ci % ns]);
    e.chead[ci] = static_cast<uint8_t>(ci / ns);
  }
  e.inv_d = 1.f / static_cast<float>(h.d);
  e.gain_q = attn_prescaled(h, L) ? L.gain_q_s : L.gain_q;
  e.gain_k = L.gain_k;
  e.q = h.save_to ? h.save_to->q : h.Qb;
  e.k = h.save_to ? h.save_to->k : h.Kb;
  e.v = h.save_to ? h.save_to->v : h.Vb;
  e.g = h.save_to ? h.save_to->g : h.Gb;
  e.Rq = L.Rq;
  e.Rkv = L.Rkv;
  if (Bpair && h.qkvg_pair)
    launch_gemm_pair(h, A, *Bpair, M, N, h.d, BN, e, &tmS, &tmR);
  else
    launch_gemm(h, A, Bm, M, N, h.d, BN, e, &tmS, &tmR);
}

static void launch_qkvg(Handle& h, const LayerDev& L, const CUtensorMap& A, const CUtensorMap& Bm,
                        int M, int N, int BN, int R, const std::vector<int>& sec,
                        const CUtensorMap& tmS, const CUtensorMap& tmR, const CUtensorMap* Bpair = nullptr) {
  if (N / h.dk > 64) throw ConfigError("unsupported: more than 64 head chunks per projection");
  switch (h.dk) {
    case 16: launch_qkvg_dk<16>(h, L, A, Bm, M, N, BN, R, sec, tmS, tmR, Bpair); break;
    case 32: launch_qkvg_dk<32>(h, L, A, Bm, M, N, BN, R, sec, tmS, tmR, Bpair); break;
    case 64: launch_qkvg_dk<64>(h, L, A, Bm, M, N, BN, R, sec, tmS, tmR, Bpair); break;
    default: throw ConfigError("unsupported head dim");
  }
}

template <int D, bool kPair>
static void launch_tail_dp(Handle& h, const LayerDev& L, float4* SSq, int M, __nv_bfloat16* x1_out) {
  ensure_smem(k_block_tail<D, kPair>, TailSmem<D>::bytes);
  TailArgs ta;
  ta.x1_out = x1_out;
  ta.ss_out = reinterpret_cast<float*>(SSq);
  ta.M = M;
  ta.m = h.m;
  ta.inv_d = 1.f / static_cast<float>(h.d);
  if constexpr (kPair) {
    const int units = (M + 255) / 256;
    const int pairs = std::min(units, h.num_sms / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kTailThreads);
    cfg.dynamicSmemBytes = TailSmem<D>::bytes;
    cfg.stream = h.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_block_tail<D, true>, L.tmA_hg, L.tmWo_p, L.tmWup_p, L.tmWdown_p, L.tmA_q, L.tmA_q,
                          ta));
  } else {
    const int num_m = (M + 127) / 128;
    const int grid = std::min(num_m, h.num_sms);
    k_block_tail<D, false><<<grid, kTailThreads, TailSmem<D>::bytes, h.stream>>>(L.tmA_hg, L.tmWo_t, L.tmWup_t,
                                                                                L.tmWdown_t, L.tmA_q, L.tmA_q, ta);
  }
  check_launch("block_tail");
  ++h.launches;
}

template <int D>
static void launch_tail_d(Handle& h, const LayerDev& L, __nv_bfloat16*, float4* SSq, int M,
                          __nv_bfloat16* x1_out = nullptr) {
  if (h.tail_pair) {
    launch_tail_dp<D, true>(h, L, SSq, M, x1_out);
  } else {
    launch_tail_dp<D, false>(h, L, SSq, M, x1_out);
  }
}

static void stage_mark(Handle& h, const std::string& name) {
  if (!h.timing) return;
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  CK(cudaEventRecord(e, h.stream));
  h.events.push_back(e);
  h.stage_names.push_back(name);
}

static TokParams tok_params(Handle& h, int B) {
  const SortConfig& c = h.cfg;
  TokParams p{};
  p.item_tab = h.item_ext ? h.item_ext : h.item;
  p.action_tab = h.action;
  p.scene_tab = h.scene;
  p.time_tab = h.time;
  p.prof_tab = h.prof;
  p.special = h.special;
  for (int f = 0; f < c.n_profile_fields; ++f) {
    p.prof_row_off[f] = h.prof_off[f];
    p.prof_vocab[f] = c.profile_vocab[f];
  }
  for (int g = 0; g < 3; ++g) {
    p.wt[g] = h.tok_wt[g];
    p.bias[g] = h.tok_b[g];
    p.gain[g] = h.tok_g[g];
  }
  p.hist_item = h.in_item;
  p.hist_action = h.in_action;
  p.hist_scene = h.in_scene;
  p.hist_ts = h.in_ts;
  p.req_ts = h.in_req;
  p.profile = h.in_prof;
  p.cand_item = h.in_cand;
  p.x = h.X[0];
  p.ss = h.SS[0];
  p.hist_time = h.hist_time;
  p.err = h.err;
  p.B = B;
  p.H = c.n_hist;
  p.P = c.n_profile_fields;
  p.N = c.n_cand;
  p.L = h.L0;
  p.d = h.d;
  p.item_dim = c.item_dim;
  p.action_dim = c.action_dim;
  p.scene_dim = c.scene_dim;
  p.time_dim = c.time_dim;
  p.prof_dim = c.profile_dim;
  p.n_items = h.item_ext ? static_cast<int>(h.item_ext_rows) : c.n_items;
  p.n_actions = c.n_actions;
  p.n_scenes = c.n_scenes;
  p.n_tb = c.n_time_buckets;
  p.special_tokens = c.special_tokens;
  p.click_seq = c.pretrain;
  p.tiles_hist = (B * c.n_hist + 127) / 128;
  p.tiles_cand = (B * c.n_cand + 127) / 128;
  p.tiles_prof = (B * c.n_profile_fields + 127) / 128;
  return p;
}

static void run_tokenizer(Handle& h, int B) {
  const TokParams p = tok_params(h, B);
  const size_t smem = tok_smem_bytes(h.d);
  ensure_smem(k_tokenize, smem);
  const int tiles = p.tiles_hist + p.tiles_cand + p.tiles_prof;
  const int grid = std::max(1, std::min(tiles, 2 * h.num_sms));
  k_tokenize<<<grid, kTokThreads, smem, h.stream>>>(p);
  check_launch("tokenizer");
  ++h.launches;
}

// MoE FFN of layer l on the T rows of X (in place): x <- x + MoE(RMSNorm(x)) (SPEC.md:375 with
// the FFN of SPEC.md:272-351), row statistics refreshed for the next layer. See moe.cuh.
static void run_moe(Handle& h, int l, __nv_bfloat16* X, float4* SS, int T) {
  LayerDev& L = h.layers[l];
  const int d = h.d, E = h.moe_E, k = h.moe_k, S = h.moe_s, me = h.moe_m;
  const int Tcap = (T + 127) / 128 * 128;
  if (static_cast<int64_t>(E + S) * Tcap > h.moe_pmax || T * (k + S) / 128 + E + S + 1 > h.moe_tiles_max)
    throw RuntimeFailure("moe: workspace too small");
  int32_t* counts = h.moe_counts + static_cast<size_t>(l) * E;
  const float* gain = h.w32.at("block." + std::to_string(l) + ".ffn_norm");
  ensure_smem(k_moe_route, (256 * kMoeMaxExperts + 8 * 32 * (kMoeMaxExperts + 1)) * 4);
  CK(cudaMemsetAsync(counts, 0, static_cast<size_t>(E) * 4, h.stream));
  if (E <= 8 && k <= 2) {  // routing and scatter in one pass; the cursors end as the loads
    const int grid = std::max(1, std::min((T + 255) / 256, kRouteCtasPerSm * h.num_sms));
    ensure_smem(k_moe_route_scatter8<1>, kRouteSmem);
    ensure_smem(k_moe_route_scatter8<2>, kRouteSmem);
    if (k == 1)
      k_moe_route_scatter8<1><<<grid, 256, kRouteSmem, h.stream>>>(X, T, d, gain, L.router, L.router_bias, E, S, Tcap,
                                                          L.moe_sel, L.moe_w, counts, h.moe_xs, h.moe_tok, h.moe_wof,
                                                          h.moe_slot, h.err);
    else
      k_moe_route_scatter8<2><<<grid, 256, kRouteSmem, h.stream>>>(X, T, d, gain, L.router, L.router_bias, E, S, Tcap,
                                                          L.moe_sel, L.moe_w, counts, h.moe_xs, h.moe_tok, h.moe_wof,
                                                          h.moe_slot, h.err);
    k_moe_plan<<<1, 256, 0, h.stream>>>(counts, E, S, T, Tcap, h.moe_off, h.moe_cursor, h.moe_tile_group,
                                        h.moe_tile_mblk, h.moe_ntiles, h.moe_tok);
    check_launch("moe route+scatter/plan");
    h.launches += 2;
  } else {
    const int rgrid = std::max(1, std::min((T + 7) / 8, h.num_sms * 8));
    if (E <= 8)  // persistent: 2 resident CTAs per SM (120 registers)
      k_moe_route8<<<std::max(1, std::min((T + 7) / 8, 2 * h.num_sms)), 256, 0, h.stream>>>(
          X, T, d, gain, L.router, L.router_bias, E, k, L.moe_sel, L.moe_w, h.moe_inv, counts, h.err);
    else
      k_moe_route<<<rgrid, 256, (static_cast<size_t>(d) * E + 8 * 32 * (E + 1)) * 4, h.stream>>>(
          X, T, d, gain, L.router, L.router_bias, E, k, L.moe_sel, L.moe_w, h.moe_inv, counts, h.err);
    k_moe_plan<<<1, 256, 0, h.stream>>>(counts, E, S, T, Tcap, h.moe_off, h.moe_cursor, h.moe_tile_group,
                                        h.moe_tile_mblk, h.moe_ntiles, h.moe_tok);
    const int sgrid = std::max(1, std::min((T + 255) / 256, h.num_sms * 8));
    k_moe_scatter<<<sgrid, 256, 0, h.stream>>>(X, T, d, gain, h.moe_inv, L.moe_sel, L.moe_w, E, k, S, h.moe_off,
                                               h.moe_cursor, h.moe_xs, h.moe_tok, h.moe_wof, h.moe_slot);
    check_launch("moe route/plan/scatter");
    h.launches += 3;
  }
  stage_mark(h, "L" + std::to_string(l) + ".moe_route");
  if (h.moe_fused && (d == 128 || d == 256)) {  // hidden chunk stays on chip (moe.cuh)
    ensure_smem(k_moe_expert<256>, TailSmem<256>::bytes);
    ensure_smem(k_moe_expert<128>, TailSmem<128>::bytes);
    const int grid = std::max(1, std::min(h.moe_tiles_max, h.num_sms));
    if (d == 256)
      k_moe_expert<256><<<grid, kTailThreads, TailSmem<256>::bytes, h.stream>>>(
          h.tmA_moe_xs, L.tmWup_moe, L.tmWdown_moe, h.tmY_moe, h.moe_tile_group, h.moe_tile_mblk, h.moe_ntiles,
          h.moe_wof, me);
    else
      k_moe_expert<128><<<grid, kTailThreads, TailSmem<128>::bytes, h.stream>>>(
          h.tmA_moe_xs, L.tmWup_moe, L.tmWdown_moe, h.tmY_moe, h.moe_tile_group, h.moe_tile_mblk, h.moe_ntiles,
          h.moe_wof, me);
    check_launch("moe expert");
    ++h.launches;
  } else {
  EpiMoeGU eg;
  eg.tile_group = h.moe_tile_group;
  eg.tile_mblk = h.moe_tile_mblk;
  eg.num_tiles = h.moe_ntiles;
  eg.group_n = 2 * me;
  eg.tok_of = h.moe_tok;
  eg.hidden = h.moe_hs;
  eg.m = me;
  launch_gemm_grouped(h, h.tmA_moe_xs, L.tmB_moe_gu, 2 * me, d, L.bn_moe_gu, eg);
  EpiMoeDown ed;
  ed.tile_group = h.moe_tile_group;
  ed.tile_mblk = h.moe_tile_mblk;
  ed.num_tiles = h.moe_ntiles;
  ed.group_n = d;
  ed.tok_of = h.moe_tok;
  ed.w_of = h.moe_wof;
  ed.y = h.moe_ys;
  ed.d = d;
  launch_gemm_grouped(h, h.tmA_moe_hs, L.tmB_moe_down, d, me, L.bn_moe_down, ed);
  }
  stage_mark(h, "L" + std::to_string(l) + ".moe_experts");
  const int cgrid = std::max(1, std::min((T + 7) / 8, h.num_sms * 8));
  k_moe_combine<<<cgrid, 256, 0, h.stream>>>(X, T, d, h.moe_ys, h.moe_slot, k, S, SS);
  check_launch("moe combine");
  ++h.launches;
  h.moe_rows[l] = T;
  stage_mark(h, "L" + std::to_string(l) + ".moe_combine");
}

// One SORT block. out_attn_only: write Attn(...) instead of the residual
// stream (op-level parity entry point).
static void run_layer(Handle& h, int l, int B, bool attn_only = false) {
  const LayerDev& L = h.layers[l];
  const LayerPlan& lp = h.plan.layers[l];
  const int d = h.d;
  __nv_bfloat16* Xin = h.X[L.in_buf];
  float4* SSin = h.SS[L.in_buf];
  __nv_bfloat16* Xq = h.X[L.q_buf];
  float4* SSq = h.SS[L.q_buf];
  if (h.training) {
    CK(cudaMemcpyAsync(h.tl[l].x_in, Xin, static_cast<size_t>(B) * L.Rkv * d * 2, cudaMemcpyDeviceToDevice,
                       h.stream));
    h.save_to = &h.tl[l];  // the projections and the attention core use the saved buffers
  } else {
    h.save_to = nullptr;
  }
  if (lp.q_identity) {
    launch_qkvg(h, L, L.tmA_in, L.tmB_all, B * L.Rkv, 4 * d, L.bn_full, L.Rkv,
                {kSecQ, kSecV, kSecK, kSecG}, h.tmSS[L.in_buf], L.tmRopeKV, &L.tmB_all_p);
  } else {
    const int rows = B * L.Rq;
    k_gather_rows<<<(rows + 7) / 8, 256, 0, h.stream>>>(Xin, SSin, Xq, SSq, L.query_rows, B, L.Rkv, L.Rq, d);
    check_launch("gather");
    ++h.launches;
    launch_qkvg(h, L, L.tmA_in, L.tmB_kv, B * L.Rkv, 2 * d, L.bn_half, L.Rkv, {kSecK, kSecV},
                h.tmSS[L.in_buf], L.tmRopeKV, &L.tmB_kv_p);
    launch_qkvg(h, L, L.tmA_q, L.tmB_qg, B * L.Rq, 2 * d, L.bn_half, L.Rq, {kSecQ, kSecG},
                h.tmSS[L.q_buf], L.tmRopeQ, &L.tmB_qg_p);
  }
  stage_mark(h, "L" + std::to_string(l) + ".qkvg");
  launch_attention(h, L, lp, B);
  stage_mark(h, "L" + std::to_string(l) + ".attention");
  h.save_to = nullptr;  // (Q / K / V / G of a training forward went straight to h.tl[l])
  if (!attn_only && h.fused_tail && tail_supported(h)) {  // training: x1 saved by the kernel
    __nv_bfloat16* x1_out = h.training ? h.tl[l].x1 : nullptr;
    if (d == 256) launch_tail_d<256>(h, L, Xq, SSq, B * L.Rq, x1_out);
    else launch_tail_d<128>(h, L, Xq, SSq, B * L.Rq, x1_out);
    stage_mark(h, "L" + std::to_string(l) + ".tail");
    return;
  }
  EpiResid eo;
  eo.resid = attn_only ? nullptr : Xq;
  eo.out = attn_only ? h.Qb : Xq;  // Q buffer is dead after attention
  eo.ss_out = reinterpret_cast<float*>(SSq);
  eo.d = d;
  launch_gemm(h, L.tmA_hg, L.tmB_o, B * L.Rq, d, d, L.bn_o, eo);
  stage_mark(h, "L" + std::to_string(l) + ".wo");
  if (attn_only) return;
  if (h.moe) {
    run_moe(h, l, Xq, SSq, B * L.Rq);
    return;
  }
  if (h.training)
    CK(cudaMemcpyAsync(h.tl[l].x1, Xq, static_cast<size_t>(B) * L.Rq * d * 2, cudaMemcpyDeviceToDevice, h.stream));
  EpiSwiGLU eu;
  eu.inv_d = 1.f / static_cast<float>(d);
  eu.hidden = h.hid;
  eu.m = h.m;
  launch_gemm(h, L.tmA_q, L.tmB_up, B * L.Rq, 2 * h.m, d, L.bn_up, eu, &h.tmSS[L.q_buf]);
  stage_mark(h, "L" + std::to_string(l) + ".ffn_up");
  EpiResid ed;
  ed.resid = Xq;
  ed.out = Xq;
  ed.ss_out = reinterpret_cast<float*>(SSq);
  ed.d = d;
  launch_gemm(h, L.tmA_hid, L.tmB_down, B * L.Rq, d, h.m, L.bn_down, ed);
  stage_mark(h, "L" + std::to_string(l) + ".ffn_down");
}


// ====================================================================== training
// Row-major C[M,N] = op(A)[M,K] op(B)[K,N] (+ beta C) through column-major cuBLAS
// (C^T = op(B)^T op(A)^T), TF32 tensor cores, fp32 in/out.
static void gemm_rm_cublas(Handle& h, bool ta, bool tb, int M, int N, int K, const float* A, int lda, const float* B,
                           int ldb, float* C, int ldc, float beta = 0.f) {
  const float alpha = 1.f;
  const cublasStatus_t st = cublasGemmEx(h.cublas, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N,
                                         N, M, K, &alpha, B, CUDA_R_32F, ldb, A, CUDA_R_32F, lda, &beta, C,
                                         CUDA_R_32F, ldc, CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT);
  if (st != CUBLAS_STATUS_SUCCESS) throw RuntimeFailure("cublasGemmEx failed: " + std::to_string(static_cast<int>(st)));
}

// Row-major C[M,N] (fp32, + beta C) = A[M,K] (bf16) . B[K,N] (bf16), fp32 accumulation.
static void gemm_rm_bf16(Handle& h, int M, int N, int K, const __nv_bfloat16* A, int lda, const __nv_bfloat16* B,
                         int ldb, void* C, int ldc, float beta = 0.f, bool c_bf16 = false) {
  const float alpha = 1.f;
  const cublasStatus_t st = cublasGemmEx(h.cublas, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &alpha, B, CUDA_R_16BF, ldb, A,
                                         CUDA_R_16BF, lda, &beta, C, c_bf16 ? CUDA_R_16BF : CUDA_R_32F, ldc,
                                         CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  if (st != CUBLAS_STATUS_SUCCESS) throw RuntimeFailure("cublasGemmEx (bf16) failed: " + std::to_string(static_cast<int>(st)));
}

static inline int warp_rows_grid(int rows) { return (rows + 7) / 8; }
static inline int ew_grid(size_t n) { return static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 16)); }

// generic-path row RMSNorm (optionally after the gathered residual add), see k_resid_rmsnorm
static void resid_rmsnorm(Handle& h, const float* x, const int32_t* map, int R, int Rsrc, const float* a,
                          const float* gain, int rows, int d, float* xo, __nv_bfloat16* y) {
  const int g = warp_rows_grid(rows);
  if (d <= 256)
    k_resid_rmsnorm<2><<<g, 256, 0, h.stream>>>(x, map, R, Rsrc, a, gain, rows, d, xo, y);
  else if (d <= 512)
    k_resid_rmsnorm<4><<<g, 256, 0, h.stream>>>(x, map, R, Rsrc, a, gain, rows, d, xo, y);
  else if (d <= 1024)
    k_resid_rmsnorm<8><<<g, 256, 0, h.stream>>>(x, map, R, Rsrc, a, gain, rows, d, xo, y);
  else
    k_resid_rmsnorm<16><<<g, 256, 0, h.stream>>>(x, map, R, Rsrc, a, gain, rows, d, xo, y);
}

// generic-path per-head Q/K/V/G preparation, see k_qkv_prep (d = H dk <= 2048)
static void qkv_prep(Handle& h, const __nv_bfloat16* raw, int ld, int rows, int R, int H, int dk, int kind,
                     const int32_t* pos, const float* gain, __nv_bfloat16* out) {
  const int g = warp_rows_grid(rows), d = H * dk;
  const float2* rope = h.rope;
  if (d <= 256)
    k_qkv_prep<1><<<g, 256, 0, h.stream>>>(raw, ld, rows, R, H, dk, kind, pos, rope, gain, out);
  else if (d <= 512)
    k_qkv_prep<2><<<g, 256, 0, h.stream>>>(raw, ld, rows, R, H, dk, kind, pos, rope, gain, out);
  else if (d <= 1024)
    k_qkv_prep<4><<<g, 256, 0, h.stream>>>(raw, ld, rows, R, H, dk, kind, pos, rope, gain, out);
  else
    k_qkv_prep<8><<<g, 256, 0, h.stream>>>(raw, ld, rows, R, H, dk, kind, pos, rope, gain, out);
}

// ---- streaming tcgen05 GEMM (gemm_stream.cuh) for the generic path
// mn_f32: an MN-major fp32 (TF32) operand, stored with the 32-byte-atom 128-byte swizzle
static const CUtensorMap& gs_map(Handle& h, const void* p, uint64_t rows, uint64_t cols, uint64_t ld,
                                 uint32_t box_rows, uint32_t box_cols = kGsBK, bool f32 = false, bool mn_f32 = false) {
  const auto key = std::make_tuple(p, rows, cols, ld,
                                   box_rows | (box_cols << 16) | (f32 ? 1u << 31 : 0u) | (mn_f32 ? 1u << 30 : 0u));
  auto it = h.gs_maps.find(key);
  if (it != h.gs_maps.end()) return it->second;
  if (!f32) return h.gs_maps[key] = make_tmap_2d(p, rows, cols, ld, box_rows, box_cols, 128);
  const uint64_t dims[2] = {cols, rows}, str[1] = {ld * 4};
  const uint32_t box[2] = {box_cols, box_rows};
  return h.gs_maps[key] = make_tmap(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, p, 2, dims, str, box, mn_f32 ? 129 : 128);
}

// C[M, N] = op(A)[M, K] x op(B)[K, N] on the streaming tcgen05 GEMM, epilogue functor epi:
//   kAMN = false: A stored [M, K] (row pitch lda);  true: A stored [K, M] (A^T, MN-major)
//   kBMN = false: B stored [N, K] (B^T, K-major);   true: B stored [K, N] (MN-major)
// k_splits > 1: K split over CTAs, epi must take the split index (GsPartialF32).
template <class Epi, bool kAMN = false, bool kBMN = false, class T = __nv_bfloat16>
static void gemm_stream(Handle& h, const T* A, int lda, int M, int K, const T* Bt, int ldb, int N, const Epi& epi,
                        int k_splits = 1) {
  if (M <= 0 || N <= 0) return;
  constexpr bool f32 = std::is_same_v<T, float>;
  constexpr uint32_t BK = 128 / sizeof(T), kAtom = 128 / sizeof(T);
  if (N % Epi::kChunk != 0) throw ConfigError("stream gemm: N must be a multiple of the epilogue chunk");
  const CUtensorMap& ta = kAMN ? gs_map(h, A, K, M, lda, BK, kAtom, f32, f32) : gs_map(h, A, M, K, lda, kGsBM, BK, f32);
  const CUtensorMap& tb = kBMN ? gs_map(h, Bt, K, N, ldb, BK, kAtom, f32, f32) : gs_map(h, Bt, N, K, ldb, kGsBN, BK, f32);
  ensure_smem(k_gemm_stream<Epi, kAMN, kBMN, T>, kGsSmem);
  const int tiles = ((M + kGsBM - 1) / kGsBM) * ((N + kGsBN - 1) / kGsBN) * k_splits;
  k_gemm_stream<Epi, kAMN, kBMN, T><<<std::min(tiles, h.num_sms), kGsThreads, kGsSmem, h.stream>>>(
      ta, tb, M, N, K, k_splits, epi);
  check_launch("stream gemm");
  ++h.launches;
}

// bf16 K-major B operand [sum N_i, ldk] of the column-concatenated [K, N_i] fp32 weights
// `parts` (reference [in, out] layout); swiglu: the two parts (w_gate, w_up) are interleaved in
// 32-row blocks [gate_j | up_j] for EpiSwiGLU. ldk = K rounded up to 8 (16-byte TMA pitch).
static const __nv_bfloat16* wT16(Handle& h, const std::string& key, const std::vector<std::string>& parts,
                                 bool swiglu = false) {
  auto it = h.wT.find(key);
  if (it != h.wT.end()) return it->second;
  const auto& g0 = h.grad_index.at(parts[0]).second;
  const int K = static_cast<int>(g0.first), ldk = (K + 7) & ~7;
  int Ntot = 0;
  for (const auto& p : parts) Ntot += static_cast<int>(h.grad_index.at(p).second.second);
  __nv_bfloat16* dst = h.dalloc<__nv_bfloat16>(static_cast<size_t>(Ntot) * ldk);
  int row0 = 0;
  for (size_t i = 0; i < parts.size(); ++i) {
    const auto& gi = h.grad_index.at(parts[i]).second;
    if (gi.first != K) throw ConfigError("wT16: parts with different input widths");
    const int N = static_cast<int>(gi.second);
    const dim3 grid((ldk + 31) / 32, (N + 31) / 32);
    k_transpose_bf16<<<grid, 256, 0, h.stream>>>(h.w32.at(parts[i]), K, N, ldk, row0, swiglu ? 32 : 0,
                                                 swiglu ? static_cast<int>(i) * 32 : 0, dst);
    row0 += N;
  }
  check_launch("weight transpose");
  return h.wT[key] = dst;
}

// Row-major C[M,N] (+ beta C) = op(A) op(B) with bf16 operands and fp32 accumulation; C fp32
// or bf16 (the training FFN backward).
static void gemm_rm16(Handle& h, bool ta, bool tb, int M, int N, int K, const __nv_bfloat16* A, int lda,
                      const __nv_bfloat16* B, int ldb, void* C, int ldc, bool c_bf16, float beta = 0.f) {
  if (M <= 0 || N <= 0) return;
  if (h.train_cublas) {  // A/B option: the library GEMM
    const float alpha = 1.f;
    const cublasStatus_t st = cublasGemmEx(h.cublas, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N,
                                           N, M, K, &alpha, B, CUDA_R_16BF, ldb, A, CUDA_R_16BF, lda, &beta, C,
                                           c_bf16 ? CUDA_R_16BF : CUDA_R_32F, ldc, CUBLAS_COMPUTE_32F,
                                           CUBLAS_GEMM_DEFAULT);
    if (st != CUBLAS_STATUS_SUCCESS)
      throw RuntimeFailure("cublasGemmEx (bf16) failed: " + std::to_string(static_cast<int>(st)));
    return;
  }
  // tcgen05 streaming GEMM: op(A) = A^T is an MN-major A, op(B) = B (not transposed) an
  // MN-major B. Few output tiles and a long K (the weight gradients, K = rows) split K over
  // the SMs into partials summed in a fixed order (deterministic).
  const int tiles = ((M + kGsBM - 1) / kGsBM) * ((N + kGsBN - 1) / kGsBN);
  const int num_k = (K + kGsBK - 1) / kGsBK;
  int splits = 1;
  if (tiles * 2 <= h.num_sms && num_k >= 16) splits = std::max(1, std::min(h.num_sms / tiles, num_k / 8));
  auto run = [&](auto epi) {
    using E = decltype(epi);
    if (ta && tb) gemm_stream<E, true, false>(h, A, lda, M, K, B, ldb, N, epi, splits);
    else if (ta) gemm_stream<E, true, true>(h, A, lda, M, K, B, ldb, N, epi, splits);
    else if (tb) gemm_stream<E, false, false>(h, A, lda, M, K, B, ldb, N, epi, splits);
    else gemm_stream<E, false, true>(h, A, lda, M, K, B, ldb, N, epi, splits);
  };
  if (splits > 1) {
    const size_t need = static_cast<size_t>(splits) * M * N;
    if (need > h.splitk_cap) {
      if (h.splitk_ws) CK(cudaFree(h.splitk_ws));
      CK(cudaMalloc(&h.splitk_ws, need * sizeof(float)));
      h.splitk_cap = need;
    }
    run(GsPartialF32{h.splitk_ws, M, N});
    const int g = static_cast<int>(std::min<size_t>((static_cast<size_t>(M) * N + 255) / 256, 148 * 8));
    if (c_bf16)
      k_splitk_reduce<__nv_bfloat16><<<g, 256, 0, h.stream>>>(h.splitk_ws, splits, M, N,
                                                              static_cast<__nv_bfloat16*>(C), ldc, beta);
    else
      k_splitk_reduce<float><<<g, 256, 0, h.stream>>>(h.splitk_ws, splits, M, N, static_cast<float*>(C), ldc, beta);
    check_launch("split-k reduce");
    ++h.launches;
    return;
  }
  if (c_bf16) {
    if (beta != 0.f) throw RuntimeFailure("gemm_rm16: bf16 output with beta is not supported");
    run(GsStore<__nv_bfloat16>{static_cast<__nv_bfloat16*>(C), ldc});
  } else if (beta != 0.f) {
    if (beta != 1.f) throw RuntimeFailure("gemm_rm16: beta must be 0 or 1");
    run(GsAccF32{static_cast<float*>(C), ldc});
  } else {
    run(GsStore<float>{static_cast<float*>(C), ldc});
  }
}

// Row-major fp32 C[M,N] (+ beta C) = op(A) op(B) (the ranking head and tokenizer products,
// fp32 per PAPER.md:243): TF32 tcgen05 streaming GEMM (split-K for the long-K weight
// gradients), or the SIMT kernel for shapes TMA cannot tile (N = 3 logits, K = 3, widths
// that are not multiples of 32 / 16-byte row pitches).
static void gemm_rm(Handle& h, bool ta, bool tb, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                    float* C, int ldc, float beta = 0.f) {
  if (M <= 0 || N <= 0) return;
  if (h.train_cublas) {
    gemm_rm_cublas(h, ta, tb, M, N, K, A, lda, B, ldb, C, ldc, beta);
    return;
  }
  const bool tma_ok = N % 32 == 0 && K >= 8 && lda % 4 == 0 && ldb % 4 == 0 && ldc % 4 == 0 &&
                      (beta == 0.f || beta == 1.f);
  if (!tma_ok) {
    const dim3 grid((N + 31) / 32, (M + 31) / 32);
    k_gemm_simt<<<grid, 256, 0, h.stream>>>(ta, tb, M, N, K, A, lda, B, ldb, C, ldc, beta);
    check_launch("simt gemm");
    ++h.launches;
    return;
  }
  const int tiles = ((M + kGsBM - 1) / kGsBM) * ((N + kGsBN - 1) / kGsBN);
  const int num_k = (K + 31) / 32;
  int splits = 1;
  if (tiles * 2 <= h.num_sms && num_k >= 16) splits = std::max(1, std::min(h.num_sms / tiles, num_k / 8));
  auto run = [&](auto epi) {
    using E = decltype(epi);
    if (ta && tb) gemm_stream<E, true, false, float>(h, A, lda, M, K, B, ldb, N, epi, splits);
    else if (ta) gemm_stream<E, true, true, float>(h, A, lda, M, K, B, ldb, N, epi, splits);
    else if (tb) gemm_stream<E, false, false, float>(h, A, lda, M, K, B, ldb, N, epi, splits);
    else gemm_stream<E, false, true, float>(h, A, lda, M, K, B, ldb, N, epi, splits);
  };
  if (splits > 1) {
    const size_t need = static_cast<size_t>(splits) * M * N;
    if (need > h.splitk_cap) {
      if (h.splitk_ws) CK(cudaFree(h.splitk_ws));
      CK(cudaMalloc(&h.splitk_ws, need * sizeof(float)));
      h.splitk_cap = need;
    }
    run(GsPartialF32{h.splitk_ws, M, N});
    const int g = static_cast<int>(std::min<size_t>((static_cast<size_t>(M) * N + 255) / 256, 148 * 8));
    k_splitk_reduce<float><<<g, 256, 0, h.stream>>>(h.splitk_ws, splits, M, N, C, ldc, beta);
    check_launch("split-k reduce");
    ++h.launches;
  } else if (beta != 0.f) {
    run(GsAccF32{C, ldc});
  } else {
    run(GsStore<float>{C, ldc});
  }
}

static float* grad_ptr(Handle& h, const std::string& name) {
  auto it = h.grad_index.find(name);
  if (it == h.grad_index.end()) throw RuntimeFailure("no gradient slot for " + name);
  return h.grads + it->second.first;
}
static const float* w32(Handle& h, const std::string& name) {
  auto it = h.w32.find(name);
  if (it == h.w32.end()) throw RuntimeFailure("no fp32 parameter " + name);
  return it->second;
}

// bf16 copy of an fp32 training weight (`n` elements), refreshed by repack_weights after every
// optimizer step.
static const __nv_bfloat16* tw16(Handle& h, const std::string& name, size_t n) {
  auto it = h.tw16.find(name);
  if (it != h.tw16.end()) return it->second.first;
  __nv_bfloat16* dst = h.dalloc<__nv_bfloat16>(n);
  k_f32_to_bf16<<<ew_grid(n), 256, 0, h.stream>>>(w32(h, name), n, dst);
  check_launch("training weight cast");
  h.tw16[name] = {dst, n};
  return dst;
}

// Work lists of the attention backward for one layer (batch-uniform): for every 32-row
// q-block the kv-column intervals any of its rows sees, for every 32-column kv-block the
// q-row intervals that see any of its columns (from the compact mask {lo, hi, self}).
static void build_bwd_lists(const LayerPlan& lp, std::vector<int32_t>& dq_off, std::vector<int2>& dq_iv,
                            std::vector<int32_t>& dkv_off, std::vector<int2>& dkv_iv) {
  auto push_runs = [](const std::vector<char>& on, std::vector<int2>& iv) {
    const int n = static_cast<int>(on.size());
    for (int i = 0; i < n;) {
      if (!on[i]) {
        ++i;
        continue;
      }
      int j = i;
      while (j < n && on[j]) ++j;
      iv.push_back(make_int2(i, j));
      i = j;
    }
  };
  const int nqb = (lp.l_q + 31) / 32, nkb = (lp.l_kv + 31) / 32;
  dq_off.assign(1, 0);
  for (int qb = 0; qb < nqb; ++qb) {
    std::vector<char> on(lp.l_kv, 0);
    for (int r = qb * 32; r < std::min(lp.l_q, qb * 32 + 32); ++r) {
      for (int c = std::max(lp.lo[r], 0); c <= lp.hi[r] && c < lp.l_kv; ++c) on[c] = 1;
      if (lp.self_idx[r] >= 0) on[lp.self_idx[r]] = 1;
    }
    push_runs(on, dq_iv);
    dq_off.push_back(static_cast<int32_t>(dq_iv.size()));
  }
  dkv_off.assign(1, 0);
  for (int kb = 0; kb < nkb; ++kb) {
    const int c0 = kb * 32, c1 = std::min(lp.l_kv, c0 + 32) - 1;
    std::vector<char> on(lp.l_q, 0);
    for (int r = 0; r < lp.l_q; ++r) {
      const bool iv = lp.lo[r] <= c1 && lp.hi[r] >= c0 && lp.hi[r] >= lp.lo[r];
      const bool self = lp.self_idx[r] >= c0 && lp.self_idx[r] <= c1;
      on[r] = iv || self;
    }
    push_runs(on, dkv_iv);
    dkv_off.push_back(static_cast<int32_t>(dkv_iv.size()));
  }
}

// Step lists of the tcgen05 attention backward (attn_bwd.cuh): for every 128-row X block the
// 64-row Y blocks sharing a visible entry, with the class of each 32 x 32 chunk (lane quarter
// q of X, half hf of Y) in bits 2 (2 q + hf): 1 = fully visible, 2 = invisible, 0 = mixed.
// dq_mode: X = query rows, Y = kv rows; else X = kv rows, Y = query rows. A chunk is "full"
// only when all its rows and columns are in range.
static void build_bwd_tc_lists(const LayerPlan& lp, bool dq_mode, std::vector<int32_t>& off, std::vector<int2>& code) {
  const int RX = dq_mode ? lp.l_q : lp.l_kv, RY = dq_mode ? lp.l_kv : lp.l_q;
  const int nX = (RX + 127) / 128, nY = (RY + 63) / 64;
  off.assign(1, 0);
  code.clear();
  auto sees = [&](int q, int k) { return (k >= lp.lo[q] && k <= lp.hi[q]) || k == lp.self_idx[q]; };
  for (int xb = 0; xb < nX; ++xb) {
    for (int yb = 0; yb < nY; ++yb) {
      uint32_t bits = 0;
      bool any = false;
      for (int qq = 0; qq < 4; ++qq)
        for (int hf = 0; hf < 2; ++hf) {
          const int x0 = xb * 128 + qq * 32, y0 = yb * 64 + hf * 32;
          bool full = x0 + 32 <= RX && y0 + 32 <= RY, none = true;
          for (int i = 0; i < 32 && (full || none); ++i)
            for (int j = 0; j < 32 && (full || none); ++j) {
              const int x = x0 + i, y = y0 + j;
              const bool v = x < RX && y < RY && (dq_mode ? sees(x, y) : sees(y, x));
              full = full && v;
              none = none && !v;
            }
          const uint32_t c = full ? 1u : (none ? 2u : 0u);
          bits |= c << (2 * (2 * qq + hf));
          any = any || !none;
        }
      if (any) code.push_back(make_int2(yb, static_cast<int32_t>(bits)));
    }
    off.push_back(static_cast<int32_t>(code.size()));
  }
  if (code.empty()) code.push_back(make_int2(0, 0));
}

// Saved-activation buffers, TMA boxes and backward work lists of one training layer
// (B requests of plan lp); the dO16 boxes are added by the caller once dO16 exists.
static void train_layer_buffers(Handle& h, const LayerPlan& lp, const LayerDev& L, int B, Handle::TrainLayer& T) {
  const int d = h.d;
  const size_t nq = static_cast<size_t>(B) * L.Rq * d, nkv = static_cast<size_t>(B) * L.Rkv * d;
  T.x_in = h.dalloc<__nv_bfloat16>(nkv);
  T.q = h.dalloc<__nv_bfloat16>(nq);
  T.k = h.dalloc<__nv_bfloat16>(nkv);
  T.v = h.dalloc<__nv_bfloat16>(nkv);
  T.g = h.dalloc<__nv_bfloat16>(nq);
  T.o_pre = h.dalloc<__nv_bfloat16>(nq);
  T.x1 = h.dalloc<__nv_bfloat16>(nq);
  T.lse = h.dalloc<float>(static_cast<size_t>(B) * h.H * L.Rq);
  {
    const int dk = h.dk;
    const uint64_t BH = static_cast<uint64_t>(B) * h.H;
    uint64_t dq[3] = {static_cast<uint64_t>(dk), static_cast<uint64_t>(L.Rq), BH};
    uint64_t sq[2] = {static_cast<uint64_t>(dk) * 2, static_cast<uint64_t>(L.Rq) * dk * 2};
    uint32_t bq[3] = {static_cast<uint32_t>(dk), 128, 1};
    T.tmQ = make_tmap_bf16(T.q, 3, dq, sq, bq, dk * 2);
    uint64_t dkd[3] = {static_cast<uint64_t>(dk), static_cast<uint64_t>(L.Rkv), BH};
    uint64_t skd[2] = {static_cast<uint64_t>(dk) * 2, static_cast<uint64_t>(L.Rkv) * dk * 2};
    T.tmK = make_tmap_bf16(T.k, 3, dkd, skd, bq, dk * 2);
    T.tmV = make_tmap_bf16(T.v, 3, dkd, skd, bq, dk * 2);
    uint32_t b64[3] = {static_cast<uint32_t>(dk), 64, 1};
    T.tmQ64 = make_tmap_bf16(T.q, 3, dq, sq, b64, dk * 2);
    T.tmK64 = make_tmap_bf16(T.k, 3, dkd, skd, b64, dk * 2);
    T.tmV64 = make_tmap_bf16(T.v, 3, dkd, skd, b64, dk * 2);
  }
  {
    std::vector<int32_t> off;
    std::vector<int2> code;
    build_bwd_tc_lists(lp, false, off, code);
    T.tc_kv_off = h.upload(off);
    T.tc_kv_code = h.upload(code);
    T.tc_kv_n = static_cast<int>(code.size());
    build_bwd_tc_lists(lp, true, off, code);
    T.tc_q_off = h.upload(off);
    T.tc_q_code = h.upload(code);
    T.tc_q_n = static_cast<int>(code.size());
  }
  {  // per kv row x the query rows that see it; kept when every row's set is <= 2 intervals
    std::vector<std::vector<int32_t>> seen(static_cast<size_t>(lp.l_kv));
    for (int r = 0; r < lp.l_q; ++r) {
      for (int c = std::max(lp.lo[r], 0); c <= lp.hi[r] && c < lp.l_kv; ++c) seen[c].push_back(r);
      if (lp.self_idx[r] >= 0 && (lp.self_idx[r] < lp.lo[r] || lp.self_idx[r] > lp.hi[r]))
        seen[lp.self_idx[r]].push_back(r);
    }
    std::vector<int4> km(static_cast<size_t>(lp.l_kv), make_int4(0, -1, 0, -1));
    bool ok = true;
    for (int x = 0; x < lp.l_kv && ok; ++x) {
      auto& v = seen[x];
      std::sort(v.begin(), v.end());
      int runs = 0;
      for (size_t i = 0; i < v.size() && ok; ++i) {
        if (i > 0 && v[i] == v[i - 1] + 1) {
          (runs == 1 ? km[x].y : km[x].w) = v[i];
          continue;
        }
        if (++runs > 2) {
          ok = false;
        } else if (runs == 1) {
          km[x].x = km[x].y = v[i];
        } else {
          km[x].z = km[x].w = v[i];
        }
      }
    }
    if (ok) T.kvmeta = h.upload(km);
  }
  std::vector<int32_t> qo, ko;
  std::vector<int2> qi, ki;
  build_bwd_lists(lp, qo, qi, ko, ki);
  if (qi.empty()) qi.push_back(make_int2(0, 0));
  if (ki.empty()) ki.push_back(make_int2(0, 0));
  T.dq_off = h.upload(qo);
  T.dq_iv = h.upload(qi);
  T.dkv_off = h.upload(ko);
  T.dkv_iv = h.upload(ki);
  {  // 64-row q blocks that see each 64-column kv block (k_attn_bwd_mma)
    std::vector<int32_t> off(1, 0), lst;
    for (int c0 = 0; c0 < lp.l_kv; c0 += 64) {
      const int c1 = std::min(lp.l_kv, c0 + 64) - 1;
      for (int qb = 0; qb * 64 < lp.l_q; ++qb) {
        bool any = false;
        for (int r = qb * 64; r < std::min(lp.l_q, qb * 64 + 64) && !any; ++r)
          any = (lp.hi[r] >= lp.lo[r] && lp.lo[r] <= c1 && lp.hi[r] >= c0) ||
                (lp.self_idx[r] >= c0 && lp.self_idx[r] <= c1);
        if (!any) continue;
        // every (q, kv) of the 64 x 64 block visible and in range: no per-element mask
        bool full = qb * 64 + 64 <= lp.l_q && c0 + 64 <= lp.l_kv;
        for (int r = qb * 64; r < qb * 64 + 64 && full; ++r) full = lp.lo[r] <= c0 && lp.hi[r] >= c1;
        lst.push_back(full ? (qb | static_cast<int32_t>(0x40000000)) : qb);
      }
      off.push_back(static_cast<int32_t>(lst.size()));
    }
    if (lst.empty()) lst.push_back(0);
    T.qb_off = h.upload(off);
    T.qb_list = h.upload(lst);
  }
}

// dO16 as token-major [B, Rq, H, dk] boxes (128- and 64-row) for the tcgen05 backward
static void train_do_boxes(Handle& h, int Rq, int B, Handle::TrainLayer& T) {
  const int dk = h.dk, d = h.d;
  const uint64_t dims[4] = {static_cast<uint64_t>(dk), static_cast<uint64_t>(h.H), static_cast<uint64_t>(Rq),
                            static_cast<uint64_t>(B)};
  const uint64_t str[3] = {static_cast<uint64_t>(dk) * 2, static_cast<uint64_t>(d) * 2,
                           static_cast<uint64_t>(Rq) * d * 2};
  const uint32_t b128[4] = {static_cast<uint32_t>(dk), 1, 128, 1}, b64[4] = {static_cast<uint32_t>(dk), 1, 64, 1};
  T.tmDO128 = make_tmap(CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, h.dO16, 4, dims, str, b128, dk * 2);
  T.tmDO64 = make_tmap(CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, h.dO16, 4, dims, str, b64, dk * 2);
}

// Unfreezing the item table: its fp32 master (from the bf16 device table), gradient, moments.
static void unfreeze_item_table(Handle& h) {
  if (h.item_master) return;
  const size_t n = static_cast<size_t>(h.cfg.n_items) * h.cfg.item_dim;
  h.item_master = h.dalloc<float>(n);
  h.item_grad = h.dalloc<float>(n);
  h.item_m = h.dalloc<float>(n);
  h.item_v = h.dalloc<float>(n);
  k_bf16_to_f32<<<ew_grid(n), 256, 0, h.stream>>>(h.item, n, h.item_master);  // master from the device table
  CK(cudaMemsetAsync(h.item_m, 0, n * 4, h.stream));
  CK(cudaMemsetAsync(h.item_v, 0, n * 4, h.stream));
  check_launch("item table master");
}

static void ensure_train_buffers(Handle& h, int B) {
  if (h.moe) throw ConfigError("training step: the MoE FFN backward is not implemented in this build");
  if (!h.frozen.count("tok.item_table")) unfreeze_item_table(h);  // (pre-training trains it by default)
  if (h.train_B >= B) return;
  if (h.cfg.pretrain) {
    if (h.cfg.n_items % 32 != 0) throw ConfigError("pre-training step: n_items must be a multiple of 32");
    h.pre_P = h.dalloc<__nv_bfloat16>(static_cast<size_t>(h.Bmax) * h.L0 * h.cfg.n_items);
    h.pre_dh = h.dalloc<float>(static_cast<size_t>(h.Bmax) * h.L0 * h.cfg.item_dim);
    h.pre_loss = h.dalloc<float>(1);
  }
  if (!h.cublas) {
    if (cublasCreate(&h.cublas) != CUBLAS_STATUS_SUCCESS) throw RuntimeFailure("cublasCreate failed");
  }
  const int d = h.d, m = h.m;
  B = h.Bmax;  // size once for max_batch
  h.grads = h.dalloc<float>(h.grad_count);
  h.t_rows = h.dalloc<int32_t>(static_cast<size_t>(h.Bmax) * h.L0);
  h.tl.resize(h.cfg.layers);
  size_t mkv_max = 0;
  for (int l = 0; l < h.cfg.layers; ++l) {
    const LayerDev& L = h.layers[l];
    train_layer_buffers(h, h.plan.layers[l], L, B, h.tl[l]);
    mkv_max = std::max(mkv_max, static_cast<size_t>(B) * L.Rkv);
  }
  const size_t rows = std::max(mkv_max, static_cast<size_t>(B) * h.L0);
  // workspace: 0 dX, 1 dX next, 2 xn, 3 xq, 4 H / dxq, 5 dH, 6 dO, 7 dgraw, 8 dQ, 9 dK, 10 dV,
  // 11 raw, 12 GU / dGU, 13 z / dz, 14 inv (rows), 15 D / head scratch
  for (int i = 0; i < 12; ++i) h.tw[i] = h.dalloc<float>(rows * d);
  h.dO16 = h.dalloc<__nv_bfloat16>(rows * d);
  for (int l = 0; l < h.cfg.layers; ++l) train_do_boxes(h, h.layers[l].Rq, B, h.tl[l]);
  h.tw[12] = h.dalloc<float>(rows * 2 * m * 2);  // GU and dGU
  h.tw[13] = h.dalloc<float>(rows * m);
  h.tw[14] = h.dalloc<float>(rows * 2);
  // head scratch: hid, dhid [BN, dh], the 32-column padded dz [BN, 32] and dW2 [dh, 32]
  h.tw[15] = h.dalloc<float>(std::max(rows * h.H, static_cast<size_t>(B) * h.cfg.n_cand * (h.dh * 2 + 32) +
                                                      static_cast<size_t>(h.dh) * 32));
  h.train_B = h.Bmax;
}


// Row RMSNorm / its backward for the training path: the vectorised kernels when d <= 256.
template <class T>
static void rms_rows(Handle& h, const T* x, const float* gain, int rows, int d, float* y, float* inv) {
  if (d <= 256 && d % 8 == 0)
    k_rmsnorm_rows_v<T><<<std::max(1, std::min((rows + 7) / 8, 8 * h.num_sms)), 256, 0, h.stream>>>(x, gain, rows, d,
                                                                                                   y, inv);
  else
    k_rmsnorm_rows<T><<<(rows + 7) / 8, 256, 0, h.stream>>>(x, gain, rows, d, nullptr, 1, 1, y, inv);
}
template <class T>
static void rms_bwd(Handle& h, const float* dy, const T* x, const float* inv, const float* gain, int rows, int d,
                    float* dx, int accum, float* dgain, __nv_bfloat16* dx16 = nullptr) {
  if (d <= 256 && d % 8 == 0) {
    k_rmsnorm_bwd_v<T><<<std::max(1, std::min((rows + 7) / 8, 4 * h.num_sms)), 256, d * 4, h.stream>>>(
        dy, x, inv, gain, rows, d, dx, accum, dgain, dx16);
  } else {
    k_rmsnorm_bwd<T><<<(rows + 63) / 64, 256, d * 4, h.stream>>>(dy, x, inv, gain, rows, d, dx, accum, dgain);
    if (dx16) k_f32_to_bf16<<<ew_grid(static_cast<size_t>(rows) * d), 256, 0, h.stream>>>(dx, static_cast<size_t>(rows) * d, dx16);
  }
}

// Pre-training head backward: loss = mean over the B n predicted positions of
// lse_t - z_t[click_t], z_t = hp_t E^T. The logits are recomputed by the tcgen05 GEMM whose
// epilogue writes dL/dz as bf16 (GsCeGrad); dh = dz E and dE += dz^T hp (the tied head's share
// of the item-table gradient) are two more tcgen05 GEMMs; then hp = RMSN(x) proj backward
// writes d(final stream) for every position into dX.
static void pretrain_head_backward(Handle& h, int B, float* dX) {
  const SortConfig& c = h.cfg;
  const int d = h.d, L = h.L0, n = L - 1, T = B * L, V = c.n_items, K = c.item_dim;
  if (h.item_ext) throw ConfigError("pre-training step: the row-sharded item table is not trained here");
  const __nv_bfloat16* Xf = h.X[h.layers.back().q_buf];
  gemm_stream(h, h.pre_hp, K, T, K, h.item, K, V,
              GsCeGrad{h.pre_P, V, h.pre_lse, h.in_item, L, n, 1.f / static_cast<float>(B * n)});
  gemm_rm16(h, false, false, T, K, V, h.pre_P, V, h.item, K, h.pre_dh, K, false);           // dh = dz E
  if (!h.frozen.count("tok.item_table"))
    gemm_rm16(h, true, false, V, K, T, h.pre_P, V, h.pre_hp, K, h.item_grad, K, false, 1.f);  // dE += dz^T hp
  float* xh = h.tw[2];
  float* inv = h.tw[14];
  rms_rows<__nv_bfloat16>(h, Xf, w32(h, "final_norm.gain"), T, d, xh, inv);
  gemm_rm(h, true, false, d, K, T, xh, d, h.pre_dh, K, grad_ptr(h, "pretrain.proj"), K);
  float* dxh = h.tw[3];
  gemm_rm(h, false, true, T, d, K, h.pre_dh, K, w32(h, "pretrain.proj"), K, dxh, d);
  rms_bwd<__nv_bfloat16>(h, dxh, Xf, inv, w32(h, "final_norm.gain"), T, d, dX, 0, grad_ptr(h, "final_norm.gain"));
  check_launch("pretrain head backward");
}

// Backward of one training forward; dz = dL/dlogits [B*N, 3] on the device.
// tcgen05 attention-core backward (attn_bwd.cuh) of one layer, B requests: pass 1 dK / dV per
// 128-row kv block (X = K, V; Y = Q, dO), pass 2 dQ per 128-row q block (X = Q, dO; Y = K, V).
// D = rowsum(dO * O) per (bh, query row); dV is also written as bf16 (dV16).
static void attn_core_backward_tc(Handle& h, const LayerDev& L, const Handle::TrainLayer& T, int B, const float* Dd,
                                  float* dQ, float* dK, float* dV, __nv_bfloat16* dV16) {
  const int H = h.H, dk = h.dk;
  AttnBwdTcArgs tb;
  tb.rowmeta = L.rowmeta;
  tb.kvmeta = T.kvmeta;
  tb.lse = T.lse;
  tb.D = Dd;
  tb.BH = B * H;
  tb.H = H;
  tb.Rq = L.Rq;
  tb.Rkv = L.Rkv;
  tb.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(dk)));
  tb.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(dk)));
  tb.x_off = T.tc_kv_off;
  tb.y_code = T.tc_kv_code;
  tb.nX = (L.Rkv + 127) / 128;
  tb.out0 = dK;
  tb.out1 = dV;
  tb.out1_16 = dV16;
  auto launch_tc = [&](auto kern, const CUtensorMap& x0, const CUtensorMap& x1, const CUtensorMap& y0,
                       const CUtensorMap& y1, size_t smem_fn_bytes) {
    ensure_smem(kern, smem_fn_bytes);
    const int grid = coprime_grid(std::min(tb.nX * tb.BH, 2 * h.num_sms), tb.nX);
    kern<<<grid, kAttnThreads, smem_fn_bytes, h.stream>>>(x0, x1, y0, y1, tb);
  };
#define SORT_BWD_TC(DKV)                                                                               \
  case DKV: {                                                                                          \
    launch_tc(k_attn_bwd_tc<DKV, false>, T.tmK, T.tmV, T.tmQ64, T.tmDO64,                              \
              BwdSmem<DKV>::bytes(tb.nX + 2 + 2 * T.tc_kv_n));                                         \
    tb.x_off = T.tc_q_off;                                                                             \
    tb.y_code = T.tc_q_code;                                                                           \
    tb.nX = (L.Rq + 127) / 128;                                                                        \
    tb.out0 = dQ;                                                                                      \
    tb.kvmeta = nullptr;                                                                               \
    tb.out1 = nullptr;                                                                                 \
    tb.out1_16 = nullptr;                                                                              \
    launch_tc(k_attn_bwd_tc<DKV, true>, T.tmQ, T.tmDO128, T.tmK64, T.tmV64,                            \
              BwdSmem<DKV>::bytes(tb.nX + 2 + 2 * T.tc_q_n));                                          \
    break;                                                                                             \
  }
  switch (dk) {
    SORT_BWD_TC(16)
    SORT_BWD_TC(32)
    SORT_BWD_TC(64)
    default: throw ConfigError("training: unsupported head dim");
  }
#undef SORT_BWD_TC
  check_launch("tcgen05 attention backward");
  h.launches += 2;
}

static void backward_device(Handle& h, int B, const float* dz) {
  const SortConfig& c = h.cfg;
  const int d = h.d, m = h.m, H = h.H, dk = h.dk, N = c.n_cand, dh = h.dh;
  CK(cudaMemsetAsync(h.grads, 0, h.grad_count * sizeof(float), h.stream));
  const bool item_train = !h.frozen.count("tok.item_table");
  const size_t n_item_el = static_cast<size_t>(c.n_items) * c.item_dim;
  if (item_train) CK(cudaMemsetAsync(h.item_grad, 0, n_item_el * sizeof(float), h.stream));
  float* dX = h.tw[0];
  float* dXn = h.tw[1];
  float* inv = h.tw[14];
  if (c.pretrain) {
    pretrain_head_backward(h, B, dX);
  } else {
  // ---- head: xc = final candidate rows, xh = RMSN(xc), hid = relu(xh W1 + b1)
  const LayerDev& last = h.layers.back();
  const int R = last.Rq, BN = B * N;
  std::vector<int32_t> cmap_h(N);
  for (int j = 0; j < N; ++j) cmap_h[j] = R - N + j;
  int32_t*& cmap = h.cand_maps[R];
  if (!cmap) cmap = h.upload(cmap_h);
  float* xc = h.tw[2];
  float* xh = h.tw[3];
  float* hid = h.tw[15];
  float* dhid = hid + static_cast<size_t>(BN) * dh;
  const __nv_bfloat16* Xf = h.X[last.q_buf];
  k_gather_f32<__nv_bfloat16><<<(BN + 7) / 8, 256, 0, h.stream>>>(Xf, cmap, N, R, BN, d, xc);
  rms_rows<float>(h, xc, w32(h, "final_norm.gain"), BN, d, xh, inv);
  check_launch("head rows");
  gemm_rm(h, false, false, BN, dh, d, xh, d, w32(h, "head.w1"), dh, hid, dh);
  k_bias_relu<<<ew_grid(static_cast<size_t>(BN) * dh), 256, 0, h.stream>>>(hid, w32(h, "head.b1"), BN, dh);
  {  // dW2 = hid^T dz: N = 3 would leave the SIMT kernel 8 CTAs over K = B*N rows; dz is
     // zero-padded to 32 columns so the TF32 tcgen05 GEMM splits K over the SMs
    float* dz32 = hid + 2 * static_cast<size_t>(BN) * dh;
    float* gw2 = dz32 + static_cast<size_t>(BN) * 32;
    CK(cudaMemsetAsync(dz32, 0, static_cast<size_t>(BN) * 32 * 4, h.stream));
    CK(cudaMemcpy2DAsync(dz32, 32 * 4, dz, 3 * 4, 3 * 4, BN, cudaMemcpyDeviceToDevice, h.stream));
    gemm_rm(h, true, false, dh, 32, BN, hid, dh, dz32, 32, gw2, 32);
    CK(cudaMemcpy2DAsync(grad_ptr(h, "head.w2"), 3 * 4, gw2, 32 * 4, 3 * 4, dh, cudaMemcpyDeviceToDevice, h.stream));
  }
  k_colsum<<<dim3(1, 64), dim3(32, 8), 0, h.stream>>>(dz, BN, 3, grad_ptr(h, "head.b2"));
  gemm_rm(h, false, true, BN, dh, 3, dz, 3, w32(h, "head.w2"), 3, dhid, dh);
  k_relu_mask<<<ew_grid(static_cast<size_t>(BN) * dh), 256, 0, h.stream>>>(dhid, hid, static_cast<size_t>(BN) * dh);
  gemm_rm(h, true, false, d, dh, BN, xh, d, dhid, dh, grad_ptr(h, "head.w1"), dh);
  k_colsum<<<dim3((dh + 31) / 32, std::min(148, (BN + 255) / 256)), dim3(32, 8), 0, h.stream>>>(dhid, BN, dh,
                                                                                    grad_ptr(h, "head.b1"));
  float* dxh = h.tw[4];
  gemm_rm(h, false, true, BN, d, dh, dhid, dh, w32(h, "head.w1"), dh, dxh, d);
  float* dxc = h.tw[5];
  rms_bwd<float>(h, dxh, xc, inv, w32(h, "final_norm.gain"), BN, d, dxc, 0, grad_ptr(h, "final_norm.gain"));
  CK(cudaMemsetAsync(dX, 0, static_cast<size_t>(B) * R * d * 4, h.stream));
  k_scatter_add_rows<<<(BN + 7) / 8, 256, 0, h.stream>>>(dxc, cmap, B, N, R, d, dX);
  check_launch("head backward");
  }
  // ---- blocks in reverse
  bool dX16_ready = false;  // tw[3] already holds dX in bf16 (written by the layer above)
  for (int l = c.layers - 1; l >= 0; --l) {
    const LayerDev& L = h.layers[l];
    const LayerPlan& lp = h.plan.layers[l];
    const auto& T = h.tl[l];
    const std::string sl = std::to_string(l);
    const std::string A = "attn." + sl + ".", F = "ffn." + sl + ".", Bk = "block." + sl + ".";
    const int M = B * L.Rq, Mkv = B * L.Rkv;
    const size_t nq = static_cast<size_t>(M) * d, nkv = static_cast<size_t>(Mkv) * d;
    // FFN: xo = xr + down(swish(xf Wg) * (xf Wu)), xf = RMSN(xr = x1)
    // bf16 operands and [M, m] / [M, 2m] intermediates, fp32 accumulation and gradients
    __nv_bfloat16* xf = reinterpret_cast<__nv_bfloat16*>(h.tw[2]);
    __nv_bfloat16* GU = reinterpret_cast<__nv_bfloat16*>(h.tw[12]);
    __nv_bfloat16* dGU = GU + static_cast<size_t>(M) * 2 * m;
    __nv_bfloat16* z = reinterpret_cast<__nv_bfloat16*>(h.tw[13]);
    __nv_bfloat16* dX16 = reinterpret_cast<__nv_bfloat16*>(h.tw[3]);
    const __nv_bfloat16* Wgu = tw16(h, F + "w_gu", static_cast<size_t>(d) * 2 * m);
    const __nv_bfloat16* Wdn = tw16(h, F + "w_down", static_cast<size_t>(m) * d);
    if (d <= 256 && d % 8 == 0) {
      k_rmsnorm_rows_v<__nv_bfloat16, __nv_bfloat16><<<std::max(1, std::min((M + 7) / 8, 8 * h.num_sms)), 256, 0,
                                                        h.stream>>>(T.x1, w32(h, Bk + "ffn_norm"), M, d, xf, inv);
    } else {
      k_rmsnorm_rows<__nv_bfloat16, __nv_bfloat16><<<(M + 7) / 8, 256, 0, h.stream>>>(
          T.x1, w32(h, Bk + "ffn_norm"), M, d, nullptr, 1, 1, xf, inv);
    }
    gemm_rm16(h, false, false, M, 2 * m, d, xf, d, Wgu, 2 * m, GU, 2 * m, true);
    k_swiglu_z<__nv_bfloat16, __nv_bfloat16><<<ew_grid(static_cast<size_t>(M) * m / 8), 256, 0, h.stream>>>(GU, M, m, z);
    if (!dX16_ready) k_f32_to_bf16<<<ew_grid(nq), 256, 0, h.stream>>>(dX, nq, dX16);
    dX16_ready = false;
    gemm_rm16(h, true, false, m, d, M, z, m, dX16, d, grad_ptr(h, F + "w_down"), d, false);
    gemm_rm16(h, false, true, M, m, d, dX16, d, Wdn, d, z, m, true);  // z <- dz
    k_swiglu_bwd16<<<ew_grid(static_cast<size_t>(M) * m / 8), 256, 0, h.stream>>>(z, GU, M, m, dGU);
    gemm_rm16(h, true, false, d, m, M, xf, d, dGU, 2 * m, grad_ptr(h, F + "w_gate"), m, false);
    gemm_rm16(h, true, false, d, m, M, xf, d, dGU + m, 2 * m, grad_ptr(h, F + "w_up"), m, false);
    float* dxf = h.tw[3];
    gemm_rm16(h, false, true, M, d, 2 * m, dGU, 2 * m, Wgu, 2 * m, dxf, d, false);
    __nv_bfloat16* dXr16 = reinterpret_cast<__nv_bfloat16*>(h.tw[11]);  // d(xr) in bf16 for the next GEMMs
    rms_bwd<__nv_bfloat16>(h, dxf, T.x1, inv, w32(h, Bk + "ffn_norm"), M, d, dX, 1, grad_ptr(h, Bk + "ffn_norm"),
                           dXr16);
    check_launch("ffn backward");
    // attention (attention.cpp:134-202); dX now holds d(xr). GEMM operands in bf16 (fp32
    // accumulation and gradients): the gated output, d(xr), the normalised rows, d(g_raw),
    // dQ / dK / dV
    __nv_bfloat16* Hm = reinterpret_cast<__nv_bfloat16*>(h.tw[4]);
    float* dH = h.tw[5];
    float* dO = h.tw[6];
    __nv_bfloat16* dgraw = reinterpret_cast<__nv_bfloat16*>(h.tw[7]);

    const __nv_bfloat16* Wo16 = tw16(h, A + "wo", static_cast<size_t>(d) * d);
    const __nv_bfloat16* Wg16 = tw16(h, A + "wg", static_cast<size_t>(d) * d);
    const __nv_bfloat16* Wq16 = tw16(h, A + "wq", static_cast<size_t>(d) * d);
    const __nv_bfloat16* Wk16 = tw16(h, A + "wk", static_cast<size_t>(d) * d);
    const __nv_bfloat16* Wv16 = tw16(h, A + "wv", static_cast<size_t>(d) * d);
    k_gate_fwd<__nv_bfloat16><<<ew_grid(nq), 256, 0, h.stream>>>(T.g, T.o_pre, nq, Hm);
    gemm_rm16(h, true, false, d, d, M, Hm, d, dXr16, d, grad_ptr(h, A + "wo"), d, false);
    gemm_rm16(h, false, true, M, d, d, dXr16, d, Wo16, d, dH, d, false);
    float* Dd = h.tw[15];
    // fp32 dO only for the SIMT attention backward; the tcgen05 / mma.sync kernels read dO16
    k_gate_bwd_rows<<<warp_rows_grid(M), 256, 0, h.stream>>>(dH, T.g, T.o_pre, M, L.Rq, H, dk,
                                                             (h.attn_bwd_tc || h.attn_bwd_mma) ? nullptr : dO, h.dO16, dgraw,
                                                             Dd);
    __nv_bfloat16* xn = reinterpret_cast<__nv_bfloat16*>(h.tw[2]);
    __nv_bfloat16* xq = reinterpret_cast<__nv_bfloat16*>(h.tw[3]);
    float* inv_a = h.tw[14] + static_cast<size_t>(h.train_B) * h.L0;
    if (d <= 256 && d % 8 == 0) {
      k_rmsnorm_rows_v<__nv_bfloat16, __nv_bfloat16><<<std::max(1, std::min((Mkv + 7) / 8, 8 * h.num_sms)), 256, 0,
                                                        h.stream>>>(T.x_in, w32(h, Bk + "attn_norm"), Mkv, d, xn,
                                                                    inv_a);
    } else {
      k_rmsnorm_rows<__nv_bfloat16, __nv_bfloat16><<<(Mkv + 7) / 8, 256, 0, h.stream>>>(
          T.x_in, w32(h, Bk + "attn_norm"), Mkv, d, nullptr, 1, 1, xn, inv_a);
    }
    const __nv_bfloat16* xqp = xn;
    if (!lp.q_identity) {
      k_gather_f32<__nv_bfloat16, __nv_bfloat16><<<(M + 7) / 8, 256, 0, h.stream>>>(xn, L.query_rows, L.Rq, L.Rkv,
                                                                                    M, d, xq);
      xqp = xq;
    }
    check_launch("attention rows");
    gemm_rm16(h, true, false, d, d, M, xqp, d, dgraw, d, grad_ptr(h, A + "wg"), d, false);
    // d(xq) = dgraw Wg^T + dQ Wq^T. When the query rows are all kv rows in order (unpruned
    // layers) d(xq) is accumulated straight into d(xn) (tw[5]: dH is dead after the gate
    // backward), so no separate [M, d] buffer is written and scattered back.
    float* dxn = h.tw[5];
    float* dxq = lp.q_identity ? dxn : h.tw[4];  // (the gated output is no longer needed) -- fp32 [M, d]
    gemm_rm16(h, false, true, M, d, d, dgraw, d, Wg16, d, dxq, d, false);
    // attention core
    AttnBwdArgs ab;
    ab.q = T.q;
    ab.k = T.k;
    ab.v = T.v;
    ab.dO = dO;
    ab.lse = T.lse;
    ab.D = Dd;
    ab.rowmeta = L.rowmeta;
    ab.H = H;
    ab.Rq = L.Rq;
    ab.Rkv = L.Rkv;
    ab.BH = B * H;
    ab.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(dk)));
    ab.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(dk)));
    float* dQ = h.tw[8];
    float* dK = h.tw[9];
    float* dV = h.tw[10];
    ab.dq = dQ;
    ab.dk = dK;
    ab.dv = dV;
    ab.blk_off = T.dq_off;
    ab.blk_iv = T.dq_iv;
    AttnBwdArgs ak = ab;
    ak.blk_off = T.dkv_off;
    ak.blk_iv = T.dkv_iv;
    if (h.attn_bwd_tc) {
      // (only the bf16 dV feeds the GEMMs below: no fp32 copy)
      attn_core_backward_tc(h, L, T, B, Dd, dQ, dK, nullptr,
                            reinterpret_cast<__nv_bfloat16*>(h.tw[12]) + 2 * static_cast<size_t>(h.train_B) * h.L0 * d);
    } else if (h.attn_bwd_mma) {
      AttnBwdMmaArgs am;
      am.q = T.q;
      am.k = T.k;
      am.v = T.v;
      am.dO16 = h.dO16;
      am.lse = T.lse;
      am.D = Dd;
      am.rowmeta = L.rowmeta;
      am.qb_off = T.qb_off;
      am.qb_list = T.qb_list;
      am.dq = dQ;
      am.dk = dK;
      am.dv = dV;
      am.dv16 = reinterpret_cast<__nv_bfloat16*>(h.tw[12]) + 2 * static_cast<size_t>(h.train_B) * h.L0 * d;
      am.H = H;
      am.Rq = L.Rq;
      am.Rkv = L.Rkv;
      am.scale = ab.scale;
      am.scale_log2 = ab.scale_log2;
      CK(cudaMemsetAsync(dQ, 0, static_cast<size_t>(M) * d * 4, h.stream));
      const dim3 grid((L.Rkv + 63) / 64, B * H);
      switch (dk) {
        case 16: k_attn_bwd_mma<16><<<grid, 128, 0, h.stream>>>(am); break;
        case 32: k_attn_bwd_mma<32><<<grid, 128, 0, h.stream>>>(am); break;
        case 64: k_attn_bwd_mma<64><<<grid, 128, 0, h.stream>>>(am); break;
        default: throw ConfigError("training: unsupported head dim");
      }
    } else {
      switch (dk) {
        case 16:
          k_attn_bwd_dq<16><<<dim3((L.Rq + 31) / 32, B * H), 32, 0, h.stream>>>(ab);
          k_attn_bwd_dkv<16><<<dim3((L.Rkv + 31) / 32, B * H), 32, 0, h.stream>>>(ak);
          break;
        case 32:
          k_attn_bwd_dq<32><<<dim3((L.Rq + 31) / 32, B * H), 32, 0, h.stream>>>(ab);
          k_attn_bwd_dkv<32><<<dim3((L.Rkv + 31) / 32, B * H), 32, 0, h.stream>>>(ak);
          break;
        case 64:
          k_attn_bwd_dq<64><<<dim3((L.Rq + 31) / 32, B * H), 32, 0, h.stream>>>(ab);
          k_attn_bwd_dkv<64><<<dim3((L.Rkv + 31) / 32, B * H), 32, 0, h.stream>>>(ak);
          break;
        default:
          throw ConfigError("training: unsupported head dim");
      }
    }
    check_launch("attention core backward");
    // QKNorm + RoPE backward against recomputed raw projections
    float* raw = h.tw[11];
    __nv_bfloat16* dQ16 = reinterpret_cast<__nv_bfloat16*>(h.tw[12]);
    __nv_bfloat16* dK16 = dQ16 + static_cast<size_t>(h.train_B) * h.L0 * d;
    __nv_bfloat16* dV16 = dK16 + static_cast<size_t>(h.train_B) * h.L0 * d;
    gemm_rm16(h, false, false, M, d, d, xqp, d, Wq16, d, raw, d, false);
    // persistent grid (register-held gain partials per warp, one smem reduction per CTA); only
    // the bf16 d(raw) feeds the GEMMs below, so the fp32 copy is not written
    const int qk_grid_q = std::max(1, std::min((M + 7) / 8, 4 * h.num_sms));
    k_qknorm_rope_bwd_v<1><<<qk_grid_q, 256, d * 4, h.stream>>>(dQ, raw, M, L.Rq, L.pos_q, h.rope, H, dk,
                                                              w32(h, A + "qk_gain_q"), nullptr, grad_ptr(h, A + "qk_gain_q"),
                                                              dQ16);
    gemm_rm16(h, false, false, Mkv, d, d, xn, d, Wk16, d, raw, d, false);
    const int qk_grid_k = std::max(1, std::min((Mkv + 7) / 8, 4 * h.num_sms));
    k_qknorm_rope_bwd_v<1><<<qk_grid_k, 256, d * 4, h.stream>>>(dK, raw, Mkv, L.Rkv, L.pos_kv, h.rope, H, dk,
                                                              w32(h, A + "qk_gain_k"), nullptr, grad_ptr(h, A + "qk_gain_k"),
                                                              dK16);
    if (!h.attn_bwd_mma && !h.attn_bwd_tc) k_f32_to_bf16<<<ew_grid(nkv), 256, 0, h.stream>>>(dV, nkv, dV16);  // (SIMT path)
    check_launch("qknorm/rope backward");
    gemm_rm16(h, true, false, d, d, M, xqp, d, dQ16, d, grad_ptr(h, A + "wq"), d, false);
    gemm_rm16(h, true, false, d, d, Mkv, xn, d, dK16, d, grad_ptr(h, A + "wk"), d, false);
    gemm_rm16(h, true, false, d, d, Mkv, xn, d, dV16, d, grad_ptr(h, A + "wv"), d, false);
    gemm_rm16(h, false, true, M, d, d, dQ16, d, Wq16, d, dxq, d, false, 1.f);
    if (lp.q_identity) {
      // d(xn) already holds d(xq); d(x_in) = d(xr) + RMSN_bwd(d(xn)) accumulated in place into dX
      // (the same fp32 sum as the scatter below, operands swapped)
      gemm_rm16(h, false, true, Mkv, d, d, dK16, d, Wk16, d, dxn, d, false, 1.f);
      gemm_rm16(h, false, true, Mkv, d, d, dV16, d, Wv16, d, dxn, d, false, 1.f);
      // ... and, below the first layer, its bf16 copy for the next layer's FFN GEMMs (tw[3]: the
      // FFN's d(xf) is dead), so that layer skips its own conversion pass
      rms_bwd<__nv_bfloat16>(h, dxn, T.x_in, inv_a, w32(h, Bk + "attn_norm"), Mkv, d, dX, 1,
                             grad_ptr(h, Bk + "attn_norm"),
                             l > 0 ? reinterpret_cast<__nv_bfloat16*>(h.tw[3]) : nullptr);
      dX16_ready = l > 0;
      check_launch("attention backward");
      continue;
    }
    gemm_rm16(h, false, true, Mkv, d, d, dK16, d, Wk16, d, dxn, d, false);
    gemm_rm16(h, false, true, Mkv, d, d, dV16, d, Wv16, d, dxn, d, false, 1.f);
    k_scatter_add_rows<<<(M + 7) / 8, 256, 0, h.stream>>>(dxq, L.query_rows, B, L.Rq, L.Rkv, d, dxn);
    // d(x_in) = RMSN_bwd(dxn) + scatter of d(xr) through P(x, L_out)
    rms_bwd<__nv_bfloat16>(h, dxn, T.x_in, inv_a, w32(h, Bk + "attn_norm"), Mkv, d, dXn, 0,
                           grad_ptr(h, Bk + "attn_norm"));
    k_scatter_add_rows<<<(M + 7) / 8, 256, 0, h.stream>>>(dX, L.query_rows, B, L.Rq, L.Rkv, d, dXn);
    check_launch("attention backward");
    std::swap(dX, dXn);
  }
  h.dtokens = dX;
  // ---- Tokenizer::backward (tokenizer.cpp:286-352); the item table is frozen
  const TokParams tp = tok_params(h, B);
  const int gcount[3] = {B * c.n_hist, B * N, B * c.n_profile_fields};
  const int gK[3] = {c.item_dim + c.action_dim + c.scene_dim + c.time_dim, c.item_dim, c.profile_dim};
  const char* gname[3] = {"hist", "cand", "prof"};
  __nv_bfloat16* catb = reinterpret_cast<__nv_bfloat16*>(h.tw[13]);
  float* catf = h.tw[12];
  float* y = h.tw[2];
  float* dy = h.tw[3];
  float* dproj = h.tw[4];
  float* dcat = h.tw[5];
  for (int g = 0; g < 3; ++g) {
    const int n = gcount[g], K = gK[g];
    if (n == 0) continue;
    const std::string W = std::string("tok.w_") + gname[g];
    k_tok_concat<<<warp_rows_grid(n), 256, 0, h.stream>>>(tp, g, K, catb, h.t_rows);
    k_bf16_to_f32<<<ew_grid(static_cast<size_t>(n) * K), 256, 0, h.stream>>>(catb, static_cast<size_t>(n) * K, catf);
    gemm_rm(h, false, false, n, d, K, catf, K, w32(h, W), d, y, d);
    k_bias_add<<<ew_grid(static_cast<size_t>(n) * d), 256, 0, h.stream>>>(y, w32(h, std::string("tok.b_") + gname[g]),
                                                                         n, d);
    rms_rows<float>(h, y, nullptr, n, d, nullptr, inv);
    k_gather_f32<float><<<warp_rows_grid(n), 256, 0, h.stream>>>(dX, h.t_rows, n, 0, n, d, dy);
    rms_bwd<float>(h, dy, y, inv, w32(h, std::string("tok.g_") + gname[g]), n, d, dproj, 0,
                   grad_ptr(h, std::string("tok.g_") + gname[g]));
    gemm_rm(h, true, false, K, d, n, catf, K, dproj, d, grad_ptr(h, W), d);
    k_colsum<<<dim3((d + 31) / 32, std::min(148, (n + 255) / 256)), dim3(32, 8), 0, h.stream>>>(
        dproj, n, d, grad_ptr(h, std::string("tok.b_") + gname[g]));
    if (g == 1 && !item_train) continue;  // the candidate concat is the item row only
    // d(concat) = dproj W^T with W zero-padded to Kp rows, so N = Kp is a multiple of 32 and the
    // product runs on the TF32 tcgen05 GEMM (N = 56 would fall back to the SIMT kernel)
    const int Kp = (K + 31) & ~31;
    const size_t wp_n = static_cast<size_t>(Kp) * d;
    if (wp_n > h.wpad_cap) {
      h.wpad = h.dalloc<float>(wp_n);
      h.wpad_cap = wp_n;
    }
    CK(cudaMemsetAsync(h.wpad, 0, wp_n * 4, h.stream));
    CK(cudaMemcpyAsync(h.wpad, w32(h, W), static_cast<size_t>(K) * d * 4, cudaMemcpyDeviceToDevice, h.stream));
    gemm_rm(h, false, true, n, Kp, d, dproj, d, h.wpad, d, dcat, Kp);
    if (item_train && g != 2)  // tokenizer.cpp:315-317, 346-352: the item columns of d(concat)
      k_item_grad_scatter<<<std::min(148 * 4, (n + 7) / 8), 256, 0, h.stream>>>(
          dcat, Kp, n, g == 0 ? tp.hist_item : tp.cand_item, c.n_items, c.item_dim, h.item_grad);
    if (g == 1) continue;
    TokTableGrads tg{};
    int tsize = 0;
    if (g == 0) {
      tg.action = grad_ptr(h, "tok.action_table");
      tg.scene = grad_ptr(h, "tok.scene_table");
      tg.time = grad_ptr(h, "tok.time_table");
      tsize = c.n_actions * c.action_dim + c.n_scenes * c.scene_dim + c.n_time_buckets * c.time_dim;
    } else {
      for (int f = 0; f < c.n_profile_fields; ++f) {
        tg.prof[f] = grad_ptr(h, "tok.profile_table." + std::to_string(f));
        tsize += c.profile_vocab[f] * c.profile_dim;
      }
    }
    if (tsize * 4 > 200 * 1024) throw ConfigError("training: feature tables too large for the scatter kernel");
    int* pvd = nullptr;
    if (g == 2) {
      int32_t*& pvd_h = h.cand_maps[-1];  // profile vocab sizes (device), cached
      if (!pvd_h) pvd_h = h.upload(std::vector<int32_t>(c.profile_vocab, c.profile_vocab + std::max(c.n_profile_fields, 1)));
      pvd = pvd_h;
    }
    if (tsize * 4 > 48 * 1024)
      CK(cudaFuncSetAttribute(k_tok_table_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, tsize * 4));
    k_tok_table_scatter<<<std::min(148 * 2, (n + 7) / 8), 256, tsize * 4, h.stream>>>(
        dcat, g == 0 ? 0 : 1, n, Kp, h.in_action, h.in_scene, h.hist_time, h.in_prof, c.n_profile_fields, c.item_dim,
        c.action_dim, c.scene_dim, c.time_dim, c.n_actions, c.n_scenes, c.n_time_buckets, pvd, c.profile_dim, tg);
  }
  if (c.special_tokens)
    k_special_grad<<<(3 * d + 255) / 256, 256, 0, h.stream>>>(dX, B, h.L0, c.n_hist, c.n_profile_fields, d,
                                                              c.pretrain ? 1 : 3, grad_ptr(h, "tok.special"));
  check_launch("tokenizer backward");
  for (const std::string& name : h.frozen) {  // frozen tensors receive zero gradient
    auto it = h.grad_index.find(name);
    if (it == h.grad_index.end()) continue;
    const size_t n = static_cast<size_t>(it->second.second.first) * it->second.second.second;
    CK(cudaMemsetAsync(h.grads + it->second.first, 0, n * sizeof(float), h.stream));
  }
}


// ====================================================================== generic forward (d > 256)
static void ensure_generic_buffers(Handle& h) {
  if (h.gX[0]) return;
  if (!h.cublas && cublasCreate(&h.cublas) != CUBLAS_STATUS_SUCCESS) throw RuntimeFailure("cublasCreate failed");
  const size_t rows = static_cast<size_t>(h.Bmax) * h.L0;
  const int d = h.d, m = h.m;
  for (int i = 0; i < 2; ++i) h.gX[i] = h.dalloc<float>(rows * d);
  // 0 xn, 1 xq / xf, 2 Qr / a, 3 Kr, 4 Vr, 5 Gr, 6 GU [rows, 2m], 7 z [rows, m], 8 tokenizer
  // concat rows [rows, 64], 9 head scratch
  for (int i = 0; i < 6; ++i) h.gw[i] = h.dalloc<float>(rows * d);
  h.gw[6] = h.dalloc<float>(rows * 2 * m);
  h.gw[7] = h.dalloc<float>(rows * m);
  h.gw[8] = h.dalloc<float>(rows * 64);
  h.gw[9] = h.dalloc<float>(static_cast<size_t>(h.Bmax) * h.cfg.n_cand * (2 * d + h.dh + 4));
  h.g_rows = h.dalloc<int32_t>(rows);
}

static const __nv_bfloat16* w16(Handle& h, const std::string& name) {
  auto it = h.w16.find(name);
  if (it != h.w16.end()) return it->second;
  auto src = h.w32.find(name);
  if (src == h.w32.end()) throw RuntimeFailure("no parameter " + name);
  size_t n = 0;
  if (auto g = h.grad_index.find(name); g != h.grad_index.end())
    n = static_cast<size_t>(g->second.second.first) * g->second.second.second;
  else if (name.rfind("tok.w_", 0) == 0)
    n = static_cast<size_t>(name == "tok.w_hist" ? h.cfg.item_dim + h.cfg.action_dim + h.cfg.scene_dim + h.cfg.time_dim
                            : name == "tok.w_cand" ? h.cfg.item_dim : h.cfg.profile_dim) * h.d;
  else if (name.size() > 5 && name.compare(name.size() - 5, 5, ".w_gu") == 0)
    n = static_cast<size_t>(h.d) * 2 * h.m;
  else
    throw RuntimeFailure("no size for parameter " + name);
  __nv_bfloat16* dst = h.dalloc<__nv_bfloat16>(n);
  k_f32_to_bf16<<<ew_grid(n), 256, 0, h.stream>>>(src->second, n, dst);
  check_launch("weight cast");
  return h.w16[name] = dst;
}

// bf16 [K, n * N] row-major weight whose column blocks are the named [K, N] parameters
// (built once per handle; the generic path's concatenated projections).
static const __nv_bfloat16* w16_cat(Handle& h, const std::string& key, const std::vector<std::string>& parts) {
  auto it = h.w16.find(key);
  if (it != h.w16.end()) return it->second;
  const auto& gi = h.grad_index.at(parts[0]);
  const int64_t K = gi.second.first, N = gi.second.second, n = static_cast<int64_t>(parts.size());
  __nv_bfloat16* dst = h.dalloc<__nv_bfloat16>(static_cast<size_t>(K * N * n));
  for (int64_t i = 0; i < n; ++i) {
    const __nv_bfloat16* src = w16(h, parts[i]);
    CK(cudaMemcpy2DAsync(dst + i * N, static_cast<size_t>(n * N) * 2, src, static_cast<size_t>(N) * 2,
                         static_cast<size_t>(N) * 2, static_cast<size_t>(K), cudaMemcpyDeviceToDevice, h.stream));
  }
  return h.w16[key] = dst;
}

static void forward_generic(Handle& h, int B) {
  ensure_generic_buffers(h);
  CK(cublasSetStream(h.cublas, h.stream) == CUBLAS_STATUS_SUCCESS ? cudaSuccess : cudaErrorUnknown);
  const SortConfig& c = h.cfg;
  const int d = h.d, m = h.m, H = h.H, dk = h.dk, N = c.n_cand;
  // ---- tokenizer: gather -> projection -> bias + RMSNorm (tokenizer.cpp:144-238)
  const TokParams tp = tok_params(h, B);
  float* X = h.gX[0];
  const int gcount[3] = {B * c.n_hist, B * N, B * c.n_profile_fields};
  const int gK[3] = {c.item_dim + c.action_dim + c.scene_dim + c.time_dim, c.item_dim, c.profile_dim};
  const char* gname[3] = {"hist", "cand", "prof"};
  for (int g = 0; g < 3; ++g) {
    if (gcount[g] == 0) continue;
    __nv_bfloat16* cat = reinterpret_cast<__nv_bfloat16*>(h.gw[8]);
    k_tok_concat<<<warp_rows_grid(gcount[g]), 256, 0, h.stream>>>(tp, g, gK[g], cat, h.g_rows);
    if (h.stream_gemm) {
      const std::string wn = std::string("tok.w_") + gname[g];
      gemm_stream(h, cat, gK[g], gcount[g], gK[g], wT16(h, wn + "^T", {wn}), (gK[g] + 7) & ~7, d,
                  GsStore<float>{h.gw[0], d});
    } else {
      gemm_rm_bf16(h, gcount[g], d, gK[g], cat, gK[g], w16(h, std::string("tok.w_") + gname[g]), d, h.gw[0], d);
    }
    k_tok_finish<<<warp_rows_grid(gcount[g]), 256, 0, h.stream>>>(h.gw[0], w32(h, std::string("tok.b_") + gname[g]),
                                                                w32(h, std::string("tok.g_") + gname[g]), h.g_rows,
                                                                gcount[g], d, X);
  }
  if (c.special_tokens)
    k_tok_specials<<<warp_rows_grid(B * 3), 256, 0, h.stream>>>(w32(h, "tok.special"), B, h.L0, c.n_hist,
                                                               c.n_profile_fields, d, X);
  check_launch("generic tokenizer");
  stage_mark(h, "tokenizer");
  // ---- blocks
  int cur = 0;
  for (int l = 0; l < c.layers; ++l) {
    const LayerDev& L = h.layers[l];
    const LayerPlan& lp = h.plan.layers[l];
    const std::string sl = std::to_string(l);
    const std::string A = "attn." + sl + ".", F = "ffn." + sl + ".", Bk = "block." + sl + ".";
    const int M = B * L.Rq, Mkv = B * L.Rkv;
    float* x = h.gX[cur];
    float* xo = h.gX[1 - cur];
    __nv_bfloat16* xn = reinterpret_cast<__nv_bfloat16*>(h.gw[0]);
    __nv_bfloat16* xq = reinterpret_cast<__nv_bfloat16*>(h.gw[1]);
    resid_rmsnorm(h, x, nullptr, 1, 1, nullptr, w32(h, Bk + "attn_norm"), Mkv, d, nullptr, xn);
    const __nv_bfloat16* xqp = xn;
    if (!lp.q_identity) {
      k_gather_f32<__nv_bfloat16, __nv_bfloat16><<<warp_rows_grid(M), 256, 0, h.stream>>>(xn, L.query_rows, L.Rq,
                                                                                          L.Rkv, M, d, xq);
      xqp = xq;
    }
    // bf16 projection outputs (fp32 accumulation), consumed by the per-head prep: two GEMMs
    // with column-concatenated weights, [Wq | Wg] on the query rows and [Wk | Wv] on all rows
    const bool sg = h.stream_gemm && dk == 64;
    if (sg) {
      // [Wq | Wg] on the query rows, [Wk | Wv] on all rows; QKNorm + RoPE + head-major layout
      // (and the sigmoid gate) in the epilogue, straight from the fp32 accumulators
      gemm_stream(h, xqp, d, M, d, wT16(h, A + "wq|wg^T", {A + "wq", A + "wg"}), d, 2 * d,
                  GsQKVG{d, H, L.Rq, L.pos_q, h.rope, attn_prescaled(h, L) ? L.gain_q_s : L.gain_q, h.Qb, h.Gb, true});
      gemm_stream(h, xn, d, Mkv, d, wT16(h, A + "wk|wv^T", {A + "wk", A + "wv"}), d, 2 * d,
                  GsQKVG{d, H, L.Rkv, L.pos_kv, h.rope, L.gain_k, h.Kb, h.Vb, false});
    } else {
      __nv_bfloat16* pqg = reinterpret_cast<__nv_bfloat16*>(h.gw[2]);  // [M, 2d]
      __nv_bfloat16* pkv = reinterpret_cast<__nv_bfloat16*>(h.gw[3]);  // [Mkv, 2d]
      gemm_rm_bf16(h, M, 2 * d, d, xqp, d, w16_cat(h, A + "wq|wg", {A + "wq", A + "wg"}), 2 * d, pqg, 2 * d, 0.f, true);
      gemm_rm_bf16(h, Mkv, 2 * d, d, xn, d, w16_cat(h, A + "wk|wv", {A + "wk", A + "wv"}), 2 * d, pkv, 2 * d, 0.f, true);
      qkv_prep(h, pqg, 2 * d, M, L.Rq, H, dk, 0, L.pos_q, attn_prescaled(h, L) ? L.gain_q_s : L.gain_q, h.Qb);
      qkv_prep(h, pkv, 2 * d, Mkv, L.Rkv, H, dk, 1, L.pos_kv, L.gain_k, h.Kb);
      qkv_prep(h, pkv + d, 2 * d, Mkv, L.Rkv, H, dk, 2, nullptr, nullptr, h.Vb);
      qkv_prep(h, pqg + d, 2 * d, M, L.Rq, H, dk, 3, nullptr, nullptr, h.Gb);
    }
    check_launch("generic projections");
    stage_mark(h, "L" + sl + ".qkvg");
    launch_attention(h, L, lp, B);  // tcgen05 core; writes the gated output to h.Hg
    stage_mark(h, "L" + sl + ".attention");
    __nv_bfloat16* xf = reinterpret_cast<__nv_bfloat16*>(h.gw[1]);
    __nv_bfloat16* z = reinterpret_cast<__nv_bfloat16*>(h.gw[7]);
    if (h.stream_gemm) {
      // x1 = P(x) + attn Wo (fp32, in xo) in the epilogue; RMSN(x1) -> bf16 FFN input; up
      // projection with SwishGLU in the epilogue -> z; down projection accumulating into x1
      gemm_stream(h, h.Hg, d, M, d, wT16(h, A + "wo^T", {A + "wo"}), d, d,
                  GsResidF32{x, L.query_rows, L.Rq, L.Rkv, d, xo});
      resid_rmsnorm(h, xo, nullptr, 1, 1, nullptr, w32(h, Bk + "ffn_norm"), M, d, nullptr, xf);
      gemm_stream(h, xf, d, M, d, wT16(h, F + "w_gate|w_up^T", {F + "w_gate", F + "w_up"}, true), d, 2 * m,
                  GsSwiGLU{z, m});
      gemm_stream(h, z, m, M, m, wT16(h, F + "w_down^T", {F + "w_down"}), m, d, GsAccF32{xo, d});
    } else {
      gemm_rm_bf16(h, M, d, d, h.Hg, d, w16(h, A + "wo"), d, h.gw[2], d);
      // x1 = P(x) + attn (kept fp32 in xo), then RMSN(x1) -> bf16 FFN input, in one pass
      resid_rmsnorm(h, x, L.query_rows, L.Rq, L.Rkv, h.gw[2], w32(h, Bk + "ffn_norm"), M, d, xo, xf);
      __nv_bfloat16* gu = reinterpret_cast<__nv_bfloat16*>(h.gw[6]);  // bf16 [gate | up] pre-activations
      gemm_rm_bf16(h, M, 2 * m, d, xf, d, w16(h, F + "w_gu"), 2 * m, gu, 2 * m, 0.f, true);
      k_swiglu_z<__nv_bfloat16, __nv_bfloat16><<<ew_grid(static_cast<size_t>(M) * m / 8), 256, 0, h.stream>>>(gu, M, m, z);
      gemm_rm_bf16(h, M, d, m, z, m, w16(h, F + "w_down"), d, xo, d, 1.f);
    }
    check_launch("generic block tail");
    stage_mark(h, "L" + sl + ".tail");
    cur = 1 - cur;
  }
  h.gX_final = cur;
  // ---- final RMSNorm + head on the candidate rows
  const LayerDev& last = h.layers.back();
  const int R = last.Rq, BN = B * N;
  std::vector<int32_t> cmap_h(N);
  for (int j = 0; j < N; ++j) cmap_h[j] = R - N + j;
  int32_t*& cmap = h.cand_maps[R];
  if (!cmap) cmap = h.upload(cmap_h);
  float* xh = h.gw[9];
  float* hid = xh + static_cast<size_t>(BN) * d;
  float* lo = hid + static_cast<size_t>(BN) * h.dh;
  k_gather_f32<float><<<warp_rows_grid(BN), 256, 0, h.stream>>>(h.gX[cur], cmap, N, R, BN, d, h.gw[0]);
  k_rmsnorm_rows<float><<<warp_rows_grid(BN), 256, 0, h.stream>>>(h.gw[0], w32(h, "final_norm.gain"), BN, d, nullptr,
                                                                  1, 1, xh, nullptr);
  gemm_rm(h, false, false, BN, h.dh, d, xh, d, w32(h, "head.w1"), h.dh, hid, h.dh);
  k_bias_relu<<<ew_grid(static_cast<size_t>(BN) * h.dh), 256, 0, h.stream>>>(hid, w32(h, "head.b1"), BN, h.dh);
  gemm_rm(h, false, false, BN, 3, h.dh, hid, h.dh, w32(h, "head.w2"), 3, lo, 3);
  k_head_out<<<(BN * 3 + 255) / 256, 256, 0, h.stream>>>(lo, w32(h, "head.b2"), BN, h.logits, h.probs);
  check_launch("generic head");
  stage_mark(h, "head");
}

// Rebuild the bf16 inference weights (and the derived fp32 W_gate|W_up) from the masters,
// and the per-layer QKNorm logit bounds from the updated gains.
static void repack_weights(Handle& h) {
  const SortConfig& c = h.cfg;
  const int d = h.d, m = h.m, H = h.H, dk = h.dk;
  auto grid = [](size_t n) { return static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 32)); };
  auto cast = [&](const std::string& name, __nv_bfloat16* dst, size_t n) {
    k_cast_bf16<<<grid(n), 256, 0, h.stream>>>(h.w32.at(name), n, dst);
  };
  cast("tok.action_table", h.action, static_cast<size_t>(c.n_actions) * c.action_dim);
  cast("tok.scene_table", h.scene, static_cast<size_t>(c.n_scenes) * c.scene_dim);
  cast("tok.time_table", h.time, static_cast<size_t>(c.n_time_buckets) * c.time_dim);
  for (int f = 0; f < c.n_profile_fields; ++f)
    cast("tok.profile_table." + std::to_string(f), h.prof + static_cast<size_t>(h.prof_off[f]) * c.profile_dim,
         static_cast<size_t>(c.profile_vocab[f]) * c.profile_dim);
  cast("tok.special", h.special, static_cast<size_t>(3) * d);
  const int gk[3] = {c.item_dim + c.action_dim + c.scene_dim + c.time_dim, c.item_dim, c.profile_dim};
  const char* gw[3] = {"tok.w_hist", "tok.w_cand", "tok.w_prof"};
  for (int g = 0; g < 3; ++g)
    if (h.tok_wt[g])
      k_repack_t<<<grid(static_cast<size_t>(d) * 64), 256, 0, h.stream>>>(h.w32.at(gw[g]), nullptr, gk[g], d, 64,
                                                                       h.tok_wt[g]);
  for (int l = 0; l < c.layers; ++l) {
    LayerDev& L = h.layers[l];
    const std::string a = "attn." + std::to_string(l) + ".", f = "ffn." + std::to_string(l) + ".",
                      bk = "block." + std::to_string(l) + ".";
    QkvgSrc src{{h.w32.at(a + "wq"), h.w32.at(a + "wk"), h.w32.at(a + "wv"), h.w32.at(a + "wg")}};
    const float* ga = h.w32.at(bk + "attn_norm");
    k_repack_qkvg<<<grid(static_cast<size_t>(4) * d * d), 256, 0, h.stream>>>(
        src, ga, make_int4(kSecQ, kSecV, kSecK, kSecG), 4, H, dk, d, L.w_all);
    k_repack_qkvg<<<grid(static_cast<size_t>(2) * d * d), 256, 0, h.stream>>>(src, ga, make_int4(kSecK, kSecV, 0, 0),
                                                                             2, H, dk, d, L.w_kv);
    k_repack_qkvg<<<grid(static_cast<size_t>(2) * d * d), 256, 0, h.stream>>>(src, ga, make_int4(kSecQ, kSecG, 0, 0),
                                                                             2, H, dk, d, L.w_qg);
    k_repack_t<<<grid(static_cast<size_t>(d) * d), 256, 0, h.stream>>>(h.w32.at(a + "wo"), nullptr, d, d, d, L.w_o);
    k_repack_up<<<grid(static_cast<size_t>(2) * m * d), 256, 0, h.stream>>>(h.w32.at(f + "w_gate"), h.w32.at(f + "w_up"),
                                                                         h.w32.at(bk + "ffn_norm"), d, m, L.w_up);
    k_repack_t<<<grid(static_cast<size_t>(d) * m), 256, 0, h.stream>>>(h.w32.at(f + "w_down"), nullptr, m, d, m,
                                                                    L.w_down);
    k_concat_gu<<<grid(static_cast<size_t>(d) * 2 * m), 256, 0, h.stream>>>(h.w32.at(f + "w_gate"), h.w32.at(f + "w_up"),
                                                                          d, m, h.w32.at(f + "w_gu"));
    std::vector<float> gq(static_cast<size_t>(H) * dk), gkv(static_cast<size_t>(H) * dk);
    CK(cudaMemcpyAsync(gq.data(), L.gain_q, gq.size() * 4, cudaMemcpyDeviceToHost, h.stream));
    CK(cudaMemcpyAsync(gkv.data(), L.gain_k, gkv.size() * 4, cudaMemcpyDeviceToHost, h.stream));
    CK(cudaStreamSynchronize(h.stream));
    float mq = 0.f, mk = 0.f;
    for (float v : gq) mq = std::max(mq, std::fabs(v));
    for (float v : gkv) mk = std::max(mk, std::fabs(v));
    L.logit_bound = 1.02f * std::sqrt(static_cast<float>(dk)) * mq * mk + 1e-3f;
    if (L.gain_q_s) {
      const float sl2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(dk)));
      for (float& v : gq) v *= sl2;
      CK(cudaMemcpyAsync(L.gain_q_s, gq.data(), gq.size() * 4, cudaMemcpyHostToDevice, h.stream));
      CK(cudaStreamSynchronize(h.stream));
    }
  }
  if (!h.tw16.empty()) {  // bf16 copies the training backward reads, one launch for all
    if (h.tw16_nseg != static_cast<int>(h.tw16.size())) {
      std::vector<CastSeg> segs;
      size_t nmax = 0;
      for (auto& kv : h.tw16) {
        segs.push_back(CastSeg{w32(h, kv.first), kv.second.first, kv.second.second});
        nmax = std::max(nmax, kv.second.second);
      }
      h.tw16_segs = h.upload(segs);
      h.tw16_nseg = static_cast<int>(segs.size());
      h.tw16_nmax = nmax;
    }
    k_cast_segs<<<dim3(static_cast<unsigned>(std::min<size_t>((h.tw16_nmax + 255) / 256, 64)), h.tw16_nseg), 256, 0,
                  h.stream>>>(h.tw16_segs);
  }
  if (h.head_wt) head_wsplit(h);
  check_launch("weight repack");
  h.w16.clear();  // generic-path bf16 copies are rebuilt on next use
}

static void upload_batch(Handle& h, const SortBatch* b, bool on_device) {
  const SortConfig& c = h.cfg;
  const int B = b->batch;
  if (B < 1 || B > h.Bmax) throw ConfigError("batch size must be in [1, max_batch]");
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  const size_t nh = static_cast<size_t>(B) * c.n_hist;
  auto cp = [&](void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    if (!src) throw ConfigError("batch array is null");
    CK(cudaMemcpyAsync(dst, src, bytes, kind, h.stream));
  };
  cp(h.in_item, b->hist_item, nh * 4);
  cp(h.in_action, b->hist_action, nh * 4);
  cp(h.in_scene, b->hist_scene, nh * 4);
  cp(h.in_ts, b->hist_ts, nh * 8);
  cp(h.in_req, b->req_ts, static_cast<size_t>(B) * 8);
  cp(h.in_prof, b->profile, static_cast<size_t>(B) * c.n_profile_fields * 4);
  cp(h.in_cand, b->cand_item, static_cast<size_t>(B) * c.n_cand * 4);
}

static void begin_timing(Handle& h) {
  for (auto e : h.events) cudaEventDestroy(e);
  h.events.clear();
  h.stage_names.clear();
  h.launches = 0;
  stage_mark(h, "start");
}

static void forward_device(Handle& h, int B) {
  if (h.generic) {
    if (h.training) throw ConfigError("training step: model_dim > 256 is not supported in this build");
    forward_generic(h, B);
    return;
  }
  // h.err is NOT cleared here: several sort_forward_async calls may be queued before one
  // sort_sync, and each batch's device checks (OOV ids, MoE non-finite router scores) must
  // survive until that sync reads them. collect_status() clears the word after reading it.
  run_tokenizer(h, B);
  stage_mark(h, "tokenizer");
  for (int l = 0; l < h.cfg.layers; ++l) run_layer(h, l, B);
  const LayerDev& last = h.layers.back();
  if (h.cfg.pretrain) {  // tied next-item head, see pretrain.cuh
    const int T = B * h.L0;
    const size_t psmem = (static_cast<size_t>(h.d) * kPreK + 8 * h.d) * sizeof(float);
    ensure_smem(k_pretrain_proj, psmem);
    const __nv_bfloat16* items = h.item_ext ? h.item_ext : h.item;
    const int V = h.item_ext ? static_cast<int>(h.item_ext_rows) : h.cfg.n_items;
    if (h.pre_proj_tc && h.d % 32 == 0) {  // projection + target logit on the streaming tcgen05 GEMM
      if (!h.pre_wt) h.pre_wt = h.dalloc<__nv_bfloat16>(static_cast<size_t>(kPreK) * h.d);
      k_pretrain_wfold<<<ew_grid(static_cast<size_t>(kPreK) * h.d), 256, 0, h.stream>>>(h.pre_proj, h.head_gain, h.d,
                                                                                         h.pre_wt);
      gemm_stream(h, h.X[last.q_buf], h.d, T, h.d, h.pre_wt, h.d, kPreK,
                  GsPretrainHead{h.SS[last.q_buf], 1.f / static_cast<float>(h.d), h.pre_hp, items, h.in_item,
                                 h.pre_tgt, h.L0, h.L0 - 1});
    } else {
      k_pretrain_proj<<<std::max(1, std::min((T + 7) / 8, 8 * h.num_sms)), 256, psmem, h.stream>>>(
          h.X[last.q_buf], T, h.L0, h.d, h.head_gain, h.pre_proj, items, h.in_item, h.pre_hp, h.pre_tgt);
    }
    if (h.ce_tc) {  // tcgen05 logits + online log-sum-exp, partials per vocabulary chunk
      const int n_chunks = (V + kCeChunk - 1) / kCeChunk;
      const size_t need = static_cast<size_t>(h.Bmax) * h.L0 * n_chunks * 2;
      if (need > h.ce_part_cap) {
        h.ce_part = h.dalloc<float2>(need);
        h.ce_part_cap = need;
      }
      CeTcArgs ca;
      ca.T = T;
      ca.V = V;
      ca.n_chunks = n_chunks;
      ca.n_items = ((T + 127) / 128) * n_chunks;
      ca.part = h.ce_part;
      const CUtensorMap tmH = make_tmap_2d(h.pre_hp, static_cast<uint64_t>(T), kPreK, kPreK, 128, kPreK, kPreK * 2);
      const CUtensorMap tmE = make_tmap_2d(items, static_cast<uint64_t>(V), kPreK, kPreK, 128, kPreK, kPreK * 2);
      ensure_smem(k_ce_tc, CeTcSmem::bytes);
      k_ce_tc<<<std::min(ca.n_items, 2 * h.num_sms), kAttnThreads, CeTcSmem::bytes, h.stream>>>(tmH, tmE, ca);
      k_ce_combine<<<(T + 255) / 256, 256, 0, h.stream>>>(h.ce_part, T, h.L0, 2 * n_chunks, h.pre_lse);
      h.launches += 1;
    } else {
      k_ce_tied<<<(T + kCeRows - 1) / kCeRows, kCeThreads, 0, h.stream>>>(h.pre_hp, T, h.L0, items, V, h.pre_lse);
    }
    check_launch("pretrain head");
    h.launches += 2;
    stage_mark(h, "head");
    return;
  }
  const int total = B * h.cfg.n_cand;
  if (h.head_tc && h.head_wt) {
    const LayerDev& lst = last;
    const int N = h.cfg.n_cand, Rq = lst.Rq;
    GsHead epi{nullptr, 0, 0, 1.f / static_cast<float>(h.d), h.head_b1, h.head_w2, h.head_b2, h.head_zp,
               h.probs, h.logits, total, h.dh};
    const __nv_bfloat16* wt = h.head_wt;
    const int K = 3 * h.d, a_kwrap = h.d / 64;
    ensure_smem(k_gemm_stream<GsHead, false, false, __nv_bfloat16>, kGsSmem);
    const CUtensorMap& tb = gs_map(h, wt, h.dh, K, K, kGsBN, 64, false);
    const int grid = std::min((total + kGsBM - 1) / kGsBM, h.num_sms);
    if (N <= kGsBM && kGsBM % N == 0) {  // candidate rows read in place: 3D view {d, N, B}
      const uint64_t dims[3] = {static_cast<uint64_t>(h.d), static_cast<uint64_t>(N), static_cast<uint64_t>(B)};
      const uint64_t strides[2] = {static_cast<uint64_t>(h.d) * 2, static_cast<uint64_t>(Rq) * h.d * 2};
      const uint32_t box[3] = {64, static_cast<uint32_t>(N), static_cast<uint32_t>(kGsBM / N)};
      const CUtensorMap ta =
          make_tmap_bf16(h.X[lst.q_buf] + static_cast<size_t>(Rq - N) * h.d, 3, dims, strides, box, 128);
      epi.ss = h.SS[lst.q_buf];
      epi.R = Rq;
      epi.N = N;
      k_gemm_stream<GsHead, false, false, __nv_bfloat16><<<grid, kGsThreads, kGsSmem, h.stream>>>(
          ta, tb, total, h.dh, K, 1, epi, a_kwrap, N);
    } else {  // gathered copy of the candidate rows
      k_gather_cand<<<std::min((total * (h.d / 8) + 255) / 256, 148 * 16), 256, 0, h.stream>>>(
          h.X[lst.q_buf], h.SS[lst.q_buf], Rq, N, total, h.d, h.head_xc, h.head_ssc);
      ++h.launches;
      epi.ss = h.head_ssc;
      const CUtensorMap& ta = gs_map(h, h.head_xc, total, h.d, h.d, kGsBM, 64, false);
      k_gemm_stream<GsHead, false, false, __nv_bfloat16><<<grid, kGsThreads, kGsSmem, h.stream>>>(
          ta, tb, total, h.dh, K, 1, epi, a_kwrap, 0);
    }
    check_launch("head");
    ++h.launches;
    stage_mark(h, "head");
    return;
  }
  const size_t hsmem = (static_cast<size_t>(kHeadPitch) * h.d + 2 * kHeadKSlice * h.dh) * sizeof(float);
  const int hgrid = (total + kHeadRows - 1) / kHeadRows;
  const LayerDev& lst = last;
#define SORT_HEAD(CPT)                                                                          \
  case CPT: {                                                                                   \
    ensure_smem(k_head<CPT>, hsmem);                                                            \
    k_head<CPT><<<hgrid, kHeadThreads, hsmem, h.stream>>>(                                      \
        h.X[lst.q_buf], h.SS[lst.q_buf], lst.Rq, h.cfg.n_cand, total, h.d, h.head_gain,         \
        h.head_w1, h.head_b1, h.head_w2, h.head_b2, h.probs, h.logits);                         \
    break;                                                                                      \
  }
  switch (h.dh / 32) {
    SORT_HEAD(1)
    SORT_HEAD(2)
    SORT_HEAD(4)
    SORT_HEAD(8)
    default: throw ConfigError("unsupported head_hidden (must be 32, 64, 128 or 256)");
  }
#undef SORT_HEAD
  check_launch("head");
  ++h.launches;
  stage_mark(h, "head");
}

// The inference forward, replayed from a CUDA graph when possible. The first call for a key
// runs eagerly (kernel attributes, plan checks) and then captures the same enqueue sequence.
static void forward_run(Handle& h, int B) {
  // (a batch-local item table changes with every batch: no graph for those calls)
  if (!h.use_graphs || h.timing || h.training || h.generic || h.stream == nullptr || h.item_ext) {
    forward_device(h, B);
    return;
  }
  const auto key = std::make_tuple(B, static_cast<const void*>(h.in_item), static_cast<const void*>(nullptr),
                                   static_cast<int64_t>(0));
  auto it = h.graphs.find(key);
  if (it != h.graphs.end()) {
    CK(cudaGraphLaunch(it->second.exec, h.stream));
    h.launches = it->second.launches;
    return;
  }
  forward_device(h, B);
  const int launches = h.launches;
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(h.stream, cudaStreamCaptureModeRelaxed));
  try {
    forward_device(h, B);
  } catch (...) {
    cudaStreamEndCapture(h.stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  CK(cudaStreamEndCapture(h.stream, &g));
  Handle::GraphEntry e;
  const cudaError_t ie = cudaGraphInstantiate(&e.exec, g, 0);
  cudaGraphDestroy(g);
  if (ie != cudaSuccess) throw RuntimeFailure(std::string("cudaGraphInstantiate failed: ") + cudaGetErrorString(ie));
  e.launches = launches;
  h.launches = launches;
  h.graphs[key] = e;
}

static void collect_status(Handle& h) {
  int32_t err[4];
  CK(cudaMemcpyAsync(err, h.err, sizeof(err), cudaMemcpyDeviceToHost, h.stream));
  CK(cudaStreamSynchronize(h.stream));
  // the sync point: everything enqueued so far has been checked, start a fresh error word
  if (err[0] | err[1] | err[2] | err[3]) CK(cudaMemsetAsync(h.err, 0, 4 * sizeof(int32_t), h.stream));
  if (h.timing && h.events.size() > 1) {
    h.stage_ms.clear();
    for (size_t i = 1; i < h.events.size(); ++i) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, h.events[i - 1], h.events[i]));
      h.stage_ms.push_back(ms);
    }
  }
  if (err[0] & kErrOOV) throw ConfigError("tokenizer: id outside vocabulary (device check)");
  if (err[0] & kErrMoeNonFinite)
    throw RuntimeFailure("moe: non-finite router score at token row " + std::to_string(err[1] - 1) +
                         " (device check)");
}

static Handle* H_(SortHandle p) {
  if (!p) throw ConfigError("null handle");
  Handle* h = reinterpret_cast<Handle*>(p);
  CK(cudaSetDevice(h->device));
  return h;
}

static Handle* ready(SortHandle p) {
  Handle* h = H_(p);
  if (!h->finalized) throw ConfigError("parameters not finalized (call sort_finalize_params)");
  return h;
}

template <class F>
static int api(F&& f) {
  try {
    f();
    return SORT_OK;
  } catch (const ConfigError& e) {
    g_last_error = e.what();
    return SORT_CONFIG_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SORT_RUNTIME_FAILURE;
  }
}

// ------------------------------------------------------------------ op-level helpers
static std::vector<float> bf16_to_f32(const std::vector<__nv_bfloat16>& v) {
  std::vector<float> o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = __bfloat162float(v[i]);
  return o;
}

}  // namespace sortk

using namespace sortk;

#include "exchange.cuh"

// ======================================================================= C ABI
extern "C" {

const char* sort_last_error(void) { return g_last_error.c_str(); }
int sort_version(void) { return 1; }

int sort_create(const SortConfig* cfg, int device, SortHandle* out) {
  return api([&] {
    if (!cfg || !out) throw ConfigError("null argument");
    auto h = std::make_unique<Handle>();
    h->cfg = *cfg;
    h->device = device;
    h->plan = make_plan(*cfg);
    h->d = cfg->model_dim;
    h->H = cfg->heads;
    h->dk = cfg->model_dim / cfg->heads;
    h->m = cfg->ffn_dim;
    h->dh = cfg->head_hidden > 0 ? cfg->head_hidden : cfg->model_dim;
    h->generic = cfg->model_dim > 256;
    h->moe = cfg->moe_experts > 0;
    h->moe_E = cfg->moe_experts;
    h->moe_k = cfg->moe_topk;
    h->moe_s = cfg->moe_shared;
    h->moe_m = cfg->moe_ffn_dim;
    if (!h->generic && h->dh != 32 && h->dh != 64 && h->dh != 128 && h->dh != 256)
      throw ConfigError("unsupported head_hidden (must be 32, 64, 128 or 256)");
    h->L0 = h->plan.L0;
    h->Bmax = cfg->max_batch;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw RuntimeFailure("no CUDA device available (libsort_b200 has no CPU path)");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw RuntimeFailure("libsort_b200 requires an sm_100 (Blackwell) GPU");
    h->num_sms = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
    *out = reinterpret_cast<SortHandle>(h.release());
  });
}

int sort_destroy(SortHandle p) {
  return api([&] { delete reinterpret_cast<Handle*>(p); });
}

int sort_set_stream(SortHandle p, void* stream) {
  return api([&] {
    Handle* h = H_(p);
    if (stream) {
      if (h->own_stream) CK(cudaStreamDestroy(h->stream));
      h->stream = static_cast<cudaStream_t>(stream);
      h->own_stream = false;
    }
  });
}

int sort_load_param(SortHandle p, const char* name, const float* data, int64_t rows, int64_t cols) {
  return api([&] {
    Handle* h = reinterpret_cast<Handle*>(p);
    if (!h || !name || !data) throw ConfigError("null argument");
    if (h->finalized) throw ConfigError("parameters already finalized");
    HostParam hp;
    hp.rows = rows;
    hp.cols = cols;
    hp.v.assign(data, data + rows * cols);
    h->host[name] = std::move(hp);
  });
}

int sort_finalize_params(SortHandle p) {
  return api([&] {
    Handle* h = H_(p);
    if (h->finalized) return;
    finalize(*h);
  });
}

int sort_forward(SortHandle p, const SortBatch* batch, int inputs_on_device, float* scores,
                 int scores_on_device) {
  return api([&] {
    Handle* h = ready(p);
    if (!batch || !scores) throw ConfigError("null argument");
    if (h->cfg.pretrain) throw ConfigError("pre-training model: use sort_pretrain_forward");
    begin_timing(*h);
    upload_batch(*h, batch, inputs_on_device != 0);
    forward_run(*h, batch->batch);
    const size_t bytes = static_cast<size_t>(batch->batch) * h->cfg.n_cand * 3 * sizeof(float);
    CK(cudaMemcpyAsync(scores, h->probs, bytes,
                       scores_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream));
    if (!(inputs_on_device && scores_on_device)) collect_status(*h);
  });
}

int sort_forward_async(SortHandle p, const SortBatch* batch, float* scores) {
  return api([&] {
    Handle* h = ready(p);
    if (!batch || !scores) throw ConfigError("null argument");
    if (h->cfg.pretrain) throw ConfigError("pre-training model: use sort_pretrain_forward");
    const SortConfig& c = h->cfg;
    const int B = batch->batch;
    if (B < 1 || B > h->Bmax) throw ConfigError("batch size must be in [1, max_batch]");
    if (!h->copy_stream) {
      CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        CK(cudaEventCreateWithFlags(&h->slot_copied[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->slot_free[i], cudaEventDisableTiming));
      }
      const size_t BH_ = static_cast<size_t>(h->Bmax) * std::max(c.n_hist, 1);
      Handle::InSlot& s1 = h->in_slot[1];
      s1.item = h->dalloc<int32_t>(BH_);
      s1.action = h->dalloc<int32_t>(BH_);
      s1.scene = h->dalloc<int32_t>(BH_);
      s1.ts = h->dalloc<int64_t>(BH_);
      s1.req = h->dalloc<int64_t>(h->Bmax);
      s1.prof = h->dalloc<int32_t>(static_cast<size_t>(h->Bmax) * std::max(c.n_profile_fields, 1));
      s1.cand = h->dalloc<int32_t>(static_cast<size_t>(h->Bmax) * c.n_cand);
    }
    const int k = static_cast<int>(h->async_steps & 1);
    Handle::InSlot& sl = h->in_slot[k];
    // the slot's previous reader (the forward two steps back) must be done before overwriting
    if (h->async_steps >= 2) CK(cudaStreamWaitEvent(h->copy_stream, h->slot_free[k], 0));
    const size_t nh = static_cast<size_t>(B) * c.n_hist;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (bytes == 0) return;
      if (!src) throw ConfigError("batch array is null");
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->copy_stream));
    };
    cp(sl.item, batch->hist_item, nh * 4);
    cp(sl.action, batch->hist_action, nh * 4);
    cp(sl.scene, batch->hist_scene, nh * 4);
    cp(sl.ts, batch->hist_ts, nh * 8);
    cp(sl.req, batch->req_ts, static_cast<size_t>(B) * 8);
    cp(sl.prof, batch->profile, static_cast<size_t>(B) * c.n_profile_fields * 4);
    cp(sl.cand, batch->cand_item, static_cast<size_t>(B) * c.n_cand * 4);
    CK(cudaEventRecord(h->slot_copied[k], h->copy_stream));
    CK(cudaStreamWaitEvent(h->stream, h->slot_copied[k], 0));
    h->in_item = sl.item;
    h->in_action = sl.action;
    h->in_scene = sl.scene;
    h->in_ts = sl.ts;
    h->in_req = sl.req;
    h->in_prof = sl.prof;
    h->in_cand = sl.cand;
    begin_timing(*h);
    forward_run(*h, B);
    CK(cudaEventRecord(h->slot_free[k], h->stream));
    CK(cudaMemcpyAsync(scores, h->probs, static_cast<size_t>(B) * c.n_cand * 3 * sizeof(float),
                       cudaMemcpyDeviceToHost, h->stream));
    ++h->async_steps;
  });
}

int sort_sync(SortHandle p) {
  return api([&] { collect_status(*ready(p)); });
}

int sort_forward_logits(SortHandle p, const SortBatch* batch, float* probs, float* logits) {
  return api([&] {
    Handle* h = ready(p);
    if (!batch || !probs) throw ConfigError("null argument");
    begin_timing(*h);
    upload_batch(*h, batch, false);
    forward_device(*h, batch->batch);
    const size_t bytes = static_cast<size_t>(batch->batch) * h->cfg.n_cand * 3 * sizeof(float);
    CK(cudaMemcpyAsync(probs, h->probs, bytes, cudaMemcpyDeviceToHost, h->stream));
    if (logits) CK(cudaMemcpyAsync(logits, h->logits, bytes, cudaMemcpyDeviceToHost, h->stream));
    collect_status(*h);
  });
}

int sort_tokenize(SortHandle p, const SortBatch* batch, float* tokens, int32_t* hist_time,
                  int32_t* position_ids, int32_t* roles, int32_t* candidate_index) {
  return api([&] {
    Handle* h = ready(p);
    if (!batch) throw ConfigError("null argument");
    begin_timing(*h);
    upload_batch(*h, batch, false);
    const int B = batch->batch;
    std::vector<__nv_bfloat16> xb(static_cast<size_t>(B) * h->L0 * h->d);
    if (h->generic) {
      throw ConfigError("sort_tokenize: model_dim > 256 tokens are only produced inside sort_forward");
    }
    run_tokenizer(*h, batch->batch);
    CK(cudaMemcpyAsync(xb.data(), h->X[0], xb.size() * 2, cudaMemcpyDeviceToHost, h->stream));
    if (hist_time && h->cfg.n_hist)
      CK(cudaMemcpyAsync(hist_time, h->hist_time, static_cast<size_t>(B) * h->cfg.n_hist * 4,
                         cudaMemcpyDeviceToHost, h->stream));
    collect_status(*h);
    if (tokens) {
      std::vector<float> f = bf16_to_f32(xb);
      std::memcpy(tokens, f.data(), f.size() * sizeof(float));
    }
    const Plan& P = h->plan;
    if (position_ids) std::copy(P.pos0.begin(), P.pos0.end(), position_ids);
    if (roles) std::copy(P.roles0.begin(), P.roles0.end(), roles);
    if (candidate_index) std::copy(P.cand_index0.begin(), P.cand_index0.end(), candidate_index);
  });
}

int sort_layer_plan(SortHandle p, int layer, int32_t* l_q, int32_t* l_kv, int32_t* query_rows,
                    int32_t* lo, int32_t* hi, int32_t* self_idx, int64_t* visible,
                    int64_t* tiles_issued, int64_t* tiles_total) {
  return api([&] {
    Handle* h = reinterpret_cast<Handle*>(p);
    if (!h) throw ConfigError("null handle");
    if (layer < 0 || layer >= h->cfg.layers) throw ConfigError("layer out of range");
    const LayerPlan& lp = h->plan.layers[layer];
    if (l_q) *l_q = lp.l_q;
    if (l_kv) *l_kv = lp.l_kv;
    if (query_rows) std::copy(lp.query_rows.begin(), lp.query_rows.end(), query_rows);
    if (lo) std::copy(lp.lo.begin(), lp.lo.end(), lo);
    if (hi) std::copy(lp.hi.begin(), lp.hi.end(), hi);
    if (self_idx) std::copy(lp.self_idx.begin(), lp.self_idx.end(), self_idx);
    if (visible) *visible = lp.visible;
    if (tiles_issued) *tiles_issued = lp.tiles_issued;
    if (tiles_total) *tiles_total = lp.tiles_total;
  });
}

int sort_attention_forward(SortHandle p, int layer, int32_t batch, const float* x, float* out) {
  return api([&] {
    Handle* h = ready(p);
    if (layer < 0 || layer >= h->cfg.layers) throw ConfigError("layer out of range");
    if (batch < 1 || batch > h->Bmax) throw ConfigError("batch out of range");
    const LayerDev& L = h->layers[layer];
    const size_t n_in = static_cast<size_t>(batch) * L.Rkv * h->d;
    std::vector<__nv_bfloat16> xb(n_in);
    std::vector<float4> ss(static_cast<size_t>(batch) * L.Rkv, make_float4(0.f, 0.f, 0.f, 0.f));
    for (size_t i = 0; i < n_in; ++i) {
      xb[i] = f2bf(x[i]);
      const float f = __bfloat162float(xb[i]);
      ss[i / h->d].x += f * f;
    }
    begin_timing(*h);
    CK(cudaMemcpyAsync(h->X[L.in_buf], xb.data(), n_in * 2, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->SS[L.in_buf], ss.data(), ss.size() * sizeof(float4), cudaMemcpyHostToDevice, h->stream));
    run_layer(*h, layer, batch, /*attn_only=*/true);
    const size_t n_out = static_cast<size_t>(batch) * L.Rq * h->d;
    std::vector<__nv_bfloat16> ob(n_out);
    CK(cudaMemcpyAsync(ob.data(), h->Qb, n_out * 2, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    for (size_t i = 0; i < n_out; ++i) out[i] = __bfloat162float(ob[i]);
  });
}

int sort_op_gemm(int32_t M, int32_t N, int32_t K, int32_t trans_a, int32_t trans_b, int32_t tf32, const float* A,
                 const float* B, float* C) {
  return api([&] {
    if (M < 0 || N < 0 || K < 1 || (M && (!A || !C)) || (N && !B)) throw ConfigError("op gemm: bad arguments");
    if (M == 0 || N == 0) return;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    Handle h;  // a bare context: default stream, no plan
    h.device = dev;
    CK(cudaDeviceGetAttribute(&h.num_sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t na = static_cast<size_t>(M) * K, nb = static_cast<size_t>(K) * N;
    const int lda = trans_a ? M : K, ldb = trans_b ? K : N;
    float* dc = h.dalloc<float>(static_cast<size_t>(M) * N);
    if (tf32) {
      std::vector<float> a(A, A + na), b(B, B + nb);
      gemm_rm(h, trans_a != 0, trans_b != 0, M, N, K, h.upload(a), lda, h.upload(b), ldb, dc, N);
    } else {
      if (lda % 8 || ldb % 8 || N % 32) throw ConfigError("op gemm (bf16): row pitches must be multiples of 8, N of 32");
      std::vector<__nv_bfloat16> a(na), b(nb);
      for (size_t i = 0; i < na; ++i) a[i] = f2bf(A[i]);
      for (size_t i = 0; i < nb; ++i) b[i] = f2bf(B[i]);
      gemm_rm16(h, trans_a != 0, trans_b != 0, M, N, K, h.upload(a), lda, h.upload(b), ldb, dc, N, false);
    }
    CK(cudaMemcpy(C, dc, sizeof(float) * M * N, cudaMemcpyDeviceToHost));
  });
}

int sort_block_attention(int32_t nh, int32_t l_q, int32_t l_kv, int32_t dk, const float* q,
                         const float* k, const float* v, const int32_t* lo, const int32_t* hi,
                         const int32_t* self_idx, float* out, int64_t* skipped, int64_t* total) {
  return api([&] {
    if (nh < 1 || l_q < 1 || l_kv < 1) throw ConfigError("block_attention: bad shape");
    if (dk != 16 && dk != 32 && dk != 64) throw ConfigError("block_attention: dk must be 16, 32 or 64");
    int dev = 0;
    CK(cudaGetDevice(&dev));
    Handle h;
    h.device = dev;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10) throw RuntimeFailure("requires an sm_100 GPU");
    h.num_sms = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&h.stream, cudaStreamNonBlocking));
    h.own_stream = true;
    h.d = dk;  // one head per "request": out rows are [nh * l_q, dk]
    h.H = 1;
    h.dk = dk;
    LayerPlan lp;
    lp.l_q = l_q;
    lp.l_kv = l_kv;
    lp.lo.assign(lo, lo + l_q);
    lp.hi.assign(hi, hi + l_q);
    lp.self_idx.assign(self_idx, self_idx + l_q);
    build_tiles(lp);
    LayerDev L;
    L.Rq = l_q;
    L.Rkv = l_kv;
    std::vector<int4> meta(static_cast<size_t>(lp.n_qtiles) * 128, make_int4(0, -1, -1, 0));
    for (int r = 0; r < l_q; ++r) meta[r] = make_int4(lo[r], hi[r], self_idx[r], 0);
    L.rowmeta = h.upload(meta);
    L.tile_off = h.upload(lp.tile_off);
    L.tile_code = h.upload(lp.tile_code.empty() ? std::vector<int32_t>{0, 0} : lp.tile_code);
    L.qtile_order = h.upload(lp.qtile_order);
    auto up = [&](const float* src, size_t n) {
      std::vector<__nv_bfloat16> b(n);
      for (size_t i = 0; i < n; ++i) b[i] = f2bf(src[i]);
      return h.upload(b);
    };
    h.Qb = up(q, static_cast<size_t>(nh) * l_q * dk);
    h.Kb = up(k, static_cast<size_t>(nh) * l_kv * dk);
    h.Vb = up(v, static_cast<size_t>(nh) * l_kv * dk);
    h.Gb = h.upload(std::vector<__nv_bfloat16>(static_cast<size_t>(nh) * l_q * dk, f2bf(1.f)));
    h.Hg = h.dalloc<__nv_bfloat16>(static_cast<size_t>(nh) * l_q * dk);
    uint64_t dq[3] = {static_cast<uint64_t>(dk), static_cast<uint64_t>(l_q), static_cast<uint64_t>(nh)};
    uint64_t sq[2] = {static_cast<uint64_t>(dk) * 2, static_cast<uint64_t>(l_q) * dk * 2};
    uint32_t bq[3] = {static_cast<uint32_t>(dk), 128, 1};
    L.tmQ = make_tmap_bf16(h.Qb, 3, dq, sq, bq, dk * 2);
    uint64_t dkd[3] = {static_cast<uint64_t>(dk), static_cast<uint64_t>(l_kv), static_cast<uint64_t>(nh)};
    uint64_t skd[2] = {static_cast<uint64_t>(dk) * 2, static_cast<uint64_t>(l_kv) * dk * 2};
    L.tmK = make_tmap_bf16(h.Kb, 3, dkd, skd, bq, dk * 2);
    L.tmV = make_tmap_bf16(h.Vb, 3, dkd, skd, bq, dk * 2);
    launch_attention(h, L, lp, nh);
    std::vector<__nv_bfloat16> ob(static_cast<size_t>(nh) * l_q * dk);
    CK(cudaMemcpyAsync(ob.data(), h.Hg, ob.size() * 2, cudaMemcpyDeviceToHost, h.stream));
    CK(cudaStreamSynchronize(h.stream));
    for (size_t i = 0; i < ob.size(); ++i) out[i] = __bfloat162float(ob[i]);
    if (skipped) *skipped = lp.tiles_total - lp.tiles_issued;
    if (total) *total = lp.tiles_total;
  });
}

int sort_time_bucket(int64_t delta_seconds, int32_t n_buckets) {
  return time_bucket_int(delta_seconds, n_buckets);
}

int sort_geometric_schedule(int32_t prefix_len, int32_t depth, int32_t target, int32_t* keep) {
  return api([&] {
    std::vector<int32_t> k = geometric_schedule(prefix_len, depth, target);
    std::copy(k.begin(), k.end(), keep);
  });
}

int sort_retained_rows(const int32_t* roles, int32_t n, int32_t keep, int32_t keep_specials,
                       int32_t* rows, int32_t* n_rows) {
  return api([&] {
    std::vector<int32_t> r(roles, roles + n);
    std::vector<int32_t> o = retained_rows(r, keep, keep_specials != 0);
    std::copy(o.begin(), o.end(), rows);
    *n_rows = static_cast<int32_t>(o.size());
  });
}

int sort_mask_intervals(int32_t l_q, int32_t l_kv, int32_t local_window, int32_t full_suffix,
                        const int32_t* roles, const int32_t* position_ids, const int32_t* query_rows,
                        int32_t* lo, int32_t* hi, int32_t* self_idx) {
  return api([&] {
    mask_intervals(l_q, l_kv, local_window, full_suffix, roles, position_ids, query_rows, lo, hi, self_idx);
  });
}

int sort_kernel_count(SortHandle p, int32_t* launches) {
  return api([&] {
    Handle* h = reinterpret_cast<Handle*>(p);
    if (!h || !launches) throw ConfigError("null argument");
    *launches = h->launches;
  });
}

int sort_enable_stage_timing(SortHandle p, int enable) {
  return api([&] {
    Handle* h = reinterpret_cast<Handle*>(p);
    if (!h) throw ConfigError("null handle");
    h->timing = enable != 0;
  });
}

int sort_train_step(SortHandle p, const SortBatch* batch, const float* dlogits, float* logits) {
  return api([&] {
    Handle* h = ready(p);
    if (!batch || !dlogits) throw ConfigError("null argument");
    const int B = batch->batch;
    begin_timing(*h);
    upload_batch(*h, batch, false);
    ensure_train_buffers(*h, B);
    h->training = true;
    try {
      forward_device(*h, B);
    } catch (...) {
      h->training = false;
      throw;
    }
    h->training = false;
    const size_t nz = static_cast<size_t>(B) * h->cfg.n_cand * 3;
    float*& dzb = h->dz_dev;
    if (!dzb) dzb = h->dalloc<float>(static_cast<size_t>(h->Bmax) * h->cfg.n_cand * 3 + 1);  // + loss slot
    CK(cudaMemcpyAsync(dzb, dlogits, nz * 4, cudaMemcpyHostToDevice, h->stream));
    CK(cublasSetStream(h->cublas, h->stream) == CUBLAS_STATUS_SUCCESS ? cudaSuccess : cudaErrorUnknown);
    backward_device(*h, B, dzb);
    if (logits) CK(cudaMemcpyAsync(logits, h->logits, nz * 4, cudaMemcpyDeviceToHost, h->stream));
    collect_status(*h);
  });
}

int sort_pretrain_train_step(SortHandle p, const SortBatch* batch, float* loss) {
  return api([&] {
    Handle* h = ready(p);
    if (!batch) throw ConfigError("null argument");
    if (!h->cfg.pretrain) throw ConfigError("sort_pretrain_train_step needs a pre-training model (pretrain = 1)");
    if (h->cfg.n_hist < 2) throw ConfigError("pretrain: sequences shorter than 2 clicks are skipped");
    const int B = batch->batch;
    begin_timing(*h);
    upload_batch(*h, batch, false);
    ensure_train_buffers(*h, B);
    h->training = true;
    try {
      forward_device(*h, B);
    } catch (...) {
      h->training = false;
      throw;
    }
    h->training = false;
    k_ce_loss<<<1, 1024, 0, h->stream>>>(h->pre_lse, h->pre_tgt, B * h->cfg.n_hist, h->pre_loss);
    check_launch("pretrain loss");
    backward_device(*h, B, nullptr);
    float hl = 0.f;
    CK(cudaMemcpyAsync(&hl, h->pre_loss, 4, cudaMemcpyDeviceToHost, h->stream));
    collect_status(*h);
    if (loss) *loss = hl;
  });
}

int sort_train_step_bce(SortHandle p, const SortBatch* batch, const float* labels, const float* obj_weights,
                        float* loss) {
  return api([&] {
    Handle* h = ready(p);
    if (!batch || !labels) throw ConfigError("null argument");
    if (h->generic) throw ConfigError("training step: model_dim > 256 is not supported in this build");
    const int B = batch->batch;
    begin_timing(*h);
    upload_batch(*h, batch, false);
    ensure_train_buffers(*h, B);
    h->training = true;
    try {
      forward_device(*h, B);
    } catch (...) {
      h->training = false;
      throw;
    }
    h->training = false;
    const int n = B * h->cfg.n_cand;
    float*& dzb = h->dz_dev;
    if (!dzb) dzb = h->dalloc<float>(static_cast<size_t>(h->Bmax) * h->cfg.n_cand * 3 + 1);
    float* lab = h->tw[15];  // scratch until the attention backward
    CK(cudaMemcpyAsync(lab, labels, static_cast<size_t>(n) * 3 * 4, cudaMemcpyHostToDevice, h->stream));
    const float w0 = obj_weights ? obj_weights[0] : 1.f, w1 = obj_weights ? obj_weights[1] : 0.5f,
                w2 = obj_weights ? obj_weights[2] : 0.5f;  // SPEC.md:416 defaults
    float* dloss = dzb + static_cast<size_t>(h->Bmax) * h->cfg.n_cand * 3;
    k_bce<<<1, 1024, 0, h->stream>>>(h->logits, lab, n, w0, w1, w2, dzb, dloss);
    check_launch("bce");
    float hl = 0.f;
    CK(cudaMemcpyAsync(&hl, dloss, 4, cudaMemcpyDeviceToHost, h->stream));
    CK(cublasSetStream(h->cublas, h->stream) == CUBLAS_STATUS_SUCCESS ? cudaSuccess : cudaErrorUnknown);
    backward_device(*h, B, dzb);
    collect_status(*h);
    if (loss) *loss = hl;
  });
}

int sort_adamw_step(SortHandle p, float lr, float beta1, float beta2, float eps, float weight_decay) {
  return api([&] {
    Handle* h = ready(p);
    if (!h->grads) throw ConfigError("no gradients yet (call sort_train_step)");
    if (h->generic) throw ConfigError("training step: model_dim > 256 is not supported in this build");
    h->drop_graphs();  // weights and QKNorm logit bounds (kernel arguments) change
    if (!h->adam_m) {
      h->adam_m = h->dalloc<float>(h->grad_count);
      h->adam_v = h->dalloc<float>(h->grad_count);
      CK(cudaMemsetAsync(h->adam_m, 0, h->grad_count * 4, h->stream));
      CK(cudaMemsetAsync(h->adam_v, 0, h->grad_count * 4, h->stream));
    }
    ++h->adam_t;
    const float bc1 = 1.f - std::pow(beta1, static_cast<float>(h->adam_t));
    const float bc2 = 1.f - std::pow(beta2, static_cast<float>(h->adam_t));
    if (!h->adam_bad) h->adam_bad = h->dalloc<unsigned long long>(1);
    unsigned long long* bad = h->adam_bad;
    const unsigned long long none = ~0ull;
    CK(cudaMemcpyAsync(bad, &none, 8, cudaMemcpyHostToDevice, h->stream));
    // one launch per run of trainable tensors (frozen ones are skipped: no update, no decay)
    std::vector<std::pair<size_t, size_t>> runs;  // [begin, end) in the flat buffer
    {
      std::vector<std::pair<size_t, size_t>> fz;
      for (const std::string& name : h->frozen) {
        auto it = h->grad_index.find(name);
        if (it != h->grad_index.end())
          fz.emplace_back(it->second.first,
                          it->second.first + static_cast<size_t>(it->second.second.first) * it->second.second.second);
      }
      std::sort(fz.begin(), fz.end());
      size_t at = 0;
      for (const auto& f : fz) {
        if (f.first > at) runs.emplace_back(at, f.first);
        at = std::max(at, f.second);
      }
      if (at < h->grad_count) runs.emplace_back(at, h->grad_count);
    }
    auto adam = [&](float* p, float* g, float* m, float* v, size_t n, size_t base) {
      k_adamw<<<static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 32)), 256, 0, h->stream>>>(
          p, g, m, v, n, lr, beta1, beta2, eps, weight_decay, bc1, bc2, bad, base);
    };
    for (const auto& r : runs)
      adam(h->master + r.first, h->grads + r.first, h->adam_m + r.first, h->adam_v + r.first, r.second - r.first,
           r.first);
    const size_t n_item = static_cast<size_t>(h->cfg.n_items) * h->cfg.item_dim;
    if (!h->frozen.count("tok.item_table")) {
      adam(h->item_master, h->item_grad, h->item_m, h->item_v, n_item, h->grad_count);
      k_cast_bf16<<<static_cast<int>(std::min<size_t>((n_item + 255) / 256, 148 * 32)), 256, 0, h->stream>>>(
          h->item_master, n_item, h->item);
    }
    check_launch("adamw");
    unsigned long long hb = 0;
    CK(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (hb != none) {
      const size_t idx = static_cast<size_t>(hb - 1);
      std::string name = idx >= h->grad_count ? "tok.item_table" : "?";
      for (auto& kv : h->grad_index)
        if (idx >= kv.second.first &&
            idx < kv.second.first + static_cast<size_t>(kv.second.second.first) * kv.second.second.second)
          name = kv.first;
      throw RuntimeFailure("adamw_step: non-finite gradient in parameter " + name);
    }
    repack_weights(*h);
  });
}

int sort_get_param(SortHandle p, const char* name, float* out) {
  return api([&] {
    Handle* h = ready(p);
    if (!name || !out) throw ConfigError("null argument");
    if (std::strcmp(name, "tok.item_table") == 0) {  // fp32 master when trained, else the bf16 table widened
      const size_t n = static_cast<size_t>(h->cfg.n_items) * h->cfg.item_dim;
      if (h->item_master) {
        CK(cudaMemcpyAsync(out, h->item_master, n * 4, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        return;
      }
      std::vector<__nv_bfloat16> b(n);
      CK(cudaMemcpyAsync(b.data(), h->item, n * 2, cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      for (size_t i = 0; i < n; ++i) out[i] = __bfloat162float(b[i]);
      return;
    }
    auto it = h->grad_index.find(name);
    if (it == h->grad_index.end()) throw ConfigError(std::string("no trainable parameter ") + name);
    const size_t n = static_cast<size_t>(it->second.second.first) * it->second.second.second;
    CK(cudaMemcpyAsync(out, h->master + it->second.first, n * 4, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  });
}

int sort_get_grad(SortHandle p, const char* name, float* out) {
  return api([&] {
    Handle* h = ready(p);
    if (!name || !out) throw ConfigError("null argument");
    if (!h->grads) throw ConfigError("no gradients yet (call sort_train_step)");
    if (std::strcmp(name, "tok.item_table") == 0) {
      if (h->frozen.count(name) || !h->item_grad) throw ConfigError("tok.item_table is frozen: no gradient");
      const size_t n = static_cast<size_t>(h->cfg.n_items) * h->cfg.item_dim;
      CK(cudaMemcpyAsync(out, h->item_grad, n * 4, cudaMemcpyDeviceToHost, h->stream));
    } else {
      auto it = h->grad_index.find(name);
      if (it == h->grad_index.end()) throw ConfigError(std::string("no trainable parameter ") + name);
      const size_t n = static_cast<size_t>(it->second.second.first) * it->second.second.second;
      CK(cudaMemcpyAsync(out, h->grads + it->second.first, n * 4, cudaMemcpyDeviceToHost, h->stream));
    }
    CK(cudaStreamSynchronize(h->stream));
  });
}


int sort_set_frozen(SortHandle p, const char* name, int32_t frozen) {
  return api([&] {
    Handle* h = ready(p);
    if (!name) throw ConfigError("null argument");
    const std::string n(name);
    if (n != "tok.item_table" && !h->grad_index.count(n)) throw ConfigError("no parameter " + n);
    if (frozen) {
      h->frozen.insert(n);
      return;
    }
    if (n == "tok.item_table") {
      if (h->item_ext) throw ConfigError("the row-sharded item table (sort_set_item_table) is not trained here");
      unfreeze_item_table(*h);
    }
    h->frozen.erase(n);
  });
}

int sort_transfer_item_table(SortHandle from, SortHandle to, int32_t freeze) {
  return api([&] {
    Handle* a = ready(from);
    Handle* b = ready(to);
    if (a->cfg.n_items != b->cfg.n_items || a->cfg.item_dim != b->cfg.item_dim)
      throw ConfigError("transfer_item_table: item vocabularies differ");
    const size_t n = static_cast<size_t>(a->cfg.n_items) * a->cfg.item_dim;
    std::vector<float> t(n);
    CK(cudaSetDevice(a->device));
    if (a->item_master) {
      CK(cudaMemcpyAsync(t.data(), a->item_master, n * 4, cudaMemcpyDeviceToHost, a->stream));
      CK(cudaStreamSynchronize(a->stream));
    } else {
      std::vector<__nv_bfloat16> hb(n);
      CK(cudaMemcpyAsync(hb.data(), a->item, n * 2, cudaMemcpyDeviceToHost, a->stream));
      CK(cudaStreamSynchronize(a->stream));
      for (size_t i = 0; i < n; ++i) t[i] = __bfloat162float(hb[i]);
    }
    CK(cudaSetDevice(b->device));
    const std::vector<__nv_bfloat16> tb = to_bf16(t);
    CK(cudaMemcpyAsync(b->item, tb.data(), n * 2, cudaMemcpyHostToDevice, b->stream));
    if (b->item_master) {
      CK(cudaMemcpyAsync(b->item_master, t.data(), n * 4, cudaMemcpyHostToDevice, b->stream));
      CK(cudaMemsetAsync(b->item_m, 0, n * 4, b->stream));
      CK(cudaMemsetAsync(b->item_v, 0, n * 4, b->stream));
    }
    CK(cudaStreamSynchronize(b->stream));
    b->drop_graphs();
    if (freeze) {
      b->frozen.insert("tok.item_table");
    } else {
      unfreeze_item_table(*b);
      b->frozen.erase("tok.item_table");
    }
  });
}

int sort_grad_info(SortHandle p, const char* name, int64_t* offset, int64_t* rows, int64_t* cols,
                   int64_t* total) {
  return api([&] {
    Handle* h = ready(p);
    if (total) *total = static_cast<int64_t>(h->grad_count);
    if (!name) return;
    auto it = h->grad_index.find(name);
    if (it == h->grad_index.end()) throw ConfigError(std::string("no gradient for parameter ") + name);
    if (offset) *offset = static_cast<int64_t>(it->second.first);
    if (rows) *rows = it->second.second.first;
    if (cols) *cols = it->second.second.second;
  });
}

int sort_grads_copy(SortHandle p, float* buf, int buf_on_device, int to_handle) {
  return api([&] {
    Handle* h = ready(p);
    if (!buf) throw ConfigError("null argument");
    if (!h->grads) throw ConfigError("no gradients yet (call sort_train_step)");
    const size_t bytes = h->grad_count * sizeof(float);
    if (to_handle)
      CK(cudaMemcpyAsync(h->grads, buf, bytes, buf_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                         h->stream));
    else
      CK(cudaMemcpyAsync(buf, h->grads, bytes, buf_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                         h->stream));
    CK(cudaStreamSynchronize(h->stream));
  });
}

int sort_dtokens(SortHandle p, int32_t batch, float* out) {
  return api([&] {
    Handle* h = ready(p);
    if (!out || !h->dtokens) throw ConfigError("no token gradients yet (call sort_train_step)");
    CK(cudaMemcpyAsync(out, h->dtokens, static_cast<size_t>(batch) * h->L0 * h->d * 4, cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
  });
}

int sort_set_item_table(SortHandle p, const void* rows, int64_t n_rows) {
  return api([&] {
    Handle* h = reinterpret_cast<Handle*>(p);
    if (!h) throw ConfigError("null handle");
    if (rows && (n_rows < 1 || n_rows > INT32_MAX)) throw ConfigError("item table rows out of range");
    h->item_ext = static_cast<const __nv_bfloat16*>(rows);
    h->item_ext_rows = rows ? n_rows : 0;
  });
}

int sort_gather_rows(const void* table, int64_t n_rows, int32_t row_bytes, const int64_t* ids, int64_t n,
                     void* out, void* stream) {
  return api([&] {
    if (!table || !ids || !out) throw ConfigError("null argument");
    if (row_bytes <= 0 || row_bytes % 16) throw ConfigError("row_bytes must be a positive multiple of 16");
    if (n == 0) return;
    int32_t* err = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&err), 4, static_cast<cudaStream_t>(stream)));
    CK(cudaMemsetAsync(err, 0, 4, static_cast<cudaStream_t>(stream)));
    const int chunks = row_bytes / 16;
    const int64_t threads = n * chunks;
    const int grid = static_cast<int>(std::min<int64_t>((threads + 255) / 256, 148 * 32));
    k_gather_table_rows<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const int4*>(table), n_rows, chunks, ids, n, static_cast<int4*>(out), err);
    check_launch("gather rows");
    int32_t herr = 0;
    CK(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)));
    CK(cudaFreeAsync(err, static_cast<cudaStream_t>(stream)));
    CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    if (herr) throw ConfigError("gather rows: id outside the table shard");
  });
}

int sort_pretrain_forward(SortHandle p, const SortBatch* batch, int inputs_on_device, float* lse,
                          float* target_logit, int outputs_on_device) {
  return api([&] {
    Handle* h = ready(p);
    if (!batch || !lse || !target_logit) throw ConfigError("null argument");
    if (!h->cfg.pretrain) throw ConfigError("sort_pretrain_forward needs a pre-training model (pretrain = 1)");
    begin_timing(*h);
    upload_batch(*h, batch, inputs_on_device != 0);
    forward_device(*h, batch->batch);
    const size_t bytes = static_cast<size_t>(batch->batch) * h->cfg.n_hist * sizeof(float);
    const cudaMemcpyKind k = outputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CK(cudaMemcpyAsync(lse, h->pre_lse, bytes, k, h->stream));
    CK(cudaMemcpyAsync(target_logit, h->pre_tgt, bytes, k, h->stream));
    if (!(inputs_on_device && outputs_on_device)) collect_status(*h);
  });
}

int sort_moe_routing(SortHandle p, int layer, int32_t capacity_rows, int32_t* rows_out, int32_t* sel,
                     float* weights) {
  return api([&] {
    Handle* h = ready(p);
    if (!h->moe) throw ConfigError("moe: the model has no MoE FFN");
    if (layer < 0 || layer >= h->cfg.layers) throw ConfigError("moe: layer out of range");
    const LayerDev& L = h->layers[layer];
    if (rows_out) *rows_out = h->moe_rows[layer];
    if ((sel || weights) && capacity_rows < h->moe_rows[layer])
      throw ConfigError("moe: routing buffers hold " + std::to_string(capacity_rows) + " rows, the last forward routed " +
                        std::to_string(h->moe_rows[layer]));
    const size_t n = static_cast<size_t>(h->moe_rows[layer]) * h->moe_k;
    if (sel) CK(cudaMemcpyAsync(sel, L.moe_sel, n * 4, cudaMemcpyDeviceToHost, h->stream));
    if (weights) CK(cudaMemcpyAsync(weights, L.moe_w, n * 4, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  });
}

int sort_moe_load(SortHandle p, int layer, int64_t* load) {
  return api([&] {
    Handle* h = ready(p);
    if (!h->moe) throw ConfigError("moe: the model has no MoE FFN");
    if (layer < 0 || layer >= h->cfg.layers || !load) throw ConfigError("moe: bad argument");
    std::vector<int32_t> c(h->moe_E);
    CK(cudaMemcpyAsync(c.data(), h->moe_counts + static_cast<size_t>(layer) * h->moe_E, c.size() * 4,
                       cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    for (int e = 0; e < h->moe_E; ++e) load[e] = c[e];
  });
}

int sort_moe_update_bias(SortHandle p, double gamma) {
  return api([&] {
    Handle* h = ready(p);
    if (!h->moe) throw ConfigError("moe: the model has no MoE FFN");
    for (int l = 0; l < h->cfg.layers; ++l)
      k_moe_update_bias<<<1, 64, 0, h->stream>>>(h->moe_counts + static_cast<size_t>(l) * h->moe_E, h->moe_E,
                                                 static_cast<float>(gamma), h->layers[l].router_bias);
    check_launch("moe bias update");
    CK(cudaStreamSynchronize(h->stream));
  });
}

int sort_moe_forward(SortHandle p, int layer, const float* x, int rows, float* out) {
  return api([&] {
    Handle* h = ready(p);
    if (!h->moe) throw ConfigError("moe: the model has no MoE FFN");
    if (layer < 0 || layer >= h->cfg.layers || !x || !out || rows < 0) throw ConfigError("moe: bad argument");
    const size_t cap = static_cast<size_t>(h->Bmax) * h->plan.layers[layer].l_q;
    if (static_cast<size_t>(rows) > cap) throw ConfigError("moe: more rows than the layer's workspace");
    const int d = h->d;
    std::vector<__nv_bfloat16> xb(static_cast<size_t>(rows) * d);
    for (size_t i = 0; i < xb.size(); ++i) xb[i] = f2bf(x[i]);
    __nv_bfloat16* X = h->X[0];
    CK(cudaMemcpyAsync(X, xb.data(), xb.size() * 2, cudaMemcpyHostToDevice, h->stream));
    if (rows > 0) run_moe(*h, layer, X, h->SS[0], rows);
    CK(cudaMemcpyAsync(xb.data(), X, xb.size() * 2, cudaMemcpyDeviceToHost, h->stream));
    collect_status(*h);
    for (size_t i = 0; i < xb.size(); ++i) out[i] = __bfloat162float(xb[i]);
  });
}

int sort_set_option(SortHandle p, const char* name, int32_t value) {
  return api([&] {
    Handle* h = reinterpret_cast<Handle*>(p);
    if (!h || !name) throw ConfigError("null argument");
    h->drop_graphs();
    if (std::strcmp(name, "graphs") == 0) {
      h->use_graphs = value != 0;
    } else if (std::strcmp(name, "fused_tail") == 0) {
      h->fused_tail = value != 0;
    } else if (std::strcmp(name, "tail_pair") == 0) {
      h->tail_pair = value != 0;
    } else if (std::strcmp(name, "attn_bwd_mma") == 0) {
      h->attn_bwd_mma = value != 0;
    } else if (std::strcmp(name, "pre_proj_tc") == 0) {
      h->pre_proj_tc = value != 0;
    } else if (std::strcmp(name, "ce_tc") == 0) {
      h->ce_tc = value != 0;
    } else if (std::strcmp(name, "head_tc") == 0) {
      h->head_tc = value != 0;
    } else if (std::strcmp(name, "attn_prescale") == 0) {
      h->attn_prescale = value != 0;
    } else if (std::strcmp(name, "qkvg_pair") == 0) {
      h->qkvg_pair = value != 0;

    } else if (std::strcmp(name, "stream_gemm") == 0) {
      h->stream_gemm = value != 0;
    } else if (std::strcmp(name, "train_cublas") == 0) {
      h->train_cublas = value != 0;
    } else if (std::strcmp(name, "attn_bwd_tc") == 0) {
      h->attn_bwd_tc = value != 0;
    } else if (std::strcmp(name, "moe_fused") == 0) {
      h->moe_fused = value != 0;
    } else {
      throw ConfigError(std::string("unknown option ") + name);
    }
  });
}

int sort_stage_times(SortHandle p, float* ms, int32_t cap, int32_t* n, char* names, int32_t names_cap) {
  return api([&] {
    Handle* h = reinterpret_cast<Handle*>(p);
    if (!h) throw ConfigError("null handle");
    const int cnt = static_cast<int>(std::min<size_t>(h->stage_ms.size(), static_cast<size_t>(cap)));
    for (int i = 0; i < cnt; ++i) ms[i] = h->stage_ms[i];
    *n = cnt;
    std::string s;
    for (int i = 0; i < cnt; ++i) s += (i ? ";" : "") + h->stage_names[i + 1];
    if (names && names_cap > 0) {
      std::strncpy(names, s.c_str(), static_cast<size_t>(names_cap) - 1);
      names[names_cap - 1] = 0;
    }
  });
}

}  // extern "C"

#include "layer_op.cuh"  // operator-level entries (rmsnorm / rope / attention layer)
