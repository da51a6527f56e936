// SPDX-License-Identifier: Apache-2.0
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace sortk {

// time_bucket (tokenizer.cpp:36-40): min(floor(log2(1 + max(d, 0))), nb - 1). For
// nb <= 32 the clamp makes the integer form 63 - clz(1 + d) exact;
// 1 + d is formed in uint64 so d = INT64_MAX cannot overflow.
int time_bucket_int(int64_t delta, int n_buckets) {
  const uint64_t d = delta > 0 ? static_cast<uint64_t>(delta) : 0ull;
  const int b = 63 - __builtin_clzll(d + 1ull);
  return std::min(b, n_buckets - 1);
}

// make_geometric_schedule (mask.cpp:97-117), evaluated in double like the reference.
std::vector<int32_t> geometric_schedule(int prefix_len, int depth, int target) {
  if (depth < 1) throw ConfigError("make_geometric_schedule: depth must be >= 1");
  if (prefix_len < 1) prefix_len = 1;
  const int final_keep = std::min(target, prefix_len);
  std::vector<int32_t> keep(depth);
  if (depth == 1) {
    keep[0] = final_keep;
    return keep;
  }
  const double ratio = static_cast<double>(final_keep) / static_cast<double>(prefix_len);
  int prev = prefix_len;
  for (int l = 0; l < depth; ++l) {
    const double t = static_cast<double>(l) / static_cast<double>(depth - 1);
    int k = static_cast<int>(std::lround(prefix_len * std::pow(ratio, t)));
    k = std::min(std::max(k, final_keep), prev);
    keep[l] = k;
    prev = k;
  }
  return keep;
}

// retained_rows (mask.cpp:132-154): the last `keep` non-candidates + all candidates
// (+ BOS/SEP when keep_specials).
std::vector<int32_t> retained_rows(const std::vector<int32_t>& roles, int keep, bool keep_specials) {
  int non_cand = 0;
  for (int32_t r : roles) non_cand += r != SORT_ROLE_CAND;
  const int drop = non_cand - std::min(keep, non_cand);
  std::vector<int32_t> out;
  out.reserve(roles.size());
  int seen = 0;
  for (size_t i = 0; i < roles.size(); ++i) {
    if (roles[i] == SORT_ROLE_CAND) {
      out.push_back(static_cast<int32_t>(i));
      continue;
    }
    const bool in_suffix = seen >= drop;
    ++seen;
    const bool special = roles[i] == SORT_ROLE_BOS || roles[i] == SORT_ROLE_SEP;
    if (in_suffix || (keep_specials && special)) out.push_back(static_cast<int32_t>(i));
  }
  return out;
}

// Compact form of build_mask (mask.cpp:14-76). For query kv-row qi:
//   candidate           -> every non-candidate kv row c <= qi, plus itself (:57-60)
//   non-candidate       -> non-candidate c <= qi (:55, :61-62)
//   ... and windowed    -> additionally pos[c] in [q_pos - W + 1, q_pos] (:52-53, :63-66)
// Non-candidate kv rows keep their original, strictly increasing positions, so the
// window is a lower_bound on the kv index and the visible set is one interval [lo, hi]
// plus `self` (brute-force checked in tests).
void mask_intervals(int l_q, int l_kv, int window, int full_suffix, const int32_t* roles,
                    const int32_t* pos, const int32_t* query_rows, int32_t* lo, int32_t* hi,
                    int32_t* self_idx) {
  if (l_q < 1 || l_kv < l_q) throw ConfigError("MaskSpec: need 1 <= l_q <= l_kv");
  if (window != -1 && window < 1)
    throw ConfigError("MaskSpec: local_window must be >= 1 or -1 (unbounded)");
  if (full_suffix < 0) throw ConfigError("MaskSpec: full_suffix must be >= 0");
  int prefix_positions = 0;
  bool has_cand = false;
  for (int i = 0; i < l_kv; ++i)
    if (roles[i] == SORT_ROLE_CAND) {
      prefix_positions = pos[i];
      has_cand = true;
      break;
    }
  if (!has_cand)
    for (int i = 0; i < l_kv; ++i) prefix_positions = std::max(prefix_positions, pos[i] + 1);
  std::vector<int32_t> nc_idx, nc_pos;
  for (int i = 0; i < l_kv; ++i)
    if (roles[i] != SORT_ROLE_CAND) {
      if (!nc_pos.empty() && pos[i] <= nc_pos.back())
        throw ConfigError("mask: non-candidate positions must be strictly increasing");
      nc_idx.push_back(i);
      nc_pos.push_back(pos[i]);
    }
  for (int r = 0; r < l_q; ++r) {
    const int qi = query_rows ? query_rows[r] : (l_kv - l_q) + r;
    if (qi < 0 || qi >= l_kv) throw ConfigError("build_mask: query row out of range");
    const int k = static_cast<int>(std::upper_bound(nc_idx.begin(), nc_idx.end(), qi) - nc_idx.begin());
    if (roles[qi] == SORT_ROLE_CAND) {
      lo[r] = k ? nc_idx[0] : 0;
      hi[r] = k ? nc_idx[k - 1] : -1;
      self_idx[r] = qi;
      continue;
    }
    const int q_pos = pos[qi];
    int first = 0;
    if (window != -1 && q_pos < prefix_positions - full_suffix) {
      first = static_cast<int>(
          std::lower_bound(nc_pos.begin(), nc_pos.begin() + k, q_pos - window + 1) - nc_pos.begin());
    }
    if (k == 0 || first >= k)
      throw ConfigError("build_mask: query row " + std::to_string(r) + " has no visible key");
    lo[r] = nc_idx[first];
    hi[r] = nc_idx[k - 1];
    self_idx[r] = -1;
  }
}

// Tile census for the attention kernel: for every 128-row q-tile, the 128-column kv tiles
// with at least one visible entry (blockwise_masked_attention's skip rule,
// block_attention.hpp:86-99, evaluated analytically from the intervals), flagged partial
// unless every valid row sees every column of the tile.
void build_tiles(LayerPlan& p) {
  const int T = kAttnTile;
  p.n_qtiles = (p.l_q + T - 1) / T;
  const int n_kv = (p.l_kv + T - 1) / T;
  p.tile_off.assign(1, 0);
  p.tile_code.clear();
  p.tiles_total = static_cast<int64_t>(p.n_qtiles) * n_kv;
  int64_t issued = 0;
  for (int t = 0; t < p.n_qtiles; ++t) {
    const int r0 = t * T, r1 = std::min(p.l_q, r0 + T);
    for (int u = 0; u < n_kv; ++u) {
      const int c0 = u * T, c1 = std::min(p.l_kv, c0 + T);  // [c0, c1)
      bool any = false;
      for (int r = r0; r < r1; ++r)
        any = any || (p.lo[r] <= c1 - 1 && p.hi[r] >= c0) || (p.self_idx[r] >= c0 && p.self_idx[r] < c1);
      if (!any) continue;
      // warp-level chunk classes: rows [r0 + 32q, +32) x columns [c0 + 32c, +32)
      uint32_t cls = 0;
      for (int q = 0; q < 4; ++q)
        for (int c = 0; c < 4; ++c) {
          const int cs = c0 + 32 * c, ce = cs + 31;
          bool full = ce < p.l_kv, none = true;
          for (int r = r0 + 32 * q; r < std::min(r1, r0 + 32 * q + 32); ++r) {
            const bool sees_all = p.lo[r] <= cs && p.hi[r] >= ce;
            const bool sees_any = (p.lo[r] <= ce && p.hi[r] >= cs) || (p.self_idx[r] >= cs && p.self_idx[r] <= ce);
            full = full && sees_all;
            none = none && !sees_any;
          }
          const int ci = 4 * q + c;
          if (none) cls |= 2u << (2 * ci);  // rows that do not exist count as "none"
          else if (full) cls |= 1u << (2 * ci);
        }
      p.tile_code.push_back(u);
      p.tile_code.push_back(static_cast<int32_t>(cls));
      ++issued;
    }
    p.tile_off.push_back(static_cast<int32_t>(issued));
  }
  p.tiles_issued = issued;
  p.qtile_order.resize(p.n_qtiles);
  std::iota(p.qtile_order.begin(), p.qtile_order.end(), 0);
  std::stable_sort(p.qtile_order.begin(), p.qtile_order.end(), [&](int a, int b) {
    return p.tile_off[a + 1] - p.tile_off[a] > p.tile_off[b + 1] - p.tile_off[b];
  });
}

void validate_config(const SortConfig& c) {
  auto need = [](bool ok, const std::string& what) {
    if (!ok) throw ConfigError(what);
  };
  // TokenizerConfig::validate (tokenizer.cpp:22-34)
  need(c.model_dim >= 1, "TokenizerConfig: model_dim must be >= 1");
  need(c.item_dim >= 1, "TokenizerConfig: item_dim must be >= 1");
  need(c.action_dim >= 1 && c.scene_dim >= 1 && c.time_dim >= 1 && c.profile_dim >= 1,
       "TokenizerConfig: feature dims must be >= 1");
  need(c.n_items >= 1, "TokenizerConfig: n_items must be >= 1");
  need(c.n_time_buckets >= 2, "TokenizerConfig: n_time_buckets must be >= 2");
  need(c.n_time_buckets <= 48, "unsupported: n_time_buckets > 48 (integer time_bucket form)");
  need(c.n_profile_fields >= 0 && c.n_profile_fields <= SORT_MAX_PROFILE_FIELDS,
       "unsupported: n_profile_fields");
  for (int f = 0; f < c.n_profile_fields; ++f)
    need(c.profile_vocab[f] >= 1, "TokenizerConfig: profile vocab sizes must be >= 1");
  // AttentionSettings::validate (attention.hpp:21-28)
  need(c.heads >= 1 && c.model_dim % c.heads == 0,
       "attention: model_dim must be a positive multiple of heads");
  const int dk = c.model_dim / std::max(c.heads, 1);
  need(dk % 2 == 0, "attention: head dim must be even for the rotary transform");
  // B200 kernel geometry
  need(dk == 16 || dk == 32 || dk == 64, "unsupported: head dim must be 16, 32 or 64 in this build");
  need(c.model_dim % 64 == 0 && c.model_dim <= 2048,
       "unsupported: model_dim must be a multiple of 64 and <= 2048 (> 256: generic path)");
  need(c.item_dim % 8 == 0 && c.action_dim % 8 == 0 && c.scene_dim % 8 == 0 &&
           c.time_dim % 8 == 0 && c.profile_dim % 8 == 0,
       "unsupported: embedding dims must be multiples of 8");
  need(c.item_dim + c.action_dim + c.scene_dim + c.time_dim <= 64 && c.profile_dim <= 64,
       "unsupported: concat widths must be <= 64");
  need(c.ffn_dim % 32 == 0, "unsupported: ffn_dim must be a multiple of 32");
  need(c.head_hidden >= 0, "head_hidden must be >= 0");
  need(c.layers >= 1 && c.layers <= SORT_MAX_LAYERS, "layers must be in [1, 64]");
  need(c.qknorm == 1 && c.gate == 1, "unsupported: qknorm and gate must be enabled");
  // MaskSpec / PruneSchedule (mask.hpp:22-30, 51-60)
  need(c.local_window == -1 || c.local_window >= 1,
       "MaskSpec: local_window must be >= 1 or -1 (unbounded)");
  need(c.full_suffix >= 0, "MaskSpec: full_suffix must be >= 0");
  for (int l = 0; l + 1 < c.layers; ++l)
    need(c.keep[l + 1] <= c.keep[l], "PruneSchedule: keep counts must be non-increasing");
  for (int l = 0; l < c.layers; ++l) need(c.keep[l] >= 1, "PruneSchedule: keep counts must be >= 1");
  if (c.pretrain) {  // click-sequence model
    need(c.n_cand == 0 && c.n_profile_fields == 0, "pretrain: sequences have no candidates or profile");
    need(c.n_hist >= 2, "pretrain: sequences shorter than 2 clicks are skipped");
    for (int l = 0; l < c.layers; ++l) need(c.keep[l] >= 1 + c.n_hist, "pretrain: query pruning must be off");
    need(c.moe_experts == 0 && c.model_dim <= 256, "unsupported: pretrain with MoE or model_dim > 256");
  } else {
    need(c.n_cand >= 1, "tokenizer: sample has zero candidates");
  }
  need(c.n_hist >= 0 && c.max_batch >= 1, "batch geometry");
  // MoE FFN: SparsityConfig invariants 1 <= k <= E
  need(c.moe_experts >= 0 && c.moe_experts <= 64, "unsupported: moe_experts must be in [0, 64]");
  if (c.moe_experts > 0) {
    need(c.moe_topk >= 1 && c.moe_topk <= c.moe_experts, "SparsityConfig: need 1 <= k <= E");
    need(c.moe_topk <= 8, "unsupported: moe_topk > 8");
    need(c.moe_shared == 0 || c.moe_shared == 1, "unsupported: moe_shared must be 0 or 1");
    need(c.moe_ffn_dim >= 64 && c.moe_ffn_dim % 64 == 0, "unsupported: moe_ffn_dim must be a multiple of 64");
    need(c.model_dim <= 256, "unsupported: the MoE FFN runs on the tcgen05 path (model_dim <= 256)");
  }
}

Plan make_plan(const SortConfig& c) {
  validate_config(c);
  Plan P;
  const bool st = c.special_tokens != 0;
  // Sequence layout [BOS; H; SEP; U; SEP; C] and positions (tokenizer.cpp:170-237).
  auto push = [&](int role, int n) {
    for (int i = 0; i < n; ++i) P.roles0.push_back(role);
  };
  if (c.pretrain) {  // [BOS; clicks] (tokenizer.cpp:243-256)
    push(SORT_ROLE_BOS, 1);
    push(SORT_ROLE_HIST, c.n_hist);
  } else {
    if (st) push(SORT_ROLE_BOS, 1);
    push(SORT_ROLE_HIST, c.n_hist);
    if (st) push(SORT_ROLE_SEP, 1);
    push(SORT_ROLE_PROF, c.n_profile_fields);
    if (st) push(SORT_ROLE_SEP, 1);
    push(SORT_ROLE_CAND, c.n_cand);
  }
  P.L0 = static_cast<int>(P.roles0.size());
  P.prefix = P.L0 - c.n_cand;
  P.pos0.resize(P.L0);
  P.cand_index0.assign(P.L0, -1);
  for (int i = 0; i < P.L0; ++i) {
    P.pos0[i] = i < P.prefix ? i : P.prefix;
    if (i >= P.prefix) P.cand_index0[i] = i - P.prefix;
  }
  P.max_pos = P.prefix;
  std::vector<int32_t> roles = P.roles0, pos = P.pos0;
  for (int l = 0; l < c.layers; ++l) {
    LayerPlan lp;
    lp.query_rows = retained_rows(roles, c.keep[l], c.keep_specials != 0);
    lp.l_q = static_cast<int>(lp.query_rows.size());
    lp.l_kv = static_cast<int>(roles.size());
    lp.q_identity = lp.l_q == lp.l_kv;  // rows are increasing, so equal size => identity
    lp.roles_kv = roles;
    lp.pos_kv = pos;
    lp.lo.resize(lp.l_q);
    lp.hi.resize(lp.l_q);
    lp.self_idx.resize(lp.l_q);
    mask_intervals(lp.l_q, lp.l_kv, c.local_window, c.full_suffix, roles.data(), pos.data(),
                   lp.query_rows.data(), lp.lo.data(), lp.hi.data(), lp.self_idx.data());
    lp.visible = 0;
    for (int r = 0; r < lp.l_q; ++r)
      lp.visible += std::max(0, lp.hi[r] - lp.lo[r] + 1) + (lp.self_idx[r] >= 0 ? 1 : 0);
    lp.pos_q.resize(lp.l_q);
    std::vector<int32_t> nroles(lp.l_q);
    for (int r = 0; r < lp.l_q; ++r) {
      lp.pos_q[r] = pos[lp.query_rows[r]];
      nroles[r] = roles[lp.query_rows[r]];
    }
    build_tiles(lp);
    roles = nroles;
    pos = lp.pos_q;
    P.layers.push_back(std::move(lp));
  }
  // Candidates must stay the contiguous suffix of every layer's rows (the head reads them there).
  const auto& last = P.layers.back();
  int nc = 0;
  for (int r = 0; r < last.l_q; ++r) nc += roles[r] == SORT_ROLE_CAND;
  if (nc != c.n_cand) throw RuntimeFailure("plan: candidates lost through pruning");
  return P;
}

}  // namespace sortk
