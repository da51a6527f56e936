// SPDX-License-Identifier: Apache-2.0
//
// rankformer::gpu -- C++ host binding of libsort_b200.so that keeps the reference's
// rankformer:: names and semantics (/root/reference/proj/include/rankformer/):
//
//   reference                                         here
//   ------------------------------------------------  -------------------------------------
//   RequestSample / ItemEvent / Candidate (data.hpp)   same structs (no side features)
//   ConfigError / RuntimeFailure (common.hpp:17-27)    same names, thrown on status 1 / 2
//   time_bucket (tokenizer.cpp:36-40)                  gpu::time_bucket
//   make_geometric_schedule (mask.cpp:97-117)          gpu::make_geometric_schedule
//   retained_rows (mask.cpp:132-154)                   gpu::retained_rows
//   build_mask (mask.cpp:14-76) -> Mat of {0,-inf}     gpu::build_mask (compact form expanded)
//   mask_visible_count (mask.cpp:87-95)                gpu::mask_visible_count
//   Tokenizer::tokenize_sample (tokenizer.cpp:144)     gpu::Model::tokenize_sample
//   model_forward                    gpu::Model::score (batched on the GPU)
//   blockwise_masked_attention (block_attention.hpp)   gpu::blockwise_masked_attention
//
// Eigen is not available in this image, so Mat is a small owning row-major matrix with the
// accessors the reference code uses (rows(), cols(), operator()(r, c), row pointer).
// Header-only; link with -lsort_b200 (or dlopen). One Model per GPU; a Model is not
// thread-safe -- drive each from its own host thread (params.hpp:12-14 concurrency model).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../sort_b200.h"

namespace rankformer {

class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& what) : std::runtime_error(what) {}
};
class RuntimeFailure : public std::runtime_error {
 public:
  explicit RuntimeFailure(const std::string& what) : std::runtime_error(what) {}
};

enum class Role : int { kBos = 0, kHist = 1, kSep = 2, kProf = 3, kCand = 4 };
enum class ActionType : int { kClick = 0, kCart = 1, kPurchase = 2 };

struct ItemEvent {
  int32_t item_id = 0;
  ActionType action_type = ActionType::kClick;
  int64_t timestamp = 0;
  int32_t scene_id = 0;
};
struct Candidate {
  int32_t item_id = 0;
  int click = 0, cart = 0, purchase = 0;
};
struct RequestSample {
  int64_t request_id = 0;
  int64_t timestamp = 0;
  std::vector<int32_t> user_profile;
  std::vector<ItemEvent> history;
  std::vector<Candidate> candidates;
};

// Owning row-major matrix (stand-in for rankformer::Mat = Eigen row-major double).
template <class T>
class MatT {
 public:
  MatT() = default;
  MatT(int64_t r, int64_t c, T fill = T(0)) : r_(r), c_(c), a_(static_cast<size_t>(r * c), fill) {}
  int64_t rows() const { return r_; }
  int64_t cols() const { return c_; }
  T& operator()(int64_t i, int64_t j) { return a_[static_cast<size_t>(i * c_ + j)]; }
  T operator()(int64_t i, int64_t j) const { return a_[static_cast<size_t>(i * c_ + j)]; }
  T* data() { return a_.data(); }
  const T* data() const { return a_.data(); }

 private:
  int64_t r_ = 0, c_ = 0;
  std::vector<T> a_;
};
using Mat = MatT<double>;

struct TokenSequence {
  Mat tokens;  // L x d (the device's bf16 token rows, widened)
  std::vector<int> position_ids;
  std::vector<Role> roles;
  std::vector<int> candidate_index;
  std::vector<int> hist_time;  // TokenizerCache::hist_time (tokenizer.hpp:68)
  int n_candidates = 0;
  int length() const { return static_cast<int>(roles.size()); }
  int prefix_len() const { return length() - n_candidates; }
};

namespace gpu {

inline void check(int status) {
  if (status == SORT_OK) return;
  const std::string msg = sort_last_error();
  if (status == SORT_CONFIG_ERROR) throw ConfigError(msg);
  throw RuntimeFailure(msg);
}

inline int time_bucket(int64_t delta_seconds, int n_buckets) {
  return sort_time_bucket(delta_seconds, n_buckets);
}

inline std::vector<int> make_geometric_schedule(int prefix_len, int depth, int target) {
  std::vector<int32_t> k(static_cast<size_t>(depth < 1 ? 1 : depth));
  check(sort_geometric_schedule(prefix_len, depth, target, k.data()));
  return std::vector<int>(k.begin(), k.end());
}

inline std::vector<int> retained_rows(const std::vector<Role>& roles, int keep, bool keep_specials) {
  std::vector<int32_t> r(roles.size()), out(roles.size());
  for (size_t i = 0; i < roles.size(); ++i) r[i] = static_cast<int32_t>(roles[i]);
  int32_t n = 0;
  check(sort_retained_rows(r.data(), static_cast<int32_t>(r.size()), keep, keep_specials, out.data(), &n));
  return std::vector<int>(out.begin(), out.begin() + n);
}

// build_mask (mask.hpp:36-42): query_rows empty = suffix overload. Entries are 0 / -inf.
inline Mat build_mask(int l_q, int local_window, int full_suffix, const std::vector<Role>& roles,
                      const std::vector<int>& position_ids, std::vector<int> query_rows = {}) {
  const int l_kv = static_cast<int>(roles.size());
  if (query_rows.empty())
    for (int i = 0; i < l_q; ++i) query_rows.push_back(l_kv - l_q + i);
  std::vector<int32_t> r(roles.size()), p(position_ids.begin(), position_ids.end()),
      q(query_rows.begin(), query_rows.end()), lo(l_q), hi(l_q), se(l_q);
  for (size_t i = 0; i < roles.size(); ++i) r[i] = static_cast<int32_t>(roles[i]);
  check(sort_mask_intervals(l_q, l_kv, local_window, full_suffix, r.data(), p.data(), q.data(),
                            lo.data(), hi.data(), se.data()));
  Mat m(l_q, l_kv, -std::numeric_limits<double>::infinity());
  for (int i = 0; i < l_q; ++i) {
    for (int c = lo[i]; c <= hi[i]; ++c) m(i, c) = 0.0;
    if (se[i] >= 0) m(i, se[i]) = 0.0;
  }
  return m;
}

inline int64_t mask_visible_count(const Mat& mask) {
  int64_t n = 0;
  for (int64_t i = 0; i < mask.rows(); ++i)
    for (int64_t j = 0; j < mask.cols(); ++j) n += mask(i, j) == 0.0;
  return n;
}

struct BlockAttentionResult {
  MatT<float> output;
  int64_t skipped_blocks = 0, total_blocks = 0;
  double skipped_fraction() const {
    return total_blocks ? static_cast<double>(skipped_blocks) / static_cast<double>(total_blocks) : 0.0;
  }
};

// blockwise_masked_attention (block_attention.hpp:58-62) with the mask given in the compact
// form build_mask rows take (one interval + self per row); tiles are the kernel's 128 x 128.
inline BlockAttentionResult blockwise_masked_attention(const MatT<float>& q, const MatT<float>& k,
                                                       const MatT<float>& v,
                                                       const std::vector<int32_t>& lo,
                                                       const std::vector<int32_t>& hi,
                                                       const std::vector<int32_t>& self_idx) {
  BlockAttentionResult res;
  res.output = MatT<float>(q.rows(), v.cols());
  check(sort_block_attention(1, static_cast<int32_t>(q.rows()), static_cast<int32_t>(k.rows()),
                             static_cast<int32_t>(q.cols()), q.data(), k.data(), v.data(), lo.data(),
                             hi.data(), self_idx.data(), res.output.data(), &res.skipped_blocks,
                             &res.total_blocks));
  return res;
}

// The SORT model on one GPU: tokenizer -> block stack -> ranking head.
class Model {
 public:
  // params: reference-named [rows, cols] row-major tensors (see sort_load_param).
  Model(const SortConfig& cfg, const std::map<std::string, std::pair<std::vector<int64_t>, std::vector<float>>>& params,
        int device = 0)
      : cfg_(cfg) {
    check(sort_create(&cfg_, device, &h_));
    for (const auto& [name, t] : params)
      check(sort_load_param(h_, name.c_str(), t.second.data(), t.first.at(0), t.first.at(1)));
    check(sort_finalize_params(h_));
  }
  ~Model() {
    if (h_) sort_destroy(h_);
  }
  Model(const Model&) = delete;
  Model& operator=(const Model&) = delete;

  // model_forward for every request: {p_click, p_cart, p_purchase} per candidate. Requests
  // are packed AoS -> SoA and scored in GPU batches of the planned geometry (n_hist, n_cand);
  // a request with another geometry is a ConfigError (issue it through a Model planned for it).
  // Batches go through the pipelined serving path (sort_forward_async: each batch's host ->
  // device copy overlaps the previous batch's kernels), one sync at the end.
  std::vector<std::vector<std::array<float, 3>>> score(const std::vector<RequestSample>& reqs) {
    std::vector<std::vector<std::array<float, 3>>> out(reqs.size());
    std::vector<Packed> packs;
    std::vector<std::vector<float>> scores;
    std::vector<size_t> first;
    for (size_t b0 = 0; b0 < reqs.size(); b0 += static_cast<size_t>(cfg_.max_batch)) {
      const size_t nb = std::min(reqs.size() - b0, static_cast<size_t>(cfg_.max_batch));
      packs.push_back(pack(reqs, b0, nb));
      scores.emplace_back(nb * static_cast<size_t>(cfg_.n_cand) * 3);
      first.push_back(b0);
    }
    for (size_t k = 0; k < packs.size(); ++k) {
      packs[k].batch = bind(packs[k]);  // (vectors moved into the list: re-point the SoA batch)
      check(sort_forward_async(h_, &packs[k].batch, scores[k].data()));
    }
    check(sort_sync(h_));
    for (size_t k = 0; k < packs.size(); ++k) {
      const size_t nb = static_cast<size_t>(packs[k].batch.batch);
      for (size_t i = 0; i < nb; ++i) {
        auto& o = out[first[k] + i];
        o.resize(static_cast<size_t>(cfg_.n_cand));
        for (int j = 0; j < cfg_.n_cand; ++j)
          for (int q = 0; q < 3; ++q)
            o[static_cast<size_t>(j)][static_cast<size_t>(q)] =
                scores[k][(i * static_cast<size_t>(cfg_.n_cand) + static_cast<size_t>(j)) * 3 + static_cast<size_t>(q)];
      }
    }
    return out;
  }

  // pretrain_forward (cfg.pretrain = 1): for every click sequence of
  // cfg.n_hist clicks, the next-item cross entropy of each position (lse - target logit).
  std::vector<std::vector<float>> pretrain_ce(const std::vector<std::vector<ItemEvent>>& seqs) {
    std::vector<std::vector<float>> out(seqs.size());
    for (size_t b0 = 0; b0 < seqs.size(); b0 += static_cast<size_t>(cfg_.max_batch)) {
      const size_t nb = std::min(seqs.size() - b0, static_cast<size_t>(cfg_.max_batch));
      Packed p;
      for (size_t i = b0; i < b0 + nb; ++i) {
        if (static_cast<int>(seqs[i].size()) != cfg_.n_hist)
          throw ConfigError("click sequence length differs from the planned n_hist");
        for (const ItemEvent& e : seqs[i]) {
          p.item.push_back(e.item_id);
          p.action.push_back(static_cast<int32_t>(e.action_type));
          p.scene.push_back(e.scene_id);
          p.ts.push_back(e.timestamp);
        }
        p.req.push_back(0);
      }
      p.batch = bind(p);
      p.batch.batch = static_cast<int32_t>(nb);
      const size_t n = nb * static_cast<size_t>(cfg_.n_hist);
      std::vector<float> lse(n), tgt(n);
      check(sort_pretrain_forward(h_, &p.batch, 0, lse.data(), tgt.data(), 0));
      for (size_t i = 0; i < nb; ++i) {
        out[b0 + i].resize(static_cast<size_t>(cfg_.n_hist));
        for (int t = 0; t < cfg_.n_hist; ++t) {
          const size_t k = i * static_cast<size_t>(cfg_.n_hist) + static_cast<size_t>(t);
          out[b0 + i][static_cast<size_t>(t)] = lse[k] - tgt[k];
        }
      }
    }
    return out;
  }

  // MoE FFN (cfg.moe_experts > 0): expert loads of `layer` in the last
  // forward, and update_balance (router_bias_e -= gamma * sign(load_e - mean)) on every layer.
  std::vector<int64_t> moe_load(int layer) {
    std::vector<int64_t> load(static_cast<size_t>(cfg_.moe_experts));
    check(sort_moe_load(h_, layer, load.data()));
    return load;
  }
  void moe_update_bias(double gamma = 1e-3) { check(sort_moe_update_bias(h_, gamma)); }

  // Tokenizer::tokenize_sample (tokenizer.hpp:84) of one request.
  TokenSequence tokenize_sample(const RequestSample& s) {
    std::vector<RequestSample> one{s};
    Packed p = pack(one, 0, 1);
    const int L = seq_len();
    TokenSequence t;
    t.tokens = Mat(L, cfg_.model_dim);
    std::vector<float> tok(static_cast<size_t>(L) * static_cast<size_t>(cfg_.model_dim));
    std::vector<int32_t> pos(L), roles(L), cidx(L), ht(static_cast<size_t>(cfg_.n_hist > 0 ? cfg_.n_hist : 1));
    check(sort_tokenize(h_, &p.batch, tok.data(), ht.data(), pos.data(), roles.data(), cidx.data()));
    for (size_t i = 0; i < tok.size(); ++i) t.tokens.data()[i] = tok[i];
    t.position_ids.assign(pos.begin(), pos.end());
    for (int32_t r : roles) t.roles.push_back(static_cast<Role>(r));
    t.candidate_index.assign(cidx.begin(), cidx.end());
    t.hist_time.assign(ht.begin(), ht.begin() + cfg_.n_hist);
    t.n_candidates = cfg_.n_cand;
    return t;
  }

  int seq_len() const {
    if (cfg_.pretrain) return 1 + cfg_.n_hist;  // [BOS; clicks]
    return (cfg_.special_tokens ? 3 : 0) + cfg_.n_hist + cfg_.n_profile_fields + cfg_.n_cand;
  }
  SortHandle handle() const { return h_; }

 private:
  struct Packed {
    std::vector<int32_t> item, action, scene, prof, cand;
    std::vector<int64_t> ts, req;
    SortBatch batch{};
  };
  // the SoA batch over a Packed's arrays (after the Packed was moved into a container)
  static SortBatch bind(const Packed& p) {
    SortBatch b = p.batch;
    b.hist_item = p.item.data();
    b.hist_action = p.action.data();
    b.hist_scene = p.scene.data();
    b.hist_ts = p.ts.data();
    b.req_ts = p.req.data();
    b.profile = p.prof.data();
    b.cand_item = p.cand.data();
    return b;
  }
  Packed pack(const std::vector<RequestSample>& reqs, size_t b0, size_t nb) const {
    Packed p;
    for (size_t i = b0; i < b0 + nb; ++i) {
      const RequestSample& s = reqs[i];
      if (static_cast<int>(s.history.size()) != cfg_.n_hist || static_cast<int>(s.candidates.size()) != cfg_.n_cand ||
          static_cast<int>(s.user_profile.size()) != cfg_.n_profile_fields)
        throw ConfigError("request geometry differs from the planned (n_hist, n_cand, profile)");
      for (const ItemEvent& e : s.history) {
        p.item.push_back(e.item_id);
        p.action.push_back(static_cast<int32_t>(e.action_type));
        p.scene.push_back(e.scene_id);
        p.ts.push_back(e.timestamp);
      }
      p.req.push_back(s.timestamp);
      p.prof.insert(p.prof.end(), s.user_profile.begin(), s.user_profile.end());
      for (const Candidate& c : s.candidates) p.cand.push_back(c.item_id);
    }
    p.batch.batch = static_cast<int32_t>(nb);
    p.batch.hist_item = p.item.data();
    p.batch.hist_action = p.action.data();
    p.batch.hist_scene = p.scene.data();
    p.batch.hist_ts = p.ts.data();
    p.batch.req_ts = p.req.data();
    p.batch.profile = p.prof.data();
    p.batch.cand_item = p.cand.data();
    return p;
  }

  SortConfig cfg_;
  SortHandle h_ = nullptr;
};

}  // namespace gpu
}  // namespace rankformer
