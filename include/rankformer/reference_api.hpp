// SPDX-License-Identifier: Apache-2.0
//
// rankformer:: drop-in facade: the reference's free functions and classes of the hot path with
// the reference's SIGNATURES, executed by libsort_b200.so (/root/reference/proj/include/rankformer/):
//
//   reference declaration                                              runs as
//   -----------------------------------------------------------------  ---------------------------------
//   struct MaskSpec (mask.hpp:15-31)                                   same fields / validate()
//   Mat build_mask(const MaskSpec&, roles, position_ids, query_rows)   host planner (sort_mask_intervals),
//     + suffix overload (mask.hpp:36-42)                               rendered 0 / -inf
//   int64_t mask_visible_count(const Mat&) (mask.hpp:44)               host count
//   struct PruneSchedule, make_geometric_schedule, make_full_schedule  sort_geometric_schedule
//     (mask.hpp:48-70)
//   Mat prune_queries(const Mat&, int) (mask.hpp:73)                   row copy
//   retained_rows(roles, keep, keep_specials) (mask.hpp:77-78)         sort_retained_rows
//   int time_bucket(int64_t, int) (tokenizer.hpp:60)                   sort_time_bucket
//   rmsnorm_forward / rmsnorm_backward (norm.hpp:17-45)                GPU: sort_op_rmsnorm(_backward)
//   rope_apply (rope.hpp:13-40)                                        GPU: sort_op_rope
//   Parameter / ParamRefs / ParamIndex / GradBuffer (params.hpp)       same semantics (frozen = no grad)
//   AttentionSettings / AttentionCache / AttentionLayer                GPU: sort_op_attention_layer
//     ::forward(xn, query_rows, mask, position_ids, cache)             (tcgen05 GEMMs + k_attention)
//     ::backward(dout, cache, grads, index)  (attention.hpp:58-63)     (tcgen05 attention backward)
//   TokenizerCache / Tokenizer::tokenize_sample(sample, cache)         GPU: k_tokenize (sort_tokenize)
//     (tokenizer.hpp:60-84)
//   transfer_item_table(from, to, freeze) (tokenizer.hpp:107)          sort_transfer_item_table
//
// Numbers: the reference computes in fp64; here the ops run on the device in fp32 (row ops) or
// bf16 operands with fp32 accumulation (attention), so results agree within the tolerances the
// tests state (tests/test_cpp_reference_api.py), not bit for bit. Masks must be of the form
// build_mask renders (per query row: one contiguous run of visible keys plus at most one more
// visible key, the candidate diagonal); any other pattern is a ConfigError.
// Header-only; link with -lsort_b200.
#pragma once

#include <algorithm>
#include <cmath>
#include <limits>
#include <string>
#include <unordered_map>
#include <vector>

#include "sort_gpu.hpp"

namespace rankformer {

using Vec = MatT<double>;  // column vector (rows x 1), indexed v(i)

// ---------------------------------------------------------------- mask.hpp
struct MaskSpec {
  int l_q = 0;
  int l_kv = 0;
  int local_window = -1;  // -1: unbounded (plain causal)
  int full_suffix = 128;  // F

  int prune_offset() const { return l_kv - l_q; }
  void validate() const {
    if (l_q < 1 || l_kv < l_q) throw ConfigError("MaskSpec: need 1 <= l_q <= l_kv");
    if (local_window != -1 && local_window < 1)
      throw ConfigError("MaskSpec: local_window must be >= 1 or -1 (unbounded)");
    if (full_suffix < 0) throw ConfigError("MaskSpec: full_suffix must be >= 0");
  }
};

inline Mat build_mask(const MaskSpec& spec, const std::vector<Role>& roles, const std::vector<int>& position_ids,
                      const std::vector<int>& query_rows) {
  spec.validate();
  if (static_cast<int>(roles.size()) != spec.l_kv || static_cast<int>(position_ids.size()) != spec.l_kv)
    throw ConfigError("build_mask: roles / position_ids must have l_kv entries");
  if (static_cast<int>(query_rows.size()) != spec.l_q) throw ConfigError("build_mask: need l_q query rows");
  return gpu::build_mask(spec.l_q, spec.local_window, spec.full_suffix, roles, position_ids, query_rows);
}

inline Mat build_mask(const MaskSpec& spec, const std::vector<Role>& roles, const std::vector<int>& position_ids) {
  std::vector<int> q(static_cast<size_t>(std::max(spec.l_q, 0)));
  for (int i = 0; i < spec.l_q; ++i) q[static_cast<size_t>(i)] = spec.l_kv - spec.l_q + i;
  return build_mask(spec, roles, position_ids, q);
}

inline int64_t mask_visible_count(const Mat& mask) { return gpu::mask_visible_count(mask); }

struct PruneSchedule {
  std::vector<int> keep;
  void validate() const {
    for (size_t i = 0; i + 1 < keep.size(); ++i)
      if (keep[i + 1] > keep[i]) throw ConfigError("PruneSchedule: keep counts must be non-increasing");
    for (int k : keep)
      if (k < 1) throw ConfigError("PruneSchedule: keep counts must be >= 1");
  }
};

inline PruneSchedule make_geometric_schedule(int prefix_len, int depth, int target) {
  return PruneSchedule{gpu::make_geometric_schedule(prefix_len, depth, target)};
}

inline PruneSchedule make_full_schedule(int prefix_len, int depth) {
  if (prefix_len < 1 || depth < 1) throw ConfigError("make_full_schedule: prefix_len and depth must be >= 1");
  return PruneSchedule{std::vector<int>(static_cast<size_t>(depth), prefix_len)};
}

inline Mat prune_queries(const Mat& x, int n) {
  if (n < 1 || n > x.rows()) throw ConfigError("prune_queries: need 1 <= n <= rows");
  Mat out(n, x.cols());
  const int64_t r0 = x.rows() - n;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < x.cols(); ++j) out(i, j) = x(r0 + i, j);
  return out;
}

inline std::vector<int> retained_rows(const std::vector<Role>& roles, int keep, bool keep_specials) {
  return gpu::retained_rows(roles, keep, keep_specials);
}

inline int time_bucket(int64_t delta_seconds, int n_buckets) { return gpu::time_bucket(delta_seconds, n_buckets); }

namespace detail {
inline std::vector<float> to_f32(const Mat& m) {
  std::vector<float> v(static_cast<size_t>(m.rows() * m.cols()));
  for (size_t i = 0; i < v.size(); ++i) v[i] = static_cast<float>(m.data()[i]);
  return v;
}
inline Mat from_f32(const std::vector<float>& v, int64_t rows, int64_t cols) {
  Mat m(rows, cols);
  for (size_t i = 0; i < v.size(); ++i) m.data()[i] = static_cast<double>(v[i]);
  return m;
}
// A rendered mask (0 visible, -inf masked) -> the compact per-row form of the attention kernel:
// visible = [lo, hi] U {self}. Rows must have at least one visible key.
inline void compact_mask(const Mat& mask, std::vector<int32_t>& lo, std::vector<int32_t>& hi,
                         std::vector<int32_t>& self_idx) {
  const int64_t R = mask.rows(), C = mask.cols();
  lo.assign(static_cast<size_t>(R), 0);
  hi.assign(static_cast<size_t>(R), -1);
  self_idx.assign(static_cast<size_t>(R), -1);
  for (int64_t i = 0; i < R; ++i) {
    std::vector<std::pair<int32_t, int32_t>> runs;
    for (int64_t j = 0; j < C; ++j) {
      const double v = mask(i, j);
      const bool vis = v == 0.0;
      if (!vis && !(std::isinf(v) && v < 0)) throw ConfigError("mask entries must be 0 or -inf (mask.hpp:11-14)");
      if (!vis) continue;
      if (!runs.empty() && runs.back().second == j - 1) runs.back().second = static_cast<int32_t>(j);
      else runs.emplace_back(static_cast<int32_t>(j), static_cast<int32_t>(j));
    }
    if (runs.empty()) throw ConfigError("mask row " + std::to_string(i) + " sees no key");
    if (runs.size() > 2) throw ConfigError("mask row " + std::to_string(i) + " is not of the build_mask form");
    size_t iv = 0;
    if (runs.size() == 2) {
      const bool second_single = runs[1].first == runs[1].second, first_single = runs[0].first == runs[0].second;
      if (!second_single && !first_single)
        throw ConfigError("mask row " + std::to_string(i) + " is not of the build_mask form");
      iv = second_single ? 0 : 1;
      self_idx[static_cast<size_t>(i)] = runs[1 - iv].first;
    }
    lo[static_cast<size_t>(i)] = runs[iv].first;
    hi[static_cast<size_t>(i)] = runs[iv].second;
  }
}
}  // namespace detail

// ---------------------------------------------------------------- norm.hpp / rope.hpp
constexpr double kRmsEps = 1e-6;

struct RmsNormCache {
  Mat x;        // pre-norm input
  Vec inv_rms;  // 1/rms per row
};

inline Mat rmsnorm_forward(const Mat& x, const Mat& gain, RmsNormCache& cache) {
  if (gain.rows() != 1 || gain.cols() != x.cols()) throw ConfigError("rmsnorm_forward: gain must be 1 x cols");
  cache.x = x;
  cache.inv_rms = Vec(x.rows(), 1);
  const std::vector<float> xf = detail::to_f32(x), gf = detail::to_f32(gain);
  std::vector<float> y(xf.size()), inv(static_cast<size_t>(x.rows()));
  gpu::check(sort_op_rmsnorm(static_cast<int32_t>(x.rows()), static_cast<int32_t>(x.cols()), xf.data(), gf.data(),
                             y.data(), inv.data()));
  for (int64_t r = 0; r < x.rows(); ++r) cache.inv_rms(r, 0) = inv[static_cast<size_t>(r)];
  return detail::from_f32(y, x.rows(), x.cols());
}

inline Mat rmsnorm_backward(const Mat& dy, const RmsNormCache& cache, const Mat& gain, Mat& dgain) {
  const int64_t R = cache.x.rows(), C = cache.x.cols();
  if (dy.rows() != R || dy.cols() != C || gain.cols() != C || dgain.rows() != 1 || dgain.cols() != C)
    throw ConfigError("rmsnorm_backward: shape mismatch");
  const std::vector<float> dyf = detail::to_f32(dy), xf = detail::to_f32(cache.x), gf = detail::to_f32(gain);
  std::vector<float> inv(static_cast<size_t>(R)), dx(dyf.size()), dg(static_cast<size_t>(C), 0.f);
  for (int64_t r = 0; r < R; ++r) inv[static_cast<size_t>(r)] = static_cast<float>(cache.inv_rms(r, 0));
  gpu::check(sort_op_rmsnorm_backward(static_cast<int32_t>(R), static_cast<int32_t>(C), dyf.data(), xf.data(),
                                      inv.data(), gf.data(), dx.data(), dg.data()));
  for (int64_t c = 0; c < C; ++c) dgain(0, c) += dg[static_cast<size_t>(c)];
  return detail::from_f32(dx, R, C);
}

inline Mat rope_apply(const Mat& x, const std::vector<int>& position_ids, double theta_base, bool inverse = false) {
  if (x.cols() % 2 != 0) throw ConfigError("rope_apply: head dim must be even");
  if (static_cast<int64_t>(position_ids.size()) != x.rows())
    throw ConfigError("rope_apply: one position id per row required");
  const std::vector<float> xf = detail::to_f32(x);
  const std::vector<int32_t> p(position_ids.begin(), position_ids.end());
  std::vector<float> out(xf.size());
  gpu::check(sort_op_rope(static_cast<int32_t>(x.rows()), static_cast<int32_t>(x.cols()), xf.data(), p.data(),
                          theta_base, inverse ? 1 : 0, out.data()));
  return detail::from_f32(out, x.rows(), x.cols());
}

// ---------------------------------------------------------------- params.hpp
struct Parameter {
  std::string name;
  Mat value;
  bool frozen = false;
  Parameter() = default;
  Parameter(std::string n, int64_t rows, int64_t cols) : name(std::move(n)), value(rows, cols) {}
  int64_t size() const { return value.rows() * value.cols(); }
};
using ParamRefs = std::vector<Parameter*>;

class ParamIndex {
 public:
  ParamIndex() = default;
  explicit ParamIndex(const ParamRefs& params) {
    for (size_t i = 0; i < params.size(); ++i) map_.emplace(params[i], i);
  }
  size_t of(const Parameter& p) const { return map_.at(&p); }

 private:
  std::unordered_map<const Parameter*, size_t> map_;
};

class GradBuffer {
 public:
  GradBuffer() = default;
  explicit GradBuffer(const ParamRefs& params) { reset_shapes(params); }
  void reset_shapes(const ParamRefs& params) {
    grads_.clear();
    for (const Parameter* p : params) grads_.emplace_back(p->value.rows(), p->value.cols());
  }
  void zero() {
    for (auto& g : grads_) std::fill(g.data(), g.data() + g.rows() * g.cols(), 0.0);
  }
  Mat& operator[](size_t i) { return grads_[i]; }
  const Mat& operator[](size_t i) const { return grads_[i]; }
  size_t size() const { return grads_.size(); }
  void add(const GradBuffer& o) {
    for (size_t i = 0; i < grads_.size(); ++i)
      for (int64_t k = 0; k < grads_[i].rows() * grads_[i].cols(); ++k) grads_[i].data()[k] += o.grads_[i].data()[k];
  }

 private:
  std::vector<Mat> grads_;
};

// ---------------------------------------------------------------- attention.hpp
struct AttentionSettings {
  int model_dim = 64;
  int heads = 4;
  bool qknorm = true;
  bool gate = true;
  double rope_theta = 10000.0;
  int head_dim() const { return model_dim / heads; }
  void validate() const {
    if (heads < 1 || model_dim % heads != 0)
      throw ConfigError("attention: model_dim must be a positive multiple of heads");
    if (head_dim() % 2 != 0) throw ConfigError("attention: head dim must be even for the rotary transform");
  }
};

// What the backward needs: the layer inputs of the forward (the device recomputes the
// projections and the softmax statistics instead of keeping per-head softmax matrices).
struct AttentionCache {
  Mat xn;
  std::vector<int> query_rows;
  std::vector<int> pos_q, pos_kv;
  std::vector<int32_t> lo, hi, self_idx;  // the mask in compact form
  Mat out;
};

class AttentionLayer {
 public:
  AttentionLayer(const AttentionSettings& s, int layer_idx) : s_(s) {
    s_.validate();
    const std::string p = "attn." + std::to_string(layer_idx) + ".";
    const int d = s.model_dim;
    wq_ = Parameter(p + "wq", d, d);
    wk_ = Parameter(p + "wk", d, d);
    wv_ = Parameter(p + "wv", d, d);
    wg_ = Parameter(p + "wg", d, d);
    wo_ = Parameter(p + "wo", d, d);
    gain_q_ = Parameter(p + "qk_gain_q", s.heads, s.head_dim());
    gain_k_ = Parameter(p + "qk_gain_k", s.heads, s.head_dim());
    for (Parameter* g : {&gain_q_, &gain_k_}) std::fill(g->value.data(), g->value.data() + g->size(), 1.0);
  }

  // parameter registry in the reference's order (attention.cpp:58-69)
  ParamRefs params() { return {&wq_, &wk_, &wv_, &wg_, &wo_, &gain_q_, &gain_k_}; }

  Mat forward(const Mat& xn, const std::vector<int>& query_rows, const Mat& mask,
              const std::vector<int>& position_ids, AttentionCache& cache) const {
    const int64_t l_in = xn.rows(), l_q = static_cast<int64_t>(query_rows.size());
    if (xn.cols() != s_.model_dim) throw ConfigError("attention: xn width != model_dim");
    if (mask.rows() != l_q || mask.cols() != l_in) throw ConfigError("attention: mask must be l_q x l_in");
    if (static_cast<int64_t>(position_ids.size()) != l_in) throw ConfigError("attention: one position id per kv row");
    cache.xn = xn;
    cache.query_rows = query_rows;
    cache.pos_kv = position_ids;
    cache.pos_q.clear();
    for (int r : query_rows) {
      if (r < 0 || r >= l_in) throw ConfigError("attention: query row out of range");
      cache.pos_q.push_back(position_ids[static_cast<size_t>(r)]);
    }
    detail::compact_mask(mask, cache.lo, cache.hi, cache.self_idx);
    cache.out = run(cache, nullptr, nullptr, nullptr);
    return cache.out;
  }

  Mat backward(const Mat& dout, const AttentionCache& cache, GradBuffer& grads, const ParamIndex& index) const {
    if (dout.rows() != static_cast<int64_t>(cache.query_rows.size()) || dout.cols() != s_.model_dim)
      throw ConfigError("attention backward: dout must be l_q x model_dim");
    const Parameter* ps[7] = {&wq_, &wk_, &wv_, &wg_, &wo_, &gain_q_, &gain_k_};
    std::vector<std::vector<float>> g(7);
    float* gp[7];
    for (int i = 0; i < 7; ++i) {
      gp[i] = nullptr;
      if (ps[i]->frozen) continue;  // params.hpp:15-25
      g[static_cast<size_t>(i)].assign(static_cast<size_t>(ps[i]->size()), 0.f);
      gp[i] = g[static_cast<size_t>(i)].data();
    }
    Mat dxn;
    run(cache, &dout, &dxn, gp);
    for (int i = 0; i < 7; ++i) {
      if (!gp[i]) continue;
      Mat& G = grads[index.of(*ps[i])];
      for (int64_t k = 0; k < ps[i]->size(); ++k) G.data()[k] += g[static_cast<size_t>(i)][static_cast<size_t>(k)];
    }
    return dxn;
  }

  const AttentionSettings& settings() const { return s_; }

 private:
  Mat run(const AttentionCache& c, const Mat* dout, Mat* dxn, float* const* gp) const {
    const int d = s_.model_dim;
    const int64_t l_in = c.xn.rows(), l_q = static_cast<int64_t>(c.query_rows.size());
    const std::vector<float> x = detail::to_f32(c.xn);
    std::vector<float> w[7];
    const Parameter* ps[7] = {&wq_, &wk_, &wv_, &wg_, &wo_, &gain_q_, &gain_k_};
    const float* wp[7];
    for (int i = 0; i < 7; ++i) {
      w[i] = detail::to_f32(ps[i]->value);
      wp[i] = w[i].data();
    }
    const std::vector<int32_t> q(c.query_rows.begin(), c.query_rows.end()), p(c.pos_kv.begin(), c.pos_kv.end());
    std::vector<float> out(static_cast<size_t>(l_q * d)), dx;
    std::vector<float> dy;
    if (dout) {
      dy = detail::to_f32(*dout);
      dx.resize(static_cast<size_t>(l_in * d));
    }
    gpu::check(sort_op_attention_layer(d, s_.heads, s_.rope_theta, s_.qknorm ? 1 : 0, s_.gate ? 1 : 0,
                                       static_cast<int32_t>(l_in), static_cast<int32_t>(l_q), x.data(), q.data(),
                                       c.lo.data(), c.hi.data(), c.self_idx.data(), p.data(), wp, out.data(),
                                       dout ? dy.data() : nullptr, dout ? dx.data() : nullptr, gp));
    if (dxn) *dxn = detail::from_f32(dx, l_in, d);
    return detail::from_f32(out, l_q, d);
  }

  AttentionSettings s_;
  Parameter wq_, wk_, wv_, wg_, wo_;
  Parameter gain_q_, gain_k_;  // heads x head_dim
};

// ---------------------------------------------------------------- tokenizer.hpp
// The index part of the reference's cache (tokenizer.hpp:63-74): the looked-up ids, time
// buckets and token rows. The fp64 concat rows and norm statistics stay on the device.
struct TokenizerCache {
  struct Group {
    std::vector<int> token_rows;
  };
  Group hist, prof, cand;
  std::vector<int> hist_item, hist_action, hist_scene, hist_time;
  std::vector<int> prof_field, prof_value;
  std::vector<int> cand_item;
  std::vector<std::pair<int, int>> specials;  // (token row, special table row)
};

// Tokenizer over a planned gpu::Model: tokenize_sample keeps the reference signature
// (tokenizer.hpp:84); the parameters are the model's (sort_load_param names "tok.*").
class Tokenizer {
 public:
  explicit Tokenizer(gpu::Model& model) : m_(&model) {}

  gpu::Model& model() const { return *m_; }

  TokenSequence tokenize_sample(const RequestSample& sample, TokenizerCache& cache) const {
    TokenSequence t = m_->tokenize_sample(sample);
    cache = TokenizerCache{};
    const int H = static_cast<int>(sample.history.size()), P = static_cast<int>(sample.user_profile.size());
    const bool sp = t.length() == 3 + H + P + t.n_candidates;
    int row = 0;
    if (sp) cache.specials.emplace_back(row++, 0);  // BOS
    for (int i = 0; i < H; ++i) {
      const ItemEvent& e = sample.history[static_cast<size_t>(i)];
      cache.hist_item.push_back(e.item_id);
      cache.hist_action.push_back(static_cast<int>(e.action_type));
      cache.hist_scene.push_back(e.scene_id);
      cache.hist_time.push_back(t.hist_time[static_cast<size_t>(i)]);
      cache.hist.token_rows.push_back(row++);
    }
    if (sp) cache.specials.emplace_back(row++, 1);  // SEP0
    for (int f = 0; f < P; ++f) {
      cache.prof_field.push_back(f);
      cache.prof_value.push_back(sample.user_profile[static_cast<size_t>(f)]);
      cache.prof.token_rows.push_back(row++);
    }
    if (sp) cache.specials.emplace_back(row++, 2);  // SEP1
    for (const Candidate& c : sample.candidates) {
      cache.cand_item.push_back(c.item_id);
      cache.cand.token_rows.push_back(row++);
    }
    return t;
  }

 private:
  gpu::Model* m_;
};

// tokenizer.cpp:376-383: copy the item table between tokenizers with identical item
// vocabularies and set the destination's frozen flag (sort_transfer_item_table).
inline void transfer_item_table(const Tokenizer& from, Tokenizer& to, bool freeze) {
  gpu::check(sort_transfer_item_table(from.model().handle(), to.model().handle(), freeze ? 1 : 0));
}

}  // namespace rankformer
