// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY -- C entry points over the REFERENCE's own code.
//
// oracle/Makefile compiles /root/reference/proj/src/{mask,tokenizer,attention}.cpp unmodified
// (against oracle/ref_shim/Eigen/Dense, with oracle/ref_shim/ref_fixups.hpp force-included
// for the three undeclared names in AttentionLayer::backward) and links them with this file
// into oracle/_ref/libref.so. tests/ use it to pin the CPU restatement (oracle/sort_oracle.cpp)
// and the CUDA path to what the reference itself computes:
//   * every integer rule: time_bucket, build_mask / mask_visible_count, retained_rows,
//     make_geometric_schedule / make_full_schedule, prune_queries (mask.cpp, tokenizer.cpp);
//   * Tokenizer::tokenize_sample / tokenize_click_sequence / backward (tokenizer.cpp:144-354);
//   * rmsnorm_forward / rmsnorm_backward (norm.hpp), rope_apply (rope.hpp);
//   * AttentionLayer::forward / backward (attention.cpp:71-202);
//   * dense_masked_attention / blockwise_masked_attention (block_attention.hpp);
//   * a model forward COMPOSED from those reference calls. The pieces the reference only
//     specifies in prose -- the pre-norm residual block, the SwishGLU FFN and the ranking
//     head -- are written here from the spec, with the
//     reference's own sigmoid / swish (common.hpp:29-37) and rmsnorm_forward.
// Nothing in the product links, loads or calls this library.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "rankformer/attention.hpp"
#include "rankformer/block_attention.hpp"
#include "rankformer/mask.hpp"
#include "rankformer/norm.hpp"
#include "rankformer/rope.hpp"
#include "rankformer/tokenizer.hpp"
#include "sort_oracle.h"

using namespace rankformer;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const RuntimeFailure& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

Mat from_rows(const double* p, int rows, int cols) {
  Mat m(rows, cols);
  std::memcpy(m.data(), p, sizeof(double) * static_cast<size_t>(rows) * cols);
  return m;
}

void to_rows(const Mat& m, double* out) { std::memcpy(out, m.data(), sizeof(double) * m.size()); }

std::vector<Role> roles_of(const int* r, int n) {
  std::vector<Role> o(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) o[static_cast<size_t>(i)] = static_cast<Role>(r[i]);
  return o;
}

RequestSample sample_of(const OrSample& s) {
  RequestSample r;
  r.timestamp = s.timestamp;
  r.user_profile.assign(s.profile, s.profile + s.n_prof);
  r.history.resize(static_cast<size_t>(s.n_hist));
  for (int i = 0; i < s.n_hist; ++i) {
    ItemEvent& e = r.history[static_cast<size_t>(i)];
    e.item_id = s.hist_item[i];
    e.action_type = static_cast<ActionType>(s.hist_action[i]);
    e.timestamp = s.hist_ts[i];
    e.scene_id = s.hist_scene[i];
  }
  r.candidates.resize(static_cast<size_t>(s.n_cand));
  for (int c = 0; c < s.n_cand; ++c) r.candidates[static_cast<size_t>(c)].item_id = s.cand_item[c];
  return r;
}

}  // namespace

struct RefModel {
  OrModelCfg cfg;
  std::unique_ptr<Tokenizer> tok;
  std::vector<std::unique_ptr<AttentionLayer>> attn;
  std::map<std::string, Mat> spec;  // spec-only parameters (norm gains, FFN, head)

  Parameter* find(const std::string& name) {
    for (Parameter* p : tok->params())
      if (p->name == name) return p;
    for (auto& a : attn)
      for (Parameter* p : a->params())
        if (p->name == name) return p;
    return nullptr;
  }
  const Mat& P(const std::string& name) const {
    auto it = spec.find(name);
    if (it == spec.end()) throw ConfigError("ref model: parameter " + name + " not set");
    return it->second;
  }
};

struct RefGrads {
  std::map<std::string, Mat> g;
};

namespace {

// SwishGLU FFN: down(swish(x W_gate) * (x W_up)), no biases.
Mat swishglu(const Mat& x, const Mat& wg, const Mat& wu, const Mat& wd) {
  Mat g = x * wg;
  Mat u = x * wu;
  Mat z = g.unaryExpr([](double v) { return swish(v); }).cwiseProduct(u);
  return z * wd;
}

// Pre-norm residual block stack over a query-pruned stream, every
// reference operator called as the reference defines it.
void model_forward(const RefModel& m, const OrSample& s, double* probs, double* logits) {
  const OrModelCfg& c = m.cfg;
  TokenizerCache tc;
  TokenSequence seq = m.tok->tokenize_sample(sample_of(s), tc);
  Mat x = seq.tokens;
  std::vector<Role> roles = seq.roles;
  std::vector<int> pos = seq.position_ids;
  const int d = c.model_dim;
  for (int l = 0; l < c.layers; ++l) {
    const std::string L = std::to_string(l);
    const std::vector<int> qrows = retained_rows(roles, c.keep[l], c.keep_specials != 0);  // mask.cpp:132
    MaskSpec spec;
    spec.l_q = static_cast<int>(qrows.size());
    spec.l_kv = static_cast<int>(x.rows());
    spec.local_window = c.local_window;
    spec.full_suffix = c.full_suffix;
    const Mat mask = build_mask(spec, roles, pos, qrows);  // mask.cpp:14
    RmsNormCache n1;
    const Mat xn = rmsnorm_forward(x, m.P("block." + L + ".attn_norm"), n1);
    AttentionCache ac;
    const Mat a = m.attn[static_cast<size_t>(l)]->forward(xn, qrows, mask, pos, ac);  // attention.cpp:71
    Mat xr(spec.l_q, d);
    std::vector<Role> nroles(qrows.size());
    std::vector<int> npos(qrows.size());
    for (size_t i = 0; i < qrows.size(); ++i) {
      xr.row(static_cast<Eigen::Index>(i)) = x.row(qrows[i]) + a.row(static_cast<Eigen::Index>(i));
      nroles[i] = roles[static_cast<size_t>(qrows[i])];
      npos[i] = pos[static_cast<size_t>(qrows[i])];
    }
    RmsNormCache n2;
    const Mat xf = rmsnorm_forward(xr, m.P("block." + L + ".ffn_norm"), n2);
    xr += swishglu(xf, m.P("ffn." + L + ".w_gate"), m.P("ffn." + L + ".w_up"), m.P("ffn." + L + ".w_down"));
    x = xr;
    roles = nroles;
    pos = npos;
  }
  // final RMSNorm + ranking head on the candidate rows, in candidate order
  std::vector<int> crows;
  for (size_t i = 0; i < roles.size(); ++i)
    if (roles[i] == Role::kCand) crows.push_back(static_cast<int>(i));
  Mat xc(static_cast<Eigen::Index>(crows.size()), d);
  for (size_t i = 0; i < crows.size(); ++i) xc.row(static_cast<Eigen::Index>(i)) = x.row(crows[i]);
  RmsNormCache nf;
  const Mat xh = rmsnorm_forward(xc, m.P("final_norm.gain"), nf);
  Mat hid = xh * m.P("head.w1");
  hid.rowwise() += m.P("head.b1").row(0);
  hid = hid.unaryExpr([](double v) { return std::max(0.0, v); });
  Mat lo = hid * m.P("head.w2");
  lo.rowwise() += m.P("head.b2").row(0);
  for (Eigen::Index i = 0; i < lo.rows(); ++i)
    for (int j = 0; j < 3; ++j) {
      if (logits) logits[i * 3 + j] = lo(i, j);
      probs[i * 3 + j] = sigmoid(lo(i, j));
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- integer rules
int ref_time_bucket(int64_t delta_seconds, int n_buckets) { return time_bucket(delta_seconds, n_buckets); }

int ref_build_mask(int l_q, int l_kv, int local_window, int full_suffix, const int* roles, const int* pos,
                   const int* query_rows, uint8_t* visible, int64_t* visible_count) {
  return guarded([&] {
    MaskSpec spec;
    spec.l_q = l_q;
    spec.l_kv = l_kv;
    spec.local_window = local_window;
    spec.full_suffix = full_suffix;
    const std::vector<Role> r = roles_of(roles, l_kv);
    const std::vector<int> p(pos, pos + l_kv);
    const Mat mask = query_rows ? build_mask(spec, r, p, std::vector<int>(query_rows, query_rows + l_q))
                                : build_mask(spec, r, p);
    for (int i = 0; i < l_q; ++i)
      for (int j = 0; j < l_kv; ++j) visible[static_cast<size_t>(i) * l_kv + j] = mask(i, j) == 0.0 ? 1 : 0;
    if (visible_count) *visible_count = mask_visible_count(mask);
  });
}

int ref_geometric_schedule(int prefix_len, int depth, int target, int* keep) {
  return guarded([&] {
    const PruneSchedule s = make_geometric_schedule(prefix_len, depth, target);
    s.validate();
    std::copy(s.keep.begin(), s.keep.end(), keep);
  });
}

int ref_full_schedule(int prefix_len, int depth, int* keep) {
  return guarded([&] {
    const PruneSchedule s = make_full_schedule(prefix_len, depth);
    std::copy(s.keep.begin(), s.keep.end(), keep);
  });
}

int ref_retained_rows(const int* roles, int n, int keep, int keep_specials, int* out, int* n_out) {
  return guarded([&] {
    const std::vector<int> r = retained_rows(roles_of(roles, n), keep, keep_specials != 0);
    std::copy(r.begin(), r.end(), out);
    *n_out = static_cast<int>(r.size());
  });
}

int ref_prune_queries(const double* x, int rows, int cols, int n, double* out) {
  return guarded([&] { to_rows(prune_queries(from_rows(x, rows, cols), n), out); });
}

// ---------------------------------------------------------------- numeric operators
int ref_rmsnorm_forward(const double* x, int rows, int cols, const double* gain, double* y, double* inv_rms) {
  return guarded([&] {
    RmsNormCache c;
    to_rows(rmsnorm_forward(from_rows(x, rows, cols), from_rows(gain, 1, cols), c), y);
    if (inv_rms)
      for (int r = 0; r < rows; ++r) inv_rms[r] = c.inv_rms(r);
  });
}

int ref_rmsnorm_backward(const double* dy, const double* x, int rows, int cols, const double* gain,
                         double* dgain_accum, double* dx) {
  return guarded([&] {
    RmsNormCache c;
    const Mat g = from_rows(gain, 1, cols);
    rmsnorm_forward(from_rows(x, rows, cols), g, c);
    Mat dg = from_rows(dgain_accum, 1, cols);
    to_rows(rmsnorm_backward(from_rows(dy, rows, cols), c, g, dg), dx);
    to_rows(dg, dgain_accum);
  });
}

int ref_rope_apply(const double* x, int rows, int dim, const int* pos, double theta, int inverse, double* out) {
  return guarded([&] {
    to_rows(rope_apply(from_rows(x, rows, dim), std::vector<int>(pos, pos + rows), theta, inverse != 0), out);
  });
}

#define REF_ATTN(S, SUF)                                                                                        \
  int ref_dense_attention_##SUF(const S* q, const S* k, const S* v, const S* mask, int l_q, int l_kv, int dk,   \
                                int dv, S* out) {                                                               \
    return guarded([&] {                                                                                        \
      using MT = MatT<S>;                                                                                       \
      auto mk = [](const S* p, int r, int c) {                                                                  \
        MT m(r, c);                                                                                             \
        std::memcpy(m.data(), p, sizeof(S) * static_cast<size_t>(r) * c);                                     \
        return m;                                                                                               \
      };                                                                                                        \
      const MT o = dense_masked_attention<S>(mk(q, l_q, dk), mk(k, l_kv, dk), mk(v, l_kv, dv),                  \
                                             mk(mask, l_q, l_kv));                                              \
      std::memcpy(out, o.data(), sizeof(S) * static_cast<size_t>(l_q) * dv);                                   \
    });                                                                                                         \
  }                                                                                                             \
  int ref_blockwise_attention_##SUF(const S* q, const S* k, const S* v, const S* mask, int l_q, int l_kv,       \
                                    int dk, int dv, int block, S* out, int64_t* skipped, int64_t* total) {      \
    return guarded([&] {                                                                                        \
      using MT = MatT<S>;                                                                                       \
      auto mk = [](const S* p, int r, int c) {                                                                  \
        MT m(r, c);                                                                                             \
        std::memcpy(m.data(), p, sizeof(S) * static_cast<size_t>(r) * c);                                     \
        return m;                                                                                               \
      };                                                                                                        \
      const auto res = blockwise_masked_attention<S>(mk(q, l_q, dk), mk(k, l_kv, dk), mk(v, l_kv, dv),          \
                                                     mk(mask, l_q, l_kv), block);                               \
      std::memcpy(out, res.output.data(), sizeof(S) * static_cast<size_t>(l_q) * dv);                          \
      *skipped = res.skipped_blocks;                                                                            \
      *total = res.total_blocks;                                                                                \
    });                                                                                                         \
  }
REF_ATTN(double, f64)
REF_ATTN(float, f32)
#undef REF_ATTN

// ---------------------------------------------------------------- model objects
int ref_model_create(const OrModelCfg* c, RefModel** out) {
  return guarded([&] {
    auto m = std::make_unique<RefModel>();
    m->cfg = *c;
    TokenizerConfig tc;
    tc.model_dim = c->model_dim;
    tc.item_dim = c->item_dim;
    tc.action_dim = c->action_dim;
    tc.scene_dim = c->scene_dim;
    tc.time_dim = c->time_dim;
    tc.profile_dim = c->profile_dim;
    tc.n_items = c->n_items;
    tc.n_actions = c->n_actions;
    tc.n_scenes = c->n_scenes;
    tc.n_time_buckets = c->n_time_buckets;
    tc.profile_vocab.assign(c->profile_vocab, c->profile_vocab + c->n_profile_fields);
    tc.special_tokens = c->special_tokens != 0;
    m->tok = std::make_unique<Tokenizer>(tc);
    AttentionSettings as;
    as.model_dim = c->model_dim;
    as.heads = c->heads;
    as.qknorm = c->qknorm != 0;
    as.gate = c->gate != 0;
    as.rope_theta = c->rope_theta;
    for (int l = 0; l < c->layers; ++l) m->attn.push_back(std::make_unique<AttentionLayer>(as, l));
    *out = m.release();
  });
}

void ref_model_destroy(RefModel* m) { delete m; }

int ref_model_set_param(RefModel* m, const char* name, const double* data, int rows, int cols) {
  return guarded([&] {
    Parameter* p = m->find(name);
    if (p) {
      if (p->value.rows() != rows || p->value.cols() != cols)
        throw ConfigError(std::string("ref model: shape mismatch for ") + name);
      p->value = from_rows(data, rows, cols);
    } else {
      m->spec[name] = from_rows(data, rows, cols);
    }
  });
}

int ref_set_frozen(RefModel* m, const char* name, int frozen) {
  return guarded([&] {
    Parameter* p = m->find(name);
    if (!p) throw ConfigError(std::string("ref model: no reference parameter ") + name);
    p->frozen = frozen != 0;
  });
}

int ref_tokenize(const RefModel* m, const OrSample* s, double* tokens, int* pos, int* roles, int* cand_index,
                 int* hist_time, int* out_len) {
  return guarded([&] {
    TokenizerCache tc;
    const TokenSequence seq = m->tok->tokenize_sample(sample_of(*s), tc);
    if (tokens) to_rows(seq.tokens, tokens);
    for (int i = 0; i < seq.length(); ++i) {
      if (pos) pos[i] = seq.position_ids[static_cast<size_t>(i)];
      if (roles) roles[i] = static_cast<int>(seq.roles[static_cast<size_t>(i)]);
      if (cand_index) cand_index[i] = seq.candidate_index[static_cast<size_t>(i)];
    }
    if (hist_time) std::copy(tc.hist_time.begin(), tc.hist_time.end(), hist_time);
    if (out_len) *out_len = seq.length();
  });
}

int ref_tokenize_clicks(const RefModel* m, const OrSample* s, double* tokens, int* hist_time) {
  return guarded([&] {
    const RequestSample r = sample_of(*s);
    TokenizerCache tc;
    const TokenSequence seq = m->tok->tokenize_click_sequence(r.history, tc);
    if (tokens) to_rows(seq.tokens, tokens);
    if (hist_time) std::copy(tc.hist_time.begin(), tc.hist_time.end(), hist_time);
  });
}

// Tokenizer::backward (tokenizer.cpp:286-354) of the sample's tokenization for dL/dtokens
// [L, d]; gradients by reference parameter name (frozen tables get none, :289-349).
int ref_tokenizer_backward(RefModel* m, const OrSample* s, const double* dtokens, RefGrads** out) {
  return guarded([&] {
    TokenizerCache tc;
    const TokenSequence seq = m->tok->tokenize_sample(sample_of(*s), tc);
    const ParamRefs ps = m->tok->params();
    GradBuffer gb(ps);
    const ParamIndex ix(ps);
    m->tok->backward(from_rows(dtokens, seq.length(), m->cfg.model_dim), tc, gb, ix);
    auto g = std::make_unique<RefGrads>();
    for (size_t i = 0; i < ps.size(); ++i) g->g[ps[i]->name] = gb[i];
    *out = g.release();
  });
}

static Mat mask_of(const double* mask, const uint8_t* visible, int l_q, int l_in) {
  if (mask) return from_rows(mask, l_q, l_in);
  Mat mk(l_q, l_in);
  for (int i = 0; i < l_q; ++i)
    for (int j = 0; j < l_in; ++j)
      mk(i, j) = visible[static_cast<size_t>(i) * l_in + j] ? 0.0 : -std::numeric_limits<double>::infinity();
  return mk;
}

int ref_attention_forward(const RefModel* m, int layer, const double* xn, int l_in, const int* query_rows, int l_q,
                          const uint8_t* visible, const int* pos, double* out) {
  return guarded([&] {
    if (layer < 0 || layer >= m->cfg.layers) throw ConfigError("ref: layer out of range");
    AttentionCache ac;
    const Mat o = m->attn[static_cast<size_t>(layer)]->forward(
        from_rows(xn, l_in, m->cfg.model_dim), std::vector<int>(query_rows, query_rows + l_q),
        mask_of(nullptr, visible, l_q, l_in), std::vector<int>(pos, pos + l_in), ac);
    to_rows(o, out);
  });
}

// AttentionLayer::backward (attention.cpp:134-202, compiled with ref_fixups.hpp): d(xn) and
// the layer's parameter gradients by name.
int ref_attention_backward(RefModel* m, int layer, const double* xn, int l_in, const int* query_rows, int l_q,
                           const uint8_t* visible, const int* pos, const double* dout, double* dxn, RefGrads** out) {
  return guarded([&] {
    if (layer < 0 || layer >= m->cfg.layers) throw ConfigError("ref: layer out of range");
    AttentionLayer& A = *m->attn[static_cast<size_t>(layer)];
    AttentionCache ac;
    A.forward(from_rows(xn, l_in, m->cfg.model_dim), std::vector<int>(query_rows, query_rows + l_q),
              mask_of(nullptr, visible, l_q, l_in), std::vector<int>(pos, pos + l_in), ac);
    const ParamRefs ps = A.params();
    GradBuffer gb(ps);
    const ParamIndex ix(ps);
    to_rows(A.backward(from_rows(dout, l_q, m->cfg.model_dim), ac, gb, ix), dxn);
    auto g = std::make_unique<RefGrads>();
    for (size_t i = 0; i < ps.size(); ++i) g->g[ps[i]->name] = gb[i];
    *out = g.release();
  });
}

int ref_grads_get(const RefGrads* g, const char* name, double* out, int* rows, int* cols) {
  return guarded([&] {
    auto it = g->g.find(name);
    if (it == g->g.end()) throw ConfigError(std::string("ref: no gradient for ") + name);
    if (rows) *rows = static_cast<int>(it->second.rows());
    if (cols) *cols = static_cast<int>(it->second.cols());
    if (out) to_rows(it->second, out);
  });
}

void ref_grads_destroy(RefGrads* g) { delete g; }

int ref_model_forward(const RefModel* m, const OrSample* s, double* probs, double* logits) {
  return guarded([&] { model_forward(*m, *s, probs, logits); });
}

}  // extern "C"
