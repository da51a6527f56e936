// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY -- CPU oracle for the SORT hot path (see sort_oracle.h).
//
// fp64 restatement of the reference algorithm, written from its semantics
// (no Eigen: the reference's Eigen dependency is absent in this image, so the
// matrix kernels below are plain loops). Each function cites the reference
// file:line it follows; paths are relative to /root/reference.
// Parity: pinned only against SPEC.md known-answer examples and SURVEY.md
// derived counts (tests/test_oracle_kat.py) -- "parity unpinned" at the
// Eigen GEMM boundary, as DESIGN.md states.

#include "sort_oracle.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct RuntimeFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
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

constexpr double kRmsEps = 1e-6;  // norm.hpp:8

// ------------------------------------------------------------------ matrices
struct M {
  int r = 0, c = 0;
  std::vector<double> a;
  M() = default;
  M(int rows, int cols) : r(rows), c(cols), a(static_cast<size_t>(rows) * cols, 0.0) {}
  double* row(int i) { return a.data() + static_cast<size_t>(i) * c; }
  const double* row(int i) const { return a.data() + static_cast<size_t>(i) * c; }
  double& operator()(int i, int j) { return a[static_cast<size_t>(i) * c + j]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(i) * c + j]; }
};

// C[M,N] = A[M,K] * B[K,N], row-major, i-k-j order (inner loop contiguous).
void matmul(const double* A, const double* B, double* C, int Mr, int K, int N) {
  std::fill(C, C + static_cast<size_t>(Mr) * N, 0.0);
  constexpr int KB = 128;
  for (int k0 = 0; k0 < K; k0 += KB) {
    const int k1 = std::min(K, k0 + KB);
    for (int i = 0; i < Mr; ++i) {
      double* c = C + static_cast<size_t>(i) * N;
      const double* a = A + static_cast<size_t>(i) * K;
      for (int k = k0; k < k1; ++k) {
        const double av = a[k];
        const double* b = B + static_cast<size_t>(k) * N;
        for (int j = 0; j < N; ++j) c[j] += av * b[j];
      }
    }
  }
}
M matmul(const M& A, const M& B) {
  M C(A.r, B.c);
  matmul(A.a.data(), B.a.data(), C.a.data(), A.r, A.c, B.c);
  return C;
}
M transpose(const M& A) {
  M T(A.c, A.r);
  for (int i = 0; i < A.r; ++i)
    for (int j = 0; j < A.c; ++j) T(j, i) = A(i, j);
  return T;
}
M cols_of(const M& A, int c0, int n) {
  M out(A.r, n);
  for (int i = 0; i < A.r; ++i) std::memcpy(out.row(i), A.row(i) + c0, sizeof(double) * n);
  return out;
}

double sigmoid(double x) {  // common.hpp:29-35
  if (x >= 0.0) return 1.0 / (1.0 + std::exp(-x));
  const double e = std::exp(x);
  return e / (1.0 + e);
}
double swish(double x) { return x * sigmoid(x); }  // common.hpp:37

// rmsnorm_forward (norm.hpp:17-29): y = x / sqrt(mean(x^2) + eps) * gain.
void rmsnorm_rows(const double* x, int rows, int cols, const double* gain, double* y,
                  double* inv_out) {
  for (int r = 0; r < rows; ++r) {
    const double* xr = x + static_cast<size_t>(r) * cols;
    double ss = 0.0;
    for (int j = 0; j < cols; ++j) ss += xr[j] * xr[j];
    const double inv = 1.0 / std::sqrt(ss / static_cast<double>(cols) + kRmsEps);
    if (inv_out) inv_out[r] = inv;
    double* yr = y + static_cast<size_t>(r) * cols;
    for (int j = 0; j < cols; ++j) yr[j] = xr[j] * inv * gain[j];
  }
}
M rmsnorm(const M& x, const double* gain) {
  M y(x.r, x.c);
  rmsnorm_rows(x.a.data(), x.r, x.c, gain, y.a.data(), nullptr);
  return y;
}

// rope_apply (rope.hpp:13-40): interleaved pairs (2j, 2j+1), freq_j = theta^(-2j/dim).
void rope_rows(const double* x, int rows, int dim, const int* pos, double theta, bool inverse,
               double* out) {
  if (dim % 2 != 0) throw ConfigError("rope_apply: head dim must be even");
  const int np = dim / 2;
  std::vector<double> freq(np);
  for (int j = 0; j < np; ++j)
    freq[j] = std::pow(theta, -2.0 * static_cast<double>(j) / static_cast<double>(dim));
  for (int r = 0; r < rows; ++r) {
    const double p = static_cast<double>(pos[r]);
    const double* xr = x + static_cast<size_t>(r) * dim;
    double* o = out + static_cast<size_t>(r) * dim;
    for (int j = 0; j < np; ++j) {
      const double ang = (inverse ? -p : p) * freq[j];
      const double cs = std::cos(ang), sn = std::sin(ang);
      const double x0 = xr[2 * j], x1 = xr[2 * j + 1];
      o[2 * j] = cs * x0 - sn * x1;
      o[2 * j + 1] = sn * x0 + cs * x1;
    }
  }
}

// time_bucket (tokenizer.cpp:36-40).
int time_bucket(int64_t delta, int nb) {
  const int64_t d = std::max<int64_t>(delta, 0);
  const int b = static_cast<int>(std::floor(std::log2(1.0 + static_cast<double>(d))));
  return std::min(b, nb - 1);
}

// build_mask (mask.cpp:14-76); visible[r*l_kv + c] = 1 where the reference writes 0.0.
void build_mask(int l_q, int l_kv, int W, int F, const int* roles, const int* pos,
                const int* query_rows, uint8_t* vis) {
  if (l_q < 1 || l_kv < l_q) throw ConfigError("MaskSpec: need 1 <= l_q <= l_kv");
  if (W != -1 && W < 1) throw ConfigError("MaskSpec: local_window must be >= 1 or -1 (unbounded)");
  if (F < 0) throw ConfigError("MaskSpec: full_suffix must be >= 0");
  // Prefix length = first candidate's position id, else one past the max position (:28-44).
  int prefix_positions = 0;
  bool has_cand = false;
  for (int i = 0; i < l_kv; ++i) {
    if (roles[i] == OR_ROLE_CAND) {
      prefix_positions = pos[i];
      has_cand = true;
      break;
    }
  }
  if (!has_cand)
    for (int i = 0; i < l_kv; ++i) prefix_positions = std::max(prefix_positions, pos[i] + 1);

  std::memset(vis, 0, static_cast<size_t>(l_q) * l_kv);
  for (int r = 0; r < l_q; ++r) {
    const int qi = query_rows ? query_rows[r] : (l_kv - l_q) + r;  // suffix overload :78-85
    if (qi < 0 || qi >= l_kv) throw ConfigError("build_mask: query row out of range");
    const bool q_cand = roles[qi] == OR_ROLE_CAND;
    const int q_pos = pos[qi];
    const bool windowed = !q_cand && W != -1 && q_pos < prefix_positions - F;  // :52-53
    bool any = false;
    uint8_t* vr = vis + static_cast<size_t>(r) * l_kv;
    for (int c = 0; c <= qi && c < l_kv; ++c) {  // causal by kv index (:55)
      const bool k_cand = roles[c] == OR_ROLE_CAND;
      if (q_cand) {
        if (k_cand && c != qi) continue;  // candidate diagonal (:57-60)
      } else if (k_cand) {
        continue;  // (:61-62)
      } else if (windowed) {
        const int k_pos = pos[c];
        if (k_pos < q_pos - W + 1 || k_pos > q_pos) continue;  // (:63-66)
      }
      vr[c] = 1;
      any = true;
    }
    if (!any) throw ConfigError("build_mask: query row " + std::to_string(r) + " has no visible key");
  }
}

// retained_rows (mask.cpp:132-154).
std::vector<int> retained_rows(const std::vector<int>& roles, int keep, bool keep_specials) {
  int non_cand = 0;
  for (int r : roles) non_cand += (r != OR_ROLE_CAND) ? 1 : 0;
  const int kept = std::min(keep, non_cand);
  const int drop = non_cand - kept;
  std::vector<int> out;
  int seen = 0;
  for (size_t i = 0; i < roles.size(); ++i) {
    if (roles[i] == OR_ROLE_CAND) {
      out.push_back(static_cast<int>(i));
      continue;
    }
    const bool in_suffix = seen >= drop;
    ++seen;
    const bool special = roles[i] == OR_ROLE_BOS || roles[i] == OR_ROLE_SEP;
    if (in_suffix || (keep_specials && special)) out.push_back(static_cast<int>(i));
  }
  return out;
}

// make_geometric_schedule (mask.cpp:97-117).
std::vector<int> geometric_schedule(int prefix_len, int depth, int target) {
  if (depth < 1) throw ConfigError("make_geometric_schedule: depth must be >= 1");
  if (prefix_len < 1) prefix_len = 1;
  const int final_keep = std::min(target, prefix_len);
  std::vector<int> keep(depth);
  if (depth == 1) {
    keep[0] = final_keep;
    return keep;
  }
  const double ratio = static_cast<double>(final_keep) / static_cast<double>(prefix_len);
  int prev = prefix_len;
  for (int l = 0; l < depth; ++l) {
    const double t = static_cast<double>(l) / static_cast<double>(depth - 1);
    int k = static_cast<int>(std::lround(prefix_len * std::pow(ratio, t)));
    k = std::clamp(k, final_keep, prev);
    keep[l] = k;
    prev = k;
  }
  return keep;
}

// dense_masked_attention<Scalar> (block_attention.hpp:29-52).
template <class S>
void dense_attention(const S* q, const S* k, const S* v, const S* mask, int lq, int lkv, int dk,
                     int dv, S* out) {
  const S scale = S(1) / std::sqrt(static_cast<S>(dk));
  std::vector<S> s(lkv);
  for (int r = 0; r < lq; ++r) {
    S m = -std::numeric_limits<S>::infinity();
    for (int c = 0; c < lkv; ++c) {
      S acc = 0;
      for (int j = 0; j < dk; ++j) acc += q[static_cast<size_t>(r) * dk + j] * k[static_cast<size_t>(c) * dk + j];
      s[c] = acc * scale + mask[static_cast<size_t>(r) * lkv + c];
      m = std::max(m, s[c]);
    }
    if (!(m > -std::numeric_limits<S>::infinity()))
      throw std::invalid_argument("dense_masked_attention: fully masked query row");
    S denom = 0;
    for (int c = 0; c < lkv; ++c) {
      s[c] = std::exp(s[c] - m);
      denom += s[c];
    }
    S* o = out + static_cast<size_t>(r) * dv;
    for (int j = 0; j < dv; ++j) o[j] = 0;
    for (int c = 0; c < lkv; ++c) {
      const S p = s[c] / denom;
      for (int j = 0; j < dv; ++j) o[j] += p * v[static_cast<size_t>(c) * dv + j];
    }
  }
}

// blockwise_masked_attention<Scalar> (block_attention.hpp:54-134).
template <class S>
void blockwise_attention(const S* q, const S* k, const S* v, const S* mask, int lq, int lkv,
                         int dk, int dv, int B, S* out, int64_t* skipped, int64_t* total) {
  if (B < 1) throw std::invalid_argument("blockwise_masked_attention: block >= 1");
  const S ninf = -std::numeric_limits<S>::infinity();
  const S scale = S(1) / std::sqrt(static_cast<S>(dk));
  *skipped = 0;
  *total = 0;
  std::vector<S> row_max, row_sum, acc, s, p;
  for (int q0 = 0; q0 < lq; q0 += B) {
    const int qn = std::min(B, lq - q0);
    row_max.assign(qn, ninf);
    row_sum.assign(qn, 0);
    acc.assign(static_cast<size_t>(qn) * dv, 0);
    for (int k0 = 0; k0 < lkv; k0 += B) {
      const int kn = std::min(B, lkv - k0);
      ++*total;
      bool any = false;  // mask preload + validation (:86-99)
      for (int r = 0; r < qn && !any; ++r)
        for (int c = 0; c < kn; ++c)
          if (mask[static_cast<size_t>(q0 + r) * lkv + k0 + c] == S(0)) {
            any = true;
            break;
          }
      if (!any) {
        ++*skipped;
        continue;
      }
      s.assign(static_cast<size_t>(qn) * kn, 0);
      p.assign(static_cast<size_t>(qn) * kn, 0);
      for (int r = 0; r < qn; ++r)
        for (int c = 0; c < kn; ++c) {
          S a = 0;
          for (int j = 0; j < dk; ++j)
            a += q[static_cast<size_t>(q0 + r) * dk + j] * k[static_cast<size_t>(k0 + c) * dk + j];
          s[static_cast<size_t>(r) * kn + c] = a * scale + mask[static_cast<size_t>(q0 + r) * lkv + k0 + c];
        }
      for (int r = 0; r < qn; ++r) {  // online softmax (:104-122)
        S tmax = ninf;
        for (int c = 0; c < kn; ++c) tmax = std::max(tmax, s[static_cast<size_t>(r) * kn + c]);
        if (!(tmax > ninf)) continue;  // p row stays zero
        const S nmax = std::max(row_max[r], tmax);
        const S corr = row_max[r] > ninf ? std::exp(row_max[r] - nmax) : S(0);
        row_sum[r] *= corr;
        for (int j = 0; j < dv; ++j) acc[static_cast<size_t>(r) * dv + j] *= corr;
        S psum = 0;
        for (int c = 0; c < kn; ++c) {
          const S sv = s[static_cast<size_t>(r) * kn + c];
          const S pv = sv > ninf ? std::exp(sv - nmax) : S(0);
          p[static_cast<size_t>(r) * kn + c] = pv;
          psum += pv;
        }
        row_sum[r] += psum;
        row_max[r] = nmax;
      }
      for (int r = 0; r < qn; ++r)  // acc += p V (:123)
        for (int c = 0; c < kn; ++c) {
          const S pv = p[static_cast<size_t>(r) * kn + c];
          if (pv == S(0)) continue;
          for (int j = 0; j < dv; ++j)
            acc[static_cast<size_t>(r) * dv + j] += pv * v[static_cast<size_t>(k0 + c) * dv + j];
        }
    }
    for (int r = 0; r < qn; ++r) {  // normalise (:126-131)
      if (!(row_sum[r] > S(0)))
        throw std::invalid_argument("blockwise_masked_attention: fully masked query row");
      for (int j = 0; j < dv; ++j)
        out[static_cast<size_t>(q0 + r) * dv + j] = acc[static_cast<size_t>(r) * dv + j] / row_sum[r];
    }
  }
}

}  // namespace

// ====================================================================== model
struct OrModel {
  OrModelCfg cfg;
  int d = 0, dk = 0, m = 0, dh = 0;
  std::map<std::string, M> p;
  bool item_trainable = false;  // Parameter::frozen of the item table (params.hpp:18), inverted

  const M& P(const std::string& name) const {
    auto it = p.find(name);
    if (it == p.end()) throw ConfigError("oracle: missing parameter " + name);
    return it->second;
  }
  int hist_width() const {
    return cfg.item_dim + cfg.action_dim + cfg.scene_dim + cfg.time_dim;  // tokenizer.hpp:46-48
  }
};

namespace {

void check_id(int id, int vocab, const char* what) {  // tokenizer.cpp:14-19
  if (id < 0 || id >= vocab)
    throw ConfigError(std::string("tokenizer: ") + what + " id " + std::to_string(id) +
                      " outside vocabulary of size " + std::to_string(vocab));
}

struct Seq {
  M tokens;
  std::vector<int> pos, roles, cand_index, hist_time;
};

// Tokenizer::tokenize_sample (tokenizer.cpp:144-238).
Seq tokenize(const OrModel& mdl, const OrSample& s) {
  const OrModelCfg& c = mdl.cfg;
  if (s.n_cand <= 0) throw ConfigError("tokenizer: sample has zero candidates");
  if (s.n_prof != c.n_profile_fields)
    throw ConfigError("tokenizer: profile has " + std::to_string(s.n_prof) + " fields, expected " +
                      std::to_string(c.n_profile_fields));
  const bool st = c.special_tokens != 0;
  const int nh = s.n_hist, np = s.n_prof, nc = s.n_cand;
  const int total = (st ? 3 : 0) + nh + np + nc;
  const int d = mdl.d;
  Seq q;
  q.tokens = M(total, d);
  q.pos.assign(total, 0);
  q.roles.assign(total, 0);
  q.cand_index.assign(total, -1);
  q.hist_time.assign(nh, 0);

  const M& special = mdl.P("tok.special");
  int row = 0;
  auto put_special = [&](int srow, int role) {
    std::memcpy(q.tokens.row(row), special.row(srow), sizeof(double) * d);
    q.roles[row] = role;
    ++row;
  };
  if (st) put_special(0, OR_ROLE_BOS);

  // History group: gather item|action|scene|time rows (history_concat_row, :95-112).
  const M& it = mdl.P("tok.item_table");
  const M& at = mdl.P("tok.action_table");
  const M& sc = mdl.P("tok.scene_table");
  const M& tt = mdl.P("tok.time_table");
  const int hw = mdl.hist_width();
  M hcat(nh, hw);
  std::vector<int> hrows(nh);
  for (int i = 0; i < nh; ++i) {
    check_id(s.hist_item[i], c.n_items, "item");
    check_id(s.hist_action[i], c.n_actions, "action");
    check_id(s.hist_scene[i], c.n_scenes, "scene");
    const int tb = time_bucket(s.timestamp - s.hist_ts[i], c.n_time_buckets);
    double* o = hcat.row(i);
    std::memcpy(o, it.row(s.hist_item[i]), sizeof(double) * c.item_dim);
    o += c.item_dim;
    std::memcpy(o, at.row(s.hist_action[i]), sizeof(double) * c.action_dim);
    o += c.action_dim;
    std::memcpy(o, sc.row(s.hist_scene[i]), sizeof(double) * c.scene_dim);
    o += c.scene_dim;
    std::memcpy(o, tt.row(tb), sizeof(double) * c.time_dim);
    q.hist_time[i] = tb;
    hrows[i] = row;
    q.roles[row] = OR_ROLE_HIST;
    ++row;
  }
  if (st) put_special(1, OR_ROLE_SEP);

  M pcat(np, c.profile_dim);
  std::vector<int> prows(np);
  for (int f = 0; f < np; ++f) {
    const int v = s.profile[f];
    check_id(v, c.profile_vocab[f], "profile");
    const M& tab = mdl.P("tok.profile_table." + std::to_string(f));
    std::memcpy(pcat.row(f), tab.row(v), sizeof(double) * c.profile_dim);
    prows[f] = row;
    q.roles[row] = OR_ROLE_PROF;
    ++row;
  }
  if (st) put_special(2, OR_ROLE_SEP);

  M ccat(nc, c.item_dim);
  std::vector<int> crows(nc);
  for (int j = 0; j < nc; ++j) {
    check_id(s.cand_item[j], c.n_items, "item");
    std::memcpy(ccat.row(j), it.row(s.cand_item[j]), sizeof(double) * c.item_dim);
    crows[j] = row;
    q.roles[row] = OR_ROLE_CAND;
    q.cand_index[row] = j;
    ++row;
  }

  // emit_group (:219-232): concat * W + b -> RMSNorm(gain) -> scatter into the sequence.
  auto emit = [&](const M& cat, const std::vector<int>& rows, const char* w, const char* b,
                  const char* g) {
    if (cat.r == 0) return;
    M proj = matmul(cat, mdl.P(w));
    const M& bias = mdl.P(b);
    for (int i = 0; i < proj.r; ++i)
      for (int j = 0; j < d; ++j) proj(i, j) += bias(0, j);
    M y = rmsnorm(proj, mdl.P(g).row(0));
    for (int i = 0; i < y.r; ++i) std::memcpy(q.tokens.row(rows[i]), y.row(i), sizeof(double) * d);
  };
  emit(hcat, hrows, "tok.w_hist", "tok.b_hist", "tok.g_hist");
  emit(pcat, prows, "tok.w_prof", "tok.b_prof", "tok.g_prof");
  emit(ccat, crows, "tok.w_cand", "tok.b_cand", "tok.g_cand");

  const int prefix = total - nc;  // :234-236
  for (int i = 0; i < prefix; ++i) q.pos[i] = i;
  for (int i = prefix; i < total; ++i) q.pos[i] = prefix;
  return q;
}

// AttentionLayer::forward (attention.cpp:71-132).
M attention_forward(const OrModel& mdl, int layer, const M& xn, const std::vector<int>& qrows,
                    const uint8_t* vis, const std::vector<int>& pos) {
  const int d = mdl.d, h = mdl.cfg.heads, dk = mdl.dk;
  const int lq = static_cast<int>(qrows.size());
  const int lkv = xn.r;
  if (xn.c != d) throw RuntimeFailure("attention: input width mismatch");
  const std::string base = "attn." + std::to_string(layer) + ".";
  M xq(lq, d);
  std::vector<int> pos_q(lq);
  for (int i = 0; i < lq; ++i) {
    std::memcpy(xq.row(i), xn.row(qrows[i]), sizeof(double) * d);  // gather_rows (:10-16)
    pos_q[i] = pos[qrows[i]];
  }
  M q_raw = matmul(xq, mdl.P(base + "wq"));
  M k_raw = matmul(xn, mdl.P(base + "wk"));
  M v = matmul(xn, mdl.P(base + "wv"));
  const double scale = 1.0 / std::sqrt(static_cast<double>(dk));
  M out_pre(lq, d);
  std::vector<double> logits(static_cast<size_t>(lq) * lkv);
  for (int i = 0; i < h; ++i) {
    M qh = cols_of(q_raw, i * dk, dk), kh = cols_of(k_raw, i * dk, dk);
    if (mdl.cfg.qknorm) {  // per-head RMSNorm before RoPE (:111-114)
      qh = rmsnorm(qh, mdl.P(base + "qk_gain_q").row(i));
      kh = rmsnorm(kh, mdl.P(base + "qk_gain_k").row(i));
    }
    M qr(lq, dk), kr(lkv, dk);
    rope_rows(qh.a.data(), lq, dk, pos_q.data(), mdl.cfg.rope_theta, false, qr.a.data());
    rope_rows(kh.a.data(), lkv, dk, pos.data(), mdl.cfg.rope_theta, false, kr.a.data());
    M krT = transpose(kr);
    matmul(qr.a.data(), krT.a.data(), logits.data(), lq, dk, lkv);
    // logits*scale + mask, then masked_softmax (:19-30, :118-119)
    M vh = cols_of(v, i * dk, dk);
    for (int r = 0; r < lq; ++r) {
      double* lr = logits.data() + static_cast<size_t>(r) * lkv;
      const uint8_t* vr = vis + static_cast<size_t>(r) * lkv;
      double mx = -std::numeric_limits<double>::infinity();
      for (int c = 0; c < lkv; ++c) {
        lr[c] = vr[c] ? lr[c] * scale : -std::numeric_limits<double>::infinity();
        mx = std::max(mx, lr[c]);
      }
      if (!(mx > -std::numeric_limits<double>::infinity()))
        throw RuntimeFailure("attention: fully masked query row");
      double sum = 0.0;
      for (int c = 0; c < lkv; ++c) {
        lr[c] = std::exp(lr[c] - mx);
        sum += lr[c];
      }
      double* o = out_pre.row(r) + i * dk;
      for (int c = 0; c < lkv; ++c) {
        const double a = lr[c] / sum;
        if (a == 0.0) continue;
        const double* vv = vh.row(c);
        for (int j = 0; j < dk; ++j) o[j] += a * vv[j];
      }
    }
  }
  M hcat = out_pre;
  if (mdl.cfg.gate) {  // sigmoid gate on the gathered rows (:124-127)
    M g = matmul(xq, mdl.P(base + "wg"));
    for (size_t t = 0; t < hcat.a.size(); ++t) hcat.a[t] = sigmoid(g.a[t]) * out_pre.a[t];
  }
  return matmul(hcat, mdl.P(base + "wo"));  // (:131)
}

// swishglu_ffn: down(swish(x Wg) * (x Wu)).
M swishglu(const M& x, const M& wg, const M& wu, const M& wd) {
  M g = matmul(x, wg), u = matmul(x, wu);
  for (size_t t = 0; t < g.a.size(); ++t) g.a[t] = swish(g.a[t]) * u.a[t];
  return matmul(g, wd);
}

struct LayerTrace {
  std::vector<int> qrows;
  int64_t visible = 0;
};

// ====================================================================== MoE FFN
// DeepSeek-style mixture of SwishGLU experts: sigmoid gate
// scores, selection by score + bias (auxiliary-loss-free balancing; the bias never enters the
// combine weights, SPEC.md "Bias-neutral combine"), ties broken toward the lower expert index,
// weights renormalised over the selected experts, one always-on shared expert (weight 1).
struct MoeRouting {
  std::vector<int> sel;        // [rows, k], descending biased score
  std::vector<double> w;       // [rows, k]
  std::vector<double> margin;  // [rows]
};

void moe_route(const M& x, const M& router, const double* bias, int k, const int* forced, MoeRouting& R) {
  const int rows = x.r, E = router.c;
  if (k < 1 || k > E) throw ConfigError("moe: need 1 <= k <= E");
  R.sel.assign(static_cast<size_t>(rows) * k, 0);
  R.w.assign(static_cast<size_t>(rows) * k, 0.0);
  R.margin.assign(rows, 0.0);
  M logit = matmul(x, router);
  std::vector<double> sc(E), bs(E);
  std::vector<int> order(E);
  for (int i = 0; i < rows; ++i) {
    for (int e = 0; e < E; ++e) {
      sc[e] = sigmoid(logit(i, e));
      bs[e] = sc[e] + (bias ? bias[e] : 0.0);
      order[e] = e;
    }
    // descending biased score, lower index first on ties (a stable sort of the identity order)
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return bs[a] > bs[b]; });
    R.margin[i] = k < E ? bs[order[k - 1]] - bs[order[k]] : std::numeric_limits<double>::infinity();
    double tot = 0.0;
    for (int j = 0; j < k; ++j) {
      int e = order[j];
      if (forced) {
        e = forced[static_cast<size_t>(i) * k + j];
        if (e < 0 || e >= E) throw ConfigError("moe: forced expert id out of range");
      }
      R.sel[static_cast<size_t>(i) * k + j] = e;
      tot += sc[e];
    }
    for (int j = 0; j < k; ++j) {
      const int e = R.sel[static_cast<size_t>(i) * k + j];
      R.w[static_cast<size_t>(i) * k + j] = sc[e] / tot;
    }
  }
}

// Rows of x routed to each expert run through that expert's SwishGLU and are added back with
// their combine weight; the shared expert sees every row with weight 1.
M moe_ffn(const M& x, const M& router, const double* bias, int k, int shared,
          const std::vector<const M*>& wg, const std::vector<const M*>& wu, const std::vector<const M*>& wd,
          const int* forced, MoeRouting& R) {
  const int rows = x.r, d = x.c, E = router.c;
  moe_route(x, router, bias, k, forced, R);
  M out(rows, d);
  for (int e = 0; e < E + shared; ++e) {
    std::vector<int> rid;
    std::vector<double> rw;
    for (int i = 0; i < rows; ++i) {
      if (e == E) {
        rid.push_back(i);
        rw.push_back(1.0);
        continue;
      }
      for (int j = 0; j < k; ++j)
        if (R.sel[static_cast<size_t>(i) * k + j] == e) {
          rid.push_back(i);
          rw.push_back(R.w[static_cast<size_t>(i) * k + j]);
        }
    }
    if (rid.empty()) continue;
    M xs(static_cast<int>(rid.size()), d);
    for (size_t t = 0; t < rid.size(); ++t) std::memcpy(xs.row(static_cast<int>(t)), x.row(rid[t]), sizeof(double) * d);
    M y = swishglu(xs, *wg[e], *wu[e], *wd[e]);
    for (size_t t = 0; t < rid.size(); ++t) {
      double* o = out.row(rid[t]);
      const double* yr = y.row(static_cast<int>(t));
      for (int c = 0; c < d; ++c) o[c] += rw[t] * yr[c];
    }
  }
  return out;
}

M model_moe_ffn(const OrModel& mdl, int l, const M& xf, const int* forced, MoeRouting& R) {
  const OrModelCfg& c = mdl.cfg;
  const std::string F = "ffn." + std::to_string(l) + ".";
  std::vector<const M*> wg, wu, wd;
  for (int e = 0; e < c.moe_experts + c.moe_shared; ++e) {
    const std::string X = e < c.moe_experts ? F + "expert." + std::to_string(e) + "." : F + "shared.";
    wg.push_back(&mdl.P(X + "w_gate"));
    wu.push_back(&mdl.P(X + "w_up"));
    wd.push_back(&mdl.P(X + "w_down"));
  }
  const M& b = mdl.P(F + "router_bias");
  return moe_ffn(xf, mdl.P(F + "router"), b.row(0), c.moe_topk, c.moe_shared, wg, wu, wd, forced, R);
}

// MoE routing control of one model_forward (see oracle_model_forward_moe).
struct MoeCtl {
  const int* forced = nullptr;
  int* out_sel = nullptr;
  double* out_margin = nullptr;
};

// model_forward: pre-norm residual blocks over a shrinking
// residual stream, final RMSNorm, ranking head on candidate rows.
// The block stack over x with its roles/positions, shrinking by query pruning.
void blocks_forward(const OrModel& mdl, M& x, std::vector<int>& roles, std::vector<int>& pos,
                    std::vector<LayerTrace>* trace, MoeCtl* moe) {
  size_t moe_off = 0, moe_row_off = 0;
  const OrModelCfg& c = mdl.cfg;
  const int d = mdl.d;
  for (int l = 0; l < c.layers; ++l) {
    const std::string L = std::to_string(l);
    std::vector<int> qrows = retained_rows(roles, c.keep[l], c.keep_specials != 0);
    const int lq = static_cast<int>(qrows.size()), lkv = x.r;
    std::vector<uint8_t> vis(static_cast<size_t>(lq) * lkv);
    build_mask(lq, lkv, c.local_window, c.full_suffix, roles.data(), pos.data(), qrows.data(),
               vis.data());
    if (trace) {
      LayerTrace t;
      t.qrows = qrows;
      for (uint8_t v : vis) t.visible += v;
      trace->push_back(std::move(t));
    }
    M xn = rmsnorm(x, mdl.P("block." + L + ".attn_norm").row(0));
    M a = attention_forward(mdl, l, xn, qrows, vis.data(), pos);
    M xr(lq, d);
    std::vector<int> nroles(lq), npos(lq);
    for (int i = 0; i < lq; ++i) {
      const double* src = x.row(qrows[i]);
      double* dst = xr.row(i);
      const double* ar = a.row(i);
      for (int j = 0; j < d; ++j) dst[j] = src[j] + ar[j];  // residual on P(x, L_out)
      nroles[i] = roles[qrows[i]];
      npos[i] = pos[qrows[i]];
    }
    M xf = rmsnorm(xr, mdl.P("block." + L + ".ffn_norm").row(0));
    M f;
    if (c.moe_experts > 0) {  // DeepSeek-style MoE FFN
      MoeRouting R;
      f = model_moe_ffn(mdl, l, xf, moe && moe->forced ? moe->forced + moe_off : nullptr, R);
      if (moe && moe->out_sel) std::copy(R.sel.begin(), R.sel.end(), moe->out_sel + moe_off);
      if (moe && moe->out_margin) std::copy(R.margin.begin(), R.margin.end(), moe->out_margin + moe_row_off);
      moe_off += R.sel.size();
      moe_row_off += R.margin.size();
    } else {
      f = swishglu(xf, mdl.P("ffn." + L + ".w_gate"), mdl.P("ffn." + L + ".w_up"), mdl.P("ffn." + L + ".w_down"));
    }
    for (size_t t = 0; t < xr.a.size(); ++t) xr.a[t] += f.a[t];
    x = std::move(xr);
    roles = std::move(nroles);
    pos = std::move(npos);
  }
}

void model_forward(const OrModel& mdl, const OrSample& s, double* probs, double* logits_out,
                   std::vector<LayerTrace>* trace, MoeCtl* moe = nullptr) {
  Seq q = tokenize(mdl, s);
  M x = q.tokens;
  std::vector<int> roles = q.roles, pos = q.pos;
  const int d = mdl.d;
  blocks_forward(mdl, x, roles, pos, trace, moe);
  // Final RMSNorm + head on candidate rows, candidates in order.
  std::vector<int> crows;
  for (int i = 0; i < x.r; ++i)
    if (roles[i] == OR_ROLE_CAND) crows.push_back(i);
  M xc(static_cast<int>(crows.size()), d);
  for (size_t i = 0; i < crows.size(); ++i)
    std::memcpy(xc.row(static_cast<int>(i)), x.row(crows[i]), sizeof(double) * d);
  M xh = rmsnorm(xc, mdl.P("final_norm.gain").row(0));
  M hid = matmul(xh, mdl.P("head.w1"));
  const M& b1 = mdl.P("head.b1");
  for (int i = 0; i < hid.r; ++i)
    for (int j = 0; j < hid.c; ++j) hid(i, j) = std::max(0.0, hid(i, j) + b1(0, j));
  M lo = matmul(hid, mdl.P("head.w2"));
  const M& b2 = mdl.P("head.b2");
  for (int i = 0; i < lo.r; ++i)
    for (int j = 0; j < 3; ++j) {
      const double z = lo(i, j) + b2(0, j);
      if (logits_out) logits_out[i * 3 + j] = z;
      probs[i * 3 + j] = sigmoid(z);
    }
}

// ====================================================================== pre-training
// Tokenizer::tokenize_click_sequence (tokenizer.cpp:240-284): [BOS; one token per click],
// history projection of item|action|scene|time where the time slice is the bucket of the gap
// to the previous click (the first click gets the bucket of INT64_MAX/4, :262-270);
// positions 0..n, roles BOS + HIST.
Seq tokenize_clicks(const OrModel& mdl, const OrSample& s) {
  const OrModelCfg& c = mdl.cfg;
  const int n = s.n_hist, d = mdl.d, total = 1 + n;
  Seq q;
  q.tokens = M(total, d);
  q.pos.resize(total);
  q.roles.assign(total, OR_ROLE_HIST);
  q.cand_index.assign(total, -1);
  q.hist_time.assign(n, 0);
  std::memcpy(q.tokens.row(0), mdl.P("tok.special").row(0), sizeof(double) * d);
  q.roles[0] = OR_ROLE_BOS;
  const M& it = mdl.P("tok.item_table");
  const M& at = mdl.P("tok.action_table");
  const M& sc = mdl.P("tok.scene_table");
  const M& tt = mdl.P("tok.time_table");
  M cat(n, mdl.hist_width());
  for (int i = 0; i < n; ++i) {
    check_id(s.hist_item[i], c.n_items, "item");
    check_id(s.hist_action[i], c.n_actions, "action");
    check_id(s.hist_scene[i], c.n_scenes, "scene");
    const int64_t gap = i == 0 ? std::numeric_limits<int64_t>::max() / 4 : s.hist_ts[i] - s.hist_ts[i - 1];
    const int tb = time_bucket(gap, c.n_time_buckets);
    double* o = cat.row(i);
    std::memcpy(o, it.row(s.hist_item[i]), sizeof(double) * c.item_dim);
    o += c.item_dim;
    std::memcpy(o, at.row(s.hist_action[i]), sizeof(double) * c.action_dim);
    o += c.action_dim;
    std::memcpy(o, sc.row(s.hist_scene[i]), sizeof(double) * c.scene_dim);
    o += c.scene_dim;
    std::memcpy(o, tt.row(tb), sizeof(double) * c.time_dim);
    q.hist_time[i] = tb;
  }
  if (n > 0) {
    M proj = matmul(cat, mdl.P("tok.w_hist"));
    const M& b = mdl.P("tok.b_hist");
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < d; ++j) proj(i, j) += b(0, j);
    M y = rmsnorm(proj, mdl.P("tok.g_hist").row(0));
    for (int i = 0; i < n; ++i) std::memcpy(q.tokens.row(1 + i), y.row(i), sizeof(double) * d);
  }
  for (int i = 0; i < total; ++i) q.pos[i] = i;
  return q;
}

// pretrain_forward: the block stack as a causal LM over [BOS; clicks]
// (no candidates, local window and pruning off by config), final RMSNorm,
// projection to the item-embedding width (pretrain.proj [d, item_dim], the builder's bridge
// between d and the table) and tied logits z_t[v] = h_t . item_table[v]. Position t (< n)
// predicts click t: lse[t] = log sum_v exp z_t[v], target[t] = z_t[click_t].
void pretrain_forward(const OrModel& mdl, const OrSample& s, double* lse, double* target, double* hproj) {
  if (s.n_hist < 2) throw ConfigError("pretrain: sequences shorter than 2 clicks are skipped");
  Seq q = tokenize_clicks(mdl, s);
  M x = q.tokens;
  std::vector<int> roles = q.roles, pos = q.pos;
  blocks_forward(mdl, x, roles, pos, nullptr, nullptr);
  if (x.r != s.n_hist + 1) throw ConfigError("pretrain: query pruning must be off");
  M h = matmul(rmsnorm(x, mdl.P("final_norm.gain").row(0)), mdl.P("pretrain.proj"));
  const M& E = mdl.P("tok.item_table");
  const int V = E.r, k = E.c;
  if (h.c != k) throw ConfigError("pretrain: projection width must equal item_dim");
  std::vector<double> z(V);
  for (int t = 0; t < s.n_hist; ++t) {
    double mx = -std::numeric_limits<double>::infinity();
    for (int v = 0; v < V; ++v) {
      double a = 0.0;
      for (int j = 0; j < k; ++j) a += h(t, j) * E(v, j);
      z[v] = a;
      mx = std::max(mx, a);
    }
    double se = 0.0;
    for (int v = 0; v < V; ++v) se += std::exp(z[v] - mx);
    lse[t] = mx + std::log(se);
    target[t] = z[s.hist_item[t]];
  }
  if (hproj) std::memcpy(hproj, h.a.data(), sizeof(double) * h.r * h.c);
}

// ====================================================================== backward
// Training-mode backward of the whole scoring path for one request, fp64: head -> final
// RMSNorm -> blocks (FFN, pre-norms, residuals, pruning scatter) -> attention layers
// (AttentionLayer::backward, attention.cpp:134-202, with the intended math: the gate
// path's d(xq) added to the query path, QKNorm gains indexed per head) -> dtokens.
// rmsnorm_backward follows norm.hpp:32-45.
using Grads = std::map<std::string, M>;

M& grad_of(Grads& g, const OrModel& mdl, const std::string& name) {
  auto it = g.find(name);
  if (it == g.end()) {
    const M& p = mdl.P(name);
    it = g.emplace(name, M(p.r, p.c)).first;
  }
  return it->second;
}

// y = x * inv * gain (per row); returns dx, accumulates dgain (norm.hpp:32-45)
M rmsnorm_backward(const M& dy, const M& x, const double* gain, double* dgain) {
  M dx(x.r, x.c);
  for (int r = 0; r < x.r; ++r) {
    const double* xr = x.row(r);
    double ss = 0.0;
    for (int j = 0; j < x.c; ++j) ss += xr[j] * xr[j];
    const double inv = 1.0 / std::sqrt(ss / static_cast<double>(x.c) + kRmsEps);
    double proj = 0.0;
    for (int j = 0; j < x.c; ++j) {
      const double xh = xr[j] * inv;
      dgain[j] += dy(r, j) * xh;
      proj += dy(r, j) * gain[j] * xh;
    }
    proj /= static_cast<double>(x.c);
    for (int j = 0; j < x.c; ++j) dx(r, j) = (dy(r, j) * gain[j] - proj * xr[j] * inv) * inv;
  }
  return dx;
}

M matmul_tn(const M& A, const M& B) { return matmul(transpose(A), B); }  // A^T B
M matmul_nt(const M& A, const M& B) { return matmul(A, transpose(B)); }  // A B^T
void add_into(M& a, const M& b) {
  for (size_t t = 0; t < a.a.size(); ++t) a.a[t] += b.a[t];
}

// AttentionLayer::backward (attention.cpp:134-202): returns d(xn) [l_kv, d].
M attention_backward(const OrModel& mdl, int layer, const M& xn, const std::vector<int>& qrows,
                     const uint8_t* vis, const std::vector<int>& pos, const M& dout, Grads& G) {
  const int d = mdl.d, h = mdl.cfg.heads, dk = mdl.dk;
  const int lq = static_cast<int>(qrows.size()), lkv = xn.r;
  const std::string base = "attn." + std::to_string(layer) + ".";
  const double scale = 1.0 / std::sqrt(static_cast<double>(dk));
  // ---- forward with caches (attention.cpp:71-132)
  M xq(lq, d);
  std::vector<int> pos_q(lq);
  for (int i = 0; i < lq; ++i) {
    std::memcpy(xq.row(i), xn.row(qrows[i]), sizeof(double) * d);
    pos_q[i] = pos[qrows[i]];
  }
  const M& Wq = mdl.P(base + "wq");
  const M& Wk = mdl.P(base + "wk");
  const M& Wv = mdl.P(base + "wv");
  const M& Wo = mdl.P(base + "wo");
  M q_raw = matmul(xq, Wq), k_raw = matmul(xn, Wk), v = matmul(xn, Wv);
  M out_pre(lq, d);
  std::vector<M> attn(h), q_rot(h), k_rot(h);
  for (int i = 0; i < h; ++i) {
    M qh = cols_of(q_raw, i * dk, dk), kh = cols_of(k_raw, i * dk, dk);
    if (mdl.cfg.qknorm) {
      qh = rmsnorm(qh, mdl.P(base + "qk_gain_q").row(i));
      kh = rmsnorm(kh, mdl.P(base + "qk_gain_k").row(i));
    }
    q_rot[i] = M(lq, dk);
    k_rot[i] = M(lkv, dk);
    rope_rows(qh.a.data(), lq, dk, pos_q.data(), mdl.cfg.rope_theta, false, q_rot[i].a.data());
    rope_rows(kh.a.data(), lkv, dk, pos.data(), mdl.cfg.rope_theta, false, k_rot[i].a.data());
    M& a = attn[i] = M(lq, lkv);
    matmul(q_rot[i].a.data(), transpose(k_rot[i]).a.data(), a.a.data(), lq, dk, lkv);
    for (int r = 0; r < lq; ++r) {
      double* ar = a.row(r);
      const uint8_t* vr = vis + static_cast<size_t>(r) * lkv;
      double mx = -std::numeric_limits<double>::infinity();
      for (int c = 0; c < lkv; ++c) {
        ar[c] = vr[c] ? ar[c] * scale : -std::numeric_limits<double>::infinity();
        mx = std::max(mx, ar[c]);
      }
      double sum = 0.0;
      for (int c = 0; c < lkv; ++c) {
        ar[c] = vr[c] ? std::exp(ar[c] - mx) : 0.0;
        sum += ar[c];
      }
      for (int c = 0; c < lkv; ++c) ar[c] /= sum;
    }
    M oh = matmul(a, cols_of(v, i * dk, dk));
    for (int r = 0; r < lq; ++r) std::memcpy(out_pre.row(r) + i * dk, oh.row(r), sizeof(double) * dk);
  }
  M gsig(lq, d), hcat = out_pre;
  if (mdl.cfg.gate) {
    M graw = matmul(xq, mdl.P(base + "wg"));
    for (size_t t = 0; t < gsig.a.size(); ++t) {
      gsig.a[t] = sigmoid(graw.a[t]);
      hcat.a[t] = gsig.a[t] * out_pre.a[t];
    }
  }
  // ---- backward (attention.cpp:134-202)
  add_into(grad_of(G, mdl, base + "wo"), matmul_tn(hcat, dout));
  M dh = matmul_nt(dout, Wo);
  M dpre = dh, dxq(lq, d);
  if (mdl.cfg.gate) {
    M dgraw(lq, d);
    for (size_t t = 0; t < dh.a.size(); ++t) {
      dpre.a[t] = dh.a[t] * gsig.a[t];
      dgraw.a[t] = dh.a[t] * out_pre.a[t] * gsig.a[t] * (1.0 - gsig.a[t]);
    }
    add_into(grad_of(G, mdl, base + "wg"), matmul_tn(xq, dgraw));
    dxq = matmul_nt(dgraw, mdl.P(base + "wg"));
  }
  M dq_raw(lq, d), dk_raw(lkv, d), dv(lkv, d);
  for (int i = 0; i < h; ++i) {
    const M& a = attn[i];
    M dO = cols_of(dpre, i * dk, dk);
    M da = matmul_nt(dO, cols_of(v, i * dk, dk));
    M dvh = matmul_tn(a, dO);
    M ds(lq, lkv);
    for (int r = 0; r < lq; ++r) {
      double dot = 0.0;
      for (int c = 0; c < lkv; ++c) dot += da(r, c) * a(r, c);
      for (int c = 0; c < lkv; ++c) ds(r, c) = a(r, c) * (da(r, c) - dot);
    }
    M dq_rot = matmul(ds, k_rot[i]), dk_rot = matmul_tn(ds, q_rot[i]);
    for (double& t : dq_rot.a) t *= scale;
    for (double& t : dk_rot.a) t *= scale;
    M dq(lq, dk), dkk(lkv, dk);
    rope_rows(dq_rot.a.data(), lq, dk, pos_q.data(), mdl.cfg.rope_theta, true, dq.a.data());
    rope_rows(dk_rot.a.data(), lkv, dk, pos.data(), mdl.cfg.rope_theta, true, dkk.a.data());
    if (mdl.cfg.qknorm) {
      M& gq = grad_of(G, mdl, base + "qk_gain_q");
      M& gk = grad_of(G, mdl, base + "qk_gain_k");
      dq = rmsnorm_backward(dq, cols_of(q_raw, i * dk, dk), mdl.P(base + "qk_gain_q").row(i), gq.row(i));
      dkk = rmsnorm_backward(dkk, cols_of(k_raw, i * dk, dk), mdl.P(base + "qk_gain_k").row(i), gk.row(i));
    }
    for (int r = 0; r < lq; ++r) std::memcpy(dq_raw.row(r) + i * dk, dq.row(r), sizeof(double) * dk);
    for (int r = 0; r < lkv; ++r) {
      std::memcpy(dk_raw.row(r) + i * dk, dkk.row(r), sizeof(double) * dk);
      std::memcpy(dv.row(r) + i * dk, dvh.row(r), sizeof(double) * dk);
    }
  }
  add_into(grad_of(G, mdl, base + "wq"), matmul_tn(xq, dq_raw));
  add_into(grad_of(G, mdl, base + "wk"), matmul_tn(xn, dk_raw));
  add_into(grad_of(G, mdl, base + "wv"), matmul_tn(xn, dv));
  add_into(dxq, matmul_nt(dq_raw, Wq));
  M dxn = matmul_nt(dk_raw, Wk);
  add_into(dxn, matmul_nt(dv, Wv));
  for (int i = 0; i < lq; ++i)
    for (int j = 0; j < d; ++j) dxn(qrows[i], j) += dxq(i, j);
  return dxn;
}

// Tokenizer::backward (tokenizer.cpp:286-352) for one request: per group
// dproj = rmsnorm_backward(dtokens[group rows]) -> dW = concat^T dproj, db = colsum(dproj),
// d(concat) = dproj W^T scattered into the feature tables; special rows take dtokens raw.
// The item table is frozen by default (SPEC.md transfer+freeze; tokenizer.cpp:315-317,
// 346-352 skip frozen tables); with item_trainable its rows take the item columns of d(concat)
// of the history and candidate groups.
void tokenizer_backward(const OrModel& mdl, const OrSample& s, const M& dtok, Grads& G) {
  const OrModelCfg& c = mdl.cfg;
  const bool st = c.special_tokens != 0;
  const int nh = s.n_hist, np = s.n_prof, nc = s.n_cand, d = mdl.d;
  if (st) {
    M& gs = grad_of(G, mdl, "tok.special");
    const int srow[3] = {0, 1 + nh, 2 + nh + np};
    for (int k = 0; k < 3; ++k)
      for (int j = 0; j < d; ++j) gs(k, j) += dtok(srow[k], j);
  }
  auto group = [&](const M& cat, int row0, const char* w, const char* b, const char* g) -> M {
    const int n = cat.r;
    M dy(n, d);
    for (int i = 0; i < n; ++i) std::memcpy(dy.row(i), dtok.row(row0 + i), sizeof(double) * d);
    M proj = matmul(cat, mdl.P(w));
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < d; ++j) proj(i, j) += mdl.P(b)(0, j);
    M dproj = rmsnorm_backward(dy, proj, mdl.P(g).row(0), grad_of(G, mdl, g).row(0));
    add_into(grad_of(G, mdl, w), matmul_tn(cat, dproj));
    M& gb = grad_of(G, mdl, b);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < d; ++j) gb(0, j) += dproj(i, j);
    return matmul_nt(dproj, mdl.P(w));
  };
  const M& it = mdl.P("tok.item_table");
  if (nh > 0) {
    M hcat(nh, mdl.hist_width());
    for (int i = 0; i < nh; ++i) {
      double* o = hcat.row(i);
      std::memcpy(o, it.row(s.hist_item[i]), sizeof(double) * c.item_dim);
      std::memcpy(o + c.item_dim, mdl.P("tok.action_table").row(s.hist_action[i]), sizeof(double) * c.action_dim);
      std::memcpy(o + c.item_dim + c.action_dim, mdl.P("tok.scene_table").row(s.hist_scene[i]),
                  sizeof(double) * c.scene_dim);
      const int tb = time_bucket(s.timestamp - s.hist_ts[i], c.n_time_buckets);
      std::memcpy(o + c.item_dim + c.action_dim + c.scene_dim, mdl.P("tok.time_table").row(tb),
                  sizeof(double) * c.time_dim);
    }
    M dc = group(hcat, st ? 1 : 0, "tok.w_hist", "tok.b_hist", "tok.g_hist");
    M& ga = grad_of(G, mdl, "tok.action_table");
    M& gsn = grad_of(G, mdl, "tok.scene_table");
    M& gt = grad_of(G, mdl, "tok.time_table");
    for (int i = 0; i < nh; ++i) {
      const int tb = time_bucket(s.timestamp - s.hist_ts[i], c.n_time_buckets);
      if (mdl.item_trainable) {  // tokenizer.cpp:315-317
        M& gi = grad_of(G, mdl, "tok.item_table");
        for (int j = 0; j < c.item_dim; ++j) gi(s.hist_item[i], j) += dc(i, j);
      }
      for (int j = 0; j < c.action_dim; ++j) ga(s.hist_action[i], j) += dc(i, c.item_dim + j);
      for (int j = 0; j < c.scene_dim; ++j) gsn(s.hist_scene[i], j) += dc(i, c.item_dim + c.action_dim + j);
      for (int j = 0; j < c.time_dim; ++j) gt(tb, j) += dc(i, c.item_dim + c.action_dim + c.scene_dim + j);
    }
  }
  if (np > 0) {
    M pcat(np, c.profile_dim);
    for (int f = 0; f < np; ++f)
      std::memcpy(pcat.row(f), mdl.P("tok.profile_table." + std::to_string(f)).row(s.profile[f]),
                  sizeof(double) * c.profile_dim);
    M dc = group(pcat, (st ? 2 : 0) + nh, "tok.w_prof", "tok.b_prof", "tok.g_prof");
    for (int f = 0; f < np; ++f) {
      M& gp = grad_of(G, mdl, "tok.profile_table." + std::to_string(f));
      for (int j = 0; j < c.profile_dim; ++j) gp(s.profile[f], j) += dc(f, j);
    }
  }
  M ccat(nc, c.item_dim);
  for (int j = 0; j < nc; ++j) std::memcpy(ccat.row(j), it.row(s.cand_item[j]), sizeof(double) * c.item_dim);
  M dcc = group(ccat, (st ? 3 : 0) + nh + np, "tok.w_cand", "tok.b_cand", "tok.g_cand");
  if (mdl.item_trainable) {  // tokenizer.cpp:346-352
    M& gi = grad_of(G, mdl, "tok.item_table");
    for (int j = 0; j < nc; ++j)
      for (int k = 0; k < c.item_dim; ++k) gi(s.cand_item[j], k) += dcc(j, k);
  }
}

// Backward of model_forward for one request given dL/dlogits [n_cand, 3]; returns dtokens.
// Saved activations of one block for the backward.
struct BlockSaved {
  M x, xr;
  std::vector<int> qrows, roles, pos;
  std::vector<uint8_t> vis;
};

// blocks_forward with every block's input, residual and plan kept (x, roles, pos advance).
std::vector<BlockSaved> blocks_forward_saved(const OrModel& mdl, M& x, std::vector<int>& roles, std::vector<int>& pos) {
  const OrModelCfg& c = mdl.cfg;
  const int d = mdl.d;
  std::vector<BlockSaved> sv(c.layers);
  for (int l = 0; l < c.layers; ++l) {
    const std::string L = std::to_string(l);
    BlockSaved& S = sv[l];
    S.x = x;
    S.roles = roles;
    S.pos = pos;
    S.qrows = retained_rows(roles, c.keep[l], c.keep_specials != 0);
    const int lq = static_cast<int>(S.qrows.size()), lkv = x.r;
    S.vis.assign(static_cast<size_t>(lq) * lkv, 0);
    build_mask(lq, lkv, c.local_window, c.full_suffix, roles.data(), pos.data(), S.qrows.data(), S.vis.data());
    M xn = rmsnorm(x, mdl.P("block." + L + ".attn_norm").row(0));
    M a = attention_forward(mdl, l, xn, S.qrows, S.vis.data(), pos);
    M xr(lq, d);
    std::vector<int> nroles(lq), npos(lq);
    for (int i = 0; i < lq; ++i) {
      for (int j = 0; j < d; ++j) xr(i, j) = x(S.qrows[i], j) + a(i, j);
      nroles[i] = roles[S.qrows[i]];
      npos[i] = pos[S.qrows[i]];
    }
    S.xr = xr;
    M xf = rmsnorm(xr, mdl.P("block." + L + ".ffn_norm").row(0));
    M f = swishglu(xf, mdl.P("ffn." + L + ".w_gate"), mdl.P("ffn." + L + ".w_up"), mdl.P("ffn." + L + ".w_down"));
    add_into(xr, f);
    x = std::move(xr);
    roles = std::move(nroles);
    pos = std::move(npos);
  }
  return sv;
}

// The blocks in reverse given d(final residual stream); returns d(tokens).
M blocks_backward(const OrModel& mdl, const std::vector<BlockSaved>& sv, M dx, Grads& G) {
  const OrModelCfg& c = mdl.cfg;
  const int d = mdl.d;
  for (int l = c.layers - 1; l >= 0; --l) {
    const std::string L = std::to_string(l);
    const BlockSaved& S = sv[l];
    const int lq = static_cast<int>(S.qrows.size());
    // FFN: x_out = xr + down(swish(xf Wg) * (xf Wu)), xf = RMSN(xr)
    const double* gf = mdl.P("block." + L + ".ffn_norm").row(0);
    M xf = rmsnorm(S.xr, gf);
    const M& Wg = mdl.P("ffn." + L + ".w_gate");
    const M& Wu = mdl.P("ffn." + L + ".w_up");
    const M& Wd = mdl.P("ffn." + L + ".w_down");
    M gp = matmul(xf, Wg), up = matmul(xf, Wu), z(gp.r, gp.c);
    for (size_t t = 0; t < z.a.size(); ++t) z.a[t] = swish(gp.a[t]) * up.a[t];
    add_into(grad_of(G, mdl, "ffn." + L + ".w_down"), matmul_tn(z, dx));
    M dz2 = matmul_nt(dx, Wd), dgp(gp.r, gp.c), dup(gp.r, gp.c);
    for (size_t t = 0; t < z.a.size(); ++t) {
      const double sg = sigmoid(gp.a[t]);
      dup.a[t] = dz2.a[t] * gp.a[t] * sg;
      dgp.a[t] = dz2.a[t] * up.a[t] * sg * (1.0 + gp.a[t] * (1.0 - sg));
    }
    add_into(grad_of(G, mdl, "ffn." + L + ".w_gate"), matmul_tn(xf, dgp));
    add_into(grad_of(G, mdl, "ffn." + L + ".w_up"), matmul_tn(xf, dup));
    M dxf = matmul_nt(dgp, Wg);
    add_into(dxf, matmul_nt(dup, Wu));
    M dxr = dx;
    add_into(dxr, rmsnorm_backward(dxf, S.xr, gf, grad_of(G, mdl, "block." + L + ".ffn_norm").row(0)));
    // attention: xr = P(x, L_out) + Attn(RMSN(x))
    const double* ga = mdl.P("block." + L + ".attn_norm").row(0);
    M xn = rmsnorm(S.x, ga);
    M dxn = attention_backward(mdl, l, xn, S.qrows, S.vis.data(), S.pos, dxr, G);
    M dxin = rmsnorm_backward(dxn, S.x, ga, grad_of(G, mdl, "block." + L + ".attn_norm").row(0));
    for (int i = 0; i < lq; ++i)
      for (int j = 0; j < d; ++j) dxin(S.qrows[i], j) += dxr(i, j);
    dx = std::move(dxin);
  }
  return dx;
}

// Backward of model_forward for one request given dL/dlogits [n_cand, 3]; returns dtokens.
M model_backward(const OrModel& mdl, const OrSample& s, const double* dlogits, Grads& G) {
  if (mdl.cfg.moe_experts > 0) throw ConfigError("oracle: backward of the MoE FFN is not implemented");
  Seq q = tokenize(mdl, s);
  const int d = mdl.d;
  M x = q.tokens;
  std::vector<int> roles = q.roles, pos = q.pos;
  std::vector<BlockSaved> sv = blocks_forward_saved(mdl, x, roles, pos);
  // ---- head backward
  std::vector<int> crows;
  for (int i = 0; i < x.r; ++i)
    if (roles[i] == OR_ROLE_CAND) crows.push_back(i);
  const int nc = static_cast<int>(crows.size());
  M xc(nc, d);
  for (int i = 0; i < nc; ++i) std::memcpy(xc.row(i), x.row(crows[i]), sizeof(double) * d);
  const double* gfin = mdl.P("final_norm.gain").row(0);
  M xh = rmsnorm(xc, gfin);
  M hid = matmul(xh, mdl.P("head.w1"));
  const M& b1 = mdl.P("head.b1");
  for (int i = 0; i < hid.r; ++i)
    for (int j = 0; j < hid.c; ++j) hid(i, j) = std::max(0.0, hid(i, j) + b1(0, j));
  M dz(nc, 3);
  std::memcpy(dz.a.data(), dlogits, sizeof(double) * nc * 3);
  add_into(grad_of(G, mdl, "head.w2"), matmul_tn(hid, dz));
  M& gb2 = grad_of(G, mdl, "head.b2");
  for (int i = 0; i < nc; ++i)
    for (int j = 0; j < 3; ++j) gb2(0, j) += dz(i, j);
  M dhid = matmul_nt(dz, mdl.P("head.w2"));
  for (size_t t = 0; t < dhid.a.size(); ++t)
    if (hid.a[t] <= 0.0) dhid.a[t] = 0.0;  // ReLU (the subgradient 0 at 0)
  add_into(grad_of(G, mdl, "head.w1"), matmul_tn(xh, dhid));
  M& gb1 = grad_of(G, mdl, "head.b1");
  for (int i = 0; i < nc; ++i)
    for (int j = 0; j < dhid.c; ++j) gb1(0, j) += dhid(i, j);
  M dxh = matmul_nt(dhid, mdl.P("head.w1"));
  M dxc = rmsnorm_backward(dxh, xc, gfin, grad_of(G, mdl, "final_norm.gain").row(0));
  M dx(x.r, d);
  for (int i = 0; i < nc; ++i) std::memcpy(dx.row(crows[i]), dxc.row(i), sizeof(double) * d);
  dx = blocks_backward(mdl, sv, std::move(dx), G);
  tokenizer_backward(mdl, s, dx, G);
  return dx;
}

// Backward of the pre-training loss for one click sequence: loss contribution
// scale * sum_t CE_t (t < n, position t predicting click t) -> every gradient, the item table
// included twice (tied head: dE += dz^T h; input embedding: tokenize_click_sequence's history
// projection, tokenizer.cpp:240-284 / 315-317). Returns sum_t CE_t.
double pretrain_backward(const OrModel& mdl, const OrSample& s, double scale, Grads& G) {
  if (s.n_hist < 2) throw ConfigError("pretrain: sequences shorter than 2 clicks are skipped");
  const OrModelCfg& c = mdl.cfg;
  const int d = mdl.d, n = s.n_hist;
  Seq q = tokenize_clicks(mdl, s);
  M x = q.tokens;
  std::vector<int> roles = q.roles, pos = q.pos;
  std::vector<BlockSaved> sv = blocks_forward_saved(mdl, x, roles, pos);
  if (x.r != n + 1) throw ConfigError("pretrain: query pruning must be off");
  const double* gfin = mdl.P("final_norm.gain").row(0);
  M xh = rmsnorm(x, gfin);
  const M& W = mdl.P("pretrain.proj");
  M h = matmul(xh, W);
  const M& E = mdl.P("tok.item_table");
  const int V = E.r, k = E.c;
  M dh(h.r, k);
  M& gE = grad_of(G, mdl, "tok.item_table");
  double loss = 0.0;
  std::vector<double> z(V);
  for (int t = 0; t < n; ++t) {
    double mx = -std::numeric_limits<double>::infinity();
    for (int v = 0; v < V; ++v) {
      double a = 0.0;
      for (int j = 0; j < k; ++j) a += h(t, j) * E(v, j);
      z[v] = a;
      mx = std::max(mx, a);
    }
    double se = 0.0;
    for (int v = 0; v < V; ++v) se += std::exp(z[v] - mx);
    const double lse = mx + std::log(se);
    const int tg = s.hist_item[t];
    loss += lse - z[tg];
    for (int v = 0; v < V; ++v) {
      const double g = scale * (std::exp(z[v] - lse) - (v == tg ? 1.0 : 0.0));
      for (int j = 0; j < k; ++j) {
        dh(t, j) += g * E(v, j);
        gE(v, j) += g * h(t, j);
      }
    }
  }
  add_into(grad_of(G, mdl, "pretrain.proj"), matmul_tn(xh, dh));
  M dxh = matmul_nt(dh, W);
  M dx = rmsnorm_backward(dxh, x, gfin, grad_of(G, mdl, "final_norm.gain").row(0));
  dx = blocks_backward(mdl, sv, std::move(dx), G);
  // tokenize_click_sequence backward: BOS = special row 0, clicks = the history projection
  M& gs = grad_of(G, mdl, "tok.special");
  for (int j = 0; j < d; ++j) gs(0, j) += dx(0, j);
  M cat(n, mdl.hist_width());
  std::vector<int> tbs(n);
  for (int i = 0; i < n; ++i) {
    const int64_t gap = i == 0 ? std::numeric_limits<int64_t>::max() / 4 : s.hist_ts[i] - s.hist_ts[i - 1];
    tbs[i] = time_bucket(gap, c.n_time_buckets);
    double* o = cat.row(i);
    std::memcpy(o, E.row(s.hist_item[i]), sizeof(double) * c.item_dim);
    std::memcpy(o + c.item_dim, mdl.P("tok.action_table").row(s.hist_action[i]), sizeof(double) * c.action_dim);
    std::memcpy(o + c.item_dim + c.action_dim, mdl.P("tok.scene_table").row(s.hist_scene[i]),
                sizeof(double) * c.scene_dim);
    std::memcpy(o + c.item_dim + c.action_dim + c.scene_dim, mdl.P("tok.time_table").row(tbs[i]),
                sizeof(double) * c.time_dim);
  }
  M dy(n, d);
  for (int i = 0; i < n; ++i) std::memcpy(dy.row(i), dx.row(1 + i), sizeof(double) * d);
  M proj = matmul(cat, mdl.P("tok.w_hist"));
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < d; ++j) proj(i, j) += mdl.P("tok.b_hist")(0, j);
  M dproj = rmsnorm_backward(dy, proj, mdl.P("tok.g_hist").row(0), grad_of(G, mdl, "tok.g_hist").row(0));
  add_into(grad_of(G, mdl, "tok.w_hist"), matmul_tn(cat, dproj));
  M& gb = grad_of(G, mdl, "tok.b_hist");
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < d; ++j) gb(0, j) += dproj(i, j);
  M dc = matmul_nt(dproj, mdl.P("tok.w_hist"));
  M& ga = grad_of(G, mdl, "tok.action_table");
  M& gsn = grad_of(G, mdl, "tok.scene_table");
  M& gt = grad_of(G, mdl, "tok.time_table");
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < c.item_dim; ++j) gE(s.hist_item[i], j) += dc(i, j);
    for (int j = 0; j < c.action_dim; ++j) ga(s.hist_action[i], j) += dc(i, c.item_dim + j);
    for (int j = 0; j < c.scene_dim; ++j) gsn(s.hist_scene[i], j) += dc(i, c.item_dim + c.action_dim + j);
    for (int j = 0; j < c.time_dim; ++j) gt(tbs[i], j) += dc(i, c.item_dim + c.action_dim + c.scene_dim + j);
  }
  return loss;
}

}  // namespace

// ====================================================================== C API
extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

int oracle_time_bucket(int64_t delta_seconds, int n_buckets) {
  return time_bucket(delta_seconds, n_buckets);
}

int oracle_build_mask(int l_q, int l_kv, int local_window, int full_suffix, const int* roles,
                      const int* position_ids, const int* query_rows, uint8_t* out_visible) {
  return guarded([&] {
    build_mask(l_q, l_kv, local_window, full_suffix, roles, position_ids, query_rows, out_visible);
  });
}

int64_t oracle_mask_visible_count(const uint8_t* visible, int64_t n) {  // mask.cpp:87-95
  int64_t c = 0;
  for (int64_t i = 0; i < n; ++i) c += visible[i] ? 1 : 0;
  return c;
}

int oracle_geometric_schedule(int prefix_len, int depth, int target, int* out_keep) {
  return guarded([&] {
    std::vector<int> k = geometric_schedule(prefix_len, depth, target);
    std::copy(k.begin(), k.end(), out_keep);
  });
}

int oracle_full_schedule(int prefix_len, int depth, int* out_keep) {  // mask.cpp:119-123
  for (int i = 0; i < depth; ++i) out_keep[i] = std::max(prefix_len, 1);
  return 0;
}

int oracle_retained_rows(const int* roles, int n, int keep, int keep_specials, int* out_rows,
                         int* out_n) {
  std::vector<int> r(roles, roles + n);
  std::vector<int> o = retained_rows(r, keep, keep_specials != 0);
  std::copy(o.begin(), o.end(), out_rows);
  *out_n = static_cast<int>(o.size());
  return 0;
}

int oracle_prune_queries(const double* x, int rows, int cols, int n, double* out) {
  return guarded([&] {  // mask.cpp:125-130
    if (n < 1 || n > rows) throw ConfigError("prune_queries: n must be in [1, rows]");
    std::memcpy(out, x + static_cast<size_t>(rows - n) * cols, sizeof(double) * n * cols);
  });
}

int oracle_rmsnorm_forward(const double* x, int rows, int cols, const double* gain, double* y,
                           double* inv_rms) {
  rmsnorm_rows(x, rows, cols, gain, y, inv_rms);
  return 0;
}

// rmsnorm_backward (norm.hpp:32-45), with dgain accumulated into the row it belongs to.
int oracle_rmsnorm_backward(const double* dy, const double* x, const double* inv_rms, int rows,
                            int cols, const double* gain, double* dgain, double* dx) {
  for (int r = 0; r < rows; ++r) {
    const double inv = inv_rms[r];
    const double* xr = x + static_cast<size_t>(r) * cols;
    const double* dyr = dy + static_cast<size_t>(r) * cols;
    double proj = 0.0;
    for (int j = 0; j < cols; ++j) {
      const double xh = xr[j] * inv;
      dgain[j] += dyr[j] * xh;
      proj += dyr[j] * gain[j] * xh;
    }
    proj /= static_cast<double>(cols);
    double* o = dx + static_cast<size_t>(r) * cols;
    for (int j = 0; j < cols; ++j) o[j] = (dyr[j] * gain[j] - proj * xr[j] * inv) * inv;
  }
  return 0;
}

int oracle_rope_apply(const double* x, int rows, int dim, const int* position_ids, double theta,
                      int inverse, double* out) {
  return guarded([&] { rope_rows(x, rows, dim, position_ids, theta, inverse != 0, out); });
}

int oracle_dense_masked_attention_f64(const double* q, const double* k, const double* v,
                                      const double* mask, int l_q, int l_kv, int dk, int dv,
                                      double* out) {
  return guarded([&] { dense_attention<double>(q, k, v, mask, l_q, l_kv, dk, dv, out); });
}
int oracle_dense_masked_attention_f32(const float* q, const float* k, const float* v,
                                      const float* mask, int l_q, int l_kv, int dk, int dv,
                                      float* out) {
  return guarded([&] { dense_attention<float>(q, k, v, mask, l_q, l_kv, dk, dv, out); });
}
int oracle_blockwise_masked_attention_f64(const double* q, const double* k, const double* v,
                                          const double* mask, int l_q, int l_kv, int dk, int dv,
                                          int block, double* out, int64_t* skipped,
                                          int64_t* total) {
  return guarded([&] {
    blockwise_attention<double>(q, k, v, mask, l_q, l_kv, dk, dv, block, out, skipped, total);
  });
}
int oracle_blockwise_masked_attention_f32(const float* q, const float* k, const float* v,
                                          const float* mask, int l_q, int l_kv, int dk, int dv,
                                          int block, float* out, int64_t* skipped,
                                          int64_t* total) {
  return guarded([&] {
    blockwise_attention<float>(q, k, v, mask, l_q, l_kv, dk, dv, block, out, skipped, total);
  });
}

int oracle_swishglu(const double* x, int rows, int d, int m, const double* w_gate,
                    const double* w_up, const double* w_down, double* out) {
  M X(rows, d), G(d, m), U(d, m), D(m, d);
  std::memcpy(X.a.data(), x, sizeof(double) * rows * d);
  std::memcpy(G.a.data(), w_gate, sizeof(double) * d * m);
  std::memcpy(U.a.data(), w_up, sizeof(double) * d * m);
  std::memcpy(D.a.data(), w_down, sizeof(double) * m * d);
  M y = swishglu(X, G, U, D);
  std::memcpy(out, y.a.data(), sizeof(double) * rows * d);
  return 0;
}

int oracle_model_forward_moe(const OrModel* m, const OrSample* s, const int* forced_sel, double* probs,
                             double* logits, int* out_sel, double* out_margin) {
  return guarded([&] {
    MoeCtl ctl;
    ctl.forced = forced_sel;
    ctl.out_sel = out_sel;
    ctl.out_margin = out_margin;
    model_forward(*m, *s, probs, logits, nullptr, &ctl);
  });
}

int oracle_moe_route(const double* x, int rows, int d, int n_experts, int k, const double* router,
                     const double* bias, int* sel, double* w, double* margin) {
  return guarded([&] {
    M X(rows, d), Rt(d, n_experts);
    std::memcpy(X.a.data(), x, sizeof(double) * rows * d);
    std::memcpy(Rt.a.data(), router, sizeof(double) * d * n_experts);
    MoeRouting R;
    moe_route(X, Rt, bias, k, nullptr, R);
    std::copy(R.sel.begin(), R.sel.end(), sel);
    std::copy(R.w.begin(), R.w.end(), w);
    if (margin) std::copy(R.margin.begin(), R.margin.end(), margin);
  });
}

int oracle_moe_ffn(const double* x, int rows, int d, int m, int n_experts, int k, int shared,
                   const double* router, const double* bias, const double* w_gate, const double* w_up,
                   const double* w_down, const int* forced_sel, double* out, int* sel, double* w) {
  return guarded([&] {
    if (shared != 0 && shared != 1) throw ConfigError("moe: shared must be 0 or 1");
    M X(rows, d), Rt(d, n_experts);
    std::memcpy(X.a.data(), x, sizeof(double) * rows * d);
    std::memcpy(Rt.a.data(), router, sizeof(double) * d * n_experts);
    const int n = n_experts + shared;
    std::vector<M> G(n, M(d, m)), U(n, M(d, m)), D(n, M(m, d));
    std::vector<const M*> pg, pu, pd;
    for (int e = 0; e < n; ++e) {
      std::memcpy(G[e].a.data(), w_gate + static_cast<size_t>(e) * d * m, sizeof(double) * d * m);
      std::memcpy(U[e].a.data(), w_up + static_cast<size_t>(e) * d * m, sizeof(double) * d * m);
      std::memcpy(D[e].a.data(), w_down + static_cast<size_t>(e) * m * d, sizeof(double) * m * d);
      pg.push_back(&G[e]);
      pu.push_back(&U[e]);
      pd.push_back(&D[e]);
    }
    MoeRouting R;
    M y = moe_ffn(X, Rt, bias, k, shared, pg, pu, pd, forced_sel, R);
    std::memcpy(out, y.a.data(), sizeof(double) * rows * d);
    if (sel) std::copy(R.sel.begin(), R.sel.end(), sel);
    if (w) std::copy(R.w.begin(), R.w.end(), w);
  });
}

int oracle_moe_update_bias(const int64_t* load, int n_experts, double gamma, double* bias) {
  return guarded([&] {
    double mean = 0.0;
    for (int e = 0; e < n_experts; ++e) mean += static_cast<double>(load[e]);
    mean /= n_experts;
    for (int e = 0; e < n_experts; ++e) {
      const double dlt = static_cast<double>(load[e]) - mean;
      bias[e] -= gamma * (dlt > 0 ? 1.0 : (dlt < 0 ? -1.0 : 0.0));
    }
  });
}

int oracle_pretrain_forward(const OrModel* m, const OrSample* s, double* lse, double* target, double* hproj) {
  return guarded([&] { pretrain_forward(*m, *s, lse, target, hproj); });
}

int oracle_tokenize_clicks(const OrModel* m, const OrSample* s, double* tokens, int* hist_time) {
  return guarded([&] {
    Seq q = tokenize_clicks(*m, *s);
    std::memcpy(tokens, q.tokens.a.data(), sizeof(double) * q.tokens.a.size());
    if (hist_time) std::copy(q.hist_time.begin(), q.hist_time.end(), hist_time);
  });
}

int oracle_model_create(const OrModelCfg* cfg, OrModel** out) {
  return guarded([&] {
    auto* m = new OrModel;
    m->cfg = *cfg;
    m->d = cfg->model_dim;
    if (cfg->heads < 1 || m->d % cfg->heads != 0)
      throw ConfigError("attention: model_dim must be a positive multiple of heads");
    m->dk = m->d / cfg->heads;
    if (m->dk % 2 != 0) throw ConfigError("attention: head dim must be even for the rotary transform");
    m->m = cfg->ffn_dim;
    m->dh = cfg->head_hidden > 0 ? cfg->head_hidden : m->d;
    std::vector<int> keep(cfg->keep, cfg->keep + cfg->layers);
    for (size_t i = 0; i + 1 < keep.size(); ++i)  // PruneSchedule::validate (mask.hpp:51-60)
      if (keep[i + 1] > keep[i]) throw ConfigError("PruneSchedule: keep counts must be non-increasing");
    for (int k : keep)
      if (k < 1) throw ConfigError("PruneSchedule: keep counts must be >= 1");
    if (cfg->moe_experts < 0 ||
        (cfg->moe_experts > 0 && (cfg->moe_topk < 1 || cfg->moe_topk > cfg->moe_experts ||
                                  (cfg->moe_shared != 0 && cfg->moe_shared != 1) || cfg->moe_ffn_dim < 1)))
      throw ConfigError("moe: need 1 <= topk <= experts, shared in {0, 1}, expert ffn dim >= 1");
    *out = m;
  });
}

void oracle_model_destroy(OrModel* m) { delete m; }

int oracle_model_set_item_trainable(OrModel* m, int trainable) {
  if (!m) return 1;
  m->item_trainable = trainable != 0;
  return 0;
}

int oracle_model_set_param(OrModel* m, const char* name, const double* data, int rows, int cols) {
  return guarded([&] {
    M t(rows, cols);
    std::memcpy(t.a.data(), data, sizeof(double) * rows * cols);
    m->p[name] = std::move(t);
  });
}

int oracle_tokenize(const OrModel* m, const OrSample* s, double* tokens, int* position_ids,
                    int* roles, int* candidate_index, int* hist_time, int* out_len) {
  return guarded([&] {
    Seq q = tokenize(*m, *s);
    const int L = q.tokens.r;
    *out_len = L;
    if (tokens) std::memcpy(tokens, q.tokens.a.data(), sizeof(double) * L * m->d);
    if (position_ids) std::copy(q.pos.begin(), q.pos.end(), position_ids);
    if (roles) std::copy(q.roles.begin(), q.roles.end(), roles);
    if (candidate_index) std::copy(q.cand_index.begin(), q.cand_index.end(), candidate_index);
    if (hist_time) std::copy(q.hist_time.begin(), q.hist_time.end(), hist_time);
  });
}

int oracle_attention_forward(const OrModel* m, int layer, const double* xn, int l_in,
                             const int* query_rows, int l_q, const uint8_t* visible,
                             const int* position_ids, double* out) {
  return guarded([&] {
    M X(l_in, m->d);
    std::memcpy(X.a.data(), xn, sizeof(double) * l_in * m->d);
    std::vector<int> qr(query_rows, query_rows + l_q), pos(position_ids, position_ids + l_in);
    M y = attention_forward(*m, layer, X, qr, visible, pos);
    std::memcpy(out, y.a.data(), sizeof(double) * l_q * m->d);
  });
}

int oracle_model_forward(const OrModel* m, const OrSample* s, double* probs, double* logits) {
  return guarded([&] { model_forward(*m, *s, probs, logits, nullptr); });
}

int oracle_model_layer_meta(const OrModel* m, const OrSample* s, int* l_q, int64_t* visible,
                            int* query_rows_concat, int* total_rows) {
  return guarded([&] {
    std::vector<LayerTrace> tr;
    std::vector<double> probs(static_cast<size_t>(s->n_cand) * 3);
    model_forward(*m, *s, probs.data(), nullptr, &tr);
    int off = 0;
    for (size_t l = 0; l < tr.size(); ++l) {
      l_q[l] = static_cast<int>(tr[l].qrows.size());
      visible[l] = tr[l].visible;
      if (query_rows_concat) std::copy(tr[l].qrows.begin(), tr[l].qrows.end(), query_rows_concat + off);
      off += l_q[l];
    }
    *total_rows = off;
  });
}

int oracle_model_forward_batch(const OrModel* m, const OrSample* samples, int B, int threads,
                               double* probs) {
  std::vector<size_t> off(B + 1, 0);
  for (int b = 0; b < B; ++b) off[b + 1] = off[b] + static_cast<size_t>(samples[b].n_cand) * 3;
  std::atomic<int> next{0};
  std::atomic<int> status{0};
  std::string first_err;
  std::mutex mu;
  auto worker = [&] {
    for (;;) {
      const int b = next.fetch_add(1);
      if (b >= B) break;
      try {
        model_forward(*m, samples[b], probs + off[b], nullptr, nullptr);
      } catch (const ConfigError& e) {
        std::lock_guard<std::mutex> lk(mu);
        int z = 0;
        if (status.compare_exchange_strong(z, 1)) first_err = e.what();
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lk(mu);
        int z = 0;
        if (status.compare_exchange_strong(z, 2)) first_err = e.what();
      }
    }
  };
  threads = std::max(1, threads);
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  if (status.load() != 0) g_err = first_err;
  return status.load();
}


struct OrGrads {
  Grads g;
};

int oracle_model_backward(const OrModel* m, const OrSample* s, const double* dlogits,
                          double* dtokens, OrGrads** out) {
  return guarded([&] {
    auto* G = new OrGrads;
    try {
      M dx = model_backward(*m, *s, dlogits, G->g);
      if (dtokens) std::memcpy(dtokens, dx.a.data(), sizeof(double) * dx.a.size());
    } catch (...) {
      delete G;
      throw;
    }
    *out = G;
  });
}

int oracle_pretrain_backward(const OrModel* m, const OrSample* s, double scale, double* ce_sum, OrGrads** out) {
  return guarded([&] {
    auto* G = new OrGrads;
    try {
      const double l = pretrain_backward(*m, *s, scale, G->g);
      if (ce_sum) *ce_sum = l;
    } catch (...) {
      delete G;
      throw;
    }
    *out = G;
  });
}

int oracle_grads_get(const OrGrads* g, const char* name, double* out, int* rows, int* cols) {
  return guarded([&] {
    auto it = g->g.find(name);
    if (it == g->g.end()) {  // parameter not on the differentiated path: zero gradient
      if (rows) *rows = 0;
      if (cols) *cols = 0;
      return;
    }
    if (rows) *rows = it->second.r;
    if (cols) *cols = it->second.c;
    if (out) std::memcpy(out, it->second.a.data(), sizeof(double) * it->second.a.size());
  });
}

void oracle_grads_destroy(OrGrads* g) { delete g; }

int oracle_attention_backward(const OrModel* m, int layer, const double* xn, int l_in, const int* query_rows,
                              int l_q, const uint8_t* visible, const int* position_ids, const double* dout,
                              double* dxn, OrGrads** out) {
  return guarded([&] {
    if (layer < 0 || layer >= m->cfg.layers) throw ConfigError("attention: layer out of range");
    M x(l_in, m->d);
    std::memcpy(x.a.data(), xn, sizeof(double) * x.a.size());
    M dy(l_q, m->d);
    std::memcpy(dy.a.data(), dout, sizeof(double) * dy.a.size());
    auto* G = new OrGrads;
    try {
      M dx = attention_backward(*m, layer, x, std::vector<int>(query_rows, query_rows + l_q), visible,
                                std::vector<int>(position_ids, position_ids + l_in), dy, G->g);
      std::memcpy(dxn, dx.a.data(), sizeof(double) * dx.a.size());
    } catch (...) {
      delete G;
      throw;
    }
    *out = G;
  });
}

int oracle_tokenizer_backward(const OrModel* m, const OrSample* s, const double* dtokens, OrGrads** out) {
  return guarded([&] {
    const int L = (m->cfg.special_tokens ? 3 : 0) + s->n_hist + s->n_prof + s->n_cand;
    M dt(L, m->d);
    std::memcpy(dt.a.data(), dtokens, sizeof(double) * dt.a.size());
    auto* G = new OrGrads;
    try {
      tokenizer_backward(*m, *s, dt, G->g);
    } catch (...) {
      delete G;
      throw;
    }
    *out = G;
  });
}
}  // extern "C"
