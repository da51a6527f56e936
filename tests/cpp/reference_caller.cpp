// A caller written against the REFERENCE's hot-path API (call sites as in tokenizer.hpp:84,
// mask.hpp:36-78, norm.hpp:17-45, rope.hpp:13, attention.hpp:58-63), compiled unchanged against
// include/rankformer/ (-I<repo>/include) and run through libsort_b200.so.
//
//   reference_caller host              host-only rules (no GPU): prints "host ok"
//   reference_caller IN OUT            reads params + one request (IN, written by
//                                      tests/test_cpp_reference_api.py), runs tokenizer -> pre-norm ->
//                                      mask -> AttentionLayer forward/backward -> rmsnorm / rope, writes
//                                      every result to OUT for the test to check against the oracle
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <string>
#include <vector>

#include "rankformer/attention.hpp"
#include "rankformer/mask.hpp"
#include "rankformer/norm.hpp"
#include "rankformer/rope.hpp"
#include "rankformer/tokenizer.hpp"

using namespace rankformer;

namespace {

template <class T>
T rd(std::ifstream& f) {
  T v{};
  f.read(reinterpret_cast<char*>(&v), sizeof(T));
  return v;
}

struct Out {
  std::ofstream f;
  void put(const std::string& name, const Mat& m) {
    const int32_t n = static_cast<int32_t>(name.size());
    const int64_t r = m.rows(), c = m.cols();
    f.write(reinterpret_cast<const char*>(&n), 4);
    f.write(name.data(), n);
    f.write(reinterpret_cast<const char*>(&r), 8);
    f.write(reinterpret_cast<const char*>(&c), 8);
    f.write(reinterpret_cast<const char*>(m.data()), static_cast<std::streamsize>(r * c * 8));
  }
  void put(const std::string& name, const std::vector<int>& v) {
    Mat m(1, static_cast<int64_t>(v.size()));
    for (size_t i = 0; i < v.size(); ++i) m(0, static_cast<int64_t>(i)) = v[i];
    put(name, m);
  }
};

int host_checks() {
  // mask.hpp:36-42 with a MaskSpec, suffix overload and explicit query rows
  std::vector<Role> roles = {Role::kBos, Role::kHist, Role::kHist, Role::kSep, Role::kCand, Role::kCand};
  std::vector<int> pos = {0, 1, 2, 3, 4, 4};
  MaskSpec spec;
  spec.l_q = 6;
  spec.l_kv = 6;
  spec.local_window = -1;
  spec.full_suffix = 128;
  Mat mask = build_mask(spec, roles, pos);
  if (mask_visible_count(mask) != 1 + 2 + 3 + 4 + 5 + 5) return std::puts("mask count mismatch"), 1;
  if (mask(4, 5) == 0.0 || mask(5, 4) == 0.0 || mask(5, 5) != 0.0) return std::puts("candidate isolation"), 1;
  PruneSchedule sched = make_geometric_schedule(1030, 4, 128);
  sched.validate();
  if (sched.keep != std::vector<int>({1030, 514, 256, 128})) return std::puts("schedule mismatch"), 1;
  std::vector<int> rows = retained_rows(roles, 1, false);
  if (rows != std::vector<int>({3, 4, 5})) return std::puts("retained rows mismatch"), 1;
  spec.l_q = 3;
  Mat pm = build_mask(spec, roles, pos, rows);
  if (pm.rows() != 3 || mask_visible_count(pm) != 4 + 5 + 5) return std::puts("pruned mask mismatch"), 1;
  if (time_bucket(1023, 32) != 10) return std::puts("time bucket mismatch"), 1;
  bool threw = false;
  try {
    MaskSpec bad;
    bad.l_q = 2;
    bad.l_kv = 1;
    build_mask(bad, roles, pos);
  } catch (const ConfigError&) {
    threw = true;
  }
  if (!threw) return std::puts("expected ConfigError"), 1;
  std::puts("host ok");
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc == 2 && std::strcmp(argv[1], "host") == 0) return host_checks();
  if (argc != 3) return std::puts("usage: reference_caller host | IN OUT"), 2;
  std::ifstream in(argv[1], std::ios::binary);
  // ---- model config, parameters, one request (written by the test)
  SortConfig c{};
  in.read(reinterpret_cast<char*>(&c), sizeof(SortConfig));
  const int n_params = rd<int32_t>(in);
  std::map<std::string, std::pair<std::vector<int64_t>, std::vector<float>>> P;
  for (int i = 0; i < n_params; ++i) {
    std::string name(static_cast<size_t>(rd<int32_t>(in)), '\0');
    in.read(name.data(), static_cast<std::streamsize>(name.size()));
    const int64_t r = rd<int64_t>(in), cc = rd<int64_t>(in);
    std::vector<float> v(static_cast<size_t>(r * cc));
    in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(v.size() * 4));
    P[name] = {{r, cc}, v};
  }
  RequestSample sample;
  sample.timestamp = rd<int64_t>(in);
  for (int i = 0; i < c.n_hist; ++i) {
    ItemEvent e;
    e.item_id = rd<int32_t>(in);
    e.action_type = static_cast<ActionType>(rd<int32_t>(in));
    e.scene_id = rd<int32_t>(in);
    e.timestamp = rd<int64_t>(in);
    sample.history.push_back(e);
  }
  for (int f = 0; f < c.n_profile_fields; ++f) sample.user_profile.push_back(rd<int32_t>(in));
  for (int j = 0; j < c.n_cand; ++j) {
    Candidate cd;
    cd.item_id = rd<int32_t>(in);
    sample.candidates.push_back(cd);
  }
  const int keep = rd<int32_t>(in);  // non-candidate rows kept as queries of the checked layer
  Mat dout_seed;                      // d(out) for the backward, l_q x d (from the test)
  {
    const int64_t r = rd<int64_t>(in), cc = rd<int64_t>(in);
    std::vector<double> v(static_cast<size_t>(r * cc));
    in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
    dout_seed = Mat(r, cc);
    std::memcpy(dout_seed.data(), v.data(), v.size() * 8);
  }
  if (!in) return std::puts("bad input file"), 2;
  gpu::Model model(c, P, 0);
  Out out{std::ofstream(argv[2], std::ios::binary)};

  // ---- the reference's call sites
  const Tokenizer tokenizer(model);
  TokenizerCache tcache;
  TokenSequence seq = tokenizer.tokenize_sample(sample, tcache);  // tokenizer.hpp:84
  out.put("tokens", seq.tokens);
  out.put("hist_time", tcache.hist_time);
  out.put("position_ids", seq.position_ids);

  Mat gain(1, c.model_dim);
  for (int k = 0; k < c.model_dim; ++k) gain(0, k) = P.at("block.0.attn_norm").second[static_cast<size_t>(k)];
  RmsNormCache ncache;
  Mat xn = rmsnorm_forward(seq.tokens, gain, ncache);  // norm.hpp:17
  out.put("xn", xn);

  std::vector<int> query_rows = retained_rows(seq.roles, keep, c.keep_specials != 0);  // mask.hpp:77
  MaskSpec spec;
  spec.l_q = static_cast<int>(query_rows.size());
  spec.l_kv = seq.length();
  spec.local_window = c.local_window;
  spec.full_suffix = c.full_suffix;
  Mat mask = build_mask(spec, seq.roles, seq.position_ids, query_rows);  // mask.hpp:36
  out.put("query_rows", query_rows);
  out.put("mask", mask);

  AttentionSettings s;
  s.model_dim = c.model_dim;
  s.heads = c.heads;
  s.rope_theta = c.rope_theta;
  AttentionLayer layer(s, 0);
  for (Parameter* p : layer.params()) {
    const auto& src = P.at(p->name).second;
    for (int64_t k = 0; k < p->size(); ++k) p->value.data()[k] = src[static_cast<size_t>(k)];
  }
  AttentionCache acache;
  Mat attn = layer.forward(xn, query_rows, mask, seq.position_ids, acache);  // attention.hpp:58
  out.put("attn_out", attn);

  ParamRefs params = layer.params();
  params[4]->frozen = true;  // wo frozen: no gradient (params.hpp:15-25)
  GradBuffer grads(params);
  ParamIndex index(params);
  Mat dxn = layer.backward(dout_seed, acache, grads, index);  // attention.hpp:62
  out.put("dxn", dxn);
  for (Parameter* p : params) out.put("grad." + p->name, grads[index.of(*p)]);

  Mat dgain(1, c.model_dim);
  Mat dx = rmsnorm_backward(dxn, ncache, gain, dgain);  // norm.hpp:32
  out.put("dx", dx);
  out.put("dgain", dgain);

  std::vector<int> qpos;
  for (int r : query_rows) qpos.push_back(seq.position_ids[static_cast<size_t>(r)]);
  Mat head0(static_cast<int64_t>(query_rows.size()), s.head_dim());
  for (int64_t r = 0; r < head0.rows(); ++r)
    for (int64_t k = 0; k < head0.cols(); ++k) head0(r, k) = attn(r, k);
  out.put("rope", rope_apply(head0, qpos, s.rope_theta));              // rope.hpp:13
  out.put("rope_inv", rope_apply(head0, qpos, s.rope_theta, true));
  out.f.close();
  std::puts("gpu ok");
  return 0;
}
