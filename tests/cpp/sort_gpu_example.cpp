// C++ drop-in check: drives libsort_b200.so through include/rankformer/sort_gpu.hpp exactly as
// a rankformer:: caller would (host planner calls need no GPU; scoring does). Prints
// "host ok" after the host-only checks and "gpu ok <p0>" after one scored request.
#include <cstdio>
#include <cstring>
#include <random>

#include "../../include/rankformer/sort_gpu.hpp"

using namespace rankformer;

int main(int argc, char** argv) {
  // host-only rules (mask.cpp / tokenizer.cpp restated in the library's planner)
  auto keep = gpu::make_geometric_schedule(1030, 4, 128);
  if (keep != std::vector<int>({1030, 514, 256, 128})) { std::puts("schedule mismatch"); return 1; }
  std::vector<Role> roles = {Role::kBos, Role::kHist, Role::kHist, Role::kCand, Role::kCand};
  Mat m = gpu::build_mask(5, -1, 128, roles, {0, 1, 2, 3, 3});
  if (gpu::mask_visible_count(m) != 1 + 2 + 3 + 4 + 4) { std::puts("mask mismatch"); return 1; }
  if (gpu::time_bucket(1023, 32) != 10) { std::puts("bucket mismatch"); return 1; }
  bool threw = false;
  try { gpu::build_mask(1, 0, 0, roles, {0, 1, 2, 3, 3}); } catch (const ConfigError&) { threw = true; }
  if (!threw) { std::puts("expected ConfigError"); return 1; }
  std::puts("host ok");
  if (argc < 2 || std::strcmp(argv[1], "--gpu") != 0) return 0;

  // tiny SORT on the GPU through the C++ model API
  SortConfig c{};
  c.model_dim = 64; c.heads = 4; c.layers = 2; c.ffn_dim = 160; c.head_hidden = 0;
  c.item_dim = 32; c.action_dim = 8; c.scene_dim = 8; c.time_dim = 8; c.profile_dim = 16;
  c.n_items = 5000; c.n_actions = 3; c.n_scenes = 4; c.n_time_buckets = 32;
  c.n_profile_fields = 3; c.profile_vocab[0] = c.profile_vocab[1] = c.profile_vocab[2] = 8;
  c.special_tokens = 1; c.qknorm = 1; c.gate = 1; c.rope_theta = 10000.0;
  c.local_window = 32; c.full_suffix = 128; c.keep[0] = c.keep[1] = 262; c.keep_specials = 0;
  c.max_batch = 2; c.n_hist = 256; c.n_cand = 16;
  std::mt19937 rng(1);
  std::normal_distribution<float> nd(0.f, 0.1f);
  std::map<std::string, std::pair<std::vector<int64_t>, std::vector<float>>> P;
  auto add = [&](const std::string& n, int64_t r, int64_t cc, float base = 0.f) {
    std::vector<float> v(static_cast<size_t>(r * cc));
    for (auto& x : v) x = base + nd(rng);
    P[n] = {{r, cc}, v};
  };
  add("tok.special", 3, 64); add("tok.item_table", 5000, 32); add("tok.action_table", 3, 8);
  add("tok.scene_table", 4, 8); add("tok.time_table", 32, 8);
  for (int f = 0; f < 3; ++f) add("tok.profile_table." + std::to_string(f), 8, 16);
  add("tok.w_hist", 56, 64); add("tok.b_hist", 1, 64); add("tok.g_hist", 1, 64, 1.f);
  add("tok.w_prof", 16, 64); add("tok.b_prof", 1, 64); add("tok.g_prof", 1, 64, 1.f);
  add("tok.w_cand", 32, 64); add("tok.b_cand", 1, 64); add("tok.g_cand", 1, 64, 1.f);
  for (int l = 0; l < 2; ++l) {
    const std::string a = "attn." + std::to_string(l) + ".";
    for (const char* w : {"wq", "wk", "wv", "wo", "wg"}) add(a + w, 64, 64);
    add(a + "qk_gain_q", 4, 16, 1.f); add(a + "qk_gain_k", 4, 16, 1.f);
    add("block." + std::to_string(l) + ".attn_norm", 1, 64, 1.f);
    add("block." + std::to_string(l) + ".ffn_norm", 1, 64, 1.f);
    add("ffn." + std::to_string(l) + ".w_gate", 64, 160); add("ffn." + std::to_string(l) + ".w_up", 64, 160);
    add("ffn." + std::to_string(l) + ".w_down", 160, 64);
  }
  add("final_norm.gain", 1, 64, 1.f); add("head.w1", 64, 64); add("head.b1", 1, 64);
  add("head.w2", 64, 3); add("head.b2", 1, 3);
  gpu::Model model(c, P, 0);
  RequestSample s;
  s.timestamp = 1'800'000'000;
  s.user_profile = {1, 2, 3};
  for (int i = 0; i < 256; ++i) s.history.push_back({i * 7 % 5000, ActionType::kClick, s.timestamp - 1000 + i, i % 4});
  for (int j = 0; j < 16; ++j) s.candidates.push_back({j * 13 % 5000});
  auto scores = model.score({s});
  TokenSequence t = model.tokenize_sample(s);
  if (t.length() != 278 || t.position_ids.back() != 262) { std::puts("tokenize mismatch"); return 1; }
  const float p0 = scores[0][0][0];
  if (!(p0 > 0.f && p0 < 1.f)) { std::puts("bad score"); return 1; }
  // five requests = three batches of max_batch 2 through the pipelined path: each request's
  // scores equal its single-request scores
  std::vector<RequestSample> many;
  for (int k = 0; k < 5; ++k) {
    RequestSample r = s;
    for (auto& cnd : r.candidates) cnd.item_id = (cnd.item_id + 17 * k) % 5000;
    many.push_back(r);
  }
  auto multi = model.score(many);
  for (int k = 0; k < 5; ++k) {
    auto single = model.score({many[static_cast<size_t>(k)]});
    if (single[0] != multi[static_cast<size_t>(k)]) { std::puts("pipelined batch mismatch"); return 1; }
  }
  s.candidates[3].item_id = 5000;  // OOV -> ConfigError (tokenizer.cpp:14-19)
  threw = false;
  try { model.score({s}); } catch (const ConfigError&) { threw = true; }
  if (!threw) { std::puts("expected OOV ConfigError"); return 1; }
  std::printf("gpu ok %.6f\n", p0);
  return 0;
}
