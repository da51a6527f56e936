/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the SORT hot path.
 *
 * A plain fp64 CPU restatement of the reference's algorithm
 * (/root/reference/proj, C++20 + Eigen, fp64). It exists so that tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * can CHECK the CUDA path and time the reference algorithm on host cores.
 * Nothing in the product (paper_2603_03988_b200/) links, loads or calls it.
 *
 * Parity status: PINNED TO THE REFERENCE'S OWN CODE. The reference cannot be built with
 * its own CMake (Eigen3 absent, its src/tools/tests CMake dirs missing,
 * attention.cpp:152,180-183,194 do not compile), but oracle/Makefile compiles its
 * mask.cpp / tokenizer.cpp / attention.cpp unmodified against a small Eigen-subset shim
 * (oracle/ref_shim) into oracle/_ref/libref.so, and tests/test_ref_pinning.py checks this
 * restatement against it: integer artifacts bit-identical, fp64 values to 1e-9 (tokenizer
 * forward/backward, masks, schedules, retained rows, rmsnorm, rope, dense/blockwise
 * attention, AttentionLayer forward/backward, and the whole-model forward composed from
 * the reference's calls plus the spec-only FFN/block/head). It is additionally pinned
 * against every known-answer example in SPEC.md (tests/test_oracle_kat.py).
 *
 * All functions return 0 on success, 1 for a ConfigError (common.hpp:17-21)
 * and 2 for a RuntimeFailure (common.hpp:23-27); oracle_last_error() gives
 * the message (thread-local).
 */
#ifndef SORT_ORACLE_H_
#define SORT_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Role ids follow rankformer::Role (tokenizer.hpp:13). */
enum { OR_ROLE_BOS = 0, OR_ROLE_HIST = 1, OR_ROLE_SEP = 2, OR_ROLE_PROF = 3, OR_ROLE_CAND = 4 };

typedef struct {
  /* TokenizerConfig (tokenizer.hpp:31-56) without side-feature groups. */
  int model_dim, item_dim, action_dim, scene_dim, time_dim, profile_dim;
  int n_items, n_actions, n_scenes, n_time_buckets;
  int n_profile_fields;
  int profile_vocab[16];
  int special_tokens;
  /* Block stack + AttentionSettings (attention.hpp:13-29). */
  int layers, heads, ffn_dim;
  int qknorm, gate;
  double rope_theta;
  /* MaskSpec (mask.hpp:15-31) + PruneSchedule (mask.hpp:48-61). */
  int local_window, full_suffix;
  int keep[64];
  int keep_specials;
  int head_hidden; /* ranking head d -> d_h; 0 means d */
  /* DeepSeek-style MoE FFN: moe_experts routed experts (0 = dense
   * SwishGLU), moe_topk active per token, moe_shared always-on shared experts (0/1),
   * moe_ffn_dim intermediate size of every expert. */
  int moe_experts, moe_topk, moe_shared, moe_ffn_dim;
} OrModelCfg;

/* One request (RequestSample, data.hpp:32-38) with no side features. */
typedef struct {
  int64_t timestamp;
  int n_hist;
  const int32_t* hist_item;
  const int32_t* hist_action;
  const int32_t* hist_scene;
  const int64_t* hist_ts;
  int n_prof;
  const int32_t* profile;
  int n_cand;
  const int32_t* cand_item;
} OrSample;

const char* oracle_last_error(void);

/* --- integer rules ---------------------------------------------------- */
int oracle_time_bucket(int64_t delta_seconds, int n_buckets);
int oracle_build_mask(int l_q, int l_kv, int local_window, int full_suffix, const int* roles,
                      const int* position_ids, const int* query_rows /* NULL = suffix */,
                      uint8_t* out_visible /* l_q*l_kv */);
int64_t oracle_mask_visible_count(const uint8_t* visible, int64_t n);
int oracle_geometric_schedule(int prefix_len, int depth, int target, int* out_keep);
int oracle_full_schedule(int prefix_len, int depth, int* out_keep);
int oracle_retained_rows(const int* roles, int n, int keep, int keep_specials, int* out_rows,
                         int* out_n);
int oracle_prune_queries(const double* x, int rows, int cols, int n, double* out);

/* --- numeric ops (fp64) ------------------------------------------------ */
int oracle_rmsnorm_forward(const double* x, int rows, int cols, const double* gain, double* y,
                           double* inv_rms /* may be NULL */);
int oracle_rmsnorm_backward(const double* dy, const double* x, const double* inv_rms, int rows,
                            int cols, const double* gain, double* dgain_accum, double* dx);
int oracle_rope_apply(const double* x, int rows, int dim, const int* position_ids, double theta,
                      int inverse, double* out);
int oracle_dense_masked_attention_f64(const double* q, const double* k, const double* v,
                                      const double* mask, int l_q, int l_kv, int dk, int dv,
                                      double* out);
int oracle_dense_masked_attention_f32(const float* q, const float* k, const float* v,
                                      const float* mask, int l_q, int l_kv, int dk, int dv,
                                      float* out);
int oracle_blockwise_masked_attention_f64(const double* q, const double* k, const double* v,
                                          const double* mask, int l_q, int l_kv, int dk, int dv,
                                          int block, double* out, int64_t* skipped,
                                          int64_t* total);
int oracle_blockwise_masked_attention_f32(const float* q, const float* k, const float* v,
                                          const float* mask, int l_q, int l_kv, int dk, int dv,
                                          int block, float* out, int64_t* skipped,
                                          int64_t* total);
int oracle_swishglu(const double* x, int rows, int d, int m, const double* w_gate,
                    const double* w_up, const double* w_down, double* out);

/* --- model ------------------------------------------------------------- */
typedef struct OrModel OrModel;
int oracle_model_create(const OrModelCfg* cfg, OrModel** out);
void oracle_model_destroy(OrModel* m);
/* Parameter names follow the reference (tokenizer.cpp:45-63, attention.cpp:37-46)
 * plus spec-named block.<l>.attn_norm / block.<l>.ffn_norm / ffn.<l>.w_gate|w_up|w_down /
 * final_norm.gain / head.w1|b1|w2|b2. Row-major [rows, cols]. */
int oracle_model_set_param(OrModel* m, const char* name, const double* data, int rows, int cols);
/* Parameter::frozen of the item table (params.hpp:18): trainable = 1 makes the backward produce
 * the "tok.item_table" gradient (tokenizer.cpp:315-317, 346-352). Default: frozen. */
int oracle_model_set_item_trainable(OrModel* m, int trainable);

/* Tokenize one request (Tokenizer::tokenize_sample, tokenizer.cpp:144-238). */
int oracle_tokenize(const OrModel* m, const OrSample* s, double* tokens /* L*d */,
                    int* position_ids, int* roles, int* candidate_index,
                    int* hist_time /* n_hist */, int* out_len);

/* Attention layer l (AttentionLayer::forward, attention.cpp:71-132). */
int oracle_attention_forward(const OrModel* m, int layer, const double* xn, int l_in,
                             const int* query_rows, int l_q, const uint8_t* visible,
                             const int* position_ids, double* out /* l_q*d */);

/* Full forward of one request: probabilities [n_cand*3] (click, cart, purchase),
 * optionally the pre-sigmoid logits [n_cand*3]. */
int oracle_model_forward(const OrModel* m, const OrSample* s, double* probs, double* logits);

/* Full forward with MoE routing control: forced_sel (NULL = route) holds, layer after layer,
 * l_q[l] x moe_topk expert ids to use instead of the oracle's own selection (combine weights
 * still come from the oracle's raw scores of those experts); out_sel (same layout) receives
 * the selection used and out_margin (l_q[l] per layer) the gap between the k-th and
 * (k+1)-th biased score (+inf when k == E). Any of the three may be NULL. */
int oracle_model_forward_moe(const OrModel* m, const OrSample* s, const int* forced_sel, double* probs,
                             double* logits, int* out_sel, double* out_margin);

/* Pre-training: click sequence = s->hist_* (n_hist clicks; timestamp,
 * profile and candidates unused). tokens [1 + n, d] (tokenize_click_sequence,
 * tokenizer.cpp:240-284); forward: lse[t], target[t] (logit of click t) for t < n, hproj
 * [1 + n, item_dim] the projected hidden rows (may be NULL). */
int oracle_tokenize_clicks(const OrModel* m, const OrSample* s, double* tokens, int* hist_time);
int oracle_pretrain_forward(const OrModel* m, const OrSample* s, double* lse, double* target, double* hproj);

/* --- MoE FFN operators -------------------------------- */
/* route_topk, DeepSeek style: s_e = sigmoid(x . router[:, e]); selection = top-k of s_e + bias_e
 * in descending order, ties -> lower index; weights w_j = s_{e_j} / sum_j s_{e_j} (bias never
 * enters the weights). router [d, E] row-major. sel/w [rows, k]; margin [rows] (may be NULL). */
int oracle_moe_route(const double* x, int rows, int d, int n_experts, int k, const double* router,
                     const double* bias, int* sel, double* w, double* margin);
/* moe_forward: out = sum_{shared} swishglu_s(x) + sum_j w_j swishglu_{e_j}(x). Expert weights
 * stacked over (n_experts + shared) experts, shared last: w_gate/w_up [n, d, m], w_down [n, m, d].
 * forced_sel [rows, k] or NULL. */
int oracle_moe_ffn(const double* x, int rows, int d, int m, int n_experts, int k, int shared,
                   const double* router, const double* bias, const double* w_gate, const double* w_up,
                   const double* w_down, const int* forced_sel, double* out, int* sel, double* w);
/* update_balance, DeepSeek style: bias_e -= gamma * sign(load_e - mean load). */
int oracle_moe_update_bias(const int64_t* load, int n_experts, double gamma, double* bias);

/* Per-layer structural artifacts of one request: for each layer l,
 * l_q[l], visible count[l], and query_rows concatenated. */
int oracle_model_layer_meta(const OrModel* m, const OrSample* s, int* l_q, int64_t* visible,
                            int* query_rows_concat, int* total_rows);

/* Batched forward over B requests on `threads` host threads (one request per
 * thread at a time, the reference's concurrency model: params.hpp:12-14). */
int oracle_model_forward_batch(const OrModel* m, const OrSample* samples, int B, int threads,
                               double* probs /* sum(n_cand)*3 */);

/* --- training backward (fp64) ------------------------------------------ */
/* Backward of oracle_model_forward for one request given dL/dlogits [n_cand*3]: the head,
 * final RMSNorm, every block (SwishGLU FFN, pre-norms, residuals, pruning scatter) and
 * AttentionLayer::backward (attention.cpp:134-202, intended math). dtokens [L*d] may be NULL.
 * Gradients are returned by parameter name (oracle_grads_get; rows = cols = 0 for a
 * parameter off the differentiated path, e.g. the tokenizer tables). */
typedef struct OrGrads OrGrads;
int oracle_model_backward(const OrModel* m, const OrSample* s, const double* dlogits,
                          double* dtokens, OrGrads** out);
/* Pre-training backward of one click sequence: gradients of
 * scale * sum_t CE_t over every parameter (item table: tied head + input embedding);
 * *ce_sum = sum_t CE_t. */
int oracle_pretrain_backward(const OrModel* m, const OrSample* s, double scale, double* ce_sum, OrGrads** out);
int oracle_grads_get(const OrGrads* g, const char* name, double* out, int* rows, int* cols);
void oracle_grads_destroy(OrGrads* g);
/* AttentionLayer::backward of layer `layer` alone (attention.cpp:134-202): d(xn) [l_in, d]
 * and the layer's gradients (attn.<l>.wq|wk|wv|wo|wg|qk_gain_q|qk_gain_k). */
int oracle_attention_backward(const OrModel* m, int layer, const double* xn, int l_in, const int* query_rows,
                              int l_q, const uint8_t* visible, const int* position_ids, const double* dout,
                              double* dxn, OrGrads** out);
/* Tokenizer::backward (tokenizer.cpp:286-354) for dL/dtokens [L, d], item table frozen. */
int oracle_tokenizer_backward(const OrModel* m, const OrSample* s, const double* dtokens, OrGrads** out);

#ifdef __cplusplus
}
#endif

#endif /* SORT_ORACLE_H_ */
