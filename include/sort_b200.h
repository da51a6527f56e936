/* SPDX-License-Identifier: Apache-2.0
 *
 * sort_b200.h -- C ABI of libsort_b200.so, the B200-native (sm_100a) SORT
 * ranking-transformer block path (arXiv 2603.03988).
 *
 * This is the drop-in boundary for the reference's C++ hot-path API
 * (/root/reference/proj/include/rankformer/ headers). Plain pointers and sizes
 * only; no CUDA/torch types. Each entry point names the reference interface
 * it replaces. A C++ binding with the reference's rankformer:: names lives
 * in include/rankformer/sort_gpu.hpp; the ctypes binding used by the tests is
 * paper_2603_03988_b200/runtime.py; INTEGRATION.md shows both.
 *
 * Conventions:
 *   - Every function returns int status: 0 = ok, 1 = config/input error
 *     (rankformer::ConfigError, common.hpp:17-21; CLI exit 1), 2 = runtime
 *     failure (rankformer::RuntimeFailure, common.hpp:23-27; CLI exit 2).
 *     sort_last_error() returns the thread-local message of the last failure.
 *   - A handle binds one CUDA device and one stream, owns device weights and
 *     workspace; calls on one handle are serialised by the caller (one handle
 *     per GPU, each driven by its own host thread -- the reference's
 *     "pure const forward, many threads" model, params.hpp:12-14).
 *   - Host buffers are caller-owned. Device-side range checks (OOV ids,
 *     tokenizer.cpp:14-19) raise a device flag that becomes status 1; an
 *     out-of-vocabulary id is never read out of bounds.
 *   - All requests of one batch share n_hist / n_cand (the batched path is
 *     planned per geometry); ragged batches are issued as several calls.
 */
#ifndef SORT_B200_H_
#define SORT_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SORT_OK 0
#define SORT_CONFIG_ERROR 1
#define SORT_RUNTIME_FAILURE 2

#define SORT_MAX_PROFILE_FIELDS 16
#define SORT_MAX_LAYERS 64

/* Role ids: rankformer::Role (tokenizer.hpp:13). */
#define SORT_ROLE_BOS 0
#define SORT_ROLE_HIST 1
#define SORT_ROLE_SEP 2
#define SORT_ROLE_PROF 3
#define SORT_ROLE_CAND 4

typedef struct SortHandle_* SortHandle;

/* Model + batch geometry. Fields mirror TokenizerConfig (tokenizer.hpp:31-56),
 * AttentionSettings (attention.hpp:13-29), MaskSpec (mask.hpp:15-31),
 * PruneSchedule (mask.hpp:48-61) and the spec's ModelConfig. */
typedef struct {
  int32_t model_dim, heads, layers, ffn_dim, head_hidden; /* head_hidden 0 -> model_dim */
  int32_t item_dim, action_dim, scene_dim, time_dim, profile_dim;
  int32_t n_items, n_actions, n_scenes, n_time_buckets;
  int32_t n_profile_fields;
  int32_t profile_vocab[SORT_MAX_PROFILE_FIELDS];
  int32_t special_tokens, qknorm, gate;
  double rope_theta;
  int32_t local_window; /* -1 = unbounded */
  int32_t full_suffix;
  int32_t keep[SORT_MAX_LAYERS]; /* per-layer non-candidate keep counts */
  int32_t keep_specials;
  int32_t max_batch, n_hist, n_cand; /* batch geometry the workspace is planned for */
  /* DeepSeek-style MoE FFN in every block instead of the dense SwishGLU:
   * moe_experts routed experts (0 = dense FFN), moe_topk active per token, moe_shared
   * always-on shared experts (0 or 1), moe_ffn_dim intermediate size of every expert.
   * Parameters ffn.<l>.router [d, E], ffn.<l>.router_bias [1, E],
   * ffn.<l>.expert.<e>.w_gate|w_up [d, m_e] / w_down [m_e, d], ffn.<l>.shared.* likewise. */
  int32_t moe_experts, moe_topk, moe_shared, moe_ffn_dim;
  /* 1 = generative pre-training model: sequences are click histories
   * tokenized as [BOS; clicks] (tokenize_click_sequence, tokenizer.cpp:240-284) with
   * n_cand = 0 and n_profile_fields = 0, no pruning, and the ranking head replaced by the
   * tied next-item head (parameter pretrain.proj [d, item_dim]; sort_pretrain_forward). */
  int32_t pretrain;
} SortConfig;

/* A batch of requests in structure-of-arrays form (RequestSample, data.hpp:32-38,
 * without side features). Row-major [batch, n] arrays. */
typedef struct {
  int32_t batch;
  const int32_t* hist_item;   /* [batch, n_hist] */
  const int32_t* hist_action; /* [batch, n_hist] */
  const int32_t* hist_scene;  /* [batch, n_hist] */
  const int64_t* hist_ts;     /* [batch, n_hist] */
  const int64_t* req_ts;      /* [batch] */
  const int32_t* profile;     /* [batch, n_profile_fields] */
  const int32_t* cand_item;   /* [batch, n_cand] */
} SortBatch;

const char* sort_last_error(void);
int sort_version(void);

/* ---------------------------------------------------------------- lifetime */
/* Replaces constructing Tokenizer + AttentionLayer x depth (tokenizer.cpp:42-64,
 * attention.cpp:34-47) and the spec's model assembly. */
int sort_create(const SortConfig* cfg, int device, SortHandle* out);
int sort_destroy(SortHandle h);
/* cudaStream_t passed as void* (NULL = the handle's own stream). */
int sort_set_stream(SortHandle h, void* stream);

/* Named parameters in the reference's [rows, cols] row-major orientation
 * (Parameter::value, params.hpp:15-25). Names: tok.* (tokenizer.cpp:45-63),
 * attn.<l>.{wq,wk,wv,wo,wg,qk_gain_q,qk_gain_k} (attention.cpp:37-46), and the
 * spec-named block.<l>.{attn_norm,ffn_norm}, ffn.<l>.{w_gate,w_up,w_down},
 * final_norm.gain, head.{w1,b1,w2,b2}. Values are converted to the device
 * layout (bf16 K-major tensors, fp32 head) by sort_finalize_params. */
int sort_load_param(SortHandle h, const char* name, const float* data, int64_t rows, int64_t cols);
int sort_finalize_params(SortHandle h);

/* ---------------------------------------------------------------- forward */
/* model_forward over a batch: scores[b, j, 0..2] =
 * {p_click, p_cart, p_purchase} for candidate j of request b. When
 * inputs_on_device != 0 the SortBatch pointers are device pointers; when
 * scores_on_device != 0 `scores` is a device pointer. Synchronous unless
 * both are device pointers (then it only enqueues on the handle's stream;
 * call sort_sync to collect the status of device-side checks). */
int sort_forward(SortHandle h, const SortBatch* batch, int inputs_on_device, float* scores,
                 int scores_on_device);
/* Pipelined serving form of sort_forward with HOST inputs and outputs: enqueue only. The
 * batch's arrays are copied on the handle's copy stream into one of two device staging slots
 * (alternating per call), so the next call's host->device copy overlaps this call's kernels;
 * scores [batch, n_cand, 3] are written back asynchronously. Host buffers should be pinned
 * and must stay untouched until sort_sync; device-side errors (OOV ids) surface at sort_sync. */
int sort_forward_async(SortHandle h, const SortBatch* batch, float* scores);
int sort_sync(SortHandle h);

/* Same as sort_forward but also returns the pre-sigmoid logits [batch, n_cand, 3]. */
int sort_forward_logits(SortHandle h, const SortBatch* batch, float* probs, float* logits);

/* ---------------------------------------------------------------- parity ops */
/* Tokenizer::tokenize_sample (tokenizer.hpp:84) over a batch, host buffers:
 * tokens [batch, L, d] (fp32 copy of the bf16 tokens), hist_time [batch, n_hist]
 * (the time-bucket part of TokenizerCache, tokenizer.hpp:68). position_ids / roles /
 * candidate_index [L] are the (batch-uniform) sequence structure. Any output may be NULL. */
int sort_tokenize(SortHandle h, const SortBatch* batch, float* tokens, int32_t* hist_time,
                  int32_t* position_ids, int32_t* roles, int32_t* candidate_index);

/* Structural plan of layer `layer` (build_mask + retained_rows, mask.hpp:36-76):
 * l_q/l_kv, the retained query rows (kv-index space), and the compact mask of each
 * query row: visible = [lo, hi] U {self} (self = -1 for non-candidates), plus the
 * number of visible entries (mask_visible_count, mask.hpp:44) and the attention
 * kernel's 128x128 tile census (issued / total). Arrays sized >= l_q; may be NULL. */
int sort_layer_plan(SortHandle h, int layer, int32_t* l_q, int32_t* l_kv, int32_t* query_rows,
                    int32_t* lo, int32_t* hi, int32_t* self_idx, int64_t* visible,
                    int64_t* tiles_issued, int64_t* tiles_total);

/* AttentionLayer::forward (attention.hpp:58-59) of layer `layer` composed with the
 * pre-norm that feeds it: out = Attn_l(RMSNorm(x; block.<l>.attn_norm)),
 * for a batch of layer inputs x [batch, l_kv, d] (host fp32), using the layer's plan
 * for query rows / mask / positions. out: [batch, l_q, d] host fp32. */
int sort_attention_forward(SortHandle h, int layer, int32_t batch, const float* x, float* out);

/* blockwise_masked_attention (block_attention.hpp:58-62) at the kernel's tile size on
 * one (q, k, v) problem per head of a batch (dk 16 or 32): q [nh, l_q, dk], k/v [nh, l_kv, dk] (host fp32,
 * rounded to bf16 on upload), visibility given in compact form (lo/hi/self per query row,
 * shared by all nh problems). out [nh, l_q, dk]; skipped/total 128x128 tiles per problem. */
int sort_block_attention(int32_t nh, int32_t l_q, int32_t l_kv, int32_t dk, const float* q,
                         const float* k, const float* v, const int32_t* lo, const int32_t* hi,
                         const int32_t* self_idx, float* out, int64_t* skipped, int64_t* total);

/* ---------------------------------------------------------------- operator-level entries */
/* The reference's free functions / AttentionLayer as standalone device ops (no handle; host fp32
 * buffers in and out). include/rankformer/reference_api.hpp binds them with the reference's
 * signatures.
 * rmsnorm_forward (norm.hpp:17-29): y [rows, cols] = x / rms(x) * gain, inv_rms [rows]. */
int sort_op_rmsnorm(int32_t rows, int32_t cols, const float* x, const float* gain, float* y, float* inv_rms);
/* rmsnorm_backward (norm.hpp:32-45): dx written, dgain [cols] ACCUMULATED (+=) like the reference. */
int sort_op_rmsnorm_backward(int32_t rows, int32_t cols, const float* dy, const float* x, const float* inv_rms,
                             const float* gain, float* dx, float* dgain);
/* rope_apply (rope.hpp:13-40): out [rows, dim], dim even (else status 1), inverse = exact adjoint. */
int sort_op_rope(int32_t rows, int32_t dim, const float* x, const int32_t* position_ids, double theta_base,
                 int32_t inverse, float* out);
/* AttentionLayer::forward (attention.hpp:58-59, attention.cpp:71-132) and, with dout != NULL,
 * AttentionLayer::backward (attention.hpp:62-63, attention.cpp:134-202) of one layer on one
 * request: xn [l_in, d] (normalised input), query_rows [l_q] strictly increasing into xn, the mask
 * as build_mask rows in compact form (visible = [lo, hi] U {self}; self -1 = none), position_ids
 * [l_in]. weights[7] = wq, wk, wv, wg, wo ([d, d], [in, out]) and qk_gain_q, qk_gain_k ([heads, dk]).
 * out [l_q, d]. Backward: dxn [l_in, d] written; dweights[i] ACCUMULATED (+=), NULL entry = frozen
 * parameter (params.hpp:15-25). dk in {16, 32, 64}; backward needs d <= 256; qknorm = gate = 1. */
int sort_op_attention_layer(int32_t model_dim, int32_t heads, double rope_theta, int32_t qknorm, int32_t gate,
                            int32_t l_in, int32_t l_q, const float* xn, const int32_t* query_rows, const int32_t* lo,
                            const int32_t* hi, const int32_t* self_idx, const int32_t* position_ids,
                            const float* const* weights, float* out, const float* dout, float* dxn,
                            float* const* dweights);

/* ---------------------------------------------------------------- host planner */
/* Host-only integer rules (no GPU needed): time_bucket (tokenizer.cpp:36-40),
 * make_geometric_schedule (mask.cpp:97-117), retained_rows (mask.cpp:132-154) and the
 * compact form of build_mask (mask.cpp:14-76). */
int sort_time_bucket(int64_t delta_seconds, int32_t n_buckets);
int sort_geometric_schedule(int32_t prefix_len, int32_t depth, int32_t target, int32_t* keep);
int sort_retained_rows(const int32_t* roles, int32_t n, int32_t keep, int32_t keep_specials,
                       int32_t* rows, int32_t* n_rows);
int sort_mask_intervals(int32_t l_q, int32_t l_kv, int32_t local_window, int32_t full_suffix,
                        const int32_t* roles, const int32_t* position_ids,
                        const int32_t* query_rows, int32_t* lo, int32_t* hi, int32_t* self_idx);

/* Op-level GEMM on the library's engines (the streaming tcgen05 GEMM of gemm_stream.cuh; small
 * or TMA-unfriendly fp32 shapes on the SIMT kernel), for tests and op-level callers: row-major
 * C[M, N] = op(A) op(B) with host fp32 buffers; A stored [M, K] (or [K, M] when trans_a),
 * B stored [K, N] (or [N, K] when trans_b). tf32 = 0: bf16 operands (row pitches multiples of
 * 8, N of 32); tf32 = 1: fp32 operands at TF32 precision. fp32 accumulation. */
int sort_op_gemm(int32_t M, int32_t N, int32_t K, int32_t trans_a, int32_t trans_b, int32_t tf32, const float* A,
                 const float* B, float* C);

/* ---------------------------------------------------------------- instrumentation */
/* Number of CUDA kernels one sort_forward launches, and per-stage device times (ms) of
 * the last sort_forward when timing was enabled with sort_enable_stage_timing(h, 1).
 * stage_names is a ';'-separated list written into names (cap bytes). */
int sort_kernel_count(SortHandle h, int32_t* launches);
int sort_enable_stage_timing(SortHandle h, int enable);
int sort_stage_times(SortHandle h, float* ms, int32_t cap, int32_t* n, char* names,
                     int32_t names_cap);
/* ---------------------------------------------------------------- training */
/* One training step of the scoring path on the handle's device: forward (saving activations)
 * + backward of the head, final norm, every block (SwishGLU FFN, pre-norms, residuals,
 * pruning scatter) and AttentionLayer::backward (attention.cpp:134-202, intended math),
 * given dL/dlogits [batch, n_cand, 3] (host). Gradients (fp32) stay on the device in one flat
 * buffer in parameter-name order; logits [batch, n_cand, 3] are returned when non-null.
 * Replaces the reference's per-request AttentionLayer::backward / rmsnorm_backward calls
 * (attention.hpp:62-63, norm.hpp:32) accumulated into a GradBuffer (params.hpp:42-70). */
int sort_train_step(SortHandle h, const SortBatch* batch, const float* dlogits, float* logits);
/* Training step with the ranking loss on the device: L = sum_obj w_obj *
 * mean BCE over candidates (labels [batch, n_cand, 3] host; obj_weights NULL = (1, .5, .5),
 * SPEC.md:416); dL/dlogits never leaves the GPU. *loss receives L. */
int sort_train_step_bce(SortHandle h, const SortBatch* batch, const float* labels,
                        const float* obj_weights, float* loss);
/* Pre-training step (cfg.pretrain = 1): forward of the click sequences, loss =
 * mean over the B * n_hist predicted positions of the full-softmax next-item CE (*loss), and the
 * backward of every parameter, the item table (tied head + input embedding) included unless
 * frozen. Follow with sort_adamw_step. Needs n_items % 32 == 0. */
int sort_pretrain_train_step(SortHandle h, const SortBatch* batch, float* loss);
/* adamw_step over every parameter not frozen (sort_set_frozen), then the bf16
 * inference weights are rebuilt from the fp32 masters on the device. Status 2 names the
 * parameter on a non-finite gradient. */
int sort_adamw_step(SortHandle h, float lr, float beta1, float beta2, float eps, float weight_decay);
/* Current fp32 master value of a trainable parameter (host copy, reference shape); for
 * "tok.item_table" the fp32 master when it is trained, else the device's bf16 table widened. */
int sort_get_param(SortHandle h, const char* name, float* out);
/* Gradient of one parameter from the last training step (host copy, reference shape),
 * "tok.item_table" included when it is not frozen. */
int sort_get_grad(SortHandle h, const char* name, float* out);
/* Parameter::frozen (params.hpp:15-25; tokenizer.cpp:289-346): a frozen parameter receives zero
 * gradient and no optimizer update (bytes unchanged). Every parameter starts
 * trainable except "tok.item_table", which starts frozen (SORT's transfer + freeze setting);
 * unfreezing it allocates its fp32 master (from the bf16 device table), gradient and moments. */
int sort_set_frozen(SortHandle h, const char* name, int32_t frozen);
/* transfer_item_table (tokenizer.cpp:376-383; transfer_sparse): copies the item
 * table of `from` (e.g. a pre-training handle) into `to` (same n_items / item_dim) and sets its
 * frozen flag. */
int sort_transfer_item_table(SortHandle from, SortHandle to, int32_t freeze);
/* Offset / shape of one parameter's gradient in the flat buffer, and its total length. */
int sort_grad_info(SortHandle h, const char* name, int64_t* offset, int64_t* rows, int64_t* cols,
                   int64_t* total);
/* Copy the flat gradient buffer out (to_handle = 0) or back in (to_handle = 1, e.g. after a
 * data-parallel all-reduce); buf is host or device memory. */
int sort_grads_copy(SortHandle h, float* buf, int buf_on_device, int to_handle);
/* d(loss)/d(tokens) of the last step, [batch, L, d] fp32 on the host. */
int sort_dtokens(SortHandle h, int32_t batch, float* out);

/* ---------------------------------------------------------------- row-sharded item table */
/* Embedding-heavy configuration (item table larger than one GPU should hold, row-sharded
 * over the ranks): the caller exchanges the batch's unique item ids with the owning ranks
 * (all-to-all), each owner gathers its rows with sort_gather_rows, the rows come back and
 * form a batch-local table; sort_set_item_table makes the tokenizer read item rows from it
 * (ids in the batch are then indices into it) until it is reset with rows = NULL.
 * Replaces the Eigen row copies of history_concat_row / candidate_concat_row
 * (tokenizer.cpp:95-127) against a table the process does not own. rows: device bf16
 * [n_rows, item_dim]. */
int sort_set_item_table(SortHandle h, const void* rows, int64_t n_rows);
/* out[i] = table[ids[i]] (device pointers; row_bytes a multiple of 16) on `stream`; status 1
 * if an id is outside [0, n_rows). */
int sort_gather_rows(const void* table, int64_t n_rows, int32_t row_bytes, const int64_t* ids,
                     int64_t n, void* out, void* stream);

/* ---- the exchange itself, in the library (replaces a host-side dedupe + torch all-to-all).
 * One SortExchange per rank. Transports: NCCL (sort_nccl_unique_id on rank 0, the 128 bytes
 * broadcast by the caller's own channel, then sort_exchange_create_nccl on every rank;
 * libnccl.so.2 is resolved from the process at run time) or a host callback (payloads staged
 * through host memory; any host collective, several ranks may share one GPU). */
typedef struct SortExchange_* SortExchange;
/* all-to-all-v of bytes between the `world` ranks: send holds world consecutive blocks of
 * send_bytes[p] bytes (block p goes to rank p), recv receives recv_bytes[p] from rank p. */
typedef int (*sort_alltoallv_fn)(void* ctx, const void* send, const int64_t* send_bytes, void* recv,
                                 const int64_t* recv_bytes, int world);
/* in-place sum over the ranks of n floats */
typedef int (*sort_allreduce_fn)(void* ctx, float* buf, int64_t n);
int sort_nccl_unique_id(void* out_128_bytes);
int sort_exchange_create_nccl(const void* unique_id_128_bytes, int rank, int world, int device, SortExchange* out);
int sort_exchange_create_host(sort_alltoallv_fn fn, sort_allreduce_fn reduce_fn, void* ctx, int rank, int world,
                              int device, SortExchange* out);
int sort_exchange_destroy(SortExchange x);
/* Row-sharded lookup: rank r owns table rows [r R, (r+1) R) as `shard` (device, row_bytes per
 * row, R = rows_per_rank); ids (device int32 [n], global row ids) -> out_rows (device
 * [n, row_bytes]) with out_rows[i] = table[ids[i]], through two all-to-all exchanges on
 * `stream`. Every rank calls it (collective). An id outside [0, world R) on ANY rank makes
 * every rank return status 1 (ConfigError) before any payload moves (tokenizer.cpp:14-19).
 * Feed out_rows to sort_set_item_table with ids replaced by their positions. */
int sort_exchange_lookup(SortExchange x, const void* shard, int64_t rows_per_rank, int32_t row_bytes,
                         const int32_t* ids, int64_t n, void* out_rows, void* stream);
/* Data-parallel gradient sum: buf (device fp32 [n]) summed over the ranks in place (training). */
int sort_exchange_allreduce_f32(SortExchange x, float* buf, int64_t n, void* stream);

/* ---------------------------------------------------------------- request ingest */
/* The reference's JSONL dataset (schema "rankformer.dataset" v1, read_dataset,
 * dataset_io.cpp:58-162) parsed on the host with its validation rules; errors are status 1
 * with "dataset line N, field 'F': what" (DatasetFormatError). Batches are packed into
 * pinned SoA arrays owned by the dataset (valid until the next sort_dataset_batch call):
 * records [first, first + count) must all have n_hist events, n_cand candidates and
 * n_profile_fields profile values (one handle serves one geometry). labels [count, n_cand,
 * 3] (click, cart, purchase) and request_ids [count] are optional. */
typedef struct SortDataset_* SortDataset;
int sort_dataset_open(const char* path, SortDataset* out);
void sort_dataset_close(SortDataset d);
int64_t sort_dataset_size(SortDataset d);
int sort_dataset_batch(SortDataset d, int64_t first, int32_t count, int32_t n_hist, int32_t n_cand,
                       int32_t n_profile_fields, SortBatch* batch, float* labels, int64_t* request_ids);

/* Kernel-selection knobs for A/B tests (no reference counterpart; defaults are the fastest
 * path): "fused_tail" (1 = one k_block_tail launch per block for Wo + residual + SwishGLU FFN
 * + residual where the shape allows it, 0 = the three separate GEMMs); "tail_pair" (1 = run
 * that kernel as CTA pairs with cta_group::2 MMAs, M = 256 per pair and the weights split by
 * N; 0 = single CTA, the default: measured faster on B200); "qkvg_pair" (the QKVG projection
 * GEMM as CTA pairs, default 0 for the same reason); "attn_bwd_mma" (1 = tensor-core
 * attention backward, the default; 0 = the fp32 SIMT kernels); "moe_fused" (1 = one fused expert kernel per MoE layer, the hidden
 * chunk kept in TMEM, the default; 0 = the grouped [gate|up] and down GEMM pair);
 * "graphs" (1 = replay the
 * inference forward from a CUDA graph per (batch size, input slot, item table), the default;
 * 0 = eager launches); "head_tc" (1 = the ranking head on tcgen05 with the fp32 weights split
 * into three exact bf16 pieces, the default; 0 = the fp32 SIMT head); "attn_prescale",
 * "ce_tc", "pre_proj_tc", "stream_gemm", "train_cublas". Status 1 on an
 * unknown name. */
int sort_set_option(SortHandle h, const char* name, int32_t value);

/* ---- pre-training (config field pretrain = 1) ---------------------------------------------
 * pretrain_forward of a batch of click sequences (hist_* arrays, n_hist
 * clicks each; req_ts/profile/cand_item unused): for every position t < n_hist of sequence
 * b, lse[b, t] = log sum_v exp z[v] and target_logit[b, t] = z[click_t.item] with
 * z = (RMSNorm(x_t; final_norm.gain) . pretrain.proj) . item_table^T over the full vocabulary.
 * The next-item cross entropy of position t is lse - target_logit. Pointers follow
 * sort_forward's host/device convention; outputs are [batch, n_hist] fp32. */
int sort_pretrain_forward(SortHandle h, const SortBatch* batch, int inputs_on_device, float* lse,
                          float* target_logit, int outputs_on_device);

/* ---- MoE FFN (config fields moe_*) ------------------------------------
 * Routing of layer `layer` in the last forward: sel/weights [rows, moe_topk] host buffers
 * (either may be NULL), rows = batch * l_q(layer) in the forward's row order; selection in
 * descending biased score, weights = renormalised raw sigmoid scores (route_topk,
 * SPEC.md:305-315). `capacity_rows` is the row capacity of sel/weights: ConfigError when the
 * last forward routed more rows. `rows_out` (may be NULL) receives the routed row count, so a
 * caller can size its buffers with a first call passing sel = weights = NULL. */
int sort_moe_routing(SortHandle h, int layer, int32_t capacity_rows, int32_t* rows_out, int32_t* sel,
                     float* weights);
/* Expert-load histogram [moe_experts] of layer `layer` in the last forward (update_balance
 * input). */
int sort_moe_load(SortHandle h, int layer, int64_t* load);
/* update_balance, DeepSeek style, on every layer from the last forward's loads:
 * router_bias_e -= gamma * sign(load_e - mean load) (gamma = 1e-3 default). */
int sort_moe_update_bias(SortHandle h, double gamma);
/* Op-level entry (moe_forward, SPEC.md:316-324 inside the block residual):
 * out = x + MoE(RMSNorm(x; block.<layer>.ffn_norm)) for `rows` host rows [rows, d], x rounded
 * to bf16 first (the residual stream's type), out read back from bf16. */
int sort_moe_forward(SortHandle h, int layer, const float* x, int rows, float* out);

#ifdef __cplusplus
}
#endif

#endif /* SORT_B200_H_ */
