// SPDX-License-Identifier: Apache-2.0
// Operator-level entries behind the reference's free functions and AttentionLayer
// (include/rankformer/reference_api.hpp binds them with the reference signatures):
//
//   rmsnorm_forward / rmsnorm_backward (norm.hpp:17-45)   sort_op_rmsnorm / sort_op_rmsnorm_backward
//   rope_apply (rope.hpp:13-40)                            sort_op_rope
//   AttentionLayer::forward / ::backward                   sort_op_attention_layer
//     (attention.hpp:58-63, attention.cpp:71-202)
//
// Each call is self-contained (no model handle): host fp32 in, host fp32 out, the work on the
// device. The attention layer runs the same kernels as the model's training step: tcgen05
// streaming GEMMs for the projections and their gradients, k_qkv_prep (QKNorm + RoPE + head
// layout + sigmoid gate), k_attention saving LSE and the pre-gate output, the tcgen05 attention
// backward (attn_bwd.cuh) and the fused QKNorm/RoPE backward. Included at the end of runtime.cu.

// ---------------------------------------------------------------- row kernels (fp32)
// y = x / rms(x) * gain, inv = 1 / sqrt(mean(x^2) + eps) (norm.hpp:17-29). Warp per row.
__global__ void k_op_rmsnorm(const float* __restrict__ x, const float* __restrict__ gain, int rows, int cols,
                             float* __restrict__ y, float* __restrict__ inv_out) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= rows) return;
  const float* xr = x + static_cast<size_t>(w) * cols;
  float ss = 0.f;
  for (int c = lane; c < cols; c += 32) ss = fmaf(xr[c], xr[c], ss);
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = rsqrtf(ss / static_cast<float>(cols) + 1e-6f);
  if (lane == 0) inv_out[w] = inv;
  for (int c = lane; c < cols; c += 32) y[static_cast<size_t>(w) * cols + c] = xr[c] * inv * gain[c];
}

// dx = (dy*g - <dy*g, xhat>/n * xhat) * inv (norm.hpp:32-45). Warp per row.
__global__ void k_op_rmsnorm_dx(const float* __restrict__ dy, const float* __restrict__ x,
                                const float* __restrict__ inv, const float* __restrict__ gain, int rows, int cols,
                                float* __restrict__ dx) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= rows) return;
  const size_t o = static_cast<size_t>(w) * cols;
  const float iv = inv[w];
  float pr = 0.f;
  for (int c = lane; c < cols; c += 32) pr = fmaf(dy[o + c] * gain[c], x[o + c] * iv, pr);
  for (int k = 16; k; k >>= 1) pr += __shfl_xor_sync(0xffffffffu, pr, k);
  const float proj = pr / static_cast<float>(cols);
  for (int c = lane; c < cols; c += 32) dx[o + c] = (dy[o + c] * gain[c] - proj * x[o + c] * iv) * iv;
}

// dgain[c] += sum_r dy[r, c] * xhat[r, c]: one thread per column, rows summed in order
// (deterministic; coalesced across the warp's columns).
__global__ void k_op_rmsnorm_dgain(const float* __restrict__ dy, const float* __restrict__ x,
                                   const float* __restrict__ inv, int rows, int cols, float* __restrict__ dgain) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float acc = 0.f;
  for (int r = 0; r < rows; ++r) {
    const size_t o = static_cast<size_t>(r) * cols + c;
    acc = fmaf(dy[o], x[o] * inv[r], acc);
  }
  dgain[c] = acc;
}

// rope_apply (rope.hpp:13-40): pairs (2j, 2j+1) rotated by pos * theta^(-2j/dim); the angle and
// its sine / cosine in fp64 like the reference (positions reach 4e3 rad), the product in fp32.
__global__ void k_op_rope(const float* __restrict__ x, const int32_t* __restrict__ pos, int rows, int dim,
                          double theta, int inverse, float* __restrict__ out) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= rows) return;
  const double p = static_cast<double>(inverse ? -pos[w] : pos[w]);
  const size_t o = static_cast<size_t>(w) * dim;
  for (int j = lane; j < dim / 2; j += 32) {
    const double ang = p * pow(theta, -2.0 * j / static_cast<double>(dim));
    double s, c;
    sincos(ang, &s, &c);
    const float x0 = x[o + 2 * j], x1 = x[o + 2 * j + 1];
    out[o + 2 * j] = static_cast<float>(c) * x0 - static_cast<float>(s) * x1;
    out[o + 2 * j + 1] = static_cast<float>(s) * x0 + static_cast<float>(c) * x1;
  }
}

// ---------------------------------------------------------------- bare op context
// A Handle without a model: device, SM count and an own stream (the op-level entries).
static void op_context(Handle& h) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  h.device = dev;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) throw RuntimeFailure("requires an sm_100 GPU");
  h.num_sms = prop.multiProcessorCount;
  CK(cudaStreamCreateWithFlags(&h.stream, cudaStreamNonBlocking));
  h.own_stream = true;
}

template <class T>
static T* op_upload(Handle& h, const T* src, size_t n) {
  T* p = h.dalloc<T>(n);
  CK(cudaMemcpyAsync(p, src, n * sizeof(T), cudaMemcpyHostToDevice, h.stream));
  return p;
}
static __nv_bfloat16* op_upload_bf16(Handle& h, const float* src, size_t n) {
  std::vector<__nv_bfloat16> b(n);
  for (size_t i = 0; i < n; ++i) b[i] = f2bf(src[i]);
  __nv_bfloat16* p = h.dalloc<__nv_bfloat16>(n);
  CK(cudaMemcpy(p, b.data(), n * 2, cudaMemcpyHostToDevice));
  return p;
}

// ---------------------------------------------------------------- attention layer op
// One request's attention layer: forward (attention.cpp:71-132) and, when dout is given, the
// backward (attention.cpp:134-202). B = 1, so the head-major layouts are [H, R, dk].
static void attn_layer_op(int d, int H, double theta, int l_in, int l_q, const float* xn, const int32_t* query_rows,
                          const int32_t* lo, const int32_t* hi, const int32_t* self_idx, const int32_t* pos,
                          const float* const* w, float* out, const float* dout, float* dxn, float* const* dw) {
  if (H < 1 || d % H != 0) throw ConfigError("attention: model_dim must be a positive multiple of heads");
  const int dk = d / H;
  if (dk != 16 && dk != 32 && dk != 64) throw ConfigError("attention op: head dim must be 16, 32 or 64");
  if (d % 32 != 0 || d > 1024) throw ConfigError("attention op: model_dim must be a multiple of 32, <= 1024");
  if (dout && d > 256) throw ConfigError("attention op backward: model_dim <= 256");
  if (l_q < 1 || l_in < l_q) throw ConfigError("attention op: need 1 <= l_q <= l_in");
  for (int i = 0; i < 7; ++i)
    if (!w[i]) throw ConfigError("attention op: missing weight");
  for (int r = 0; r < l_q; ++r) {
    if (query_rows[r] < 0 || query_rows[r] >= l_in || (r && query_rows[r] <= query_rows[r - 1]))
      throw ConfigError("attention op: query_rows must be strictly increasing indices into xn");
    const bool iv = lo[r] <= hi[r];
    if ((iv && (lo[r] < 0 || hi[r] >= l_in)) || self_idx[r] < -1 || self_idx[r] >= l_in)
      throw ConfigError("attention op: mask entry out of range");
    if (!iv && self_idx[r] < 0) throw ConfigError("attention op: a query row sees no key");
  }
  int max_pos = 0;
  for (int i = 0; i < l_in; ++i) {
    if (pos[i] < 0) throw ConfigError("attention op: negative position id");
    max_pos = std::max(max_pos, pos[i]);
  }
  Handle h;
  op_context(h);
  h.d = d;
  h.H = H;
  h.dk = dk;
  h.Bmax = 1;
  // RoPE table (rope.hpp:23-38; fp64 angles, fp32 cos/sin) as in finalize
  {
    std::vector<float2> tab(static_cast<size_t>(max_pos + 1) * (dk / 2));
    for (int p = 0; p <= max_pos; ++p)
      for (int j = 0; j < dk / 2; ++j) {
        const double ang = static_cast<double>(p) * std::pow(theta, -2.0 * j / static_cast<double>(dk));
        tab[static_cast<size_t>(p) * (dk / 2) + j] =
            make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
      }
    h.rope = h.upload(tab);
  }
  // the layer plan of this call
  LayerPlan lp;
  lp.l_q = l_q;
  lp.l_kv = l_in;
  lp.query_rows.assign(query_rows, query_rows + l_q);
  lp.q_identity = l_q == l_in;
  lp.lo.assign(lo, lo + l_q);
  lp.hi.assign(hi, hi + l_q);
  lp.self_idx.assign(self_idx, self_idx + l_q);
  lp.pos_kv.assign(pos, pos + l_in);
  for (int r = 0; r < l_q; ++r) lp.pos_q.push_back(pos[query_rows[r]]);
  build_tiles(lp);
  h.layers.resize(1);
  LayerDev& L = h.layers[0];
  L.Rq = l_q;
  L.Rkv = l_in;
  {
    std::vector<int4> meta(static_cast<size_t>(lp.n_qtiles) * 128, make_int4(0, -1, -1, 0));
    for (int r = 0; r < l_q; ++r) meta[r] = make_int4(lp.lo[r], lp.hi[r], lp.self_idx[r], 0);
    L.rowmeta = h.upload(meta);
  }
  L.tile_off = h.upload(lp.tile_off);
  L.tile_code = h.upload(lp.tile_code.empty() ? std::vector<int32_t>{0, 0} : lp.tile_code);
  L.qtile_order = h.upload(lp.qtile_order);
  L.pos_q = h.upload(lp.pos_q);
  L.pos_kv = h.upload(lp.pos_kv);
  L.query_rows = h.upload(lp.query_rows);
  L.gain_q = op_upload(h, w[5], static_cast<size_t>(d));
  L.gain_k = op_upload(h, w[6], static_cast<size_t>(d));
  L.logit_bound = 0.f;  // online-max softmax (no bound assumed for caller-supplied gains)
  h.tl.resize(1);
  auto& T = h.tl[0];
  h.dO16 = h.dalloc<__nv_bfloat16>(static_cast<size_t>(l_q) * d);
  train_layer_buffers(h, lp, L, 1, T);
  train_do_boxes(h, l_q, 1, T);
  h.training = true;
  h.save_to = &T;
  // ---- forward
  const size_t nq = static_cast<size_t>(l_q) * d, nkv = static_cast<size_t>(l_in) * d;
  __nv_bfloat16* xn16 = op_upload_bf16(h, xn, nkv);
  const __nv_bfloat16* xq16 = xn16;
  __nv_bfloat16* xq_buf = nullptr;
  if (!lp.q_identity) {
    xq_buf = h.dalloc<__nv_bfloat16>(nq);
    k_gather_f32<__nv_bfloat16, __nv_bfloat16><<<(l_q + 7) / 8, 256, 0, h.stream>>>(xn16, L.query_rows, l_q, l_in,
                                                                                   l_q, d, xq_buf);
    xq16 = xq_buf;
  }
  // bf16 [in, out] weights; projections [Wq | Wg] on the query rows, [Wk | Wv] on all rows
  std::vector<float> cat(static_cast<size_t>(d) * 2 * d);
  auto cat2 = [&](const float* a, const float* b) {
    for (int r = 0; r < d; ++r) {
      std::copy(a + static_cast<size_t>(r) * d, a + static_cast<size_t>(r + 1) * d, cat.begin() + static_cast<size_t>(r) * 2 * d);
      std::copy(b + static_cast<size_t>(r) * d, b + static_cast<size_t>(r + 1) * d,
                cat.begin() + static_cast<size_t>(r) * 2 * d + d);
    }
    return op_upload_bf16(h, cat.data(), cat.size());
  };
  const __nv_bfloat16* Wqg = cat2(w[0], w[3]);
  const __nv_bfloat16* Wkv = cat2(w[1], w[2]);
  const __nv_bfloat16* Wo16 = op_upload_bf16(h, w[4], static_cast<size_t>(d) * d);
  __nv_bfloat16* pqg = h.dalloc<__nv_bfloat16>(2 * nq);
  __nv_bfloat16* pkv = h.dalloc<__nv_bfloat16>(2 * nkv);
  gemm_rm16(h, false, false, l_q, 2 * d, d, xq16, d, Wqg, 2 * d, pqg, 2 * d, true);
  gemm_rm16(h, false, false, l_in, 2 * d, d, xn16, d, Wkv, 2 * d, pkv, 2 * d, true);
  qkv_prep(h, pqg, 2 * d, l_q, l_q, H, dk, 0, L.pos_q, L.gain_q, T.q);
  qkv_prep(h, pkv, 2 * d, l_in, l_in, H, dk, 1, L.pos_kv, L.gain_k, T.k);
  qkv_prep(h, pkv + d, 2 * d, l_in, l_in, H, dk, 2, nullptr, nullptr, T.v);
  qkv_prep(h, pqg + d, 2 * d, l_q, l_q, H, dk, 3, nullptr, nullptr, T.g);
  check_launch("attention op projections");
  h.Hg = h.dalloc<__nv_bfloat16>(nq);
  launch_attention(h, L, lp, 1);  // gated output -> Hg; LSE and the pre-gate output -> T
  float* out_d = h.dalloc<float>(nq);
  gemm_rm16(h, false, false, l_q, d, d, h.Hg, d, Wo16, d, out_d, d, false);
  check_launch("attention op output projection");
  CK(cudaMemcpyAsync(out, out_d, nq * 4, cudaMemcpyDeviceToHost, h.stream));
  if (!dout) {
    CK(cudaStreamSynchronize(h.stream));
    return;
  }
  // ---- backward (attention.cpp:134-202); weight gradients in fp32 (dw order: wq wk wv wg wo gq gk)
  float* g[7];
  const size_t gsz[7] = {static_cast<size_t>(d) * d, static_cast<size_t>(d) * d, static_cast<size_t>(d) * d,
                         static_cast<size_t>(d) * d, static_cast<size_t>(d) * d, static_cast<size_t>(d),
                         static_cast<size_t>(d)};
  for (int i = 0; i < 7; ++i) {
    g[i] = h.dalloc<float>(gsz[i]);
    CK(cudaMemsetAsync(g[i], 0, gsz[i] * 4, h.stream));
  }
  const __nv_bfloat16* Wq16 = op_upload_bf16(h, w[0], static_cast<size_t>(d) * d);
  const __nv_bfloat16* Wk16 = op_upload_bf16(h, w[1], static_cast<size_t>(d) * d);
  const __nv_bfloat16* Wv16 = op_upload_bf16(h, w[2], static_cast<size_t>(d) * d);
  const __nv_bfloat16* Wg16 = op_upload_bf16(h, w[3], static_cast<size_t>(d) * d);
  const __nv_bfloat16* dout16 = op_upload_bf16(h, dout, nq);
  __nv_bfloat16* Hm = h.dalloc<__nv_bfloat16>(nq);
  float* dH = h.dalloc<float>(nq);
  float* dO = h.dalloc<float>(nq);
  __nv_bfloat16* dgraw = h.dalloc<__nv_bfloat16>(nq);
  float* Dd = h.dalloc<float>(static_cast<size_t>(H) * l_q);
  k_gate_fwd<__nv_bfloat16><<<ew_grid(nq), 256, 0, h.stream>>>(T.g, T.o_pre, nq, Hm);
  gemm_rm16(h, true, false, d, d, l_q, Hm, d, dout16, d, g[4], d, false);
  gemm_rm16(h, false, true, l_q, d, d, dout16, d, Wo16, d, dH, d, false);
  k_gate_bwd_rows<<<warp_rows_grid(l_q), 256, 0, h.stream>>>(dH, T.g, T.o_pre, l_q, l_q, H, dk, dO, h.dO16, dgraw, Dd);
  gemm_rm16(h, true, false, d, d, l_q, xq16, d, dgraw, d, g[3], d, false);
  float* dxq = h.dalloc<float>(nq);
  gemm_rm16(h, false, true, l_q, d, d, dgraw, d, Wg16, d, dxq, d, false);
  float* dQ = h.dalloc<float>(nq);
  float* dK = h.dalloc<float>(nkv);
  float* dV = h.dalloc<float>(nkv);
  __nv_bfloat16* dQ16 = h.dalloc<__nv_bfloat16>(nq);
  __nv_bfloat16* dK16 = h.dalloc<__nv_bfloat16>(nkv);
  __nv_bfloat16* dV16 = h.dalloc<__nv_bfloat16>(nkv);
  attn_core_backward_tc(h, L, T, 1, Dd, dQ, dK, dV, dV16);
  // QKNorm + RoPE backward against the recomputed raw projections
  float* raw = h.dalloc<float>(nkv);
  gemm_rm16(h, false, false, l_q, d, d, xq16, d, Wq16, d, raw, d, false);
  k_qknorm_rope_bwd_v<1><<<std::max(1, std::min((l_q + 7) / 8, 4 * h.num_sms)), 256, d * 4, h.stream>>>(
      dQ, raw, l_q, l_q, L.pos_q, h.rope, H, dk, L.gain_q, dQ, g[5], dQ16);
  gemm_rm16(h, false, false, l_in, d, d, xn16, d, Wk16, d, raw, d, false);
  k_qknorm_rope_bwd_v<1><<<std::max(1, std::min((l_in + 7) / 8, 4 * h.num_sms)), 256, d * 4, h.stream>>>(
      dK, raw, l_in, l_in, L.pos_kv, h.rope, H, dk, L.gain_k, dK, g[6], dK16);
  check_launch("attention op qknorm/rope backward");
  gemm_rm16(h, true, false, d, d, l_q, xq16, d, dQ16, d, g[0], d, false);
  gemm_rm16(h, true, false, d, d, l_in, xn16, d, dK16, d, g[1], d, false);
  gemm_rm16(h, true, false, d, d, l_in, xn16, d, dV16, d, g[2], d, false);
  gemm_rm16(h, false, true, l_q, d, d, dQ16, d, Wq16, d, dxq, d, false, 1.f);
  float* dxn_d = h.dalloc<float>(nkv);
  gemm_rm16(h, false, true, l_in, d, d, dK16, d, Wk16, d, dxn_d, d, false);
  gemm_rm16(h, false, true, l_in, d, d, dV16, d, Wv16, d, dxn_d, d, false, 1.f);
  k_scatter_add_rows<<<(l_q + 7) / 8, 256, 0, h.stream>>>(dxq, L.query_rows, 1, l_q, l_in, d, dxn_d);
  check_launch("attention op backward");
  CK(cudaMemcpyAsync(dxn, dxn_d, nkv * 4, cudaMemcpyDeviceToHost, h.stream));
  std::vector<std::vector<float>> gh(7);
  for (int i = 0; i < 7; ++i) {
    if (!dw || !dw[i]) continue;  // frozen parameter (params.hpp:15-25): no gradient
    gh[i].resize(gsz[i]);
    CK(cudaMemcpyAsync(gh[i].data(), g[i], gsz[i] * 4, cudaMemcpyDeviceToHost, h.stream));
  }
  CK(cudaStreamSynchronize(h.stream));
  for (int i = 0; i < 7; ++i)
    for (size_t k = 0; k < gh[i].size(); ++k) dw[i][k] += gh[i][k];
}

extern "C" {

int sort_op_rmsnorm(int32_t rows, int32_t cols, const float* x, const float* gain, float* y, float* inv_rms) {
  return api([&] {
    if (rows < 0 || cols < 1 || (rows && (!x || !gain || !y || !inv_rms))) throw ConfigError("rmsnorm: bad arguments");
    if (rows == 0) return;
    Handle h;
    op_context(h);
    const size_t n = static_cast<size_t>(rows) * cols;
    const float* xd = op_upload(h, x, n);
    const float* gd = op_upload(h, gain, static_cast<size_t>(cols));
    float* yd = h.dalloc<float>(n);
    float* id = h.dalloc<float>(static_cast<size_t>(rows));
    k_op_rmsnorm<<<warp_rows_grid(rows), 256, 0, h.stream>>>(xd, gd, rows, cols, yd, id);
    check_launch("rmsnorm op");
    CK(cudaMemcpyAsync(y, yd, n * 4, cudaMemcpyDeviceToHost, h.stream));
    CK(cudaMemcpyAsync(inv_rms, id, static_cast<size_t>(rows) * 4, cudaMemcpyDeviceToHost, h.stream));
    CK(cudaStreamSynchronize(h.stream));
  });
}

int sort_op_rmsnorm_backward(int32_t rows, int32_t cols, const float* dy, const float* x, const float* inv_rms,
                             const float* gain, float* dx, float* dgain) {
  return api([&] {
    if (rows < 0 || cols < 1 || !gain || !dgain || (rows && (!dy || !x || !inv_rms || !dx)))
      throw ConfigError("rmsnorm backward: bad arguments");
    if (rows == 0) return;
    Handle h;
    op_context(h);
    const size_t n = static_cast<size_t>(rows) * cols;
    const float* dyd = op_upload(h, dy, n);
    const float* xd = op_upload(h, x, n);
    const float* id = op_upload(h, inv_rms, static_cast<size_t>(rows));
    const float* gd = op_upload(h, gain, static_cast<size_t>(cols));
    float* dxd = h.dalloc<float>(n);
    float* dgd = h.dalloc<float>(static_cast<size_t>(cols));
    k_op_rmsnorm_dx<<<warp_rows_grid(rows), 256, 0, h.stream>>>(dyd, xd, id, gd, rows, cols, dxd);
    k_op_rmsnorm_dgain<<<(cols + 127) / 128, 128, 0, h.stream>>>(dyd, xd, id, rows, cols, dgd);
    check_launch("rmsnorm backward op");
    std::vector<float> dg(static_cast<size_t>(cols));
    CK(cudaMemcpyAsync(dx, dxd, n * 4, cudaMemcpyDeviceToHost, h.stream));
    CK(cudaMemcpyAsync(dg.data(), dgd, dg.size() * 4, cudaMemcpyDeviceToHost, h.stream));
    CK(cudaStreamSynchronize(h.stream));
    for (int c = 0; c < cols; ++c) dgain[c] += dg[static_cast<size_t>(c)];  // accumulates (norm.hpp:39)
  });
}

int sort_op_rope(int32_t rows, int32_t dim, const float* x, const int32_t* position_ids, double theta_base,
                 int32_t inverse, float* out) {
  return api([&] {
    if (dim % 2 != 0) throw ConfigError("rope_apply: head dim must be even");
    if (rows < 0 || dim < 0 || (rows && dim && (!x || !position_ids || !out))) throw ConfigError("rope_apply: bad arguments");
    if (rows == 0 || dim == 0) return;
    Handle h;
    op_context(h);
    const size_t n = static_cast<size_t>(rows) * dim;
    const float* xd = op_upload(h, x, n);
    const int32_t* pd = op_upload(h, position_ids, static_cast<size_t>(rows));
    float* od = h.dalloc<float>(n);
    k_op_rope<<<warp_rows_grid(rows), 256, 0, h.stream>>>(xd, pd, rows, dim, theta_base, inverse, od);
    check_launch("rope op");
    CK(cudaMemcpyAsync(out, od, n * 4, cudaMemcpyDeviceToHost, h.stream));
    CK(cudaStreamSynchronize(h.stream));
  });
}

int sort_op_attention_layer(int32_t model_dim, int32_t heads, double rope_theta, int32_t qknorm, int32_t gate,
                            int32_t l_in, int32_t l_q, const float* xn, const int32_t* query_rows, const int32_t* lo,
                            const int32_t* hi, const int32_t* self_idx, const int32_t* position_ids,
                            const float* const* weights, float* out, const float* dout, float* dxn,
                            float* const* dweights) {
  return api([&] {
    if (!qknorm || !gate)
      throw ConfigError("attention op: the SORT attention is built with qknorm = gate = 1 (AttentionSettings)");
    if (!xn || !query_rows || !lo || !hi || !self_idx || !position_ids || !weights || !out || (dout && !dxn))
      throw ConfigError("attention op: bad arguments");
    attn_layer_op(model_dim, heads, rope_theta, l_in, l_q, xn, query_rows, lo, hi, self_idx, position_ids, weights,
                  out, dout, dxn, dweights);
  });
}

}  // extern "C"
