// SPDX-License-Identifier: Apache-2.0
// Training backward of the SORT scoring path (the builder's GPU restatement of
// AttentionLayer::backward, attention.cpp:134-202 with its intended math; rmsnorm_backward,
// norm.hpp:32-45; and the spec's SwishGLU FFN / pre-norm blocks / ranking head,
// SPEC.md:291-299,362-376). The dense GEMMs of the backward are plain library GEMMs
// (cuBLAS, TF32 tensor cores, fp32 gradients, runtime.cu); the kernels here are the
// row-wise pieces in between and the masked attention core backward.
//
// Gradients are fp32. Saved forward activations are the bf16 tensors the inference
// kernels produce (layer input rows, rotated Q/K, V, sigmoid gate, pre-gate attention
// output, x1) plus the attention's per-row log2-sum-exp.
#pragma once

#include "ptx.cuh"

namespace sortk {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// y = RMSNorm(x[src_row(r)]; gain) in fp32, inv_rms per row (norm.hpp:17-29). x is bf16 or
// fp32; rows may be gathered: src row = (r / R) * Rsrc + map[r % R] when map != null.
__device__ __forceinline__ void store_as(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_as(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

template <class T, class O = float>
__global__ void k_rmsnorm_rows(const T* __restrict__ x, const float* __restrict__ gain, int rows, int d,
                               const int32_t* __restrict__ map, int R, int Rsrc, O* __restrict__ y,
                               float* __restrict__ inv_out) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= rows) return;
  size_t src = w;
  if (map) src = static_cast<size_t>(w / R) * Rsrc + map[w % R];
  const T* xr = x + src * d;
  float ss = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float v = static_cast<float>(xr[c]);
    ss = fmaf(v, v, ss);
  }
  ss = warp_sum(ss);
  const float inv = rsqrtf(ss / static_cast<float>(d) + 1e-6f);
  if (inv_out && lane == 0) inv_out[w] = inv;
  if (y) {
    O* yr = y + static_cast<size_t>(w) * d;
    for (int c = lane; c < d; c += 32) store_as(yr + c, static_cast<float>(xr[c]) * inv * (gain ? gain[c] : 1.f));
  }
}

// out[r] = x[(r / R) * Rsrc + map[r % R]] as fp32 (row gather; map = null -> identity).
template <class T, class O = float>
__global__ void k_gather_f32(const T* __restrict__ x, const int32_t* __restrict__ map, int R, int Rsrc, int rows, int d,
                             O* __restrict__ out) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= rows) return;
  size_t src = w;
  if (map) src = static_cast<size_t>(w / R) * Rsrc + map[w % R];
  for (int c = lane; c < d; c += 32) store_as(out + static_cast<size_t>(w) * d + c, static_cast<float>(x[src * d + c]));
}

// rmsnorm_backward (norm.hpp:32-45): dx = (dy*g - <dy*g, xhat>/n * xhat) * inv, dgain +=
// sum_r dy*xhat. x is bf16 [rows, d]; dx is written (accum = 0) or added (accum = 1).
// 8 rows per warp, dgain partials reduced in shared memory, one atomic per column per CTA.
constexpr int kNormBwdRowsPerWarp = 8;
template <class T>
__global__ void __launch_bounds__(256) k_rmsnorm_bwd(const float* __restrict__ dy, const T* __restrict__ x,
                                                     const float* __restrict__ inv, const float* __restrict__ gain,
                                                     int rows, int d, float* __restrict__ dx, int accum,
                                                     float* __restrict__ dgain) {
  extern __shared__ float sg[];  // [d]
  for (int c = threadIdx.x; c < d; c += blockDim.x) sg[c] = 0.f;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = (blockIdx.x * (blockDim.x >> 5) + warp) * kNormBwdRowsPerWarp;
  constexpr int kMaxCols = 8;  // register-held dgain partials for d <= 256; larger d spill to smem atomics
  float gacc[kMaxCols];
#pragma unroll
  for (int i = 0; i < kMaxCols; ++i) gacc[i] = 0.f;
  for (int r = r0; r < r0 + kNormBwdRowsPerWarp && r < rows; ++r) {
    const float iv = inv[r];
    const float* dyr = dy + static_cast<size_t>(r) * d;
    const T* xr = x + static_cast<size_t>(r) * d;
    float proj = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxCols; ++i) {
      const int c = lane + 32 * i;
      if (c < d) {
        const float xh = static_cast<float>(xr[c]) * iv;
        const float g = dyr[c];
        gacc[i] = fmaf(g, xh, gacc[i]);
        proj = fmaf(g * gain[c], xh, proj);
      }
    }
    for (int c = lane + 32 * kMaxCols; c < d; c += 32) {
      const float xh = static_cast<float>(xr[c]) * iv;
      const float g = dyr[c];
      atomicAdd(&sg[c], g * xh);
      proj = fmaf(g * gain[c], xh, proj);
    }
    proj = warp_sum(proj) / static_cast<float>(d);
    float* dxr = dx + static_cast<size_t>(r) * d;
    for (int c = lane; c < d; c += 32) {
      const float xh = static_cast<float>(xr[c]) * iv;
      const float v = (dyr[c] * gain[c] - proj * xh) * iv;
      dxr[c] = accum ? dxr[c] + v : v;
    }
  }
#pragma unroll
  for (int i = 0; i < kMaxCols; ++i)
    if (lane + 32 * i < d) atomicAdd(&sg[lane + 32 * i], gacc[i]);
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) atomicAdd(&dgain[c], sg[c]);
}

// Vectorised row forms for d <= 256 (d % 8 == 0): one warp per row, lane owns 8 contiguous
// columns (32-byte fp32 / 16-byte bf16 accesses), grid-stride over rows.
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&v)[8]) {
  const int4 r = *reinterpret_cast<const int4*>(p);
  const __nv_bfloat162* q = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(q[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void store8(float* p, const float (&v)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

// y = RMSNorm(x; gain) (fp32 or bf16 out, gain may be null), inv_rms per row (norm.hpp:17-29).
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&v)[8]) {
  *reinterpret_cast<int4*>(p) = make_int4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                                          pack_bf16x2(v[6], v[7]));
}
template <class T, class O = float>
__global__ void __launch_bounds__(256) k_rmsnorm_rows_v(const T* __restrict__ x, const float* __restrict__ gain,
                                                        int rows, int d, O* __restrict__ y,
                                                        float* __restrict__ inv_out) {
  const int lane = threadIdx.x & 31, c0 = lane * 8;
  const bool act = c0 < d;
  float g[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) g[k] = act && gain ? gain[c0 + k] : 1.f;
  const int warps = gridDim.x * (blockDim.x >> 5);
  // one row ahead: the next row's load is in flight while this row is reduced and stored
  int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  float nx[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (act && w < rows) load8(x + static_cast<size_t>(w) * d + c0, nx);
  for (; w < rows; w += warps) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = nx[k];
    if (act && w + warps < rows) load8(x + static_cast<size_t>(w + warps) * d + c0, nx);
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) ss = fmaf(v[k], v[k], ss);
    const float inv = rsqrtf(warp_sum(ss) / static_cast<float>(d) + 1e-6f);
    if (inv_out && lane == 0) inv_out[w] = inv;
    if (y && act) {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] *= inv * g[k];
      store8(y + static_cast<size_t>(w) * d + c0, v);
    }
  }
}

// rmsnorm_backward (norm.hpp:32-45), vectorised form of k_rmsnorm_bwd (same math).
template <class T>
__global__ void __launch_bounds__(256) k_rmsnorm_bwd_v(const float* __restrict__ dy, const T* __restrict__ x,
                                                       const float* __restrict__ inv, const float* __restrict__ gain,
                                                       int rows, int d, float* __restrict__ dx, int accum,
                                                       float* __restrict__ dgain, __nv_bfloat16* __restrict__ dx16) {
  extern __shared__ float sg[];  // [d]
  for (int c = threadIdx.x; c < d; c += blockDim.x) sg[c] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, c0 = lane * 8;
  const bool act = c0 < d;
  float g[8], gacc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    g[k] = act ? gain[c0 + k] : 0.f;
    gacc[k] = 0.f;
  }
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const float iv = inv[r];
    float dyv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, xv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (act) {
      load8(dy + static_cast<size_t>(r) * d + c0, dyv);
      load8(x + static_cast<size_t>(r) * d + c0, xv);
    }
    float proj = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float xh = xv[k] * iv;
      gacc[k] = fmaf(dyv[k], xh, gacc[k]);
      proj = fmaf(dyv[k] * g[k], xh, proj);
    }
    proj = warp_sum(proj) / static_cast<float>(d);
    if (act) {
      float o[8];
      float* dxr = dx + static_cast<size_t>(r) * d + c0;
      if (accum) load8(dxr, o);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float v = (dyv[k] * g[k] - proj * xv[k] * iv) * iv;
        o[k] = accum ? o[k] + v : v;
      }
      store8(dxr, o);
      if (dx16) store8(dx16 + static_cast<size_t>(r) * d + c0, o);  // bf16 copy (a GEMM operand)
    }
  }
  if (act)
#pragma unroll
    for (int k = 0; k < 8; ++k) atomicAdd(&sg[c0 + k], gacc[k]);
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) atomicAdd(&dgain[c], sg[c]);
}

// SwishGLU pieces. GU = [gp | up] (fp32 [M, 2m]).
__device__ __forceinline__ float sigmoid_f(float x) { return 1.f / (1.f + __expf(-x)); }
template <class O = float, class I = float>
__global__ void k_swiglu_z(const I* __restrict__ gu, int M, int m, O* __restrict__ z) {
  // block-rows x columns (no 64-bit division per element)
  for (int r = blockIdx.x; r < M; r += gridDim.x) {
    const I* gr = gu + static_cast<size_t>(r) * 2 * m;
    O* zr = z + static_cast<size_t>(r) * m;
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      const float g = static_cast<float>(gr[j]), u = static_cast<float>(gr[m + j]);
      store_as(zr + j, g * sigmoid_f(g) * u);
    }
  }
}
// bf16 -> bf16 form with 16-byte vectors (m % 8 == 0): the HBM-bound case. The (row, vector)
// pairs are flattened over the grid so every thread has work whatever m is.
template <>
__global__ void k_swiglu_z<__nv_bfloat16, __nv_bfloat16>(const __nv_bfloat16* __restrict__ gu, int M, int m,
                                                         __nv_bfloat16* __restrict__ z) {
  const int m8 = m / 8;
  const size_t total = static_cast<size_t>(M) * m8;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = i / m8;
    const int j = static_cast<int>(i - r * m8);
    const int4* gr = reinterpret_cast<const int4*>(gu + r * 2 * m);
    const int4 gv = gr[j], uv = gr[m8 + j];
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
    const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uv);
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 g = __bfloat1622float2(g2[e]), u = __bfloat1622float2(u2[e]);
      o[e] = pack_bf16x2(g.x * sigmoid_f(g.x) * u.x, g.y * sigmoid_f(g.y) * u.y);
    }
    reinterpret_cast<int4*>(z + r * m)[j] = make_int4(o[0], o[1], o[2], o[3]);
  }
}
// bf16 form of k_swiglu_bwd (16-byte vectors, m % 8 == 0): the training FFN backward keeps its
// [M, m] / [M, 2m] intermediates in bf16.
__global__ void k_swiglu_bwd16(const __nv_bfloat16* __restrict__ dz, const __nv_bfloat16* __restrict__ gu, int M,
                               int m, __nv_bfloat16* __restrict__ dgu) {
  const int m8 = m / 8;
  const size_t total = static_cast<size_t>(M) * m8;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = i / m8;
    const int j = static_cast<int>(i - r * m8);
    const int4* gr = reinterpret_cast<const int4*>(gu + r * 2 * m);
    const int4 gv = gr[j], uv = gr[m8 + j], dv = reinterpret_cast<const int4*>(dz + r * m)[j];
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
    const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uv);
    const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&dv);
    uint32_t og[4], ou[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 g = __bfloat1622float2(g2[e]), u = __bfloat1622float2(u2[e]), dzv = __bfloat1622float2(d2[e]);
      const float sx = sigmoid_f(g.x), sy = sigmoid_f(g.y);
      og[e] = pack_bf16x2(dzv.x * u.x * sx * (1.f + g.x * (1.f - sx)), dzv.y * u.y * sy * (1.f + g.y * (1.f - sy)));
      ou[e] = pack_bf16x2(dzv.x * g.x * sx, dzv.y * g.y * sy);
    }
    int4* o = reinterpret_cast<int4*>(dgu + r * 2 * m);
    o[j] = make_int4(og[0], og[1], og[2], og[3]);
    o[m8 + j] = make_int4(ou[0], ou[1], ou[2], ou[3]);
  }
}

// dgu = [dz * u * swish'(g) | dz * swish(g)], swish'(g) = s (1 + g (1 - s))
__global__ void k_swiglu_bwd(const float* __restrict__ dz, const float* __restrict__ gu, int M, int m,
                             float* __restrict__ dgu) {
  for (int r = blockIdx.x; r < M; r += gridDim.x) {
    const float* gr = gu + static_cast<size_t>(r) * 2 * m;
    const float* dzr = dz + static_cast<size_t>(r) * m;
    float* o = dgu + static_cast<size_t>(r) * 2 * m;
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      const float g = gr[j], u = gr[m + j], dzv = dzr[j];
      const float s = sigmoid_f(g);
      o[j] = dzv * u * s * (1.f + g * (1.f - s));
      o[m + j] = dzv * g * s;
    }
  }
}

// Gate (attention.cpp:124-127): H = G * O (recomputed for the Wo weight gradient). G, O bf16 [M, d].
template <class T = float>
__global__ void k_gate_fwd(const __nv_bfloat16* __restrict__ G, const __nv_bfloat16* __restrict__ O, size_t n,
                           T* __restrict__ H) {
  if ((n & 7) == 0) {  // 16-byte vectors
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n / 8;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
      float g[8], o[8];
      load8(G + i * 8, g);
      load8(O + i * 8, o);
#pragma unroll
      for (int k = 0; k < 8; ++k) g[k] *= o[k];
      store8(H + i * 8, g);
    }
    return;
  }
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    store_as(H + i, __bfloat162float(G[i]) * __bfloat162float(O[i]));
}

// Gate backward and the softmax row term in one pass (attention.cpp:124-131, 144-152, 169-172): per
// row, dO = dH * g (fp32 and a bf16 copy for the tensor-core backward), d(g_raw) =
// dH * o * g (1 - g) (bf16: a GEMM operand only), and D[bh, r] = <dO_head, O_head>. Warp per row, lane owns 8 contiguous
// columns, a head = dk / 8 lanes (shuffle reduction). d <= 256.
__global__ void __launch_bounds__(256) k_gate_bwd_rows(const float* __restrict__ dH, const __nv_bfloat16* __restrict__ G,
                                                       const __nv_bfloat16* __restrict__ O, int rows, int Rq, int H,
                                                       int dk, float* __restrict__ dO, __nv_bfloat16* __restrict__ dO16,
                                                       __nv_bfloat16* __restrict__ dgraw, float* __restrict__ D) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= rows) return;
  const int d = H * dk, c0 = lane * 8;
  const bool act = c0 < d;
  float dot = 0.f;
  if (act) {
    const size_t o = static_cast<size_t>(w) * d + c0;
    const float4 h0 = reinterpret_cast<const float4*>(dH + o)[0], h1 = reinterpret_cast<const float4*>(dH + o)[1];
    const int4 gv = *reinterpret_cast<const int4*>(G + o), ov = *reinterpret_cast<const int4*>(O + o);
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
    const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov);
    const float hh[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
    float dov[8], dgr[8];
    uint32_t pk[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 g = __bfloat1622float2(g2[q]), ob = __bfloat1622float2(o2[q]);
      dov[2 * q] = hh[2 * q] * g.x;
      dov[2 * q + 1] = hh[2 * q + 1] * g.y;
      dgr[2 * q] = hh[2 * q] * ob.x * g.x * (1.f - g.x);
      dgr[2 * q + 1] = hh[2 * q + 1] * ob.y * g.y * (1.f - g.y);
      dot = fmaf(dov[2 * q], ob.x, fmaf(dov[2 * q + 1], ob.y, dot));
      pk[q] = pack_bf16x2(dov[2 * q], dov[2 * q + 1]);
    }
    if (dO) {  // (null: the tensor-core attention backward reads only dO16)
      reinterpret_cast<float4*>(dO + o)[0] = make_float4(dov[0], dov[1], dov[2], dov[3]);
      reinterpret_cast<float4*>(dO + o)[1] = make_float4(dov[4], dov[5], dov[6], dov[7]);
    }
    *reinterpret_cast<int4*>(dgraw + o) = make_int4(pack_bf16x2(dgr[0], dgr[1]), pack_bf16x2(dgr[2], dgr[3]),
                                                    pack_bf16x2(dgr[4], dgr[5]), pack_bf16x2(dgr[6], dgr[7]));
    *reinterpret_cast<int4*>(dO16 + o) = make_int4(pk[0], pk[1], pk[2], pk[3]);
  }
  for (int off = dk / 16; off; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
  if (act && (c0 & (dk - 1)) == 0) {
    const int h = c0 / dk, b = w / Rq, r = w - b * Rq;
    D[(static_cast<size_t>(b) * H + h) * Rq + r] = dot;
  }
}

// ---------------------------------------------------------------- masked attention backward
// Per (request, head): P = exp2(s * scale_log2 - lse2) on visible entries (rows' compact mask
// {lo, hi, self}), dP = dO V^T, dS = P (dP - D), dQ = scale dS K, dK = scale dS^T Q,
// dV = P^T dO (attention.cpp:160-176). Lane-per-row SIMT with fp32 pair math: the q-centric
// kernel gives one query row per lane and streams the block's visible kv rows (broadcast
// loads); the kv-centric kernel gives one kv row per lane and streams the query rows that
// see its block, so neither needs atomics. Work lists (row / column intervals per 32-block)
// come from the host plan.
struct AttnBwdArgs {
  const __nv_bfloat16 *q, *k, *v;  // rotated Q [BH, Rq, dk], rotated K / V [BH, Rkv, dk]
  const float* dO;                 // [B*Rq, H*dk] (row-major, head column blocks)
  const float* lse;                // [BH, Rq] log2-domain
  const float* D;                  // [BH, Rq]
  const int4* rowmeta;             // [Rq] {lo, hi, self, 0}
  const int32_t* blk_off;          // CSR over 32-blocks
  const int2* blk_iv;              // [begin, end) intervals
  float* dq;                       // [B*Rq, H*dk]
  float* dk;                       // [B*Rkv, H*dk]
  float* dv;                       // [B*Rkv, H*dk]
  int BH, H, Rq, Rkv;
  float scale_log2, scale;
};

template <int DK>
__device__ __forceinline__ void load_row_bf16(const __nv_bfloat16* p, float2 (&o)[DK / 2]) {
#pragma unroll
  for (int i = 0; i < DK / 8; ++i) {
    const int4 v = reinterpret_cast<const int4*>(p)[i];
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int e = 0; e < 4; ++e) o[4 * i + e] = __bfloat1622float2(b[e]);
  }
}
template <int DK>
__device__ __forceinline__ float dot2(const float2 (&a)[DK / 2], const float2 (&b)[DK / 2]) {
  float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < DK / 2; i += 2) {
    s0 = ffma2(a[i], b[i], s0);
    s1 = ffma2(a[i + 1], b[i + 1], s1);
  }
  s0 = fadd2(s0, s1);
  return s0.x + s0.y;
}
__device__ __forceinline__ bool row_sees(int4 m, int c) { return (c >= m.x && c <= m.y) || c == m.z; }

// grid: (ceil(Rq / 32), BH), 32 threads. blk lists = kv-column intervals per 32-row q-block.
// kv rows are staged 32 at a time in shared memory by coalesced warp loads and read back
// as broadcasts.
template <int DK>
__global__ void __launch_bounds__(32) k_attn_bwd_dq(const AttnBwdArgs a) {
  __shared__ int4 sk[32][DK / 8], sv[32][DK / 8];
  const int qb = blockIdx.x, bh = blockIdx.y, lane = threadIdx.x;
  const int b = bh / a.H, h = bh - b * a.H;
  const int r = qb * 32 + lane;
  const bool valid = r < a.Rq;
  float2 q[DK / 2], go[DK / 2], acc[DK / 2];
  int4 meta = make_int4(0, -1, -1, 0);
  float lse = 0.f, Dr = 0.f;
  if (valid) {
    load_row_bf16<DK>(a.q + (static_cast<size_t>(bh) * a.Rq + r) * DK, q);
    const float* gp = a.dO + (static_cast<size_t>(b) * a.Rq + r) * a.H * DK + h * DK;
#pragma unroll
    for (int i = 0; i < DK / 2; ++i) go[i] = reinterpret_cast<const float2*>(gp)[i];
    meta = a.rowmeta[r];
    lse = a.lse[static_cast<size_t>(bh) * a.Rq + r];
    Dr = a.D[static_cast<size_t>(bh) * a.Rq + r];
  } else {
#pragma unroll
    for (int i = 0; i < DK / 2; ++i) q[i] = go[i] = make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int i = 0; i < DK / 2; ++i) acc[i] = make_float2(0.f, 0.f);
  const int4* kb = reinterpret_cast<const int4*>(a.k + static_cast<size_t>(bh) * a.Rkv * DK);
  const int4* vb = reinterpret_cast<const int4*>(a.v + static_cast<size_t>(bh) * a.Rkv * DK);
  for (int iv = a.blk_off[qb]; iv < a.blk_off[qb + 1]; ++iv) {
    const int2 range = a.blk_iv[iv];
    for (int c0 = range.x; c0 < range.y; c0 += 32) {
      const int n = min(32, range.y - c0);
      __syncwarp();
      if (lane < n) {
#pragma unroll
        for (int i = 0; i < DK / 8; ++i) {
          sk[lane][i] = kb[static_cast<size_t>(c0 + lane) * (DK / 8) + i];
          sv[lane][i] = vb[static_cast<size_t>(c0 + lane) * (DK / 8) + i];
        }
      }
      __syncwarp();
      for (int jj = 0; jj < n; ++jj) {
        const int c = c0 + jj;
        float2 kk[DK / 2], vv[DK / 2];
        load_row_bf16<DK>(reinterpret_cast<const __nv_bfloat16*>(sk[jj]), kk);
        load_row_bf16<DK>(reinterpret_cast<const __nv_bfloat16*>(sv[jj]), vv);
        if (!valid || !row_sees(meta, c)) continue;
        const float p = exp2f(dot2<DK>(q, kk) * a.scale_log2 - lse);
        const float ds = p * (dot2<DK>(go, vv) - Dr) * a.scale;
        const float2 ds2 = make_float2(ds, ds);
#pragma unroll
        for (int i = 0; i < DK / 2; ++i) acc[i] = ffma2(ds2, kk[i], acc[i]);
      }
    }
  }
  if (valid) {
    float* out = a.dq + (static_cast<size_t>(b) * a.Rq + r) * a.H * DK + h * DK;
#pragma unroll
    for (int i = 0; i < DK / 2; ++i) reinterpret_cast<float2*>(out)[i] = acc[i];
  }
}

// grid: (ceil(Rkv / 32), BH), 32 threads. blk lists = q-row intervals per 32-column kv-block.
// Query rows (Q, dO, lse, D, mask row) are staged 32 at a time in shared memory.
template <int DK>
__global__ void __launch_bounds__(32) k_attn_bwd_dkv(const AttnBwdArgs a) {
  __shared__ int4 sq[32][DK / 8];
  __shared__ float4 sdo[32][DK / 4];
  __shared__ int4 smeta[32];
  __shared__ float2 sld[32];
  const int kb_ = blockIdx.x, bh = blockIdx.y, lane = threadIdx.x;
  const int b = bh / a.H, h = bh - b * a.H;
  const int c = kb_ * 32 + lane;
  const bool valid = c < a.Rkv;
  float2 kk[DK / 2], vv[DK / 2], dk[DK / 2], dv[DK / 2];
  if (valid) {
    load_row_bf16<DK>(a.k + (static_cast<size_t>(bh) * a.Rkv + c) * DK, kk);
    load_row_bf16<DK>(a.v + (static_cast<size_t>(bh) * a.Rkv + c) * DK, vv);
  } else {
#pragma unroll
    for (int i = 0; i < DK / 2; ++i) kk[i] = vv[i] = make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int i = 0; i < DK / 2; ++i) dk[i] = dv[i] = make_float2(0.f, 0.f);
  const int4* qb = reinterpret_cast<const int4*>(a.q + static_cast<size_t>(bh) * a.Rq * DK);
  for (int iv = a.blk_off[kb_]; iv < a.blk_off[kb_ + 1]; ++iv) {
    const int2 range = a.blk_iv[iv];
    for (int r0 = range.x; r0 < range.y; r0 += 32) {
      const int n = min(32, range.y - r0);
      __syncwarp();
      if (lane < n) {
        const int r = r0 + lane;
#pragma unroll
        for (int i = 0; i < DK / 8; ++i) sq[lane][i] = qb[static_cast<size_t>(r) * (DK / 8) + i];
        const float4* gp = reinterpret_cast<const float4*>(a.dO + (static_cast<size_t>(b) * a.Rq + r) * a.H * DK + h * DK);
#pragma unroll
        for (int i = 0; i < DK / 4; ++i) sdo[lane][i] = gp[i];
        smeta[lane] = a.rowmeta[r];
        sld[lane] = make_float2(a.lse[static_cast<size_t>(bh) * a.Rq + r], a.D[static_cast<size_t>(bh) * a.Rq + r]);
      }
      __syncwarp();
      for (int jj = 0; jj < n; ++jj) {
        if (!valid || !row_sees(smeta[jj], c)) continue;
        float2 q[DK / 2], go[DK / 2];
        load_row_bf16<DK>(reinterpret_cast<const __nv_bfloat16*>(sq[jj]), q);
#pragma unroll
        for (int i = 0; i < DK / 4; ++i) {
          const float4 t = sdo[jj][i];
          go[2 * i] = make_float2(t.x, t.y);
          go[2 * i + 1] = make_float2(t.z, t.w);
        }
        const float2 ld = sld[jj];
        const float p = exp2f(dot2<DK>(q, kk) * a.scale_log2 - ld.x);
        const float ds = p * (dot2<DK>(go, vv) - ld.y) * a.scale;
        const float2 ds2 = make_float2(ds, ds), p2 = make_float2(p, p);
#pragma unroll
        for (int i = 0; i < DK / 2; ++i) {
          dk[i] = ffma2(ds2, q[i], dk[i]);
          dv[i] = ffma2(p2, go[i], dv[i]);
        }
      }
    }
  }
  if (valid) {
    const size_t o = (static_cast<size_t>(b) * a.Rkv + c) * a.H * DK + h * DK;
#pragma unroll
    for (int i = 0; i < DK / 2; ++i) {
      reinterpret_cast<float2*>(a.dk + o)[i] = dk[i];
      reinterpret_cast<float2*>(a.dv + o)[i] = dv[i];
    }
  }
}

// ---------------------------------------------------------------- tensor-core attention backward
// FlashAttention-2-style backward on bf16 mma.sync (m16n8k16, fp32 accumulation), one CTA per
// (request*head, 64-row kv block), 4 warps of 16 kv rows each. For every 64-row q block that
// sees the kv block (host list): S^T = K Q^T, P^T = exp2(S^T log2e/sqrt(dk) - lse) masked by the
// compact rows {lo, hi, self}, dP^T = V dO^T, dS^T = P^T (dP^T - D); dV += P^T dO and
// dK += dS^T Q stay in registers across q blocks; dQ += dS K goes through dS^T in shared
// memory and fp32 atomics (several kv blocks contribute to a q block).
struct AttnBwdMmaArgs {
  const __nv_bfloat16 *q, *k, *v;  // [BH, Rq, DK], [BH, Rkv, DK], [BH, Rkv, DK]
  const __nv_bfloat16* dO16;       // [B*Rq, H*DK] bf16
  const float* lse;                // [BH, Rq]
  const float* D;                  // [BH, Rq]
  const int4* rowmeta;             // [Rq]
  const int32_t* qb_off;           // CSR over 64-row kv blocks -> 64-row q blocks
  const int32_t* qb_list;
  float *dq, *dk, *dv;             // dq zeroed by the caller; dk/dv written
  __nv_bfloat16* dv16;             // optional bf16 copy of dv (a GEMM operand)
  int H, Rq, Rkv;
  float scale_log2, scale;
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int DK>
__global__ void __launch_bounds__(128, 4) k_attn_bwd_mma(const AttnBwdMmaArgs a) {
  constexpr int LD = DK + 8;  // padded bf16 row (conflict-free ldmatrix)
  constexpr int LDS = 64 + 8;
  constexpr int NT = DK / 8;  // n-tiles of the dK / dV / dQ accumulators
  constexpr int KS = DK / 16; // k-steps of S^T and dP^T
  // Q / dO (bf16) / lse / D / row metadata of a q block, double-buffered: the next q block's
  // tiles stream in (cp.async) while this one is computed
  constexpr int NBUF = DK <= 32 ? 2 : 1;  // dk = 64: single-buffered (48 KB static smem)
  __shared__ __align__(16) __nv_bfloat16 sK[64 * LD], sV[64 * LD], sQb[NBUF][64 * LD], sOb[NBUF][64 * LD];
  __shared__ __align__(16) __nv_bfloat16 sS[64 * LDS];  // dS^T [kv][q]
  __shared__ __align__(16) float sLb[NBUF][64], sDb[NBUF][64];
  __shared__ __align__(16) int4 sMb[NBUF][64];
  const int kvb = blockIdx.x, bh = blockIdx.y;
  const int b = bh / a.H, h = bh - b * a.H;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int c0 = kvb * 64;
  auto cp16 = [](void* dst, const void* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
  };
  auto cp4 = [](void* dst, const void* src, bool ok) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 4 : 0)
                 : "memory");
  };
  const int it0 = a.qb_off[kvb], it1 = a.qb_off[kvb + 1];
  auto stage = [&](int it, int buf) {
    const int r0 = (a.qb_list[it] & 0x3fffffff) * 64;
    for (int i = tid; i < 64 * (DK / 8); i += 128) {
      const int r = i / (DK / 8), cc = i % (DK / 8);
      const bool ok = r0 + r < a.Rq;
      const int rr = ok ? r0 + r : 0;
      cp16(sQb[buf] + r * LD + cc * 8, a.q + (static_cast<size_t>(bh) * a.Rq + rr) * DK + cc * 8, ok);
      cp16(sOb[buf] + r * LD + cc * 8, a.dO16 + (static_cast<size_t>(b) * a.Rq + rr) * a.H * DK + h * DK + cc * 8, ok);
    }
    for (int i = tid; i < 64; i += 128) {
      const bool ok = r0 + i < a.Rq;
      const size_t li = static_cast<size_t>(bh) * a.Rq + (ok ? r0 + i : 0);
      cp4(&sLb[buf][i], a.lse + li, ok);
      cp4(&sDb[buf][i], a.D + li, ok);
      if (ok) cp16(&sMb[buf][i], a.rowmeta + r0 + i, true);
      else sMb[buf][i] = make_int4(0, -1, -1, 0);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (it0 < it1) stage(it0, 0);
  for (int i = tid; i < 64 * (DK / 8); i += 128) {  // K, V rows of the block (zero past Rkv)
    const int r = i / (DK / 8), cc = i % (DK / 8);
    int4 kv = make_int4(0, 0, 0, 0), vv = kv;
    if (c0 + r < a.Rkv) {
      kv = reinterpret_cast<const int4*>(a.k + (static_cast<size_t>(bh) * a.Rkv + c0 + r) * DK)[cc];
      vv = reinterpret_cast<const int4*>(a.v + (static_cast<size_t>(bh) * a.Rkv + c0 + r) * DK)[cc];
    }
    *reinterpret_cast<int4*>(sK + r * LD + cc * 8) = kv;
    *reinterpret_cast<int4*>(sV + r * LD + cc * 8) = vv;
  }
  float dk[NT][4], dv[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[n][e] = dv[n][e] = 0.f;
  const uint32_t sKa = smem_u32(sK), sVa = smem_u32(sV), sSa = smem_u32(sS);
  const int kv_lo = c0 + warp * 16 + g;  // this thread's two kv rows: kv_lo, kv_lo + 8
  for (int it = it0; it < it1; ++it) {
    const int buf = (it - it0) % NBUF;
    const int qbe = a.qb_list[it];
    const int r0 = (qbe & 0x3fffffff) * 64;
    const bool full = (qbe & 0x40000000) != 0;  // the whole 64 x 64 block is visible (host plan)
    __syncthreads();  // previous iteration done with sS and with the other buffer
    if constexpr (NBUF == 2) {
      if (it + 1 < it1) {
        stage(it + 1, buf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
    } else {
      if (it > it0) stage(it, 0);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const uint32_t sQa = smem_u32(sQb[buf]), sOa = smem_u32(sOb[buf]);
    const float* sL = sLb[buf];
    const float* sD = sDb[buf];
    const int4* sM = sMb[buf];
    // S^T and dP^T: [16 kv (this warp) x 64 q]
    float st[8][4], dp[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[n][e] = dp[n][e] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      uint32_t ak[4], av[4];
      const int arow = warp * 16 + (lane & 15), acol = ks * 16 + (lane >> 4) * 8;
      ldsm_x4(sKa + (arow * LD + acol) * 2, ak);
      ldsm_x4(sVa + (arow * LD + acol) * 2, av);
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // pairs of q n-tiles
        uint32_t bq[4], bo[4];
        const int brow = np * 16 + (lane & 7) + ((lane >> 4) << 3), bcol = ks * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(sQa + (brow * LD + bcol) * 2, bq);
        ldsm_x4(sOa + (brow * LD + bcol) * 2, bo);
        mma16816(st[2 * np], ak, bq[0], bq[1]);
        mma16816(st[2 * np + 1], ak, bq[2], bq[3]);
        mma16816(dp[2 * np], av, bo[0], bo[1]);
        mma16816(dp[2 * np + 1], av, bo[2], bo[3]);
      }
    }
    // P^T, dS^T as bf16 A fragments: C n-tiles 2s, 2s+1 form the k-slice s
    uint32_t pa[4][4], sa[4][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float p[4], ds[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int q = n * 8 + 2 * t4 + (e & 1);
        const int kv = kv_lo + ((e >> 1) << 3);
        bool vis = true;
        if (!full) {
          const int4 m = sM[q];
          vis = kv < a.Rkv && ((kv >= m.x && kv <= m.y) || kv == m.z);
        }
        p[e] = vis ? ex2_approx(st[n][e] * a.scale_log2 - sL[q]) : 0.f;  // argument <= 0 (P <= 1)
        ds[e] = p[e] * (dp[n][e] - sD[q]);
      }
      const int s = n >> 1, hi = n & 1;
      // A fragment regs: {rows g, k 0-7}, {rows g+8, k 0-7}, {rows g, k 8-15}, {rows g+8, k 8-15}
      pa[s][hi * 2 + 0] = pack_bf16x2(p[0], p[1]);
      pa[s][hi * 2 + 1] = pack_bf16x2(p[2], p[3]);
      sa[s][hi * 2 + 0] = pack_bf16x2(ds[0], ds[1]);
      sa[s][hi * 2 + 1] = pack_bf16x2(ds[2], ds[3]);
      const int kl = warp * 16 + g;  // dS^T (bf16) rows kv (local), cols q, for the dQ product
      *reinterpret_cast<uint32_t*>(sS + kl * LDS + n * 8 + 2 * t4) = sa[s][hi * 2 + 0];
      *reinterpret_cast<uint32_t*>(sS + (kl + 8) * LDS + n * 8 + 2 * t4) = sa[s][hi * 2 + 1];
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {  // k = q
#pragma unroll
      for (int np = 0; np < NT / 2; ++np) {  // pairs of dk n-tiles; B from [q][dk] rows -> .trans
        uint32_t bo[4], bq[4];
        const int brow = s * 16 + (lane & 15), bcol = np * 16 + (lane >> 4) * 8;
        ldsm_x4_t(sOa + (brow * LD + bcol) * 2, bo);
        ldsm_x4_t(sQa + (brow * LD + bcol) * 2, bq);
        mma16816(dv[2 * np], pa[s], bo[0], bo[1]);
        mma16816(dv[2 * np + 1], pa[s], bo[2], bo[3]);
        mma16816(dk[2 * np], sa[s], bq[0], bq[1]);
        mma16816(dk[2 * np + 1], sa[s], bq[2], bq[3]);
      }
    }
    __syncthreads();  // dS^T of all warps in smem
    // dQ rows [16 w, 16 w + 16) of the q block = dS (q x 64 kv) . K (64 kv x DK)
    float dq[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) dq[n][e] = 0.f;
#pragma unroll
    for (int s = 0; s < 4; ++s) {  // k = kv
      uint32_t as[4];
      const int arow = s * 16 + (lane & 7) + ((lane >> 4) << 3), acol = warp * 16 + ((lane >> 3) & 1) * 8;
      ldsm_x4_t(sSa + (arow * LDS + acol) * 2, as);
#pragma unroll
      for (int np = 0; np < NT / 2; ++np) {
        uint32_t bk[4];
        const int brow = s * 16 + (lane & 15), bcol = np * 16 + (lane >> 4) * 8;
        ldsm_x4_t(sKa + (brow * LD + bcol) * 2, bk);
        mma16816(dq[2 * np], as, bk[0], bk[1]);
        mma16816(dq[2 * np + 1], as, bk[2], bk[3]);
      }
    }
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int e2 = 0; e2 < 2; ++e2) {  // two adjacent columns per vector reduction
        const int q = r0 + warp * 16 + g + (e2 << 3);
        if (q < a.Rq) {
          float* dst = a.dq + (static_cast<size_t>(b) * a.Rq + q) * a.H * DK + h * DK + n * 8 + 2 * t4;
          asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(dst), "f"(dq[n][2 * e2] * a.scale),
                       "f"(dq[n][2 * e2 + 1] * a.scale)
                       : "memory");
        }
      }
  }
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int e2 = 0; e2 < 2; ++e2) {  // two adjacent columns per store
      const int kv = kv_lo + (e2 << 3);
      if (kv < a.Rkv) {
        const size_t o = (static_cast<size_t>(b) * a.Rkv + kv) * a.H * DK + h * DK + n * 8 + 2 * t4;
        *reinterpret_cast<float2*>(a.dk + o) = make_float2(dk[n][2 * e2] * a.scale, dk[n][2 * e2 + 1] * a.scale);
        *reinterpret_cast<float2*>(a.dv + o) = make_float2(dv[n][2 * e2], dv[n][2 * e2 + 1]);
        if (a.dv16) *reinterpret_cast<uint32_t*>(a.dv16 + o) = pack_bf16x2(dv[n][2 * e2], dv[n][2 * e2 + 1]);
      }
    }
}

// QKNorm + RoPE backward (attention.cpp:177-183): dx_rot -> inverse RoPE at the row's position
// (rope.hpp:13-40, angle -> -angle) -> per-head RMSNorm backward against the raw projection
// `raw` with gain g[h]; drot and draw may alias (each lane reads its elements before writing
// them); draw may be null when only the bf16 copy draw16 is wanted. One warp per row, lane owns 8 contiguous
// elements (4 rotation pairs) of chunk c = lane + 32 i, so a head spans dk / 8 aligned lanes and
// both per-head reductions are 1-3 shuffle steps; 32-byte loads and stores. Gain-gradient
// partials stay in registers across the warp's rows (grid-stride), then one shared-memory
// reduction per CTA. d = H * dk <= 256 * kV.
template <int kV>
__global__ void __launch_bounds__(256) k_qknorm_rope_bwd_v(const float* drot, const float* __restrict__ raw,
                                                           int rows, int R, const int32_t* __restrict__ pos,
                                                           const float2* __restrict__ rope_tab, int H, int dk,
                                                           const float* __restrict__ gain, float* draw,
                                                           float* __restrict__ dgain, __nv_bfloat16* __restrict__ draw16) {
  extern __shared__ float sg[];  // [H * dk]
  const int d = H * dk, d8 = d >> 3;
  for (int c = threadIdx.x; c < d; c += blockDim.x) sg[c] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int e = (lane * 8) & (dk - 1);  // offset inside the head (same for every chunk: 256 % dk == 0)
  float g[kV][8], gacc[kV][8];
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    const int c = lane + 32 * i;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      g[i][k] = c < d8 ? gain[c * 8 + k] : 0.f;
      gacc[i][k] = 0.f;
    }
  }
  const int warps = gridDim.x * (blockDim.x >> 5);
  // one row ahead: the next row's dQ / raw / (cos, sin) loads are in flight while this row is
  // computed and stored (rows are distinct, so the in-place draw == drot stores cannot alias them)
  struct RowIn {
    float4 g[kV][2], x[kV][2], cs[2];
  };
  auto load_row = [&](int w, RowIn& in) {
    const float4* t = reinterpret_cast<const float4*>(rope_tab + static_cast<size_t>(pos[w % R]) * (dk / 2) + e / 2);
    in.cs[0] = t[0];
    in.cs[1] = t[1];
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const int c = lane + 32 * i;
      if (c < d8) {
        const float4* gp = reinterpret_cast<const float4*>(drot + static_cast<size_t>(w) * d + c * 8);
        const float4* xp = reinterpret_cast<const float4*>(raw + static_cast<size_t>(w) * d + c * 8);
        in.g[i][0] = gp[0];
        in.g[i][1] = gp[1];
        in.x[i][0] = xp[0];
        in.x[i][1] = xp[1];
      }
    }
  };
  int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  RowIn cur;
  if (w < rows) load_row(w, cur);
  for (; w < rows; w += warps) {
    RowIn nxt;
    if (w + warps < rows) load_row(w + warps, nxt);
    const float cs[8] = {cur.cs[0].x, cur.cs[0].y, cur.cs[0].z, cur.cs[0].w,
                         cur.cs[1].x, cur.cs[1].y, cur.cs[1].z, cur.cs[1].w};  // (cos, sin) of 4 pairs
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const int c = lane + 32 * i;
      const bool act = c < d8;
      float dq[8], x[8];
      if (act) {
        const float4 g0 = cur.g[i][0], g1 = cur.g[i][1], x0 = cur.x[i][0], x1 = cur.x[i][1];
        const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        x[0] = x0.x; x[1] = x0.y; x[2] = x0.z; x[3] = x0.w;
        x[4] = x1.x; x[5] = x1.y; x[6] = x1.z; x[7] = x1.w;
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // inverse rotation of pair q (rope.hpp:13-40, -angle)
          const float cc = cs[2 * q], sn = cs[2 * q + 1];
          dq[2 * q] = cc * gg[2 * q] + sn * gg[2 * q + 1];
          dq[2 * q + 1] = -sn * gg[2 * q] + cc * gg[2 * q + 1];
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) dq[k] = x[k] = 0.f;
      }
      float ss = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) ss = fmaf(x[k], x[k], ss);
      for (int o = dk / 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const float inv = rsqrtf(ss / static_cast<float>(dk) + 1e-6f);
      float pr = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) pr = fmaf(dq[k] * g[i][k], x[k] * inv, pr);
      for (int o = dk / 16; o; o >>= 1) pr += __shfl_xor_sync(0xffffffffu, pr, o);
      const float proj = pr / static_cast<float>(dk);
      if (act) {
        float out[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float xh = x[k] * inv;
          gacc[i][k] = fmaf(dq[k], xh, gacc[i][k]);
          out[k] = (dq[k] * g[i][k] - proj * xh) * inv;
        }
        if (draw) {  // (null: only the bf16 copy is consumed -- the training GEMMs)
          float4* op = reinterpret_cast<float4*>(draw + static_cast<size_t>(w) * d + c * 8);
          op[0] = make_float4(out[0], out[1], out[2], out[3]);
          op[1] = make_float4(out[4], out[5], out[6], out[7]);
        }
        if (draw16) store8(draw16 + static_cast<size_t>(w) * d + c * 8, out);
      }
    }
    cur = nxt;
  }
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    const int c = lane + 32 * i;
    if (c < d8)
#pragma unroll
      for (int k = 0; k < 8; ++k) atomicAdd(&sg[c * 8 + k], gacc[i][k]);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) atomicAdd(&dgain[c], sg[c]);
}

// dst[b*Rdst + map[r]] (+)= src[b*Rsrc + r] over B*Rsrc rows (unique destinations).
__global__ void k_scatter_add_rows(const float* __restrict__ src, const int32_t* __restrict__ map, int B, int Rsrc,
                                   int Rdst, int d, float* __restrict__ dst) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= B * Rsrc) return;
  const int b = w / Rsrc, r = w - b * Rsrc;
  float* o = dst + (static_cast<size_t>(b) * Rdst + map[r]) * d;
  const float* s = src + static_cast<size_t>(w) * d;
  if ((d & 3) == 0) {  // 16-byte vectors
    for (int c = lane; c < d / 4; c += 32) {
      const float4 a = reinterpret_cast<const float4*>(s)[c];
      float4 t = reinterpret_cast<float4*>(o)[c];
      t.x += a.x;
      t.y += a.y;
      t.z += a.z;
      t.w += a.w;
      reinterpret_cast<float4*>(o)[c] = t;
    }
  } else {
    for (int c = lane; c < d; c += 32) o[c] += s[c];
  }
}

// Column sums: out[c] += sum_r a[r, c] (bias gradients).
// Block (32, 8): 32 columns x 8 row lanes, 4 independent partial sums per thread, the 8 row
// lanes combined in shared memory, one atomic per column per block.
__global__ void __launch_bounds__(256) k_colsum(const float* __restrict__ a, int rows, int cols,
                                                float* __restrict__ out) {
  __shared__ float red[8][33];
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int r0 = blockIdx.y * 8 + threadIdx.y, rs = gridDim.y * 8;
  float s[4] = {0.f, 0.f, 0.f, 0.f};
  if (c < cols) {
    int r = r0, k = 0;
    for (; r < rows; r += rs, k = (k + 1) & 3) s[k] += a[static_cast<size_t>(r) * cols + c];
  }
  red[threadIdx.y][threadIdx.x] = (s[0] + s[1]) + (s[2] + s[3]);
  __syncthreads();
  if (threadIdx.y == 0 && c < cols) {
    float t = 0.f;
#pragma unroll
    for (int y = 0; y < 8; ++y) t += red[y][threadIdx.x];
    atomicAdd(&out[c], t);
  }
}

// ---------------------------------------------------------------- tokenizer backward
// (Tokenizer::backward, tokenizer.cpp:286-352): d(concat) rows scattered into the small
// feature tables. History: [item | action | scene | time] (item frozen, skipped); profile:
// the field's table. Per-CTA shared-memory accumulation (the tables have a few hundred
// entries that every row hits), one global atomic per entry per CTA.
struct TokTableGrads {
  float* action;  // [n_actions, action_dim]
  float* scene;   // [n_scenes, scene_dim]
  float* time;    // [n_tb, time_dim]
  float* prof[SORT_MAX_PROFILE_FIELDS];  // per field [vocab_f, prof_dim]
};
// K: the row stride of dcat (>= the concat width)
__global__ void __launch_bounds__(256) k_tok_table_scatter(const float* __restrict__ dcat, int group, int n, int K,
                                                           const int32_t* __restrict__ hist_action,
                                                           const int32_t* __restrict__ hist_scene,
                                                           const int32_t* __restrict__ hist_time,
                                                           const int32_t* __restrict__ profile, int P, int item_dim,
                                                           int action_dim, int scene_dim, int time_dim, int n_actions,
                                                           int n_scenes, int n_tb, const int* __restrict__ prof_vocab,
                                                           int prof_dim, TokTableGrads g) {
  extern __shared__ float acc[];
  int total = 0;
  int prof_off[SORT_MAX_PROFILE_FIELDS] = {0};
  if (group == 0) {
    total = n_actions * action_dim + n_scenes * scene_dim + n_tb * time_dim;
  } else {
    for (int f = 0; f < P; ++f) {
      prof_off[f] = total;
      total += prof_vocab[f] * prof_dim;
    }
  }
  for (int i = threadIdx.x; i < total; i += blockDim.x) acc[i] = 0.f;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = blockIdx.x * 8 + warp; r < n; r += gridDim.x * 8) {
    const float* row = dcat + static_cast<size_t>(r) * K;
    if (group == 0) {
      const int a = hist_action[r], sc = hist_scene[r], tb = hist_time[r];
      for (int j = lane; j < action_dim; j += 32) atomicAdd(&acc[a * action_dim + j], row[item_dim + j]);
      for (int j = lane; j < scene_dim; j += 32)
        atomicAdd(&acc[n_actions * action_dim + sc * scene_dim + j], row[item_dim + action_dim + j]);
      for (int j = lane; j < time_dim; j += 32)
        atomicAdd(&acc[n_actions * action_dim + n_scenes * scene_dim + tb * time_dim + j],
                  row[item_dim + action_dim + scene_dim + j]);
    } else {
      const int f = r % P, v = profile[r];
      for (int j = lane; j < prof_dim; j += 32) atomicAdd(&acc[prof_off[f] + v * prof_dim + j], row[j]);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    if (acc[i] == 0.f) continue;
    if (group == 0) {
      const int na = n_actions * action_dim, ns = n_scenes * scene_dim;
      if (i < na) atomicAdd(&g.action[i], acc[i]);
      else if (i < na + ns) atomicAdd(&g.scene[i - na], acc[i]);
      else atomicAdd(&g.time[i - na - ns], acc[i]);
    } else {
      int f = 0;
      while (f + 1 < P && i >= prof_off[f + 1]) ++f;
      atomicAdd(&g.prof[f][i - prof_off[f]], acc[i]);
    }
  }
}

// d(special table) rows: BOS = row 0, SEPs = rows 1 + H and 2 + H + P of every request.
__global__ void k_special_grad(const float* __restrict__ dX, int B, int L, int H, int P, int d, int n_special,
                               float* __restrict__ gspecial) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_special * d) return;  // click sequences carry BOS only
  const int k = i / d, c = i - k * d;
  const int row = k == 0 ? 0 : (k == 1 ? 1 + H : 2 + H + P);
  float s = 0.f;
  for (int b = 0; b < B; ++b) s += dX[(static_cast<size_t>(b) * L + row) * d + c];
  gspecial[i] += s;
}

__global__ void k_bias_add(float* __restrict__ x, const float* __restrict__ b, int rows, int cols) {
  const size_t n = static_cast<size_t>(rows) * cols;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    x[i] += b[i % cols];
}

// ---------------------------------------------------------------- optimizer step
// adamw_step: bias-corrected moments, decoupled weight decay, over the
// flat master buffer (every trainable tensor; the frozen item table is not in it).
// Non-finite gradients set *bad to (index + 1) of the first one seen (host names it).
__global__ void k_adamw(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                        float* __restrict__ v, size_t n, float lr, float b1, float b2, float eps, float wd,
                        float bc1, float bc2, unsigned long long* bad, size_t base) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const float gi = g[i];
    if (!isfinite(gi)) {
      atomicMin(bad, static_cast<unsigned long long>(base + i) + 1ull);
      continue;
    }
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float mh = mi / bc1, vh = vi / bc2;
    p[i] = p[i] - lr * wd * p[i] - lr * (mh / (sqrtf(vh) + eps));
  }
}

// Item-table gradient (tokenizer.cpp:315-317, 346-352) when the table is not frozen: row r of
// d(concat) (row stride ld) adds its first item_dim columns into ditem[ids[r]]. Warp per row;
// fp32 atomics (rows sharing an item add in arbitrary order: last-ulp nondeterminism).
__global__ void k_item_grad_scatter(const float* __restrict__ dcat, int ld, int n, const int32_t* __restrict__ ids,
                                    int n_items, int item_dim, float* __restrict__ ditem) {
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += gridDim.x * (blockDim.x >> 5)) {
    const int id = ids[r];
    if (static_cast<unsigned>(id) >= static_cast<unsigned>(n_items)) continue;  // OOV is reported by the forward
    for (int j = lane; j < item_dim; j += 32)
      atomicAdd(ditem + static_cast<size_t>(id) * item_dim + j, dcat[static_cast<size_t>(r) * ld + j]);
  }
}

// Ranking loss: L = sum_obj w_obj * mean over candidates of BCE(p, y) with
// eps-clamped logs; dL/dz = w_obj (p - y) / n. One block of 1024 threads, fixed-order reduction.
__global__ void __launch_bounds__(1024) k_bce(const float* __restrict__ logits, const float* __restrict__ labels, int n,
                      float w0, float w1, float w2, float* __restrict__ dz, float* __restrict__ loss) {
  __shared__ float red[1024];
  float acc = 0.f;
  const float w[3] = {w0, w1, w2};
  for (int i = threadIdx.x; i < n * 3; i += blockDim.x) {
    const int o = i % 3;
    const float p = sigmoidf_stable(logits[i]), y = labels[i];
    const float pc = fminf(fmaxf(p, 1e-7f), 1.f - 1e-7f);
    acc += w[o] * -(y * logf(pc) + (1.f - y) * logf(1.f - pc));
    dz[i] = w[o] * (p - y) / static_cast<float>(n);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = red[0] / static_cast<float>(n);
}

// ---------------------------------------------------------------- weight repacking
// After an optimizer step the inference kernels' bf16 weights are rebuilt from the fp32
// masters with the transforms finalize() applies on the host: W^T (K-major), pre-norm gain
// folded into the input rows, QKVG rows interleaved head by head in `order`, SwishGLU up rows
// interleaved in 32-column [gate | up] blocks.
struct QkvgSrc {
  const float* w[4];  // kSecQ, kSecK, kSecV, kSecG  ([d, d], [in, out])
};
__global__ void k_repack_qkvg(QkvgSrc src, const float* __restrict__ gain, int4 order, int n_sec, int H, int dk,
                              int d, __nv_bfloat16* __restrict__ out) {
  const size_t n = static_cast<size_t>(n_sec) * d * d;
  const int ord[4] = {order.x, order.y, order.z, order.w};
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % d);
    const int row = static_cast<int>(i / d);
    const int hd = row / (n_sec * dk), rem = row - hd * n_sec * dk;
    const int sec = ord[rem / dk], j = rem % dk;
    out[i] = __float2bfloat16_rn(src.w[sec][static_cast<size_t>(k) * d + hd * dk + j] * gain[k]);
  }
}
// out[n, k] = bf16(W[k, n] * (gain ? gain[k] : 1)) for W [K, N]; out row pitch Kpad (zeros past K).
__global__ void k_repack_t(const float* __restrict__ W, const float* __restrict__ gain, int K, int N, int Kpad,
                           __nv_bfloat16* __restrict__ out) {
  const size_t n = static_cast<size_t>(N) * Kpad;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % Kpad), c = static_cast<int>(i / Kpad);
    out[i] = k < K ? __float2bfloat16_rn(W[static_cast<size_t>(k) * N + c] * (gain ? gain[k] : 1.f))
                   : __float2bfloat16_rn(0.f);
  }
}
__global__ void k_repack_up(const float* __restrict__ wg, const float* __restrict__ wu, const float* __restrict__ gain,
                            int d, int m, __nv_bfloat16* __restrict__ out) {
  const size_t n = static_cast<size_t>(2) * m * d;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % d), row = static_cast<int>(i / d);
    const int j = row / 64, r = row % 64;
    const float* src = r < 32 ? wg : wu;
    out[i] = __float2bfloat16_rn(src[static_cast<size_t>(k) * m + 32 * j + (r & 31)] * gain[k]);
  }
}
__global__ void k_concat_gu(const float* __restrict__ wg, const float* __restrict__ wu, int d, int m,
                            float* __restrict__ out) {
  const size_t n = static_cast<size_t>(d) * 2 * m;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = i / (2 * m);
    const int c = static_cast<int>(i % (2 * m));
    out[i] = c < m ? wg[r * m + c] : wu[r * m + c - m];
  }
}
// Many fp32 -> bf16 casts in one launch (the training GEMMs' bf16 weight copies refreshed after
// every optimizer step: ~30 tensors that were one launch each). blockIdx.y = segment.
struct CastSeg {
  const float* src;
  __nv_bfloat16* dst;
  size_t n;
};
__global__ void k_cast_segs(const CastSeg* __restrict__ segs) {
  const CastSeg sg = segs[blockIdx.y];
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < sg.n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    sg.dst[i] = __float2bfloat16_rn(sg.src[i]);
}

__global__ void k_cast_bf16(const float* __restrict__ x, size_t n, __nv_bfloat16* __restrict__ y) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
}

// Ranking head forward pieces in fp32: hid = relu(pre + b1); and its backward mask.
__global__ void k_bias_relu(float* __restrict__ x, const float* __restrict__ b, int rows, int cols) {
  const size_t n = static_cast<size_t>(rows) * cols;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    x[i] = fmaxf(x[i] + b[i % cols], 0.f);
}
__global__ void k_relu_mask(float* __restrict__ g, const float* __restrict__ hid, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    if (hid[i] <= 0.f) g[i] = 0.f;
}
__global__ void k_add_f32(float* __restrict__ a, const float* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    a[i] += b[i];
}

}  // namespace sortk
