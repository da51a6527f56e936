// SPDX-License-Identifier: Apache-2.0
// Row-sharded embedding lookup across ranks (BASELINE configs[4]):
// the reference gathers item rows with item_table_.value.row(id) (tokenizer.cpp:95-127)
// from one in-memory table; here the 100M-row table is split into contiguous row shards, one
// per rank (GPU), and every rank serves its batch's rows through two all-to-all exchanges:
//
//   ids (device) --count by owner--> send_ids grouped by owner  --alltoallv-->  owner
//   owner: rows = shard[local id]   --alltoallv-->  requester: rows in send order
//   requester: out[i] = row of ids[i] (scatter through the send permutation)
//
// All index work runs on the device; only the per-owner counts (world integers) cross to the
// host, because NCCL's grouped send/recv needs the message sizes on the host. Two transports:
//   * NCCL (the production path, one communicator per rank, grouped ncclSend/ncclRecv on the
//     caller's stream; libnccl.so.2 is resolved at run time from the process -- the copy
//     torch loaded -- so this library has no link-time NCCL dependency);
//   * a host callback (device buffers staged through pinned host memory): lets the exchange
//     logic run with several ranks on ONE GPU (tests) and any host collective (gloo).
// Out-of-vocabulary ids are agreed on before any payload moves: the counts message carries
// an error flag, so every rank raises ConfigError together instead of one rank blocking the
// others inside a collective (check_id, tokenizer.cpp:14-19).
// Included by runtime.cu after its error plumbing (ConfigError / api / sort_last_error).
#pragma once

#include <dlfcn.h>

#include <mutex>

namespace sortk {
namespace xchg {

using XConfigError = ConfigError;

inline void xck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- NCCL, resolved at run time
typedef struct { char internal[128]; } NcclUid;
typedef void* NcclComm;
struct Nccl {
  int (*GetUniqueId)(NcclUid*) = nullptr;
  int (*CommInitRank)(NcclComm*, int, NcclUid, int) = nullptr;
  int (*CommDestroy)(NcclComm) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Send)(const void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool ok = false;
};
constexpr int kNcclInt8 = 0, kNcclFloat32 = 7, kNcclSum = 0;

inline Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return;
    auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::decay_t<decltype(f)>>(dlsym(lib, name)); };
    sym(n.GetUniqueId, "ncclGetUniqueId");
    sym(n.CommInitRank, "ncclCommInitRank");
    sym(n.CommDestroy, "ncclCommDestroy");
    sym(n.GroupStart, "ncclGroupStart");
    sym(n.GroupEnd, "ncclGroupEnd");
    sym(n.Send, "ncclSend");
    sym(n.Recv, "ncclRecv");
    sym(n.AllReduce, "ncclAllReduce");
    sym(n.GetErrorString, "ncclGetErrorString");
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.GroupStart && n.GroupEnd && n.Send && n.Recv &&
           n.AllReduce;
  });
  if (!n.ok) throw std::runtime_error("NCCL (libnccl.so.2) is not available in this process");
  return n;
}
inline void nck(int r, const char* what) {
  if (r != 0)
    throw std::runtime_error(std::string(what) + ": " +
                             (nccl().GetErrorString ? nccl().GetErrorString(r) : std::to_string(r)));
}

// ---------------------------------------------------------------- kernels
// per-owner counts (block-local histogram, one global atomic per owner and block) and the
// out-of-range flag
__global__ void k_xchg_count(const int32_t* __restrict__ ids, int64_t n, int64_t rows_per_rank, int world,
                             int64_t* __restrict__ counts, int32_t* __restrict__ err) {
  __shared__ unsigned long long hist[64];
  for (int i = threadIdx.x; i < world; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int64_t limit = rows_per_rank * world;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t id = ids[i];
    if (id < 0 || id >= limit) {
      atomicOr(err, 1);
      continue;
    }
    atomicAdd(&hist[id / rows_per_rank], 1ull);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < world; i += blockDim.x)
    if (hist[i]) atomicAdd(reinterpret_cast<unsigned long long*>(counts + i), hist[i]);
}

// group ids by owner: position = offsets[owner] + atomic cursor; the permutation src[] keeps
// which batch position each sent id came from (order inside a group is not fixed, values are)
__global__ void k_xchg_scatter(const int32_t* __restrict__ ids, int64_t n, int64_t rows_per_rank,
                               const int64_t* __restrict__ offsets, unsigned long long* __restrict__ cursor,
                               int32_t* __restrict__ send_ids, int64_t* __restrict__ src) {
  // warp-aggregated slots: the lanes of a warp with the same owner take one atomicAdd (a
  // single global counter per owner would otherwise serialise every id, e.g. at world 1)
  const int lane = threadIdx.x & 31;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t base = blockIdx.x * static_cast<int64_t>(blockDim.x); base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool act = i < n;
    const int64_t id = act ? ids[i] : 0;
    const int owner = act ? static_cast<int>(id / rows_per_rank) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, owner);
    const int leader = __ffs(peers) - 1;
    unsigned long long first = 0;
    if (act && lane == leader) first = atomicAdd(cursor + owner, static_cast<unsigned long long>(__popc(peers)));
    first = __shfl_sync(0xffffffffu, first, leader);
    if (act) {
      const int64_t pos = offsets[owner] + static_cast<int64_t>(first) + __popc(peers & ((1u << lane) - 1u));
      send_ids[pos] = static_cast<int32_t>(id - owner * rows_per_rank);
      src[pos] = i;
    }
  }
}

// owner side: rows of the requested local ids, 16-byte vectors (range-checked)
__global__ void k_xchg_gather(const int4* __restrict__ shard, int64_t rows, int chunks, const int32_t* __restrict__ ids,
                              int64_t n, int4* __restrict__ out, int32_t* __restrict__ err) {
  const int64_t total = n * chunks;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = t / chunks;
    const int c = static_cast<int>(t - i * chunks);
    int64_t id = ids[i];
    if (id < 0 || id >= rows) {
      atomicOr(err, 2);
      id = 0;
    }
    out[t] = __ldg(shard + id * chunks + c);
  }
}

// requester side: out[src[j]] = received row j
__global__ void k_xchg_unpermute(const int4* __restrict__ recv, const int64_t* __restrict__ src, int64_t n, int chunks,
                                 int4* __restrict__ out) {
  const int64_t total = n * chunks;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = t / chunks;
    const int c = static_cast<int>(t - j * chunks);
    out[src[j] * chunks + c] = recv[t];
  }
}

inline int grid_for(int64_t work) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 16)));
}

}  // namespace xchg
}  // namespace sortk

using namespace sortk::xchg;

// ---------------------------------------------------------------- the exchange object
struct SortExchange_ {
  int rank = 0, world = 1, device = 0;
  NcclComm comm = nullptr;            // NCCL transport
  sort_alltoallv_fn host_fn = nullptr;  // host transport
  sort_allreduce_fn host_reduce = nullptr;
  void* host_ctx = nullptr;
  // device scratch (grown on demand)
  int64_t* d_counts = nullptr;  // [world] counts, then [world] offsets
  unsigned long long* d_cursor = nullptr;
  int32_t* d_err = nullptr;
  int32_t* send_ids = nullptr;
  int64_t* src = nullptr;
  int32_t* recv_ids = nullptr;
  void* rows_out = nullptr;  // owner side gathered rows
  void* rows_in = nullptr;   // requester side received rows
  size_t cap_ids = 0, cap_src = 0, cap_recv = 0, cap_rows_out = 0, cap_rows_in = 0;
  std::vector<uint8_t> h_send, h_recv;  // host transport staging
  int64_t* h_pin = nullptr;  // pinned [4 world + 1]: own counts, peer counts, offsets, error flag
  int64_t* d_xc = nullptr;   // device [2 world]: counts message out / in (NCCL transport)

  template <class T>
  void grow(T*& p, size_t& cap, size_t n) {
    if (n <= cap) return;
    if (p) cudaFree(p);
    cap = std::max(n, cap * 3 / 2 + 1);
    xck(cudaMalloc(reinterpret_cast<void**>(&p), cap), "exchange buffer");
  }

  // all-to-all-v of bytes: send[offsets by peer] -> recv[offsets by peer]
  void alltoallv(const void* send, const std::vector<int64_t>& sc, void* recv, const std::vector<int64_t>& rc,
                 cudaStream_t st) {
    std::vector<int64_t> so(world + 1, 0), ro(world + 1, 0);
    for (int p = 0; p < world; ++p) {
      so[p + 1] = so[p] + sc[p];
      ro[p + 1] = ro[p] + rc[p];
    }
    if (comm) {
      Nccl& n = nccl();
      nck(n.GroupStart(), "ncclGroupStart");
      for (int p = 0; p < world; ++p) {
        if (sc[p]) nck(n.Send(static_cast<const uint8_t*>(send) + so[p], sc[p], kNcclInt8, p, comm, st), "ncclSend");
        if (rc[p]) nck(n.Recv(static_cast<uint8_t*>(recv) + ro[p], rc[p], kNcclInt8, p, comm, st), "ncclRecv");
      }
      nck(n.GroupEnd(), "ncclGroupEnd");
      return;
    }
    h_send.resize(static_cast<size_t>(so[world]));
    h_recv.resize(static_cast<size_t>(ro[world]));
    if (so[world]) xck(cudaMemcpyAsync(h_send.data(), send, so[world], cudaMemcpyDeviceToHost, st), "exchange d2h");
    xck(cudaStreamSynchronize(st), "exchange sync");
    if (host_fn(host_ctx, h_send.data(), sc.data(), h_recv.data(), rc.data(), world) != 0)
      throw std::runtime_error("exchange: host all-to-all callback failed");
    if (ro[world]) xck(cudaMemcpyAsync(recv, h_recv.data(), ro[world], cudaMemcpyHostToDevice, st), "exchange h2d");
  }

  // counts (one int64 per peer) through the same transport, plus the agreed error flag
  std::vector<int64_t> exchange_counts(const std::vector<int64_t>& mine, bool bad, bool& any_bad, cudaStream_t st) {
    std::vector<int64_t> send(world), recv(world);
    for (int p = 0; p < world; ++p) send[p] = bad ? -1 : mine[p];
    std::vector<int64_t> b8(world, 8);
    if (comm) {  // through a persistent device buffer and pinned host memory (no pageable staging)
      if (!d_xc) xck(cudaMalloc(reinterpret_cast<void**>(&d_xc), 16 * world), "counts buffer");
      int64_t* hp = h_pin + world;
      std::memcpy(hp, send.data(), 8 * world);
      xck(cudaMemcpyAsync(d_xc, hp, 8 * world, cudaMemcpyHostToDevice, st), "counts h2d");
      alltoallv(d_xc, b8, d_xc + world, b8, st);
      xck(cudaMemcpyAsync(hp, d_xc + world, 8 * world, cudaMemcpyDeviceToHost, st), "counts d2h");
      xck(cudaStreamSynchronize(st), "counts sync");
      std::memcpy(recv.data(), hp, 8 * world);
    } else {
      if (host_fn(host_ctx, send.data(), b8.data(), recv.data(), b8.data(), world) != 0)
        throw std::runtime_error("exchange: host all-to-all callback failed");
    }
    any_bad = bad;
    for (int p = 0; p < world; ++p) any_bad |= recv[p] < 0;
    return recv;
  }

  ~SortExchange_() {
    for (void* p : {static_cast<void*>(d_counts), static_cast<void*>(d_cursor), static_cast<void*>(d_err),
                    static_cast<void*>(send_ids), static_cast<void*>(src), static_cast<void*>(recv_ids), rows_out,
                    rows_in})
      if (p) cudaFree(p);
    if (d_xc) cudaFree(d_xc);
    if (h_pin) cudaFreeHost(h_pin);
    if (comm) nccl().CommDestroy(comm);
  }
};

#define xapi sortk::api

extern "C" {

int sort_nccl_unique_id(void* out128) {
  return xapi([&] {
    if (!out128) throw XConfigError("null argument");
    NcclUid u;
    nck(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(out128, &u, sizeof(u));
  });
}

int sort_exchange_create_nccl(const void* unique_id128, int rank, int world, int device, SortExchange* out) {
  return xapi([&] {
    if (!unique_id128 || !out || world < 1 || rank < 0 || rank >= world || world > 64)
      throw XConfigError("exchange: bad arguments");
    xck(cudaSetDevice(device), "cudaSetDevice");
    auto* x = new SortExchange_;
    x->rank = rank;
    x->world = world;
    x->device = device;
    NcclUid u;
    std::memcpy(&u, unique_id128, sizeof(u));
    try {
      nck(nccl().CommInitRank(&x->comm, world, u, rank), "ncclCommInitRank");
    } catch (...) {
      delete x;
      throw;
    }
    *out = x;
  });
}

int sort_exchange_create_host(sort_alltoallv_fn fn, sort_allreduce_fn reduce_fn, void* ctx, int rank, int world,
                              int device, SortExchange* out) {
  return xapi([&] {
    if (!fn || !out || world < 1 || rank < 0 || rank >= world || world > 64)
      throw XConfigError("exchange: bad arguments");
    auto* x = new SortExchange_;
    x->rank = rank;
    x->world = world;
    x->device = device;
    x->host_fn = fn;
    x->host_reduce = reduce_fn;
    x->host_ctx = ctx;
    *out = x;
  });
}

int sort_exchange_destroy(SortExchange x) {
  return xapi([&] {
    if (x) {
      cudaSetDevice(x->device);
      delete x;
    }
  });
}

int sort_exchange_lookup(SortExchange x, const void* shard, int64_t rows_per_rank, int32_t row_bytes,
                         const int32_t* ids, int64_t n, void* out_rows, void* stream) {
  return xapi([&] {
    if (!x || !shard || (!ids && n) || (!out_rows && n)) throw XConfigError("exchange: null argument");
    if (row_bytes <= 0 || row_bytes % 16) throw XConfigError("exchange: row_bytes must be a positive multiple of 16");
    if (rows_per_rank < 1 || rows_per_rank > INT32_MAX) throw XConfigError("exchange: rows_per_rank out of range");
    xck(cudaSetDevice(x->device), "cudaSetDevice");
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int W = x->world;
    const int chunks = row_bytes / 16;
    if (!x->d_counts) {
      size_t c0 = 0, c1 = 0, c2 = 0;
      x->grow(x->d_counts, c0, sizeof(int64_t) * 2 * W);
      x->grow(x->d_cursor, c1, sizeof(unsigned long long) * W);
      x->grow(x->d_err, c2, sizeof(int32_t));
      xck(cudaHostAlloc(reinterpret_cast<void**>(&x->h_pin), sizeof(int64_t) * (4 * W + 1), cudaHostAllocDefault),
          "pinned counts");
    }
    // ---- 1. count ids per owner (+ range flag)
    xck(cudaMemsetAsync(x->d_counts, 0, sizeof(int64_t) * W, st), "memset");
    xck(cudaMemsetAsync(x->d_cursor, 0, sizeof(unsigned long long) * W, st), "memset");
    xck(cudaMemsetAsync(x->d_err, 0, sizeof(int32_t), st), "memset");
    if (n) k_xchg_count<<<grid_for(n), 256, 0, st>>>(ids, n, rows_per_rank, W, x->d_counts, x->d_err);
    xck(cudaGetLastError(), "exchange count");
    int64_t* hp = x->h_pin;  // [0, W): own counts; [4W]: error flag (pinned: truly async copies)
    hp[4 * W] = 0;
    xck(cudaMemcpyAsync(hp, x->d_counts, sizeof(int64_t) * W, cudaMemcpyDeviceToHost, st), "d2h");
    xck(cudaMemcpyAsync(hp + 4 * W, x->d_err, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "d2h");
    xck(cudaStreamSynchronize(st), "sync");
    const std::vector<int64_t> sc_ids(hp, hp + W);
    const int32_t herr = static_cast<int32_t>(hp[4 * W] & 0xffffffff);
    // ---- 2. agree on the error flag, learn how many ids every peer will ask this rank for
    bool any_bad = false;
    const std::vector<int64_t> rc_ids = x->exchange_counts(sc_ids, herr != 0, any_bad, st);
    if (any_bad)
      throw XConfigError("tokenizer: item id outside vocabulary of size " + std::to_string(rows_per_rank * W) +
                         " (sharded table, detected on rank " + std::string(herr ? "this" : "another") + ")");
    // ---- 3. group ids by owner
    std::vector<int64_t> off(W + 1, 0);
    for (int p = 0; p < W; ++p) off[p + 1] = off[p] + sc_ids[p];
    int64_t n_recv = 0;
    for (int p = 0; p < W; ++p) n_recv += rc_ids[p];
    x->grow(x->send_ids, x->cap_ids, sizeof(int32_t) * std::max<int64_t>(n, 1));
    x->grow(x->src, x->cap_src, sizeof(int64_t) * std::max<int64_t>(n, 1));
    std::memcpy(hp + 2 * W, off.data(), sizeof(int64_t) * W);
    xck(cudaMemcpyAsync(x->d_counts + W, hp + 2 * W, sizeof(int64_t) * W, cudaMemcpyHostToDevice, st), "h2d");
    if (n)
      k_xchg_scatter<<<grid_for(n), 256, 0, st>>>(ids, n, rows_per_rank, x->d_counts + W, x->d_cursor, x->send_ids,
                                                   x->src);
    xck(cudaGetLastError(), "exchange scatter");
    // ---- 4. ids to their owners
    x->grow(x->recv_ids, x->cap_recv, sizeof(int32_t) * std::max<int64_t>(n_recv, 1));
    std::vector<int64_t> sb(W), rb(W);
    for (int p = 0; p < W; ++p) {
      sb[p] = sc_ids[p] * 4;
      rb[p] = rc_ids[p] * 4;
    }
    x->alltoallv(x->send_ids, sb, x->recv_ids, rb, st);
    // ---- 5. owner-side gather
    x->grow(x->rows_out, x->cap_rows_out, static_cast<size_t>(row_bytes) * std::max<int64_t>(n_recv, 1));
    if (n_recv)
      k_xchg_gather<<<grid_for(n_recv * chunks), 256, 0, st>>>(static_cast<const int4*>(shard), rows_per_rank, chunks,
                                                               x->recv_ids, n_recv, static_cast<int4*>(x->rows_out),
                                                               x->d_err);
    xck(cudaGetLastError(), "exchange gather");
    // ---- 6. rows back to the requesters (the reverse message sizes), 7. into batch order
    x->grow(x->rows_in, x->cap_rows_in, static_cast<size_t>(row_bytes) * std::max<int64_t>(n, 1));
    for (int p = 0; p < W; ++p) {
      sb[p] = rc_ids[p] * row_bytes;
      rb[p] = sc_ids[p] * row_bytes;
    }
    x->alltoallv(x->rows_out, sb, x->rows_in, rb, st);
    if (n)
      k_xchg_unpermute<<<grid_for(n * chunks), 256, 0, st>>>(static_cast<const int4*>(x->rows_in), x->src, n, chunks,
                                                             static_cast<int4*>(out_rows));
    xck(cudaGetLastError(), "exchange unpermute");
  });
}

int sort_exchange_allreduce_f32(SortExchange x, float* buf, int64_t n, void* stream) {
  return xapi([&] {
    if (!x || (!buf && n)) throw XConfigError("exchange: null argument");
    xck(cudaSetDevice(x->device), "cudaSetDevice");
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n == 0 || x->world == 1) return;
    if (x->comm) {
      nck(nccl().AllReduce(buf, buf, static_cast<size_t>(n), kNcclFloat32, kNcclSum, x->comm, st), "ncclAllReduce");
      return;
    }
    if (!x->host_reduce) throw XConfigError("exchange: host transport without an all-reduce callback");
    std::vector<float> h(static_cast<size_t>(n));
    xck(cudaMemcpyAsync(h.data(), buf, sizeof(float) * n, cudaMemcpyDeviceToHost, st), "d2h");
    xck(cudaStreamSynchronize(st), "sync");
    if (x->host_reduce(x->host_ctx, h.data(), n) != 0) throw std::runtime_error("exchange: host all-reduce failed");
    xck(cudaMemcpyAsync(buf, h.data(), sizeof(float) * n, cudaMemcpyHostToDevice, st), "h2d");
    xck(cudaStreamSynchronize(st), "sync");
  });
}

}  // extern "C"
