#include <atomic>
// Dual-index build on the device: the sm_100a replacement of
// EdgeStore::build (edge_store.cpp:27-254).
//
// Pipeline (all device kernels on the ctx stream; three 8-byte host reads
// size the outputs: V, Z, Q):
//   1. k_edge_stats       min/max time, max id, negative-input flags  (:32-38)
//   2. densify            dense ids: presence flags + scan (rank table) when
//                         the id range is compact, else sort-unique + binary
//                         search. Internal id = rank of the external id among
//                         the snapshot's endpoints, exactly as :57-89.
//   3. canonical order    one stable LSD radix sort of the packed key
//                         (t - tmin | src | dst) when it fits 64 bits (the
//                         sorted key IS the edge: no gather), else two stable
//                         passes (src|dst, then t) + gather.          (:42-55)
//   4. ts view            flag + scan -> ts_off, ts_time             (:91-98)
//                         ts_w: exact zero prefix + serial <=746-group tail (:100-110)
//   5. node view          stable radix sort of entries by owner; entries
//                         materialised as 16-byte {nbr, edge, t}; region
//                         bounds from run boundaries; marks by flag+scan (:112-214)
//   6. node weights       zero prefix + per-node serial tail over the entries
//                         within 745 time units of the node's anchor (:159,:208-209)
//   7. adjacency          radix sort of (owner|nbr), unique, bounds  (:216-250)
//
// Exactness: every weight is exp(t - anchor) with an
// integer argument <= 0. glibc gives exp(-k) = +0 for k >= 746, so every
// prefix before the first entry with t >= anchor - 745 is exactly +0.0 and
// only the tail needs the serial in-order fp64 sum; its terms come from a
// table of glibc exp(-k) computed on the host (ctx.d_exp_neg).
#include "primitives.cuh"
#include "store.cuh"

namespace twg {

namespace {

constexpr int kBlock = 256;

// scalars: [0] neg time flag, [1] neg id flag, [2] max id, [3] min t, [4] max t
__global__ void k_edge_stats(EdgesSoA in, u64* scalars) {
  u64 neg_t = 0, neg_id = 0, max_id = 0, min_t = ~0ull, max_t = 0;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < in.n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const i64 s = in.src[i], d = in.dst[i], t = in.t[i];
    if (t < 0) neg_t = 1;
    if (s < 0 || d < 0) neg_id = 1;
    const u64 hi = static_cast<u64>(s > d ? s : d);
    if (hi > max_id) max_id = hi;
    if (static_cast<u64>(t) < min_t) min_t = static_cast<u64>(t);
    if (static_cast<u64>(t) > max_t) max_t = static_cast<u64>(t);
  }
  for (int o = 16; o > 0; o >>= 1) {
    neg_t |= __shfl_xor_sync(0xffffffffu, neg_t, o);
    neg_id |= __shfl_xor_sync(0xffffffffu, neg_id, o);
    max_id = max(max_id, __shfl_xor_sync(0xffffffffu, max_id, o));
    min_t = min(min_t, __shfl_xor_sync(0xffffffffu, min_t, o));
    max_t = max(max_t, __shfl_xor_sync(0xffffffffu, max_t, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (neg_t) atomicOr(reinterpret_cast<unsigned long long*>(&scalars[0]), 1ull);
    if (neg_id) atomicOr(reinterpret_cast<unsigned long long*>(&scalars[1]), 1ull);
    atomicMax(reinterpret_cast<unsigned long long*>(&scalars[2]), max_id);
    atomicMin(reinterpret_cast<unsigned long long*>(&scalars[3]), min_t);
    atomicMax(reinterpret_cast<unsigned long long*>(&scalars[4]), max_t);
  }
}

__global__ void k_init_stats(u64* scalars) {
  scalars[0] = 0;
  scalars[1] = 0;
  scalars[2] = 0;
  scalars[3] = ~0ull;
  scalars[4] = 0;
}

__global__ void k_mark_present(EdgesSoA in, u32* present) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < in.n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    present[in.src[i]] = 1u;
    present[in.dst[i]] = 1u;
  }
}

struct PresentFn {
  const u32* p;
  __device__ __forceinline__ u32 operator()(u64 i) const { return p[i]; }
};

__global__ void k_fill_ext_dense(const u32* present, const u32* rank, u64 range, i64* ext) {
  for (u64 id = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; id < range;
       id += static_cast<u64>(gridDim.x) * blockDim.x) {
    if (present[id]) ext[rank[id]] = static_cast<i64>(id);
  }
}

__global__ void k_map_dense(EdgesSoA in, const u32* rank, u32* src_i, u32* dst_i) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < in.n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    src_i[i] = rank[in.src[i]];
    dst_i[i] = rank[in.dst[i]];
  }
}

__global__ void k_endpoints(EdgesSoA in, u64* keys) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < in.n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    keys[2 * i] = static_cast<u64>(in.src[i]);
    keys[2 * i + 1] = static_cast<u64>(in.dst[i]);
  }
}

struct UniqueFlagFn {
  const u64* k;
  __device__ __forceinline__ u32 operator()(u64 i) const { return (i == 0 || k[i] != k[i - 1]) ? 1u : 0u; }
};

__global__ void k_fill_ext_unique(const u64* keys, const u32* rank, u64 n, i64* ext) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    if (i == 0 || keys[i] != keys[i - 1]) ext[rank[i]] = static_cast<i64>(keys[i]);
  }
}

__device__ __forceinline__ u32 find_ext(const i64* ext, u64 V, u64 id) {
  u64 lo = 0, hi = V;
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if (static_cast<u64>(ext[mid]) < id) lo = mid + 1;
    else hi = mid;
  }
  return static_cast<u32>(lo);
}

__global__ void k_map_sparse(EdgesSoA in, const i64* ext, u64 V, u32* src_i, u32* dst_i) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < in.n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    src_i[i] = find_ext(ext, V, static_cast<u64>(in.src[i]));
    dst_i[i] = find_ext(ext, V, static_cast<u64>(in.dst[i]));
  }
}

__global__ void k_pack_canonical(const u32* src_i, const u32* dst_i, const i64* t, u64 n, i64 tmin, int vb,
                                 u64* keys, u32* perm) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    keys[i] = (static_cast<u64>(t[i] - tmin) << (2 * vb)) | (static_cast<u64>(src_i[i]) << vb) | dst_i[i];
    perm[i] = static_cast<u32>(i);
  }
}

__global__ void k_unpack_canonical(const u64* keys, u64 n, i64 tmin, int vb, u32* e_src, u32* e_dst, i64* e_t) {
  const u64 mask = vb == 0 ? 0ull : ((1ull << vb) - 1);
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 k = keys[i];
    e_dst[i] = static_cast<u32>(k & mask);
    e_src[i] = static_cast<u32>((k >> vb) & mask);
    e_t[i] = static_cast<i64>(k >> (2 * vb)) + tmin;
  }
}

__global__ void k_pack_pair(const u32* src_i, const u32* dst_i, u64 n, int vb, u64* keys, u32* perm) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    keys[i] = (static_cast<u64>(src_i[i]) << vb) | dst_i[i];
    perm[i] = static_cast<u32>(i);
  }
}

__global__ void k_gather_time_key(const i64* t, const u32* perm, u64 n, i64 tmin, u64* keys) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    keys[i] = static_cast<u64>(t[perm[i]] - tmin);
  }
}

__global__ void k_gather_edges(const u32* src_i, const u32* dst_i, const i64* t, const u32* perm, u64 n,
                               u32* e_src, u32* e_dst, i64* e_t) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 p = perm[i];
    e_src[i] = src_i[p];
    e_dst[i] = dst_i[p];
    e_t[i] = t[p];
  }
}

struct TimeChangeFn {
  const i64* t;
  __device__ __forceinline__ u32 operator()(u64 i) const { return (i == 0 || t[i] != t[i - 1]) ? 1u : 0u; }
};


// ts_w[g] = sum_{h<=g} exp(t_h - t_last) (edge_store.cpp:100-110). Zero
// prefix by memset; this one-warp kernel does the <=746-group serial tail.
__global__ void k_ts_weights(const i64* ts_time, u64 Z, const double* exp_neg, double* ts_w) {
  if (threadIdx.x != 0 || Z == 0) return;
  const i64 anchor = ts_time[Z - 1];
  const u32 g0 = lb_i64(ts_time, 0, static_cast<u32>(Z), anchor - (kExpTableSize - 1));
  double acc = 0.0;
  for (u32 g = g0; g < Z; ++g) {
    acc = __dadd_rn(acc, exp_neg[anchor - ts_time[g]]);
    ts_w[g] = acc;
  }
}

// entries in canonical order: j -> owner (edge_store.cpp:120-124)
__global__ void k_owner_keys(const u32* e_src, const u32* e_dst, u64 m, int mode, u32* keys, u32* vals) {
  const u64 P = mode == TWG_UNDIRECTED ? 2 * m : m;
  for (u64 j = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; j < P;
       j += static_cast<u64>(gridDim.x) * blockDim.x) {
    u32 owner;
    if (mode == TWG_UNDIRECTED) owner = (j & 1) ? e_dst[j >> 1] : e_src[j >> 1];
    else if (mode == TWG_BACKWARD) owner = e_dst[j];
    else owner = e_src[j];
    keys[j] = owner;
    vals[j] = static_cast<u32>(j);
  }
}

// edge_store.hpp:133-140 ref_neighbor, materialised per entry
__global__ void k_entries(const u32* owners, const u32* jidx, u64 P, int mode, const u32* e_src,
                          const u32* e_dst, const i64* e_t, Entry* ent) {
  for (u64 pos = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; pos < P;
       pos += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 j = jidx[pos];
    const u32 e = mode == TWG_UNDIRECTED ? (j >> 1) : j;
    const u32 owner = owners[pos];
    u32 nbr;
    if (mode == TWG_FORWARD) nbr = e_dst[e];
    else if (mode == TWG_BACKWARD) nbr = e_src[e];
    else nbr = e_src[e] == owner ? e_dst[e] : e_src[e];
    Entry x;
    x.nbr = nbr;
    x.edge = e;
    x.t = e_t[e];
    ent[pos] = x;
  }
}


struct GroupStartFn {
  const u32* owners;
  const Entry* ent;
  __device__ __forceinline__ u32 operator()(u64 p) const {
    return (p == 0 || owners[p] != owners[p - 1] || ent[p].t != ent[p - 1].t) ? 1u : 0u;
  }
};



// node_weight_prefix_ (edge_store.cpp:159, :208-209): per node, serial sum of
// exp(t - anchor_v) over the entries within 745 time units of the anchor.
__global__ void k_node_weights(StoreView s, const double* exp_neg, double* wp) {
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < s.V;
       v += static_cast<u64>(gridDim.x) * blockDim.x) {
    const uint2 a = s.nmeta[v], b = s.nmeta[v + 1];
    if (a.x == b.x) continue;
    const i64 anchor = s.ent[b.x - 1].t;
    const u32 g0 = lb_i64(s.mk_time, a.y, b.y, anchor - (kExpTableSize - 1));
    double acc = 0.0;
    for (u32 pos = s.mk_start[g0]; pos < b.x; ++pos) {
      acc = __dadd_rn(acc, exp_neg[anchor - s.ent[pos].t]);
      wp[pos] = acc;
    }
  }
}

// newest incident time per node (check-before-max: hub slots are hot)
__global__ void k_node_last_t(const u32* s, const u32* d, const i64* t, u64 m, i64* last) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const i64 ti = t[i];
    const u32 a = s[i], b = d[i];
    if (last[a] < ti) atomicMax(reinterpret_cast<long long*>(last + a), static_cast<long long>(ti));
    if (last[b] < ti) atomicMax(reinterpret_cast<long long*>(last + b), static_cast<long long>(ti));
  }
}

__global__ void k_adj_keys(const u32* owners, const Entry* ent, u64 P, int vb, u64* keys) {
  for (u64 p = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; p < P;
       p += static_cast<u64>(gridDim.x) * blockDim.x) {
    keys[p] = (static_cast<u64>(owners[p]) << vb) | ent[p].nbr;
  }
}

__global__ void k_adj_fill(const u64* keys, const u32* uscan, u64 P, int vb, u32* adj, u32* adj_owner) {
  const u64 mask = (1ull << vb) - 1;
  for (u64 p = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; p < P;
       p += static_cast<u64>(gridDim.x) * blockDim.x) {
    if (p == 0 || keys[p] != keys[p - 1]) {
      adj[uscan[p]] = static_cast<u32>(keys[p] & mask);
      adj_owner[uscan[p]] = static_cast<u32>(keys[p] >> vb);
    }
  }
}

__global__ void k_region_bounds_u32(const u32* owners, u64 P, u64 V, u32* off) {
  for (u64 pos = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; pos <= P;
       pos += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 lo = pos == 0 ? 0 : static_cast<u64>(owners[pos - 1]) + 1;
    const u64 hi = pos == P ? V : static_cast<u64>(owners[pos]);
    if (pos == 0 || pos == P || owners[pos] != owners[pos - 1]) {
      for (u64 v = lo; v <= hi && v <= V; ++v) off[v] = static_cast<u32>(pos);
    }
  }
}

unsigned grid(Ctx& ctx, u64 n) { return grid_for(n, kBlock, static_cast<unsigned>(ctx.sm_count) * 16); }

}  // namespace

namespace {
__global__ void k_read_scalars(const u64* src, volatile u64* mapped, int n, u64 seq) {
  if (static_cast<int>(threadIdx.x) < n) mapped[threadIdx.x] = src[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // the values reach the host before the flag
    mapped[kMappedFlag] = seq;
  }
}
}  // namespace

void mapped_wait(Ctx& ctx, u64 seq) {
  volatile u64* flag = ctx.h_pinned + kMappedFlag;
  for (u32 spin = 1;; ++spin) {
    if (*flag == seq) break;
    if ((spin & 4095) == 0) {  // every few microseconds: the stream failed or drained without the flag?
      const cudaError_t e = cudaStreamQuery(ctx.stream);
      if (e == cudaSuccess) {
        if (*flag == seq) break;
        fail(TWG_ECUDA, "mapped read-back: stream drained without publishing");
      }
      if (e != cudaErrorNotReady) cuda_check(e, "mapped read-back", __FILE__, __LINE__);
    }
    __builtin_ia32_pause();
  }
  std::atomic_thread_fence(std::memory_order_acquire);
}

// Small device->host reads go through mapped pinned memory written by a
// one-warp kernel: no copy engine is involved, so the read never queues
// behind a multi-GB walk download running on the D2H engine. The host
// polls the mapped flag instead of synchronising the stream (a stream
// synchronisation costs several microseconds more per read-back).
void read_scalars(Ctx& ctx, const u64* d_src, u64* host_dst, int n) {
  const u64 seq = ++ctx.mapped_seq;
  k_read_scalars<<<1, 64, 0, ctx.stream>>>(d_src, ctx.d_mapped, n, seq);
  TWG_LAUNCHED(ctx);
  mapped_wait(ctx, seq);
  for (int i = 0; i < n; ++i) host_dst[i] = reinterpret_cast<volatile u64*>(ctx.h_pinned)[i];
}

// streaming stores: ts_w[g] = sum_{h<=g} exp(t_h - t_last) is +0 before the
// first group within 745 time units of t_last; only that tail (<= 746 values)
// is materialised. The per-node prefixes are evaluated by the walk kernels
// from the node's tail entries (walk.cu draw_weighted_ring), exactly.
__global__ void k_ts_wtail(StoreView s, const double* exp_neg, double* tail, u64* t0) {
  if (threadIdx.x != 0 || s.Z == 0) return;
  const i64 anchor = s.ts_time[s.zrg(static_cast<u32>(s.Z - 1))];
  u64 lo = 0, hi = s.Z;  // first group with time >= anchor - 745
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if (s.ts_time[s.zrg(static_cast<u32>(mid))] < anchor - (kExpTableSize - 1)) lo = mid + 1;
    else hi = mid;
  }
  *t0 = lo;
  double acc = 0.0;
  for (u64 g = lo; g < s.Z; ++g) {
    acc = __dadd_rn(acc, exp_neg[anchor - s.ts_time[s.zrg(static_cast<u32>(g))]]);
    tail[g - lo] = acc;
  }
}

void ensure_weights(Ctx& ctx, Store& s) {
  std::lock_guard<std::mutex> lk(s.lazy_mu);
  if (s.has_weights) return;
  if (s.gapped) {
    cudaStream_t st = ctx.stream;
    s.ts_wtail.alloc(kExpTableSize + 1, st);
    TWG_CUDA(cudaMemsetAsync(ctx.d_scalars + 20, 0, sizeof(u64), st));
    if (s.Z) {
      k_ts_wtail<<<1, 32, 0, st>>>(s.view(), ctx.d_exp_neg, s.ts_wtail.p, ctx.d_scalars + 20);
      TWG_LAUNCHED(ctx);
    }
    u64 t0[1];
    read_scalars(ctx, ctx.d_scalars + 20, t0, 1);
    s.ts_wt0 = t0[0];
    s.has_weights = true;
    return;
  }
  cudaStream_t st = ctx.stream;
  s.ts_w.alloc(s.Z ? s.Z : 1, st);
  TWG_CUDA(cudaMemsetAsync(s.ts_w.p, 0, s.ts_w.bytes(), st));
  if (s.Z) {
    k_ts_weights<<<1, 32, 0, st>>>(s.ts_time.p, s.Z, ctx.d_exp_neg, s.ts_w.p);
    TWG_LAUNCHED(ctx);
  }
  s.wp.alloc(s.P ? s.P : 1, st);
  TWG_CUDA(cudaMemsetAsync(s.wp.p, 0, s.wp.bytes(), st));
  if (s.P) {
    k_node_weights<<<grid(ctx, s.V), kBlock, 0, st>>>(s.view(), ctx.d_exp_neg, s.wp.p);
    TWG_LAUNCHED(ctx);
  }
  TWG_CUDA(cudaStreamSynchronize(st));  // complete before any other stream may see the flag
  s.has_weights = true;
}

// Sorted unique traversal neighbours (edge_store.cpp:216-250).
static void build_adjacency(Ctx& ctx, Store& s, const u32* owners) {
  cudaStream_t st = ctx.stream;
  const u64 P = s.P, V = s.V;
  s.adj_off.alloc(V + 1, st);
  if (P == 0) {
    TWG_CUDA(cudaMemsetAsync(s.adj_off.p, 0, s.adj_off.bytes(), st));
    s.adj.alloc(1, st);
    s.A = 0;
    s.has_adjacency = true;
    return;
  }
  const int vb = V > 1 ? bit_width_u64(V - 1) : 1;
  DevBuf<u64> k0(P, st), k1(P, st);
  k_adj_keys<<<grid(ctx, P), kBlock, 0, st>>>(owners, s.ent.p, P, vb, k0.p);
  TWG_LAUNCHED(ctx);
  u64* kp = k0.p;
  u64* ka = k1.p;
  u32* vnull = nullptr;
  u32* vnull2 = nullptr;
  radix_sort_pairs<u64>(ctx, &kp, &ka, &vnull, &vnull2, P, 2 * vb);
  DevBuf<u32> uscan(P + 1, st);
  exclusive_scan<u32>(ctx, UniqueFlagFn{kp}, P, uscan.p);
  u64 A = 0;
  {
    u64 tmp[1];
    TWG_CUDA(cudaMemcpyAsync(ctx.d_scalars, uscan.p + P, sizeof(u32), cudaMemcpyDeviceToDevice, st));
    read_scalars(ctx, ctx.d_scalars, tmp, 1);
    A = tmp[0] & 0xffffffffull;
  }
  s.adj.alloc(A ? A : 1, st);
  DevBuf<u32> adj_owner(A ? A : 1, st);
  k_adj_fill<<<grid(ctx, P), kBlock, 0, st>>>(kp, uscan.p, P, vb, s.adj.p, adj_owner.p);
  TWG_LAUNCHED(ctx);
  k_region_bounds_u32<<<grid(ctx, A + 1), kBlock, 0, st>>>(adj_owner.p, A, V, s.adj_off.p);
  TWG_LAUNCHED(ctx);
  s.A = A;
  TWG_CUDA(cudaStreamSynchronize(st));  // complete before any other stream may see the flag
  s.has_adjacency = true;
}

namespace {
__global__ void k_nm_from_nmeta(const uint2* nmeta, u64 V, NodeMeta* nm) {
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<u64>(gridDim.x) * blockDim.x) {
    const uint2 a = nmeta[v], b = nmeta[v + 1];
    nm[v] = NodeMeta{a.x, b.x, a.y, b.y, 0u, kIdentityCap, 0u, 0u};
  }
}

struct EntSizeFn {
  const NodeMeta* nm;
  __device__ __forceinline__ u32 operator()(u64 v) const { return nm[v].ee - nm[v].eb; }
};
struct MarkSizeFn {
  const NodeMeta* nm;
  __device__ __forceinline__ u32 operator()(u64 v) const { return nm[v].ge - nm[v].gb; }
};

__global__ void k_pack_nmeta(const u32* off, const u32* goff, u64 V, uint2* nmeta) {
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v <= V;
       v += static_cast<u64>(gridDim.x) * blockDim.x)
    nmeta[v] = make_uint2(off[v], goff[v]);
}

__global__ void k_ts_rebase(const u32* ts_off, const i64* ts_time, Ring zr, u64 Z, u32 seq0, u64 m, u32* out,
                            i64* tout) {
  for (u64 g = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; g <= Z;
       g += static_cast<u64>(gridDim.x) * blockDim.x) {
    out[g] = g < Z ? ts_off[zr(static_cast<u32>(g))] - seq0 : static_cast<u32>(m);
    if (g < Z) tout[g] = ts_time[zr(static_cast<u32>(g))];
  }
}

// ring slice of the edge log -> contiguous columns
__global__ void k_unring_edges(StoreView v, u64 m, u32* os, u32* od, i64* ot) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const EdgeRec r = edge_at(v, i);
    os[i] = r.src;
    od[i] = r.dst;
    ot[i] = r.t;
  }
}

// gapped regions -> contiguous regions, one warp per node (lanes stride the
// region): entries get snapshot-relative edge indices, marks contiguous
// positions, and every entry its owner.
__global__ void k_compact_regions(const NodeMeta* nm, u64 V, const Entry* ent, const i64* mk_time,
                                  const u32* mk_start, u32 seq0, const uint2* nmeta, Entry* ent_c, u32* owner_c,
                                  i64* mk_time_c, u32* mk_start_c) {
  const int lane = threadIdx.x & 31;
  const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
  for (u64 v = (blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) >> 5; v < V; v += warps) {
    const NodeMeta r = nm[v];
    const Ring er = entry_ring(r), mr = mark_ring(r);
    const uint2 o = nmeta[v];
    for (u32 i = lane; i < r.ee - r.eb; i += 32) {
      Entry e = ent[er(r.eb + i)];
      e.edge -= seq0;
      ent_c[o.x + i] = e;
      owner_c[o.x + i] = static_cast<u32>(v);
    }
    if (implicit_marks(r)) {  // single-entry groups: mark k is entry k (marks not stored)
      for (u32 i = lane; i < r.ge - r.gb; i += 32) {
        mk_time_c[o.y + i] = ent[er(r.eb + i)].t;
        mk_start_c[o.y + i] = o.x + i;
      }
    } else {
      for (u32 i = lane; i < r.ge - r.gb; i += 32) {
        mk_time_c[o.y + i] = mk_time[mr(r.gb + i)];
        mk_start_c[o.y + i] = mk_start[mr(r.gb + i)] - r.eb + o.x;
      }
    }
  }
}

__global__ void k_entry_owners(const uint2* nmeta, u64 V, u32* owners) {
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<u64>(gridDim.x) * blockDim.x) {
    for (u32 p = nmeta[v].x; p < nmeta[v + 1].x; ++p) owners[p] = static_cast<u32>(v);
  }
}
}  // namespace

// walk records of a contiguous store (identity ring): bounds + the newest
// kWalkTail entries of each region, newest first (store.cuh WalkRec)
__global__ void k_wrec_from_nm(const NodeMeta* nm, const Entry* ent, u64 V, WalkRec* wrec) {
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<u64>(gridDim.x) * blockDim.x) {
    const NodeMeta m = nm[v];
    WalkRec w;
    w.eb = m.eb;
    w.ee = m.ee;
    w.base = m.base;
    w.cap = m.cap;
    w.eorg = m.eorg;
    w.g = m.ge - m.gb;
    w.pad = 0;
    const Ring er = entry_ring(m);
#pragma unroll
    for (u32 i = 0; i < kWalkTail; ++i) {
      const bool in = i < m.ee - m.eb;
      const Entry e = in ? ent[er(m.ee - 1 - i)] : Entry{0u, 0u, 0};
      w.nbr[i] = e.nbr;
      w.t[i] = e.t;
    }
    wrec[v] = w;
  }
}

void build_nm(Ctx& ctx, Store& s) {
  s.nm.alloc(s.V ? s.V : 1, ctx.stream);
  if (s.V) {
    k_nm_from_nmeta<<<grid(ctx, s.V), kBlock, 0, ctx.stream>>>(s.nmeta.p, s.V, s.nm.p);
    TWG_LAUNCHED(ctx);
    s.wrec.alloc(s.V, ctx.stream);
    k_wrec_from_nm<<<grid(ctx, s.V), kBlock, 0, ctx.stream>>>(s.nm.p, s.ent.p, s.V, s.wrec.p);
    TWG_LAUNCHED(ctx);
  }
}

Store& ensure_compact(Ctx& ctx, const Store& g) {
  if (!g.gapped) return const_cast<Store&>(g);
  std::lock_guard<std::mutex> lock(g.compact_mu);
  if (g.compact) return *g.compact;
  cudaStream_t st = ctx.stream;
  auto c = std::make_unique<Store>();
  c->ctx = &ctx;
  c->mode = g.mode;
  c->m = g.m;
  c->V = g.V;
  c->Z = g.Z;
  c->P = g.P;
  c->ext_identity = g.ext_identity;
  c->seq0 = 0;
  c->ext.alias(g.ext.p, g.ext.n);
  c->last_t.alias(g.last_t.p, g.last_t.n);
  c->e_src.alloc(g.m ? g.m : 1, st);
  c->e_dst.alloc(g.m ? g.m : 1, st);
  c->e_t.alloc(g.m ? g.m : 1, st);
  if (g.m) {
    k_unring_edges<<<grid(ctx, g.m), kBlock, 0, st>>>(g.view(), g.m, c->e_src.p, c->e_dst.p, c->e_t.p);
    TWG_LAUNCHED(ctx);
  }
  c->ts_time.alloc(g.Z ? g.Z : 1, st);
  c->ts_off.alloc(g.Z + 1, st);
  k_ts_rebase<<<grid(ctx, g.Z + 1), kBlock, 0, st>>>(g.ts_off.p, g.ts_time.p, Ring{0u, g.z_cap, g.z_org}, g.Z, g.seq0,
                                                     g.m, c->ts_off.p, c->ts_time.p);
  TWG_LAUNCHED(ctx);
  const u64 V = g.V;
  DevBuf<u32> off(V + 1, st), goff(V + 1, st);
  exclusive_scan<u32>(ctx, EntSizeFn{g.nm.p}, V, off.p);
  exclusive_scan<u32>(ctx, MarkSizeFn{g.nm.p}, V, goff.p);
  c->nmeta.alloc(V + 1, st);
  k_pack_nmeta<<<grid(ctx, V + 1), kBlock, 0, st>>>(off.p, goff.p, V, c->nmeta.p);
  TWG_LAUNCHED(ctx);
  TWG_CUDA(cudaMemsetAsync(ctx.d_scalars + 18, 0, 16, st));
  TWG_CUDA(cudaMemcpyAsync(ctx.d_scalars + 18, off.p + V, 4, cudaMemcpyDeviceToDevice, st));
  TWG_CUDA(cudaMemcpyAsync(ctx.d_scalars + 19, goff.p + V, 4, cudaMemcpyDeviceToDevice, st));
  u64 pq[2];
  read_scalars(ctx, ctx.d_scalars + 18, pq, 2);
  if (pq[0] != g.P) fail(TWG_ECUDA, "ensure_compact: region sizes do not add up to the entry count");
  c->Q = pq[1];
  c->ent.alloc(g.P ? g.P : 1, st);
  c->owner.alloc(g.P ? g.P : 1, st);
  c->mk_time.alloc(c->Q ? c->Q : 1, st);
  c->mk_start.alloc(c->Q ? c->Q : 1, st);
  if (V) {
    k_compact_regions<<<grid(ctx, 32 * V), kBlock, 0, st>>>(g.nm.p, V, g.ent.p, g.mk_time.p, g.mk_start.p, g.seq0,
                                                            c->nmeta.p, c->ent.p, c->owner.p, c->mk_time.p,
                                                            c->mk_start.p);
    TWG_LAUNCHED(ctx);
  }
  build_nm(ctx, *c);
  c->has_weights = false;
  c->has_adjacency = false;
  TWG_CUDA(cudaStreamSynchronize(st));  // complete before another context's stream may read it
  g.compact = std::move(c);
  return *g.compact;
}

void ensure_adjacency(Ctx& ctx, Store& s) {
  if (s.gapped) return;  // streaming stores answer adjacency from the node view (walk.cu adjacent)
  std::lock_guard<std::mutex> lk(s.lazy_mu);
  if (s.has_adjacency) return;
  DevBuf<u32> owners(s.P ? s.P : 1, ctx.stream);
  if (s.P) {
    k_entry_owners<<<grid(ctx, s.V), kBlock, 0, ctx.stream>>>(s.nmeta.p, s.V, owners.p);
    TWG_LAUNCHED(ctx);
  }
  build_adjacency(ctx, s, owners.p);
}


// Canonical (time, src, dst) order of n edges given dense internal ids
// (edge_store.cpp:42-55; ties between identical triples are content-equal).
void sort_canonical(Ctx& ctx, const u32* src_i, const u32* dst_i, const i64* t, u64 m, i64 tmin, i64 tmax, int vb,
                    u32* o_src, u32* o_dst, i64* o_t) {
  if (m == 0) return;
  cudaStream_t st = ctx.stream;
  const int tb = bit_width_u64(static_cast<u64>(tmax - tmin));
  DevBuf<u64> k0(m, st), k1(m, st);
  u64* kp = k0.p;
  u64* ka = k1.p;
  if (tb + 2 * vb <= 64) {
    DevBuf<u32> v0(m, st);
    k_pack_canonical<<<grid(ctx, m), kBlock, 0, st>>>(src_i, dst_i, t, m, tmin, vb, kp, v0.p);
    TWG_LAUNCHED(ctx);
    u32* vnull = nullptr;
    u32* vnull2 = nullptr;
    radix_sort_pairs<u64>(ctx, &kp, &ka, &vnull, &vnull2, m, tb + 2 * vb);
    k_unpack_canonical<<<grid(ctx, m), kBlock, 0, st>>>(kp, m, tmin, vb, o_src, o_dst, o_t);
    TWG_LAUNCHED(ctx);
  } else {
    DevBuf<u32> v0(m, st), v1(m, st);
    u32* vp = v0.p;
    u32* va = v1.p;
    k_pack_pair<<<grid(ctx, m), kBlock, 0, st>>>(src_i, dst_i, m, vb, kp, vp);
    TWG_LAUNCHED(ctx);
    radix_sort_pairs<u64>(ctx, &kp, &ka, &vp, &va, m, 2 * vb);
    k_gather_time_key<<<grid(ctx, m), kBlock, 0, st>>>(t, vp, m, tmin, kp);
    TWG_LAUNCHED(ctx);
    radix_sort_pairs<u64>(ctx, &kp, &ka, &vp, &va, m, tb);
    k_gather_edges<<<grid(ctx, m), kBlock, 0, st>>>(src_i, dst_i, t, vp, m, o_src, o_dst, o_t);
    TWG_LAUNCHED(ctx);
  }
}

namespace {

// ts view scatter (edge_store.cpp:91-98): group starts -> ts_off / ts_time
struct TsScatter {
  const i64* t;
  u32* ts_off;
  i64* ts_time;
  __device__ __forceinline__ void operator()(u64 i, u64 g, u32 f) const {
    if (f) {
      ts_off[g] = static_cast<u32>(i);
      ts_time[g] = t[i];
    }
  }
};

__global__ void k_ts_tail(const u64* Z, u64 m, u32* ts_off) { ts_off[*Z] = static_cast<u32>(m); }

// node view scatter (edge_store.cpp:164-214): per-node timestamp-group
// marks, and at every region start the (entry, group) offsets of the node
// and of the empty-region nodes before it
struct NodeViewScatter {
  const u32* owner;
  const Entry* ent;
  i64* mk_time;
  u32* mk_start;
  uint2* nmeta;
  __device__ __forceinline__ void operator()(u64 p, u64 g, u32 f) const {
    if (!f) return;
    mk_time[g] = ent[p].t;
    mk_start[g] = static_cast<u32>(p);
    if (p == 0 || owner[p] != owner[p - 1]) {
      const u64 lo = p == 0 ? 0 : static_cast<u64>(owner[p - 1]) + 1;
      for (u64 v = lo; v <= owner[p]; ++v) nmeta[v] = make_uint2(static_cast<u32>(p), static_cast<u32>(g));
    }
  }
};

__global__ void k_node_tail(const u32* owner, u64 P, u64 V, const u64* Q, uint2* nmeta) {
  const u64 lo = P ? static_cast<u64>(owner[P - 1]) + 1 : 0;
  const uint2 x = make_uint2(static_cast<u32>(P), static_cast<u32>(*Q));
  for (u64 v = lo + blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v <= V;
       v += static_cast<u64>(gridDim.x) * blockDim.x)
    nmeta[v] = x;
}

}  // namespace

// ts_off / ts_time from the canonical time column (edge_store.cpp:91-98).
// One pass (flag + look-back scan + scatter); Z stays on the device in
// ctx.d_scalars[16] until finish_node_view reads Z and Q together.
void build_ts_view(Ctx& ctx, Store& s) {
  cudaStream_t st = ctx.stream;
  const u64 m = s.m;
  s.ts_off.alloc(m + 1, st);
  s.ts_time.alloc(m ? m : 1, st);
  scan_scatter(ctx, TimeChangeFn{s.e_t.p}, m, ctx.d_scalars + 16, TsScatter{s.e_t.p, s.ts_off.p, s.ts_time.p});
  k_ts_tail<<<1, 1, 0, st>>>(ctx.d_scalars + 16, m, s.ts_off.p);
  TWG_LAUNCHED(ctx);
}

// Region bounds, timestamp-group marks and group offsets from the node-sorted
// owner column + entries (edge_store.cpp:164-214), then the optional views.
void finish_node_view(Ctx& ctx, Store& s, BuildOpts opts) {
  cudaStream_t st = ctx.stream;
  const u64 P = s.P, V = s.V;
  const u32* okp = s.owner.p;
  s.nmeta.alloc(V + 1, st);
  s.mk_time.alloc(P ? P : 1, st);  // Q <= P
  s.mk_start.alloc(P ? P : 1, st);
  scan_scatter(ctx, GroupStartFn{okp, s.ent.p}, P, ctx.d_scalars + 17,
               NodeViewScatter{okp, s.ent.p, s.mk_time.p, s.mk_start.p, s.nmeta.p});
  k_node_tail<<<grid(ctx, V + 1), kBlock, 0, st>>>(okp, P, V, ctx.d_scalars + 17, s.nmeta.p);
  TWG_LAUNCHED(ctx);
  build_nm(ctx, s);
  u64 zq[2];
  read_scalars(ctx, ctx.d_scalars + 16, zq, 2);  // the build's one read-back of Z and Q
  s.Z = zq[0];
  s.Q = zq[1];
  s.has_weights = false;
  s.has_adjacency = false;
  if (opts.weights) ensure_weights(ctx, s);
  if (opts.adjacency) build_adjacency(ctx, s, okp);
}

Store* build_store(Ctx& ctx, EdgesSoA in, int mode, BuildOpts opts, u64* scratch_peak) {
  cudaStream_t st = ctx.stream;
  const u64 m = in.n;
  if (mode < 0 || mode > 2) fail(TWG_EINVAL, "edge store: unknown direction mode");
  if (m >= 0xffffffffull / 2) fail(TWG_EINVAL, "edge store: edge count exceeds 32-bit reference space");
  auto s = std::make_unique<Store>();
  s->ctx = &ctx;
  s->mode = mode;
  s->m = m;
  const u64 P = mode == TWG_UNDIRECTED ? 2 * m : m;
  s->P = P;
  u64 scratch = 0;

  if (m == 0) {
    s->nmeta.alloc(1, st);
    TWG_CUDA(cudaMemsetAsync(s->nmeta.p, 0, sizeof(uint2), st));
    s->nm.alloc(1, st);
    TWG_CUDA(cudaMemsetAsync(s->nm.p, 0, sizeof(NodeMeta), st));
    s->ts_off.alloc(1, st);
    TWG_CUDA(cudaMemsetAsync(s->ts_off.p, 0, sizeof(u32), st));
    s->adj_off.alloc(1, st);
    TWG_CUDA(cudaMemsetAsync(s->adj_off.p, 0, sizeof(u32), st));
    s->has_weights = true;
    s->has_adjacency = true;
    if (scratch_peak) *scratch_peak = 0;
    return s.release();
  }

  // 1. input statistics + validation (edge_store.cpp:32-38)
  u64 sc[5];
  k_init_stats<<<1, 1, 0, st>>>(ctx.d_scalars);
  TWG_LAUNCHED(ctx);
  k_edge_stats<<<grid(ctx, m), kBlock, 0, st>>>(in, ctx.d_scalars);
  TWG_LAUNCHED(ctx);
  read_scalars(ctx, ctx.d_scalars, sc, 5);
  if (sc[0]) fail(TWG_EINVAL, "edge store: negative timestamp");
  if (sc[1]) fail(TWG_EINVAL, "edge store: negative node id");
  const u64 max_id = sc[2];
  const i64 tmin = static_cast<i64>(sc[3]), tmax = static_cast<i64>(sc[4]);

  // 2. densify (edge_store.cpp:57-89)
  DevBuf<u32> src_i(m, st), dst_i(m, st);
  scratch += 8 * m;
  u64 V = 0;
  const bool dense = max_id < (1ull << 31) && max_id + 1 <= std::max<u64>(8 * m, 1ull << 22);
  if (dense) {
    const u64 range = max_id + 1;
    DevBuf<u32> present(range, st), rank(range + 1, st);
    scratch += 8 * range;
    TWG_CUDA(cudaMemsetAsync(present.p, 0, present.bytes(), st));
    k_mark_present<<<grid(ctx, m), kBlock, 0, st>>>(in, present.p);
    TWG_LAUNCHED(ctx);
    exclusive_scan<u32>(ctx, PresentFn{present.p}, range, rank.p);
    TWG_CUDA(cudaMemcpyAsync(ctx.d_scalars, rank.p + range, sizeof(u32), cudaMemcpyDeviceToDevice, st));
    TWG_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(ctx.d_scalars) + 4, 0, 4, st));
    read_scalars(ctx, ctx.d_scalars, sc, 1);
    V = sc[0];
    s->ext.alloc(V, st);
    k_fill_ext_dense<<<grid(ctx, range), kBlock, 0, st>>>(present.p, rank.p, range, s->ext.p);
    TWG_LAUNCHED(ctx);
    k_map_dense<<<grid(ctx, m), kBlock, 0, st>>>(in, rank.p, src_i.p, dst_i.p);
    TWG_LAUNCHED(ctx);
  } else {
    const u64 n2 = 2 * m;
    DevBuf<u64> k0(n2, st), k1(n2, st);
    scratch += 16 * n2;
    k_endpoints<<<grid(ctx, m), kBlock, 0, st>>>(in, k0.p);
    TWG_LAUNCHED(ctx);
    u64* kp = k0.p;
    u64* ka = k1.p;
    u32* vn = nullptr;
    u32* vn2 = nullptr;
    radix_sort_pairs<u64>(ctx, &kp, &ka, &vn, &vn2, n2, bit_width_u64(max_id));
    DevBuf<u32> uscan(n2 + 1, st);
    exclusive_scan<u32>(ctx, UniqueFlagFn{kp}, n2, uscan.p);
    TWG_CUDA(cudaMemcpyAsync(ctx.d_scalars, uscan.p + n2, sizeof(u32), cudaMemcpyDeviceToDevice, st));
    TWG_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(ctx.d_scalars) + 4, 0, 4, st));
    read_scalars(ctx, ctx.d_scalars, sc, 1);
    V = sc[0];
    s->ext.alloc(V, st);
    k_fill_ext_unique<<<grid(ctx, n2), kBlock, 0, st>>>(kp, uscan.p, n2, s->ext.p);
    TWG_LAUNCHED(ctx);
    k_map_sparse<<<grid(ctx, m), kBlock, 0, st>>>(in, s->ext.p, V, src_i.p, dst_i.p);
    TWG_LAUNCHED(ctx);
  }
  s->V = V;
  s->ext_identity = V > 0 && V == max_id + 1;  // every id 0..max present: rank == id

  // 3. canonical (time, src, dst) order (edge_store.cpp:42-55)
  const int vb = V > 1 ? bit_width_u64(V - 1) : 0;
  const int tb = bit_width_u64(static_cast<u64>(tmax - tmin));
  (void)tb;
  s->e_src.alloc(m, st);
  s->e_dst.alloc(m, st);
  s->e_t.alloc(m, st);
  scratch += 24 * m;
  sort_canonical(ctx, src_i.p, dst_i.p, in.t, m, tmin, tmax, vb, s->e_src.p, s->e_dst.p, s->e_t.p);
  s->last_t.alloc(V, st);
  TWG_CUDA(cudaMemsetAsync(s->last_t.p, 0xff, s->last_t.bytes(), st));  // -1: before every (non-negative) time
  k_node_last_t<<<grid(ctx, m), kBlock, 0, st>>>(src_i.p, dst_i.p, in.t, m, s->last_t.p);
  TWG_LAUNCHED(ctx);
  src_i.release();
  dst_i.release();

  // 4. timestamp-grouped view (edge_store.cpp:91-110)
  build_ts_view(ctx, *s);

  // 5. node-and-timestamp-grouped view (edge_store.cpp:112-214)
  DevBuf<u32> ok0(P, st), ok1(P, st), ov0(P, st), ov1(P, st);
  scratch += 16 * P;
  u32* okp = ok0.p;
  u32* oka = ok1.p;
  u32* ovp = ov0.p;
  u32* ova = ov1.p;
  k_owner_keys<<<grid(ctx, P), kBlock, 0, st>>>(s->e_src.p, s->e_dst.p, m, mode, okp, ovp);
  TWG_LAUNCHED(ctx);
  radix_sort_pairs<u32>(ctx, &okp, &oka, &ovp, &ova, P, vb);
  s->ent.alloc(P, st);
  k_entries<<<grid(ctx, P), kBlock, 0, st>>>(okp, ovp, P, mode, s->e_src.p, s->e_dst.p, s->e_t.p, s->ent.p);
  TWG_LAUNCHED(ctx);
  // owners of the sorted entries become the store's owner column
  s->owner = std::move(okp == ok0.p ? ok0 : ok1);
  finish_node_view(ctx, *s, opts);
  if (scratch_peak) *scratch_peak = scratch;
  return s.release();
}

}  // namespace twg
