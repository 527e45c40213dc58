// Multi-GPU replica group (include/twg.h "multi-GPU replica group"; SURVEY
// §8e): the per-batch loop of replay_stream (replay.cpp:16-53) across GPUs,
// one process per GPU.
//
//  * Index: REPLICATED. The root packs its batch into the wire format (16 B
//    per edge — u32 src, u32 dst, i64 t, three planes — when every id is in
//    [0, 2^32), else the 24-B triple) and ONE ncclBroadcast over NVLink moves
//    it into every rank's staging slot on the group's copy stream, so batch
//    k+1 travels while batch k is ingested and walked. Every rank (the root
//    included) unpacks the same wire bytes and runs the same deterministic
//    ingest, so replicas are identical by construction; a 64-bit hash of each
//    new snapshot is all-reduced (max of {h, ~h}) and a disagreement is
//    reported on the batch that causes it.
//  * Walks: PARTITIONED. Rank r generates slice r of the global walk-id
//    range; RNG draws are keyed by global walk ids (rng.hpp:22-43), so the
//    union of the shards is byte-identical to one GPU generating every id.
//    Walk counters are all-reduced (sums; wall time = max).
//
// Two communicators: `data` (broadcasts, copy stream) and `ctl` (reductions,
// the ctx stream), so a broadcast in flight never orders the control path.
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <cstring>

#include "handles.cuh"

using namespace twg;

namespace twg {
namespace {

// NCCL is resolved at run time (dlopen), not linked: a process that imports
// PyTorch already holds PyTorch's own libnccl.so.2, and a second NCCL linked
// into this library would claim the same soname first and break it. The
// copy already loaded in the process wins (RTLD_NOLOAD); otherwise
// TWG_NCCL_LIB, else the system libnccl.so.2.
struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

const Nccl& nccl() {
  static Nccl api = [] {
    Nccl a{};
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) {
      const char* e = std::getenv("TWG_NCCL_LIB");
      h = dlopen(e && *e ? e : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) fail(TWG_ECUDA, std::string("multi-GPU group: cannot load NCCL (libnccl.so.2): ") + dlerror());
    auto sym = [h](const char* n) {
      void* f = dlsym(h, n);
      if (!f) fail(TWG_ECUDA, std::string("multi-GPU group: NCCL lacks ") + n);
      return f;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommSplit = reinterpret_cast<decltype(a.CommSplit)>(sym("ncclCommSplit"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    std::string m = std::string("NCCL: ") + what + ": " + nccl().GetErrorString(r);
    fail(TWG_ECUDA, m);
  }
}
#define TWG_NCCL(x) nccl_check((x), #x)

constexpr int kB = 256;
unsigned gridn(const Ctx& c, u64 n) { return grid_for(n, kB, static_cast<unsigned>(c.sm_count) * 8); }

// root: 24-B SoA batch -> 16-B wire planes; flag[0] |= 1 when an id is outside [0, 2^32)
__global__ void k_pack(const i64* s, const i64* d, const i64* t, u64 n, u32* ws, u32* wd, i64* wt, u64* flag) {
  u32 bad = 0;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const i64 a = s[i], b = d[i];
    bad |= (static_cast<u64>(a) >> 32) | (static_cast<u64>(b) >> 32) ? 1u : 0u;
    ws[i] = static_cast<u32>(a);
    wd[i] = static_cast<u32>(b);
    wt[i] = t[i];
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(reinterpret_cast<unsigned long long*>(flag), 1ull);
}

// root, host batch: AoS triples (after one H2D) -> wire planes
__global__ void k_pack_aos(const twg_edge* e, u64 n, int narrow, u32* ws, u32* wd, i64* wt, i64* ws64, i64* wd64,
                           u64* flag) {
  u32 bad = 0;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const twg_edge x = e[i];
    bad |= (static_cast<u64>(x.src) >> 32) | (static_cast<u64>(x.dst) >> 32) ? 1u : 0u;
    if (narrow) {
      ws[i] = static_cast<u32>(x.src);
      wd[i] = static_cast<u32>(x.dst);
    } else {
      ws64[i] = x.src;
      wd64[i] = x.dst;
    }
    wt[i] = x.t;
  }
  if (flag && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    atomicOr(reinterpret_cast<unsigned long long*>(flag), 1ull);
}

__global__ void k_scan_ids(const twg_edge* e, u64 n, u64* flag) {
  u32 bad = 0;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    bad |= (static_cast<u64>(e[i].src) >> 32) | (static_cast<u64>(e[i].dst) >> 32) ? 1u : 0u;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(reinterpret_cast<unsigned long long*>(flag), 1ull);
}

// every rank: 16-B wire planes -> the i64 SoA columns the ingest reads
__global__ void k_unpack(const u32* ws, const u32* wd, u64 n, i64* s, i64* d) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    s[i] = ws[i];
    d[i] = wd[i];
  }
}

__device__ __forceinline__ u64 hmix(u64 x) {  // splitmix64 finaliser
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// Order-independent hash of a snapshot's logical content: per node its
// bounds (eb, ee, gb, ge, cap — the ring base comes from a bump allocator
// and differs between replicas), its newest entry and its external id; the
// newest `tail` edges of the time-sorted edge sequence; the counts.
__global__ void k_replica_hash(StoreView v, u64 tail_from, u64* out) {
  u64 h = 0;
  const u64 tid = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 x = tid; x < v.V; x += stride) {
    const NodeMeta m = v.nm[x];
    u64 k = hmix(x ^ (static_cast<u64>(m.eb) << 32 | m.ee));
    k = hmix(k ^ (static_cast<u64>(m.gb) << 32 | m.ge));
    k = hmix(k ^ m.cap);
    if (m.ee != m.eb) {
      const Entry e = v.ent[entry_ring(m)(m.ee - 1)];
      k = hmix(k ^ (static_cast<u64>(e.nbr) << 32 | (e.edge - v.seq0)));
      k = hmix(k ^ static_cast<u64>(e.t));
    }
    if (v.ext) k = hmix(k ^ static_cast<u64>(v.ext[x]));
    h += k;
  }
  for (u64 i = tail_from + tid; i < v.m; i += stride) {
    const EdgeRec r = edge_at(v, i);
    h += hmix(hmix(i ^ (static_cast<u64>(r.src) << 32 | r.dst)) ^ static_cast<u64>(r.t));
  }
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(reinterpret_cast<unsigned long long*>(out), static_cast<unsigned long long>(h));
}

__global__ void k_hash_pair(const u64* h, u64 counts_mix, u64* pair) {
  pair[0] = h[0] ^ counts_mix;
  pair[1] = ~pair[0];
}

u64 counts_mix(const Store& s) {
  auto mix = [](u64 x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
  };
  return mix(mix(mix(mix(mix(s.m) ^ s.V) ^ s.Z) ^ s.P) ^ s.Q);
}

// device-side hash of s into d_out (one u64; d_out zeroed here)
void replica_hash_dev(Ctx& c, const Store& s, u64 tail, u64* d_out) {
  TWG_CUDA(cudaMemsetAsync(d_out, 0, sizeof(u64), c.stream));
  const u64 from = (tail == 0 || tail >= s.m) ? 0 : s.m - tail;
  k_replica_hash<<<gridn(c, s.V + (s.m - from) + 1), kB, 0, c.stream>>>(s.view(), from, d_out);
  TWG_LAUNCHED(c);
}

// a small device->host read on an arbitrary stream (the copy stream's header)
__global__ void k_publish(const u64* src, volatile u64* mapped, int n, u64 seq) {
  if (static_cast<int>(threadIdx.x) < n) mapped[threadIdx.x] = src[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    mapped[31] = seq;
  }
}

}  // namespace
}  // namespace twg

struct twg_group {
  twg_ctx* ctx = nullptr;
  int nranks = 1, rank = 0;
  ncclComm_t data = nullptr, ctl = nullptr;
  cudaStream_t copy = nullptr;     // broadcasts (and the root's pack / H2D)
  u64* h_map = nullptr;            // mapped pinned words for header read-backs on the copy stream
  u64* d_map = nullptr;
  u64 seq = 0;
  u64* d_small = nullptr;          // device scratch: [0..1] header, [2] pack flag, [4..5] hash pair, [8..] stats
  struct Slot {
    void* wire = nullptr;          // broadcast target: planes src | dst | t
    u64 cap_bytes = 0;
    void* host_stage = nullptr;    // root, host variant: the H2D'd AoS batch
    u64 host_cap = 0;
    u64 n = 0;
    int narrow = 1;
    cudaEvent_t ready = nullptr;   // broadcast landed (copy stream)
    cudaEvent_t consumed = nullptr;// the ctx stream finished unpacking it
  } slots[2];

  Ctx& c() { return ctx->c; }

  // host wait for `n` words of d_src written in copy-stream order
  void read_copy_stream(const u64* d_src, u64* out, int n) {
    const u64 s = ++seq;
    k_publish<<<1, 32, 0, copy>>>(d_src, d_map, n, s);
    TWG_LAUNCHED(c());
    volatile u64* f = h_map + 31;
    for (u32 spin = 1; *f != s; ++spin) {
      if ((spin & 4095) == 0) {
        const cudaError_t e = cudaStreamQuery(copy);
        if (e == cudaSuccess && *f != s) fail(TWG_ECUDA, "group: copy stream drained without publishing");
        if (e != cudaSuccess && e != cudaErrorNotReady) cuda_check(e, "group read-back", __FILE__, __LINE__);
      }
      __builtin_ia32_pause();
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    for (int i = 0; i < n; ++i) out[i] = reinterpret_cast<volatile u64*>(h_map)[i];
  }

  void ensure_wire(Slot& sl, u64 bytes) {
    if (bytes <= sl.cap_bytes) return;
    // the slot's previous contents must be consumed before it is replaced
    TWG_CUDA(cudaEventSynchronize(sl.consumed));
    TWG_CUDA(cudaStreamSynchronize(copy));
    if (sl.wire) TWG_CUDA(cudaFree(sl.wire));
    TWG_CUDA(cudaMalloc(&sl.wire, bytes));
    sl.cap_bytes = bytes;
  }
};

namespace {

template <class F>
int gguarded(F&& f) {
  try {
    f();
    return TWG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return TWG_ECUDA;
  }
}

// Broadcast header {n, narrow} from the root, then the wire planes.
// root_prep: on the root, fills the wire planes of `sl` for n edges (copy
// stream) and returns narrow (1: 16 B/edge).
template <class RootPrep>
void stage(twg_group& g, int slot, int root, u64 n_root, RootPrep root_prep) {
  if (slot != 0 && slot != 1) fail(TWG_EINVAL, "group stage: slot must be 0 or 1");
  if (root < 0 || root >= g.nranks) fail(TWG_EINVAL, "group stage: root outside the group");
  Ctx& c = g.c();
  auto& sl = g.slots[slot];
  // never overwrite a slot the ctx stream has not finished reading
  TWG_CUDA(cudaStreamWaitEvent(g.copy, sl.consumed, 0));
  u64 hdr[2] = {0, 1};
  if (g.rank == root) {
    hdr[0] = n_root;
    hdr[1] = static_cast<u64>(root_prep(sl));  // packs on the copy stream (may read back its flag)
    TWG_CUDA(cudaMemcpyAsync(g.d_small, hdr, sizeof(hdr), cudaMemcpyHostToDevice, g.copy));
  }
  if (g.nranks > 1) {
    TWG_NCCL(nccl().Broadcast(g.d_small, g.d_small, 2, ncclUint64, root, g.data, g.copy));
    if (g.rank != root) g.read_copy_stream(g.d_small, hdr, 2);
  }
  const u64 n = hdr[0];
  const int narrow = hdr[1] != 0;
  const u64 bytes = n * (narrow ? 16 : 24);
  if (g.rank != root) g.ensure_wire(sl, bytes ? bytes : 16);
  if (g.nranks > 1 && bytes)
    TWG_NCCL(nccl().Broadcast(sl.wire, sl.wire, bytes, ncclUint8, root, g.data, g.copy));
  TWG_CUDA(cudaEventRecord(sl.ready, g.copy));
  sl.n = n;
  sl.narrow = narrow;
  (void)c;
}

void ingest_staged(twg_group& g, twg_window* w, int slot, twg_group_batch_stats* out) {
  if (slot != 0 && slot != 1) fail(TWG_EINVAL, "group ingest: slot must be 0 or 1");
  Ctx& c = g.c();
  if (w->w->ctx != &c) fail(TWG_EINVAL, "group ingest: the window belongs to another context");
  auto& sl = g.slots[slot];
  const u64 n = sl.n;
  TWG_CUDA(cudaStreamWaitEvent(c.stream, sl.ready, 0));
  DevBuf<i64> s64, d64;
  const i64* ps;
  const i64* pd;
  const i64* pt;
  if (sl.narrow) {
    const u32* ws = static_cast<const u32*>(sl.wire);
    s64.alloc(n ? n : 1, c.stream);
    d64.alloc(n ? n : 1, c.stream);
    if (n) {
      k_unpack<<<gridn(c, n), kB, 0, c.stream>>>(ws, ws + n, n, s64.p, d64.p);
      TWG_LAUNCHED(c);
    }
    ps = s64.p;
    pd = d64.p;
    pt = reinterpret_cast<const i64*>(ws + 2 * n);
  } else {
    const i64* wi = static_cast<const i64*>(sl.wire);
    ps = wi;
    pd = wi + n;
    pt = wi + 2 * n;
  }
  twg_batch_stats st{};
  window_ingest(*w->w, ps, pd, pt, n, &st);
  TWG_CUDA(cudaEventRecord(sl.consumed, c.stream));
  // replica agreement: hash of the new snapshot, all-reduced as max{h, ~h}
  u64 pair[2] = {0, 0};
  replica_hash_dev(c, *w->w->store, n, g.d_small + 4);
  k_hash_pair<<<1, 1, 0, c.stream>>>(g.d_small + 4, counts_mix(*w->w->store), g.d_small + 6);
  TWG_LAUNCHED(c);
  if (g.nranks > 1) TWG_NCCL(nccl().AllReduce(g.d_small + 6, g.d_small + 8, 2, ncclUint64, ncclMax, g.ctl, c.stream));
  else TWG_CUDA(cudaMemcpyAsync(g.d_small + 8, g.d_small + 6, 16, cudaMemcpyDeviceToDevice, c.stream));
  TWG_CUDA(cudaMemcpyAsync(g.d_small + 10, g.d_small + 6, 8, cudaMemcpyDeviceToDevice, c.stream));
  u64 r[3];
  read_scalars(c, g.d_small + 8, r, 3);  // [0] max h, [1] max ~h, [2] own h
  pair[0] = r[2];
  if (out) {
    out->local = st;
    out->replica_hash = pair[0];
    out->replicas_agree = (r[0] == ~r[1]) ? 1 : 0;  // max h == min h
    out->wire_bytes_per_edge = sl.narrow ? 16 : 24;
    out->edges = n;
  }
}

}  // namespace

extern "C" {

int twg_group_unique_id(uint8_t id[TWG_GROUP_ID_BYTES]) {
  return gguarded([&] {
    static_assert(sizeof(ncclUniqueId) == TWG_GROUP_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    TWG_NCCL(nccl().GetUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
  });
}

int twg_group_create(twg_ctx* ctx, int nranks, int rank, const uint8_t id[TWG_GROUP_ID_BYTES], twg_group** out) {
  return gguarded([&] {
    if (!ctx || nranks < 1 || rank < 0 || rank >= nranks) fail(TWG_EINVAL, "group: bad rank / size");
    auto* g = new twg_group;
    try {
      g->ctx = ctx;
      g->nranks = nranks;
      g->rank = rank;
      Ctx& c = ctx->c;
      TWG_CUDA(cudaSetDevice(c.device));
      ncclUniqueId u;
      std::memcpy(&u, id, sizeof(u));
      TWG_NCCL(nccl().CommInitRank(&g->data, nranks, u, rank));
      TWG_NCCL(nccl().CommSplit(g->data, 0, rank, &g->ctl, nullptr));
      TWG_CUDA(cudaStreamCreateWithFlags(&g->copy, cudaStreamNonBlocking));
      TWG_CUDA(cudaHostAlloc(&g->h_map, 32 * sizeof(u64), cudaHostAllocMapped));
      std::memset(g->h_map, 0, 32 * sizeof(u64));
      TWG_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&g->d_map), g->h_map, 0));
      TWG_CUDA(cudaMalloc(&g->d_small, 32 * sizeof(u64)));
      for (auto& sl : g->slots) {
        TWG_CUDA(cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
        TWG_CUDA(cudaEventCreateWithFlags(&sl.consumed, cudaEventDisableTiming));
      }
    } catch (...) {
      twg_group_destroy(g);
      throw;
    }
    *out = g;
  });
}

int twg_group_destroy(twg_group* g) {
  return gguarded([&] {
    if (!g) return;
    if (g->copy) cudaStreamSynchronize(g->copy);
    if (g->ctx) cudaStreamSynchronize(g->ctx->c.stream);
    for (auto& sl : g->slots) {
      if (sl.wire) cudaFree(sl.wire);
      if (sl.host_stage) cudaFree(sl.host_stage);
      if (sl.ready) cudaEventDestroy(sl.ready);
      if (sl.consumed) cudaEventDestroy(sl.consumed);
    }
    if (g->d_small) cudaFree(g->d_small);
    if (g->h_map) cudaFreeHost(g->h_map);
    if (g->copy) cudaStreamDestroy(g->copy);
    if (g->ctl) nccl().CommDestroy(g->ctl);
    if (g->data) nccl().CommDestroy(g->data);
    delete g;
  });
}

int twg_group_info(twg_group* g, int* nranks, int* rank) {
  return gguarded([&] {
    if (nranks) *nranks = g->nranks;
    if (rank) *rank = g->rank;
  });
}

int twg_group_stage_device(twg_group* g, int slot, int root, const int64_t* d_src, const int64_t* d_dst,
                           const int64_t* d_t, uint64_t n) {
  return gguarded([&] {
    Ctx& c = g->c();
    // the root's columns are ready in ctx-stream order
    cudaEvent_t ev;
    TWG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TWG_CUDA(cudaEventRecord(ev, c.stream));
    TWG_CUDA(cudaStreamWaitEvent(g->copy, ev, 0));
    TWG_CUDA(cudaEventDestroy(ev));
    stage(*g, slot, root, n, [&](twg_group::Slot& sl) -> int {
      g->ensure_wire(sl, n ? 16 * n : 16);
      TWG_CUDA(cudaMemsetAsync(g->d_small + 2, 0, 8, g->copy));
      u32* ws = static_cast<u32*>(sl.wire);
      if (n) {
        k_pack<<<gridn(c, n), kB, 0, g->copy>>>(d_src, d_dst, d_t, n, ws, ws + n, reinterpret_cast<i64*>(ws + 2 * n),
                                               g->d_small + 2);
        TWG_LAUNCHED(c);
      }
      u64 bad[1];
      g->read_copy_stream(g->d_small + 2, bad, 1);
      if (!bad[0]) return 1;
      // an id outside 32 bits: the 24-B triple goes on the wire
      g->ensure_wire(sl, 24 * n);
      i64* wi = static_cast<i64*>(sl.wire);
      TWG_CUDA(cudaMemcpyAsync(wi, d_src, 8 * n, cudaMemcpyDeviceToDevice, g->copy));
      TWG_CUDA(cudaMemcpyAsync(wi + n, d_dst, 8 * n, cudaMemcpyDeviceToDevice, g->copy));
      TWG_CUDA(cudaMemcpyAsync(wi + 2 * n, d_t, 8 * n, cudaMemcpyDeviceToDevice, g->copy));
      return 0;
    });
  });
}

int twg_group_stage_host(twg_group* g, int slot, int root, const twg_edge* batch, uint64_t n) {
  return gguarded([&] {
    Ctx& c = g->c();
    stage(*g, slot, root, n, [&](twg_group::Slot& sl) -> int {
      if (n > sl.host_cap) {
        TWG_CUDA(cudaStreamSynchronize(g->copy));
        if (sl.host_stage) TWG_CUDA(cudaFree(sl.host_stage));
        TWG_CUDA(cudaMalloc(&sl.host_stage, n * sizeof(twg_edge)));
        sl.host_cap = n;
      }
      const twg_edge* de = static_cast<const twg_edge*>(sl.host_stage);
      if (n) TWG_CUDA(cudaMemcpyAsync(sl.host_stage, batch, n * sizeof(twg_edge), cudaMemcpyHostToDevice, g->copy));
      TWG_CUDA(cudaMemsetAsync(g->d_small + 2, 0, 8, g->copy));
      if (n) {
        k_scan_ids<<<gridn(c, n), kB, 0, g->copy>>>(de, n, g->d_small + 2);
        TWG_LAUNCHED(c);
      }
      u64 bad[1];
      g->read_copy_stream(g->d_small + 2, bad, 1);
      const int narrow = bad[0] ? 0 : 1;
      g->ensure_wire(sl, n ? n * (narrow ? 16 : 24) : 16);
      if (n) {
        u32* ws = static_cast<u32*>(sl.wire);
        i64* wi = static_cast<i64*>(sl.wire);
        k_pack_aos<<<gridn(c, n), kB, 0, g->copy>>>(de, n, narrow, ws, ws + n,
                                                    narrow ? reinterpret_cast<i64*>(ws + 2 * n) : wi + 2 * n, wi,
                                                    wi + n, nullptr);
        TWG_LAUNCHED(c);
      }
      return narrow;
    });
  });
}

int twg_group_staged_edges(twg_group* g, int slot, uint64_t* n) {
  return gguarded([&] {
    if (slot != 0 && slot != 1) fail(TWG_EINVAL, "group: slot must be 0 or 1");
    *n = g->slots[slot].n;
  });
}

int twg_group_ingest_staged(twg_group* g, twg_window* w, int slot, twg_group_batch_stats* out) {
  return gguarded([&] { ingest_staged(*g, w, slot, out); });
}

int twg_group_ingest_device(twg_group* g, twg_window* w, int root, const int64_t* d_src, const int64_t* d_dst,
                            const int64_t* d_t, uint64_t n, twg_group_batch_stats* out) {
  const int rc = twg_group_stage_device(g, 0, root, d_src, d_dst, d_t, n);
  if (rc != TWG_OK) return rc;
  return twg_group_ingest_staged(g, w, 0, out);
}

int twg_group_ingest(twg_group* g, twg_window* w, int root, const twg_edge* batch, uint64_t n,
                     twg_group_batch_stats* out) {
  const int rc = twg_group_stage_host(g, 0, root, batch, n);
  if (rc != TWG_OK) return rc;
  return twg_group_ingest_staged(g, w, 0, out);
}

int twg_group_generate(twg_group* g, twg_store* s, const twg_walk_config* config, const twg_thresholds* thresholds,
                       int variant, twg_walkset** out, twg_walk_stats* local, twg_walk_stats* global) {
  return gguarded([&] {
    if (variant < 0 || variant > 2) fail(TWG_EINVAL, "generate_walks: unknown variant");
    Ctx& c = g->c();
    const twg_thresholds th = thresholds ? *thresholds : twg_thresholds{4, 256, 8192, 512, 4096};
    twg_walk_stats st{};
    WalkSetDev* w = generate_walks(c, *s->s, *config, th, variant, &st, g->rank, g->nranks);
    *out = new twg_walkset{w};
    if (local) *local = st;
    if (global) {
      // counters (u64 words of twg_walk_stats except wall_seconds) summed, wall time max
      constexpr int kWords = 9;
      u64 words[kWords + 2] = {st.walks, st.hops, st.steps, st.solo, st.warp_cached, st.warp_direct,
                               st.block_cached, st.block_direct, st.multi_block, st.ambiguous_draws,
                               st.alg_bytes};
      u64 tw = 0;
      std::memcpy(&tw, &st.wall_seconds, 8);  // non-negative doubles order like their bits
      u64* d = g->d_small + 12;
      TWG_CUDA(cudaMemcpyAsync(d, words, sizeof(words), cudaMemcpyHostToDevice, c.stream));
      TWG_CUDA(cudaMemcpyAsync(d + 11, &tw, 8, cudaMemcpyHostToDevice, c.stream));
      if (g->nranks > 1) {
        TWG_NCCL(nccl().AllReduce(d, d, kWords + 2, ncclUint64, ncclSum, g->ctl, c.stream));
        TWG_NCCL(nccl().AllReduce(d + 11, d + 11, 1, ncclUint64, ncclMax, g->ctl, c.stream));
      }
      u64 r[12];
      read_scalars(c, d, r, 12);
      twg_walk_stats gs{};
      gs.walks = r[0];
      gs.hops = r[1];
      gs.steps = r[2];
      gs.solo = r[3];
      gs.warp_cached = r[4];
      gs.warp_direct = r[5];
      gs.block_cached = r[6];
      gs.block_direct = r[7];
      gs.multi_block = r[8];
      gs.ambiguous_draws = r[9];
      gs.alg_bytes = r[10];
      std::memcpy(&gs.wall_seconds, &r[11], 8);
      *global = gs;
    }
  });
}

int twg_store_replica_hash(twg_store* s, uint64_t tail, uint64_t* hash) {
  return gguarded([&] {
    Store& st = *s->s;
    Ctx& c = *st.ctx;
    replica_hash_dev(c, st, tail, c.d_scalars + 60);
    k_hash_pair<<<1, 1, 0, c.stream>>>(c.d_scalars + 60, counts_mix(st), c.d_scalars + 61);
    TWG_LAUNCHED(c);
    u64 r[1];
    read_scalars(c, c.d_scalars + 61, r, 1);
    *hash = r[0];
  });
}

}  // extern "C"
