// The C ABI (include/twg.h): object lifetimes, host<->device staging, error
// mapping. Every compute call is a device kernel; there is no CPU path.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "primitives.cuh"
#include "rng.cuh"
#include "walk.cuh"
#include "window.cuh"
#include "handles.cuh"

using namespace twg;

struct twg_edges {  // a device edge list (SoA columns)
  twg::Ctx* c = nullptr;
  twg::u64 n = 0;
  twg::DevBuf<twg::i64> src, dst, t;
};

namespace {

thread_local std::string g_error;
}  // namespace

void twg::set_last_error(const char* what) { g_error = what; }

namespace {

// CounterRng state for a seed (rng.hpp:25)
inline u64 mix64_host(u64 seed) { return mix64(seed ^ 0x6a09e667f3bcc909ULL); }

template <class F>
int guarded(F&& f) {
  try {
    f();
    return TWG_OK;
  } catch (const Error& e) {
    g_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_error = e.what();
    return TWG_ENOMEM;
  } catch (const std::exception& e) {
    g_error = e.what();
    return TWG_ECUDA;
  }
}

void require(bool ok, const char* what) {
  if (!ok) fail(TWG_EINVAL, what);
}

BuildOpts to_opts(const twg_build_opts* o) {
  BuildOpts b;
  if (o) {
    b.weights = o->weights != 0;
    b.adjacency = o->adjacency != 0;
  }
  return b;
}

template <class T>
void h2d(Ctx& c, DevBuf<T>& d, const T* h, u64 n) {
  d.alloc(n ? n : 1, c.stream);
  if (n) TWG_CUDA(cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, c.stream));
}

template <class T>
void d2h(Ctx& c, T* h, const T* d, u64 n) {
  if (n) TWG_CUDA(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, c.stream));
}

void sync(Ctx& c) { TWG_CUDA(cudaStreamSynchronize(c.stream)); }

__global__ void k_split_aos(const twg_edge* e, u64 n, i64* s, i64* d, i64* t) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const twg_edge x = e[i];
    s[i] = x.src;
    d[i] = x.dst;
    t[i] = x.t;
  }
}

struct SoA {
  DevBuf<i64> s, d, t;
};

void upload_edges(Ctx& c, const twg_edge* edges, u64 n, SoA& out) {
  DevBuf<twg_edge> raw;
  h2d(c, raw, edges, n);
  out.s.alloc(n ? n : 1, c.stream);
  out.d.alloc(n ? n : 1, c.stream);
  out.t.alloc(n ? n : 1, c.stream);
  if (n) {
    k_split_aos<<<grid_for(n, 256, c.sm_count * 16), 256, 0, c.stream>>>(raw.p, n, out.s.p, out.d.p, out.t.p);
    TWG_LAUNCHED(c);
  }
}

// ---- synthetic stream (C5 law; draws as synthetic.cpp:17-20, :92-96)
__host__ __device__ inline void stream_edge(u64 nodes, u64 i, u64 key, i64* s, i64* d, i64* t) {
  auto mix = [](u64 x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
  };
  auto bits = [&](u64 walk, u64 hop, u64 ord) { return mix(mix(mix(key ^ walk) ^ hop) ^ ord); };
  const double u = static_cast<double>(bits(2, i, 1) >> 11) * 0x1.0p-53;
#ifdef __CUDA_ARCH__
  i64 dv = static_cast<i64>(__dmul_rn(__dmul_rn(__dmul_rn(static_cast<double>(nodes), u), u), u));
#else
  i64 dv = static_cast<i64>(static_cast<double>(nodes) * u * u * u);
#endif
  if (dv > static_cast<i64>(nodes) - 1) dv = static_cast<i64>(nodes) - 1;
  *s = static_cast<i64>(bits(1, i, 0) % nodes);
  *d = dv;
  *t = static_cast<i64>(i / 4);
}

__global__ void k_synth_stream(u64 nodes, u64 first, u64 count, u64 key, i64* s, i64* d, i64* t) {
  for (u64 k = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; k < count;
       k += static_cast<u64>(gridDim.x) * blockDim.x)
    stream_edge(nodes, first + k, key, s + k, d + k, t + k);
}

// make_uniform_graph (synthetic.cpp:24-36)
__global__ void k_synth_uniform(u64 nodes, u64 count, i64 t_max, u64 key, i64* s, i64* d, i64* t) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    auto mix = [](u64 x) {
      x += 0x9e3779b97f4a7c15ULL;
      x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
      x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
      return x ^ (x >> 31);
    };
    auto bits = [&](u64 walk, u64 hop, u64 ord) { return mix(mix(mix(key ^ walk) ^ hop) ^ ord); };
    s[i] = static_cast<i64>(bits(1, i, 0) % nodes);
    d[i] = static_cast<i64>(bits(2, i, 0) % nodes);
    t[i] = static_cast<i64>(bits(3, i, 0) % (static_cast<u64>(t_max) + 1));
  }
}

}  // namespace

extern "C" {

int twg_abi_version(void) { return TWG_ABI_VERSION; }
const char* twg_last_error(void) { return g_error.c_str(); }

int twg_ctx_create(int device, twg_ctx** out) { return twg_ctx_create_prio(device, 0, out); }

int twg_ctx_create_prio(int device, int priority, twg_ctx** out) {
  return guarded([&] {
    auto* h = new twg_ctx;
    Ctx& c = h->c;
    try {
      c.device = device;
      TWG_CUDA(cudaSetDevice(device));
      TWG_CUDA(cudaDeviceGetAttribute(&c.sm_count, cudaDevAttrMultiProcessorCount, device));
      if (priority > 0) {  // the device's greatest priority: its kernels' blocks dispatch first
        int least = 0, greatest = 0;
        TWG_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        TWG_CUDA(cudaStreamCreateWithPriority(&c.stream, cudaStreamNonBlocking, greatest));
      } else {
        TWG_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
      }
      arena_register(c.stream);
      // glibc tables: same libm as the reference
      std::vector<double> e(kExpTableSize), x(701);
      for (int k = 0; k < kExpTableSize; ++k) e[k] = std::exp(static_cast<double>(-k));
      for (int n = 0; n <= 700; ++n) x[n] = std::expm1(static_cast<double>(n));
      TWG_CUDA(cudaMalloc(&c.d_exp_neg, e.size() * sizeof(double)));
      TWG_CUDA(cudaMalloc(&c.d_expm1, x.size() * sizeof(double)));
      TWG_CUDA(cudaMemcpy(c.d_exp_neg, e.data(), e.size() * sizeof(double), cudaMemcpyHostToDevice));
      TWG_CUDA(cudaMemcpy(c.d_expm1, x.data(), x.size() * sizeof(double), cudaMemcpyHostToDevice));
      TWG_CUDA(cudaHostAlloc(&c.h_pinned, 64 * sizeof(u64), cudaHostAllocMapped));
      TWG_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c.d_mapped), c.h_pinned, 0));
      for (int i = 0; i < 64; ++i) c.h_pinned[i] = 0;  // kMappedFlag starts below the first sequence number
      TWG_CUDA(cudaMalloc(&c.d_scalars, 64 * sizeof(u64)));
      TWG_CUDA(cudaStreamCreateWithFlags(&c.h2d_stream, cudaStreamNonBlocking));
      TWG_CUDA(cudaStreamCreateWithFlags(&c.d2h_stream, cudaStreamNonBlocking));
      for (auto& sl : c.slots) {
        TWG_CUDA(cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
        TWG_CUDA(cudaEventCreateWithFlags(&sl.consumed, cudaEventDisableTiming));
      }
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int twg_ctx_destroy(twg_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    Ctx& c = ctx->c;
    cudaStreamSynchronize(c.stream);
    if (c.svc_stream) {  // the picker service exits after its idle timeout
      cudaStreamSynchronize(c.svc_stream);
      cudaStreamDestroy(c.svc_stream);
      cudaFreeHost(c.pick_mbox);
    }
    cudaFree(c.d_exp_neg);
    cudaFree(c.d_expm1);
    cudaFree(c.d_scalars);
    cudaFreeHost(c.h_pinned);
    cudaStreamSynchronize(c.h2d_stream);
    cudaStreamSynchronize(c.d2h_stream);
    for (auto& sl : c.slots) {
      if (sl.buf) cudaFree(sl.buf);
      cudaEventDestroy(sl.ready);
      cudaEventDestroy(sl.consumed);
    }
    cudaStreamDestroy(c.h2d_stream);
    cudaStreamDestroy(c.d2h_stream);
    arena_unregister(c.stream);
    cudaStreamDestroy(c.stream);
    delete ctx;
  });
}

int twg_ctx_sync(twg_ctx* ctx) {
  return guarded([&] { sync(ctx->c); });
}

int twg_ctx_stream(twg_ctx* ctx, void** stream) {
  return guarded([&] { *stream = static_cast<void*>(ctx->c.stream); });
}

int twg_ctx_launch_count(twg_ctx* ctx, uint64_t* count) {
  return guarded([&] { *count = ctx->c.launches; });
}

// ---- store ------------------------------------------------------------------

int twg_store_build(twg_ctx* ctx, const twg_edge* edges, uint64_t n, int mode, const twg_build_opts* opts,
                    twg_store** out) {
  return guarded([&] {
    Ctx& c = ctx->c;
    if (n >= 0xffffffffull / 2) fail(TWG_EINVAL, "edge store: edge count exceeds 32-bit reference space");
    SoA soa;
    upload_edges(c, edges, n, soa);
    Store* s = build_store(c, EdgesSoA{soa.s.p, soa.d.p, soa.t.p, n}, mode, to_opts(opts));
    sync(c);
    *out = new twg_store{s};
  });
}

int twg_store_build_device(twg_ctx* ctx, const int64_t* d_src, const int64_t* d_dst, const int64_t* d_t, uint64_t n,
                           int mode, const twg_build_opts* opts, twg_store** out) {
  return guarded([&] {
    Store* s = build_store(ctx->c, EdgesSoA{d_src, d_dst, d_t, n}, mode, to_opts(opts));
    *out = new twg_store{s};
  });
}

int twg_store_retain(twg_store* s) {
  return guarded([&] { s->s->refs.fetch_add(1); });
}

int twg_store_release(twg_store* s) {
  return guarded([&] {
    if (!s) return;
    release_store(s->s);
    delete s;
  });
}

int twg_store_get_info(twg_store* h, twg_store_info* out) {
  return guarded([&] {
    const Store& s = *h->s;
    twg_store_info i{};
    i.edges = s.m;
    i.nodes = s.V;
    i.ts_groups = s.Z;
    i.entries = s.P;
    i.node_groups = s.Q;
    // a streaming store's optional views live on its contiguous form
    const Store& v = s.gapped && s.compact ? *s.compact : s;
    i.adjacency = v.has_adjacency ? v.A : 0;
    i.mode = s.mode;
    i.has_weights = v.has_weights;
    i.has_adjacency = v.has_adjacency;
    i.streaming = s.gapped ? 1 : 0;
    i.device_bytes = s.device_bytes();
    *out = i;
  });
}

namespace {
__global__ void k_max_ring_end(const NodeMeta* nm, u64 V, u64* out) {
  u32 mx = 0;
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<u64>(gridDim.x) * blockDim.x)
    mx = max(mx, nm[v].ee);
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(reinterpret_cast<unsigned long long*>(out), static_cast<u64>(mx));
}
}  // namespace

int twg_store_get_layout(twg_store* h, twg_store_layout* out) {
  return guarded([&] {
    const Store& s = *h->s;
    twg_store_layout l{};
    if (s.gapped) {
      Ctx& c = *s.ctx;
      l.log_cap = s.log->cap;
      l.log_first = s.log_first;
      l.ts_first = s.ts_first;
      l.arena_cap = s.arena->cap;
      l.arena_used = s.arena->used;
      l.arena_serial = s.arena->serial;
      l.relocated_rings = s.relocated;
      if (s.V) {
        TWG_CUDA(cudaMemsetAsync(c.d_scalars, 0, 8, c.stream));
        k_max_ring_end<<<grid_for(s.V, 256, c.sm_count * 8), 256, 0, c.stream>>>(s.nm.p, s.V, c.d_scalars);
        TWG_LAUNCHED(c);
        u64 r[1];
        read_scalars(c, c.d_scalars, r, 1);
        l.max_ring_end = r[0];
      }
    }
    *out = l;
  });
}

namespace {
__global__ void k_widen_u32(const u32* in, u64 n, u64* out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}
__global__ void k_ext_of(const u32* ids, const i64* ext, u64 n, i64* out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    out[i] = ext[ids[i]];
}
__global__ void k_meta_field(const uint2* meta, u64 n, int which, u64* out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    out[i] = which ? meta[i].y : meta[i].x;
}
__global__ void k_entry_field(const Entry* ent, u64 n, int which, u32* out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    out[i] = which ? ent[i].nbr : ent[i].edge;
}
}  // namespace

int twg_store_download(twg_store* h, int field, void* dst) {
  return guarded([&] {
    Store& s = ensure_compact(*h->s->ctx, *h->s);  // reference layout for accessors
    Ctx& c = *s.ctx;
    cudaStream_t st = c.stream;
    const unsigned g = grid_for(s.P + s.m + s.V + 1, 256, c.sm_count * 16);
    switch (field) {
      case 0: case 1: {
        DevBuf<i64> tmp(s.m ? s.m : 1, st);
        if (s.m) {
          k_ext_of<<<g, 256, 0, st>>>(field == 0 ? s.e_src.p : s.e_dst.p, s.ext.p, s.m, tmp.p);
          TWG_LAUNCHED(c);
        }
        d2h(c, static_cast<i64*>(dst), tmp.p, s.m);
        sync(c);
        break;
      }
      case 2: d2h(c, static_cast<i64*>(dst), s.e_t.p, s.m); break;
      case 3: d2h(c, static_cast<u32*>(dst), s.e_src.p, s.m); break;
      case 4: d2h(c, static_cast<u32*>(dst), s.e_dst.p, s.m); break;
      case 5: {
        DevBuf<u64> tmp(s.Z + 1, st);
        k_widen_u32<<<g, 256, 0, st>>>(s.ts_off.p, s.Z + 1, tmp.p);
        TWG_LAUNCHED(c);
        d2h(c, static_cast<u64*>(dst), tmp.p, s.Z + 1);
        sync(c);
        break;
      }
      case 6: d2h(c, static_cast<i64*>(dst), s.ts_time.p, s.Z); break;
      case 7: ensure_weights(c, s); d2h(c, static_cast<double*>(dst), s.ts_w.p, s.Z); break;
      case 8: case 9: {
        DevBuf<u64> tmp(s.V + 1, st);
        k_meta_field<<<g, 256, 0, st>>>(s.nmeta.p, s.V + 1, field == 9, tmp.p);
        TWG_LAUNCHED(c);
        d2h(c, static_cast<u64*>(dst), tmp.p, s.V + 1);
        sync(c);
        break;
      }
      case 10: d2h(c, static_cast<i64*>(dst), s.mk_time.p, s.Q); break;
      case 11: d2h(c, static_cast<u32*>(dst), s.mk_start.p, s.Q); break;
      case 12: case 15: {
        DevBuf<u32> tmp(s.P ? s.P : 1, st);
        if (s.P) {
          k_entry_field<<<g, 256, 0, st>>>(s.ent.p, s.P, field == 15, tmp.p);
          TWG_LAUNCHED(c);
        }
        d2h(c, static_cast<u32*>(dst), tmp.p, s.P);
        sync(c);
        break;
      }
      case 13: ensure_weights(c, s); d2h(c, static_cast<double*>(dst), s.wp.p, s.P); break;
      case 14: d2h(c, static_cast<i64*>(dst), s.ext.p, s.V); break;
      case 16: {
        ensure_adjacency(c, s);
        DevBuf<u64> tmp(s.V + 1, st);
        k_widen_u32<<<g, 256, 0, st>>>(s.adj_off.p, s.V + 1, tmp.p);
        TWG_LAUNCHED(c);
        d2h(c, static_cast<u64*>(dst), tmp.p, s.V + 1);
        sync(c);
        break;
      }
      case 17: ensure_adjacency(c, s); d2h(c, static_cast<u32*>(dst), s.adj.p, s.A); break;
      default: fail(TWG_EINVAL, "twg_store_download: unknown field");
    }
    sync(c);
  });
}

int twg_store_neighborhood(twg_store* h, const int64_t* v_ext, const int64_t* t, uint64_t n, int dir,
                           uint64_t* out3) {
  return guarded([&] {
    Store& s = ensure_compact(*h->s->ctx, *h->s);  // reference layout for accessors
    Ctx& c = *s.ctx;
    DevBuf<i64> dv, dt;
    h2d(c, dv, v_ext, n);
    h2d(c, dt, t, n);
    DevBuf<u64> o(3 * n + 1, c.stream);
    neighborhood_batch(c, s, dv.p, dt.p, n, dir, o.p);
    d2h(c, out3, o.p, 3 * n);
    sync(c);
  });
}

int twg_store_find_nodes(twg_store* h, const int64_t* v_ext, uint64_t n, uint32_t* internal, uint8_t* found) {
  return guarded([&] {
    Store& s = ensure_compact(*h->s->ctx, *h->s);  // reference layout for accessors
    Ctx& c = *s.ctx;
    DevBuf<i64> dv;
    h2d(c, dv, v_ext, n);
    DevBuf<u32> di(n + 1, c.stream);
    DevBuf<u8> df(n + 1, c.stream);
    find_nodes_batch(c, s, dv.p, n, di.p, df.p);
    d2h(c, internal, di.p, n);
    d2h(c, found, df.p, n);
    sync(c);
  });
}

int twg_store_adjacent(twg_store* h, const uint32_t* a, const uint32_t* b, uint64_t n, int temporal,
                       const int64_t* t, int dir, uint8_t* out) {
  return guarded([&] {
    Store& s = ensure_compact(*h->s->ctx, *h->s);  // reference layout for accessors
    Ctx& c = *s.ctx;
    for (u64 i = 0; i < n; ++i) require(a[i] < s.V && b[i] < s.V, "twg_store_adjacent: node id out of range");
    DevBuf<u32> da, db;
    DevBuf<i64> dt;
    h2d(c, da, a, n);
    h2d(c, db, b, n);
    if (temporal) h2d(c, dt, t, n);
    DevBuf<u8> o(n + 1, c.stream);
    adjacent_batch(c, s, da.p, db.p, n, temporal, dt.p, dir, o.p);
    d2h(c, out, o.p, n);
    sync(c);
  });
}

// ---- window -------------------------------------------------------------------

int twg_window_create(twg_ctx* ctx, int64_t duration, int mode, const twg_build_opts* opts, twg_window** out) {
  return guarded([&] {
    Window* w = window_create(ctx->c, duration, mode, to_opts(opts));
    *out = new twg_window{w, ctx};
  });
}

int twg_window_destroy(twg_window* w) {
  return guarded([&] {
    if (!w) return;
    window_destroy(w->w);
    delete w;
  });
}

int twg_window_ingest(twg_window* w, const twg_edge* batch, uint64_t n, twg_batch_stats* out) {
  return guarded([&] {
    Ctx& c = *w->w->ctx;
    SoA soa;
    upload_edges(c, batch, n, soa);
    window_ingest(*w->w, soa.s.p, soa.d.p, soa.t.p, n, out);
    sync(c);
  });
}

int twg_window_ingest_device(twg_window* w, const int64_t* d_src, const int64_t* d_dst, const int64_t* d_t,
                             uint64_t n, twg_batch_stats* out) {
  return guarded([&] { window_ingest(*w->w, d_src, d_dst, d_t, n, out); });
}

int twg_stage_batch(twg_ctx* ctx, int slot, const twg_edge* batch, uint64_t n) {
  return guarded([&] {
    require(slot == 0 || slot == 1, "twg_stage_batch: slot must be 0 or 1");
    Ctx& c = ctx->c;
    auto& sl = c.slots[slot];
    if (n > sl.cap) {  // grow (rare): the slot's previous contents must be consumed first
      TWG_CUDA(cudaEventSynchronize(sl.consumed));
      TWG_CUDA(cudaStreamSynchronize(c.h2d_stream));
      if (sl.buf) TWG_CUDA(cudaFree(sl.buf));
      TWG_CUDA(cudaMalloc(&sl.buf, n * sizeof(twg_edge)));
      sl.cap = n;
    }
    // never overwrite a slot the compute stream has not finished reading
    TWG_CUDA(cudaStreamWaitEvent(c.h2d_stream, sl.consumed, 0));
    if (n) TWG_CUDA(cudaMemcpyAsync(sl.buf, batch, n * sizeof(twg_edge), cudaMemcpyHostToDevice, c.h2d_stream));
    TWG_CUDA(cudaEventRecord(sl.ready, c.h2d_stream));
    sl.n = n;
  });
}

int twg_window_ingest_staged(twg_window* w, int slot, twg_batch_stats* out) {
  return guarded([&] {
    require(slot == 0 || slot == 1, "twg_window_ingest_staged: slot must be 0 or 1");
    Ctx& c = *w->w->ctx;
    auto& sl = c.slots[slot];
    const u64 n = sl.n;
    TWG_CUDA(cudaStreamWaitEvent(c.stream, sl.ready, 0));
    SoA soa;
    soa.s.alloc(n ? n : 1, c.stream);
    soa.d.alloc(n ? n : 1, c.stream);
    soa.t.alloc(n ? n : 1, c.stream);
    if (n) {
      k_split_aos<<<grid_for(n, 256, c.sm_count * 16), 256, 0, c.stream>>>(static_cast<const twg_edge*>(sl.buf), n,
                                                                           soa.s.p, soa.d.p, soa.t.p);
      TWG_LAUNCHED(c);
    }
    TWG_CUDA(cudaEventRecord(sl.consumed, c.stream));
    window_ingest(*w->w, soa.s.p, soa.d.p, soa.t.p, n, out);
  });
}

int twg_window_snapshot(twg_window* w, twg_store** out) {
  return guarded([&] {
    w->w->store->refs.fetch_add(1);
    *out = new twg_store{w->w->store};
  });
}

int twg_window_bounds(twg_window* w, int64_t* lo, int64_t* hi) {
  return guarded([&] {
    const Window& x = *w->w;
    if (x.batch_count == 0 || x.t_high == kTimeUnset)  // window_manager.cpp:65-66
      fail(TWG_ELOGIC, "window_bounds: no batch ingested yet");
    *lo = x.cutoff_for(x.t_high);
    *hi = x.t_high;
  });
}

int twg_window_state(twg_window* w, int64_t* t_high, uint64_t* batch_count, twg_batch_stats* last) {
  return guarded([&] {
    if (t_high) *t_high = w->w->t_high;
    if (batch_count) *batch_count = w->w->batch_count;
    if (last) *last = w->w->stats;
  });
}

// ---- walks -----------------------------------------------------------------------

int twg_generate(twg_ctx* ctx, twg_store* s, const twg_walk_config* config, const twg_thresholds* thresholds,
                 int variant, twg_walkset** out, twg_walk_stats* stats) {
  return guarded([&] {
    require(variant >= 0 && variant <= 2, "generate_walks: unknown variant");
    const twg_thresholds th = thresholds ? *thresholds : twg_thresholds{4, 256, 8192, 512, 4096};
    WalkSetDev* w = generate_walks(ctx->c, *s->s, *config, th, variant, stats);
    *out = new twg_walkset{w};
  });
}

int twg_walkset_destroy(twg_walkset* w) {
  return guarded([&] {
    if (!w) return;
    delete w->w;
    delete w;
  });
}

int twg_walkset_info(twg_walkset* w, uint32_t* stride, uint64_t* walk_count, uint64_t* first_walk, uint64_t* hops) {
  return guarded([&] {
    if (stride) *stride = w->w->stride;
    if (walk_count) *walk_count = w->w->count;
    if (first_walk) *first_walk = w->w->first;
    if (hops) *hops = w->w->hops;
  });
}

int twg_walkset_download(twg_walkset* w, int64_t* nodes, int64_t* times, uint32_t* lengths) {
  return guarded([&] {
    WalkSetDev& x = *w->w;
    Ctx& c = *x.ctx;
    const u64 cells = x.count * x.stride;
    DevBuf<i64> wn, wt;
    if (nodes || times) walk_major_image(c, x, wn, wt);  // device layout is slot-major
    if (nodes) d2h(c, nodes, wn.p, cells);
    if (times) d2h(c, times, wt.p, cells);
    if (lengths) d2h(c, lengths, x.lengths.p, x.count);
    sync(c);
  });
}

int twg_walkset_text(twg_walkset* w, void* dst, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    require(len != nullptr, "twg_walkset_text: len");
    WalkSetDev& x = *w->w;
    Ctx& c = *x.ctx;
    DevBuf<char> text;
    u64 bytes = 0;
    walks_text(c, x, text, &bytes);
    *len = bytes;
    if (dst) {
      require(cap >= bytes, "twg_walkset_text: buffer too small");
      if (bytes) d2h(c, static_cast<char*>(dst), text.p, bytes);
    }
    sync(c);
  });
}

int twg_walkset_binary(twg_walkset* w, void* dst, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    require(len != nullptr, "twg_walkset_binary: len");
    WalkSetDev& x = *w->w;
    Ctx& c = *x.ctx;
    const u64 bytes = walks_binary_size(x);
    *len = bytes;
    if (!dst) return;
    require(cap >= bytes, "twg_walkset_binary: buffer too small");
    char* p = static_cast<char*>(dst);
    std::memcpy(p, "TMPW0002", 8);  // kWalkBinaryMagic (io.hpp:29), then write_raw fields (io.cpp:175-176)
    const u32 stride = x.stride;
    const u64 count = x.count;
    std::memcpy(p + 8, &stride, 4);
    std::memcpy(p + 12, &count, 8);
    const u64 cells = count * stride;
    char* pn = p + kWalkBinaryHeader;
    char* pt = pn + 8 * cells;
    char* pl = pt + 8 * cells;
    DevBuf<i64> wn, wt;
    if (cells) {
      walk_major_image(c, x, wn, wt);
      TWG_CUDA(cudaMemcpyAsync(pn, wn.p, 8 * cells, cudaMemcpyDeviceToHost, c.stream));
      TWG_CUDA(cudaMemcpyAsync(pt, wt.p, 8 * cells, cudaMemcpyDeviceToHost, c.stream));
    }
    if (count) TWG_CUDA(cudaMemcpyAsync(pl, x.lengths.p, 4 * count, cudaMemcpyDeviceToHost, c.stream));
    sync(c);
  });
}

}  // extern "C"

namespace {

// The reference's ParseError text for a bad line (io.cpp:14-22, :52-59):
// re-derived on the host from the line's bytes and the device's verdict.
std::string edge_line_message(const char* text, u64 bytes, u64 line, u8 kind) {
  u64 b = 0;
  for (u64 n = 1; n < line && b < bytes; ++b)
    if (text[b] == '\n') ++n;
  u64 e = b;
  while (e < bytes && text[e] != '\n') ++e;
  if (e > b && text[e - 1] == '\r') --e;
  if (kind == kLineErrTabs) return "expected source<TAB>target<TAB>timestamp";
  const std::string l(text + b, e - b);
  const size_t t1 = l.find('\t'), t2 = l.find('\t', t1 + 1);
  static const char* names[3] = {"source", "target", "timestamp"};
  const int f = kind >= kLineErrNegative ? kind - kLineErrNegative : kind - kLineErrInvalid;
  if (kind >= kLineErrNegative) return std::string("negative ") + names[f];
  const std::string tok = f == 0 ? l.substr(0, t1) : f == 1 ? l.substr(t1 + 1, t2 - t1 - 1) : l.substr(t2 + 1);
  return std::string("invalid ") + names[f] + " '" + tok + "'";
}

void parse_tsv(Ctx& c, const char* text, u64 bytes, DevBuf<i64>& s, DevBuf<i64>& d, DevBuf<i64>& t, u64* count,
               uint64_t* error_line) {
  u64 line = 0;
  u8 kind = 0;
  parse_edges_tsv(c, text, bytes, s, d, t, count, &line, &kind);
  if (error_line) *error_line = line;
  if (line) throw Error(TWG_EPARSE, edge_line_message(text, bytes, line, kind));
}

__global__ void k_unpack_edges(const twg_edge* in, u64 n, i64* s, i64* d, i64* t) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const twg_edge x = in[i];
    s[i] = x.src;
    d[i] = x.dst;
    t[i] = x.t;
  }
}

__global__ void k_pack_edges(const i64* s, const i64* d, const i64* t, u64 n, twg_edge* out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    out[i] = twg_edge{s[i], d[i], t[i]};
}

}  // namespace

extern "C" {

int twg_parse_edges_tsv(twg_ctx* ctx, const char* text, uint64_t bytes, twg_edges** out, uint64_t* error_line) {
  return guarded([&] {
    require(out != nullptr && (bytes == 0 || text), "twg_parse_edges_tsv: arguments");
    auto e = std::make_unique<twg_edges>();
    e->c = &ctx->c;
    parse_tsv(ctx->c, text, bytes, e->src, e->dst, e->t, &e->n, error_line);
    *out = e.release();
  });
}

int twg_edges_from_host(twg_ctx* ctx, const twg_edge* edges, uint64_t n, twg_edges** out) {
  return guarded([&] {
    require(out != nullptr && (n == 0 || edges), "twg_edges_from_host: arguments");
    Ctx& c = ctx->c;
    auto e = std::make_unique<twg_edges>();
    e->c = &c;
    e->n = n;
    e->src.alloc(n ? n : 1, c.stream);
    e->dst.alloc(n ? n : 1, c.stream);
    e->t.alloc(n ? n : 1, c.stream);
    if (n) {
      DevBuf<twg_edge> aos(n, c.stream);
      TWG_CUDA(cudaMemcpyAsync(aos.p, edges, n * sizeof(twg_edge), cudaMemcpyHostToDevice, c.stream));
      k_unpack_edges<<<grid_for(n, 256, static_cast<unsigned>(c.sm_count) * 16), 256, 0, c.stream>>>(
          aos.p, n, e->src.p, e->dst.p, e->t.p);
      TWG_LAUNCHED(c);
      sync(c);
    }
    *out = e.release();
  });
}

int twg_edges_info(twg_edges* e, uint64_t* count) {
  return guarded([&] {
    require(count != nullptr, "twg_edges_info: count");
    *count = e->n;
  });
}

int twg_edges_download(twg_edges* e, twg_edge* out) {
  return guarded([&] {
    Ctx& c = *e->c;
    if (!e->n) return;
    require(out != nullptr, "twg_edges_download: out");
    DevBuf<twg_edge> aos(e->n, c.stream);
    k_pack_edges<<<grid_for(e->n, 256, static_cast<unsigned>(c.sm_count) * 16), 256, 0, c.stream>>>(
        e->src.p, e->dst.p, e->t.p, e->n, aos.p);
    TWG_LAUNCHED(c);
    d2h(c, out, aos.p, e->n);
    sync(c);
  });
}

int twg_edges_device(twg_edges* e, int64_t** d_src, int64_t** d_dst, int64_t** d_t) {
  return guarded([&] {
    if (d_src) *d_src = e->src.p;
    if (d_dst) *d_dst = e->dst.p;
    if (d_t) *d_t = e->t.p;
  });
}

int twg_edges_format_tsv(twg_edges* e, char* dst, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    require(len != nullptr, "twg_edges_format_tsv: len");
    Ctx& c = *e->c;
    DevBuf<char> text;
    u64 bytes = 0;
    format_edges_tsv(c, e->src.p, e->dst.p, e->t.p, e->n, text, &bytes);
    *len = bytes;
    if (dst) {
      require(cap >= bytes, "twg_edges_format_tsv: buffer too small");
      if (bytes) d2h(c, dst, text.p, bytes);
    }
    sync(c);
  });
}

int twg_edges_destroy(twg_edges* e) {
  delete e;
  return TWG_OK;
}

int twg_walkset_from_host(twg_ctx* ctx, uint32_t stride, uint64_t walk_count, const int64_t* nodes,
                          const int64_t* times, const uint32_t* lengths, twg_walkset** out) {
  return guarded([&] {
    require(out != nullptr, "twg_walkset_from_host: out");
    require(walk_count == 0 || (lengths && (stride == 0 || (nodes && times))), "twg_walkset_from_host: arrays");
    for (u64 i = 0; i < walk_count; ++i) require(lengths[i] <= stride, "twg_walkset_from_host: length > stride");
    auto w = std::make_unique<WalkSetDev>();
    walks_from_host(ctx->c, stride, walk_count, nodes, times, lengths, *w);
    *out = new twg_walkset{w.release()};
  });
}

int twg_walkset_audit(twg_walkset* w, twg_store* s, int direction, int strict, int64_t* first_violation,
                      twg_audit_report* out) {
  return guarded([&] {
    WalkSetDev& x = *w->w;
    Ctx& c = *x.ctx;
    require(direction == 0 || direction == 1, "twg_walkset_audit: direction");
    DevBuf<i64> first;
    if (first_violation) first.alloc(x.count ? x.count : 1, c.stream);
    u64 r[4];
    audit_walks(c, x, *s->s, direction, strict != 0, first_violation ? first.p : nullptr, r);
    if (first_violation && x.count) d2h(c, first_violation, first.p, x.count);
    sync(c);
    if (out) *out = twg_audit_report{r[0], r[1], r[2], r[3]};
  });
}

int twg_walkset_download_compact(twg_walkset* w, uint64_t* offsets, int64_t* nodes, int64_t* times) {
  return guarded([&] {
    WalkSetDev& x = *w->w;
    Ctx& c = *x.ctx;
    DevBuf<u64> offs;
    DevBuf<i64> cn, ct;
    u64 total = 0;
    compact_walks(c, x, offs, cn, ct, &total);
    if (offsets) d2h(c, offsets, offs.p, x.count + 1);
    if (nodes) d2h(c, nodes, cn.p, total);
    if (times) d2h(c, times, ct.p, total);
    sync(c);
  });
}

int twg_walkset_download_compact_async(twg_walkset* w, uint64_t* offsets, int64_t* nodes, int64_t* times,
                                       uint64_t capacity, uint64_t* total_entries) {
  return guarded([&] {
    WalkSetDev& x = *w->w;
    Ctx& c = *x.ctx;
    if (x.d2h_done) TWG_CUDA(cudaEventSynchronize(x.d2h_done));  // a previous download still reads the buffers
    u64 total = 0;
    compact_walks(c, x, x.c_off, x.c_nodes, x.c_times, &total);
    if (total_entries) *total_entries = total;
    if (total > capacity) fail(TWG_EINVAL, "twg_walkset_download_compact_async: host capacity too small");
    if (!x.d2h_done) TWG_CUDA(cudaEventCreateWithFlags(&x.d2h_done, cudaEventDisableTiming));
    cudaEvent_t compacted;
    TWG_CUDA(cudaEventCreateWithFlags(&compacted, cudaEventDisableTiming));
    TWG_CUDA(cudaEventRecord(compacted, c.stream));
    TWG_CUDA(cudaStreamWaitEvent(c.d2h_stream, compacted, 0));
    cudaEventDestroy(compacted);
    if (offsets)
      TWG_CUDA(cudaMemcpyAsync(offsets, x.c_off.p, (x.count + 1) * 8, cudaMemcpyDeviceToHost, c.d2h_stream));
    if (nodes && total) TWG_CUDA(cudaMemcpyAsync(nodes, x.c_nodes.p, total * 8, cudaMemcpyDeviceToHost, c.d2h_stream));
    if (times && total) TWG_CUDA(cudaMemcpyAsync(times, x.c_times.p, total * 8, cudaMemcpyDeviceToHost, c.d2h_stream));
    TWG_CUDA(cudaEventRecord(x.d2h_done, c.d2h_stream));
  });
}

int twg_walkset_wait(twg_walkset* w) {
  return guarded([&] {
    if (w->w->d2h_done) TWG_CUDA(cudaEventSynchronize(w->w->d2h_done));
  });
}

int twg_walkset_device(twg_walkset* w, int64_t** d_nodes, int64_t** d_times, uint32_t** d_lengths) {
  return guarded([&] {
    if (d_nodes) *d_nodes = w->w->nodes.p;
    if (d_times) *d_times = w->w->times.p;
    if (d_lengths) *d_lengths = w->w->lengths.p;
  });
}

int twg_sample_start_edges(twg_store* h, int bias, const double* u1, const double* u2, uint64_t n, uint64_t* out) {
  return guarded([&] {
    Store& s = ensure_compact(*h->s->ctx, *h->s);  // reference layout for accessors
    Ctx& c = *s.ctx;
    for (u64 i = 0; i < n; ++i)
      require(u1[i] >= 0.0 && u1[i] < 1.0 && u2[i] >= 0.0 && u2[i] < 1.0, "picker: u outside [0,1)");
    DevBuf<double> a, b;
    h2d(c, a, u1, n);
    h2d(c, b, u2, n);
    DevBuf<u64> o(n + 1, c.stream);
    sample_start_edges(c, s, bias, a.p, b.p, n, o.p);
    d2h(c, out, o.p, n);
    sync(c);
  });
}

int twg_schedule_step(twg_store* h, const uint32_t* node_of_walk, const uint8_t* alive, uint64_t n,
                      const twg_thresholds* thresholds, uint64_t* sizes5, uint32_t* rows, uint64_t cap,
                      uint32_t* walk_ids) {
  return guarded([&] {
    Store& s = ensure_compact(*h->s->ctx, *h->s);  // reference layout for accessors
    Ctx& c = *s.ctx;
    const twg_thresholds th = thresholds ? *thresholds : twg_thresholds{4, 256, 8192, 512, 4096};
    for (u64 i = 0; i < n; ++i) require(!alive[i] || node_of_walk[i] < s.V, "schedule_step: node id out of range");
    DevBuf<u32> dn;
    DevBuf<u8> da;
    h2d(c, dn, node_of_walk, n);
    h2d(c, da, alive, n);
    schedule_step_explicit(c, s, dn.p, da.p, n, th, sizes5, rows, cap, walk_ids);
  });
}

int twg_init_walks(twg_ctx* ctx, twg_store* s, const twg_walk_config* config, uint32_t* stride, uint64_t* walk_count,
                   uint32_t* current, int64_t* time, uint32_t* prev, uint8_t* has_prev, uint8_t* alive,
                   uint32_t* length, int64_t* nodes, int64_t* times) {
  return guarded([&] {
    HostWalkArrays out{current, time, prev, has_prev, alive, length, nodes, times};
    const bool fill = current && time && prev && has_prev && alive && length && nodes && times;
    init_walks_dev(ctx->c, *s->s, *config, stride, walk_count, fill ? &out : nullptr);
  });
}

int twg_hop_walks(twg_ctx* ctx, twg_store* s, const twg_walk_config* config, const uint32_t* walk_ids, uint64_t n_ids,
                  uint64_t walk_count, uint32_t stride, uint32_t* current, int64_t* time, uint32_t* prev,
                  uint8_t* has_prev, uint8_t* alive, uint32_t* length, int64_t* nodes, int64_t* times) {
  return guarded([&] {
    for (u64 i = 0; i < n_ids; ++i) require(walk_ids[i] < walk_count, "hop_walks: walk id out of range");
    for (u64 i = 0; i < n_ids; ++i)
      require(current[walk_ids[i]] < s->s->V && length[walk_ids[i]] < stride, "hop_walks: walk state out of range");
    HostWalkArrays io{current, time, prev, has_prev, alive, length, nodes, times};
    hop_walks_dev(ctx->c, *s->s, *config, walk_ids, n_ids, walk_count, stride, io);
  });
}

int twg_radix_sort_pairs(twg_ctx* ctx, uint64_t* keys, uint32_t* values, uint64_t n) {
  return guarded([&] {
    Ctx& c = ctx->c;
    require(n < (1ull << 32), "radix_sort_pairs: n");
    DevBuf<u64> k;
    DevBuf<u32> v;
    h2d(c, k, keys, n);
    h2d(c, v, values, n);
    radix_sort_pairs_dev(c, k.p, v.p, n);
    d2h(c, keys, k.p, n);
    d2h(c, values, v.p, n);
    sync(c);
  });
}

int twg_exclusive_scan(twg_ctx* ctx, const uint64_t* in, uint64_t* out, uint64_t n, uint64_t* total) {
  return guarded([&] {
    Ctx& c = ctx->c;
    DevBuf<u64> a, b(n + 1, c.stream);
    h2d(c, a, in, n);
    exclusive_scan_dev(c, a.p, b.p, n);
    d2h(c, out, b.p, n);
    u64 t[1];
    read_scalars(c, b.p + n, t, 1);
    if (total) *total = t[0];
  });
}

int twg_run_length_encode(twg_ctx* ctx, const uint64_t* sorted_keys, uint64_t n, uint64_t* out_rows, uint64_t* runs) {
  return guarded([&] {
    Ctx& c = ctx->c;
    DevBuf<u64> k, rows(3 * n + 3, c.stream);
    h2d(c, k, sorted_keys, n);
    const u64 r = run_length_encode_dev(c, k.p, n, rows.p);
    d2h(c, out_rows, rows.p, 3 * r);
    sync(c);
    *runs = r;
  });
}

int twg_partition_flagged(twg_ctx* ctx, const uint32_t* items, uint64_t n, const uint8_t* flags, uint64_t flags_len,
                          uint32_t* out, uint64_t* kept) {
  return guarded([&] {
    Ctx& c = ctx->c;
    for (u64 i = 0; i < n; ++i) require(items[i] < flags_len, "partition_flagged: item outside flags");
    DevBuf<u32> it, o(n + 1, c.stream);
    DevBuf<u8> fl;
    h2d(c, it, items, n);
    h2d(c, fl, flags, flags_len);
    const u64 k = partition_flagged_dev(c, it.p, n, fl.p, o.p);
    d2h(c, out, o.p, k);
    sync(c);
    *kept = k;
  });
}

int twg_pick_index(twg_ctx* ctx, int kind, const double* u, const uint64_t* n, uint64_t count, uint64_t* out) {
  return guarded([&] {
    require(kind >= 0 && kind <= 2, "twg_pick_index: kind");
    for (u64 i = 0; i < count; ++i) {  // samplers.cpp:10-13
      if (n[i] == 0) fail(TWG_EINVAL, "picker: empty candidate set");
      if (!(u[i] >= 0.0) || u[i] >= 1.0) fail(TWG_EINVAL, "picker: u outside [0,1)");
    }
    Ctx& c = ctx->c;
    if (count <= PickSmall::kMax) {  // scalar façade calls: no device buffers, no copies
      pick_index_small(c, kind, u, n, static_cast<u32>(count), out);
      return;
    }
    DevBuf<double> du;
    DevBuf<u64> dn;
    h2d(c, du, u, count);
    h2d(c, dn, n, count);
    DevBuf<u64> o(count + 1, c.stream);
    pick_index_batch(c, kind, du.p, dn.p, count, o.p);
    d2h(c, out, o.p, count);
    sync(c);
  });
}

int twg_pick_weighted_range(twg_ctx* ctx, const double* u, const double* prefix, uint64_t len, const uint64_t* begin,
                            const uint64_t* end, const double* base, uint64_t count, uint64_t* out) {
  return guarded([&] {
    for (u64 i = 0; i < count; ++i) require(begin[i] < end[i] && end[i] <= len, "pick_weighted_range: bad range");
    Ctx& c = ctx->c;
    DevBuf<double> du, dp, db;
    DevBuf<u64> dbeg, dend;
    h2d(c, du, u, count);
    h2d(c, dp, prefix, len);
    h2d(c, db, base, count);
    h2d(c, dbeg, begin, count);
    h2d(c, dend, end, count);
    DevBuf<u64> o(count + 1, c.stream);
    pick_weighted_range_batch(c, du.p, dp.p, dbeg.p, dend.p, db.p, count, o.p);
    d2h(c, out, o.p, count);
    sync(c);
  });
}

int twg_rng_bits(twg_ctx* ctx, int rng, uint64_t seed, const uint64_t* walk, const uint64_t* hop,
                 const uint64_t* ordinal, uint64_t count, uint64_t* out) {
  return guarded([&] {
    require(rng == TWG_RNG_SPLITMIX || rng == TWG_RNG_PHILOX, "twg_rng_bits: rng");
    Ctx& c = ctx->c;
    DevBuf<u64> dw, dh, dor;
    h2d(c, dw, walk, count);
    h2d(c, dh, hop, count);
    h2d(c, dor, ordinal, count);
    DevBuf<u64> o(count + 1, c.stream);
    rng_bits_batch(c, rng, seed, dw.p, dh.p, dor.p, count, o.p);
    d2h(c, out, o.p, count);
    sync(c);
  });
}

// ---- synthetic inputs -----------------------------------------------------------------

int twg_synth_stream_host(uint64_t nodes, uint64_t first, uint64_t count, uint64_t seed, twg_edge* out) {
  return guarded([&] {
    require(nodes > 0, "twg_synth_stream_host: nodes");
    const u64 key = mix64_host(seed);
#pragma omp parallel for schedule(static)
    for (long long k = 0; k < static_cast<long long>(count); ++k)
      stream_edge(nodes, first + static_cast<u64>(k), key, &out[k].src, &out[k].dst, &out[k].t);
  });
}

int twg_synth_stream_device(twg_ctx* ctx, uint64_t nodes, uint64_t first, uint64_t count, uint64_t seed,
                            int64_t* d_src, int64_t* d_dst, int64_t* d_t) {
  return guarded([&] {
    require(nodes > 0, "twg_synth_stream_device: nodes");
    Ctx& c = ctx->c;
    if (!count) return;
    k_synth_stream<<<grid_for(count, 256, c.sm_count * 32), 256, 0, c.stream>>>(nodes, first, count, mix64_host(seed),
                                                                                d_src, d_dst, d_t);
    TWG_LAUNCHED(c);
  });
}

int twg_synth_graph(twg_ctx* ctx, int kind, uint64_t a, uint64_t b, int64_t t_max, uint64_t seed, twg_edge* out,
                    uint64_t cap, uint64_t* count) {
  return guarded([&] {
    require(count != nullptr && kind >= 0 && kind <= 3, "twg_synth_graph: kind");
    require(kind != 0 || (a > 0 && t_max >= 0), "twg_synth_graph: uniform needs nodes > 0 and t_max >= 0");
    require(kind != 1 || a > 0, "twg_synth_graph: hub-skewed needs background nodes > 0");
    require(kind != 3 || b > 0, "twg_synth_graph: time ladder needs rungs > 0");
    const u64 n = synth_graph_size(kind, a, b);
    *count = n;
    if (!out) return;
    require(cap >= n, "twg_synth_graph: buffer too small");
    synth_graph(ctx->c, kind, a, b, t_max, mix64_host(seed), out);
  });
}

int twg_synth_uniform_device(twg_ctx* ctx, uint64_t nodes, uint64_t count, int64_t t_max, uint64_t seed,
                             int64_t* d_src, int64_t* d_dst, int64_t* d_t) {
  return guarded([&] {
    require(nodes > 0 && t_max >= 0, "twg_synth_uniform_device: args");
    Ctx& c = ctx->c;
    if (!count) return;
    k_synth_uniform<<<grid_for(count, 256, c.sm_count * 32), 256, 0, c.stream>>>(nodes, count, t_max,
                                                                                 mix64_host(seed), d_src, d_dst, d_t);
    TWG_LAUNCHED(c);
  });
}

}  // extern "C"
