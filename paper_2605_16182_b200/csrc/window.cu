// WindowManager on the device (window_manager.cpp:9-69).
//
// Per batch: batch_high by a device max-reduction; cutoff_for(new_high)
// (window_manager.hpp:51-53); survivors = the suffix of the time-sorted
// store at lower_bound(e_t, cutoff) (export_suffix, edge_store.cpp:325-332),
// gathered back to external ids on the device; admitted batch edges
// (t >= cutoff, window_manager.cpp:39-46) compacted by flag+scan behind them;
// then the full dual-index rebuild over the merged set. Snapshot swap keeps
// exactly one retired snapshot alive (window_manager.cpp:56-57); callers may
// hold any snapshot longer through the store's reference count.
#include <chrono>

#include "primitives.cuh"
#include "window.cuh"

namespace twg {

namespace {

constexpr int kBlock = 256;

__global__ void k_init_max(i64* v) { *v = kTimeUnset; }

__global__ void k_batch_max(const i64* t, u64 n, i64* out) {
  i64 m = kTimeUnset;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    m = max(m, t[i]);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<long long*>(out), static_cast<long long>(m));
}

// lower_bound(time_, cutoff) (edge_store.cpp:326)
__global__ void k_lower_bound(const i64* t, u64 m, i64 cutoff, u64* out) {
  u64 lo = 0, hi = m;
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if (t[mid] < cutoff) lo = mid + 1;
    else hi = mid;
  }
  *out = lo;
}

__global__ void k_gather_survivors(StoreView s, u64 from, i64* src, i64* dst, i64* t) {
  const u64 n = s.m - from;
  for (u64 k = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 i = from + k;
    src[k] = s.ext[s.e_src[i]];
    dst[k] = s.ext[s.e_dst[i]];
    t[k] = s.e_t[i];
  }
}

struct AdmitFn {
  const i64* t;
  i64 cutoff;
  __device__ __forceinline__ u32 operator()(u64 i) const { return t[i] >= cutoff ? 1u : 0u; }
};

__global__ void k_compact_batch(const i64* bs, const i64* bd, const i64* bt, u64 n, i64 cutoff, const u32* pos,
                                u64 base, i64* src, i64* dst, i64* t) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    if (bt[i] >= cutoff) {
      const u64 k = base + pos[i];
      src[k] = bs[i];
      dst[k] = bd[i];
      t[k] = bt[i];
    }
  }
}

unsigned grid(Ctx& ctx, u64 n) { return grid_for(n, kBlock, static_cast<unsigned>(ctx.sm_count) * 16); }

}  // namespace

void release_store(Store* s) {
  if (s && s->refs.fetch_sub(1) == 1) delete s;
}

Window* window_create(Ctx& ctx, i64 duration, int mode, BuildOpts opts) {
  if (duration <= 0) fail(TWG_EINVAL, "window duration must be positive");  // window_manager.cpp:10
  if (mode < 0 || mode > 2) fail(TWG_EINVAL, "window: unknown direction mode");
  auto w = new Window;
  w->ctx = &ctx;
  w->duration = duration;
  w->mode = mode;
  w->opts = opts;
  try {
    w->store = build_store(ctx, EdgesSoA{nullptr, nullptr, nullptr, 0}, mode, opts);
  } catch (...) {
    delete w;
    throw;
  }
  return w;
}

void window_destroy(Window* w) {
  if (!w) return;
  release_store(w->store);
  release_store(w->previous);
  delete w;
}

void window_ingest(Window& w, const i64* d_src, const i64* d_dst, const i64* d_t, u64 n, twg_batch_stats* out) {
  using clock = std::chrono::steady_clock;
  const auto started = clock::now();
  Ctx& ctx = *w.ctx;
  cudaStream_t st = ctx.stream;
  twg_batch_stats stats{};
  stats.ingested = n;
  if (n == 0) {  // window_manager.cpp:21-28
    stats.retained = w.store->m;
    stats.peak_bytes = w.store->device_bytes();
    w.stats = stats;
    ++w.batch_count;
    if (out) *out = stats;
    return;
  }
  // batch_high, new_high, cutoff (window_manager.cpp:30-33)
  k_init_max<<<1, 1, 0, st>>>(reinterpret_cast<i64*>(ctx.d_scalars));
  TWG_LAUNCHED(ctx);
  k_batch_max<<<grid(ctx, n), kBlock, 0, st>>>(d_t, n, reinterpret_cast<i64*>(ctx.d_scalars));
  TWG_LAUNCHED(ctx);
  const Store& old = *w.store;
  u64 sc[1];
  read_scalars(ctx, ctx.d_scalars, sc, 1);
  const i64 batch_high = static_cast<i64>(sc[0]);
  const i64 new_high = w.t_high > batch_high ? w.t_high : batch_high;
  const i64 cutoff = w.cutoff_for(new_high);

  // survivors: suffix of the old time-sorted store (export_suffix)
  k_lower_bound<<<1, 1, 0, st>>>(old.e_t.p, old.m, cutoff, ctx.d_scalars + 1);
  TWG_LAUNCHED(ctx);
  DevBuf<u32> pos(n + 1, st);
  exclusive_scan<u32>(ctx, AdmitFn{d_t, cutoff}, n, pos.p);
  TWG_CUDA(cudaMemsetAsync(ctx.d_scalars + 2, 0, 8, st));
  TWG_CUDA(cudaMemcpyAsync(ctx.d_scalars + 2, pos.p + n, 4, cudaMemcpyDeviceToDevice, st));
  u64 r[3];
  read_scalars(ctx, ctx.d_scalars, r, 3);
  const u64 from = r[1];
  const u64 survivors = old.m - from;
  const u64 admitted = r[2];
  stats.evicted = old.m - survivors;
  stats.dropped_late = n - admitted;

  const u64 total = survivors + admitted;
  DevBuf<i64> ms(total ? total : 1, st), md(total ? total : 1, st), mt(total ? total : 1, st);
  if (survivors) {
    k_gather_survivors<<<grid(ctx, survivors), kBlock, 0, st>>>(old.view(), from, ms.p, md.p, mt.p);
    TWG_LAUNCHED(ctx);
  }
  if (admitted) {
    k_compact_batch<<<grid(ctx, n), kBlock, 0, st>>>(d_src, d_dst, d_t, n, cutoff, pos.p, survivors, ms.p, md.p,
                                                     mt.p);
    TWG_LAUNCHED(ctx);
  }
  pos.release();
  u64 scratch = 0;
  Store* rebuilt = build_store(ctx, EdgesSoA{ms.p, md.p, mt.p, total}, w.mode, w.opts, &scratch);

  stats.retained = rebuilt->m;
  stats.peak_bytes = old.device_bytes() + 24 * total + rebuilt->device_bytes() + scratch;
  TWG_CUDA(cudaStreamSynchronize(st));
  stats.rebuild_duration = std::chrono::duration<double>(clock::now() - started).count();
  release_store(w.previous);
  w.previous = w.store;
  w.store = rebuilt;
  w.t_high = new_high;
  w.stats = stats;
  ++w.batch_count;
  if (out) *out = stats;
}

}  // namespace twg
