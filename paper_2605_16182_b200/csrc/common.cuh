// Shared host/device plumbing for libtimewalk_b200: errors, the per-context
// stream + stream-ordered pool, device buffers, launch accounting.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>

#include "twg.h"

namespace twg {

using u8 = uint8_t;
using u16 = uint16_t;
using u32 = uint32_t;
using u64 = uint64_t;
using i64 = int64_t;

constexpr i64 kTimeUnset = INT64_MIN;     // types.hpp:23
constexpr i64 kTimeInfinite = INT64_MAX;  // types.hpp:25
constexpr int kExpTableSize = 746;        // exp(-k), k = 0..745 (glibc); exp(-746) == +0

// Error carrying a TWG_* status (mapped onto the reference exception types).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "%s failed at %s:%d: %s", what, file, line,
                  cudaGetErrorString(e));
    fail(e == cudaErrorMemoryAllocation ? TWG_ENOMEM : TWG_ECUDA, buf);
  }
}
#define TWG_CUDA(x) ::twg::cuda_check((x), #x, __FILE__, __LINE__)
#define TWG_LAUNCHED(ctx) \
  do {                    \
    ::twg::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); \
    (ctx).launches++;     \
  } while (0)

// start the DRAM fetch of the line holding p into L2 (no register, no wait)
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

struct Ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  cudaMemPool_t pool = nullptr;
  u64 launches = 0;
  // glibc exp(-k) for k = 0..745 and expm1(n) for n = 0..700, computed on the
  // host by the same libm the reference links (App. A of SURVEY.md).
  double* d_exp_neg = nullptr;
  double* d_expm1 = nullptr;
  // pinned scratch for small device->host reads
  u64* h_pinned = nullptr;   // mapped pinned host scalars (see read_scalars)
  u64* d_mapped = nullptr;   // device alias of h_pinned
  u64* d_scalars = nullptr;  // 64 u64 scratch scalars on the device
  u64 mapped_seq = 0;        // sequence number of the last mapped read-back (h_pinned[kMappedFlag])
  // scalar picker service (queries.cu): a one-warp kernel on its own stream
  // serving requests posted in mapped pinned memory while they keep coming
  void* pick_mbox = nullptr;     // host view of the mailbox (PickMailbox)
  void* pick_mbox_d = nullptr;   // device view
  cudaStream_t svc_stream = nullptr;
  u64 pick_seq = 0;
  // Streaming pipeline: host batches are staged into device slots on a copy
  // stream (H2D overlaps the compute stream) and walk downloads run on a D2H
  // stream. Slot buffers are plain cudaMalloc (used across streams).
  cudaStream_t h2d_stream = nullptr;
  cudaStream_t d2h_stream = nullptr;
  struct Slot {
    void* buf = nullptr;
    u64 cap = 0;  // edges
    u64 n = 0;
    cudaEvent_t ready = nullptr;     // H2D done
    cudaEvent_t consumed = nullptr;  // compute stream finished reading it
  } slots[2];
};

// Per-stream caching allocator (arena.cu). Every ctx owns one, keyed by its
// stream. Blocks are rounded to size classes (<= 12.5% slack) and recycled
// in stream order, so the steady-state ingest/walk loop performs no device
// allocation at all (cudaMallocAsync pool growth cost up to 200 ms per batch
// in round-1 measurements, profiles/r1_baseline_fullrebuild.md).
void arena_register(cudaStream_t s);
void arena_unregister(cudaStream_t s);
void* arena_alloc(cudaStream_t s, size_t bytes);
void arena_free(cudaStream_t s, void* p, size_t bytes);
size_t arena_bytes_in_use(cudaStream_t s);
size_t arena_bytes_reserved(cudaStream_t s);

// Device buffer allocated from the ctx arena of `stream`.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  bool own = true;  // false: a view into memory owned elsewhere (shared logs / arenas)

  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s), own(o.own) { o.p = nullptr; o.n = 0; o.own = true; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s; own = o.own;
      o.p = nullptr; o.n = 0; o.own = true;
    }
    return *this;
  }
  ~DevBuf() { release(); }

  // non-owning view of count elements at q (the owner outlives this buffer)
  void alias(T* q, size_t count) {
    release();
    p = q;
    n = count;
    own = false;
  }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    own = true;
    s = stream;
    n = count;
    if (count) p = static_cast<T*>(arena_alloc(stream, count * sizeof(T)));
  }
  // grow-only reallocation (contents not preserved)
  void reserve(size_t count, cudaStream_t stream) {
    if (count > n || p == nullptr) alloc(count < 1 ? 1 : count, stream);
  }
  void release() {
    if (p && own) arena_free(s, p, n * sizeof(T));
    p = nullptr;
    n = 0;
    own = true;
  }
  size_t bytes() const { return n * sizeof(T); }
  T* get() const { return p; }
};

// Opt-in phase timing (TWG_PHASES=1): CUDA events on the ctx stream between
// named phases, printed to stderr at the end of the scope. Zero cost when off.
struct PhaseTimer {
  Ctx& ctx;
  const char* scope;
  bool on;
  int n = 0;
  cudaEvent_t ev[48];
  const char* name[48];
  // NVTX: the scope is a range and every phase boundary a mark on the
  // host timeline (nvtx3 is header-only; free when no tool is attached)
  PhaseTimer(Ctx& c, const char* s) : ctx(c), scope(s) {
    static const bool enabled = [] {
      const char* e = std::getenv("TWG_PHASES");
      return e && e[0] == '1';
    }();
    on = enabled;
    nvtxRangePushA(s);
    mark("start");
  }
  void mark(const char* what) {
    nvtxMarkA(what);
    if (!on || n >= 48) return;
    cudaEventCreate(&ev[n]);
    cudaEventRecord(ev[n], ctx.stream);
    name[n++] = what;
  }
  ~PhaseTimer() {
    nvtxRangePop();
    if (!on) return;
    mark("end");
    cudaEventSynchronize(ev[n - 1]);
    std::fprintf(stderr, "[twg phases] %s:", scope);
    float total = 0.f;
    for (int i = 1; i < n; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      total += ms;
      std::fprintf(stderr, " %s=%.2f", name[i], ms);
    }
    std::fprintf(stderr, " | total=%.2f ms\n", total);
    for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
  }
};

// an NVTX range over a host scope (walk generation, one ingest, ...)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

inline int bit_width_u64(u64 x) {
  int b = 0;
  while (x) { ++b; x >>= 1; }
  return b;
}

inline unsigned grid_for(u64 n, unsigned block, unsigned cap = 1u << 20) {
  u64 g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// small synchronous device -> host read of n u64 scalars via pinned memory
void read_scalars(Ctx& ctx, const u64* d_src, u64* host_dst, int n);
// h_pinned[kMappedFlag] receives the sequence number of a mapped read-back
// once its values are visible to the host (written after a system fence)
constexpr int kMappedFlag = 63;
// spin until the kernel that publishes `seq` has written it (no stream
// synchronisation: the host polls the mapped word; a failed or drained
// stream without the flag raises)
void mapped_wait(Ctx& ctx, u64 seq);

}  // namespace twg
