// Per-stream caching device allocator (see common.cuh). Size classes: powers
// of two up to 1 MiB, then 8 classes per octave. A freed block goes back to
// its class list and is handed to the next request of that class on the same
// stream — stream order makes the reuse safe without events. On an
// allocation failure every cached block of every class is released and the
// request retried once.
//
// TWG_GUARD=1 (a debug mode for the guard test, tests/test_gpu_sanitizer.py):
// every block is poisoned (0xA5) when handed out, so a read of memory no
// kernel wrote changes results, and carries a 4 KiB guard past the requested
// bytes that is checked when the block is freed (a synchronous read-back), so
// a write past the end of an allocation is reported on stderr.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace twg {

namespace {

struct Arena {
  std::map<size_t, std::vector<void*>> free_lists;
  std::unordered_map<void*, size_t> owned;  // live block -> its class
  size_t in_use = 0;
  size_t reserved = 0;
  std::unordered_map<void*, size_t> asked;  // TWG_GUARD: live block -> requested bytes
};

constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kPoison = 0xA5;
size_t guard_bytes() {
  static const size_t g = [] {
    const char* e = std::getenv("TWG_GUARD");
    return (e && *e && *e != '0') ? kGuardBytes : size_t(0);
  }();
  return g;
}

std::mutex g_mu;
std::unordered_map<cudaStream_t, Arena*>& arenas() {
  static auto* m = new std::unordered_map<cudaStream_t, Arena*>;
  return *m;
}

size_t size_class(size_t bytes) {
  if (bytes <= 256) return 256;
  if (bytes <= (1u << 20)) {
    size_t c = 256;
    while (c < bytes) c <<= 1;
    return c;
  }
  int top = 63 - __builtin_clzll(bytes);
  const size_t step = size_t(1) << (top - 3);
  return (bytes + step - 1) / step * step;
}

Arena* find(cudaStream_t s) {
  auto it = arenas().find(s);
  return it == arenas().end() ? nullptr : it->second;
}

}  // namespace

void arena_register(cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!find(s)) arenas()[s] = new Arena;
}

void arena_unregister(cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_mu);
  Arena* a = find(s);
  if (!a) return;
  cudaStreamSynchronize(s);
  for (auto& kv : a->free_lists)
    for (void* p : kv.second) cudaFree(p);
  arenas().erase(s);
  delete a;
}

namespace {
void* guarded(Arena* a, cudaStream_t s, void* p, size_t bytes) {
  if (a && guard_bytes()) {
    a->asked[p] = bytes;
    cuda_check(cudaMemsetAsync(p, kPoison, bytes + guard_bytes(), s), "TWG_GUARD poison", __FILE__, __LINE__);
  }
  return p;
}
}  // namespace

void* arena_alloc(cudaStream_t s, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  Arena* a = find(s);
  const size_t c = size_class(bytes + guard_bytes());
  if (a) {
    // smallest cached block of class in [c, 2c): batch-to-batch size jitter
    // (a few more nodes or groups) must not trigger a fresh cudaMalloc,
    // which synchronises the device
    for (auto it = a->free_lists.lower_bound(c); it != a->free_lists.end() && it->first < 2 * c; ++it) {
      if (!it->second.empty()) {
        void* p = it->second.back();
        it->second.pop_back();
        a->in_use += it->first;
        a->owned[p] = it->first;
        return guarded(a, s, p, bytes);
      }
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, c);
  if (e == cudaErrorMemoryAllocation && a) {
    cudaGetLastError();
    cudaStreamSynchronize(s);
    for (auto& kv : a->free_lists) {
      for (void* q : kv.second) {
        cudaFree(q);
        a->reserved -= kv.first;
      }
      kv.second.clear();
    }
    e = cudaMalloc(&p, c);
  }
  cuda_check(e, "cudaMalloc (arena)", __FILE__, __LINE__);
  if (a) {
    a->in_use += c;
    a->reserved += c;
    a->owned[p] = c;
  }
  return guarded(a, s, p, bytes);
}

void arena_free(cudaStream_t s, void* p, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  Arena* a = find(s);
  if (!a) {  // ctx already gone: release for real
    cudaFree(p);
    return;
  }
  if (auto g = guard_bytes() ? a->asked.find(p) : a->asked.end(); g != a->asked.end()) {  // TWG_GUARD: tail intact?
    std::vector<unsigned char> tail(guard_bytes());
    cudaMemcpyAsync(tail.data(), static_cast<char*>(p) + g->second, tail.size(), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    for (size_t i = 0; i < tail.size(); ++i) {
      if (tail[i] != kPoison) {
        std::fprintf(stderr, "TWG_GUARD: write past the end of a %zu-byte block (byte +%zu of its guard)\n",
                     g->second, i);
        break;
      }
    }
    a->asked.erase(g);
  }
  auto it = a->owned.find(p);
  const size_t c = it != a->owned.end() ? it->second : size_class(bytes);
  if (it != a->owned.end()) a->owned.erase(it);
  a->free_lists[c].push_back(p);
  a->in_use -= c;
}

size_t arena_bytes_in_use(cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_mu);
  Arena* a = find(s);
  return a ? a->in_use : 0;
}

size_t arena_bytes_reserved(cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_mu);
  Arena* a = find(s);
  return a ? a->reserved : 0;
}

}  // namespace twg
