// The reference's synthetic graph generators (synthetic.cpp:24-140) on the
// device, bit-identical: every random endpoint / time is the reference's
// CounterRng draw for (stream, edge, ordinal) (rng.hpp:22-43), so each edge
// is generated independently by one thread. The planted (RNG-free) funnel
// and ladder structures of the hub-skewed and mega-hub graphs are a few
// thousand edges laid out by the host in the reference's order; the random
// backgrounds follow them.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace twg {

namespace {

__device__ __forceinline__ u64 mix64d(u64 x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__device__ __forceinline__ u64 bits(u64 key, u64 stream, u64 i, u64 ord) {
  return mix64d(mix64d(mix64d(key ^ stream) ^ i) ^ ord);
}

// kind 1: hub-skewed background (synthetic.cpp:92-97); kind 2: mega-hub
// background (:117-121, ids offset by `base`); kind 3: time ladder (:130-137)
__global__ void k_synth_graph(int kind, u64 key, u64 n, u64 a, u64 base, u32 rungs, twg_edge* out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    twg_edge e;
    if (kind == 0) {  // make_uniform_graph (:24-36); base = t_max + 1
      e.src = static_cast<i64>(bits(key, 1, i, 0) % a);
      e.dst = static_cast<i64>(bits(key, 2, i, 0) % a);
      e.t = static_cast<i64>(bits(key, 3, i, 0) % base);
    } else if (kind == 1) {
      const double u = static_cast<double>(bits(key, 2, i, 1) >> 11) * 0x1.0p-53;
      const i64 dv = static_cast<i64>(__dmul_rn(__dmul_rn(__dmul_rn(static_cast<double>(a), u), u), u));
      e.src = static_cast<i64>(bits(key, 1, i, 0) % a);
      e.dst = dv < static_cast<i64>(a) - 1 ? dv : static_cast<i64>(a) - 1;
      e.t = static_cast<i64>(bits(key, 3, i, 0) % 20000u);
    } else if (kind == 2) {
      e.src = static_cast<i64>(base + bits(key, 1, i, 0) % 100u);
      e.dst = static_cast<i64>(base + bits(key, 2, i, 0) % 100u);
      e.t = static_cast<i64>(bits(key, 3, i, 0) % 5000u);
    } else {
      e.src = static_cast<i64>(i / rungs);
      e.dst = static_cast<i64>(bits(key, 2, i, 0) % a);
      e.t = static_cast<i64>(i % rungs);
    }
    out[i] = e;
  }
}

}  // namespace

// kind: 0 uniform (a = nodes, b = edges, t_max), 1 hub-skewed (a = background
// nodes, b = background edges), 2 mega hub (a = feeders), 3 time ladder (a =
// edge count, b = rungs). Host prefix of planted edges + device background.
u64 synth_graph_size(int kind, u64 a, u64 b) {
  if (kind == 0) return b;
  if (kind == 1) return 2600 + 5000 + 40 + 4500 + 40 + 150 + 3 + 700 + 3 + 60 + 40 + b;
  if (kind == 2) return a + 64 + 1000;
  return std::max<u64>(2, a / b) * b;
}

void synth_graph(Ctx& ctx, int kind, u64 a, u64 b, i64 t_max, u64 key, twg_edge* out) {
  cudaStream_t st = ctx.stream;
  std::vector<twg_edge> pre;
  u64 n_bg = 0, base = 0, node_arg = 0;
  u32 rungs = 0;
  if (kind == 1) {
    i64 next = static_cast<i64>(a);
    auto funnel = [&](u64 width, i64 t0) {  // width single-out-degree feeders into a fresh hub
      const i64 hub = next++;
      for (u64 i = 0; i < width; ++i) pre.push_back(twg_edge{next++, hub, t0 + static_cast<i64>(i)});
      return hub;
    };
    auto ladder = [&](i64 hub, u64 groups, i64 t0, u64 sinks) {  // hub -> sinks at `groups` times
      const i64 s0 = next;
      next += static_cast<i64>(sinks);
      for (u64 g = 0; g < groups; ++g) pre.push_back(twg_edge{hub, s0 + static_cast<i64>(g % sinks), t0 + static_cast<i64>(g)});
    };
    const i64 mega = funnel(2600, 1000);
    ladder(mega, 5000, 10000, 200);
    const i64 bd = funnel(40, 1000);
    ladder(bd, 4500, 10000, 50);
    const i64 bc = funnel(40, 1000);
    ladder(bc, 150, 10000, 50);
    const i64 wd = funnel(3, 1000);
    ladder(wd, 700, 10000, 20);
    const i64 wc = funnel(3, 1000);
    ladder(wc, 60, 10000, 20);
    ladder(next++, 40, 500, 40);  // spreader
    n_bg = b;
    node_arg = a;
  } else if (kind == 2) {
    const u64 feeders = a;
    i64 next = 1;
    for (u64 i = 0; i < feeders; ++i) pre.push_back(twg_edge{next++, 0, 100 + static_cast<i64>(i)});
    const i64 s0 = next;
    next += 16;
    const i64 t0 = 100 + static_cast<i64>(feeders) + 100;
    for (u64 g = 0; g < 64; ++g) pre.push_back(twg_edge{0, s0 + static_cast<i64>(g % 16), t0 + static_cast<i64>(g)});
    base = static_cast<u64>(next);
    n_bg = 1000;
  } else if (kind == 3) {
    rungs = static_cast<u32>(b);
    node_arg = std::max<u64>(2, a / b);
    n_bg = node_arg * rungs;
  } else {
    node_arg = a;
    base = static_cast<u64>(t_max) + 1;
    n_bg = b;
  }
  std::copy(pre.begin(), pre.end(), out);
  if (n_bg) {
    DevBuf<twg_edge> d(n_bg, st);
    k_synth_graph<<<grid_for(n_bg, 256, static_cast<unsigned>(ctx.sm_count) * 16), 256, 0, st>>>(
        kind, key, n_bg, node_arg, base, rungs, d.p);
    TWG_LAUNCHED(ctx);
    TWG_CUDA(cudaMemcpyAsync(out + pre.size(), d.p, n_bg * sizeof(twg_edge), cudaMemcpyDeviceToHost, st));
    TWG_CUDA(cudaStreamSynchronize(st));
  }
}

}  // namespace twg
