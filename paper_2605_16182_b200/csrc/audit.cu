// Walk validity audit on the device: the sm_100a equivalent of
// timewalk::check_walkset / check_timed_walk (validity.cpp:32-66, :108-120).
//
// Like the reference's EdgeOracle (validity.cpp:14-30) the audit is
// independent of the engine's node view: it sorts a copy of the snapshot's
// edge list by (source, target) — stably, so the times of one pair stay
// ascending — and answers "does edge a->b exist at time t" by two binary
// searches. Undirected stores accept either orientation (the oracle inserts
// both). Hop j of a walk is valid iff its edge exists at times[j+1] and the
// time strictly advances in the walk direction (non-strict when asked); a
// start sentinel (kTimeUnset / kTimeInfinite) at entry 0 imposes no order.
// Walks shorter than 2 entries are skipped, as the reference does.
#include "primitives.cuh"
#include "walk.cuh"

namespace twg {

namespace {

constexpr int kBlock = 256;

unsigned grid(Ctx& ctx, u64 n) { return grid_for(n, kBlock, static_cast<unsigned>(ctx.sm_count) * 16); }

__global__ void k_pair_keys(const u32* s, const u32* d, const i64* t, u64 m, u64* keys, i64* vals) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    keys[i] = (static_cast<u64>(s[i]) << 32) | d[i];
    vals[i] = t[i];
  }
}

__device__ __forceinline__ bool internal_id(const i64* ext, u64 V, bool identity, i64 x, u32* out) {
  if (x < 0) return false;
  if (identity) {
    if (static_cast<u64>(x) >= V) return false;
    *out = static_cast<u32>(x);
    return true;
  }
  u64 lo = 0, hi = V;
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if (ext[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  if (lo == V || ext[lo] != x) return false;
  *out = static_cast<u32>(lo);
  return true;
}

// EdgeOracle::contains (validity.cpp:27-30) over the (pair, time)-sorted copy
__device__ __forceinline__ bool contains(const u64* keys, const i64* times, u64 m, u32 a, u32 b, i64 t) {
  const u64 key = (static_cast<u64>(a) << 32) | b;
  u64 lo = 0, hi = m;  // the pair's run [lo, end)
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if (keys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  u64 x = lo, end = m;
  while (x < end) {
    const u64 mid = (x + end) >> 1;
    if (keys[mid] <= key) x = mid + 1;
    else end = mid;
  }
  u64 y = lo;  // lower_bound(t) in the run's ascending times (std::binary_search)
  x = end;
  while (y < x) {
    const u64 mid = (y + x) >> 1;
    if (times[mid] < t) y = mid + 1;
    else x = mid;
  }
  return y < end && times[y] == t;
}

struct AuditArgs {
  const u64* off;  // compact walk image
  const i64* nodes;
  const i64* times;
  u64 count;
  const i64* ext;
  u64 V;
  bool ext_identity;
  const u64* keys;
  const i64* ktimes;
  u64 m;
  int forward;
  int strict;
  int undirected;
  i64* first_violation;  // per walk, -1 when valid (or skipped)
  u64* report;           // [0] walks, [1] valid walks, [2] hops, [3] valid hops
};

__global__ void k_audit(AuditArgs a) {
  u64 walks = 0, vwalks = 0, hops = 0, vhops = 0;
  for (u64 w = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; w < a.count;
       w += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 b = a.off[w], len = a.off[w + 1] - b;
    i64 first = -1;
    if (len >= 2) {
      ++walks;
      u64 valid = 0;
      for (u64 j = 0; j + 1 < len; ++j) {
        const i64 u = a.nodes[b + j], v = a.nodes[b + j + 1];
        const i64 tp = a.times[b + j], th = a.times[b + j + 1];
        u32 iu, iv;
        bool edge_ok = false;
        if (internal_id(a.ext, a.V, a.ext_identity, u, &iu) && internal_id(a.ext, a.V, a.ext_identity, v, &iv)) {
          // a backward walk traverses the stored edge target -> source (validity.cpp:46-48)
          const u32 s = a.forward ? iu : iv, d = a.forward ? iv : iu;
          edge_ok = contains(a.keys, a.ktimes, a.m, s, d, th) ||
                    (a.undirected && contains(a.keys, a.ktimes, a.m, d, s, th));
        }
        bool time_ok;
        if (j == 0 && (tp == kTimeUnset || tp == kTimeInfinite)) time_ok = true;
        else if (a.forward) time_ok = a.strict ? th > tp : th >= tp;
        else time_ok = a.strict ? th < tp : th <= tp;
        if (edge_ok && time_ok) ++valid;
        else if (first < 0) first = static_cast<i64>(j);
      }
      hops += len - 1;
      vhops += valid;
      if (valid == len - 1) ++vwalks;
    }
    if (a.first_violation) a.first_violation[w] = first;
  }
  for (int o = 16; o > 0; o >>= 1) {
    walks += __shfl_xor_sync(0xffffffffu, walks, o);
    vwalks += __shfl_xor_sync(0xffffffffu, vwalks, o);
    hops += __shfl_xor_sync(0xffffffffu, hops, o);
    vhops += __shfl_xor_sync(0xffffffffu, vhops, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (walks) atomicAdd(reinterpret_cast<unsigned long long*>(&a.report[0]), walks);
    if (vwalks) atomicAdd(reinterpret_cast<unsigned long long*>(&a.report[1]), vwalks);
    if (hops) atomicAdd(reinterpret_cast<unsigned long long*>(&a.report[2]), hops);
    if (vhops) atomicAdd(reinterpret_cast<unsigned long long*>(&a.report[3]), vhops);
  }
}

}  // namespace

void audit_walks(Ctx& ctx, const WalkSetDev& w, const Store& g, int direction, bool strict, i64* d_first,
                 u64 report[4]) {
  cudaStream_t st = ctx.stream;
  const Store& s = ensure_compact(ctx, g);  // SoA edge columns with internal ids
  const u64 m = s.m;
  DevBuf<u64> k0(m ? m : 1, st), k1(m ? m : 1, st);
  DevBuf<i64> v0(m ? m : 1, st), v1(m ? m : 1, st);
  u64* kp = k0.p;
  u64* ka = k1.p;
  i64* vp = v0.p;
  i64* va = v1.p;
  if (m) {
    k_pair_keys<<<grid(ctx, m), kBlock, 0, st>>>(s.e_src.p, s.e_dst.p, s.e_t.p, m, kp, vp);
    TWG_LAUNCHED(ctx);
    const int vb = s.V > 1 ? bit_width_u64(s.V - 1) : 1;
    // low key word = target: bits [0, vb); high word = source: bits [32, 32 + vb)
    radix_sort_pairs<u64, i64>(ctx, &kp, &ka, &vp, &va, m, vb);
    radix_sort_pairs<u64, i64>(ctx, &kp, &ka, &vp, &va, m, 32 + vb, 32);
  }
  DevBuf<u64> off;
  DevBuf<i64> nodes, times;
  u64 total = 0;
  compact_walks(ctx, w, off, nodes, times, &total);
  DevBuf<u64> rep(4, st);
  TWG_CUDA(cudaMemsetAsync(rep.p, 0, rep.bytes(), st));
  AuditArgs a{off.p, nodes.p, times.p, w.count, s.ext.p, s.V, s.ext_identity, kp, vp, m, direction == 0 ? 1 : 0,
              strict ? 1 : 0, s.mode == TWG_UNDIRECTED ? 1 : 0, d_first, rep.p};
  if (w.count) {
    k_audit<<<grid(ctx, w.count), kBlock, 0, st>>>(a);
    TWG_LAUNCHED(ctx);
  }
  read_scalars(ctx, rep.p, report, 4);
}

}  // namespace twg
