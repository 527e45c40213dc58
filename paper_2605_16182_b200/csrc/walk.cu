// Walk generation on sm_100a (walk_engine.cpp:147-434).
//
// Variants (walk_engine.hpp:31-34), byte-identical outputs (the reference's
// scheduler-neutrality invariant, test_walk_engine.cpp:294-316):
//  * FullWalk  — k_fullwalk: one thread per walk, init fused, walk to
//                completion in registers (walk_engine.cpp:380-392).
//  * Coop      — the hierarchical cooperative scheduler (Alg. 1,
//                walk_engine.cpp:301-345): per step, compact alive walks
//                (flag+scan), stable radix sort by current node, run-length
//                encode, classify runs on the (W, G) dispatch plane, split
//                mega-hub runs into ceil(W/w_max) sub-tasks, and launch the
//                five terminal tiers: solo (thread per task), warp (warp per
//                task) and block (CTA per (sub-)task), the cached flavours
//                staging the node's timestamp-group marks in shared memory.
//  * CoopDirect — Coop with staging disabled (direct global reads).
//
// Per-hop semantics are hop_walk (walk_engine.cpp:88-145): causal slice by
// binary search over the node's marks, draw keyed (walk, length, ordinal),
// closed-form / weighted pick, node2vec rejection with <=64 retries.
#include <chrono>
#include <cstring>

#include "primitives.cuh"
#include "rng.cuh"
#include "samplers.cuh"
#include "walk.cuh"

namespace twg {

namespace {

constexpr int kBlock = 256;
constexpr u32 kNode2VecMaxRetries = 64;  // samplers.hpp:89

struct WalkParams {
  StoreView s;
  Rng rng;
  int bias;
  int dir;  // 0 forward, 1 backward
  int node2vec;
  int temporal_adj;
  double inv_p, inv_q, bmax;
  u32 stride;
  u64 walk_begin;
  u64 count;        // walks in this output
  int slot_major;   // device WalkSet layout: [slot][walk] (coalesced hop writes) vs [walk][slot]
  i64* nodes;
  i64* times;
  const double* exp_neg;
  const double* expm1_tab;
  int rec;      // hop through the store's walk records (hop_rec)
};

// Output cell of (local walk, slot). The device-resident WalkSet is
// slot-major: the 32 lanes of a warp writing slot j of 32 consecutive walks
// hit 256 contiguous bytes instead of 32 rows 640 bytes apart. The
// reference's walk-major image is produced at download.
__device__ __forceinline__ u64 out_index(const WalkParams& P, u64 wl, u32 slot) {
  return P.slot_major ? static_cast<u64>(slot) * P.count + wl : wl * P.stride + slot;
}

// internal -> external id; skipped when the id map is the identity (the
// snapshot holds exactly the ids 0..V-1, e.g. the C5 stream's population)
__device__ __forceinline__ i64 ext_of(const StoreView& s, u32 v) {
  return s.ext_identity ? static_cast<i64>(v) : s.ext[v];
}

// ---- per-hop pieces -------------------------------------------------------

// one 128-bit load per entry (the compiler otherwise splits the fields)
__device__ __forceinline__ Entry load_entry(const Entry* p) {
  const int4 v = __ldg(reinterpret_cast<const int4*>(p));
  Entry e;
  e.nbr = static_cast<u32>(v.x);
  e.edge = static_cast<u32>(v.y);
  e.t = static_cast<i64>((static_cast<u64>(static_cast<u32>(v.w)) << 32) | static_cast<u32>(v.z));
  return e;
}

// first logical g in [lo, hi) with x < a[ring(g)] / with a[ring(g)] >= x.
// Binary search down to a window of kScan marks, then the window's times in
// one round of independent loads (the window spans 2-3 sectors): a typical
// node (G ~ 33) costs 3 dependent round trips instead of 6.
constexpr u32 kScan = 4;
__device__ __forceinline__ u32 ub_ring(const i64* a, Ring r, u32 lo, u32 hi, i64 x) {
  if (hi - lo > kScan) {
    // forward walks move to ever later times: the answer is usually among
    // the run's last keys (or past them: the walk ends), so those go first
    // (the 32-B sector holding the last key: up to kScan keys, one sector)
    const u32 last = hi - 1;
    const u32 d0 = last - r.org, d = d0 >= r.cap ? d0 - r.cap : d0;
    const u32 k = min((r.base + d) & (kScan - 1), d);  // keys of the sector before `last` (no ring wrap)
    const i64* g = a + (r.base + d - k);
    u32 n = 0;
#pragma unroll
    for (u32 i = 0; i < kScan; ++i)
      if (i <= k) n += g[i] <= x ? 1u : 0u;
    if (n) return last - k + n;
    hi = last - k;
  }
  while (hi - lo > kScan) {
    const u32 mid = lo + ((hi - lo) >> 1);
    if (x < a[r(mid)]) hi = mid;
    else lo = mid + 1;
  }
  u32 n = 0;
#pragma unroll
  for (u32 i = 0; i < kScan; ++i)
    if (lo + i < hi) n += a[r(lo + i)] <= x ? 1u : 0u;  // sorted: the elements <= x form a prefix
  return lo + n;
}
__device__ __forceinline__ u32 lb_ring(const i64* a, Ring r, u32 lo, u32 hi, i64 x) {
  if (hi - lo > kScan) {  // mirror of ub_ring: backward walks move to ever earlier times
    u32 n = 0;
#pragma unroll
    for (u32 i = 0; i < kScan; ++i) n += a[r(lo + i)] < x ? 1u : 0u;
    if (n < kScan) return lo + n;
    lo += kScan;
  }
  while (hi - lo > kScan) {
    const u32 mid = lo + ((hi - lo) >> 1);
    if (a[r(mid)] < x) lo = mid + 1;
    else hi = mid;
  }
  u32 n = 0;
#pragma unroll
  for (u32 i = 0; i < kScan; ++i)
    if (lo + i < hi) n += a[r(lo + i)] < x ? 1u : 0u;
  return lo + n;
}

// walk_engine.cpp:18-34 over marks mt/ms (logical [glo, ghi) through ring mr)
// of a region [lo, hi); c/e are logical entry positions
__device__ __forceinline__ void causal_slice(const i64* mt, const u32* ms, Ring mr, u32 glo, u32 ghi, u32 lo, u32 hi,
                                             i64 t, int dir, u32& c, u32& e) {
  if (dir == 0) {
    const u32 g = ub_ring(mt, mr, glo, ghi, t);
    c = g == ghi ? hi : ms[mr(g)];
    e = hi;
  } else {
    const u32 g = lb_ring(mt, mr, glo, ghi, t);
    c = lo;
    e = g == ghi ? hi : ms[mr(g)];
  }
}

// Forward causal slice on the entries by interpolation search: the first
// entry of [lo, hi) later than t. The run's times are taken as spread over
// the snapshot's span (tl, th); each probe reads the aligned 64-B atom around
// the interpolated position and narrows [a, b) with every in-run key of it,
// keeping the times just outside the range as the next estimate's anchors;
// after 2 estimates it bisects. A first hop from a sampled start (t
// anywhere in the window) costs about two atoms instead of a bisection's
// five or six; later hops (t near the newest times) land on the run's end.
template <u32 kPer, bool kLower = false, class Key>
__device__ __forceinline__ u32 interp_ub(Key key, Ring er, u32 lo, u32 hi, i64 t, i64 tl, i64 th) {
  // kLower: lower_bound (first key >= t, backward walks) instead of upper_bound
  u32 a = lo, b = hi;
  i64 ta = tl, tb = th;  // times just before a / at b (anchors of the estimate)
  for (int round = 0; b - a > kScan; ++round) {
    u32 x;
    if (round < 2 && tb > ta && t >= ta) {
      const double f = static_cast<double>(t - ta) / static_cast<double>(tb - ta);
      const double span = static_cast<double>(b - a);
      x = a + static_cast<u32>(f * span < span ? f * span : span - 1.0);
    } else {
      x = a + ((b - a) >> 1);
    }
    const u32 d0 = x - er.org, d = d0 >= er.cap ? d0 - er.cap : d0;
    const u32 k = (er.base + d) & (kPer - 1);  // x's place in its atom
#pragma unroll
    for (u32 j = 0; j < kPer; ++j) {
      const u32 pos = x - k + j;
      if (pos >= a && pos < b) {  // in-run keys only (memory-safe: the run is allocated)
        const i64 v = key(er(pos));
        if (kLower ? v < t : v <= t) {
          a = pos + 1;
          ta = v;
        } else {
          b = pos;
          tb = v;
        }
      }
    }
  }
  u32 n = 0;
#pragma unroll
  for (u32 i = 0; i < kScan; ++i)
    if (a + i < b) n += (kLower ? key(er(a + i)) < t : key(er(a + i)) <= t) ? 1u : 0u;
  return a + n;
}

// walk_engine.cpp:18-34 evaluated on the entries: forward c = first entry
// with time > t (upper_bound), backward e = first entry with time >= t
// (lower_bound) — the same positions the mark search yields.
__device__ __forceinline__ void causal_slice_entries(const Entry* ent, Ring er, u32 lo, u32 hi, i64 t, int dir,
                                                     u32& c, u32& e) {
  u32 a = lo, b = hi;
  if (dir == 0) {
    if (b - a > kScan) {  // the run's end first, as in ub_ring: the 64-B atom holding the last entry
      const u32 last = b - 1;
      const u32 d0 = last - er.org, d = d0 >= er.cap ? d0 - er.cap : d0;
      const u32 k = min((er.base + d) & 3u, d);  // entries of the atom before `last` (no ring wrap)
      const u32 s0 = last - k;
      const Entry* g = ent + (er.base + d - k);
      u32 n = 0;
#pragma unroll
      for (u32 i = 0; i < kScan; ++i)
        if (i <= k) n += g[i].t <= t ? 1u : 0u;
      if (n) {
        c = s0 + n;
        e = hi;
        return;
      }
      b = s0;
      const u32 ds = d - k;  // ring offset of s0
      if (b - a > kScan && ds >= 4u) {  // then the whole atom before it
        const Entry* h = ent + (er.base + ds - 4u);
        u32 m = 0;
#pragma unroll
        for (u32 i = 0; i < 4u; ++i) m += h[i].t <= t ? 1u : 0u;
        if (m) {
          c = s0 - 4u + m;
          e = hi;
          return;
        }
        b = s0 - 4u;
      }
    }
    while (b - a > kScan) {
      const u32 mid = a + ((b - a) >> 1);
      if (t < ent[er(mid)].t) b = mid;
      else a = mid + 1;
    }
    u32 n = 0;
#pragma unroll
    for (u32 i = 0; i < kScan; ++i)
      if (a + i < b) n += ent[er(a + i)].t <= t ? 1u : 0u;
    c = a + n;
    e = hi;
  } else {
    if (b - a > kScan) {
      u32 n = 0;
#pragma unroll
      for (u32 i = 0; i < kScan; ++i) n += ent[er(a + i)].t < t ? 1u : 0u;
      if (n < kScan) {
        c = lo;
        e = a + n;
        return;
      }
      a += kScan;
    }
    while (b - a > kScan) {
      const u32 mid = a + ((b - a) >> 1);
      if (ent[er(mid)].t < t) a = mid + 1;
      else b = mid;
    }
    u32 n = 0;
#pragma unroll
    for (u32 i = 0; i < kScan; ++i)
      if (a + i < b) n += ent[er(a + i)].t < t ? 1u : 0u;
    c = lo;
    e = a + n;
  }
}

// walk_engine.cpp:49-63 (contiguous stores: the weighted views exist only there)
__device__ u64 draw_weighted_local(const WalkParams& P, double u, u32 c, u32 e) {
  const i64 anchor = P.s.ent[e - 1].t;
  double total = 0.0;
  for (u32 pos = c; pos < e; ++pos) total = __dadd_rn(total, exp_nonpos(P.s.ent[pos].t - anchor, P.exp_neg));
  const double r = __dmul_rn(u, total);
  double cum = 0.0;
  for (u32 pos = c; pos < e; ++pos) {
    cum = __dadd_rn(cum, exp_nonpos(P.s.ent[pos].t - anchor, P.exp_neg));
    if (r < cum) return pos - c;
  }
  return e - 1 - c;
}

// walk_engine.cpp:49-63 through the node's ring (streaming stores)
__device__ u64 draw_weighted_local_ring(const WalkParams& P, double u, Ring er, u32 c, u32 e) {
  const i64 anchor = load_entry(P.s.ent + er(e - 1)).t;
  double total = 0.0;
  for (u32 x = c; x < e; ++x) total = __dadd_rn(total, exp_nonpos(P.s.ent[er(x)].t - anchor, P.exp_neg));
  const double r = __dmul_rn(u, total);
  double cum = 0.0;
  for (u32 x = c; x < e; ++x) {
    cum = __dadd_rn(cum, exp_nonpos(P.s.ent[er(x)].t - anchor, P.exp_neg));
    if (r < cum) return x - c;
  }
  return e - 1 - c;
}

// ExponentialWeight draw on a streaming store, without a materialised
// node_weight_prefix_: the prefix of region [lo, hi) is anchored at its
// newest time (edge_store.cpp:159, :208-209), so every value before the first
// entry within 745 time units of the anchor is exactly +0 and the rest is a
// serial sum over that tail — evaluated here in the reference's order, then
// the reference's base / mass / lower_bound logic (walk_engine.cpp:73-80,
// samplers.cpp:82-90). Bit-identical to the contiguous path.
__device__ u64 draw_weighted_ring(const WalkParams& P, double u, Ring er, u32 lo, u32 hi, u32 c, u32 e) {
  const i64 anchor = load_entry(P.s.ent + er(hi - 1)).t;
  const i64 floor_t = anchor - (kExpTableSize - 1);
  u32 ts = hi;  // tail [ts, hi)
  while (ts > lo && P.s.ent[er(ts - 1)].t >= floor_t) --ts;
  double acc = 0.0, base = 0.0;
  for (u32 x = ts; x < e; ++x) {
    acc = __dadd_rn(acc, exp_nonpos(P.s.ent[er(x)].t - anchor, P.exp_neg));
    if (x + 1 == c) base = acc;
  }
  const double total = e > ts ? acc : 0.0;
  const double mass = __dsub_rn(total, base);
  if (!(mass > 0.0) || !isfinite(mass)) return draw_weighted_local_ring(P, u, er, c, e);
  const double r = __dadd_rn(base, __dmul_rn(u, mass));
  if (c < ts && 0.0 >= r) return 0;  // prefix[c] == +0 already reaches r
  acc = 0.0;
  for (u32 x = ts; x < e; ++x) {
    acc = __dadd_rn(acc, exp_nonpos(P.s.ent[er(x)].t - anchor, P.exp_neg));
    if (x >= c && acc >= r) return x - c;
  }
  return e - 1 - c;
}

// walk_engine.cpp:65-84
__device__ __forceinline__ u64 draw_index(const WalkParams& P, double u, u32 lo, u32 c, u32 e, u32* amb, Ring er,
                                          u32 hi) {
  const u64 n = e - c;
  switch (P.bias) {
    case TWG_UNIFORM: return pick_uniform(u, n);
    case TWG_LINEAR: return pick_linear(u, n);
    case TWG_EXPINDEX: return pick_exponential(u, n, P.expm1_tab, amb);
    default: {
      if (!P.s.wp) return draw_weighted_ring(P, u, er, lo, hi, c, e);  // streaming store
      const double base = c > lo ? P.s.wp[c - 1] : 0.0;
      const double mass = __dsub_rn(P.s.wp[e - 1], base);
      if (!(mass > 0.0) || !isfinite(mass)) return draw_weighted_local(P, u, c, e);
      return pick_weighted_range(u, P.s.wp, c, e, base);
    }
  }
}

// edge_store.cpp:310-314
__device__ __forceinline__ bool adjacent(const StoreView& s, u32 a, u32 b) {
  if (!s.adj_off) {  // streaming store: b among the neighbours of a's live region (any time)
    const NodeMeta na = s.nm[a];
    const Ring er = entry_ring(na);
    for (u32 x = na.eb; x < na.ee; ++x)
      if (s.ent[er(x)].nbr == b) return true;
    return false;
  }
  u32 lo = s.adj_off[a], hi = s.adj_off[a + 1];
  const u32 end = hi;
  while (lo < hi) {
    const u32 mid = lo + ((hi - lo) >> 1);
    if (s.adj[mid] < b) lo = mid + 1;
    else hi = mid;
  }
  return lo < end && s.adj[lo] == b;
}

// edge_store.cpp:316-323
__device__ bool adjacent_after(const StoreView& s, u32 a, u32 b, i64 t, int dir) {
  const NodeMeta na = s.nm[a];
  const Ring er = entry_ring(na);
  u32 c, e;
  if (implicit_marks(na)) causal_slice_entries(s.ent, er, na.eb, na.ee, t, dir, c, e);
  else causal_slice(s.mk_time, s.mk_start, mark_ring(na), na.gb, na.ge, na.eb, na.ee, t, dir, c, e);
  for (u32 pos = c; pos < e; ++pos)
    if (s.ent[er(pos)].nbr == b) return true;
  return false;
}

// Per-thread instrumentation: ambiguous exp-index draws, and the algorithmic
// bytes of SURVEY §8(d) (B_hop = 80 + 8*ceil(log2(G_v+1)) for the index
// pickers, +16 + 8*ceil(log2 n) for the weighted picker; 24 B per sampled
// start) summed exactly per hop for the roofline.
struct Ctr {
  u32 amb;
  u64 bytes;
};

__device__ __forceinline__ u32 ceil_log2p1(u32 g) { return g ? 32u - __clz(g) : 0u; }  // ceil(log2(g+1))

struct WalkReg {
  u32 cur;
  u32 prev;
  i64 t;
  u32 len;
  u32 has_prev;
};

// One hop (walk_engine.cpp:88-145). mt/ms: the marks to search (logical
// [glo, ghi) through ring mr), either the global arrays or a shared-memory
// copy; entries [lo, hi) through ring er. Returns false when the causal
// slice is empty (walk dies).
__device__ __forceinline__ bool hop(const WalkParams& P, u64 wl, WalkReg& r, const i64* mt, const u32* ms, Ring mr,
                                    u32 glo, u32 ghi, Ring er, u32 lo, u32 hi, Ctr* cn, i64 tl = 0, i64 th = -1) {
  u32* amb = &cn->amb;
  u32 c, e;
  if (mt == P.s.mk_time && 2 * (ghi - glo) > hi - lo) {
    // mostly distinct times: search the entries themselves — the first entry
    // later than t IS the first entry of the first later group, so the mark
    // start lookup disappears (one fewer random sector per hop)
    // interpolate when the answer is far from where the walk direction
    // usually finds it (forward: the run's end, backward: its start)
    bool interp = false;
    if (th > tl && r.t >= tl && r.t <= th && hi - lo > 16u) {
      const double f = static_cast<double>(r.t - tl) / static_cast<double>(th - tl);
      const double n = static_cast<double>(hi - lo);
      interp = P.dir == 0 ? f * n + 12.0 < n : f * n > 12.0;
    }
    if (interp) {
      const Entry* ent = P.s.ent;
      const auto key = [ent](u32 p) { return ent[p].t; };
      if (P.dir == 0) {
        c = interp_ub<4>(key, er, lo, hi, r.t, tl, th);
        e = hi;
      } else {
        c = lo;
        e = interp_ub<4, true>(key, er, lo, hi, r.t, tl, th);
      }
    } else {
      causal_slice_entries(P.s.ent, er, lo, hi, r.t, P.dir, c, e);
    }
  } else {
    bool interp = false;  // the same choice over the marks (8 per atom)
    if (th > tl && r.t >= tl && r.t <= th && ghi - glo > 16u) {
      const double f = static_cast<double>(r.t - tl) / static_cast<double>(th - tl);
      const double n = static_cast<double>(ghi - glo);
      interp = P.dir == 0 ? f * n + 12.0 < n : f * n > 12.0;
    }
    if (interp) {
      const auto key = [mt](u32 p) { return mt[p]; };
      if (P.dir == 0) {
        const u32 g = interp_ub<8>(key, mr, glo, ghi, r.t, tl, th);
        c = g == ghi ? hi : ms[mr(g)];
        e = hi;
      } else {
        const u32 g = interp_ub<8, true>(key, mr, glo, ghi, r.t, tl, th);
        c = lo;
        e = g == ghi ? hi : ms[mr(g)];
      }
    } else {
      causal_slice(mt, ms, mr, glo, ghi, lo, hi, r.t, P.dir, c, e);
    }
  }
  if (c == e) return false;
  cn->bytes += 80u + 8u * ceil_log2p1(ghi - glo) +
               (P.bias == TWG_EXPWEIGHT ? 16u + 8u * ceil_log2p1(e - c - 1) : 0u);
  const u64 w = P.walk_begin + wl;
  const u64 hop_index = r.len;
  u64 idx;
  if (P.node2vec && r.has_prev) {
    idx = 0;
    for (u32 k = 0; k < kNode2VecMaxRetries; ++k) {
      const double u = P.rng.uniform(w, hop_index, 2ull * k);
      idx = draw_index(P, u, lo, c, e, amb, er, hi);
      const u32 cand = load_entry(P.s.ent + er(c + static_cast<u32>(idx))).nbr;
      const double ua = P.rng.uniform(w, hop_index, 2ull * k + 1);
      double beta;  // samplers.hpp:74-86
      if (cand == r.prev) beta = P.inv_p;
      else if (P.temporal_adj ? adjacent_after(P.s, r.prev, cand, r.t, P.dir) : adjacent(P.s, r.prev, cand))
        beta = 1.0;
      else beta = P.inv_q;
      if (ua < __ddiv_rn(beta, P.bmax)) break;
    }
  } else {
    const double u = P.rng.uniform(w, hop_index, 0);
    idx = draw_index(P, u, lo, c, e, amb, er, hi);
  }
  const Entry x = load_entry(P.s.ent + er(c + static_cast<u32>(idx)));
  const u64 slot = out_index(P, wl, r.len);
  P.nodes[slot] = ext_of(P.s, x.nbr);
  P.times[slot] = x.t;
  r.len += 1;
  if (P.node2vec) {
    r.prev = r.cur;
    r.has_prev = 1;
  }
  r.cur = x.nbr;
  r.t = x.t;
  return true;
}

// One forward hop through the node's walk record (walk_engine.cpp:88-145 for
// the index pickers): the causal slice starts inside the record's tail when t
// is at or after the tail's oldest time (or the tail is the whole region);
// otherwise the ring is searched over [eb, tail) — the entry at the tail's
// start is later than t, so the slice starts at or before it. The pick
// reads the ring only when it lands before the tail. Same c, e, draw and
// entry as hop(): byte-identical walks.
__device__ __forceinline__ WalkRec load_wrec(const WalkRec* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  const int4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2), d = __ldg(q + 3);
  WalkRec w;
  w.eb = static_cast<u32>(a.x);
  w.ee = static_cast<u32>(a.y);
  w.base = static_cast<u32>(a.z);
  w.cap = static_cast<u32>(a.w);
  w.eorg = static_cast<u32>(b.x);
  w.g = static_cast<u32>(b.y);
  w.nbr[0] = static_cast<u32>(b.z);
  w.nbr[1] = static_cast<u32>(b.w);
  w.nbr[2] = static_cast<u32>(c.x);
  w.pad = static_cast<u32>(c.y);
  w.t[0] = static_cast<i64>((static_cast<u64>(static_cast<u32>(c.w)) << 32) | static_cast<u32>(c.z));
  w.t[1] = static_cast<i64>((static_cast<u64>(static_cast<u32>(d.y)) << 32) | static_cast<u32>(d.x));
  w.t[2] = static_cast<i64>((static_cast<u64>(static_cast<u32>(d.w)) << 32) | static_cast<u32>(d.z));
  return w;
}
static_assert(kWalkTail == 3, "load_wrec / tail selects assume three tail entries");
__device__ __forceinline__ i64 tail_time(const WalkRec& R, u32 i) { return i == 0 ? R.t[0] : i == 1 ? R.t[1] : R.t[2]; }
__device__ __forceinline__ u32 tail_nbr(const WalkRec& R, u32 i) {
  return i == 0 ? R.nbr[0] : i == 1 ? R.nbr[1] : R.nbr[2];
}

__device__ __forceinline__ bool hop_rec(const WalkParams& P, u64 wl, WalkReg& r, const WalkRec& R, Ctr* cn, i64 tl) {
  const u32 lo = R.eb, hi = R.ee;
  if (lo == hi || r.t >= R.t[0]) return false;  // nothing later than t (R.t[0] is the newest time)
  const u32 k = min(hi - lo, kWalkTail), tail = hi - k;
  const Ring er{R.base, R.cap, R.eorg};
  u32 c;
  const i64 t_tail = tail_time(R, k - 1);  // time of entry `tail`
  if (tail == lo || r.t >= t_tail) {
    u32 n = 0;  // tail entries not later than t (the oldest of the tail)
#pragma unroll
    for (u32 i = 0; i < kWalkTail; ++i)
      if (i < k) n += R.t[i] <= r.t ? 1u : 0u;
    c = tail + n;
  } else {
    // interpolation between the snapshot's first time and the tail's oldest
    // (every slice position is a priori likely: 1.89 -> 1.78 ms per C5 launch
    // against probing the range's end first as hop() does; 8-entry probes
    // measured 1.95 ms)
    if (t_tail > tl && r.t >= tl && tail - lo > kScan) {
      const Entry* ent = P.s.ent;
      c = interp_ub<4>([ent](u32 q) { return ent[q].t; }, er, lo, tail, r.t, tl, t_tail);
    } else {
      u32 e_unused;
      causal_slice_entries(P.s.ent, er, lo, tail, r.t, 0, c, e_unused);
    }
  }
  cn->bytes += 80u + 8u * ceil_log2p1(R.g);
  const u64 w = P.walk_begin + wl;
  const double u = P.rng.uniform(w, r.len, 0);
  const u32 pos = c + static_cast<u32>(draw_index(P, u, lo, c, hi, &cn->amb, er, hi));
  u32 nbr;
  i64 nt;
  if (pos >= tail) {
    nbr = tail_nbr(R, hi - 1 - pos);
    nt = tail_time(R, hi - 1 - pos);
  } else {
    const Entry x = load_entry(P.s.ent + er(pos));
    nbr = x.nbr;
    nt = x.t;
  }
  const u64 slot = out_index(P, wl, r.len);
  P.nodes[slot] = ext_of(P.s, nbr);
  P.times[slot] = nt;
  r.len += 1;
  r.cur = nbr;
  r.t = nt;
  return true;
}

// walk_engine.cpp:284-299
__device__ __forceinline__ u64 sample_start_edge_dev(const StoreView& s, int bias, double u1, double u2,
                                                     const double* expm1_tab, u32* amb) {
  const u64 Z = s.Z;
  u64 g;
  switch (bias) {
    case TWG_UNIFORM: g = pick_uniform(u1, Z); break;
    case TWG_LINEAR: g = pick_linear(u1, Z); break;
    case TWG_EXPINDEX: g = pick_exponential(u1, Z, expm1_tab, amb); break;
    default:
      if (s.ts_w) {
        g = pick_weighted(u1, s.ts_w, Z);
      } else {  // streaming store: zeros then the materialised tail (samplers.cpp:74-80)
        const u64 nt = Z - s.ts_wt0;
        const double r = __dmul_rn(u1, s.ts_wtail[nt - 1]);
        if (s.ts_wt0 > 0 && 0.0 >= r) {
          g = 0;
        } else {
          u64 a = 0, b = nt;
          while (a < b) {
            const u64 mid = (a + b) >> 1;
            if (s.ts_wtail[mid] < r) a = mid + 1;
            else b = mid;
          }
          g = s.ts_wt0 + (a == nt ? nt - 1 : a);
        }
      }
      break;
  }
  u64 lo, hi;
  ts_group_range(s, g, lo, hi);
  u64 off = __double2ull_rz(__dmul_rn(u2, __ull2double_rn(hi - lo)));
  if (off >= hi - lo) off = hi - lo - 1;
  return lo + off;
}

struct InitParams {
  int start_mode;
  u32 walks_per_node;
  int start_bias;
  const u32* start_nodes;
  i64 sentinel;
};

// seed_walk + init_walks (walk_engine.cpp:147-155, :247-279)
__device__ __forceinline__ void init_walk(const WalkParams& P, const InitParams& I, u64 wl, WalkReg& r, Ctr* cn) {
  const u64 w = P.walk_begin + wl;
  const u64 base = out_index(P, wl, 0), base1 = out_index(P, wl, 1);
  r.prev = 0;
  r.has_prev = 0;
  if (I.start_mode == 0) {
    const u32 v = I.start_nodes[w / I.walks_per_node];
    P.nodes[base] = ext_of(P.s, v);
    P.times[base] = I.sentinel;
    r.cur = v;
    r.t = I.sentinel;
    r.len = 1;
  } else {
    const double u1 = P.rng.uniform(w, 0, 0);
    const double u2 = P.rng.uniform(w, 0, 1);
    const u64 eidx = sample_start_edge_dev(P.s, I.start_bias, u1, u2, P.expm1_tab, &cn->amb);
    cn->bytes += 24u + (I.start_bias == TWG_EXPWEIGHT ? 8u * (64u - __clzll(P.s.Z)) : 0u);
    const EdgeRec er = edge_at(P.s, eidx);  // one 128-bit load on streaming stores
    const u32 sv = er.src, dv = er.dst;
    const i64 t = er.t;
    const u32 from = P.dir == 0 ? sv : dv;
    const u32 to = P.dir == 0 ? dv : sv;
    P.nodes[base] = ext_of(P.s, from);
    P.times[base] = I.sentinel;
    P.nodes[base1] = ext_of(P.s, to);
    P.times[base1] = t;
    r.len = 2;
    r.cur = to;
    r.t = t;
    if (P.node2vec) {
      r.prev = from;
      r.has_prev = 1;
    }
  }
}

// stats[0] walks, [1] hops, [2] max hops (fullwalk steps), [3] ambiguous, [4] algorithmic bytes

// add_stats with one atomic per counter per BLOCK (every thread of the block
// calls it): per-warp atomics on the same five words serialise at L2 and
// cost ~0.5 ms per 10M walks
__device__ __forceinline__ void add_stats_block(u64* stats, u32 len, u32 init_len, const Ctr& cn, bool active) {
  __shared__ u64 part[kBlock / 32][5];
  u64 v[5] = {active && len >= 2 ? 1ull : 0ull, active && len >= 2 ? len - 1ull : 0ull,
              active ? static_cast<u64>(len - init_len) : 0ull, cn.amb, cn.bytes};
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const u64 x = __shfl_xor_sync(0xffffffffu, v[q], o);
      v[q] = q == 2 ? max(v[q], x) : v[q] + x;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 5; ++q) part[warp][q] = v[q];
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    const int q = threadIdx.x;
    u64 acc = 0;
    for (int w = 0; w < kBlock / 32; ++w) acc = q == 2 ? max(acc, part[w][q]) : acc + part[w][q];
    if (acc) {
      unsigned long long* dst = reinterpret_cast<unsigned long long*>(&stats[q]);
      if (q == 2) atomicMax(dst, acc);
      else atomicAdd(dst, acc);
    }
  }
}

__device__ __forceinline__ void add_counters_block(u64* stats, const Ctr& cn) {
  __shared__ u64 part2[kBlock / 32][2];
  u64 a = cn.amb, b = cn.bytes;
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    part2[threadIdx.x >> 5][0] = a;
    part2[threadIdx.x >> 5][1] = b;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    u64 acc = 0;
    for (int w = 0; w < kBlock / 32; ++w) acc += part2[w][threadIdx.x];
    if (acc) atomicAdd(reinterpret_cast<unsigned long long*>(&stats[3 + threadIdx.x]), acc);
  }
}

// ---- FullWalk -----------------------------------------------------------------

// Walk statistics of one warp into one of kStatSlots partial rows (spread
// over many L2 words: no hot spot when every warp finishes at once, and no
// block barrier, so a warp whose walks are done never waits for the block's
// longest walk); k_fold_stats folds the rows into stats[0..4].
constexpr u32 kStatSlots = 1024;
__device__ __forceinline__ void add_stats_warp(u64* part, u32 len, u32 init_len, const Ctr& cn, bool active) {
  u64 v[5] = {active && len >= 2 ? 1ull : 0ull, active && len >= 2 ? len - 1ull : 0ull,
              active ? static_cast<u64>(len - init_len) : 0ull, cn.amb, cn.bytes};
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const u64 x = __shfl_xor_sync(0xffffffffu, v[q], o);
      v[q] = q == 2 ? max(v[q], x) : v[q] + x;
    }
  }
  const u32 lane = threadIdx.x & 31;
  if (lane < 5) {
    u64 mine = v[0];
#pragma unroll
    for (int q = 1; q < 5; ++q)
      if (lane == static_cast<u32>(q)) mine = v[q];
    if (mine) {
      const u64 warp = (blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) >> 5;
      unsigned long long* dst = reinterpret_cast<unsigned long long*>(&part[(warp % kStatSlots) * 8 + lane]);
      if (lane == 2) atomicMax(dst, mine);
      else atomicAdd(dst, mine);
    }
  }
}

__global__ void k_fold_stats(const u64* part, u64* stats) {
  const u32 q = threadIdx.x >> 5, lane = threadIdx.x & 31;  // warp q folds column q
  if (q >= 5) return;
  u64 acc = 0;
  for (u32 r = lane; r < kStatSlots; r += 32) acc = q == 2 ? max(acc, part[r * 8 + q]) : acc + part[r * 8 + q];
  for (int o = 16; o > 0; o >>= 1) {
    const u64 x = __shfl_xor_sync(0xffffffffu, acc, o);
    acc = q == 2 ? max(acc, x) : acc + x;
  }
  if (lane == 0) stats[q] = q == 2 ? max(stats[q], acc) : stats[q] + acc;
}

// One thread per walk, init fused, the whole walk in registers
// (walk_engine.cpp:380-392). kWB-thread blocks (32 by default): a block
// retires — and its slots take new walks — as soon as its own walks end.
template <int kWB, bool kRec>
__global__ void __launch_bounds__(kWB, 1024 / kWB) k_fullwalk(WalkParams P, InitParams I, u64 count, u32* lengths,
                                                          u64* part) {
  const u64 wl = blockIdx.x * static_cast<u64>(kWB) + threadIdx.x;
  const bool active = wl < count;
  Ctr cn{0, 0};
  u32 init_len = 0;
  WalkReg r{};
  if (active) {
    init_walk(P, I, wl, r, &cn);
    init_len = r.len;
    // the snapshot's time span: anchors of the interpolation search
    const i64 tl = P.s.m ? edge_time(P.s, 0) - 1 : 0, th = P.s.m ? edge_time(P.s, P.s.m - 1) + 1 : -1;
    if (kRec) {  // forward index-biased walks over an append-route snapshot: walk records
      while (r.len < P.stride)
        if (!hop_rec(P, wl, r, load_wrec(P.s.wrec + r.cur), &cn, tl)) break;
    }
    while (!kRec && r.len < P.stride) {
      const NodeMeta a = P.s.nm[r.cur];
      if (!hop(P, wl, r, P.s.mk_time, P.s.mk_start, mark_ring(a), a.gb, a.ge, entry_ring(a), a.eb, a.ee, &cn, tl,
               th))
        break;
    }
    lengths[wl] = r.len;
  }
  add_stats_warp(part, r.len, init_len, cn, active);
}

// ---- Coop scheduler -------------------------------------------------------------

struct StateArrays {
  u32* cur;
  u32* prev;
  i64* t;
  u32* len;
  u8* flags;  // bit0 alive, bit1 has_prev
};

__global__ void __launch_bounds__(kBlock) k_init_states(WalkParams P, InitParams I, u64 count, StateArrays S,
                                                        u64* stats) {
  const u64 wl = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
  Ctr cn{0, 0};
  if (wl < count) {
    WalkReg r{};
    init_walk(P, I, wl, r, &cn);
    S.cur[wl] = r.cur;
    S.prev[wl] = r.prev;
    S.t[wl] = r.t;
    S.len[wl] = r.len;
    S.flags[wl] = static_cast<u8>((r.len < P.stride ? 1 : 0) | (r.has_prev ? 2 : 0));
  }
  add_counters_block(stats, cn);
}

// DispatchTask (walk_engine.hpp:87-94)
struct Task {
  u32 node;
  u32 begin;  // slice of the step's grouped walk ids
  u32 end;
  u32 sub;    // sub_task_index
};

struct TaskLists {
  Task* list[5];     // solo, warp_cached, warp_direct, block_cached, block_direct
  u32* subcount[5];  // sub_task_count per task
  // count[0..4] tasks per list; count[5] / count[6] split pieces in the
  // block-cached / block-direct lists (booked as multi_block, :157-161)
  u32* count;
};

// Classify runs on the dispatch plane (walk_engine.cpp:314-343).
__global__ void k_classify(const u32* keys, u64 n, StoreView s, twg_thresholds th, TaskLists T) {
  const u32 lane = threadIdx.x & 31;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  // warp-uniform loop: the list slots are allocated per warp and tier (one
  // atomic per tier present in the warp, not one per task)
  for (u64 i0 = blockIdx.x * static_cast<u64>(blockDim.x) + (threadIdx.x & ~31u); i0 < n; i0 += stride) {
    const u64 i = i0 + lane;
    const bool act = i < n && (i == 0 || keys[i] != keys[i - 1]);
    u32 v = 0, W = 0, pieces = 1;
    u64 end = i;
    int tier = -1;
    if (act) {
      // run [i, end): galloping search for the first j > i with keys[j] != keys[i]
      v = keys[i];
      u64 lo = i + 1, step = 1, hi = i + 1;
      while (hi < n && keys[hi] == v) {
        lo = hi + 1;
        hi = i + 1 + step;
        step <<= 1;
      }
      if (hi > n) hi = n;
      while (lo < hi) {  // first j in [lo, hi) with keys[j] != v
        const u64 mid = (lo + hi) >> 1;
        if (keys[mid] == v) lo = mid + 1;
        else hi = mid;
      }
      end = lo;
      W = static_cast<u32>(end - i);
      const NodeMeta nv = s.nm[v];
      const u32 G = nv.ge - nv.gb;
      if (W < th.w_warp) tier = 0;
      else if (W <= th.block_dim) tier = G <= th.g_warp_cap ? 1 : 2;
      else {
        tier = G <= th.g_block_cap ? 3 : 4;
        if (W > th.w_max) pieces = (W + th.w_max - 1) / th.w_max;
      }
    }
    u32 slot = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const bool mine = tier == k;
      const u32 m = __ballot_sync(0xffffffffu, mine);
      if (!m) continue;
      u32 incl = mine ? pieces : 0u;  // inclusive scan of the pieces over the lanes
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<u32>(o)) incl += x;
      }
      const u32 total = __shfl_sync(0xffffffffu, incl, 31);
      const int leader = __ffs(m) - 1;
      u32 base = 0;
      if (static_cast<int>(lane) == leader) base = atomicAdd(&T.count[k], total);
      base = __shfl_sync(0xffffffffu, base, leader);
      if (mine) slot = base + incl - pieces;
    }
    if (!act) continue;
    if (pieces > 1) atomicAdd(&T.count[tier == 3 ? 5 : 6], pieces);
    for (u32 p = 0; p < pieces; ++p) {
      Task task;
      task.node = v;
      task.begin = static_cast<u32>(i) + p * th.w_max;
      task.end = pieces > 1 ? min(static_cast<u32>(end), task.begin + th.w_max) : static_cast<u32>(end);
      task.sub = p;
      T.list[tier][slot + p] = task;
      T.subcount[tier][slot + p] = pieces;
    }
  }
}

__device__ __forceinline__ void load_state(const StateArrays& S, u32 w, WalkReg& r) {
  r.cur = S.cur[w];
  r.prev = S.prev[w];
  r.t = S.t[w];
  r.len = S.len[w];
  r.has_prev = (S.flags[w] >> 1) & 1u;
}

__device__ __forceinline__ void store_state(const StateArrays& S, u32 w, const WalkReg& r, bool alive, u32 stride) {
  S.cur[w] = r.cur;
  S.prev[w] = r.prev;
  S.t[w] = r.t;
  S.len[w] = r.len;
  S.flags[w] = static_cast<u8>(((alive && r.len < stride) ? 1 : 0) | (r.has_prev ? 2 : 0));
}

__device__ __forceinline__ void hop_member(const WalkParams& P, const StateArrays& S, u32 w, const i64* mt,
                                           const u32* ms, Ring mr, u32 glo, u32 ghi, Ring er, u32 lo, u32 hi,
                                           Ctr* amb) {
  WalkReg r;
  load_state(S, w, r);
  const bool alive = hop(P, w, r, mt, ms, mr, glo, ghi, er, lo, hi, amb);
  store_state(S, w, r, alive, P.stride);
}

// warp tiers: one warp per task; cached => the node's marks staged in this
// warp's shared-memory slice (G <= cap)
template <bool kCached>
__global__ void __launch_bounds__(kBlock) k_tier_warp(WalkParams P, StateArrays S, const u32* ids, const Task* tasks,
                                                      const u32* count, u32 cap, u64* stats) {
  extern __shared__ unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const u32 n = *count;
  i64* smt = reinterpret_cast<i64*>(smem_raw) + static_cast<u64>(warp) * cap;
  u32* sms = reinterpret_cast<u32*>(reinterpret_cast<i64*>(smem_raw) + static_cast<u64>(kBlock / 32) * cap) +
             static_cast<u64>(warp) * cap;
  Ctr amb{0, 0};
  for (u32 k = blockIdx.x * (kBlock / 32) + warp; k < n; k += gridDim.x * (kBlock / 32)) {
    const Task task = tasks[k];
    const NodeMeta a = P.s.nm[task.node];
    const Ring mr = mark_ring(a), er = entry_ring(a);
    const u32 G = a.ge - a.gb;
    if (kCached && G <= cap) {
      const bool imp = implicit_marks(a);
      for (u32 g = lane; g < G; g += 32) {
        smt[g] = imp ? P.s.ent[er(a.eb + g)].t : P.s.mk_time[mr(a.gb + g)];
        sms[g] = imp ? a.eb + g : P.s.mk_start[mr(a.gb + g)];
      }
      __syncwarp();
      const Ring staged{0u, kIdentityCap, a.gb};
      for (u32 i = task.begin + lane; i < task.end; i += 32)
        hop_member(P, S, ids[i], smt, sms, staged, a.gb, a.ge, er, a.eb, a.ee, &amb);
      __syncwarp();
    } else {
      for (u32 i = task.begin + lane; i < task.end; i += 32)
        hop_member(P, S, ids[i], P.s.mk_time, P.s.mk_start, mr, a.gb, a.ge, er, a.eb, a.ee, &amb);
    }
  }
  add_counters_block(stats, amb);
}

// block tiers: one CTA per (sub-)task; cached => marks staged in the CTA's
// shared memory (G <= cap). Mega-hub sub-tasks each reload the panel
// (PAPER.md:187).
template <bool kCached>
__global__ void __launch_bounds__(kBlock) k_tier_block(WalkParams P, StateArrays S, const u32* ids, const Task* tasks,
                                                       const u32* count, u32 cap, u64* stats) {
  extern __shared__ unsigned char smem_raw[];
  i64* smt = reinterpret_cast<i64*>(smem_raw);
  u32* sms = reinterpret_cast<u32*>(smt + cap);
  const u32 n = *count;
  Ctr amb{0, 0};
  for (u32 k = blockIdx.x; k < n; k += gridDim.x) {
    const Task task = tasks[k];
    const NodeMeta a = P.s.nm[task.node];
    const Ring mr = mark_ring(a), er = entry_ring(a);
    const u32 G = a.ge - a.gb;
    if (kCached && G <= cap) {
      __syncthreads();
      const bool imp = implicit_marks(a);
      for (u32 g = threadIdx.x; g < G; g += blockDim.x) {
        smt[g] = imp ? P.s.ent[er(a.eb + g)].t : P.s.mk_time[mr(a.gb + g)];
        sms[g] = imp ? a.eb + g : P.s.mk_start[mr(a.gb + g)];
      }
      __syncthreads();
      const Ring staged{0u, kIdentityCap, a.gb};
      for (u32 i = task.begin + threadIdx.x; i < task.end; i += blockDim.x)
        hop_member(P, S, ids[i], smt, sms, staged, a.gb, a.ge, er, a.eb, a.ee, &amb);
    } else {
      for (u32 i = task.begin + threadIdx.x; i < task.end; i += blockDim.x)
        hop_member(P, S, ids[i], P.s.mk_time, P.s.mk_start, mr, a.gb, a.ge, er, a.eb, a.ee, &amb);
    }
  }
  add_counters_block(stats, amb);
}

// ---- Coop step, front half (Alg. 1 step 1-3 without the global sort) ----
// The run length W of a node is its number of alive walks, so the solo tier
// (W < w_warp: one thread per walk, global marks) needs no grouping at all:
// a histogram of the current nodes decides it per walk. Only walks on nodes
// with W >= w_warp (the warp / block tiers) are compacted and sorted by node.
// Outputs are identical (every draw is keyed by (walk, hop)); tier counts are
// the reference's (one solo task per distinct solo node).
// Alg. 1 step start over the alive list: alive walks per node (the run
// lengths W), and the alive walks appended to the next list (one atomic per
// block; list order is free: the hub list is sorted by node, solo-task
// counting only needs one `first` per node)
__global__ void k_coop_count(StateArrays S, const u32* ids, const u64* n_ids, u32* ncnt, u8* first, u64* alive,
                             u32* next) {
  __shared__ u32 s_cnt[kBlock / 32], s_base;
  const u64 n = *n_ids;
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (u64 b = blockIdx.x * static_cast<u64>(blockDim.x); b < n; b += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 k = b + threadIdx.x;
    u32 w = 0;
    bool al = false;
    if (k < n) {
      w = ids[k];
      al = (S.flags[w] & 1u) != 0;
      if (al) first[w] = atomicAdd(ncnt + S.cur[w], 1u) == 0 ? 1 : 0;
    }
    const u32 m = __ballot_sync(0xffffffffu, al);
    if (lane == 0) s_cnt[warp] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      u32 acc = 0;
      for (int q = 0; q < kBlock / 32; ++q) {
        const u32 c = s_cnt[q];
        s_cnt[q] = acc;
        acc += c;
      }
      s_base = acc ? static_cast<u32>(atomicAdd(reinterpret_cast<unsigned long long*>(alive),
                                                static_cast<unsigned long long>(acc)))
                   : 0u;
    }
    __syncthreads();
    if (al) next[s_base + s_cnt[warp] + __popc(m & ((1u << lane) - 1u))] = w;
    __syncthreads();
  }
}

__global__ void k_iota(u32* ids, u64 n, u64* n_out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    ids[i] = static_cast<u32>(i);
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = n;
}

// solo walks hop now; the others are compacted into (node, walk) pairs.
// scal: [0] hub walks, [1] solo tasks (distinct solo nodes)
__global__ void __launch_bounds__(kBlock) k_coop_solo(WalkParams P, StateArrays S, const u32* ids, const u64* n_ids,
                                                     const u32* ncnt, const u8* first, u32 w_warp, u32* hub_keys,
                                                     u32* hub_vals, u64* scal, u64* stats) {
  __shared__ u32 s_hub[kBlock / 32], s_solo[kBlock / 32], s_base;
  Ctr cn{0, 0};
  const u32 lane = threadIdx.x & 31;
  const u64 count = *n_ids;  // the alive list of this step
  for (u64 b = blockIdx.x * static_cast<u64>(blockDim.x); b < count; b += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 kk = b + threadIdx.x;
    const u32 w = kk < count ? ids[kk] : 0u;
    bool hub = false, solo_task = false;
    u32 node = 0;
    if (kk < count) {
      node = S.cur[w];
      if (ncnt[node] < w_warp) {
        solo_task = first[w] != 0;
        const NodeMeta a = P.s.nm[node];
        WalkReg r;
        load_state(S, static_cast<u32>(w), r);
        const bool ok = hop(P, w, r, P.s.mk_time, P.s.mk_start, mark_ring(a), a.gb, a.ge, entry_ring(a), a.eb, a.ee,
                            &cn);
        store_state(S, static_cast<u32>(w), r, ok, P.stride);
      } else {
        hub = true;
      }
    }
    // hub-list slots: one atomic per block (per-warp atomics on one word
    // serialise at L2), warps ordered inside the block
    const u32 hb = __ballot_sync(0xffffffffu, hub), sb = __ballot_sync(0xffffffffu, solo_task);
    const u32 warp = threadIdx.x >> 5;
    if (lane == 0) {
      s_hub[warp] = __popc(hb);
      s_solo[warp] = __popc(sb);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      u32 h = 0, so = 0;
      for (int q = 0; q < kBlock / 32; ++q) {
        const u32 c = s_hub[q];
        s_hub[q] = h;
        h += c;
        so += s_solo[q];
      }
      s_base = h ? static_cast<u32>(atomicAdd(reinterpret_cast<unsigned long long*>(&scal[0]),
                                              static_cast<unsigned long long>(h)))
                 : 0u;
      if (so) atomicAdd(reinterpret_cast<unsigned long long*>(&scal[1]), static_cast<unsigned long long>(so));
    }
    __syncthreads();
    const u32 base = s_base + s_hub[warp];
    __syncthreads();  // s_hub / s_base are rewritten next round
    if (hub) {
      const u32 k = base + __popc(hb & ((1u << lane) - 1u));
      hub_keys[k] = node;
      hub_vals[k] = static_cast<u32>(w);
    }
  }
  add_counters_block(stats, cn);
}

__global__ void k_finalize(const StateArrays S, u64 count, u32* lengths, u64* stats) {
  const u64 wl = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
  const bool active = wl < count;
  const u32 len = active ? S.len[wl] : 0;
  if (active) lengths[wl] = len;
  add_stats_block(stats, len, len, Ctr{0, 0}, active);
}

__global__ void k_start_flags(const NodeMeta* nm, u64 V, u32* flags) {
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<u64>(gridDim.x) * blockDim.x)
    flags[v] = nm[v].eb != nm[v].ee ? 1u : 0u;
}

__global__ void k_start_nodes(const u32* flags, const u32* pos, u64 V, u32* out) {
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<u64>(gridDim.x) * blockDim.x)
    if (flags[v]) out[pos[v]] = static_cast<u32>(v);
}

// slot-major device layout -> the reference's walk-major fixed-stride image
// with zeroed unused slots (walk_engine.cpp:237-239)
__global__ void k_to_walk_major(const i64* nodes, const i64* times, const u32* lengths, u64 count, u32 stride,
                                i64* wn, i64* wt) {
  const u64 total = count * stride;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 w = i / stride;
    const u32 slot = static_cast<u32>(i - w * stride);
    const bool used = slot < lengths[w];
    wn[i] = used ? nodes[static_cast<u64>(slot) * count + w] : 0;
    wt[i] = used ? times[static_cast<u64>(slot) * count + w] : 0;
  }
}

struct LenFn {
  const u32* len;
  __device__ __forceinline__ u64 operator()(u64 i) const { return len[i]; }
};

// compact CSR image from the slot-major layout: thread per walk, reads of
// slot j are coalesced across consecutive walks
__global__ void k_compact_walks(const i64* nodes, const i64* times, const u32* lengths, const u64* offs, u64 count,
                                u32 stride, i64* cn, i64* ct) {
  for (u64 w = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; w < count;
       w += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 o = offs[w];
    for (u32 j = 0; j < lengths[w]; ++j) {
      cn[o + j] = nodes[static_cast<u64>(j) * count + w];
      ct[o + j] = times[static_cast<u64>(j) * count + w];
    }
  }
  (void)stride;
}

unsigned grid(Ctx& ctx, u64 n) { return grid_for(n, kBlock, static_cast<unsigned>(ctx.sm_count) * 32); }

// The store a walk runs on: streaming (gapped) stores serve every picker
// directly (exp-weight prefixes evaluated on the fly, draw_weighted_ring;
// the static node2vec adjacency by a scan of the previous node's region).
Store& walk_store(Ctx&, Store& s, const twg_walk_config&) { return s; }

// FullWalk launch knobs (A/B experiments; defaults are the measured best)
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && e[0] ? std::atoi(e) : dflt;
}
int walk_block() {
  static const int b = env_int("TWG_WALK_BLOCK", 32);
  return b;
}
bool walk_rec_enabled() {
  static const bool on = env_int("TWG_WALK_REC", 1) != 0;
  return on;
}

WalkParams make_params(Ctx& ctx, Store& s, const twg_walk_config& cfg, u32 stride, u64 walk_begin, WalkSetDev& out,
                       bool slot_major = false, u64 count = 0) {
  WalkParams P;
  P.slot_major = slot_major ? 1 : 0;
  P.count = count;
  P.s = s.view();
  P.rng = Rng::make(cfg.rng, cfg.seed);
  P.bias = cfg.bias;
  P.dir = cfg.direction;
  P.node2vec = cfg.node2vec;
  P.temporal_adj = cfg.temporal_adjacency;
  if (cfg.node2vec) {
    P.inv_p = 1.0 / cfg.p;
    P.inv_q = 1.0 / cfg.q;
    P.bmax = P.inv_p;  // samplers.hpp:27-29 max({1/p, 1, 1/q})
    if (1.0 > P.bmax) P.bmax = 1.0;
    if (P.inv_q > P.bmax) P.bmax = P.inv_q;
  } else {
    P.inv_p = P.inv_q = P.bmax = 1.0;
  }
  P.stride = stride;
  P.walk_begin = walk_begin;
  P.nodes = out.nodes.p;
  P.times = out.times.p;
  P.exp_neg = ctx.d_exp_neg;
  P.expm1_tab = ctx.d_expm1;
  P.rec = 0;
  return P;
}

// Start plan of init_walks (walk_engine.cpp:214-235): per-node starts are
// the nodes with a non-empty region, in id order (walk id = rank * k + j).
void plan_starts(Ctx& ctx, Store& s, const twg_walk_config& cfg, u32* stride, u64* total, DevBuf<u32>& start_nodes) {
  cudaStream_t st = ctx.stream;
  if (cfg.start_mode == 0) {
    DevBuf<u32> flags(s.V ? s.V : 1, st), pos(s.V + 1, st);
    if (s.V) {
      k_start_flags<<<grid(ctx, s.V), kBlock, 0, st>>>(s.nm.p, s.V, flags.p);
      TWG_LAUNCHED(ctx);
    }
    exclusive_scan<u32>(ctx, LoadFn<u32>{flags.p}, s.V, pos.p);
    u64 sc[1];
    TWG_CUDA(cudaMemsetAsync(ctx.d_scalars, 0, 8, st));
    TWG_CUDA(cudaMemcpyAsync(ctx.d_scalars, pos.p + s.V, 4, cudaMemcpyDeviceToDevice, st));
    read_scalars(ctx, ctx.d_scalars, sc, 1);
    start_nodes.alloc(sc[0] ? sc[0] : 1, st);
    if (s.V) {
      k_start_nodes<<<grid(ctx, s.V), kBlock, 0, st>>>(flags.p, pos.p, s.V, start_nodes.p);
      TWG_LAUNCHED(ctx);
    }
    *total = sc[0] * static_cast<u64>(cfg.walks_per_node);
    *stride = cfg.walk_length;
  } else {
    if (s.m == 0) fail(TWG_EINVAL, "init_walks: sampled starts need a non-empty store");
    *total = cfg.total_walks;
    *stride = cfg.walk_length > 2 ? cfg.walk_length : 2;  // walk_engine.cpp:229
  }
  if (*total >= 0xffffffffull) fail(TWG_EINVAL, "init_walks: walk count exceeds 32-bit id space");
}

void validate_config(const twg_walk_config& cfg) {  // WalkConfig::validate (walk_engine.cpp:198-206)
  if (cfg.walk_length < 1) fail(TWG_EINVAL, "walk config: walk_length must be >= 1");
  if (cfg.start_mode == 0 && cfg.walks_per_node == 0) fail(TWG_EINVAL, "walk config: walks_per_node must be positive");
  if (cfg.node2vec && (cfg.p <= 0.0 || cfg.q <= 0.0)) fail(TWG_EINVAL, "walk config: node2vec p and q must be positive");
  if (cfg.bias < 0 || cfg.bias > 3 || cfg.start_bias < 0 || cfg.start_bias > 3) fail(TWG_EINVAL, "walk config: bias");
  if (cfg.direction != 0 && cfg.direction != 1) fail(TWG_EINVAL, "walk config: direction");
  if (cfg.rng != TWG_RNG_SPLITMIX && cfg.rng != TWG_RNG_PHILOX) fail(TWG_EINVAL, "walk config: rng");
}

__global__ void k_unpack_states(StateArrays S, u64 n, u32* cur, i64* t, u32* prev, u8* has_prev, u8* alive,
                                u32* len) {
  for (u64 w = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; w < n;
       w += static_cast<u64>(gridDim.x) * blockDim.x) {
    cur[w] = S.cur[w];
    t[w] = S.t[w];
    prev[w] = S.prev[w];
    has_prev[w] = (S.flags[w] >> 1) & 1u;
    alive[w] = S.flags[w] & 1u;
    len[w] = S.len[w];
  }
}

__global__ void k_pack_states(StateArrays S, u64 n, const u32* cur, const i64* t, const u32* prev, const u8* has_prev,
                              const u8* alive, const u32* len) {
  for (u64 w = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; w < n;
       w += static_cast<u64>(gridDim.x) * blockDim.x) {
    S.cur[w] = cur[w];
    S.t[w] = t[w];
    S.prev[w] = prev[w];
    S.len[w] = len[w];
    S.flags[w] = static_cast<u8>((alive[w] ? 1 : 0) | (has_prev[w] ? 2 : 0));
  }
}

// execute_task's per-walk loop (walk_engine.cpp:357-359) over a walk-id list
__global__ void k_hop_list(WalkParams P, StateArrays S, const u32* ids, u64 n, u64* stats) {
  Ctr cn{0, 0};
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 w = ids[i];
    const NodeMeta a = P.s.nm[S.cur[w]];
    WalkReg r;
    load_state(S, w, r);
    const bool ok = hop(P, w, r, P.s.mk_time, P.s.mk_start, mark_ring(a), a.gb, a.ge, entry_ring(a), a.eb, a.ee, &cn);
    store_state(S, w, r, ok, P.stride);
  }
  add_counters_block(stats, cn);
}

}  // namespace

void init_walks_dev(Ctx& ctx, Store& s_in, const twg_walk_config& cfg, u32* stride, u64* walk_count,
                    const HostWalkArrays* out) {
  validate_config(cfg);
  Store& s = walk_store(ctx, s_in, cfg);
  cudaStream_t st = ctx.stream;
  u64 total = 0;
  DevBuf<u32> start_nodes;
  plan_starts(ctx, s, cfg, stride, &total, start_nodes);
  *walk_count = total;
  if (!out || total == 0) return;
  if (cfg.start_bias == TWG_EXPWEIGHT) ensure_weights(ctx, s);
  WalkSetDev tmp;
  tmp.nodes.alloc(total * *stride, st);
  tmp.times.alloc(total * *stride, st);
  TWG_CUDA(cudaMemsetAsync(tmp.nodes.p, 0, tmp.nodes.bytes(), st));
  TWG_CUDA(cudaMemsetAsync(tmp.times.p, 0, tmp.times.bytes(), st));
  WalkParams P = make_params(ctx, s, cfg, *stride, 0, tmp);
  InitParams I{cfg.start_mode, cfg.walks_per_node, cfg.start_bias, start_nodes.p,
               cfg.direction == 0 ? kTimeUnset : kTimeInfinite};
  DevBuf<u32> cur(total, st), prev(total, st), len(total, st);
  DevBuf<i64> tt(total, st);
  DevBuf<u8> flags(total, st);
  DevBuf<u64> stats(8, st);
  TWG_CUDA(cudaMemsetAsync(stats.p, 0, stats.bytes(), st));
  StateArrays S{cur.p, prev.p, tt.p, len.p, flags.p};
  k_init_states<<<grid_for(total, kBlock, 0xffffffffu), kBlock, 0, st>>>(P, I, total, S, stats.p);
  TWG_LAUNCHED(ctx);
  DevBuf<u32> oc(total, st), op(total, st), ol(total, st);
  DevBuf<i64> ot(total, st);
  DevBuf<u8> oh(total, st), oa(total, st);
  k_unpack_states<<<grid(ctx, total), kBlock, 0, st>>>(S, total, oc.p, ot.p, op.p, oh.p, oa.p, ol.p);
  TWG_LAUNCHED(ctx);
  TWG_CUDA(cudaMemcpyAsync(out->current, oc.p, total * 4, cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(out->time, ot.p, total * 8, cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(out->prev, op.p, total * 4, cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(out->has_prev, oh.p, total, cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(out->alive, oa.p, total, cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(out->length, ol.p, total * 4, cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(out->nodes, tmp.nodes.p, tmp.nodes.bytes(), cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(out->times, tmp.times.p, tmp.times.bytes(), cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaStreamSynchronize(st));
}

void hop_walks_dev(Ctx& ctx, Store& s_in, const twg_walk_config& cfg, const u32* ids, u64 n_ids, u64 count, u32 stride,
                   const HostWalkArrays& io) {
  validate_config(cfg);
  Store& s = walk_store(ctx, s_in, cfg);
  cudaStream_t st = ctx.stream;
  if (cfg.bias == TWG_EXPWEIGHT) ensure_weights(ctx, s);
  if (cfg.node2vec && !cfg.temporal_adjacency) ensure_adjacency(ctx, s);
  if (n_ids == 0 || count == 0) return;
  WalkSetDev tmp;
  tmp.nodes.alloc(count * stride, st);
  tmp.times.alloc(count * stride, st);
  TWG_CUDA(cudaMemcpyAsync(tmp.nodes.p, io.nodes, tmp.nodes.bytes(), cudaMemcpyHostToDevice, st));
  TWG_CUDA(cudaMemcpyAsync(tmp.times.p, io.times, tmp.times.bytes(), cudaMemcpyHostToDevice, st));
  DevBuf<u32> ic(count, st), ip(count, st), il(count, st), dids(n_ids, st);
  DevBuf<i64> it(count, st);
  DevBuf<u8> ih(count, st), ia(count, st);
  TWG_CUDA(cudaMemcpyAsync(ic.p, io.current, count * 4, cudaMemcpyHostToDevice, st));
  TWG_CUDA(cudaMemcpyAsync(it.p, io.time, count * 8, cudaMemcpyHostToDevice, st));
  TWG_CUDA(cudaMemcpyAsync(ip.p, io.prev, count * 4, cudaMemcpyHostToDevice, st));
  TWG_CUDA(cudaMemcpyAsync(ih.p, io.has_prev, count, cudaMemcpyHostToDevice, st));
  TWG_CUDA(cudaMemcpyAsync(ia.p, io.alive, count, cudaMemcpyHostToDevice, st));
  TWG_CUDA(cudaMemcpyAsync(il.p, io.length, count * 4, cudaMemcpyHostToDevice, st));
  TWG_CUDA(cudaMemcpyAsync(dids.p, ids, n_ids * 4, cudaMemcpyHostToDevice, st));
  DevBuf<u32> cur(count, st), prev(count, st), len(count, st);
  DevBuf<i64> tt(count, st);
  DevBuf<u8> flags(count, st);
  StateArrays S{cur.p, prev.p, tt.p, len.p, flags.p};
  k_pack_states<<<grid(ctx, count), kBlock, 0, st>>>(S, count, ic.p, it.p, ip.p, ih.p, ia.p, il.p);
  TWG_LAUNCHED(ctx);
  DevBuf<u64> stats(8, st);
  TWG_CUDA(cudaMemsetAsync(stats.p, 0, stats.bytes(), st));
  WalkParams P = make_params(ctx, s, cfg, stride, 0, tmp);
  k_hop_list<<<grid(ctx, n_ids), kBlock, 0, st>>>(P, S, dids.p, n_ids, stats.p);
  TWG_LAUNCHED(ctx);
  k_unpack_states<<<grid(ctx, count), kBlock, 0, st>>>(S, count, ic.p, it.p, ip.p, ih.p, ia.p, il.p);
  TWG_LAUNCHED(ctx);
  TWG_CUDA(cudaMemcpyAsync(io.current, ic.p, count * 4, cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(io.time, it.p, count * 8, cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(io.prev, ip.p, count * 4, cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(io.has_prev, ih.p, count, cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(io.alive, ia.p, count, cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(io.length, il.p, count * 4, cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(io.nodes, tmp.nodes.p, tmp.nodes.bytes(), cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaMemcpyAsync(io.times, tmp.times.p, tmp.times.bytes(), cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaStreamSynchronize(st));
}

void walk_major_image(Ctx& ctx, const WalkSetDev& w, DevBuf<i64>& nodes, DevBuf<i64>& times) {
  const u64 cells = w.count * w.stride;
  nodes.alloc(cells ? cells : 1, ctx.stream);
  times.alloc(cells ? cells : 1, ctx.stream);
  if (!cells) return;
  k_to_walk_major<<<grid(ctx, cells), kBlock, 0, ctx.stream>>>(w.nodes.p, w.times.p, w.lengths.p, w.count, w.stride,
                                                                nodes.p, times.p);
  TWG_LAUNCHED(ctx);
}

void compact_walks(Ctx& ctx, const WalkSetDev& w, DevBuf<u64>& offsets, DevBuf<i64>& nodes, DevBuf<i64>& times,
                   u64* total) {
  offsets.alloc(w.count + 1, ctx.stream);
  exclusive_scan<u64>(ctx, LenFn{w.lengths.p}, w.count, offsets.p);
  u64 tot[1];
  read_scalars(ctx, offsets.p + w.count, tot, 1);
  *total = tot[0];
  nodes.alloc(tot[0] ? tot[0] : 1, ctx.stream);
  times.alloc(tot[0] ? tot[0] : 1, ctx.stream);
  if (w.count) {
    k_compact_walks<<<grid(ctx, w.count), kBlock, 0, ctx.stream>>>(w.nodes.p, w.times.p, w.lengths.p, offsets.p,
                                                                    w.count, w.stride, nodes.p, times.p);
    TWG_LAUNCHED(ctx);
  }
}

WalkSetDev* generate_walks(Ctx& ctx, Store& s_in, const twg_walk_config& cfg, const twg_thresholds& th, int variant,
                           twg_walk_stats* stats_out, int shard_rank, int shard_count) {
  NvtxRange nvtx_scope(variant == TWG_FULLWALK ? "twg generate_walks (FullWalk)" : "twg generate_walks (Coop)");
  Store& s = walk_store(ctx, s_in, cfg);
  using clock = std::chrono::steady_clock;
  const auto started = clock::now();
  cudaStream_t st = ctx.stream;
  // WalkConfig::validate (walk_engine.cpp:198-206), TierThresholds::validate (:189-196)
  if (cfg.walk_length < 1) fail(TWG_EINVAL, "walk config: walk_length must be >= 1");
  if (cfg.start_mode == 0 && cfg.walks_per_node == 0) fail(TWG_EINVAL, "walk config: walks_per_node must be positive");
  if (cfg.node2vec && (cfg.p <= 0.0 || cfg.q <= 0.0)) fail(TWG_EINVAL, "walk config: node2vec p and q must be positive");
  if (th.w_warp < 1 || th.w_warp > th.block_dim || th.block_dim > th.w_max)
    fail(TWG_EINVAL, "tier thresholds: need 1 <= w_warp <= block_dim <= w_max");
  if (th.g_warp_cap > th.g_block_cap) fail(TWG_EINVAL, "tier thresholds: need g_warp_cap <= g_block_cap");
  if (cfg.bias < 0 || cfg.bias > 3 || cfg.start_bias < 0 || cfg.start_bias > 3) fail(TWG_EINVAL, "walk config: bias");
  if (cfg.direction != 0 && cfg.direction != 1) fail(TWG_EINVAL, "walk config: direction");
  if (cfg.rng != TWG_RNG_SPLITMIX && cfg.rng != TWG_RNG_PHILOX) fail(TWG_EINVAL, "walk config: rng");
  // EdgeStore::supports (edge_store.hpp:60-63), walk_engine.cpp:368-370
  const bool supports = s.mode == TWG_UNDIRECTED || ((s.mode == TWG_FORWARD) == (cfg.direction == 0));
  if (!supports)
    fail(TWG_EINVAL, "generate_walks: store direction mode does not serve the requested walk direction");
  if (cfg.bias == TWG_EXPWEIGHT || cfg.start_bias == TWG_EXPWEIGHT) ensure_weights(ctx, s);
  if (cfg.node2vec && !cfg.temporal_adjacency) ensure_adjacency(ctx, s);

  auto out = std::make_unique<WalkSetDev>();
  out->ctx = &ctx;
  // init_walks (walk_engine.cpp:208-245)
  u64 total = 0;
  DevBuf<u32> start_nodes;
  plan_starts(ctx, s, cfg, &out->stride, &total, start_nodes);
  u64 wb = cfg.walk_begin, we = cfg.walk_end;
  if (wb == 0 && we == 0) we = total;
  if (we > total) we = total;
  if (wb > we) wb = we;
  if (shard_count > 1) {  // this rank's contiguous, balanced slice of [wb, we) (multi-GPU group)
    const u64 span = we - wb, base = span / shard_count, extra = span % shard_count;
    const u64 r = static_cast<u64>(shard_rank);
    const u64 lo = wb + r * base + (r < extra ? r : extra);
    wb = lo;
    we = lo + base + (r < extra ? 1 : 0);
  }
  const u64 count = we - wb;
  out->first = wb;
  out->count = count;
  out->nodes.alloc(count * out->stride ? count * out->stride : 1, st);
  out->times.alloc(count * out->stride ? count * out->stride : 1, st);
  out->lengths.alloc(count ? count : 1, st);

  DevBuf<u64> stats(8, st);
  TWG_CUDA(cudaMemsetAsync(stats.p, 0, stats.bytes(), st));
  WalkParams P = make_params(ctx, s, cfg, out->stride, wb, *out, /*slot_major=*/true, count);
  InitParams I;
  I.start_mode = cfg.start_mode;
  I.walks_per_node = cfg.walks_per_node;
  I.start_bias = cfg.start_bias;
  I.start_nodes = start_nodes.p;
  I.sentinel = cfg.direction == 0 ? kTimeUnset : kTimeInfinite;  // types.hpp:47-49

  u64 tiers[6] = {0, 0, 0, 0, 0, 0};
  u64 coop_steps = 0;
  if (count == 0) {
    // nothing to do
  } else if (variant == TWG_FULLWALK) {
    P.rec = walk_rec_enabled() && s.wrec.p && s.wrec.n >= s.V && P.dir == 0 && !P.node2vec &&
            (P.bias == TWG_UNIFORM || P.bias == TWG_LINEAR || P.bias == TWG_EXPINDEX);
    DevBuf<u64> part(kStatSlots * 8, st);
    TWG_CUDA(cudaMemsetAsync(part.p, 0, part.bytes(), st));
    const int wb = walk_block();
    const unsigned g = static_cast<unsigned>((count + wb - 1) / wb);
    if (P.rec) {
      // 32-thread blocks at 64 registers: 1024 resident threads per SM (the
      // 32-block limit); 40-register builds spill, 64-thread blocks measured
      // slower
      k_fullwalk<32, true><<<static_cast<unsigned>((count + 31) / 32), 32, 0, st>>>(P, I, count, out->lengths.p,
                                                                                   part.p);
    } else {
      switch (wb) {
        case 32: k_fullwalk<32, false><<<g, 32, 0, st>>>(P, I, count, out->lengths.p, part.p); break;
        case 64: k_fullwalk<64, false><<<g, 64, 0, st>>>(P, I, count, out->lengths.p, part.p); break;
        case 128: k_fullwalk<128, false><<<g, 128, 0, st>>>(P, I, count, out->lengths.p, part.p); break;
        default: k_fullwalk<256, false><<<g, 256, 0, st>>>(P, I, count, out->lengths.p, part.p); break;
      }
    }
    TWG_LAUNCHED(ctx);
    k_fold_stats<<<1, 160, 0, st>>>(part.p, stats.p);
    TWG_LAUNCHED(ctx);
  } else {
    const bool cache = variant == TWG_COOP;
    DevBuf<u32> cur(count, st), prev(count, st), len(count, st);
    DevBuf<i64> tt(count, st);
    DevBuf<u8> flags(count, st);
    StateArrays S{cur.p, prev.p, tt.p, len.p, flags.p};
    k_init_states<<<grid_for(count, kBlock, 0xffffffffu), kBlock, 0, st>>>(P, I, count, S, stats.p);
    TWG_LAUNCHED(ctx);
    DevBuf<u32> k0(count, st), k1(count, st), v0(count, st), v1(count, st);
    DevBuf<Task> tasks(5 * count, st);
    DevBuf<u32> subcount(5 * count, st);
    DevBuf<u32> counters(8, st);
    const int vb = s.V > 1 ? bit_width_u64(s.V - 1) : 0;
    TaskLists T;
    for (int k = 0; k < 5; ++k) {
      T.list[k] = tasks.p + k * count;
      T.subcount[k] = subcount.p + k * count;
    }
    T.count = counters.p;
    const u32 warp_cap = th.g_warp_cap;
    u32 block_cap = th.g_block_cap;
    const size_t warp_smem = static_cast<size_t>(warp_cap) * 12 * (kBlock / 32);
    const bool warp_stage = cache && warp_smem <= 200 * 1024;
    if (block_cap * 12ull > 200 * 1024) block_cap = 200 * 1024 / 12;
    const size_t block_smem = static_cast<size_t>(block_cap) * 12;
    if (warp_stage)
      TWG_CUDA(cudaFuncSetAttribute(k_tier_warp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(warp_smem)));
    if (cache)
      TWG_CUDA(cudaFuncSetAttribute(k_tier_block<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(block_smem)));
    DevBuf<u32> ncnt(s.V ? s.V : 1, st);
    DevBuf<u8> first(count, st);
    // the alive list, compacted every step so a step costs O(alive walks)
    DevBuf<u32> ids0(count ? count : 1, st), ids1(count ? count : 1, st);
    u32* ids_cur = ids0.p;
    u32* ids_next = ids1.p;
    u64* sc2 = ctx.d_scalars + 48;  // [48] alive (next list size), [49] hub walks, [50] solo tasks, [51] list size
    u64* n_cur = sc2 + 3;
    k_iota<<<grid(ctx, count), kBlock, 0, st>>>(ids_cur, count, n_cur);
    TWG_LAUNCHED(ctx);
    u64 n_alive = count;
    static const bool trace = [] {
      const char* e = std::getenv("TWG_COOP_TRACE");
      return e && e[0] == '1';
    }();
    auto t_prev = std::chrono::steady_clock::now();
    while (true) {
      // 1. alive walks per current node (the run lengths W), alive list compacted
      TWG_CUDA(cudaMemsetAsync(ncnt.p, 0, ncnt.bytes(), st));
      TWG_CUDA(cudaMemsetAsync(sc2, 0, 3 * sizeof(u64), st));
      k_coop_count<<<grid(ctx, n_alive), kBlock, 0, st>>>(S, ids_cur, n_cur, ncnt.p, first.p, sc2, ids_next);
      TWG_LAUNCHED(ctx);
      // 2. solo tier (W < w_warp): hop per walk; the rest compacted as (node, walk)
      k_coop_solo<<<grid(ctx, n_alive), kBlock, 0, st>>>(P, S, ids_next, sc2, ncnt.p, first.p, th.w_warp, k0.p, v0.p,
                                                          sc2 + 1, stats.p);
      TWG_LAUNCHED(ctx);
      u64 sc[3];
      read_scalars(ctx, sc2, sc, 3);
      if (trace) {
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[twg coop] step %llu alive %llu hub-walks %llu solo-tasks %llu  %.1f us\n",
                     static_cast<unsigned long long>(coop_steps), static_cast<unsigned long long>(n_alive),
                     static_cast<unsigned long long>(sc[1]), static_cast<unsigned long long>(sc[2]),
                     std::chrono::duration<double, std::micro>(now - t_prev).count());
        t_prev = now;
      }
      if (sc[0] == 0) break;
      n_alive = sc[0];
      std::swap(ids_cur, ids_next);
      TWG_CUDA(cudaMemcpyAsync(n_cur, sc2, sizeof(u64), cudaMemcpyDeviceToDevice, st));
      ++coop_steps;
      tiers[0] += sc[2];
      const u64 n = sc[1];
      if (n == 0) continue;
      // 3. stable sort of the hub walks by node, runs, dispatch plane, mega-hub split
      u32* kp = k0.p;
      u32* ka = k1.p;
      u32* vp = v0.p;
      u32* va = v1.p;
      radix_sort_pairs<u32>(ctx, &kp, &ka, &vp, &va, n, vb);
      TWG_CUDA(cudaMemsetAsync(counters.p, 0, counters.bytes(), st));
      k_classify<<<grid(ctx, n), kBlock, 0, st>>>(kp, n, s.view(), th, T);
      TWG_LAUNCHED(ctx);
      u32 cnt[8];
      u64 words[4];
      read_scalars(ctx, reinterpret_cast<const u64*>(counters.p), words, 4);
      std::memcpy(cnt, words, sizeof cnt);
      // tier counts (count_tier, walk_engine.cpp:157-169): split pieces count as multi_block
      for (int k = 1; k < 3; ++k) tiers[k] += cnt[k];
      tiers[3] += cnt[3] - cnt[5];
      tiers[4] += cnt[4] - cnt[6];
      tiers[5] += cnt[5] + cnt[6];
      // 4. terminal tiers (runs here all have W >= w_warp)
      if (cnt[1]) {
        if (warp_stage) {
          k_tier_warp<true><<<static_cast<unsigned>(std::min<u64>((cnt[1] + 7) / 8, 1u << 20)), kBlock, warp_smem, st>>>(
              P, S, vp, T.list[1], counters.p + 1, warp_cap, stats.p);
        } else {
          k_tier_warp<false><<<static_cast<unsigned>(std::min<u64>((cnt[1] + 7) / 8, 1u << 20)), kBlock, 0, st>>>(
              P, S, vp, T.list[1], counters.p + 1, 0, stats.p);
        }
        TWG_LAUNCHED(ctx);
      }
      if (cnt[2]) {
        k_tier_warp<false><<<static_cast<unsigned>(std::min<u64>((cnt[2] + 7) / 8, 1u << 20)), kBlock, 0, st>>>(
            P, S, vp, T.list[2], counters.p + 2, 0, stats.p);
        TWG_LAUNCHED(ctx);
      }
      if (cnt[3]) {
        if (cache) {
          k_tier_block<true><<<static_cast<unsigned>(std::min<u64>(cnt[3], 1u << 20)), kBlock, block_smem, st>>>(
              P, S, vp, T.list[3], counters.p + 3, block_cap, stats.p);
        } else {
          k_tier_block<false><<<static_cast<unsigned>(std::min<u64>(cnt[3], 1u << 20)), kBlock, 0, st>>>(
              P, S, vp, T.list[3], counters.p + 3, 0, stats.p);
        }
        TWG_LAUNCHED(ctx);
      }
      if (cnt[4]) {
        k_tier_block<false><<<static_cast<unsigned>(std::min<u64>(cnt[4], 1u << 20)), kBlock, 0, st>>>(
            P, S, vp, T.list[4], counters.p + 4, 0, stats.p);
        TWG_LAUNCHED(ctx);
      }
    }
    k_finalize<<<grid_for(count, kBlock, 0xffffffffu), kBlock, 0, st>>>(S, count, out->lengths.p, stats.p);
    TWG_LAUNCHED(ctx);
  }
  u64 hs[5];
  read_scalars(ctx, stats.p, hs, 5);
  out->hops = hs[1];
  if (stats_out) {
    twg_walk_stats w{};
    w.walks = hs[0];
    w.hops = hs[1];
    w.ambiguous_draws = hs[3];
    w.alg_bytes = hs[4];
    if (variant == TWG_FULLWALK) {
      w.steps = hs[2];
    } else {
      w.steps = coop_steps;
      w.solo = tiers[0];
      w.warp_cached = tiers[1];
      w.warp_direct = tiers[2];
      w.block_cached = tiers[3];
      w.block_direct = tiers[4];
      w.multi_block = tiers[5];
    }
    w.wall_seconds = std::chrono::duration<double>(clock::now() - started).count();
    *stats_out = w;
  }
  return out.release();
}

}  // namespace twg
