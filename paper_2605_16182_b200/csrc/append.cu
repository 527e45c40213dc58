// Streaming append ingest: the time-ordered fast path of
// WindowManager::ingest_batch (window_manager.cpp:14-62) on the shared
// EdgeLog / NodeArena representation (store.cuh).
//
// Preconditions (checked by the caller, window.cu ingest_streaming): the
// admitted batch sorts after every survivor in canonical order (the merge
// is a concatenation) and the node population is unchanged (new dense ids
// == old dense ids), so every id, every surviving entry and every surviving
// mark keeps its value. The snapshot the reference would rebuild from
// scratch is then
//   edges   = old edges [from, m) ++ sorted batch          -> a log append
//   ts view = old groups with time >= cutoff ++ batch groups -> a log append
//   node v  = v's entries with t >= cutoff ++ v's batch entries (canonical
//             order), marks likewise                          -> region append
// and the cost per batch is O(batch + V) instead of O(window):
//   1. log append of the sorted batch; ts groups of the batch by flag+scan;
//   2. batch entries stable-sorted by owner (radix), run bounds per node;
//   3. per node: eviction = galloping lower_bound(cutoff) on the region's
//      entry times and mark times; slack check; regions without room are
//      relocated (block-aggregated bump allocation), all regions when the
//      arena is replaced;
//   4. one decoupled-look-back pass over the sorted batch entries places
//      them at their region ends and numbers the new marks; a per-mark pass
//      scatters the marks; a per-node pass publishes {eb, ee, gb, ge}.
// Results are bit-identical to the full rebuild (tests compare every array
// after every batch against the oracle and the reference).
#include "primitives.cuh"
#include "window.cuh"

namespace twg {

namespace {

#ifndef TWG_PLACE_CHUNK
#define TWG_PLACE_CHUNK 2048
#endif
#ifndef TWG_PLACE_MINB
#define TWG_PLACE_MINB 4
#endif
constexpr int kBlock = 256;
constexpr int kPB = 256;           // nodes per bucket = threads per placement CTA
constexpr u32 kBucketShift = 8;
constexpr int kChunk = TWG_PLACE_CHUNK;  // bucket entries staged per placement round
constexpr int kChunkItems = kChunk / kPB;
static_assert(kChunk % kPB == 0, "whole rounds per chunk");
static_assert(kPB == 1 << kBucketShift, "one thread per bucket node");

unsigned grid(Ctx& ctx, u64 n) { return grid_for(n, kBlock, static_cast<unsigned>(ctx.sm_count) * 16); }

// first k in [0, n) with t[zr(k)] >= x (one warp)
__global__ void k_lb_time(const i64* t, Ring zr, u64 n, i64 x, u64* out) {
  const u64 r = warp_lower_bound([&](u64 k) { return t[zr(static_cast<u32>(k))]; }, n, x);
  if (threadIdx.x == 0) *out = r;
}

// survivors [from, from + n) of a snapshot -> the start of a new log
__global__ void k_copy_cols(StoreView v, u64 from, u64 n, EdgeRec* out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    out[i] = edge_at(v, from + i);
}

// surviving ts groups [g_cut, Z) of the old snapshot -> a fresh log
__global__ void k_copy_groups(const u32* off, const i64* tt, Ring zr, u64 Z, const u64* g_cut, u32* ooff, i64* ott) {
  const u64 g0 = *g_cut;
  for (u64 g = g0 + blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; g < Z;
       g += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 p = zr(static_cast<u32>(g));
    ooff[g - g0] = off[p];
    ott[g - g0] = tt[p];
  }
}

// batch group starts: the first batch edge starts a group unless it shares
// the last survivor's time
struct BatchGroupFn {
  const EdgeRec* b;
  Ring br;                     // batch index -> slot of b
  const i64* last_survivor_t;  // null when there are no survivors
  const i64* bt;               // the batch's time column in batch order, when at hand (8 B/edge, not 16)
  __device__ __forceinline__ i64 time(u64 k) const { return bt ? bt[k] : b[br(static_cast<u32>(k))].t; }
  __device__ __forceinline__ u32 operator()(u64 k) const {
    const i64 tk = time(k);
    if (k == 0) return last_survivor_t ? (tk != *last_survivor_t ? 1u : 0u) : 1u;
    return tk != time(k - 1) ? 1u : 0u;
  }
};

struct BatchGroupScatter {
  const EdgeRec* b;
  Ring br;
  u32 seq_b;
  u64 zbase;              // host-known logical write position, or
  const u64* zbase_dev;   // device-resident one (fresh log: Z_old - g_cut)
  u64 cap;                // ring slots
  u32* ts_off;
  i64* ts_time;
  const i64* bt;
  __device__ __forceinline__ void operator()(u64 k, u64 g, u32 f) const {
    if (!f) return;
    // zbase < cap (reduced on the host; the device-resident one is a fresh
    // log's count, below its capacity) and g < cap: one compare, no division
    const u64 x = (zbase_dev ? *zbase_dev : zbase) + g;
    const u64 z = x >= cap ? x - cap : x;
    ts_off[z] = seq_b + static_cast<u32>(k);
    ts_time[z] = bt ? bt[k] : b[br(static_cast<u32>(k))].t;
  }
};

__global__ void k_zbase(u64 Z, const u64* g_cut, u64* out) { *out = Z - *g_cut; }

// first logical x in [lo, hi) with time >= c, galloping from lo through
// the node's ring (eviction removes a short prefix of most regions)
template <class TimeAt>
__device__ __forceinline__ u32 gallop_lb(TimeAt at, u32 lo, u32 hi, i64 c) {
  if (lo >= hi || at(lo) >= c) return lo;
  u32 prev = lo, step = 1, bound = hi;
  while (true) {  // at(prev) < c
    const u64 nx = static_cast<u64>(prev) + step;
    if (nx >= hi) break;
    if (at(static_cast<u32>(nx)) >= c) {
      bound = static_cast<u32>(nx);
      break;
    }
    prev = static_cast<u32>(nx);
    step <<= 1;
  }
  u32 a = prev + 1, b = bound;
  while (a < b) {
    const u32 mid = a + ((b - a) >> 1);
    if (at(mid) < c) a = mid + 1;
    else b = mid;
  }
  return a;
}

using Rec = BatchRec16;

#ifndef TWG_BOUNDS_KEYS
#define TWG_BOUNDS_KEYS 8  // k_bucket_bounds keys per thread (a multiple of 4)
#endif

// the admitted batch into the log ring
__global__ void k_append_batch(const EdgeRec* b, Ring br, u64 n, EdgeRec* log, Ring wr) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    log[wr(static_cast<u32>(i))] = b[br(static_cast<u32>(i))];
}

__device__ __forceinline__ u32 nbr_of(int mode, const Rec& r, u32 j) {
  if (mode == TWG_FORWARD) return r.dst;
  if (mode == TWG_BACKWARD) return r.src;
  return (j & 1) ? r.src : r.dst;  // side 1 (owner dst) -> src; self-loops give the owner
}

// Bucket-sort payloads: the finished node-view entry (16 B), or — when the
// batch's times span less than 2^32 — the same entry with its time as a u32
// offset from the batch minimum (12 B: every radix pass and the placement
// move 16 B per item with the key instead of 20).
struct alignas(4) PEnt {
  u32 nbr, edge, dt;
};
template <class V>
struct Payload;
template <>
struct Payload<Entry> {
  __device__ __forceinline__ static Entry make(u32 nbr, u32 edge, i64 t, i64) { return Entry{nbr, edge, t}; }
  __device__ __forceinline__ static Entry entry(const Entry& e, i64) { return e; }
  __device__ __forceinline__ static i64 time(const Entry& e, i64) { return e.t; }
};
template <>
struct Payload<PEnt> {
  __device__ __forceinline__ static PEnt make(u32 nbr, u32 edge, i64 t, i64 tb) {
    return PEnt{nbr, edge, static_cast<u32>(t - tb)};
  }
  __device__ __forceinline__ static Entry entry(const PEnt& e, i64 tb) {
    return Entry{e.nbr, e.edge, tb + static_cast<i64>(e.dt)};
  }
  __device__ __forceinline__ static i64 time(const PEnt& e, i64 tb) { return tb + static_cast<i64>(e.dt); }
};

// batch entry j: key = owner, payload = the finished node-view entry (carried
// through the bucket sort, so the placement reads it in order)
template <class V>
__global__ void k_owner_keys(const Rec* rec, Ring br, u64 A, int mode, u32 seq_b, i64 tb, u32* keys, V* vals) {
  const u64 Yn = mode == TWG_UNDIRECTED ? 2 * A : A;
  for (u64 j = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; j < Yn;
       j += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 k = mode == TWG_UNDIRECTED ? static_cast<u32>(j >> 1) : static_cast<u32>(j);
    const Rec r = rec[br(k)];
    keys[j] = mode == TWG_UNDIRECTED ? ((j & 1) ? r.dst : r.src) : (mode == TWG_BACKWARD ? r.dst : r.src);
    vals[j] = Payload<V>::make(nbr_of(mode, r, static_cast<u32>(j)), seq_b + k, r.t, tb);
  }
}

// (owner, node-view entry) of batch entry j, computed from the log records
template <class V>
struct OwnerIn {
  const Rec* rec;
  Ring br;
  int mode;
  u32 seq_b;
  i64 tb;  // time base of a PEnt payload
  __device__ __forceinline__ u32 key(u64 j) const {
    const Rec r = rec[br(mode == TWG_UNDIRECTED ? static_cast<u32>(j >> 1) : static_cast<u32>(j))];
    return mode == TWG_UNDIRECTED ? ((j & 1) ? r.dst : r.src) : (mode == TWG_BACKWARD ? r.dst : r.src);
  }
  __device__ __forceinline__ V val(u64 j) const {
    const u32 k = mode == TWG_UNDIRECTED ? static_cast<u32>(j >> 1) : static_cast<u32>(j);
    const Rec r = rec[br(k)];
    return Payload<V>::make(nbr_of(mode, r, static_cast<u32>(j)), seq_b + k, r.t, tb);
  }
  __device__ __forceinline__ bool has_val() const { return true; }
  __device__ __forceinline__ void prefetch_val(u64) const {}  // the key's record load brings it
  // the record itself held from the key load to the payload (kPre pass)
  using Item = Rec;
  __device__ __forceinline__ Rec item(u64 j) const {
    return rec[br(mode == TWG_UNDIRECTED ? static_cast<u32>(j >> 1) : static_cast<u32>(j))];
  }
  __device__ __forceinline__ u32 key_of(const Rec& r, u64 j) const {
    return mode == TWG_UNDIRECTED ? ((j & 1) ? r.dst : r.src) : (mode == TWG_BACKWARD ? r.dst : r.src);
  }
  __device__ __forceinline__ V val_of(const Rec& r, u64 j) const {
    const u32 k = mode == TWG_UNDIRECTED ? static_cast<u32>(j >> 1) : static_cast<u32>(j);
    return Payload<V>::make(nbr_of(mode, r, static_cast<u32>(j)), seq_b + k, r.t, tb);
  }
  // the same multiset of keys from the batch's own id columns (input order,
  // 8 B per item instead of a 16-B record) when they are at hand
  const i64* bs = nullptr;
  const i64* bd = nullptr;
  __device__ __forceinline__ u32 hist_key(u64 j) const {
    if (!bs) return key(j);
    if (mode == TWG_UNDIRECTED) return static_cast<u32>((j & 1) ? bd[j >> 1] : bs[j >> 1]);
    return static_cast<u32>(mode == TWG_BACKWARD ? bd[j] : bs[j]);
  }
  // (directed modes, one entry per edge; one warp) the first pass's tile
  // offsets come from the statistics pass's per-tile counts in INPUT order;
  // the log holds the CANONICAL order, which permutes edges only inside
  // equal-time runs of <= kSegMax edges (the fast route's admission). Below
  // `base` the two orders differ only in the run straddling it, [rs, base):
  // corr[d] += its canonical entries' digits - its input entries' digits.
  __device__ __forceinline__ void run_fix(u64 base, int shift, int* corr) const {
    if (base == 0) return;
    const int lane = threadIdx.x & 31;
    const i64 tb = rec[br(static_cast<u32>(base))].t;
    const i64 q = static_cast<i64>(base) - 32 + lane;
    if (q < 0) return;
    const Rec r = rec[br(static_cast<u32>(q))];
    if (r.t != tb) return;  // times ascend: the lanes left are the run's part below base
    const u32 oc = mode == TWG_BACKWARD ? r.dst : r.src;
    const u32 oi = static_cast<u32>(mode == TWG_BACKWARD ? bd[q] : bs[q]);
    atomicAdd(&corr[(oc >> shift) & (kRadix - 1)], 1);
    atomicAdd(&corr[(oi >> shift) & (kRadix - 1)], -1);
  }
};

// bucket b = owner >> 8 of the bucket-sorted entries starts at bstart[b]
// (empty buckets included); bstart[nb] = Yn. TWG_BOUNDS_KEYS keys per thread
// (128-bit loads; the key before them re-read from the neighbouring group).
__global__ void k_bucket_bounds(const u32* keys, u64 Yn, u64 nb, u32* bstart) {
  constexpr int kK = TWG_BOUNDS_KEYS;  // keys per thread (kK / 4 128-bit loads)
  const u64 groups = (Yn + kK) / kK;   // positions 0..Yn (Yn itself closes the last bucket)
  const bool aligned = (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
  for (u64 g = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; g < groups;
       g += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 q0 = kK * g;
    i64 cur[kK];
    if (q0 + kK <= Yn && aligned) {
#pragma unroll
      for (int h = 0; h < kK / 4; ++h) {
        const uint4 k4 = __ldg(reinterpret_cast<const uint4*>(keys + q0) + h);
        cur[4 * h] = k4.x >> kBucketShift, cur[4 * h + 1] = k4.y >> kBucketShift,
                cur[4 * h + 2] = k4.z >> kBucketShift, cur[4 * h + 3] = k4.w >> kBucketShift;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kK; ++j)
        cur[j] = q0 + j < Yn ? static_cast<i64>(keys[q0 + j] >> kBucketShift) : static_cast<i64>(nb);
    }
    i64 prev = q0 == 0 ? -1 : static_cast<i64>(keys[q0 - 1] >> kBucketShift);
#pragma unroll
    for (int j = 0; j < kK; ++j) {
      const u64 q = q0 + j;
      if (q > Yn) break;
      for (i64 b = prev + 1; b <= cur[j]; ++b) bstart[b] = static_cast<u32>(q);
      prev = cur[j];
    }
  }
}

// Eviction bound: first logical x in [lo, hi) with time >= c. The times
// from lo to the end of lo's 128-B line (kLine keys of the array) are loaded
// at once (independent loads, one round trip, one DRAM line — the whole line
// comes in anyway): a batch evicts only a few entries of a typical node;
// longer prefixes continue by galloping.
template <u32 kLine, class TimeAt>
__device__ __forceinline__ u32 evict_lb(TimeAt at, u32 slot_lo, u32 lo, u32 hi, i64 c) {
  const u32 k = min(hi - lo, kLine - (slot_lo & (kLine - 1)));
  i64 tt[kLine];
#pragma unroll
  for (u32 i = 0; i < kLine; ++i) tt[i] = i < k ? at(lo + i) : c;
  u32 n = 0;
#pragma unroll
  for (u32 i = 0; i < kLine; ++i) n += tt[i] < c ? 1u : 0u;
  if (n < k || k == hi - lo) return lo + n;
  return gallop_lb(at, lo + k, hi, c);
}

__device__ __forceinline__ u32 adjust_org(u32 org, u32 x, u32 cap) {  // org' = org (mod cap), 0 <= x - org' < cap
  return x - org >= cap ? org + cap : org;
}

struct Reloc {
  u32 v, src_e, src_g;
};

template <class PV>
struct PlanArgs {
  const NodeMeta* onm;  // the current snapshot
  const NodeMeta* rnm;  // the retired one when it shares the arena (its rings stay readable), else null
  u64 V;
  const Entry* oent;
  const i64* omt;
  const u32* oms;
  i64 cutoff;
  int need_last;        // a batch time may equal a node's newest live time (mark merge)
  int relocate_all;     // repack every ring into a fresh arena
  u32 rebase_at;        // a ring whose logical end would pass this is relocated (positions rebased to 0)
  u64 arena_cap;
  NodeMeta* plan;       // new bounds / ring; ee, ge = where the batch's entries / marks start
  i64* last_t;          // time of the last live entry (valid iff need_last and plan.ee > plan.eb)
  Reloc* reloc;
  u64* scal;            // [0] bump, [1] overflow, [2] relocations
  // the batch's per-node counts, from the bucket-sorted keys (one bucket per
  // CTA iteration), and the newest-time update (see the note at k_plan)
  const u32* keys;
  const PV* vals;
  const u32* bstart;
  i64 tb;               // time base of PEnt payloads
  const i64* old_last;  // null: node_last is updated in place
  i64* node_last;       // the new snapshot's newest incident time per node (null: none)
  u64* dead;            // null, or: count the nodes whose newest time falls before the cutoff
};

// Per node: eviction (cutoff lower bound on the ring's entry and mark
// times), room check against the oldest live begin in the ring (the retired
// snapshot's, while it shares the ring), otherwise a new ring from the bump
// allocator (CTA-aggregated) with logical positions rebased to 0.
//
// One CTA iteration = one bucket of kPB nodes: the bucket's batch entries are
// counted per node first (shared-memory atomics over the bucket-sorted keys;
// a node's last entry in canonical order carries its newest batch time), which
// also updates the newest-incident-time array (owner side; max with the old
// snapshot's) and counts nodes about to leave the window — the former
// k_bucket_count pass, without its per-node count array round trip.
template <class PV>
__global__ void __launch_bounds__(kBlock) k_plan(PlanArgs<PV> a) {
  static_assert(kBlock == kPB, "one bucket per CTA iteration");
  __shared__ u64 s_base;
  __shared__ u32 s_rbase;
  __shared__ u32 cnt[kPB], lastq[kPB];
  for (u64 b0 = static_cast<u64>(blockIdx.x) * kBlock; b0 < a.V; b0 += static_cast<u64>(gridDim.x) * kBlock) {
    const u64 v = b0 + threadIdx.x;
    const bool valid = v < a.V;
    // the node's own rows go out before the bucket's key counting
    NodeMeta o{}, rm{};
    i64 lt_old = 0;
    if (valid) {
      o = a.onm[v];
      if (a.rnm) rm = a.rnm[v];
      if (a.node_last) lt_old = a.old_last ? a.old_last[v] : a.node_last[v];
    }
    cnt[threadIdx.x] = 0;
    lastq[threadIdx.x] = 0;
    __syncthreads();
    {
      const u64 bkt = b0 >> kBucketShift;
      const u32 bs = a.bstart[bkt], be = a.bstart[bkt + 1];
      for (u32 q = bs + threadIdx.x; q < be; q += kPB) {
        const u32 nd = a.keys[q] & (kPB - 1);
        atomicAdd(&cnt[nd], 1u);
        atomicMax(&lastq[nd], q + 1);
      }
    }
    __syncthreads();
    u32 eb = 0, gb = 0, req = 0, y = 0;
    bool fits = true;
    u64 d = 0;
    if (valid) {
      y = cnt[threadIdx.x];
      if (a.node_last) {
        i64 lt = lt_old;
        if (y) {
          const i64 t = Payload<PV>::time(a.vals[lastq[threadIdx.x] - 1], a.tb);
          if (lt < t) lt = t;
        }
        if (a.old_last || y) a.node_last[v] = lt;
        d = lt < a.cutoff ? 1u : 0u;
      }
      const Ring oer = entry_ring(o), omr = mark_ring(o);
      if (implicit_marks(o)) {
        // single-entry groups (distinct times: the common case): marks are
        // not stored, mark k is entry k — search the entry times
        eb = evict_lb<8>([&](u32 x) { return a.oent[oer(x)].t; }, oer(o.eb), o.eb, o.ee, a.cutoff);
        gb = o.gb + (eb - o.eb);
      } else {
        // the first surviving mark starts the first surviving entry (a group
        // is evicted whole: eviction is by time), so one search over the
        // marks gives both bounds
        gb = evict_lb<8>([&](u32 x) { return a.omt[omr(x)]; }, omr(o.gb), o.gb, o.ge, a.cutoff);
        eb = gb == o.ge ? o.ee : a.oms[omr(gb)];
      }
      u32 low = o.eb;
      if (a.rnm && rm.base == o.base && rm.cap == o.cap) low = rm.eb;  // same ring: the retired snapshot reads [rm.eb, ..)
      // Logical positions are u32 and only rebased when a ring moves: a ring
      // that keeps fitting would otherwise count past 2^32 over a long
      // stream and break every [eb, ee) comparison, so it moves first.
      fits = !a.relocate_all && static_cast<u64>(o.ee - low) + y <= o.cap &&
             static_cast<u64>(o.ee) + y <= a.rebase_at;
      if (!fits) {
        const u32 need = (o.ee - eb) + y;
        req = 2 * need + 4;  // 2x slack: a typical ring absorbs ~10 batches before it moves
      }
      if (a.need_last && o.ee > eb) a.last_t[v] = a.oent[oer(o.ee - 1)].t;
    }
    u32 tot, mtot;
    const u32 off = block_excl_scan<u32>(req, &tot);
    const u32 midx = block_excl_scan<u32>(fits ? 0u : 1u, &mtot);
    if (threadIdx.x == 0) {
      s_base = tot ? atomicAdd(reinterpret_cast<unsigned long long*>(&a.scal[0]), static_cast<unsigned long long>(tot))
                   : 0ull;
      s_rbase = mtot ? atomicAdd(reinterpret_cast<unsigned int*>(&a.scal[2]), mtot) : 0u;
    }
    __syncthreads();
    if (valid) {
      if (fits) {
        a.plan[v] = NodeMeta{eb, o.ee, gb, o.ge, o.base, o.cap, adjust_org(o.eorg, eb, o.cap),
                             adjust_org(o.gorg, gb, o.cap)};
      } else {
        const u64 dst = s_base + off;
        if (dst + req > a.arena_cap) atomicOr(reinterpret_cast<unsigned long long*>(&a.scal[1]), 1ull);
        a.plan[v] = NodeMeta{0u, o.ee - eb, 0u, o.ge - gb, static_cast<u32>(dst), req, 0u, 0u};
        a.reloc[s_rbase + midx] = Reloc{static_cast<u32>(v), eb, gb};
      }
    }
    if (a.dead) block_atomic_add(reinterpret_cast<unsigned long long*>(a.dead), d);
    __syncthreads();
  }
}

// live entries and marks into the new rings (rebased to logical 0), one warp per ring
__global__ void k_reloc_copy(const Reloc* list, const u64* scal, const NodeMeta* onm, const NodeMeta* plan,
                             const Entry* oent, const i64* omt, const u32* oms, Entry* ent, i64* mt, u32* ms) {
  if (scal[1] | scal[13]) return;  // the plan failed (arena exhausted / a node leaves): queued speculatively
  const u64 n = scal[2] & 0xffffffffull;
  const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
  const u32 lane = threadIdx.x & 31;
  for (u64 k = (blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) >> 5; k < n; k += warps) {
    const Reloc r = list[k];
    const NodeMeta on = onm[r.v], p = plan[r.v];
    const Ring er = entry_ring(on), mr = mark_ring(on);
    for (u32 j = lane; j < p.ee; j += 32) ent[p.base + j] = oent[er(r.src_e + j)];
    if (p.ge == p.ee) continue;  // implicit marks (single-entry groups): nothing stored to copy
    for (u32 j = lane; j < p.ge; j += 32) {
      mt[p.base + j] = omt[mr(r.src_g + j)];
      ms[p.base + j] = oms[mr(r.src_g + j)] - r.src_e;
    }
  }
}

template <class PV>
struct PlaceArgs {
  u64 V;
  i64 tb;  // time base of PEnt payloads
  const NodeMeta* plan;
  const i64* last_t;
  const u32* keys;      // batch entries bucket-sorted (owner >> 8), canonical order inside a bucket
  const PV* vals;       // their node-view entries
  const u32* bstart;
  Entry* ent;
  i64* mt;
  u32* ms;
  NodeMeta* nm_new;
  WalkRec* wrec_new;
  const WalkRec* owrec;  // the previous snapshot's walk records (null: read its tail from the ring)
  u64* q_total;
  const u64* abort;  // the plan's scalars: [1] arena exhausted, [13] a node leaves the window -> do nothing
};

template <class PV>
struct PlaceSmem {  // ~47 KB with 12-B staged payloads, ~55 KB with 16-B ones (kChunk 2048)
  u16 wcnt[kPB / 32][kPB];  // chunk counts fit 16 bits (kChunk <= 65535)
  u32 off[kPB + 1];
  u32 cur[kPB], gcur[kPB], base[kPB], cap[kPB], eorg[kPB], gorg[kPB];
  i64 last_t[kPB];
  u32 has_last[kPB];
  u8 expl[kPB];  // node stores its marks (a repeated time in its region)
  u8 tie[kPB];   // this chunk holds an entry of the node that continues a group
  u32 mtotal;
  u32 rwcnt[kChunkItems][kPB / 32];
  u8 snode[kChunk];
  u8 flag[kChunk];
  u16 mscan[kChunk];
  PV sent[kChunk];  // the chunk's payloads in node order, as sorted (expanded to entries on the way out)
};
static_assert(kChunk < 65536, "16-bit chunk counters");
static_assert(sizeof(PlaceSmem<Entry>) <= 56 * 1024, "placement: 4 CTAs per SM (228 KB of shared memory)");

// One CTA per bucket of 256 nodes (thread t <-> node (bucket << 8) + t):
// the bucket's entries in rounds of kChunk: stable rank per node
// (warp-private match/ballot counters + cross-warp scan), records gathered
// and staged in node order in shared memory, mark flags + block scan, then
// written in node order (a node's new entries / marks are contiguous in its
// ring, so the stores coalesce); finally publish {eb, ee, gb, ge, ring}.
template <class PV>
__global__ void __launch_bounds__(kPB, TWG_PLACE_MINB) k_bucket_place(PlaceArgs<PV> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PlaceSmem<PV>& sm = *reinterpret_cast<PlaceSmem<PV>*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const u64 bkt = blockIdx.x;
  if (a.abort[1] | a.abort[13]) return;  // queued before the host saw the plan fail
  const u64 v = (bkt << kBucketShift) + t;
  const bool valid = v < a.V;
  const u32 bs = a.bstart[bkt], be = a.bstart[bkt + 1];
  // the first chunk's keys and payload prefetch go out before the plan row,
  // so the CTA's first DRAM round trips overlap
  // (item i = warp*R*32 + r*32 + lane of a chunk belongs to this lane in round r)
  u32 dk[kChunkItems];
  auto load_chunk = [&](u32 c0, u32 n) {
#pragma unroll
    for (int r = 0; r < kChunkItems; ++r) {  // the payloads' DRAM fetch starts now, into L2
      const u32 i = warp * (32 * kChunkItems) + r * 32 + lane;
      if (i < n) prefetch_l2(a.vals + c0 + i);
    }
#pragma unroll
    for (int r = 0; r < kChunkItems; ++r) {
      const u32 i = warp * (32 * kChunkItems) + r * 32 + lane;
      dk[r] = i < n ? (a.keys[c0 + i] & (kPB - 1)) : 0u;
    }
  };
  if (be > bs) load_chunk(bs, min(static_cast<u32>(kChunk), be - bs));
  NodeMeta p{};
  i64 lt_v = 0;
  if (valid) {  // independent loads, in flight together
    p = a.plan[v];
    if (a.last_t) lt_v = a.last_t[v];
  }
  sm.cur[t] = p.ee;
  sm.gcur[t] = p.ge;
  sm.base[t] = p.base;
  sm.cap[t] = p.cap;
  sm.eorg[t] = p.eorg;
  sm.gorg[t] = p.gorg;
  const bool has = valid && a.last_t && p.ee > p.eb && be > bs;
  sm.has_last[t] = has ? 1u : 0u;
  sm.last_t[t] = has ? lt_v : 0;
  sm.expl[t] = implicit_marks(p) ? 0 : 1;

  const u32 lt = (1u << lane) - 1u;
  for (u32 c0 = bs; c0 < be; c0 += kChunk) {
    const u32 n = min(static_cast<u32>(kChunk), be - c0);
    __syncthreads();
    if (c0 != bs) load_chunk(c0, n);  // later chunks (the first one is in flight since the start)
    for (int i = t; i < (kPB / 32) * kPB; i += kPB) (&sm.wcnt[0][0])[i] = 0;
    sm.tie[t] = 0;
    __syncthreads();
    // stable rank: warp w owns items [w*R*32, (w+1)*R*32) in R rounds of 32
    u32 rank[kChunkItems];
#pragma unroll
    for (int r = 0; r < kChunkItems; ++r) {
      const u32 i = warp * (32 * kChunkItems) + r * 32 + lane;
      const bool ok = i < n;
      const u32 d = dk[r];
      const u32 peers = digit_peers<kBucketShift>(d, ok);
      const u32 before = ok ? sm.wcnt[warp][d] : 0u;
      __syncwarp();
      if (ok && (__ffs(peers) - 1) == lane) sm.wcnt[warp][d] = static_cast<u16>(before + __popc(peers));
      __syncwarp();
      rank[r] = before + __popc(peers & lt);
    }
    __syncthreads();
    {  // per node: exclusive prefix across warps, node offset in the staged order
      u32 acc = 0;
#pragma unroll
      for (int w = 0; w < kPB / 32; ++w) {
        const u32 c = sm.wcnt[w][t];
        sm.wcnt[w][t] = static_cast<u16>(acc);
        acc += c;
      }
      u32 total;
      sm.off[t] = block_excl_scan<u32>(acc, &total);
      if (t == 0) sm.off[kPB] = total;
      // a node this batch gives fewer entries than the walk-record tail takes
      // the rest from the previous record: fetch its line into L2 now
      if (c0 == bs && valid && a.owrec && c0 + n >= be && acc < kWalkTail) prefetch_l2(a.owrec + v);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kChunkItems; ++r) {  // payloads loaded only now: not live across the ranking
      const u32 i = warp * (32 * kChunkItems) + r * 32 + lane;
      if (i < n) {
        const u32 nd = dk[r];
        const u32 sp = sm.off[nd] + sm.wcnt[warp][nd] + rank[r];
        sm.sent[sp] = a.vals[c0 + i];
        sm.snode[sp] = static_cast<u8>(nd);
      }
    }
    __syncthreads();
    // mark flags over the staged order; item i = r*256 + t (conflict-free
    // smem reads), prefixes from per-(round, warp) ballot counts
    u32 fl[kChunkItems];
#pragma unroll
    for (int r = 0; r < kChunkItems; ++r) {
      const u32 i = r * kPB + t;
      u32 f = 0;
      if (i < n) {
        const u32 nd = sm.snode[i];
        const i64 ti = Payload<PV>::time(sm.sent[i], a.tb);
        if (i == sm.off[nd]) f = (!sm.has_last[nd] || ti != sm.last_t[nd]) ? 1u : 0u;
        else f = ti != Payload<PV>::time(sm.sent[i - 1], a.tb) ? 1u : 0u;
        if (!f) sm.tie[nd] = 1;
      }
      fl[r] = __ballot_sync(0xffffffffu, f != 0);
      if (lane == 0) sm.rwcnt[r][warp] = __popc(fl[r]);
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the kChunkItems x 8 counts in item order
      constexpr int kCounts = kChunkItems * (kPB / 32);
      u32 carry = 0;
#pragma unroll
      for (int base = 0; base < kCounts; base += 32) {
        const int i = base + lane;
        const u32 c = i < kCounts ? (&sm.rwcnt[0][0])[i] : 0u;
        const u32 incl = warp_incl_scan(c);
        if (i < kCounts) (&sm.rwcnt[0][0])[i] = carry + incl - c;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) sm.mtotal = carry;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kChunkItems; ++r) {
      const u32 i = r * kPB + t;
      sm.mscan[i] = static_cast<u16>(sm.rwcnt[r][warp] + __popc(fl[r] & lt));
      sm.flag[i] = static_cast<u8>((fl[r] >> lane) & 1u);
    }
    if (sm.tie[t] && !sm.expl[t]) {
      // the node's region gets a repeated time: its marks become explicit —
      // store the implicit ones of everything placed so far (mark k = entry
      // k over [eb, cur)); rare (ties inside a node's region)
      const Ring er{sm.base[t], sm.cap[t], sm.eorg[t]}, mr{sm.base[t], sm.cap[t], sm.gorg[t]};
      for (u32 x = p.eb; x < sm.cur[t]; ++x) {
        const u32 g = p.gb + (x - p.eb);
        a.mt[mr(g)] = a.ent[er(x)].t;
        a.ms[mr(g)] = x;
      }
      sm.expl[t] = 1;
    }
    __syncthreads();
    // write out in staged (node) order
    for (u32 i = t; i < n; i += kPB) {
      const u32 nd = sm.snode[i];
      const u32 pos = sm.cur[nd] + (i - sm.off[nd]);
      const Ring er{sm.base[nd], sm.cap[nd], sm.eorg[nd]};
      const Entry e = Payload<PV>::entry(sm.sent[i], a.tb);
      a.ent[er(pos)] = e;
      if (sm.flag[i] && sm.expl[nd]) {
        const Ring mr{sm.base[nd], sm.cap[nd], sm.gorg[nd]};
        const u32 g = sm.gcur[nd] + (sm.mscan[i] - sm.mscan[sm.off[nd]]);
        a.mt[mr(g)] = e.t;
        a.ms[mr(g)] = pos;
      }
    }
    __syncthreads();
    {  // advance the node cursors
      const u32 o1 = sm.off[t], c = sm.off[t + 1] - o1;
      if (c) {
        const u32 mend = o1 + c < n ? sm.mscan[o1 + c] : sm.mtotal;
        sm.cur[t] += c;
        sm.gcur[t] += mend - sm.mscan[o1];
        sm.last_t[t] = Payload<PV>::time(sm.sent[o1 + c - 1], a.tb);
        sm.has_last[t] = 1u;
      }
    }
  }
  __syncthreads();

  u64 q = 0;
  if (valid) {
    const NodeMeta r{p.eb, sm.cur[t], p.gb, sm.gcur[t], p.base, p.cap, p.eorg, p.gorg};
    a.nm_new[v] = r;
    q = r.ge - r.gb;
    // the walk record; its tail (the newest entries, newest first) comes
    // from the last chunk still staged in shared memory, then from this
    // batch's earlier chunks (ring slots this CTA wrote, visible after the
    // barrier), then from the previous snapshot's record (or its ring)
    WalkRec w;
    w.eb = r.eb;
    w.ee = r.ee;
    w.base = r.base;
    w.cap = r.cap;
    w.eorg = r.eorg;
    w.g = r.ge - r.gb;
    w.pad = 0;
    const Ring er = entry_ring(r);
    const u32 total = r.ee - p.ee;  // this batch's entries of the node
    const u32 o1 = be > bs ? sm.off[t] : 0u, cl = be > bs ? sm.off[t + 1] - o1 : 0u;  // in the last chunk
    const u32 k = min(r.ee - r.eb, kWalkTail);
    WalkRec o;
    if (a.owrec && total < k) o = a.owrec[v];
#pragma unroll
    for (u32 i = 0; i < kWalkTail; ++i) {
      u32 nb = 0;
      i64 tj = 0;
      if (i < k) {
        if (i < cl || i < total) {
          const Entry e = i < cl ? Payload<PV>::entry(sm.sent[o1 + cl - 1 - i], a.tb) : a.ent[er(r.ee - 1 - i)];
          nb = e.nbr;
          tj = e.t;
        } else if (a.owrec) {
          const u32 j = i - total;
          nb = j == 0 ? o.nbr[0] : j == 1 ? o.nbr[1] : o.nbr[2];
          tj = j == 0 ? o.t[0] : j == 1 ? o.t[1] : o.t[2];
        } else {
          const Entry e = a.ent[entry_ring(p)(p.ee - 1 - (i - total))];
          nb = e.nbr;
          tj = e.t;
        }
      }
      if (i == 0) w.nbr[0] = nb, w.t[0] = tj;
      else if (i == 1) w.nbr[1] = nb, w.t[1] = tj;
      else w.nbr[2] = nb, w.t[2] = tj;
    }
    a.wrec_new[v] = w;
  }
  block_atomic_add(reinterpret_cast<unsigned long long*>(a.q_total), q);
}

// logical ring end beyond which a ring is rebased (TWG_RING_REBASE lowers it
// for tests; the default keeps every position below 2^31 + one batch)
u32 ring_rebase_at() {  // read per batch (one getenv), so a test can lower it mid-process
  const char* e = std::getenv("TWG_RING_REBASE");
  const unsigned long long x = e ? std::strtoull(e, nullptr, 10) : 0ull;
  return x ? static_cast<u32>(std::min<unsigned long long>(x, 0x80000000ull)) : 0x80000000u;
}

bool append_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TWG_APPEND");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

bool append_ingest_enabled() { return append_enabled(); }

// O's log can take A more edges (and up to A groups) in place: O is the
// log's newest slice, no snapshot older than the retired one holds it, and
// the ring slots the batch reuses lie before every live slice (O, and the
// retired R when it shares the log).
bool log_room(const Store& O, const Store* R, u64 A) {
  const EdgeLog* L = O.gapped ? O.log.get() : nullptr;
  if (!L || L->len != O.log_first + O.m) return false;
  const bool shared = R && R->gapped && R->log.get() == L;
  if (O.log.use_count() > (shared ? 2 : 1)) return false;
  const u64 lo = shared ? std::min(O.log_first, R->log_first) : O.log_first;
  const u64 zlo = shared ? std::min(O.ts_first, R->ts_first) : O.ts_first;
  return (L->len + A) - lo <= L->cap && (L->zlen + A) - zlo <= L->cap;
}

bool append_log_slot(const Store& O, const Store* R, u64 A, Ring* wr) {
  if (!log_room(O, R, A)) return false;
  *wr = log_ring(O.log->cap, O.log_first + O.m);  // == the new slice start (O.log_first + from) + survivors
  return true;
}

Store* ingest_append(Window& w, const Store& O, std::unique_ptr<Store> s, const EdgeRec* batch, Ring bring, u64 A,
                     u64 from, i64 cutoff, bool no_ties, bool in_log, bool check_dead, const i64* bt,
                     const i64* const* bcols, const u64* groups_done, i64 tbase, bool compact,
                     const i64* old_last, u32* pre_hist, const u32* pre_rows, const u32* stat_rows) {
  Ctx& ctx = *w.ctx;
  cudaStream_t st = ctx.stream;
  PhaseTimer pt(ctx, "ingest_append");
  const int mode = w.mode;
  const u64 S = O.m - from;
  const u64 m = S + A;
  const u64 V = s->V;
  const u64 sides = mode == TWG_UNDIRECTED ? 2 : 1;
  const u64 Yn = sides * A;
  s->P = sides * m;
  u64* sc = ctx.d_scalars + 32;  // 32..47 private to this path
  TWG_CUDA(cudaMemsetAsync(sc, 0, 16 * sizeof(u64), st));
  const u64* d_gcut = sc + 9;  // first surviving ts group of O
  k_lb_time<<<1, 32, 0, st>>>(O.ts_time.p, O.view().zrg, O.Z, cutoff, sc + 9);
  TWG_LAUNCHED(ctx);

  // 1. edge log + ts groups
  const Store* R = w.previous;
  const bool in_place = log_room(O, R, A);
  if (in_log && !in_place) fail(TWG_ECUDA, "ingest_append: batch staged in a log without room");
  std::shared_ptr<EdgeLog> log = in_place ? O.log : nullptr;
  const u32 seq0 = O.seq0 + static_cast<u32>(from);
  const u32 seq_b = seq0 + static_cast<u32>(S);
  const StoreView ov = O.view();
  u64 zbase = 0;
  const u64* zbase_dev = nullptr;
  if (in_place) {
    s->log_first = O.log_first + from;
    zbase = log->zlen;
  } else {  // a new log (first streaming batch, window growth, or an older snapshot holding the log)
    auto nl = std::make_shared<EdgeLog>();
    nl->cap = std::max<u64>((3 * m) / 2 + 2 * A, 1024);
    nl->rec.alloc(nl->cap, st);
    nl->ts_off.alloc(nl->cap, st);
    nl->ts_time.alloc(nl->cap, st);
    if (S) {
      k_copy_cols<<<grid(ctx, S), kBlock, 0, st>>>(ov, from, S, nl->rec.p);
      TWG_LAUNCHED(ctx);
    }
    if (O.Z) {
      k_copy_groups<<<grid(ctx, O.Z), kBlock, 0, st>>>(O.ts_off.p, O.ts_time.p, ov.zrg, O.Z, d_gcut, nl->ts_off.p,
                                                       nl->ts_time.p);
      TWG_LAUNCHED(ctx);
    }
    k_zbase<<<1, 1, 0, st>>>(O.Z, d_gcut, sc + 4);
    TWG_LAUNCHED(ctx);
    zbase_dev = sc + 4;
    nl->len = S;
    log = std::move(nl);
    s->log_first = 0;
  }
  const u64 lpos = s->log_first + S;  // logical log position of batch edge 0
  const Ring wr = log_ring(log->cap, lpos);
  if (!in_log) {  // the batch into the log ring (the fast route wrote it there already)
    k_append_batch<<<grid(ctx, A), kBlock, 0, st>>>(batch, bring, A, log->rec.p, wr);
    TWG_LAUNCHED(ctx);
  }
  const Rec* brec = log->rec.p;  // batch edge k at log slot wr(k) from here on
  const i64* last_surv = nullptr;  // the last survivor's time: the first batch group merges with it on a tie
  if (S) last_surv = O.gapped ? &O.e_rec.p[(O.log_first + O.m - 1) % O.log->cap].t : O.e_t.p + (O.m - 1);
  if (groups_done) {  // the statistics pass numbered and wrote them (fast route, batch in the log)
    if (!in_place || !in_log) fail(TWG_ECUDA, "ingest_append: ts groups staged without the log");
    TWG_CUDA(cudaMemcpyAsync(sc + 5, groups_done, sizeof(u64), cudaMemcpyDeviceToDevice, st));
  } else {
    scan_scatter(ctx, BatchGroupFn{brec, wr, last_surv, bt}, A, sc + 5,
                 BatchGroupScatter{brec, wr, seq_b, zbase % log->cap, zbase_dev, log->cap, log->ts_off.p,
                                   log->ts_time.p, bt});
  }
  pt.mark("log+ts");

  // 2.-3. with the compact 12-B payload when the batch's times span < 2^32
  std::shared_ptr<NodeArena> arena;
  u64 r[14];  // the closing read-back (sc[0..13])
  auto sort_and_place = [&](auto tag) -> bool {
    using PV = decltype(tag);
    // 2. batch entries grouped into 256-node buckets: stable radix sort of
    //    (owner, entry) pairs on the owner bits above the bucket (canonical
    //    order inside a bucket), bucket bounds
    const int vb = V > 1 ? bit_width_u64(V - 1) : 0;
    const u64 nb = (V + kPB - 1) / kPB;
    DevBuf<u32> k0(Yn, st), k1(Yn, st);
    DevBuf<PV> v0(Yn, st), v1(Yn, st);
    u32* kp = k0.p;
    u32* ka = k1.p;
    PV* vp = v0.p;
    PV* va = v1.p;
    if (vb > static_cast<int>(kBucketShift)) {  // the first pass builds (owner, entry) from the log records
      OwnerIn<PV> oin{brec, wr, mode, seq_b, tbase};
      oin.bs = bcols ? bcols[0] : nullptr;
      oin.bd = bcols ? bcols[1] : nullptr;
      radix_sort_pairs_from<u32, PV>(ctx, oin, &kp, &ka, &vp, &va, Yn, vb, kBucketShift, pre_hist,
                                     pre_rows, (mode != TWG_UNDIRECTED && oin.bs) ? stat_rows : nullptr);
    } else {
      k_owner_keys<PV><<<grid(ctx, Yn), kBlock, 0, st>>>(brec, wr, A, mode, seq_b, tbase, kp, vp);
      TWG_LAUNCHED(ctx);
    }
    DevBuf<u32> bstart(nb + 1, st);
    k_bucket_bounds<<<grid(ctx, (Yn + TWG_BOUNDS_KEYS) / TWG_BOUNDS_KEYS), kBlock, 0, st>>>(kp, Yn, nb, bstart.p);
    TWG_LAUNCHED(ctx);
    (kp == k0.p ? k1 : k0).release();  // the pass count decides which buffer holds the result
    (vp == v0.p ? v1 : v0).release();
    pt.mark("bucket_sort");

    // 3. per node: eviction, ring room / relocation; then per bucket:
    //    placement, marks, publish
    s->nm.alloc(V, st);
    s->wrec.alloc(V, st);
    // fast route: the population must not shrink — the dead count (sc[13]) is
    // read back with the plan's scalars; nothing is published before
    bool dead = false;
    arena = O.gapped ? O.arena : nullptr;
    // a snapshot older than the retired one still holding this arena may read
    // any slot: then nothing of it is reused (fresh arena)
    if (arena) {
      const long expected = 2 + ((R && R->gapped && R->arena == arena) ? 1 : 0);  // O, R, this local copy
      if (arena.use_count() > expected) arena.reset();
    }
    DevBuf<NodeMeta> plan(V, st);
    DevBuf<i64> last_t(V, st);
    DevBuf<Reloc> reloc(V, st);
    // run_plan: k_plan into dst; with readback, its scalars come back at once
    // (relocations + 1, 0 = exhausted; `dead` set when the population would
    // shrink), else the closing read-back below collects them
    auto run_plan = [&](NodeArena& dst, bool all, bool readback) -> u64 {
      TWG_CUDA(cudaMemsetAsync(sc, 0, 3 * sizeof(u64), st));
      if (check_dead) TWG_CUDA(cudaMemsetAsync(sc + 13, 0, sizeof(u64), st));
      TWG_CUDA(cudaMemcpyAsync(sc, &dst.used, sizeof(u64), cudaMemcpyHostToDevice, st));
      PlanArgs<PV> pa;
      pa.onm = O.nm.p;
      pa.rnm = (!all && R && R->gapped && R->arena.get() == &dst) ? R->nm.p : nullptr;
      pa.V = V;
      pa.oent = O.ent.p;
      pa.omt = O.mk_time.p;
      pa.oms = O.mk_start.p;
      pa.keys = kp;
      pa.vals = vp;
      pa.bstart = bstart.p;
      pa.tb = tbase;
      pa.old_last = old_last;
      pa.node_last = s->last_t.p;
      pa.dead = check_dead ? sc + 13 : nullptr;
      pa.need_last = no_ties ? 0 : 1;
      pa.cutoff = cutoff;
      pa.relocate_all = all ? 1 : 0;
      pa.rebase_at = ring_rebase_at();
      pa.arena_cap = dst.cap;
      pa.plan = plan.p;
      pa.last_t = last_t.p;
      pa.reloc = reloc.p;
      pa.scal = sc;
      k_plan<PV><<<grid(ctx, V), kBlock, 0, st>>>(pa);
      TWG_LAUNCHED(ctx);
      if (!readback) return 0;
      u64 r3[14];
      read_scalars(ctx, sc, r3, check_dead ? 14 : 3);
      if (check_dead && r3[13]) {
        dead = true;
        return u64{1};
      }
      dst.used = r3[0];
      return r3[1] == 0 ? static_cast<u64>(r3[2] & 0xffffffffull) + 1 : 0;  // relocations + 1, 0 = exhausted
    };
    static bool attr_set = false;
    if (!attr_set) {
      TWG_CUDA(cudaFuncSetAttribute(k_bucket_place<Entry>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(sizeof(PlaceSmem<Entry>))));
      TWG_CUDA(cudaFuncSetAttribute(k_bucket_place<PEnt>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(sizeof(PlaceSmem<PEnt>))));
      attr_set = true;
    }
    // relocation copies (count read on the device: sc[2]) and the placement;
    // both return at once when the plan failed (sc[1]: arena exhausted,
    // sc[13]: a node leaves the window), so they can be queued before the
    // plan's scalars are known
    auto copy_and_place = [&](NodeArena& ar, u64 rel_bound) {
      k_reloc_copy<<<grid(ctx, 32 * std::max<u64>(rel_bound, 1)), kBlock, 0, st>>>(
          reloc.p, sc, O.nm.p, plan.p, O.ent.p, O.mk_time.p, O.mk_start.p, ar.ent.p, ar.mk_time.p, ar.mk_start.p);
      TWG_LAUNCHED(ctx);
      PlaceArgs<PV> pl;
      pl.V = V;
      pl.tb = tbase;
      pl.plan = plan.p;
      pl.last_t = no_ties ? nullptr : last_t.p;
      pl.keys = kp;
      pl.vals = vp;
      pl.bstart = bstart.p;
      pl.ent = ar.ent.p;
      pl.mt = ar.mk_time.p;
      pl.ms = ar.mk_start.p;
      pl.nm_new = s->nm.p;
      pl.wrec_new = s->wrec.p;
      pl.owrec = O.wrec.n >= V ? O.wrec.p : nullptr;
      pl.q_total = sc + 7;
      pl.abort = sc;
      TWG_CUDA(cudaMemsetAsync(sc + 7, 0, sizeof(u64), st));
      k_bucket_place<PV><<<static_cast<unsigned>(nb), kPB, sizeof(PlaceSmem<PV>), st>>>(pl);
      TWG_LAUNCHED(ctx);
    };
    // the closing read-back: the plan's scalars [0..2], [13] with g_cut,
    // batch groups, marks, Q [5..8]
    auto closing = [&]() {
      TWG_CUDA(cudaMemcpyAsync(sc + 8, d_gcut, sizeof(u64), cudaMemcpyDeviceToDevice, st));
      read_scalars(ctx, sc, r, 14);
    };
    auto fresh_arena = [&]() -> bool {  // every ring relocated into a new arena (synchronous plan)
      auto na = std::make_shared<NodeArena>();
      static std::atomic<u64> serials{0};
      na->serial = ++serials;
      na->V = V;
      // >= 2 P + 4 V: the repack fits (TWG_ARENA_TIGHT=1, for tests: exactly that, so later
      // batches exhaust it and take the speculative plan's exhausted path)
      const char* tight = std::getenv("TWG_ARENA_TIGHT");
      na->cap = std::min<u64>((tight && tight[0] == '1') ? 2 * s->P + 4 * V + 1024 : (5 * s->P) / 2 + 12 * V + 1024,
                              0xffffff00ull);
      na->ent.alloc(na->cap, st);
      na->mk_time.alloc(na->cap, st);
      na->mk_start.alloc(na->cap, st);
      na->used = 0;
      arena = std::move(na);
      const u64 n1 = run_plan(*arena, true, true);
      if (dead) return false;
      if (n1 == 0) fail(TWG_ENOMEM, "ingest: node arena sized below the live regions");
      copy_and_place(*arena, n1 - 1);
      closing();
      return true;
    };
    bool fresh = false;
    u64 nrel = 0;
    if (arena) {  // speculative: plan, copies and placement queued back to back, one read-back
      run_plan(*arena, false, false);
      copy_and_place(*arena, 4096);  // grid-stride over the device's relocation count
      closing();
      if (check_dead && r[13]) return false;
      if (r[1] == 0) {
        arena->used = r[0];
        nrel = r[2] & 0xffffffffull;
      } else {  // the arena is exhausted: the queued copies and placement did nothing
        if (!fresh_arena()) return false;
        fresh = true;
        nrel = r[2] & 0xffffffffull;
        arena->used = r[0];
      }
    } else {
      if (!fresh_arena()) return false;
      fresh = true;
      nrel = r[2] & 0xffffffffull;
      arena->used = r[0];
    }
    s->relocated = nrel;
    reloc.release();
    pt.mark(fresh ? "plan+place+repack" : "plan+place");
    if (pt.on) std::fprintf(stderr, "[twg phases] relocated rings: %llu of %llu\n", static_cast<unsigned long long>(nrel),
                            static_cast<unsigned long long>(V));
    return true;
  };
  if (!(compact ? sort_and_place(PEnt{}) : sort_and_place(Entry{}))) return nullptr;
  const u64 Zb = r[5], Q = r[7], g_cut = r[8];
  const u64 Z = (O.Z - g_cut) + Zb;
  s->ts_first = in_place ? O.ts_first + g_cut : 0;
  log->len = lpos + A;
  log->zlen = s->ts_first + Z;

  s->gapped = true;
  s->seq0 = seq0;
  s->m = m;
  s->Z = Z;
  s->Q = Q;
  s->e_rec.alias(log->rec.p, log->cap);
  s->ts_off.alias(log->ts_off.p, log->cap);
  s->ts_time.alias(log->ts_time.p, log->cap);
  const Ring er = log_ring(log->cap, s->log_first), zr = log_ring(log->cap, s->ts_first);
  s->e_cap = er.cap;
  s->e_org = er.org;
  s->z_cap = zr.cap;
  s->z_org = zr.org;
  s->ent.alias(arena->ent.p, arena->cap);
  s->mk_time.alias(arena->mk_time.p, arena->cap);
  s->mk_start.alias(arena->mk_start.p, arena->cap);
  s->log = std::move(log);
  s->arena = std::move(arena);
  s->has_weights = false;
  s->has_adjacency = false;
  return s.release();
}

}  // namespace twg
