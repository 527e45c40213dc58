// WindowManager on the device (window_manager.cpp:9-69), streaming design.
//
// Semantics are the reference's: batch_high / new_high / cutoff_for
// (window_manager.cpp:30-33, .hpp:51-53); survivors = the time-sorted suffix
// at lower_bound(time, cutoff) (export_suffix, edge_store.cpp:325-332);
// batch edges with t >= cutoff admitted, the rest dropped_late (:39-46);
// the snapshot is rebuilt with re-densified ids (edge_store.cpp:57-89) and
// exactly one retired snapshot is kept (:56-57).
//
// What changes is the cost: instead of re-sorting the whole window
// (O(W log W) per batch, the reference's and our v1 path), only the batch is
// sorted and then MERGED into the survivors, which are already in canonical
// order:
//   1. ids: presence flags over the external-id range from (a) the old nodes
//      still referenced by a survivor and (b) admitted batch endpoints; an
//      exclusive scan gives the new dense ids (= ranks, as the reference);
//      old->new id table for the survivors.
//   2. canonical order: radix sort of the admitted batch by (t, src, dst),
//      merge-path merge with the survivors -> new edge columns + the new
//      position of every survivor / batch edge.
//   3. node view: the old node view's surviving entries (a suffix of every
//      region) keep their order; re-keyed (new owner, new position) they are
//      merged with the batch's entries (stable-sorted by owner) -> the new
//      node view with payloads carried, no gathers.
//   4. marks / offsets / ts view by flag + scan as in the full build.
// Ids outside the dense fast path (huge or sparse external ids) take the v1
// route: gather survivors back to external ids and run the full build.
#include <chrono>

#include "primitives.cuh"
#include "window.cuh"

namespace twg {

namespace {

constexpr int kBlock = 256;

unsigned grid(Ctx& ctx, u64 n) { return grid_for(n, kBlock, static_cast<unsigned>(ctx.sm_count) * 16); }

// scal: [0] batch max t (i64), [1] max non-negative id, [2] from, [3] admitted, [4] admitted negative id flag,
//       [5] V_new, [6] max present id
__global__ void k_init_scalars(u64* s) {
  reinterpret_cast<i64*>(s)[0] = kTimeUnset;
  for (int i = 1; i < 10; ++i) s[i] = 0;
  reinterpret_cast<i64*>(s)[8] = kTimeInfinite;
}

// scal[7]: bit0 = batch not time-ordered, bit1 = some equal-time run > kSegMax
constexpr int kSegMax = 32;

// the fast append route's speculative work, prepared before the statistics pass
struct FastSpec {
  bool on = false, in_log = false;
  Ring wring{0u, kIdentityCap, 0u};
  DevBuf<EdgeRec> tmp;
  EdgeRec* rec = nullptr;
  u64 from = 0;
  const i64* bt = nullptr;  // the batch's time column (device): equals the canonical order's times
  const i64* cols[2] = {nullptr, nullptr};  // its source / target columns (input order)
  DevBuf<u64> ts_state;  // look-back words of the statistics pass's ts-group numbering
  bool groups = false;   // the statistics pass wrote the batch's ts groups into the log (total: d_scalars[14])
  DevBuf<u32> hist_rows, hist;  // the fused owner-digit histogram (rows per tile, their sum)
  DevBuf<u32> hist_csum;        // k_hist_rows' per-block sums, then their exclusive prefixes (rows_pre)
  bool rows_pre = false;        // the first bucket-sort pass takes its offsets from hist_csum + hist_rows
};

// scal[8]: batch min t, scal[9]: some id negative.
// rec != null: speculatively also emit the canonical records of a
// time-ordered batch (each edge ranked by (src, dst) inside its equal-time
// run, runs scanned up to kSegMax each way) through the ring wr — used only
// when the statistics admit the fast append route, ignored otherwise.
//
// Tiled: a CTA stages kStatTile edges plus a kSegMax halo on each side in
// shared memory with coalesced column loads (24 B per edge read once from
// HBM; every load of the tile issued before the first shared store), then
// every edge finds its run and its rank from shared memory.
//
// kGroups: the same pass also writes the batch's timestamp groups (the
// append route's step 1, otherwise a second read of the time column): a
// group starts at every edge whose time differs from its predecessor's —
// and at edge 0, since the fast route admits only batches strictly newer
// than the window — numbered by a decoupled look-back over tiles taken by
// ticket, written as {start sequence, time} through the log's ts ring.
#ifndef TWG_STAT_ITEMS
#define TWG_STAT_ITEMS 6
#endif
constexpr int kStatItems = TWG_STAT_ITEMS;
constexpr int kStatTile = kBlock * kStatItems;
constexpr int kStatSpan = kStatTile + 2 * kSegMax;
static_assert(kStatSpan % 32 == 0 && kSegMax == 32, "span words and the one-word run-bound search");

bool compact_payload_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TWG_COMPACT_PAYLOAD");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool stats_hist_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TWG_STATS_HIST");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool sort_pre_enabled() {  // TWG_SORT_PRE=0: the first bucket-sort pass resolves its offsets by look-back
  static const bool on = [] {
    const char* e = std::getenv("TWG_SORT_PRE");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool stats_groups_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TWG_STATS_GROUPS");
    return !(e && e[0] == '0');
  }();
  return on;
}

struct TsSpec {
  u64* tile_state;  // tiles + 1 words, zeroed (the last one is the ticket)
  u32* ts_off;
  i64* ts_time;
  u64 zbase;        // ring slot of the batch's first group (< cap)
  u64 cap;
  u32 seq_b;        // sequence number of batch edge 0
  u64* total;       // groups of the batch
};

// shared memory of one statistics tile: the span's three columns as they
// lie in HBM (i64), staged by TMA bulk copies
struct StatSmem {
  i64 t[kStatSpan], a[kStatSpan], b[kStatSpan];
};

// the owner-digit histogram of the bucket sort, fused (fast route): per tile
// one row of 2 x 256 counts (digits of bits 8-15 and 16-23 of each entry's
// owner), summed by k_hist_rows
struct HistSpec {
  u32* rows;   // null: not fused
  int passes;  // 1 or 2
  int mode;    // direction mode: which endpoint(s) own the entries
};

template <bool kGroups>
__global__ void __launch_bounds__(kBlock) k_batch_stats(const i64* bs, const i64* bd, const i64* bt, u64 n, u64* scal,
                                                        EdgeRec* rec, Ring wr, TsSpec ts, HistSpec hs) {
  extern __shared__ __align__(128) unsigned char stat_smem[];
  StatSmem& S = *reinterpret_cast<StatSmem*>(stat_smem);
  i64* st_t = S.t;
  i64* st_a = S.a;
  i64* st_b = S.b;
  __shared__ u32 s_tile;
  __shared__ u32 s_cnt[kStatItems][kBlock / 32];
  __shared__ u64 s_prefix;
  __shared__ alignas(8) u64 s_bar;
  __shared__ u32 s_hist[2][kRadix];
  __shared__ u32 s_start[kStatSpan / 32];  // bit j: an equal-time run starts at span position j
  static_assert(kBlock == kRadix, "one histogram bin per thread");
  const bool fuse_hist = kGroups && hs.rows != nullptr;
  if (fuse_hist) s_hist[0][threadIdx.x] = 0, s_hist[1][threadIdx.x] = 0;  // kBlock == kRadix
  i64 mt = kTimeUnset, lt = kTimeInfinite;
  u64 mid = 0;
  u32 shape = 0, neg = 0;
  if (kGroups) {
    if (threadIdx.x == 0) s_tile = atomicAdd(reinterpret_cast<u32*>(ts.tile_state + gridDim.x), 1u);
    __syncthreads();
  }
  const u64 tile = kGroups ? s_tile : blockIdx.x;
  const u64 base = tile * kStatTile;
  const i64 lo_g = static_cast<i64>(base) - kSegMax;  // global index of st_*[0]
  // interior tiles (the whole span inside the batch, 16-B aligned columns):
  // three 1-D TMA bulk copies; the first and last tiles: per-thread loads
  const bool bulk = lo_g >= 0 && static_cast<u64>(lo_g) + kStatSpan <= n &&
                    ((reinterpret_cast<uintptr_t>(bt) | reinterpret_cast<uintptr_t>(bs) |
                      reinterpret_cast<uintptr_t>(bd)) & 15) == 0;
  if (bulk) {
    constexpr u32 kBytes = kStatSpan * sizeof(i64);
    static_assert(kBytes % 16 == 0, "bulk copy size");
    if (threadIdx.x == 0) {
      mbar_init(&s_bar, 1);
      mbar_arrive_expect_tx(&s_bar, 3 * kBytes);
      bulk_g2s(st_t, bt + lo_g, kBytes, &s_bar);
      bulk_g2s(st_a, bs + lo_g, kBytes, &s_bar);
      bulk_g2s(st_b, bd + lo_g, kBytes, &s_bar);
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    mbar_wait(&s_bar, 0);
  } else {
    for (int j = threadIdx.x; j < kStatSpan; j += kBlock) {
      const i64 g = lo_g + j;
      if (g >= 0 && static_cast<u64>(g) < n) {
        st_t[j] = bt[g];
        st_a[j] = bs[g];
        st_b[j] = bd[g];
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 jn = static_cast<i64>(n) - lo_g;
  const int jmin = lo_g < 0 ? static_cast<int>(-lo_g) : 0;            // span index of edge 0
  const int jend = jn < kStatSpan ? static_cast<int>(jn) : kStatSpan;  // of edge n (clamped)
  // run starts as a bitmask over the span (one ballot per 32 positions);
  // edge 0 and everything outside [jmin, jend) count as starts, so a run's
  // bounds never leave the staged edges
  // (the same pass flags a descending pair (j-1, j) of this tile's own edges:
  // the batch is not time-ordered)
  for (int w0 = warp * 32; w0 < kStatSpan; w0 += kBlock) {
    const int j = w0 + lane;
    bool f = true;
    if (j > jmin && j < jend) {
      const i64 tj = st_t[j], tp = st_t[j - 1];
      f = tj != tp;
      if (tj < tp && j > kSegMax && j <= kSegMax + kStatTile) shape |= 1u;
    }
    const u32 word = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_start[w0 >> 5] = word;
  }
  __syncthreads();
  u32 gbal[kStatItems];
  if (kGroups) {
    // group starts = run starts of the tile's own edges; the tile's count is
    // posted at once: the successors' look-backs wait on it while this tile
    // ranks its runs
#pragma unroll
    for (int k = 0; k < kStatItems; ++k) {
      const u64 i0 = base + k * kBlock + warp * 32;  // edge of lane 0
      const u32 valid = i0 >= n ? 0u : (n - i0 >= 32 ? 0xffffffffu : (1u << (n - i0)) - 1u);
      gbal[k] = s_start[(kSegMax + k * kBlock) / 32 + warp] & valid;
      if (lane == 0) s_cnt[k][warp] = __popc(gbal[k]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // exclusive offsets of (round, warp) in position order
      u32 acc = 0;
      for (int k = 0; k < kStatItems; ++k)
        for (int w = 0; w < kBlock / 32; ++w) {
          const u32 c = s_cnt[k][w];
          s_cnt[k][w] = acc;
          acc += c;
        }
      s_prefix = acc;
      lb_store(ts.tile_state + tile, (tile == 0 ? kLbInclusive : kLbAggregate) | acc);
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < kStatItems; ++k) {
    const int j = kSegMax + k * kBlock + threadIdx.x;  // smem index of edge i
    const u64 i = base + k * kBlock + threadIdx.x;
    if (i >= n) continue;
    const i64 t = st_t[j];
    {  // this tile's own edges: statistics
      const i64 a = st_a[j], b = st_b[j];
      mt = max(mt, t);
      lt = min(lt, t);
      if (a > 0) mid = max(mid, static_cast<u64>(a));
      if (b > 0) mid = max(mid, static_cast<u64>(b));
      if (a < 0 || b < 0) neg = 1;
      if (fuse_hist) {
        const u32 o1 = static_cast<u32>(hs.mode == TWG_BACKWARD ? b : a);
        atomicAdd(&s_hist[0][(o1 >> 8) & (kRadix - 1)], 1u);
        if (hs.passes > 1) atomicAdd(&s_hist[1][(o1 >> 16) & (kRadix - 1)], 1u);
        if (hs.mode == TWG_UNDIRECTED) {
          const u32 o2 = static_cast<u32>(b);
          atomicAdd(&s_hist[0][(o2 >> 8) & (kRadix - 1)], 1u);
          if (hs.passes > 1) atomicAdd(&s_hist[1][(o2 >> 16) & (kRadix - 1)], 1u);
        }
      }
    }
    if (i + kSegMax < n && t == st_t[j + kSegMax]) shape |= 2u;
    if (rec) {
      // the run [lo, hi) around j from the start bitmask: the last start at
      // or before j, the first after it, each within one word either side (a
      // run longer than kSegMax sets shape bit 1; its records are not used)
      const int w = j >> 5, b = j & 31;
      const u32 upto = 0xffffffffu >> (31 - b);  // bits 0..b
      u32 m = s_start[w] & upto;
      int lo, hi;
      if (m) {
        lo = (w << 5) + 31 - __clz(m);
      } else {
        m = s_start[w - 1];
        lo = m ? ((w - 1) << 5) + 31 - __clz(m) : j - (kSegMax - 1);
      }
      m = s_start[w] & ~upto;
      if (m) {
        hi = (w << 5) + __ffs(m) - 1;
      } else {
        m = w + 1 < kStatSpan / 32 ? s_start[w + 1] : 1u;
        hi = m ? ((w + 1) << 5) + __ffs(m) - 1 : j + kSegMax;
      }
      // ids below 2^32 (the fast route's dense population): the low words of
      // the staged i64 columns (32-bit shared loads, little-endian)
      const u32* a32 = reinterpret_cast<const u32*>(st_a);
      const u32* b32 = reinterpret_cast<const u32*>(st_b);
      const u32 aj = a32[2 * j], bj = b32[2 * j];
      const u64 key = (static_cast<u64>(aj) << 32) | bj;
      u32 rank = 0;
      for (int q = lo; q < hi; ++q) {
        const u64 kq = (static_cast<u64>(a32[2 * q]) << 32) | b32[2 * q];
        rank += (kq < key || (kq == key && q < j)) ? 1u : 0u;
      }
      rec[wr(static_cast<u32>(lo_g + lo + rank))] = EdgeRec{aj, bj, t};
    }
  }
  if (kGroups) {
    if (warp == 0) {  // warp-parallel decoupled look-back (as k_scan_scatter)
      const u64 agg = s_prefix;
      u64* st = ts.tile_state;
      u64 prefix = 0;
      if (tile > 0) {
        long long p = static_cast<long long>(tile) - 1;
        while (true) {
          const long long idx = p - lane;
          u64 sv = kLbInclusive;
          if (idx >= 0) {
            do {
              sv = lb_load(st + idx);
            } while ((sv >> 62) == 0);
          }
          const u32 incl = __ballot_sync(0xffffffffu, (sv >> 62) == 2);
          const int stop = incl ? __ffs(incl) - 1 : 31;
          u64 v = lane <= stop ? (sv & kLbValueMask) : 0;
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          prefix += v;
          if (incl) break;
          p -= 32;
        }
        if (lane == 0) lb_store(st + tile, kLbInclusive | (prefix + agg));
      }
      __syncwarp();
      if (lane == 0) {
        if (base + kStatTile >= n) *ts.total = prefix + agg;
        s_prefix = prefix;
      }
    }
    __syncthreads();
    const u64 pre = s_prefix;
    const u32 lt32 = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < kStatItems; ++k) {
      if (!(gbal[k] >> lane & 1u)) continue;
      const int j = kSegMax + k * kBlock + threadIdx.x;
      const u64 i = base + k * kBlock + threadIdx.x;
      const u64 x = ts.zbase + pre + s_cnt[k][warp] + __popc(gbal[k] & lt32);
      const u64 z = x >= ts.cap ? x - ts.cap : x;
      ts.ts_off[z] = ts.seq_b + static_cast<u32>(i);
      ts.ts_time[z] = st_t[j];
    }
  }
  if (fuse_hist) {
    __syncthreads();
    hs.rows[tile * 512 + threadIdx.x] = s_hist[0][threadIdx.x];
    hs.rows[tile * 512 + kRadix + threadIdx.x] = s_hist[1][threadIdx.x];
  }
  // one set of atomics per block (the whole grid finishes at once: per-warp
  // atomics on these words would serialise at L2); signed times through the
  // order-preserving flip of the sign bit
  const u64 kSign = 1ull << 63;
  const u64 bmt = block_reduce_u64<1>(static_cast<u64>(mt) ^ kSign);
  const u64 blt = block_reduce_u64<2>(static_cast<u64>(lt) ^ kSign);
  const u64 bmid = block_reduce_u64<1>(mid);
  const u64 bflags = block_reduce_u64<3>(static_cast<u64>(shape) | (static_cast<u64>(neg) << 32));
  if (threadIdx.x == 0) {
    atomicMax(reinterpret_cast<long long*>(&scal[0]), static_cast<long long>(bmt ^ kSign));
    atomicMin(reinterpret_cast<long long*>(&scal[8]), static_cast<long long>(blt ^ kSign));
    atomicMax(reinterpret_cast<unsigned long long*>(&scal[1]), bmid);
    if (bflags & 0xffffffffull) atomicOr(reinterpret_cast<unsigned long long*>(&scal[7]), bflags & 0xffffffffull);
    if (bflags >> 32) atomicOr(reinterpret_cast<unsigned long long*>(&scal[9]), 1ull);
  }
}

// lower_bound of the cutoff implied by the batch maximum (scal[0]) over a snapshot's edges
__global__ void k_lower_bound_cut(StoreView s, i64 t_high, i64 duration, const u64* scal, u64* out) {
  const i64 bh = static_cast<i64>(scal[0]);
  const i64 high = t_high > bh ? t_high : bh;
  const i64 cutoff = high > duration ? high - duration : 0;
  const u64 r = warp_lower_bound([&](u64 k) { return edge_time(s, k); }, s.m, cutoff);
  if (threadIdx.x == 0) *out = r;
}

// Canonical order of a time-ordered batch whose equal-time runs are short
// (the common streaming case): sort each run by (src, dst) in registers —
// one thread per run — instead of a 72-bit LSD radix sort.
__global__ void k_segment_sort(const u32* s, const u32* d, const i64* t, u64 A, u32* os, u32* od, i64* ot) {
  for (u64 k = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; k < A;
       k += static_cast<u64>(gridDim.x) * blockDim.x) {
    const i64 tk = t[k];
    if (k > 0 && t[k - 1] == tk) continue;
    u64 key[kSegMax];
    int len = 0;
    while (len < kSegMax && k + len < A && t[k + len] == tk) {
      u64 x = (static_cast<u64>(s[k + len]) << 32) | d[k + len];
      int j = len++;
      while (j > 0 && key[j - 1] > x) {  // insertion sort (stable for equal keys: content-equal)
        key[j] = key[j - 1];
        --j;
      }
      key[j] = x;
    }
    for (int j = 0; j < len; ++j) {
      os[k + j] = static_cast<u32>(key[j] >> 32);
      od[k + j] = static_cast<u32>(key[j]);
      ot[k + j] = tk;
    }
  }
}



__global__ void k_pack_rec(const u32* s, const u32* d, const i64* t, u64 n, EdgeRec* out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    out[i] = EdgeRec{s[i], d[i], t[i]};
}

// lower_bound(time_, cutoff) (edge_store.cpp:326) over the snapshot's edges
__global__ void k_lower_bound(StoreView s, i64 cutoff, u64* out) {
  const u64 r = warp_lower_bound([&](u64 k) { return edge_time(s, k); }, s.m, cutoff);
  if (threadIdx.x == 0) *out = r;
}

struct AdmitFn {
  const i64* t;
  i64 cutoff;
  __device__ __forceinline__ u32 operator()(u64 i) const { return t[i] >= cutoff ? 1u : 0u; }
};

__global__ void k_admitted_neg(const i64* bs, const i64* bd, const i64* bt, u64 n, i64 cutoff, u64* flag) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    if (bt[i] >= cutoff && (bs[i] < 0 || bd[i] < 0)) atomicOr(reinterpret_cast<unsigned long long*>(flag), 1ull);
}

// ---- v1 route (full rebuild) -------------------------------------------------

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

// ---- streaming route ---------------------------------------------------------------


// old node v is an endpoint of a surviving edge iff its newest incident
// edge is not evicted (all of v's edges are in the old window)
__global__ void k_alive_from_last(const i64* last, u64 V, i64 cutoff, u8* alive) {
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<u64>(gridDim.x) * blockDim.x)
    alive[v] = last[v] >= cutoff ? 1 : 0;
}

// exact newest incident time of every node of a snapshot (over all its edges)
__global__ void k_store_last_t(StoreView s, i64* last) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < s.m;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const EdgeRec r = edge_at(s, i);
    if (last[r.src] < r.t) atomicMax(reinterpret_cast<long long*>(last + r.src), static_cast<long long>(r.t));
    if (last[r.dst] < r.t) atomicMax(reinterpret_cast<long long*>(last + r.dst), static_cast<long long>(r.t));
  }
}

__global__ void k_carry_last_t(const i64* old_last, const u8* alive, const u32* o2n, u64 V, i64* new_last) {
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<u64>(gridDim.x) * blockDim.x)
    if (alive[v]) new_last[o2n[v]] = old_last[v];
}

// max-combine (node, t) pairs of a warp before touching memory: hub nodes
// (dst = floor(N u^3) puts ~0.5% of a batch on node 0) otherwise serialise
// in the L2 atomic unit
// time_ordered: lanes hold non-decreasing times, so the highest peer lane
// carries the group's max and is the only one to touch memory
template <bool kTimeOrdered>
__device__ __forceinline__ void agg_max(i64* last, u32 key, i64 t, bool valid) {
  const u32 peers = __match_any_sync(0xffffffffu, valid ? key : 0xffffffffu);
  i64 m = t;
  int leader;
  if (kTimeOrdered) {
    leader = 31 - __clz(peers);
  } else {
#pragma unroll
    for (int src = 0; src < 32; ++src) {
      const i64 v = __shfl_sync(0xffffffffu, t, src);
      if ((peers >> src) & 1u) m = v > m ? v : m;
    }
    leader = __ffs(peers) - 1;
  }
  if (valid && leader == static_cast<int>(threadIdx.x & 31) && last[key] < m)
    atomicMax(reinterpret_cast<long long*>(last + key), static_cast<long long>(m));
}

template <bool kTimeOrdered>
__global__ void k_batch_last_t(const u32* s, const u32* d, const i64* t, u64 m, i64* last) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < ((m + 31) & ~31ull);
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const bool valid = i < m;
    const i64 ti = valid ? t[i] : 0;
    agg_max<kTimeOrdered>(last, valid ? s[i] : 0u, ti, valid);
    agg_max<kTimeOrdered>(last, valid ? d[i] : 0u, ti, valid);
  }
}

// present[ext[v]] for the old nodes still referenced; counts them
// (scal[0] max present id, scal[4] alive count)
__global__ void k_present_old(const u8* alive, const i64* ext, u64 V, u8* present, u64* scal) {
  u64 mx = 0, cnt = 0;
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<u64>(gridDim.x) * blockDim.x) {
    if (alive[v]) {
      present[ext[v]] = 1;
      mx = max(mx, static_cast<u64>(ext[v]));
      ++cnt;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (mx) atomicMax(reinterpret_cast<unsigned long long*>(scal), mx);
    if (cnt) atomicAdd(reinterpret_cast<unsigned long long*>(scal + 4), cnt);
  }
}

// old->new id: identity when the node set is unchanged (the common steady
// state of a stream over a fixed population), then kernels skip the remap
__device__ __forceinline__ u32 remap(const u32* o2n, u32 v) { return o2n ? o2n[v] : v; }

__global__ void k_present_batch(const i64* bs, const i64* bd, const i64* bt, u64 n, i64 cutoff, u8* present,
                                u64* max_id) {
  u64 mx = 0;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    if (bt[i] >= cutoff) {
      const u64 a = static_cast<u64>(bs[i]), b = static_cast<u64>(bd[i]);
      if (!present[a]) present[a] = 1;
      if (!present[b]) present[b] = 1;
      mx = max(mx, max(a, b));
    }
  }
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(reinterpret_cast<unsigned long long*>(max_id), mx);
}

struct U8Fn {
  const u8* p;
  __device__ __forceinline__ u32 operator()(u64 i) const { return p[i]; }
};

__global__ void k_fill_ext_u8(const u8* present, const u32* rank, u64 range, i64* ext) {
  for (u64 id = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; id < range;
       id += static_cast<u64>(gridDim.x) * blockDim.x)
    if (present[id]) ext[rank[id]] = static_cast<i64>(id);
}

__global__ void k_old_to_new(const u8* alive, const i64* ext, const u32* rank, u64 V, u32* o2n) {
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<u64>(gridDim.x) * blockDim.x)
    o2n[v] = alive[v] ? rank[ext[v]] : 0xffffffffu;
}

__global__ void k_batch_internal(const i64* bs, const i64* bd, const i64* bt, u64 n, i64 cutoff, const u32* pos,
                                 const u32* rank, u32* s_i, u32* d_i, i64* t_c) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    if (bt[i] >= cutoff) {
      const u32 k = pos[i];
      s_i[k] = rank[bs[i]];
      d_i[k] = rank[bd[i]];
      t_c[k] = bt[i];
    }
  }
}

// canonical key (t, src, dst) with new internal ids
struct K3 {
  i64 t;
  u64 sd;
  __device__ __forceinline__ bool operator<(const K3& o) const { return t < o.t || (t == o.t && sd < o.sd); }
};

struct SurvivorKey {
  StoreView s;
  const u32* o2n;
  u64 from;
  __device__ __forceinline__ K3 operator()(u64 i) const {
    const EdgeRec r = edge_at(s, from + i);
    return K3{r.t, (static_cast<u64>(remap(o2n, r.src)) << 32) | remap(o2n, r.dst)};
  }
};

struct SurvivorKeySoA {  // contiguous stores (the merge route)
  const u32* e_src;
  const u32* e_dst;
  const i64* e_t;
  const u32* o2n;
  u64 from;
  __device__ __forceinline__ K3 operator()(u64 i) const {
    const u64 p = from + i;
    return K3{e_t[p], (static_cast<u64>(remap(o2n, e_src[p])) << 32) | remap(o2n, e_dst[p])};
  }
};

struct BatchKey {
  const u32* s;
  const u32* d;
  const i64* t;
  __device__ __forceinline__ K3 operator()(u64 j) const {
    return K3{t[j], (static_cast<u64>(s[j]) << 32) | d[j]};
  }
};

struct CanonicalEmit {
  u32* e_src;
  u32* e_dst;
  i64* e_t;
  u32* spos;
  u32* bpos;
  __device__ __forceinline__ void operator()(u64 o, bool from_a, u64 idx, const K3& k) const {
    e_src[o] = static_cast<u32>(k.sd >> 32);
    e_dst[o] = static_cast<u32>(k.sd);
    e_t[o] = k.t;
    if (from_a) spos[idx] = static_cast<u32>(o);
    else bpos[idx] = static_cast<u32>(o);
  }
};

struct SurvivingEntryFn {
  const Entry* ent;
  u32 from;
  __device__ __forceinline__ u32 operator()(u64 p) const { return ent[p].edge >= from ? 1u : 0u; }
};

// X: the old node view's surviving entries, re-keyed (new owner, new pos)
// New position of surviving edge i (0-based among survivors): survivors
// before the first batch edge keep i (no batch edge precedes them) — for a
// time-ordered stream that is all but the boundary tail, so the random
// gather from spos is almost never issued. Fused into the compaction scan.
struct XScatter {
  const Entry* ent;
  const u32* owner;
  u32 from;
  const u32* o2n;
  const u32* spos;
  const u32* bpos;
  u64 A, S;
  u64* xkey;
  u32* xnbr;
  i64* xt;
  __device__ __forceinline__ void operator()(u64 p, u64 k, u32 f) const {
    if (!f) return;
    const Entry e = ent[p];
    const u64 i0 = A ? bpos[0] : S;
    const u32 i = e.edge - from;
    const u32 np = i < i0 ? i : spos[i];
    xkey[k] = (static_cast<u64>(remap(o2n, owner[p])) << 32) | np;
    xnbr[k] = remap(o2n, e.nbr);
    xt[k] = e.t;
  }
};

// ---- node view by placement (time-ordered append case) ---------------------------
//
// When the canonical merge is a concatenation, every batch entry of a node
// follows all of its surviving entries, so the new region of v is
// [survivors of v in old order | batch entries of v in position order].
// Region sizes = old size - evicted entries + batch entries (two count
// passes), one scan gives the new regions, survivors are written straight to
// their final slots (no compaction scan, no merge), batch entries are placed
// with per-node cursors and each node's (short) batch segment is re-sorted by
// position (a stable radix sort of the batch's entries by owner).

__device__ __forceinline__ u32 owner_of_side(int mode, u32 s, u32 d, int side) {
  if (mode == TWG_UNDIRECTED) return side ? d : s;
  return mode == TWG_BACKWARD ? d : s;
}

// warp-aggregated increment: lanes with the same key add once
__device__ __forceinline__ void agg_inc(u32* cnt, u32 key, bool valid) {
  const u32 peers = __match_any_sync(0xffffffffu, valid ? key : 0xffffffffu);
  if (valid && (__ffs(peers) - 1) == static_cast<int>(threadIdx.x & 31)) atomicAdd(cnt + key, __popc(peers));
}

__global__ void k_count_evicted(const u32* e_src, const u32* e_dst, u64 from, int mode, u32* evicted) {
  const int sides = mode == TWG_UNDIRECTED ? 2 : 1;
  const u64 n = from * sides;
  for (u64 j = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; j < ((n + 31) & ~31ull);
       j += static_cast<u64>(gridDim.x) * blockDim.x) {
    const bool valid = j < n;
    const u64 i = sides == 2 ? (j >> 1) : j;
    const u32 o = valid ? owner_of_side(mode, e_src[i], e_dst[i], sides == 2 ? static_cast<int>(j & 1) : 0) : 0;
    agg_inc(evicted, o, valid);
  }
}

__global__ void k_count_y(const u32* s, const u32* d, u64 A, int mode, u32* ycnt) {
  const int sides = mode == TWG_UNDIRECTED ? 2 : 1;
  const u64 n = A * sides;
  for (u64 j = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; j < ((n + 31) & ~31ull);
       j += static_cast<u64>(gridDim.x) * blockDim.x) {
    const bool valid = j < n;
    const u64 k = sides == 2 ? (j >> 1) : j;
    const u32 o = valid ? owner_of_side(mode, s[k], d[k], sides == 2 ? static_cast<int>(j & 1) : 0) : 0;
    agg_inc(ycnt, o, valid);
  }
}

// new region sizes (surviving entries + batch entries) per new node; the
// survivors' count is written at the NEW id; max batch segment -> scal[0]
__global__ void k_region_sizes(const uint2* old_meta, const u32* evicted, const u8* alive_or_null, const u32* o2n,
                               u64 Vo, u32* xcnt_new) {
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < Vo;
       v += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 x = old_meta[v + 1].x - old_meta[v].x - evicted[v];
    if (x) xcnt_new[remap(o2n, static_cast<u32>(v))] = x;
  }
}


struct SizeFn {
  const u32* x;
  const u32* y;
  __device__ __forceinline__ u32 operator()(u64 v) const { return x[v] + y[v]; }
};


// survivors straight to their final slots: slot = new_off[v'] + (p - first surviving entry of v)
__global__ void k_place_x(const Entry* ent, const u32* owner, u64 Po, u32 from, const uint2* old_meta,
                          const u32* evicted, const u32* o2n, const u32* new_off, Entry* out_ent, u32* out_owner) {
  for (u64 p = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; p < Po;
       p += static_cast<u64>(gridDim.x) * blockDim.x) {
    const Entry e = ent[p];
    if (e.edge < from) continue;
    const u32 v = owner[p];
    const u32 vn = remap(o2n, v);
    const u64 slot = new_off[vn] + (p - (old_meta[v].x + evicted[v]));
    Entry x;
    x.nbr = remap(o2n, e.nbr);
    x.edge = e.edge - from;  // concatenation: survivors keep their index
    x.t = e.t;
    out_ent[slot] = x;
    out_owner[slot] = vn;
  }
}



struct BatchRec;
__global__ void k_place_y_sorted(const u32* owners, const u32* jidx, u64 Yn, int mode, const BatchRec* rec,
                                 const u32* new_off, const u32* xcnt, const u32* ystart, Entry* out_ent, u32* out_owner);

// one 24-byte record per sorted batch edge, so the node-view entries of the
// batch gather one sector instead of four
struct BatchRec {
  u32 pos;
  u32 src;
  u32 dst;
  u32 pad;
  i64 t;
};

// the canonical merge degenerates to a concatenation iff the first batch
// edge does not sort before the last survivor (survivors first on ties)
__global__ void k_concat_check(SurvivorKey ka, u64 S, BatchKey kb, u64* out) { *out = (kb(0) < ka(S - 1)) ? 0 : 1; }

__global__ void k_copy_survivors(const u32* s, const u32* d, const i64* t, const u32* o2n, u64 n, u32* os, u32* od,
                                 i64* ot) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    os[i] = remap(o2n, s[i]);
    od[i] = remap(o2n, d[i]);
    ot[i] = t[i];
  }
}

__global__ void k_pack_batch_rec(const u32* s, const u32* d, const i64* t, const u32* bpos, u64 S, u64 A,
                                 BatchRec* rec) {
  for (u64 k = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; k < A;
       k += static_cast<u64>(gridDim.x) * blockDim.x) {
    BatchRec r;
    r.pos = bpos ? bpos[k] : static_cast<u32>(S + k);
    r.src = s[k];
    r.dst = d[k];
    r.pad = 0;
    r.t = t[k];
    rec[k] = r;
  }
}

// batch entries (stable-sorted by owner) to their final slots: after the
// node's survivors, in position order; consecutive q write consecutive slots
__global__ void k_place_y_sorted(const u32* owners, const u32* jidx, u64 Yn, int mode, const BatchRec* rec,
                                 const u32* new_off, const u32* xcnt, const u32* ystart, Entry* out_ent,
                                 u32* out_owner) {
  for (u64 q = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; q < Yn;
       q += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 o = owners[q];
    const u32 j = jidx[q];
    const BatchRec r = rec[mode == TWG_UNDIRECTED ? (j >> 1) : j];
    u32 nbr;
    if (mode == TWG_FORWARD) nbr = r.dst;
    else if (mode == TWG_BACKWARD) nbr = r.src;
    else nbr = (j & 1) ? r.src : r.dst;
    const u64 slot = static_cast<u64>(new_off[o]) + xcnt[o] + (q - ystart[o]);
    Entry x;
    x.nbr = nbr;
    x.edge = r.pos;
    x.t = r.t;
    out_ent[slot] = x;
    out_owner[slot] = o;
  }
}

__global__ void k_make_y_rec(const u32* owners, const u32* jidx, u64 P, int mode, const BatchRec* rec, u64* ykey,
                             u32* ynbr, i64* yt) {
  for (u64 q = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; q < P;
       q += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 j = jidx[q];
    const BatchRec r = rec[mode == TWG_UNDIRECTED ? (j >> 1) : j];
    u32 nbr;
    if (mode == TWG_FORWARD) nbr = r.dst;
    else if (mode == TWG_BACKWARD) nbr = r.src;
    else nbr = (j & 1) ? r.src : r.dst;
    ykey[q] = (static_cast<u64>(owners[q]) << 32) | r.pos;
    ynbr[q] = nbr;
    yt[q] = r.t;
  }
}


// batch entries in canonical order: j -> owner (edge_store.cpp:120-124)
__global__ void k_batch_owner_keys(const u32* s, const u32* d, u64 A, int mode, u32* keys, u32* vals) {
  const u64 P = mode == TWG_UNDIRECTED ? 2 * A : A;
  for (u64 j = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; j < P;
       j += static_cast<u64>(gridDim.x) * blockDim.x) {
    u32 o;
    if (mode == TWG_UNDIRECTED) o = (j & 1) ? d[j >> 1] : s[j >> 1];
    else if (mode == TWG_BACKWARD) o = d[j];
    else o = s[j];
    keys[j] = o;
    vals[j] = static_cast<u32>(j);
  }
}


struct U64Key {
  const u64* k;
  __device__ __forceinline__ u64 operator()(u64 i) const { return k[i]; }
};

struct EntryEmit {
  const u32* xnbr;
  const i64* xt;
  const u32* ynbr;
  const i64* yt;
  u32* owner;
  Entry* ent;
  __device__ __forceinline__ void operator()(u64 o, bool from_a, u64 idx, const u64& key) const {
    Entry e;
    e.nbr = from_a ? xnbr[idx] : ynbr[idx];
    e.edge = static_cast<u32>(key);
    e.t = from_a ? xt[idx] : yt[idx];
    ent[o] = e;
    owner[o] = static_cast<u32>(key >> 32);
  }
};


// The streaming rebuild (file header, steps 1-4). `pos` = admitted-batch
// compaction offsets. Returns the new snapshot.
Store* ingest_streaming(Window& w, const i64* bs, const i64* bd, const i64* bt, u64 n, i64 cutoff, u64 from,
                        u64 A, u64 R, const u32* pos, u64* scratch_out) {
  Ctx& ctx = *w.ctx;
  cudaStream_t st = ctx.stream;
  const Store& Og = *w.store;
  const u64 S = Og.m - from;
  const u64 Vo = Og.V;
  u64 scratch = 0;
  PhaseTimer pt(ctx, "ingest_streaming");

  // 1. new dense ids
  DevBuf<u8> alive(Vo ? Vo : 1, st);
  DevBuf<u8> present(R, st);
  DevBuf<u32> rank(R + 1, st);
  scratch += Vo + 5 * R;
  TWG_CUDA(cudaMemsetAsync(present.p, 0, R, st));
  TWG_CUDA(cudaMemsetAsync(ctx.d_scalars + 6, 0, 8, st));
  // O's newest incident times; exact ones recomputed from its edges when the
  // streaming route left a lower bound (directed modes)
  DevBuf<i64> exact_last;
  const i64* o_last = Og.last_t.p;
  if (Vo && !Og.last_t_exact) {
    exact_last.alloc(Vo, st);
    TWG_CUDA(cudaMemsetAsync(exact_last.p, 0xff, Vo * sizeof(i64), st));
    k_store_last_t<<<grid(ctx, Og.m), kBlock, 0, st>>>(Og.view(), exact_last.p);
    TWG_LAUNCHED(ctx);
    o_last = exact_last.p;
  }
  if (Vo) {  // O(V) instead of a pass over every survivor's endpoints
    k_alive_from_last<<<grid(ctx, Vo), kBlock, 0, st>>>(o_last, Vo, cutoff, alive.p);
    TWG_LAUNCHED(ctx);
  }
  TWG_CUDA(cudaMemsetAsync(ctx.d_scalars + 10, 0, 8, st));
  if (Vo) {
    k_present_old<<<grid(ctx, Vo), kBlock, 0, st>>>(alive.p, Og.ext.p, Vo, present.p, ctx.d_scalars + 6);
    TWG_LAUNCHED(ctx);
  }
  if (A) {
    k_present_batch<<<grid(ctx, n), kBlock, 0, st>>>(bs, bd, bt, n, cutoff, present.p, ctx.d_scalars + 6);
    TWG_LAUNCHED(ctx);
  }
  exclusive_scan<u32>(ctx, U8Fn{present.p}, R, rank.p);
  TWG_CUDA(cudaMemsetAsync(ctx.d_scalars + 5, 0, 8, st));
  TWG_CUDA(cudaMemcpyAsync(ctx.d_scalars + 5, rank.p + R, 4, cudaMemcpyDeviceToDevice, st));
  u64 sc[6];
  read_scalars(ctx, ctx.d_scalars + 5, sc, 6);
  const u64 Vn = sc[0];
  w.max_ext = static_cast<i64>(sc[1]);
  // every old node survives and none is new <=> the ranks are unchanged
  const bool identity = Vo > 0 && sc[5] == Vo && Vn == Vo;

  auto s = std::make_unique<Store>();
  s->ctx = &ctx;
  s->mode = w.mode;
  s->m = S + A;
  s->V = Vn;
  s->ext_identity = Vn > 0 && w.max_ext >= 0 && static_cast<u64>(w.max_ext) == Vn - 1;
  s->ext.alloc(Vn ? Vn : 1, st);
  k_fill_ext_u8<<<grid(ctx, R), kBlock, 0, st>>>(present.p, rank.p, R, s->ext.p);
  TWG_LAUNCHED(ctx);
  DevBuf<u32> o2n_buf;
  const u32* o2n = nullptr;  // null = identity remap
  if (Vo && !identity) {
    o2n_buf.alloc(Vo, st);
    k_old_to_new<<<grid(ctx, Vo), kBlock, 0, st>>>(alive.p, Og.ext.p, rank.p, Vo, o2n_buf.p);
    TWG_LAUNCHED(ctx);
    o2n = o2n_buf.p;
  }
  // newest incident time per new node: survivors carry theirs, the batch maxes in below
  s->last_t.alloc(Vn ? Vn : 1, st);
  if (identity) {
    TWG_CUDA(cudaMemcpyAsync(s->last_t.p, o_last, Vn * sizeof(i64), cudaMemcpyDeviceToDevice, st));
  } else {
    TWG_CUDA(cudaMemsetAsync(s->last_t.p, 0xff, s->last_t.bytes(), st));
    if (Vo) {
      k_carry_last_t<<<grid(ctx, Vo), kBlock, 0, st>>>(o_last, alive.p, o2n, Vo, s->last_t.p);
      TWG_LAUNCHED(ctx);
    }
  }
  present.release();
  alive.release();

  // 2. canonical order: sort the admitted batch, merge with the survivors
  const int vb = Vn > 1 ? bit_width_u64(Vn - 1) : 0;
  DevBuf<u32> bsi(A ? A : 1, st), bdi(A ? A : 1, st);
  DevBuf<i64> btc(A ? A : 1, st);
  DevBuf<u32> bS(A ? A : 1, st), bD(A ? A : 1, st);
  DevBuf<i64> bT(A ? A : 1, st);
  scratch += 32 * A;
  if (A) {
    k_batch_internal<<<grid(ctx, n), kBlock, 0, st>>>(bs, bd, bt, n, cutoff, pos, rank.p, bsi.p, bdi.p, btc.p);
    TWG_LAUNCHED(ctx);
    if ((w.batch_shape & 1u) == 0)  // admitted edges in time order
      k_batch_last_t<true><<<grid(ctx, A), kBlock, 0, st>>>(bsi.p, bdi.p, btc.p, A, s->last_t.p);
    else
      k_batch_last_t<false><<<grid(ctx, A), kBlock, 0, st>>>(bsi.p, bdi.p, btc.p, A, s->last_t.p);
    TWG_LAUNCHED(ctx);
    if (w.batch_shape == 0) {
      k_segment_sort<<<grid(ctx, A), kBlock, 0, st>>>(bsi.p, bdi.p, btc.p, A, bS.p, bD.p, bT.p);
      TWG_LAUNCHED(ctx);
    } else {
      // admitted times lie in [cutoff, new_high]
      sort_canonical(ctx, bsi.p, bdi.p, btc.p, A, cutoff, w.t_high_pending, vb, bS.p, bD.p, bT.p);
    }
  }
  rank.release();
  bsi.release();
  bdi.release();
  btc.release();
  pt.mark("ids+batch_sort");
  // A time-ordered stream appends: if the first batch edge does not sort
  // before the last survivor, the merge is a concatenation (survivors keep
  // their index, batch edge k lands at S + k) — two streaming copies instead
  // of a merge-path pass.
  bool concat = A == 0 || S == 0;
  if (!concat) {
    k_concat_check<<<1, 1, 0, st>>>(SurvivorKey{Og.view(), o2n, from}, S, BatchKey{bS.p, bD.p, bT.p},
                                    ctx.d_scalars + 11);
    TWG_LAUNCHED(ctx);
    u64 c[1];
    read_scalars(ctx, ctx.d_scalars + 11, c, 1);
    concat = c[0] != 0;
  }
  // Time-ordered batch over an unchanged node population: append to the
  // shared log / node arena instead of rewriting the window (append.cu).
  if (concat && identity && A > 0 && append_ingest_enabled()) {
    pt.mark("append_handoff");
    if (scratch_out) *scratch_out = scratch + 48 * (w.mode == TWG_UNDIRECTED ? 2 * A : A) + 40 * Vn;
    DevBuf<EdgeRec> brec(A, st);
    k_pack_rec<<<grid(ctx, A), kBlock, 0, st>>>(bS.p, bD.p, bT.p, A, brec.p);
    TWG_LAUNCHED(ctx);
    return ingest_append(w, Og, std::move(s), brec.p, Ring{0u, kIdentityCap, 0u}, A, from, cutoff, false);
  }
  const Store& O = ensure_compact(ctx, Og);  // the rewrite routes below read the contiguous node view
  s->e_src.alloc(s->m ? s->m : 1, st);
  s->e_dst.alloc(s->m ? s->m : 1, st);
  s->e_t.alloc(s->m ? s->m : 1, st);
  DevBuf<u32> spos, bpos;
  if (concat) {
    if (S) {
      k_copy_survivors<<<grid(ctx, S), kBlock, 0, st>>>(O.e_src.p + from, O.e_dst.p + from, O.e_t.p + from, o2n, S,
                                                        s->e_src.p, s->e_dst.p, s->e_t.p);
      TWG_LAUNCHED(ctx);
    }
    if (A) {
      k_copy_survivors<<<grid(ctx, A), kBlock, 0, st>>>(bS.p, bD.p, bT.p, nullptr, A, s->e_src.p + S, s->e_dst.p + S,
                                                        s->e_t.p + S);
      TWG_LAUNCHED(ctx);
    }
  } else {
    spos.alloc(S ? S : 1, st);
    bpos.alloc(A ? A : 1, st);
    scratch += 4 * (S + A);
    merge_path<K3>(ctx, SurvivorKeySoA{O.e_src.p, O.e_dst.p, O.e_t.p, o2n, from}, S, BatchKey{bS.p, bD.p, bT.p}, A,
                   CanonicalEmit{s->e_src.p, s->e_dst.p, s->e_t.p, spos.p, bpos.p});
  }
  pt.mark(concat ? "canonical_concat" : "canonical_merge");
  build_ts_view(ctx, *s);
  pt.mark("ts_view");

  // 3. node view: surviving old entries (X) merged with the batch's entries (Y)
  const u64 Po = O.P;
  const u64 sides = w.mode == TWG_UNDIRECTED ? 2 : 1;
  const u64 Xn = Po - sides * from;  // every surviving edge keeps all of its entries
  const u64 Yn = sides * A;
  bool placed = false;
  if (concat && Vn > 0) {
    DevBuf<u32> evicted(Vo ? Vo : 1, st), ycnt(Vn, st), xcnt(Vn, st);
    if (Vo) TWG_CUDA(cudaMemsetAsync(evicted.p, 0, Vo * 4, st));
    TWG_CUDA(cudaMemsetAsync(ycnt.p, 0, Vn * 4, st));
    TWG_CUDA(cudaMemsetAsync(xcnt.p, 0, Vn * 4, st));
    TWG_CUDA(cudaMemsetAsync(ctx.d_scalars + 12, 0, 8, st));
    if (from) {
      k_count_evicted<<<grid(ctx, sides * from), kBlock, 0, st>>>(O.e_src.p, O.e_dst.p, from, w.mode, evicted.p);
      TWG_LAUNCHED(ctx);
    }
    if (A) {
      k_count_y<<<grid(ctx, Yn), kBlock, 0, st>>>(bS.p, bD.p, A, w.mode, ycnt.p);
      TWG_LAUNCHED(ctx);
    }
    pt.mark("place_counts");
    {
      if (Vo) {
        k_region_sizes<<<grid(ctx, Vo), kBlock, 0, st>>>(O.nmeta.p, evicted.p, nullptr, o2n, Vo, xcnt.p);
        TWG_LAUNCHED(ctx);
      }
      DevBuf<u32> new_off(Vn + 1, st), ystart(Vn + 1, st);
      exclusive_scan<u32>(ctx, SizeFn{xcnt.p, ycnt.p}, Vn, new_off.p);
      s->P = Xn + Yn;
      s->ent.alloc(s->P ? s->P : 1, st);
      s->owner.alloc(s->P ? s->P : 1, st);
      pt.mark("place_offsets");
      if (Po) {
        k_place_x<<<grid(ctx, Po), kBlock, 0, st>>>(O.ent.p, O.owner.p, Po, static_cast<u32>(from), O.nmeta.p,
                                                    evicted.p, o2n, new_off.p, s->ent.p, s->owner.p);
        TWG_LAUNCHED(ctx);
      }
      pt.mark("place_x");
      if (Yn) {
        // batch entries stable-sorted by owner: rank within owner = q - ystart[owner]
        exclusive_scan<u32>(ctx, LoadFn<u32>{ycnt.p}, Vn, ystart.p);
        DevBuf<BatchRec> rec(A, st);
        k_pack_batch_rec<<<grid(ctx, A), kBlock, 0, st>>>(bS.p, bD.p, bT.p, nullptr, S, A, rec.p);
        TWG_LAUNCHED(ctx);
        DevBuf<u32> k0(Yn, st), k1(Yn, st), v0(Yn, st), v1(Yn, st);
        u32* kp = k0.p;
        u32* ka = k1.p;
        u32* vp = v0.p;
        u32* va = v1.p;
        k_batch_owner_keys<<<grid(ctx, Yn), kBlock, 0, st>>>(bS.p, bD.p, A, w.mode, kp, vp);
        TWG_LAUNCHED(ctx);
        radix_sort_pairs<u32>(ctx, &kp, &ka, &vp, &va, Yn, vb);
        pt.mark("place_y_sort");
        k_place_y_sorted<<<grid(ctx, Yn), kBlock, 0, st>>>(kp, vp, Yn, w.mode, rec.p, new_off.p, xcnt.p, ystart.p,
                                                           s->ent.p, s->owner.p);
        TWG_LAUNCHED(ctx);
      }
      placed = true;
      pt.mark("place_y");
    }
  }
  if (!placed) {
  DevBuf<u64> xkey(Xn ? Xn : 1, st);
  DevBuf<u32> xnbr(Xn ? Xn : 1, st);
  DevBuf<i64> xt(Xn ? Xn : 1, st);
  scratch += 20 * Xn;
  scan_scatter(ctx, SurvivingEntryFn{O.ent.p, static_cast<u32>(from)}, Po, ctx.d_scalars + 9,
               XScatter{O.ent.p, O.owner.p, static_cast<u32>(from), o2n, spos.p, concat ? nullptr : bpos.p,
                        concat ? 0 : A, S, xkey.p, xnbr.p, xt.p});
  pt.mark("node_x");
  DevBuf<u64> ykey(Yn ? Yn : 1, st);
  DevBuf<u32> ynbr(Yn ? Yn : 1, st);
  DevBuf<i64> yt(Yn ? Yn : 1, st);
  scratch += 36 * Yn;
  if (Yn) {
    DevBuf<BatchRec> rec(A, st);
    k_pack_batch_rec<<<grid(ctx, A), kBlock, 0, st>>>(bS.p, bD.p, bT.p, concat ? nullptr : bpos.p, S, A, rec.p);
    TWG_LAUNCHED(ctx);
    DevBuf<u32> k0(Yn, st), k1(Yn, st), v0(Yn, st), v1(Yn, st);
    u32* kp = k0.p;
    u32* ka = k1.p;
    u32* vp = v0.p;
    u32* va = v1.p;
    k_batch_owner_keys<<<grid(ctx, Yn), kBlock, 0, st>>>(bS.p, bD.p, A, w.mode, kp, vp);
    TWG_LAUNCHED(ctx);
    radix_sort_pairs<u32>(ctx, &kp, &ka, &vp, &va, Yn, vb);
    k_make_y_rec<<<grid(ctx, Yn), kBlock, 0, st>>>(kp, vp, Yn, w.mode, rec.p, ykey.p, ynbr.p, yt.p);
    TWG_LAUNCHED(ctx);
  }
  pt.mark("node_y");
  s->P = Xn + Yn;
  s->ent.alloc(s->P ? s->P : 1, st);
  s->owner.alloc(s->P ? s->P : 1, st);
  merge_path<u64>(ctx, U64Key{xkey.p}, Xn, U64Key{ykey.p}, Yn,
                  EntryEmit{xnbr.p, xt.p, ynbr.p, yt.p, s->owner.p, s->ent.p});
  pt.mark("node_merge");
  }
  // 4. marks, offsets, optional views
  finish_node_view(ctx, *s, w.opts);
  pt.mark("marks+views");
  if (scratch_out) *scratch_out = scratch;
  return s.release();
}

// The fast append route (append.cu) when the batch shape allows it from
// the batch statistics alone: time-ordered with short equal-time runs, all
// admitted (min t >= cutoff), strictly after the window's newest time (the
// canonical merge is a concatenation), ids inside the current dense
// population 0..V-1 (internal == external), and no old node leaving the
// window (checked on the device after the newest-time update; otherwise the
// general route runs from scratch and the speculative work is discarded).
Store* ingest_fast(Window& w, FastSpec& spec, u64 n, const u64* sc, i64 cutoff, twg_batch_stats* stats) {
  Ctx& ctx = *w.ctx;
  cudaStream_t st = ctx.stream;
  const Store& O = *w.store;
  const i64 batch_min = static_cast<i64>(sc[8]);
  const u32 shape = static_cast<u32>(sc[7]);
  if (!spec.on || shape != 0 || sc[9] || batch_min < cutoff || batch_min <= w.t_high || sc[1] >= O.V) return nullptr;
  const u64 V = O.V;
  auto s = std::make_unique<Store>();
  s->ctx = &ctx;
  s->mode = w.mode;
  s->V = V;
  s->ext_identity = true;
  // the id map is the identity 0..V-1 on this route: one immutable copy shared by the snapshots
  if (O.ext_keep) {
    s->ext_keep = O.ext_keep;
  } else {
    s->ext_keep = std::make_shared<DevBuf<i64>>(V, st);
    TWG_CUDA(cudaMemcpyAsync(s->ext_keep->p, O.ext.p, V * sizeof(i64), cudaMemcpyDeviceToDevice, st));
  }
  s->ext.alias(s->ext_keep->p, V);
  // newest incident time: only the owner side is tracked here (merged by the
  // placement's bucket counts); in directed modes the non-owner side would
  // cost one random atomic per edge, so last_t becomes a lower bound — the
  // population check stays sound (a node it cannot prove alive sends the
  // batch to the general route, which recomputes exact times)
  s->last_t.alloc(V, st);  // filled from O.last_t by the bucket counts (ingest_append old_last)
  s->last_t_exact = w.mode == TWG_UNDIRECTED && O.last_t_exact;
  const u64 from = spec.from;
  s->m = O.m - from + n;
  stats->evicted = from;
  stats->dropped_late = 0;
  w.max_ext = static_cast<i64>(V - 1);
  Store* out =
      ingest_append(w, O, std::move(s), spec.rec, spec.wring, n, from, cutoff, true, spec.in_log, true, spec.bt,
                    spec.cols, spec.groups ? ctx.d_scalars + 14 : nullptr, batch_min,
                    compact_payload_enabled() && static_cast<u64>(static_cast<i64>(sc[0]) - batch_min) < (1ull << 32),
                    O.last_t.p, spec.hist.n ? spec.hist.p : nullptr, spec.rows_pre ? spec.hist_csum.p : nullptr,
                    spec.rows_pre ? spec.hist_rows.p : nullptr);
  if (!out) {  // an old node leaves the window: the general route recomputes everything
    stats->evicted = stats->dropped_late = 0;
    return nullptr;
  }
  return out;
}

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
  NvtxRange nvtx_scope("twg ingest_batch");
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
  const Store& old = *w.store;
  // batch_high, new_high, cutoff (window_manager.cpp:30-33)
  k_init_scalars<<<1, 1, 0, st>>>(ctx.d_scalars);
  TWG_LAUNCHED(ctx);
  // Fast-route speculation: over a dense population 0..V-1 the statistics
  // pass also writes the canonical records (into the log ring when it has
  // room) and the survivor bound is found on the device — one read-back
  // decides, nothing is published if the route does not apply.
  FastSpec spec;
  spec.on = append_ingest_enabled() && old.m > 0 && old.V > 0 && old.ext_identity && n < 0xffffffffull / 2;
  spec.bt = d_t;
  spec.cols[0] = d_src;
  spec.cols[1] = d_dst;
  if (spec.on) {
    spec.in_log = append_log_slot(old, w.previous, n, &spec.wring);
    if (!spec.in_log) {
      spec.tmp.alloc(n, st);
      spec.rec = spec.tmp.p;
    } else {
      spec.rec = old.log->rec.p;
    }
    TWG_CUDA(cudaMemsetAsync(ctx.d_scalars + 12, 0, 8, st));
  }
  const u64 stat_tiles = (n + kStatTile - 1) / kStatTile;
  static const bool stat_attr = [] {
    TWG_CUDA(cudaFuncSetAttribute(k_batch_stats<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(StatSmem))));
    TWG_CUDA(cudaFuncSetAttribute(k_batch_stats<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(StatSmem))));
    return true;
  }();
  (void)stat_attr;
  TsSpec ts{};
  spec.groups = spec.on && spec.in_log && stats_groups_enabled();
  if (spec.groups) {
    const EdgeLog& L = *old.log;
    spec.ts_state.alloc(stat_tiles + 1, st);
    TWG_CUDA(cudaMemsetAsync(spec.ts_state.p, 0, spec.ts_state.bytes(), st));
    ts = TsSpec{spec.ts_state.p, L.ts_off.p, L.ts_time.p, L.zlen % L.cap, L.cap,
                old.seq0 + static_cast<u32>(old.m), ctx.d_scalars + 14};
    // the bucket sort's owner-digit histogram, fused (<= 2 digit passes above the 256-node bucket)
    HistSpec hs{nullptr, 0, w.mode};
    const int vb = old.V > 1 ? bit_width_u64(old.V - 1) : 0;
    const int passes = vb > 8 ? (vb - 8 + 7) / 8 : 0;
    if (passes >= 1 && passes <= 2 && stats_hist_enabled()) {
      spec.hist_rows.alloc(stat_tiles * 512, st);
      spec.hist.alloc(512, st);
      TWG_CUDA(cudaMemsetAsync(spec.hist.p, 0, spec.hist.bytes(), st));
      hs = HistSpec{spec.hist_rows.p, passes, w.mode};
    }
    k_batch_stats<true><<<static_cast<unsigned>(stat_tiles), kBlock, sizeof(StatSmem), st>>>(
        d_src, d_dst, d_t, n, ctx.d_scalars, spec.rec, spec.wring, ts, hs);
    if (hs.rows) {
      TWG_LAUNCHED(ctx);
      static_assert(kStatTile == kPreItems * kSortBlock, "the first sort pass's tiles are the statistics tiles");
      // one entry per edge; k_csum_scan covers <= kCsumPer * 1024 blocks of kPreRowsPerBlock rows
      spec.rows_pre = w.mode != TWG_UNDIRECTED && sort_pre_enabled() &&
                      stat_tiles <= static_cast<u64>(kCsumPer) * 1024 * kPreRowsPerBlock;
      const u64 rpb = spec.rows_pre ? kPreRowsPerBlock : 256;
      const u64 hblocks = (stat_tiles + rpb - 1) / rpb;
      if (spec.rows_pre) spec.hist_csum.alloc(hblocks * 512, st);
      k_hist_rows<<<static_cast<unsigned>(hblocks), 512, 0, st>>>(spec.hist_rows.p, stat_tiles, rpb, spec.hist.p,
                                                                   spec.rows_pre ? spec.hist_csum.p : nullptr);
      if (spec.rows_pre) {
        TWG_LAUNCHED(ctx);
        k_csum_scan<<<512, 1024, 0, st>>>(spec.hist_csum.p, static_cast<u32>(hblocks), spec.hist.p);
      }
    }
  } else {
    k_batch_stats<false><<<static_cast<unsigned>(stat_tiles), kBlock, sizeof(StatSmem), st>>>(
        d_src, d_dst, d_t, n, ctx.d_scalars, spec.rec, spec.wring, ts, HistSpec{nullptr, 0, 0});
  }
  TWG_LAUNCHED(ctx);
  if (spec.on) {
    k_lower_bound_cut<<<1, 32, 0, st>>>(old.view(), w.t_high, w.duration, ctx.d_scalars, ctx.d_scalars + 12);
    TWG_LAUNCHED(ctx);
  }
  u64 sc[13];
  read_scalars(ctx, ctx.d_scalars, sc, 13);
  spec.from = sc[12];
  const i64 batch_high = static_cast<i64>(sc[0]);
  const u64 batch_max_id = sc[1];
  w.batch_shape = static_cast<u32>(sc[7]);
  const i64 new_high = w.t_high > batch_high ? w.t_high : batch_high;
  const i64 cutoff = w.cutoff_for(new_high);
  if (Store* fast = ingest_fast(w, spec, n, sc, cutoff, &stats)) {
    stats.retained = fast->m;
    stats.peak_bytes = old.device_bytes() + fast->device_bytes();
    TWG_CUDA(cudaStreamSynchronize(st));
    stats.rebuild_duration = std::chrono::duration<double>(clock::now() - started).count();
    release_store(w.previous);
    w.previous = w.store;
    w.store = fast;
    w.t_high = new_high;
    w.stats = stats;
    ++w.batch_count;
    if (out) *out = stats;
    return;
  }

  // survivors (export_suffix) and admitted batch edges
  k_lower_bound<<<1, 32, 0, st>>>(old.view(), cutoff, ctx.d_scalars + 2);
  TWG_LAUNCHED(ctx);
  DevBuf<u32> pos(n + 1, st);
  exclusive_scan<u32>(ctx, AdmitFn{d_t, cutoff}, n, pos.p);
  TWG_CUDA(cudaMemcpyAsync(ctx.d_scalars + 3, pos.p + n, 4, cudaMemcpyDeviceToDevice, st));
  k_admitted_neg<<<grid(ctx, n), kBlock, 0, st>>>(d_src, d_dst, d_t, n, cutoff, ctx.d_scalars + 4);
  TWG_LAUNCHED(ctx);
  u64 r[3];
  read_scalars(ctx, ctx.d_scalars + 2, r, 3);
  const u64 from = r[0];
  const u64 admitted = r[1] & 0xffffffffull;
  if (r[2]) fail(TWG_EINVAL, "edge store: negative node id");  // edge_store.cpp:37, state unchanged
  const u64 survivors = old.m - from;
  stats.evicted = old.m - survivors;
  stats.dropped_late = n - admitted;
  const u64 total = survivors + admitted;
  if (total >= 0xffffffffull / 2) fail(TWG_EINVAL, "edge store: edge count exceeds 32-bit reference space");

  // dense id fast path: the external-id range is compact
  const u64 R = std::max<u64>(w.max_ext >= 0 ? static_cast<u64>(w.max_ext) : 0, batch_max_id) + 1;
  const bool dense = R < (1ull << 31) && R <= std::max<u64>(8 * total, 1ull << 22);
  u64 scratch = 0;
  Store* rebuilt = nullptr;
  if (dense) {
    w.t_high_pending = new_high;
    rebuilt = ingest_streaming(w, d_src, d_dst, d_t, n, cutoff, from, admitted, R, pos.p, &scratch);
  } else {
    DevBuf<i64> ms(total ? total : 1, st), md(total ? total : 1, st), mt(total ? total : 1, st);
    if (survivors) {
      k_gather_survivors<<<grid(ctx, survivors), kBlock, 0, st>>>(ensure_compact(ctx, old).view(), from, ms.p, md.p,
                                                                  mt.p);
      TWG_LAUNCHED(ctx);
    }
    if (admitted) {
      k_compact_batch<<<grid(ctx, n), kBlock, 0, st>>>(d_src, d_dst, d_t, n, cutoff, pos.p, survivors, ms.p, md.p,
                                                       mt.p);
      TWG_LAUNCHED(ctx);
    }
    pos.release();
    rebuilt = build_store(ctx, EdgesSoA{ms.p, md.p, mt.p, total}, w.mode, w.opts, &scratch);
    scratch += 24 * total;
    if (rebuilt->V) {
      u64 mx[1];
      read_scalars(ctx, reinterpret_cast<const u64*>(rebuilt->ext.p + rebuilt->V - 1), mx, 1);
      w.max_ext = static_cast<i64>(mx[0]);
    }
  }

  stats.retained = rebuilt->m;
  stats.peak_bytes = old.device_bytes() + rebuilt->device_bytes() + scratch;
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
