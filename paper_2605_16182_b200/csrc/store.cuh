// Device-resident dual index (one immutable snapshot), SoA in HBM.
//
// Replaces the reference's EdgeStore members (edge_store.hpp:168-199):
//   endpoints_/time_            -> e_src, e_dst (u32 internal ids), e_t (i64)
//   internal_to_external_       -> ext (i64, ascending: internal id == rank)
//   external_to_internal_       -> binary search over ext (no hash map)
//   ts_group_offsets_/time_/weight_prefix_ -> ts_off (u32), ts_time, ts_w
//   node_group_offsets_ + node_ts_index_   -> nmeta (uint2 {entry_off, group_off}, V+1)
//   node_ts_groups_ (16 B AoS)  -> mk_time (i64) + mk_start (u32) SoA: the
//                                  per-hop search touches only mk_time
//   node_ref_edge_              -> ent (16 B {nbr u32, edge u32, t i64}):
//                                  one aligned 16-byte load per hop gives the
//                                  neighbour AND the entry time, removing the
//                                  reference's dependent ref->endpoints->time
//                                  gathers (edge_store.hpp:133-140, walk_engine.cpp:39-44)
//   node_weight_prefix_         -> wp (f64)
//   node_adj_offsets_/node_adj_ -> adj_off (u32, V+1) + adj (u32)
#pragma once

#include <atomic>
#include <memory>
#include <mutex>

#include "common.cuh"

namespace twg {

// One edge of the streaming log (internal ids): the AoS record a walk start
// reads in one 128-bit load.
struct alignas(16) EdgeRec {
  u32 src, dst;
  i64 t;
};

struct alignas(16) Entry {  // one 128-bit load per hop
  u32 nbr;   // ref_neighbor(pos, owner)
  u32 edge;  // ref_edge(pos): index into the time-sorted edge array
  i64 t;     // time_[ref_edge(pos)]
};
static_assert(sizeof(Entry) == 16, "Entry must be 16 bytes");

// Per-node view of one snapshot (32 bytes: one sector per hop). Positions
// are LOGICAL: node v's entries are [eb, ee), its timestamp marks [gb, ge),
// and mark starts hold logical entry positions. They live in a ring of
// `cap` slots at `base` (entries and marks in parallel arrays): logical x
// maps to base + ((x - org) mod cap), with org chosen per snapshot so that
// x - org < 2 cap for every live x (one compare + select, no division).
// Contiguous stores use the identity ring {base 0, cap 2^32-1, org 0}.
struct alignas(32) NodeMeta {
  u32 eb, ee, gb, ge;
  u32 base, cap, eorg, gorg;
};
static_assert(sizeof(NodeMeta) == 32, "NodeMeta must be one 32-byte sector");

// Walk record of a streaming snapshot's node (64 B, one DRAM line access
// per hop — a random access moves a whole line, so the line carries what a
// forward hop usually needs beyond the bounds): the entry ring, the mark
// count, and the node's kWalkTail newest entries (newest first). A forward
// walk at time t whose causal slice starts inside the tail (t at or after the
// tail's oldest time — later hops, which move to the newest times, and every
// terminal hop) and whose pick lands in it never touches the ring.
constexpr u32 kWalkTail = 3;
struct alignas(64) WalkRec {
  u32 eb, ee;           // logical entry bounds
  u32 base, cap, eorg;  // entry ring
  u32 g;                // marks (ge - gb)
  u32 nbr[kWalkTail];   // nbr[i]: neighbour of entry ee - 1 - i (i < min(kWalkTail, ee - eb))
  u32 pad;
  i64 t[kWalkTail];     // its time
};
static_assert(sizeof(WalkRec) == 64, "WalkRec must be 64 bytes");

struct Ring {
  u32 base, cap, org;
  __device__ __forceinline__ u32 operator()(u32 x) const {
    const u32 d = x - org;
    return base + (d >= cap ? d - cap : d);
  }
};
// Implicit marks: a region whose timestamp groups are all single entries
// (as many groups as entries — distinct times, the common case of a
// streaming window) has mark k == {time of entry k, position of entry k}.
// The streaming ingest then does not store its marks (append.cu), and every
// reader derives them from the entries; explicit marks are stored whenever
// a region holds a repeated time.
__device__ __forceinline__ bool implicit_marks(const NodeMeta& m) { return m.ge - m.gb == m.ee - m.eb; }
__device__ __forceinline__ Ring entry_ring(const NodeMeta& m) { return Ring{m.base, m.cap, m.eorg}; }
__device__ __forceinline__ Ring mark_ring(const NodeMeta& m) { return Ring{m.base, m.cap, m.gorg}; }
constexpr u32 kIdentityCap = 0xffffffffu;

// Raw pointers + counts of one snapshot, passed by value to kernels.
//
// Edge numbering: entry .edge fields and ts_off hold edge SEQUENCE numbers
// (u32, wrapping); the snapshot's edge i has sequence seq0 + i. Contiguous
// (built) stores have seq0 == 0, so the values are the reference's 0-based
// indices; streaming stores share an append-only edge log whose numbering
// runs across batches (store.cuh EdgeLog).
struct StoreView {
  int mode;
  u64 m, V, Z, P, Q, A;
  const u32* e_src;    // contiguous stores: SoA edge columns
  const u32* e_dst;
  const i64* e_t;
  const EdgeRec* erec; // streaming stores: the log's AoS records (e_* null)
  const i64* ext;
  const u32* ts_off;   // group start sequence numbers, Z (+1 terminal in contiguous stores, unused)
  const i64* ts_time;
  const double* ts_w;
  const uint2* nmeta;  // {entry offset, group offset}, V+1 (contiguous stores only)
  const NodeMeta* nm;  // per-node bounds + ring (every store)
  const i64* mk_time;
  const u32* mk_start;
  const Entry* ent;
  const double* wp;
  const u32* adj_off;
  const u32* adj;
  int ext_identity;  // ext[v] == v for all v (the id map can be skipped)
  u32 seq0;
  Ring erg;  // snapshot edge i -> slot erg(i) of e_src/e_dst/e_t (identity in contiguous stores)
  Ring zrg;  // snapshot ts group g -> slot zrg(g) of ts_off/ts_time
  // streaming stores (no ts_w): the nonzero tail of the ts weight prefix,
  // ts_wtail[g - ts_wt0] for groups g >= ts_wt0 (every earlier value is +0)
  const double* ts_wtail;
  u64 ts_wt0;
  const WalkRec* wrec;  // streaming stores built by the append route: per-node walk records (else null)
};

// snapshot edge i
__device__ __forceinline__ i64 edge_time(const StoreView& s, u64 i) {
  const u32 p = s.erg(static_cast<u32>(i));
  return s.erec ? s.erec[p].t : s.e_t[p];
}
__device__ __forceinline__ EdgeRec edge_at(const StoreView& s, u64 i) {
  const u32 p = s.erg(static_cast<u32>(i));
  if (s.erec) return s.erec[p];
  return EdgeRec{s.e_src[p], s.e_dst[p], s.e_t[p]};
}

// Edge range [lo, hi) (snapshot-relative) of timestamp group g < Z.
__device__ __forceinline__ void ts_group_range(const StoreView& s, u64 g, u64& lo, u64& hi) {
  lo = static_cast<u32>(s.ts_off[s.zrg(static_cast<u32>(g))] - s.seq0);
  hi = g + 1 < s.Z ? static_cast<u64>(static_cast<u32>(s.ts_off[s.zrg(static_cast<u32>(g + 1))] - s.seq0)) : s.m;
}

// host: the ring slot of relative index i of a log slice starting at logical
// position `first` (slots = logical mod cap)
inline Ring log_ring(u64 cap, u64 first) {
  return Ring{0u, static_cast<u32>(cap), static_cast<u32>(0u - static_cast<u32>(first % cap))};
}

struct BuildOpts {
  bool weights = true;
  bool adjacency = true;
};

// ---- streaming (append) representation ------------------------------------
//
// A time-ordered stream only ever appends to the window's newest end and
// evicts from its oldest end, per node as well as globally. The streaming
// snapshots therefore share two append-only structures instead of
// rewriting the whole window every batch:
//  * EdgeLog: the canonical edge columns and the timestamp-group view; a
//    snapshot is a contiguous slice of it.
//  * NodeArena: one ring per node (NodeMeta); new entries and marks are
//    written at the logical ends ee/ge, eviction advances eb/gb, and the
//    slots freed by eviction are reused once no live snapshot can read them.
//    A ring without room is relocated to fresh arena space (bigger); when
//    the arena is exhausted, or a snapshot older than the retired one is
//    still held, every live ring is repacked into a new arena.
// Nothing a live snapshot can read is ever overwritten: a ring only accepts
// new entries while ee + y - (oldest live eb in that ring) <= cap, and a
// replaced log/arena stays alive (shared_ptr) while any snapshot uses it.
struct EdgeLog {  // two rings of `cap` slots; positions are logical (slot = position mod cap)
  DevBuf<EdgeRec> rec;
  DevBuf<u32> ts_off;  // group start sequence numbers
  DevBuf<i64> ts_time;
  u64 cap = 0;     // edges (and groups)
  u64 len = 0;     // edges written (logical end)
  u64 zlen = 0;    // groups written (logical end)
};

struct NodeArena {
  u64 serial = 0;    // distinct per arena (diagnostics: twg_store_get_layout)
  DevBuf<Entry> ent;
  DevBuf<i64> mk_time;
  DevBuf<u32> mk_start;
  u64 cap = 0;       // slots
  u64 used = 0;      // bump pointer (host copy, updated after each ingest)
  u64 V = 0;
};

struct Store {
  std::atomic<int> refs{1};
  Ctx* ctx = nullptr;
  int mode = 0;
  u64 m = 0, V = 0, Z = 0, P = 0, Q = 0, A = 0;
  bool has_weights = false, has_adjacency = false;
  bool ext_identity = false;
  DevBuf<u32> e_src, e_dst;
  DevBuf<i64> e_t, ext;
  std::shared_ptr<DevBuf<i64>> ext_keep;  // owner of ext when it is shared between snapshots (ext aliases it)
  DevBuf<EdgeRec> e_rec;  // streaming stores: alias of the log's records
  DevBuf<u32> ts_off;
  DevBuf<i64> ts_time;
  DevBuf<double> ts_w;
  DevBuf<uint2> nmeta;
  DevBuf<i64> mk_time;
  DevBuf<u32> mk_start;
  DevBuf<Entry> ent;
  DevBuf<double> wp;
  DevBuf<u32> adj_off, adj;
  DevBuf<u32> owner;  // owner node of each node-view entry (drives the next batch's merge)
  DevBuf<i64> last_t; // newest incident edge time per node: v survives a cutoff c iff last_t[v] >= c
  bool last_t_exact = true;  // false: a lower bound (the streaming route tracks only the owner side)
  DevBuf<NodeMeta> nm;  // per-node bounds + ring: the walk kernels' node meta (every store)
  DevBuf<WalkRec> wrec; // append-route snapshots: nm + the newest entries per node (forward walks)
  u32 seq0 = 0;       // sequence number of edge 0 (StoreView)
  // streaming representation (gapped == true): slices of a shared log/arena
  bool gapped = false;
  std::shared_ptr<EdgeLog> log;
  std::shared_ptr<NodeArena> arena;
  u64 log_first = 0;  // logical log position of edge 0
  u64 ts_first = 0;   // logical log group position of group 0
  u64 relocated = 0;  // rings moved by the ingest that made this snapshot (diagnostics)
  u32 e_cap = kIdentityCap, e_org = 0, z_cap = kIdentityCap, z_org = 0;  // StoreView::erg / zrg
  DevBuf<double> ts_wtail;  // streaming stores: the nonzero tail of the ts weight prefix
  u64 ts_wt0 = 0;
  // contiguous materialisation of a gapped store (reference layout), built on
  // first use by the accessors / downloads / weighted views (ensure_compact)
  mutable std::unique_ptr<Store> compact;
  mutable std::mutex compact_mu;
  // the lazily completed views (weights, adjacency): built under this lock and
  // published (flag set) only after their kernels finished, so a walk on
  // another context's stream never reads a half-built view
  std::mutex lazy_mu;

  StoreView view() const {
    return StoreView{mode,     m,         V,         Z,          P,         Q,        A,
                     e_src.p,  e_dst.p,   e_t.p,     e_rec.p,    ext.p,     ts_off.p,  ts_time.p,
                     ts_w.p,   nmeta.p,   nm.p,      mk_time.p,  mk_start.p, ent.p,   wp.p,
                     adj_off.p, adj.p,  ext_identity ? 1 : 0, seq0,
                     Ring{0u, e_cap, e_org}, Ring{0u, z_cap, z_org}, ts_wtail.p, ts_wt0, wrec.p};
  }
  u64 device_bytes() const {
    return e_src.bytes() + e_dst.bytes() + e_t.bytes() + e_rec.bytes() + ext.bytes() + ts_off.bytes() +
           ts_time.bytes() + ts_w.bytes() + nmeta.bytes() + mk_time.bytes() + mk_start.bytes() +
           ent.bytes() + wp.bytes() + adj_off.bytes() + adj.bytes() + owner.bytes() + nm.bytes() +
           last_t.bytes() + wrec.bytes();
  }
};

// canonical (t, src, dst) order of edges with dense internal ids (edge_store.cpp:42-55)
void sort_canonical(Ctx& ctx, const u32* src_i, const u32* dst_i, const i64* t, u64 m, i64 tmin, i64 tmax, int vb,
                    u32* o_src, u32* o_dst, i64* o_t);
// ts_off / ts_time from s.e_t (edge_store.cpp:91-98)
void build_ts_view(Ctx& ctx, Store& s);
// nmeta / marks / group offsets (+ optional weights, adjacency) from the
// node-sorted s.owner and s.ent (edge_store.cpp:164-250)
void finish_node_view(Ctx& ctx, Store& s, BuildOpts opts);

// Canonical-order edges of a build input, device SoA, external ids.
struct EdgesSoA {
  const i64* src;
  const i64* dst;
  const i64* t;
  u64 n;
};

// Full dual-index build over device-resident edges (any order).
// edge_store.cpp:27-254. Throws Error(TWG_EINVAL) on negative ids/times or
// n >= 2^31-1 (edge_store.cpp:32-38).
Store* build_store(Ctx& ctx, EdgesSoA in, int mode, BuildOpts opts, u64* scratch_peak = nullptr);

// Lazily complete optional views.
void ensure_weights(Ctx& ctx, Store& s);
void ensure_adjacency(Ctx& ctx, Store& s);
// nm from nmeta (contiguous stores)
void build_nm(Ctx& ctx, Store& s);
// The contiguous (reference-layout) form of s: s itself unless s is gapped,
// else its lazily built contiguous copy (sharing the edge columns).
Store& ensure_compact(Ctx& ctx, const Store& s);

// Device binary-search helpers shared by the walk and query kernels.
__device__ __forceinline__ u32 ub_i64(const i64* a, u32 lo, u32 hi, i64 x) {
  // first k in [lo, hi) with x < a[k]
  while (lo < hi) {
    const u32 mid = lo + ((hi - lo) >> 1);
    if (x < a[mid]) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}
__device__ __forceinline__ u32 lb_i64(const i64* a, u32 lo, u32 hi, i64 x) {
  // first k in [lo, hi) with a[k] >= x
  while (lo < hi) {
    const u32 mid = lo + ((hi - lo) >> 1);
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

}  // namespace twg
