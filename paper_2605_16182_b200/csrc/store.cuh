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

#include "common.cuh"

namespace twg {

struct Entry {
  u32 nbr;   // ref_neighbor(pos, owner)
  u32 edge;  // ref_edge(pos): index into the time-sorted edge array
  i64 t;     // time_[ref_edge(pos)]
};
static_assert(sizeof(Entry) == 16, "Entry must be 16 bytes");

// Raw pointers + counts of one snapshot, passed by value to kernels.
struct StoreView {
  int mode;
  u64 m, V, Z, P, Q, A;
  const u32* e_src;
  const u32* e_dst;
  const i64* e_t;
  const i64* ext;
  const u32* ts_off;
  const i64* ts_time;
  const double* ts_w;
  const uint2* nmeta;  // {entry offset, group offset}, V+1
  const i64* mk_time;
  const u32* mk_start;
  const Entry* ent;
  const double* wp;
  const u32* adj_off;
  const u32* adj;
  int ext_identity;  // ext[v] == v for all v (the id map can be skipped)
};

struct BuildOpts {
  bool weights = true;
  bool adjacency = true;
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

  StoreView view() const {
    return StoreView{mode,     m,         V,         Z,          P,         Q,       A,
                     e_src.p,  e_dst.p,   e_t.p,     ext.p,      ts_off.p,  ts_time.p,
                     ts_w.p,   nmeta.p,   mk_time.p, mk_start.p, ent.p,     wp.p,
                     adj_off.p, adj.p,  ext_identity ? 1 : 0};
  }
  u64 device_bytes() const {
    return e_src.bytes() + e_dst.bytes() + e_t.bytes() + ext.bytes() + ts_off.bytes() +
           ts_time.bytes() + ts_w.bytes() + nmeta.bytes() + mk_time.bytes() + mk_start.bytes() +
           ent.bytes() + wp.bytes() + adj_off.bytes() + adj.bytes() + owner.bytes();
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
