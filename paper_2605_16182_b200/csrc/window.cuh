// Sliding-window ingestion on the device (window_manager.cpp:9-69).
#pragma once

#include "store.cuh"

namespace twg {

struct Window {
  Ctx* ctx = nullptr;
  i64 duration = 0;
  int mode = 0;
  BuildOpts opts;
  Store* store = nullptr;     // current snapshot (holds one reference)
  Store* previous = nullptr;  // exactly one retired snapshot (window_manager.hpp:40, :57-58)
  i64 t_high = kTimeUnset;
  u64 batch_count = 0;
  twg_batch_stats stats{};
  i64 max_ext = -1;            // largest external id in the current snapshot (dense-id fast path)
  i64 t_high_pending = 0;      // new_high of the batch being ingested
  u32 batch_shape = 0;         // bit0 not time-ordered, bit1 long equal-time runs

  i64 cutoff_for(i64 high) const { return high > duration ? high - duration : 0; }  // window_manager.hpp:51-53
};

void release_store(Store* s);

// Streaming append ingest (append.cu): the time-ordered, stable-population
// fast path. s carries the new snapshot's ids (ext, last_t, V); bS/bD/bT
// is the admitted batch in canonical order with internal ids; no_ties:
// every batch time is newer than every window time (no mark merges).
bool append_ingest_enabled();
using BatchRec16 = EdgeRec;  // one record per admitted batch edge (internal ids)
// when the shared log of O can take A more edges in place: the ring that
// maps batch edge k to its log slot (the batch can be written there directly)
bool append_log_slot(const Store& O, const Store* R, u64 A, Ring* wr);
// batch[bring(k)] = admitted batch edge k (canonical order, internal ids).
// in_log: the batch already sits in O's log through the ring append_log_slot
// returned (batch is then the log's record array).
// check_dead: s->last_t holds only the non-owner side of the batch; the owner
// side is merged here and the ingest returns null (nothing published) when an
// old node would leave the window.
// groups_done (device count): the batch's ts groups already sit in O's log
// (written by the statistics pass, in_log only) — the group scan is skipped.
// compact: every batch time lies in [tbase, tbase + 2^32): the bucket sort
// carries 12-B payloads (time as a u32 offset from tbase).
// old_last: s->last_t is unfilled; it becomes max(old_last, the batch's
// owner-side newest) per node (else s->last_t is updated in place).
// pre_hist: the bucket sort's digit histogram, already computed (fused into
// the statistics pass); stat_rows / pre_rows: its per-tile digit rows and the
// exclusive prefixes of their block sums (k_csum_scan) — the first pass skips
// its look-back.
Store* ingest_append(Window& w, const Store& O, std::unique_ptr<Store> s, const EdgeRec* batch, Ring bring, u64 A,
                     u64 from, i64 cutoff, bool no_ties, bool in_log = false, bool check_dead = false,
                     const i64* bt = nullptr, const i64* const* bcols = nullptr,
                     const u64* groups_done = nullptr, i64 tbase = 0, bool compact = false,
                     const i64* old_last = nullptr, u32* pre_hist = nullptr, const u32* pre_rows = nullptr,
                     const u32* stat_rows = nullptr);

Window* window_create(Ctx& ctx, i64 duration, int mode, BuildOpts opts);
void window_destroy(Window* w);
// Device-resident SoA batch. stats may be null.
void window_ingest(Window& w, const i64* d_src, const i64* d_dst, const i64* d_t, u64 n, twg_batch_stats* out);

}  // namespace twg
