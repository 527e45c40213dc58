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
// is the admitted batch in canonical order with internal ids.
bool append_ingest_enabled();
Store* ingest_append(Window& w, const Store& O, std::unique_ptr<Store> s, const u32* bS, const u32* bD,
                     const i64* bT, u64 A, u64 from, i64 cutoff);

Window* window_create(Ctx& ctx, i64 duration, int mode, BuildOpts opts);
void window_destroy(Window* w);
// Device-resident SoA batch. stats may be null.
void window_ingest(Window& w, const i64* d_src, const i64* d_dst, const i64* d_t, u64 n, twg_batch_stats* out);

}  // namespace twg
