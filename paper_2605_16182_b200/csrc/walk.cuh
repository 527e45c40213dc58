// Walk generation on the device (walk_engine.cpp:147-434).
#pragma once

#include "store.cuh"

namespace twg {

struct WalkSetDev {
  Ctx* ctx = nullptr;
  u32 stride = 0;
  u64 count = 0;       // walks in this shard
  u64 first = 0;       // global id of local walk 0
  u64 hops = 0;
  DevBuf<i64> nodes;   // [count * stride] walk-major, external ids
  DevBuf<i64> times;   // [count * stride]
  DevBuf<u32> lengths; // [count]
  bool tails_zeroed = false;
  // asynchronous compact download (twg_walkset_download_compact_async)
  DevBuf<u64> c_off;
  DevBuf<i64> c_nodes, c_times;
  cudaEvent_t d2h_done = nullptr;
  ~WalkSetDev() {
    if (d2h_done) {
      cudaEventSynchronize(d2h_done);  // the D2H stream may still read the compact buffers
      cudaEventDestroy(d2h_done);
    }
  }
};

// Validates like walk_engine.cpp:189-206 / :366-370 (throws Error(TWG_EINVAL)).
// shard_count > 1: generate only slice shard_rank of the resolved walk-id
// range (contiguous, balanced; the multi-GPU group's partition).
WalkSetDev* generate_walks(Ctx& ctx, Store& s, const twg_walk_config& cfg, const twg_thresholds& th,
                           int variant, twg_walk_stats* stats, int shard_rank = 0, int shard_count = 1);

// Host-side WalkStates + WalkSet columns (walk_engine.hpp:55-82).
struct HostWalkArrays {
  u32* current;
  i64* time;
  u32* prev;
  u8* has_prev;
  u8* alive;
  u32* length;
  i64* nodes;
  i64* times;
};

// init_walks / execute_task as device round trips (reference unit-test API)
void init_walks_dev(Ctx& ctx, Store& s, const twg_walk_config& cfg, u32* stride, u64* walk_count,
                    const HostWalkArrays* out);
void hop_walks_dev(Ctx& ctx, Store& s, const twg_walk_config& cfg, const u32* ids, u64 n_ids, u64 count, u32 stride,
                   const HostWalkArrays& io);

// zero the unused slots so the fixed-stride image equals the reference's
// zero-initialised WalkSet (walk_engine.cpp:237-239)
void walk_major_image(Ctx& ctx, const WalkSetDev& w, DevBuf<i64>& nodes, DevBuf<i64>& times);

// walk writers (walkio.cu, io.cpp:119-135 / :173-183): the text image on the
// device (bytes = its length), the binary image size, and a device walk set
// from a host walk-major image (the façade's io over host WalkSets)
constexpr u64 kWalkBinaryHeader = 20;  // "TMPW0002" + u32 stride + u64 walk_count
void walks_text(Ctx& ctx, const WalkSetDev& w, DevBuf<char>& text, u64* bytes);
u64 walks_binary_size(const WalkSetDev& w);
void walks_from_host(Ctx& ctx, u32 stride, u64 count, const i64* nodes, const i64* times, const u32* lengths,
                     WalkSetDev& out);

// edge files (edgeio.cu, io.cpp:40-69): TSV parse into device SoA columns
// (count data lines; on a bad line: error_line 1-based + its kind, no
// output) and TSV formatting of device edges
enum : u8 {
  kLineSkip = 0,
  kLineEdge = 1,
  kLineErrTabs = 2,
  kLineErrInvalid = 3,   // + field (0 source, 1 target, 2 timestamp)
  kLineErrNegative = 6,  // + field
};
void parse_edges_tsv(Ctx& ctx, const char* text, u64 bytes, DevBuf<i64>& src, DevBuf<i64>& dst, DevBuf<i64>& t,
                     u64* count, u64* error_line, u8* error_kind);
void format_edges_tsv(Ctx& ctx, const i64* src, const i64* dst, const i64* t, u64 n, DevBuf<char>& text,
                      u64* bytes);

// the reference's synthetic graphs (synth.cu, synthetic.cpp:24-140)
u64 synth_graph_size(int kind, u64 a, u64 b);
void synth_graph(Ctx& ctx, int kind, u64 a, u64 b, i64 t_max, u64 key, twg_edge* out);

// compact (CSR) image on the device: offsets[count+1], nodes/times[total]
void compact_walks(Ctx& ctx, const WalkSetDev& w, DevBuf<u64>& offsets, DevBuf<i64>& nodes,
                   DevBuf<i64>& times, u64* total);

void sample_start_edges(Ctx& ctx, Store& s, int bias, const double* d_u1, const double* d_u2, u64 n,
                        u64* d_out);

// schedule_step over explicit populations; returns list sizes + rows (host)
void schedule_step_explicit(Ctx& ctx, Store& s, const u32* d_nodes, const u8* d_alive, u64 n,
                            const twg_thresholds& th, u64* sizes5, u32* rows, u64 cap, u32* walk_ids);

void pick_index_batch(Ctx& ctx, int kind, const double* d_u, const u64* d_n, u64 count, u64* d_out);
struct PickSmall {
  static constexpr u32 kMax = 16;
  u32 count;
  double u[kMax];
  u64 n[kMax];
};
// count <= PickSmall::kMax host values -> host results (one launch, one sync)
void pick_index_small(Ctx& ctx, int kind, const double* u, const u64* n, u32 count, u64* out);
void pick_weighted_range_batch(Ctx& ctx, const double* d_u, const double* d_prefix, const u64* d_begin,
                               const u64* d_end, const double* d_base, u64 count, u64* d_out);
void rng_bits_batch(Ctx& ctx, int rng, u64 seed, const u64* d_walk, const u64* d_hop, const u64* d_ord,
                    u64 count, u64* d_out);

// primitives.hpp:11-31 on device buffers
void radix_sort_pairs_dev(Ctx& ctx, u64* keys, u32* vals, u64 n);
void exclusive_scan_dev(Ctx& ctx, const u64* in, u64* out, u64 n);
u64 run_length_encode_dev(Ctx& ctx, const u64* keys, u64 n, u64* rows);
u64 partition_flagged_dev(Ctx& ctx, const u32* items, u64 n, const u8* flags, u32* out);

// check_walkset (validity.cpp:108-120) on the device: report = {walks,
// valid walks, hops, valid hops}; d_first (optional, count entries) gets each
// walk's first invalid hop or -1
void audit_walks(Ctx& ctx, const WalkSetDev& w, const Store& s, int direction, bool strict, i64* d_first,
                 u64 report[4]);

// batched queries on a store
void neighborhood_batch(Ctx& ctx, Store& s, const i64* d_v, const i64* d_t, u64 n, int dir, u64* d_out3);
void find_nodes_batch(Ctx& ctx, Store& s, const i64* d_v, u64 n, u32* d_internal, u8* d_found);
void adjacent_batch(Ctx& ctx, Store& s, const u32* d_a, const u32* d_b, u64 n, int temporal, const i64* d_t,
                    int dir, u8* d_out);

}  // namespace twg
