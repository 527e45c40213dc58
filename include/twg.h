/*
 * twg.h — C ABI of the B200-native streaming temporal-random-walk engine
 * (libtimewalk_b200.so). Plain pointers and sizes only; no CUDA or torch
 * types cross this boundary.
 *
 * This is the thin C layer the drop-in C++ façade (include/timewalk/<name>.hpp,
 * same public API as the reference's proj/core) calls into, and what a
 * ctypes / cffi binding loads. Each entry point cites the reference
 * interface it replaces:
 *   twg_store_build       <- timewalk::EdgeStore::build            (edge_store.hpp:51-52, edge_store.cpp:27-254)
 *   twg_store_download    <- EdgeStore accessors                    (edge_store.hpp:54-166)
 *   twg_store_neighborhood<- EdgeStore::temporal_neighborhood[_internal] (edge_store.hpp:86-90, edge_store.cpp:270-302)
 *   twg_store_adjacent    <- EdgeStore::adjacent / adjacent_after   (edge_store.hpp:131-136, edge_store.cpp:310-323)
 *   twg_window_*          <- timewalk::WindowManager                (window_manager.hpp:31-62, window_manager.cpp:9-69)
 *   twg_generate          <- timewalk::generate_walks / generate_walks_fullwalk (walk_engine.hpp:161-171, walk_engine.cpp:362-434)
 *   twg_sample_start_edges<- timewalk::sample_start_edge            (walk_engine.hpp:159, walk_engine.cpp:284-299)
 *   twg_schedule_step     <- timewalk::schedule_step                (walk_engine.hpp:143-144, walk_engine.cpp:301-345)
 *   twg_pick_index        <- pick_index_{uniform,linear,exponential}(samplers.hpp:42-52, samplers.cpp:17-55)
 *   twg_pick_weighted_range <- pick_weighted_range                  (samplers.hpp:62-63, samplers.cpp:82-90)
 * replay_stream (replay.cpp:16-53) is host control flow over twg_window_ingest
 * + twg_generate; the façade and the Python mirror implement it there.
 *
 * Status codes map onto the reference's exception types:
 *   TWG_EINVAL -> std::invalid_argument, TWG_ERANGE -> std::out_of_range,
 *   TWG_ELOGIC -> std::logic_error, TWG_ECUDA/TWG_ENOMEM -> std::runtime_error/bad_alloc.
 * twg_last_error() returns the message of the last failure on this thread.
 *
 * Threading: one twg_ctx per (host thread, GPU); calls on a ctx are
 * stream-ordered on the ctx's stream and not thread-safe per ctx (the
 * reference's single-writer rule, window_manager.hpp:27-30). Stores are
 * immutable and reference counted; any number of generations may read a
 * store while a window ingests the next batch.
 */
#ifndef TWG_H
#define TWG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TWG_ABI_VERSION 1

enum {
  TWG_OK = 0,
  TWG_EINVAL = 1,
  TWG_ERANGE = 2,
  TWG_ELOGIC = 3,
  TWG_ECUDA = 4,
  TWG_ENOMEM = 5,
  TWG_EPARSE = 6  /* timewalk::ParseError (io.hpp:15-23): see *error_line */
};

/* types.hpp:28-34 — AoS, 24 bytes, layout-identical to timewalk::TemporalEdge */
typedef struct twg_edge {
  int64_t src;
  int64_t dst;
  int64_t t;
} twg_edge;

/* types.hpp:39-45 */
enum { TWG_FORWARD = 0, TWG_BACKWARD = 1, TWG_UNDIRECTED = 2 };   /* DirectionMode */
enum { TWG_WALK_FORWARD = 0, TWG_WALK_BACKWARD = 1 };              /* WalkDirection */
/* samplers.hpp:11-16 BiasKind */
enum { TWG_UNIFORM = 0, TWG_LINEAR = 1, TWG_EXPINDEX = 2, TWG_EXPWEIGHT = 3 };
/* walk_engine.hpp:34 Variant */
enum { TWG_COOP = 0, TWG_COOP_DIRECT = 1, TWG_FULLWALK = 2 };
/* RNG stream: the reference's splitmix CounterRng (rng.hpp:22-43, default,
 * bit-exact with the unmodified reference) or Philox4x32-10 keyed by
 * (seed; walk, hop, ordinal) (bit-exact with oracle/philox_shadow). */
enum { TWG_RNG_SPLITMIX = 0, TWG_RNG_PHILOX = 1 };

typedef struct twg_ctx twg_ctx;
typedef struct twg_store twg_store;
typedef struct twg_window twg_window;
typedef struct twg_walkset twg_walkset;

int twg_abi_version(void);
const char* twg_last_error(void);

/* ---- context: device, stream, stream-ordered memory pool ---------------- */
int twg_ctx_create(int device, twg_ctx** out);
/* priority > 0: the compute stream gets the device's greatest priority (e.g.
 * the ingest context of a pipeline whose walks run on a second context). */
int twg_ctx_create_prio(int device, int priority, twg_ctx** out);
int twg_ctx_destroy(twg_ctx* ctx);
int twg_ctx_sync(twg_ctx* ctx);
/* the cudaStream_t (as void*) all calls on ctx are ordered on */
int twg_ctx_stream(twg_ctx* ctx, void** stream);
/* device kernels launched by this ctx since creation (instrumentation) */
int twg_ctx_launch_count(twg_ctx* ctx, uint64_t* count);

/* ---- EdgeStore ----------------------------------------------------------- */
typedef struct twg_build_opts {
  int32_t weights;    /* 1: build node/ts exp-weight prefixes (reference always does) */
  int32_t adjacency;  /* 1: build sorted unique neighbour lists (node2vec) */
} twg_build_opts;   /* NULL = both on (reference behaviour, edge_store.cpp:100-110,216-250) */

/* EdgeStore::build over host edges (any order). mode: TWG_FORWARD/... */
int twg_store_build(twg_ctx* ctx, const twg_edge* edges, uint64_t n, int mode,
                    const twg_build_opts* opts, twg_store** out);
/* Same over device-resident SoA arrays (no host copy). */
int twg_store_build_device(twg_ctx* ctx, const int64_t* d_src, const int64_t* d_dst,
                           const int64_t* d_t, uint64_t n, int mode, const twg_build_opts* opts,
                           twg_store** out);
int twg_store_retain(twg_store* s);
int twg_store_release(twg_store* s);

typedef struct twg_store_info {
  uint64_t edges;        /* m   edge_count()        */
  uint64_t nodes;        /* V   node_count()        */
  uint64_t ts_groups;    /* Z   ts_group_count()    */
  uint64_t entries;      /* P   node-view entries (m, or 2m undirected) */
  uint64_t node_groups;  /* Q   per-node timestamp groups */
  uint64_t adjacency;    /* A   unique (node, neighbour) pairs; 0 if not built */
  int32_t mode;
  int32_t has_weights;
  int32_t has_adjacency;
  int32_t streaming;     /* 1: slice of the shared append log / node arena (time-ordered stream fast path) */
  uint64_t device_bytes; /* bytes held by the snapshot's device arrays */
} twg_store_info;
int twg_store_get_info(twg_store* s, twg_store_info* out);

/* Streaming-representation layout of a snapshot (diagnostics and tests: the
 * regime a parity run reached). Zero for contiguous stores. */
typedef struct twg_store_layout {
  uint64_t log_cap;         /* edge-log ring slots */
  uint64_t log_first;       /* logical position of edge 0 (wrapped iff log_first + edges > log_cap) */
  uint64_t ts_first;        /* logical position of ts group 0 */
  uint64_t arena_cap;       /* node-arena slots */
  uint64_t arena_used;      /* bump pointer after the ingest that made this snapshot */
  uint64_t arena_serial;    /* changes when the arena is replaced (repack) */
  uint64_t relocated_rings; /* rings moved by the ingest that made this snapshot */
  uint64_t max_ring_end;    /* largest logical entry end (ee) over the snapshot's nodes */
} twg_store_layout;
int twg_store_get_layout(twg_store* s, twg_store_layout* out);

/* Field ids for twg_store_download (host destination, exact element types):
 *  0 edge src external i64[m]      1 edge dst external i64[m]    2 edge time i64[m]
 *  3 edge src internal u32[m]      4 edge dst internal u32[m]
 *  5 ts offsets u64[Z+1]           6 ts times i64[Z]             7 ts weight prefix f64[Z]
 *  8 node offsets u64[V+1]         9 node ts index u64[V+1]
 * 10 mark times i64[Q]            11 mark starts u32[Q]
 * 12 ref edge u32[P]              13 node weight prefix f64[P]   14 external ids i64[V]
 * 15 ref neighbour u32[P]         16 adjacency offsets u64[V+1]  17 adjacency u32[A]
 * Lazily builds weights / adjacency if the store was built without them. */
int twg_store_download(twg_store* s, int field, void* host_dst);

/* Batched temporal_neighborhood on external ids: out3 = (start, end,
 * group_count) per query; unknown ids give an empty range at 0. */
int twg_store_neighborhood(twg_store* s, const int64_t* v_ext, const int64_t* t, uint64_t n,
                           int walk_direction, uint64_t* out3);
/* Batched external -> internal lookup; found[i] = 0/1. */
int twg_store_find_nodes(twg_store* s, const int64_t* v_ext, uint64_t n, uint32_t* internal,
                         uint8_t* found);
/* Batched adjacency on internal ids. temporal=0: adjacent(a,b);
 * temporal=1: adjacent_after(a,b,t[i],walk_direction). */
int twg_store_adjacent(twg_store* s, const uint32_t* a, const uint32_t* b, uint64_t n,
                       int temporal, const int64_t* t, int walk_direction, uint8_t* out);

/* ---- WindowManager -------------------------------------------------------- */
/* window_manager.hpp:18-25 */
typedef struct twg_batch_stats {
  uint64_t ingested;
  uint64_t dropped_late;
  uint64_t evicted;
  uint64_t retained;
  double rebuild_duration; /* seconds */
  uint64_t peak_bytes;     /* device bytes: live snapshots + batch + scratch high-water */
} twg_batch_stats;

int twg_window_create(twg_ctx* ctx, int64_t duration, int mode, const twg_build_opts* opts,
                      twg_window** out);
int twg_window_destroy(twg_window* w);
int twg_window_ingest(twg_window* w, const twg_edge* batch, uint64_t n, twg_batch_stats* out);
/* Device-resident batch (SoA). stats may be NULL to skip the statistics
 * read-back. The call is NOT asynchronous: the route decision (append vs
 * rebuild), the ring plan and the new snapshot's counts are read back to the
 * host (a few scalar read-backs per batch), so it returns with the snapshot
 * published and the stream drained up to that point. */
int twg_window_ingest_device(twg_window* w, const int64_t* d_src, const int64_t* d_dst,
                             const int64_t* d_t, uint64_t n, twg_batch_stats* out);
/* Streaming pipeline (double-buffered host ingest). twg_stage_batch enqueues
 * the H2D copy of a host batch (pinned memory for real overlap) into device
 * slot 0 or 1 on the ctx's copy stream and returns; twg_window_ingest_staged
 * ingests a staged slot on the compute stream after its copy lands. Staging
 * batch k+1 before ingesting batch k overlaps PCIe with the rebuild. The
 * host buffer must stay untouched until the slot is re-staged or the ctx is
 * synchronised. */
int twg_stage_batch(twg_ctx* ctx, int slot, const twg_edge* batch, uint64_t n);
int twg_window_ingest_staged(twg_window* w, int slot, twg_batch_stats* out);
/* current snapshot (+1 reference; release with twg_store_release) */
int twg_window_snapshot(twg_window* w, twg_store** out);
int twg_window_bounds(twg_window* w, int64_t* lo, int64_t* hi);
int twg_window_state(twg_window* w, int64_t* t_high, uint64_t* batch_count,
                     twg_batch_stats* last);

/* ---- walks ------------------------------------------------------------------ */
/* walk_engine.hpp:16-24 */
typedef struct twg_thresholds {
  uint32_t w_warp;      /* 4    */
  uint32_t block_dim;   /* 256  */
  uint32_t w_max;       /* 8192 */
  uint32_t g_warp_cap;  /* 512  */
  uint32_t g_block_cap; /* 4096 */
} twg_thresholds;

/* walk_engine.hpp:36-49, plus the RNG stream and an optional shard of the
 * global walk-id space [walk_begin, walk_end) for multi-GPU partitioning
 * (0,0 = all walks). RNG draws are keyed by GLOBAL walk ids, so the union of
 * shards equals the unsharded WalkSet byte for byte. */
typedef struct twg_walk_config {
  uint32_t walk_length;     /* 80 */
  int32_t start_mode;       /* 0 per-node, 1 sampled */
  uint32_t walks_per_node;  /* 10 */
  uint32_t _pad0;
  uint64_t total_walks;     /* sampled mode */
  int32_t bias;             /* TWG_EXPWEIGHT */
  int32_t start_bias;       /* TWG_UNIFORM */
  int32_t node2vec;         /* 0/1 */
  int32_t temporal_adjacency;
  double p, q;
  int32_t direction;        /* TWG_WALK_FORWARD */
  int32_t rng;              /* TWG_RNG_SPLITMIX */
  uint64_t seed;
  uint64_t walk_begin;
  uint64_t walk_end;
} twg_walk_config;

/* walk_engine.hpp:112-131 (+ draws whose floor could differ from glibc by
 * one ulp: counted, expected 0) */
typedef struct twg_walk_stats {
  uint64_t walks;
  uint64_t hops;
  uint64_t steps;
  uint64_t solo, warp_cached, warp_direct, block_cached, block_direct, multi_block;
  double wall_seconds;
  uint64_t ambiguous_draws;
  uint64_t alg_bytes;  /* SURVEY §8(d) algorithmic bytes summed over the hops (roofline numerator) */
} twg_walk_stats;

/* generate_walks. The WalkSet stays on the device until downloaded.
 * thresholds may be NULL (defaults). */
int twg_generate(twg_ctx* ctx, twg_store* s, const twg_walk_config* config,
                 const twg_thresholds* thresholds, int variant, twg_walkset** out,
                 twg_walk_stats* stats);
int twg_walkset_destroy(twg_walkset* w);
/* stride, walk_count (of this shard), first global walk id, total hops */
int twg_walkset_info(twg_walkset* w, uint32_t* stride, uint64_t* walk_count,
                     uint64_t* first_walk, uint64_t* hops);
/* Fixed-stride image (walk_engine.hpp:55-70): nodes/times [walk_count*stride],
 * unused slots zero; lengths [walk_count]. Any pointer may be NULL. */
int twg_walkset_download(twg_walkset* w, int64_t* nodes, int64_t* times, uint32_t* lengths);
/* Compact image: offsets[walk_count+1] (u64) into nodes/times of total
 * sum(lengths) entries — only the recorded entries cross PCIe. */
int twg_walkset_download_compact(twg_walkset* w, uint64_t* offsets, int64_t* nodes,
                                 int64_t* times);
/* Asynchronous compact download: compaction on the compute stream, the D2H
 * copies on the ctx's download stream (overlapping the next batch). Host
 * buffers (pinned for real overlap) must hold `capacity` entries; *total
 * receives the entry count. twg_walkset_wait blocks until the data landed
 * (destroy also waits). */
int twg_walkset_download_compact_async(twg_walkset* w, uint64_t* offsets, int64_t* nodes, int64_t* times,
                                       uint64_t capacity, uint64_t* total_entries);
int twg_walkset_wait(twg_walkset* w);
/* Device views (valid until destroy). The device layout is SLOT-MAJOR:
 * cell (walk w, slot j) is at [j * walk_count + w]; slots >= lengths[w] are
 * undefined. (The downloads above produce the walk-major images.) */
int twg_walkset_device(twg_walkset* w, int64_t** d_nodes, int64_t** d_times,
                       uint32_t** d_lengths);

/* Causality audit on the device: timewalk::check_walkset (validity.cpp:108-120,
 * check_timed_walk :32-66) of every emitted walk (length >= 2) of w against
 * the edges of s, independent of the node view (a (source, target, time)-
 * sorted copy of the edge list, as EdgeOracle, :14-30). direction: 0 forward,
 * 1 backward; strict: strict time order. first_violation (optional, host,
 * walk_count entries): each walk's first invalid hop, or -1. */
typedef struct twg_audit_report {
  uint64_t walks, valid_walks, hops, valid_hops;
} twg_audit_report;
int twg_walkset_audit(twg_walkset* w, twg_store* s, int direction, int strict, int64_t* first_violation,
                      twg_audit_report* out);

/* Walk writers (io.cpp:119-135 write_walks_text, io.cpp:173-183
 * write_walks_binary), serialised on the device so only the finished bytes
 * cross PCIe. Each call sets *len to the image size; with dst != NULL the
 * image is copied there (cap >= *len, else TWG_EINVAL). Text: one line per
 * walk of length >= 2, `node@time` entries separated by ' ', a start
 * sentinel as `node@-`, '\n' per line. Binary: "TMPW0002", u32 stride,
 * u64 walk_count, walk-major i64 nodes and times (zero past each length),
 * u32 lengths — byte-identical to the reference's writers. */
int twg_walkset_text(twg_walkset* w, void* dst, uint64_t cap, uint64_t* len);
int twg_walkset_binary(twg_walkset* w, void* dst, uint64_t cap, uint64_t* len);
/* Edge lists on the device and the edge-file formats (io.cpp:40-69).
 * twg_parse_edges_tsv: read_edges_tsv on the device — `source<TAB>target<TAB>
 * timestamp` lines, '#' and blank lines skipped, a trailing '\r' dropped,
 * non-negative int64 fields; text = host bytes (one H2D). A malformed line
 * returns TWG_EPARSE with *error_line = its 1-based number and
 * twg_last_error() = the reference's ParseError text without the
 * " (line N)" suffix. The result stays on the device: count, AoS download,
 * SoA device views (ready for twg_window_ingest_device; valid until
 * destroy). twg_edges_format_tsv: write_edges_tsv on the device (*len =
 * size; copied to dst when non-NULL, cap >= *len). */
typedef struct twg_edges twg_edges;
int twg_parse_edges_tsv(twg_ctx* ctx, const char* text, uint64_t bytes, twg_edges** out,
                        uint64_t* error_line);
int twg_edges_from_host(twg_ctx* ctx, const twg_edge* edges, uint64_t n, twg_edges** out);
int twg_edges_info(twg_edges* e, uint64_t* count);
int twg_edges_download(twg_edges* e, twg_edge* out);
int twg_edges_device(twg_edges* e, int64_t** d_src, int64_t** d_dst, int64_t** d_t);
int twg_edges_format_tsv(twg_edges* e, char* dst, uint64_t cap, uint64_t* len);
int twg_edges_destroy(twg_edges* e);
/* A device walk set from a host WalkSet image (walk_engine.hpp:55-70:
 * walk-major nodes/times [walk_count * stride], lengths [walk_count]) — the
 * façade's io over host WalkSets. */
int twg_walkset_from_host(twg_ctx* ctx, uint32_t stride, uint64_t walk_count, const int64_t* nodes,
                          const int64_t* times, const uint32_t* lengths, twg_walkset** out);

/* sample_start_edge over the store for n (u1, u2) pairs -> time-sorted edge index */
int twg_sample_start_edges(twg_store* s, int bias, const double* u1, const double* u2, uint64_t n,
                           uint64_t* out);

/* schedule_step for explicit walk populations (the reference unit-test
 * fixture, test_walk_engine.cpp:16-29): walks at internal nodes with alive
 * flags; returns the five list sizes and per-task rows
 * (node, begin, end, sub_index, sub_count, tier) in list order, up to cap. */
int twg_schedule_step(twg_store* s, const uint32_t* node_of_walk, const uint8_t* alive, uint64_t n,
                      const twg_thresholds* thresholds, uint64_t* sizes5, uint32_t* rows,
                      uint64_t cap, uint32_t* walk_ids);

/* init_walks (walk_engine.hpp:136-137) as a device round trip. Call once with
 * all array pointers NULL to get stride and walk_count, then again with host
 * arrays of walk_count (states) and walk_count*stride (walks) elements.
 * WalkStates columns: current u32, time i64, prev u32, has_prev u8, alive u8,
 * length u32. Walk slots not written by init are zero. */
int twg_init_walks(twg_ctx* ctx, twg_store* s, const twg_walk_config* config, uint32_t* stride,
                   uint64_t* walk_count, uint32_t* current, int64_t* time, uint32_t* prev,
                   uint8_t* has_prev, uint8_t* alive, uint32_t* length, int64_t* nodes, int64_t* times);

/* execute_task (walk_engine.hpp:153-155): one hop (hop_walk,
 * walk_engine.cpp:88-145) for each listed walk id, updating the host
 * WalkStates / WalkSet arrays in place (device round trip). */
int twg_hop_walks(twg_ctx* ctx, twg_store* s, const twg_walk_config* config, const uint32_t* walk_ids,
                  uint64_t n_ids, uint64_t walk_count, uint32_t stride, uint32_t* current, int64_t* time,
                  uint32_t* prev, uint8_t* has_prev, uint8_t* alive, uint32_t* length, int64_t* nodes,
                  int64_t* times);

/* ---- multi-GPU replica group (replaces the loop of replay_stream,
 * replay.cpp:16-53, across GPUs) ---------------------------------------------
 * One process per GPU, each with its own twg_ctx; the group owns two NCCL
 * communicators over NVLink (data: batch broadcasts on the group's copy
 * stream; control: replica hashes and walk-statistic reductions on the ctx
 * stream). The window index is REPLICATED: every batch is broadcast once from
 * the root into every rank's staging slot (16 B/edge: u32 ids + i64 time when
 * every id fits 32 bits, else the 24-B triple) and every rank runs the same
 * deterministic ingest; a 64-bit hash of each replica's new index is
 * all-reduced so disagreement is detected on the batch that causes it. Walks
 * are PARTITIONED: rank r generates a contiguous slice of the GLOBAL walk-id
 * range (RNG draws are keyed by global ids, so the union of the ranks' walk
 * sets equals one GPU generating every id, byte for byte).
 * Every rank calls every group function, in the same order. */
typedef struct twg_group twg_group;
#define TWG_GROUP_ID_BYTES 128
/* the rendezvous id (ncclUniqueId): created by one rank, shared out of band */
int twg_group_unique_id(uint8_t id[TWG_GROUP_ID_BYTES]);
int twg_group_create(twg_ctx* ctx, int nranks, int rank, const uint8_t id[TWG_GROUP_ID_BYTES],
                     twg_group** out);
int twg_group_destroy(twg_group* g);
int twg_group_info(twg_group* g, int* nranks, int* rank);

typedef struct twg_group_batch_stats {
  twg_batch_stats local;          /* this replica's BatchStats (equal on every rank) */
  uint64_t replica_hash;          /* hash of this replica's snapshot after the batch */
  int32_t replicas_agree;         /* 1 iff every rank's hash is equal (all-reduced min == max) */
  int32_t wire_bytes_per_edge;    /* bytes per edge the broadcast moved (16 or 24) */
  uint64_t edges;                 /* batch size as broadcast by the root */
} twg_group_batch_stats;

/* Broadcast one batch from `root` into staging slot 0/1 of every rank, on the
 * group's copy stream (returns once enqueued: stage batch k+1 while batch k is
 * ingested/walked). The root passes its batch as device SoA columns (staged
 * variant) or host AoS edges (host variant: one H2D on the root); the other
 * ranks pass NULL / 0 and learn n from the root. */
int twg_group_stage_device(twg_group* g, int slot, int root, const int64_t* d_src, const int64_t* d_dst,
                           const int64_t* d_t, uint64_t n);
int twg_group_stage_host(twg_group* g, int slot, int root, const twg_edge* batch, uint64_t n);
/* edge count of the batch staged in a slot (as broadcast by the root; 0 is
 * the replay end-of-stream marker) */
int twg_group_staged_edges(twg_group* g, int slot, uint64_t* n);
/* Ingest a staged slot into this rank's replica (ctx stream waits for the
 * slot's broadcast), then hash the new snapshot and all-reduce the hashes. */
int twg_group_ingest_staged(twg_group* g, twg_window* w, int slot, twg_group_batch_stats* out);
/* stage + ingest in one call */
int twg_group_ingest_device(twg_group* g, twg_window* w, int root, const int64_t* d_src, const int64_t* d_dst,
                            const int64_t* d_t, uint64_t n, twg_group_batch_stats* out);
int twg_group_ingest(twg_group* g, twg_window* w, int root, const twg_edge* batch, uint64_t n,
                     twg_group_batch_stats* out);
/* This rank's shard of generate_walks: the walk-id range [walk_begin,
 * walk_end) of config (0,0 = every walk) split into nranks contiguous,
 * balanced slices. local: this rank's WalkStats; global (optional): the
 * counters summed over ranks (wall_seconds = max over ranks). */
int twg_group_generate(twg_group* g, twg_store* s, const twg_walk_config* config,
                       const twg_thresholds* thresholds, int variant, twg_walkset** out,
                       twg_walk_stats* local, twg_walk_stats* global);
/* The replica hash of one snapshot (what twg_group_ingest_staged all-reduces):
 * node meta, external ids, counts and the newest `tail` edges (0 = all). */
int twg_store_replica_hash(twg_store* s, uint64_t tail, uint64_t* hash);

/* ---- primitives (primitives.hpp:11-31), device implementations -------------- */
/* stable LSD radix sort of (u64 key, u32 value) pairs, in place (host arrays) */
int twg_radix_sort_pairs(twg_ctx* ctx, uint64_t* keys, uint32_t* values, uint64_t n);
/* exclusive scan of u64 (out may alias in); returns the total */
int twg_exclusive_scan(twg_ctx* ctx, const uint64_t* in, uint64_t* out, uint64_t n, uint64_t* total);
/* run-length encode of a sorted key sequence: runs (key u64, start u32,
 * length u32) into out (capacity n rows of 3 u64); *runs = count */
int twg_run_length_encode(twg_ctx* ctx, const uint64_t* sorted_keys, uint64_t n, uint64_t* out_rows,
                          uint64_t* runs);
/* stable compaction of items whose flags[item] != 0 (flags indexed by item) */
int twg_partition_flagged(twg_ctx* ctx, const uint32_t* items, uint64_t n, const uint8_t* flags,
                          uint64_t flags_len, uint32_t* out, uint64_t* kept);

/* ---- samplers (device evaluation of the closed forms) ----------------------- */
/* kind 0 uniform, 1 linear, 2 exponential; u in [0,1), n >= 1 */
int twg_pick_index(twg_ctx* ctx, int kind, const double* u, const uint64_t* n, uint64_t count,
                   uint64_t* out);
int twg_pick_weighted_range(twg_ctx* ctx, const double* u, const double* prefix, uint64_t len,
                            const uint64_t* begin, const uint64_t* end, const double* base,
                            uint64_t count, uint64_t* out);
/* raw RNG draws (walk, hop, ordinal) for the chosen stream */
int twg_rng_bits(twg_ctx* ctx, int rng, uint64_t seed, const uint64_t* walk, const uint64_t* hop,
                 const uint64_t* ordinal, uint64_t count, uint64_t* out);

/* ---- synthetic inputs (generators for the benches; synthetic.cpp:17-99) ---- */
/* C5 stream law, edges [first, first+count), written to host
 * memory (pinned or not) by the host's cores. */
int twg_synth_stream_host(uint64_t nodes, uint64_t first, uint64_t count, uint64_t seed,
                          twg_edge* out);
/* Same law generated directly into device SoA arrays on the ctx stream. */
int twg_synth_stream_device(twg_ctx* ctx, uint64_t nodes, uint64_t first, uint64_t count,
                            uint64_t seed, int64_t* d_src, int64_t* d_dst, int64_t* d_t);
/* The reference's synthetic graphs (synthetic.hpp:10-35) into host AoS
 * edges, bit-identical: kind 0 make_uniform_graph(a nodes, b edges, t_max),
 * 1 make_hub_skewed_graph(a background nodes, b background edges),
 * 2 make_mega_hub_graph(a feeders), 3 make_time_ladder_graph(a edges, b
 * rungs). *count = the edge count; out (cap >= *count) may be NULL. */
int twg_synth_graph(twg_ctx* ctx, int kind, uint64_t a, uint64_t b, int64_t t_max, uint64_t seed,
                    twg_edge* out, uint64_t cap, uint64_t* count);
/* make_uniform_graph (synthetic.cpp:24-36) into device SoA arrays */
int twg_synth_uniform_device(twg_ctx* ctx, uint64_t nodes, uint64_t count, int64_t t_max,
                             uint64_t seed, int64_t* d_src, int64_t* d_dst, int64_t* d_t);

#ifdef __cplusplus
}
#endif
#endif /* TWG_H */
