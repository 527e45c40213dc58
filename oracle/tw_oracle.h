/* TEST INFRASTRUCTURE ONLY — the CPU oracle of the streaming temporal-walk
 * hot path. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it, and only as the checker. The product (libtimewalk_b200.so)
 * never links it and has no CPU fallback.
 *
 * Plain-C restatement of the reference core `timewalk`
 * (/root/reference/proj/core), function by function; every function cites
 * the reference file:line it follows. Pinned against the compiled reference
 * (oracle/_ref, see tests/test_oracle_pin.py) and the reference's own
 * known-answer tests (tests/test_oracle_known_answers.py).
 */
#ifndef TW_ORACLE_H
#define TW_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* types.hpp:28-34 TemporalEdge (AoS, 24 bytes) */
typedef struct {
  int64_t src, dst, t;
} two_edge;

enum { TWO_FORWARD = 0, TWO_BACKWARD = 1, TWO_UNDIRECTED = 2 }; /* types.hpp:39-43 */
enum { TWO_UNIFORM = 0, TWO_LINEAR = 1, TWO_EXPINDEX = 2, TWO_EXPWEIGHT = 3 }; /* samplers.hpp:11-16 */
enum { TWO_RNG_SPLITMIX = 0, TWO_RNG_PHILOX = 1 };
enum { TWO_OK = 0, TWO_EINVAL = 1, TWO_ERANGE = 2, TWO_ELOGIC = 3, TWO_ENOMEM = 4 };

/* rng.hpp:8-43 (splitmix CounterRng) and the Philox shadow
 * (oracle/philox_shadow/timewalk/rng.hpp). */
uint64_t two_mix64(uint64_t x);
uint64_t two_rng_bits(int kind, uint64_t seed, uint64_t walk, uint64_t hop, uint64_t ordinal);
double two_rng_uniform(int kind, uint64_t seed, uint64_t walk, uint64_t hop, uint64_t ordinal);

/* synthetic.cpp:24-141 generators; caller frees *out with two_free. */
uint64_t two_gen_uniform(uint64_t nodes, uint64_t edges, int64_t t_max, uint64_t seed, two_edge** out);
uint64_t two_gen_hub_skewed(uint64_t bg_nodes, uint64_t bg_edges, uint64_t seed, two_edge** out);
uint64_t two_gen_mega_hub(uint32_t feeders, uint64_t seed, two_edge** out);
uint64_t two_gen_time_ladder(uint64_t edges, uint32_t rungs, uint64_t seed, two_edge** out);
/* C5 stream law: edge i has src = bits(1,i,0) % N,
 * dst = min(floor(N*u^3), N-1) with u from bits(2,i,1), t = floor(i/4). */
void two_gen_stream(uint64_t nodes, uint64_t first, uint64_t count, uint64_t seed, two_edge* out);
void two_free(void* p);

/* samplers.cpp:17-103 */
int two_pick_index(int kind, double u, uint64_t n, uint64_t* out);
uint64_t two_pick_weighted(double u, const double* prefix, uint64_t n);
uint64_t two_pick_weighted_range(double u, const double* prefix, uint64_t begin, uint64_t end, double base);
uint64_t two_oracle_pick(double u, const double* weights, uint64_t n);

/* edge_store.hpp:168-199 — the dual index, SoA. */
typedef struct {
  int mode;
  uint64_t m, V, Z, P, Q, A;
  uint32_t *src, *dst; /* internal ids, canonical (time, src, dst) order */
  int64_t* t;
  int64_t* ext;        /* internal -> external id (ascending) */
  uint64_t* ts_off;    /* Z+1 */
  int64_t* ts_time;    /* Z */
  double* ts_w;        /* Z */
  uint64_t* n_off;     /* V+1 node_group_offsets_ */
  uint64_t* n_tsidx;   /* V+1 node_ts_index_ */
  int64_t* mk_time;    /* Q */
  uint32_t* mk_start;  /* Q */
  uint32_t* ref_edge;  /* P node_ref_edge_ */
  double* wprefix;     /* P node_weight_prefix_ */
  uint64_t* adj_off;   /* V+1 */
  uint32_t* adj;       /* A */
} two_store;

two_store* two_build(const two_edge* edges, uint64_t n, int mode, int* status);
void two_store_free(two_store* s);
uint32_t two_ref_neighbor(const two_store* s, uint64_t pos, uint32_t owner);
int two_find_node(const two_store* s, int64_t external, uint32_t* out);
/* out3 = start, end, group_count (edge_store.cpp:270-302) */
int two_temporal_neighborhood(const two_store* s, int64_t v, int64_t t, int dir, uint64_t* out3);
int two_adjacent(const two_store* s, uint32_t a, uint32_t b);
int two_adjacent_after(const two_store* s, uint32_t a, uint32_t b, int64_t t, int dir);
/* export_suffix (edge_store.cpp:325-332); returns count, *out malloc'ed */
uint64_t two_export_suffix(const two_store* s, int64_t cutoff, two_edge** out);

/* window_manager.hpp:11-25 / window_manager.cpp */
typedef struct {
  uint64_t ingested, dropped_late, evicted, retained;
  double rebuild_duration;
  uint64_t peak_bytes;
} two_batch_stats;

typedef struct {
  int64_t duration;
  int mode;
  two_store* store;
  int64_t t_high;
  uint64_t batch_count;
  two_batch_stats stats;
} two_window;

two_window* two_window_create(int64_t duration, int mode, int* status);
void two_window_free(two_window* w);
int two_window_ingest(two_window* w, const two_edge* batch, uint64_t n, two_batch_stats* out);
int two_window_bounds(const two_window* w, int64_t* lo, int64_t* hi);

/* walk_engine.hpp:16-131 */
typedef struct {
  uint32_t w_warp, block_dim, w_max, g_warp_cap, g_block_cap;
} two_thresholds;

typedef struct {
  uint32_t walk_length;
  int32_t start_mode; /* 0 per-node, 1 sampled */
  uint32_t walks_per_node;
  uint32_t _pad0;
  uint64_t total_walks;
  int32_t bias, start_bias;
  int32_t node2vec, temporal_adjacency;
  double p, q;
  int32_t direction, rng; /* rng: TWO_RNG_* */
  uint64_t seed;
} two_walk_config;

typedef struct {
  uint64_t walks, hops, steps;
  uint64_t solo, warp_cached, warp_direct, block_cached, block_direct, multi_block;
  double wall_seconds;
} two_walk_stats;

typedef struct {
  uint32_t stride;
  uint64_t walk_count;
  int64_t* nodes;
  int64_t* times;
  uint32_t* lengths;
} two_walkset;

/* variant: 0 Coop, 1 CoopDirect, 2 FullWalk (walk_engine.hpp:34) */
int two_generate(const two_store* s, const two_walk_config* c, const two_thresholds* t, int variant,
                 two_walkset* out, two_walk_stats* stats);
void two_walkset_free(two_walkset* w);
uint64_t two_sample_start_edge(const two_store* s, int bias, double u1, double u2);

/* replay.cpp:16-53. Records per batch. keep_walks!=0 keeps each WalkSet. */
typedef struct {
  int64_t batch_duration, window_duration;
  int32_t mode, variant, generate, keep_walks;
  two_walk_config walk;
  two_thresholds thresholds;
} two_replay_config;

typedef struct {
  uint64_t batches;
  two_batch_stats* ingest;
  two_walk_stats* walk;
  two_walkset* walks;
} two_replay_result;

int two_replay(const two_edge* edges, uint64_t n, const two_replay_config* c, two_replay_result* out);
void two_replay_free(two_replay_result* r);

#ifdef __cplusplus
}
#endif
#endif
