// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference core (`/root/reference/proj/core`,
// public API only). `oracle/Makefile` compiles this file together with the
// reference's own sources into `oracle/_ref/libtimewalk_ref*.so`. It is used
//   * by tests/ to pin the C restatement (`oracle/tw_oracle.c`) against the
//     real reference, and to make the golden fixtures under tests/golden/;
//   * by bench.py's `cpu_baseline` leg and `--impl reference` arm, which time
//     the reference's own CPU implementation of the hot path.
//
// Every accessor below goes through the reference's public headers
// (edge_store.hpp:54-166, window_manager.hpp:31-62, walk_engine.hpp:136-171,
// replay.hpp:36-37, samplers.hpp:42-89, synthetic.hpp).

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <sstream>

#include "timewalk/edge_store.hpp"
#include "timewalk/io.hpp"
#include "timewalk/replay.hpp"
#include "timewalk/rng.hpp"
#include "timewalk/samplers.hpp"
#include "timewalk/synthetic.hpp"
#include "timewalk/validity.hpp"
#include "timewalk/walk_engine.hpp"
#include "timewalk/window_manager.hpp"

using namespace timewalk;

namespace {

thread_local std::string g_error;

// 0 ok, 1 invalid_argument, 2 out_of_range, 3 logic_error, 4 other
int classify(const std::exception& e) {
  g_error = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::out_of_range*>(&e)) return 2;
  if (dynamic_cast<const std::logic_error*>(&e)) return 3;
  return 4;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

struct StoreH {
  std::shared_ptr<const EdgeStore> store;
};

struct WindowH {
  std::unique_ptr<WindowManager> window;
};

struct ReplayH {
  std::vector<BatchRecord> records;
  std::vector<WalkSet> walks;
};

}  // namespace

extern "C" {

struct twref_edge {
  int64_t src, dst, t;
};
static_assert(sizeof(twref_edge) == sizeof(TemporalEdge));

struct twref_walk_config {
  uint32_t walk_length;
  int32_t start_mode;  // 0 per-node, 1 sampled
  uint32_t walks_per_node;
  uint32_t _pad0;
  uint64_t total_walks;
  int32_t bias;
  int32_t start_bias;
  int32_t node2vec;  // 0/1
  int32_t temporal_adjacency;
  double p, q;
  int32_t direction;  // 0 forward, 1 backward
  int32_t _pad1;
  uint64_t seed;
};

struct twref_thresholds {
  uint32_t w_warp, block_dim, w_max, g_warp_cap, g_block_cap;
};

struct twref_walk_stats {
  uint64_t walks, hops, steps;
  uint64_t solo, warp_cached, warp_direct, block_cached, block_direct, multi_block;
  double wall_seconds;
};

struct twref_batch_stats {
  uint64_t ingested, dropped_late, evicted, retained;
  double rebuild_duration;
  uint64_t peak_bytes;
};

const char* twref_last_error() { return g_error.c_str(); }

// ---- generators (synthetic.hpp) ---------------------------------------------

void* twref_gen_uniform(uint64_t nodes, uint64_t edges, int64_t t_max, uint64_t seed) {
  return new std::vector<TemporalEdge>(make_uniform_graph(nodes, edges, t_max, seed));
}
void* twref_gen_hub_skewed(uint64_t bg_nodes, uint64_t bg_edges, uint64_t seed) {
  return new std::vector<TemporalEdge>(make_hub_skewed_graph(bg_nodes, bg_edges, seed));
}
void* twref_gen_mega_hub(uint32_t feeders, uint64_t seed) {
  return new std::vector<TemporalEdge>(make_mega_hub_graph(feeders, seed));
}
void* twref_gen_time_ladder(uint64_t edges, uint32_t rungs, uint64_t seed) {
  return new std::vector<TemporalEdge>(make_time_ladder_graph(edges, rungs, seed));
}
uint64_t twref_edges_size(void* h) { return static_cast<std::vector<TemporalEdge>*>(h)->size(); }
void twref_edges_copy(void* h, twref_edge* out) {
  auto* v = static_cast<std::vector<TemporalEdge>*>(h);
  std::memcpy(out, v->data(), v->size() * sizeof(TemporalEdge));
}
void twref_edges_free(void* h) { delete static_cast<std::vector<TemporalEdge>*>(h); }

uint64_t twref_rng_bits(uint64_t seed, uint64_t walk, uint64_t hop, uint64_t ordinal) {
  return CounterRng(seed).bits(walk, hop, ordinal);
}
double twref_rng_uniform(uint64_t seed, uint64_t walk, uint64_t hop, uint64_t ordinal) {
  return CounterRng(seed).uniform(walk, hop, ordinal);
}

// ---- samplers (samplers.hpp:42-89) ------------------------------------------

// kind: 0 uniform, 1 linear, 2 exponential index pickers
int twref_pick(int kind, const double* u, const uint64_t* n, uint64_t count, uint64_t* out) {
  return guarded([&] {
    for (uint64_t i = 0; i < count; ++i) {
      switch (kind) {
        case 0: out[i] = pick_index_uniform(u[i], n[i]); break;
        case 1: out[i] = pick_index_linear(u[i], n[i]); break;
        case 2: out[i] = pick_index_exponential(u[i], n[i]); break;
        default: throw std::invalid_argument("twref_pick: kind");
      }
    }
  });
}

int twref_pick_weighted_range(double u, const double* prefix, uint64_t len, uint64_t begin,
                              uint64_t end, double base, uint64_t* out) {
  return guarded([&] {
    *out = pick_weighted_range(u, std::span<const double>(prefix, len), begin, end, base);
  });
}

int twref_oracle_pick(double u, const double* weights, uint64_t n, uint64_t* out) {
  return guarded([&] { *out = oracle_pick(u, std::span<const double>(weights, n)); });
}

// ---- edge store (edge_store.hpp) --------------------------------------------

void* twref_store_build(const twref_edge* edges, uint64_t n, int mode, int* status) {
  StoreH* h = nullptr;
  *status = guarded([&] {
    auto span = std::span<const TemporalEdge>(reinterpret_cast<const TemporalEdge*>(edges), n);
    h = new StoreH{std::make_shared<const EdgeStore>(
        EdgeStore::build(span, static_cast<DirectionMode>(mode)))};
  });
  return h;
}

void twref_store_free(void* h) { delete static_cast<StoreH*>(h); }

// out: m, V, Z, P (entries), Q (node ts groups), mode, memory_bytes
void twref_store_counts(void* h, uint64_t* out) {
  const EdgeStore& s = *static_cast<StoreH*>(h)->store;
  uint64_t entries = 0, groups = 0;
  for (InternalNode v = 0; v < s.node_count(); ++v) {
    const auto [lo, hi] = s.node_region(v);
    entries += hi - lo;
    groups += s.timestamp_group_count_internal(v);
  }
  out[0] = s.edge_count();
  out[1] = s.node_count();
  out[2] = s.ts_group_count();
  out[3] = entries;
  out[4] = groups;
  out[5] = static_cast<uint64_t>(s.direction_mode());
  out[6] = s.memory_bytes();
}

// Field ids (keep in sync with oracle/tw_oracle.h TWO_F_*).
//  0 edge src ext i64[m]   1 edge dst ext i64[m]   2 edge time i64[m]
//  3 edge src int u32[m]   4 edge dst int u32[m]
//  5 ts_off u64[Z+1]       6 ts_time i64[Z]        7 ts_weight f64[Z]
//  8 node_off u64[V+1]     9 node_tsidx u64[V+1]
// 10 mark time i64[Q]     11 mark start u32[Q]
// 12 ref_edge u32[P]      13 weight_prefix f64[P]  14 ext_id i64[V]
// 15 ref_neighbor u32[P]
int twref_store_dump(void* hh, int field, void* out) {
  return guarded([&] {
    const EdgeStore& s = *static_cast<StoreH*>(hh)->store;
    const uint64_t m = s.edge_count(), V = s.node_count(), Z = s.ts_group_count();
    switch (field) {
      case 0: case 1: case 2: {
        auto* o = static_cast<int64_t*>(out);
        for (uint64_t i = 0; i < m; ++i) {
          const TemporalEdge e = s.edge_at(i);
          o[i] = field == 0 ? e.source : field == 1 ? e.target : e.time;
        }
        break;
      }
      case 3: case 4: {
        auto* o = static_cast<uint32_t*>(out);
        for (uint64_t i = 0; i < m; ++i) {
          o[i] = field == 3 ? s.edge_source_internal(i) : s.edge_target_internal(i);
        }
        break;
      }
      case 5: {
        auto* o = static_cast<uint64_t*>(out);
        for (uint64_t g = 0; g < Z; ++g) o[g] = s.edge_slice_for_ts_group(g).first;
        o[Z] = m;
        break;
      }
      case 6: {
        auto* o = static_cast<int64_t*>(out);
        for (uint64_t g = 0; g < Z; ++g) o[g] = s.ts_group_time(g);
        break;
      }
      case 7: {
        const auto w = s.ts_group_weight_prefix();
        std::memcpy(out, w.data(), w.size() * sizeof(double));
        break;
      }
      case 8: case 9: {
        auto* o = static_cast<uint64_t*>(out);
        uint64_t acc = 0;
        for (InternalNode v = 0; v < V; ++v) {
          if (field == 8) {
            o[v] = s.node_region(v).first;
          } else {
            o[v] = acc;
            acc += s.timestamp_group_count_internal(v);
          }
        }
        if (V == 0) {
          o[0] = 0;
        } else {
          o[V] = field == 8 ? s.node_region(static_cast<InternalNode>(V - 1)).second : acc;
        }
        break;
      }
      case 10: case 11: {
        uint64_t q = 0;
        for (InternalNode v = 0; v < V; ++v) {
          for (const TsGroupMark& mk : s.group_marks(v)) {
            if (field == 10) static_cast<int64_t*>(out)[q] = mk.time;
            else static_cast<uint32_t*>(out)[q] = mk.start;
            ++q;
          }
        }
        break;
      }
      case 12: case 15: {
        auto* o = static_cast<uint32_t*>(out);
        for (InternalNode v = 0; v < V; ++v) {
          const auto [lo, hi] = s.node_region(v);
          for (uint64_t pos = lo; pos < hi; ++pos) {
            o[pos] = field == 12 ? s.ref_edge(pos) : s.ref_neighbor(pos, v);
          }
        }
        break;
      }
      case 13: {
        const auto w = s.weight_prefix();
        std::memcpy(out, w.data(), w.size() * sizeof(double));
        break;
      }
      case 14: {
        auto* o = static_cast<int64_t*>(out);
        for (InternalNode v = 0; v < V; ++v) o[v] = s.external_id(v);
        break;
      }
      default:
        throw std::invalid_argument("twref_store_dump: unknown field");
    }
  });
}

int twref_store_adjacent(void* hh, const uint32_t* a, const uint32_t* b, uint64_t n,
                         uint8_t* out) {
  return guarded([&] {
    const EdgeStore& s = *static_cast<StoreH*>(hh)->store;
    for (uint64_t i = 0; i < n; ++i) out[i] = s.adjacent(a[i], b[i]) ? 1 : 0;
  });
}

// out3: start, end, group_count per query
int twref_store_neighborhood(void* hh, const int64_t* v, const int64_t* t, uint64_t n, int dir,
                             uint64_t* out3) {
  return guarded([&] {
    const EdgeStore& s = *static_cast<StoreH*>(hh)->store;
    for (uint64_t i = 0; i < n; ++i) {
      const NeighborRange r = s.temporal_neighborhood(v[i], t[i], static_cast<WalkDirection>(dir));
      out3[3 * i] = r.start;
      out3[3 * i + 1] = r.end;
      out3[3 * i + 2] = r.group_count;
    }
  });
}

// ---- window (window_manager.hpp) --------------------------------------------

void* twref_window_create(int64_t duration, int mode, int* status) {
  WindowH* h = nullptr;
  *status = guarded([&] {
    h = new WindowH{std::make_unique<WindowManager>(
        WindowConfig{duration, static_cast<DirectionMode>(mode)})};
  });
  return h;
}
void twref_window_free(void* h) { delete static_cast<WindowH*>(h); }

int twref_window_ingest(void* hh, const twref_edge* edges, uint64_t n, twref_batch_stats* out) {
  return guarded([&] {
    auto span = std::span<const TemporalEdge>(reinterpret_cast<const TemporalEdge*>(edges), n);
    const BatchStats& s = static_cast<WindowH*>(hh)->window->ingest_batch(span);
    *out = {s.ingested, s.dropped_late, s.evicted, s.retained, s.rebuild_duration, s.peak_bytes};
  });
}

void* twref_window_snapshot(void* hh) {
  return new StoreH{static_cast<WindowH*>(hh)->window->snapshot()};
}

int twref_window_bounds(void* hh, int64_t* lo, int64_t* hi) {
  return guarded([&] {
    const auto [a, b] = static_cast<WindowH*>(hh)->window->window_bounds();
    *lo = a;
    *hi = b;
  });
}

void twref_window_info(void* hh, int64_t* t_high, uint64_t* batch_count) {
  const WindowManager& w = *static_cast<WindowH*>(hh)->window;
  *t_high = w.t_high();
  *batch_count = w.batch_count();
}

// ---- walks (walk_engine.hpp) ------------------------------------------------

static WalkConfig to_config(const twref_walk_config* c) {
  WalkConfig cfg;
  cfg.walk_length = c->walk_length;
  cfg.start_mode = static_cast<StartMode>(c->start_mode);
  cfg.walks_per_node = c->walks_per_node;
  cfg.total_walks = c->total_walks;
  cfg.bias = static_cast<BiasKind>(c->bias);
  cfg.start_bias = static_cast<BiasKind>(c->start_bias);
  if (c->node2vec) cfg.node2vec = Node2VecParams{c->p, c->q};
  cfg.node2vec_temporal_adjacency = c->temporal_adjacency != 0;
  cfg.direction = static_cast<WalkDirection>(c->direction);
  cfg.seed = c->seed;
  return cfg;
}

static TierThresholds to_thresholds(const twref_thresholds* t) {
  TierThresholds th;
  if (t) {
    th.w_warp = t->w_warp;
    th.block_dim = t->block_dim;
    th.w_max = t->w_max;
    th.g_warp_cap = t->g_warp_cap;
    th.g_block_cap = t->g_block_cap;
  }
  return th;
}

static void to_stats(const WalkStats& s, twref_walk_stats* out) {
  *out = {s.walks, s.hops, s.steps, s.tiers.solo, s.tiers.warp_cached, s.tiers.warp_direct,
          s.tiers.block_cached, s.tiers.block_direct, s.tiers.multi_block, s.wall_seconds};
}

void* twref_generate(void* hh, const twref_walk_config* c, const twref_thresholds* t, int variant,
                     twref_walk_stats* stats, int* status) {
  WalkSet* out = nullptr;
  *status = guarded([&] {
    const EdgeStore& s = *static_cast<StoreH*>(hh)->store;
    WalkStats ws;
    out = new WalkSet(generate_walks(s, to_config(c), to_thresholds(t),
                                     static_cast<Variant>(variant), &ws));
    if (stats) to_stats(ws, stats);
  });
  return out;
}

uint32_t twref_walks_stride(void* h) { return static_cast<WalkSet*>(h)->stride; }
uint64_t twref_walks_count(void* h) { return static_cast<WalkSet*>(h)->walk_count; }
void twref_walks_copy(void* h, int64_t* nodes, int64_t* times, uint32_t* lengths) {
  const WalkSet& w = *static_cast<WalkSet*>(h);
  if (nodes) std::memcpy(nodes, w.nodes.data(), w.nodes.size() * sizeof(int64_t));
  if (times) std::memcpy(times, w.times.data(), w.times.size() * sizeof(int64_t));
  if (lengths) std::memcpy(lengths, w.lengths.data(), w.lengths.size() * sizeof(uint32_t));
}
void twref_walks_free(void* h) { delete static_cast<WalkSet*>(h); }

// The reference's edge TSV reader / writer (io.cpp:40-69). read: *count
// edges copied to out when cap allows; a ParseError returns 5 with its line
// in *error_line and the full what() in twref_last_error().
int twref_read_edges_tsv(const char* text, uint64_t bytes, twref_edge* out, uint64_t cap, uint64_t* count,
                         uint64_t* error_line) {
  *error_line = 0;
  try {
    std::istringstream in(std::string(text, bytes));
    const auto edges = read_edges_tsv(in);
    *count = edges.size();
    if (out && cap >= edges.size()) std::memcpy(out, edges.data(), edges.size() * sizeof(TemporalEdge));
    return 0;
  } catch (const ParseError& e) {
    g_error = e.what();
    *error_line = e.line();
    return 5;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

int twref_write_edges_tsv(const twref_edge* edges, uint64_t n, char* dst, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    std::ostringstream out;
    write_edges_tsv(out, std::span<const TemporalEdge>(reinterpret_cast<const TemporalEdge*>(edges), n));
    const std::string b = out.str();
    *len = b.size();
    if (dst && cap >= b.size()) std::memcpy(dst, b.data(), b.size());
  });
}

// The reference's walk writers (io.cpp:119-135 write_walks_text, :173-183
// write_walks_binary) over a WalkSet image: *len = bytes; copied to dst when
// dst != NULL and cap >= *len.
int twref_walks_serialize(uint32_t stride, uint64_t count, const int64_t* nodes, const int64_t* times,
                          const uint32_t* lengths, int binary, char* dst, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    WalkSet w;
    w.stride = stride;
    w.walk_count = count;
    w.nodes.assign(nodes, nodes + count * stride);
    w.times.assign(times, times + count * stride);
    w.lengths.assign(lengths, lengths + count);
    std::ostringstream out;
    if (binary) write_walks_binary(out, w);
    else write_walks_text(out, w);
    const std::string b = out.str();
    *len = b.size();
    if (dst && cap >= b.size()) std::memcpy(dst, b.data(), b.size());
  });
}

// Tier counts of one schedule_step over given walk populations at internal
// nodes (test_walk_engine.cpp:16-29 style fixtures). out: 5 task-list sizes +
// per-task (node, begin, end, sub_index, sub_count, tier) rows, up to cap rows.
int twref_schedule_step(void* hh, const uint32_t* node_of_walk, const uint8_t* alive, uint64_t n,
                        const twref_thresholds* t, uint64_t* sizes5, uint32_t* rows,
                        uint64_t cap) {
  return guarded([&] {
    const EdgeStore& s = *static_cast<StoreH*>(hh)->store;
    WalkStates st;
    st.current.assign(node_of_walk, node_of_walk + n);
    st.time.assign(n, kTimeUnset);
    st.prev.assign(n, 0);
    st.has_prev.assign(n, 0);
    st.alive.assign(alive, alive + n);
    st.length.assign(n, 1);
    std::vector<uint32_t> cand(n);
    for (uint64_t i = 0; i < n; ++i) cand[i] = static_cast<uint32_t>(i);
    const StepPlan plan = schedule_step(st, cand, s, to_thresholds(t));
    const std::vector<DispatchTask>* lists[5] = {&plan.solo, &plan.warp_cached, &plan.warp_direct,
                                                 &plan.block_cached, &plan.block_direct};
    uint64_t r = 0;
    for (int k = 0; k < 5; ++k) {
      sizes5[k] = lists[k]->size();
      for (const DispatchTask& task : *lists[k]) {
        if (r < cap) {
          uint32_t* row = rows + 6 * r;
          row[0] = task.node;
          row[1] = task.begin;
          row[2] = task.end;
          row[3] = task.sub_task_index;
          row[4] = task.sub_task_count;
          row[5] = static_cast<uint32_t>(task.tier);
        }
        ++r;
      }
    }
  });
}

// ---- replay (replay.hpp:36-37) ------------------------------------------------

struct twref_replay_config {
  int64_t batch_duration;
  int64_t window_duration;
  int32_t mode;
  int32_t variant;
  int32_t generate;
  int32_t keep_walks;
  twref_walk_config walk;
  twref_thresholds thresholds;
};

void* twref_replay(const twref_edge* edges, uint64_t n, const twref_replay_config* c,
                   uint64_t* batches, int* status) {
  ReplayH* h = new ReplayH;
  *status = guarded([&] {
    ReplayConfig cfg;
    cfg.batch_duration = c->batch_duration;
    cfg.window_duration = c->window_duration;
    cfg.mode = static_cast<DirectionMode>(c->mode);
    cfg.walk = to_config(&c->walk);
    cfg.thresholds = to_thresholds(&c->thresholds);
    cfg.variant = static_cast<Variant>(c->variant);
    cfg.generate = c->generate != 0;
    const bool keep = c->keep_walks != 0;
    auto span = std::span<const TemporalEdge>(reinterpret_cast<const TemporalEdge*>(edges), n);
    *batches = replay_stream(span, cfg, [&](const BatchRecord& r, const WalkSet& w) {
      h->records.push_back(r);
      h->walks.push_back(keep ? w : WalkSet{});
    });
  });
  if (*status != 0) {
    delete h;
    return nullptr;
  }
  return h;
}

void twref_replay_record(void* hh, uint64_t b, twref_batch_stats* ingest, twref_walk_stats* walk) {
  const BatchRecord& r = static_cast<ReplayH*>(hh)->records[b];
  const BatchStats& s = r.ingest;
  *ingest = {s.ingested, s.dropped_late, s.evicted, s.retained, s.rebuild_duration, s.peak_bytes};
  to_stats(r.walk, walk);
}
void* twref_replay_walks(void* hh, uint64_t b) { return &static_cast<ReplayH*>(hh)->walks[b]; }
void twref_replay_free(void* hh) { delete static_cast<ReplayH*>(hh); }

// ---- causality auditor (validity.hpp) ----------------------------------------

// returns (valid_walks, total_walks, valid_hops, total_hops)
int twref_check_walkset(const twref_edge* edges, uint64_t n, int undirected, uint32_t stride,
                        uint64_t walk_count, const int64_t* nodes, const int64_t* times,
                        const uint32_t* lengths, int direction, uint64_t* out4) {
  return guarded([&] {
    auto span = std::span<const TemporalEdge>(reinterpret_cast<const TemporalEdge*>(edges), n);
    const EdgeOracle oracle(span, undirected != 0);
    WalkSet ws;
    ws.stride = stride;
    ws.walk_count = walk_count;
    ws.nodes.assign(nodes, nodes + walk_count * stride);
    ws.times.assign(times, times + walk_count * stride);
    ws.lengths.assign(lengths, lengths + walk_count);
    const ValidityReport r = check_walkset(ws, oracle, static_cast<WalkDirection>(direction));
    out4[0] = r.valid_walks;
    out4[1] = r.total_walks;
    out4[2] = r.valid_hops;
    out4[3] = r.total_hops;
  });
}

}  // extern "C"
