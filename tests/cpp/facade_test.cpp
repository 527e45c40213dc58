// Drop-in check: the reference's public C++ API, compiled against OUR
// headers (include/timewalk/*.hpp) and linked to libtimewalk_b200.so.
// Known-answer cases restate the reference's own unit tests
// (proj/tests/test_edge_store.cpp, test_window.cpp, test_samplers.cpp,
// test_walk_engine.cpp, test_replay.cpp, test_primitives.cpp); each block
// cites the test it follows. Exit code = number of failed checks.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <optional>
#include <span>
#include <numeric>
#include <set>
#include <stdexcept>
#include <thread>
#include <vector>

#include <sstream>

#include "timewalk/io.hpp"
#include "timewalk/primitives.hpp"
#include "timewalk/replay.hpp"
#include "timewalk/rng.hpp"
#include "timewalk/samplers.hpp"
#include "timewalk/synthetic.hpp"
#include "timewalk/validity.hpp"
#include "timewalk/walk_engine.hpp"
#include "timewalk/window_manager.hpp"

using namespace timewalk;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    ++g_checks;                                                         \
    if (!(cond)) {                                                      \
      ++g_fail;                                                         \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, T)      \
  do {                                \
    bool thrown_ = false;             \
    try {                             \
      (void)(expr);                   \
    } catch (const T&) {              \
      thrown_ = true;                 \
    } catch (...) {                   \
    }                                 \
    CHECK(thrown_ && #expr);          \
  } while (0)

// make_uniform_graph's law (synthetic.cpp:24-36), local to this test
static std::vector<TemporalEdge> uniform_graph(std::uint64_t nodes, std::uint64_t edges, Timestamp t_max,
                                               std::uint64_t seed) {
  const CounterRng rng(seed);
  std::vector<TemporalEdge> out;
  for (std::uint64_t i = 0; i < edges; ++i) {
    out.push_back({static_cast<NodeId>(rng.bits(1, i, 0) % nodes), static_cast<NodeId>(rng.bits(2, i, 0) % nodes),
                   static_cast<Timestamp>(rng.bits(3, i, 0) % (static_cast<std::uint64_t>(t_max) + 1))});
  }
  return out;
}

static void edge_store_cases() {
  {  // test_edge_store.cpp:31-39
    const auto s = EdgeStore::build({}, DirectionMode::DirectedForward);
    CHECK(s.edge_count() == 0 && s.node_count() == 0 && s.ts_group_count() == 0 && s.empty());
    CHECK(s.temporal_neighborhood(5, 0, WalkDirection::Forward).empty());
    CHECK(s.timestamp_group_count(5) == 0);
  }
  {  // :41-58
    const std::vector<TemporalEdge> e{{1, 2, 5}, {1, 3, 5}, {1, 4, 9}};
    const auto s = EdgeStore::build(e, DirectionMode::DirectedForward);
    CHECK(s.ts_group_count() == 2);
    CHECK((s.edge_slice_for_ts_group(0) == std::pair<std::size_t, std::size_t>{0, 2}));
    CHECK((s.edge_slice_for_ts_group(1) == std::pair<std::size_t, std::size_t>{2, 3}));
    CHECK(s.ts_group_time(0) == 5 && s.ts_group_time(1) == 9);
    const auto a = s.find_node(1);
    CHECK(a.has_value());
    const auto [lo, hi] = s.node_region(*a);
    CHECK(hi - lo == 3);
    CHECK(s.timestamp_group_count(1) == 2);
    CHECK_THROWS_AS(s.edge_slice_for_ts_group(2), std::out_of_range);
  }
  {  // :67-83 undirected mirrors entries
    const auto s = EdgeStore::build(std::vector<TemporalEdge>{{1, 2, 3}, {2, 1, 3}}, DirectionMode::Undirected);
    std::size_t total = 0;
    for (InternalNode v = 0; v < s.node_count(); ++v) total += s.node_region(v).second - s.node_region(v).first;
    CHECK(total == 4);
  }
  {  // :85-103
    const auto s = EdgeStore::build(std::vector<TemporalEdge>{{1, 2, 2}, {1, 3, 2}, {1, 4, 5}, {1, 5, 9}},
                                    DirectionMode::DirectedForward);
    CHECK(s.temporal_neighborhood(1, 2, WalkDirection::Forward).size() == 2);
    CHECK(s.temporal_neighborhood(1, 9, WalkDirection::Forward).empty());
    CHECK(s.temporal_neighborhood(1, 0, WalkDirection::Forward).size() == 4);
    CHECK(s.temporal_neighborhood(1, 2, WalkDirection::Forward).group_count == 2);
    CHECK(s.timestamp_group_count(1) == 3);
    CHECK(s.timestamp_group_count(999) == 0);
    CHECK(s.timestamp_group_count(2) == 0);
  }
  {  // :105-117
    const std::vector<TemporalEdge> e{{1, 2, 2}, {3, 2, 5}, {4, 2, 9}};
    const auto s = EdgeStore::build(e, DirectionMode::DirectedBackward);
    CHECK(s.temporal_neighborhood(2, 6, WalkDirection::Backward).size() == 2);
    CHECK(s.temporal_neighborhood(2, 2, WalkDirection::Backward).empty());
    CHECK(s.temporal_neighborhood(2, 10, WalkDirection::Backward).size() == 3);
    CHECK_THROWS_AS(s.temporal_neighborhood(2, 6, WalkDirection::Forward), std::invalid_argument);
  }
  {  // :203-213 self-loops
    const std::vector<TemporalEdge> e{{1, 1, 3}, {1, 2, 3}, {1, 2, 3}};
    CHECK(EdgeStore::build(e, DirectionMode::DirectedForward).temporal_neighborhood(1, 0, WalkDirection::Forward).size() ==
          3);
    const auto u = EdgeStore::build(e, DirectionMode::Undirected);
    const auto v = *u.find_node(1);
    CHECK(u.node_region(v).second - u.node_region(v).first == 4);
  }
  {  // :215-230 adjacency
    const std::vector<TemporalEdge> e{{1, 2, 1}, {2, 3, 2}};
    const auto s = EdgeStore::build(e, DirectionMode::DirectedForward);
    const auto n1 = *s.find_node(1), n2 = *s.find_node(2), n3 = *s.find_node(3);
    CHECK(s.adjacent(n1, n2) && !s.adjacent(n2, n1) && s.adjacent(n2, n3) && !s.adjacent(n1, n3));
    CHECK(s.adjacent_after(n1, n2, 0, WalkDirection::Forward));
    CHECK(!s.adjacent_after(n1, n2, 1, WalkDirection::Forward));
  }
  {  // :232-241 export_suffix
    const auto s = EdgeStore::build(std::vector<TemporalEdge>{{1, 2, 5}, {3, 4, 1}, {5, 6, 9}, {7, 8, 5}},
                                    DirectionMode::DirectedForward);
    const auto tail = s.export_suffix(5);
    CHECK(tail.size() == 3 && tail.front().time == 5 && tail.back().time == 9);
    CHECK(s.export_suffix(10).empty() && s.export_edges().size() == 4);
  }
  {  // :243-250
    CHECK_THROWS_AS(EdgeStore::build(std::vector<TemporalEdge>{{1, 2, -3}}, DirectionMode::DirectedForward),
                    std::invalid_argument);
    CHECK_THROWS_AS(EdgeStore::build(std::vector<TemporalEdge>{{-1, 2, 3}}, DirectionMode::DirectedForward),
                    std::invalid_argument);
  }
  {  // :184-201 permutation determinism
    auto e = uniform_graph(20, 500, 5, 77);
    const auto a = EdgeStore::build(e, DirectionMode::DirectedForward);
    std::reverse(e.begin(), e.end());
    const auto b = EdgeStore::build(e, DirectionMode::DirectedForward);
    bool same = a.edge_count() == b.edge_count();
    for (std::size_t i = 0; same && i < a.edge_count(); ++i) same = a.edge_at(i) == b.edge_at(i);
    for (InternalNode v = 0; same && v < a.node_count(); ++v) same = a.node_region(v) == b.node_region(v);
    CHECK(same);
  }
}

static std::vector<TemporalEdge> edges_at(std::initializer_list<Timestamp> times) {
  std::vector<TemporalEdge> out;
  NodeId id = 1;
  for (Timestamp t : times) {
    out.push_back({id, id + 1, t});
    id += 2;
  }
  return out;
}

static void window_cases() {
  {  // test_window.cpp:25-38
    WindowManager w({10, DirectionMode::DirectedForward});
    w.ingest_batch(edges_at({16, 18, 22, 25}));
    CHECK(w.last_batch_stats().retained == 4);
    const auto& st = w.ingest_batch(edges_at({18, 26, 30}));
    CHECK(w.t_high() == 30);
    CHECK((w.window_bounds() == std::pair<Timestamp, Timestamp>{20, 30}));
    CHECK(st.ingested == 3 && st.dropped_late == 1 && st.evicted == 2 && st.retained == 4);
  }
  {  // :40-48 empty batch: same snapshot object
    WindowManager w({10, DirectionMode::DirectedForward});
    w.ingest_batch(edges_at({5, 7}));
    const auto before = w.snapshot();
    w.ingest_batch({});
    CHECK(w.batch_count() == 2 && w.snapshot() == before && w.t_high() == 7);
  }
  {  // :50-60
    std::vector<TemporalEdge> b;
    for (Timestamp t = 1; t <= 100; ++t) b.push_back({t, t + 1000, t});
    WindowManager w({10, DirectionMode::DirectedForward});
    CHECK(w.ingest_batch(b).retained == 11);
    CHECK((w.window_bounds() == std::pair<Timestamp, Timestamp>{90, 100}));
  }
  {  // :81-85
    WindowManager w({10, DirectionMode::DirectedForward});
    CHECK_THROWS_AS(w.window_bounds(), std::logic_error);
    CHECK_THROWS_AS(WindowManager({0, DirectionMode::DirectedForward}), std::invalid_argument);
  }
  {  // :133-142 immutability
    WindowManager w({10, DirectionMode::DirectedForward});
    w.ingest_batch(edges_at({5, 7}));
    const auto old = w.snapshot();
    w.ingest_batch(edges_at({50, 60}));
    CHECK(old->edge_count() == 2 && old->edge_at(0).time == 5 && w.snapshot()->edge_count() == 2);
  }
}

static void sampler_cases() {
  // test_samplers.cpp:31-61, :95-103
  CHECK(oracle_pick(0.3, std::vector<double>{1, 2, 3}) == 1);
  CHECK(pick_index_uniform(0.0, 5) == 0 && pick_index_uniform(0.999, 5) == 4 && pick_index_uniform(0.5, 10) == 5);
  CHECK_THROWS_AS(pick_index_uniform(0.5, 0), std::invalid_argument);
  CHECK(pick_index_linear(0.0, 4) == 0 && pick_index_linear(0.3, 3) == 1 && pick_index_linear(0.95, 3) == 2);
  CHECK(pick_index_exponential(1e-12, 5) == 0 && pick_index_exponential(0.5, 2) == 1);
  CHECK(pick_index_exponential(0.1, 3) == 1 && pick_index_exponential(0.0, 7) == 0);
  CHECK(pick_index_exponential(0.99, 100000) == 99999);
  CHECK(pick_index_exponential(1e-300, 100000) == 100000 - 691);
  CumulativeWeights cw;
  cw.prefix = {1.0, 2.0, 9.389};
  CHECK(pick_weighted(0.5, cw) == 2 && pick_weighted(0.1, cw) == 0);
  // closed forms == oracle on a sweep (test_samplers.cpp:63-75)
  int mism = 0;
  const CounterRng rng(55);
  for (std::uint64_t i = 0; i < 300; ++i) {
    const double u = rng.uniform(i, 7, 0);
    const std::size_t n = 1 + rng.bits(i, 0, 0) % 200;
    std::vector<double> lin(n);
    for (std::size_t k = 0; k < n; ++k) lin[k] = static_cast<double>(k + 1);
    if (pick_index_linear(u, n) != oracle_pick(u, lin)) ++mism;
  }
  CHECK(mism == 0);
}

static void walk_cases() {
  {  // test_walk_engine.cpp:41-57
    const auto s = EdgeStore::build(std::vector<TemporalEdge>{{1, 4, 1}, {2, 4, 2}, {3, 4, 3}},
                                    DirectionMode::DirectedForward);
    WalkConfig c;
    c.walks_per_node = 2;
    c.walk_length = 5;
    WalkStates st;
    WalkSet w;
    init_walks(s, c, st, w);
    CHECK(w.walk_count == 6 && w.stride == 5);
    for (std::uint64_t i = 0; i < 6; ++i) CHECK(w.lengths[i] == 1 && w.time_at(i, 0) == kTimeUnset);
  }
  {  // :104-136 tiering known answers
    const auto s = EdgeStore::build(std::vector<TemporalEdge>{{10, 1, 1}, {11, 1, 1}, {12, 1, 1}},
                                    DirectionMode::DirectedForward);
    const auto x = *s.find_node(10), y = *s.find_node(11), z = *s.find_node(12);
    WalkStates st;
    for (auto [node, count] : {std::pair{x, 3u}, {y, 100u}, {z, 20000u}}) {
      for (std::uint32_t i = 0; i < count; ++i) {
        st.current.push_back(node);
        st.time.push_back(kTimeUnset);
        st.prev.push_back(0);
        st.has_prev.push_back(0);
        st.alive.push_back(1);
        st.length.push_back(1);
      }
    }
    std::vector<std::uint32_t> ids(st.size());
    std::iota(ids.begin(), ids.end(), 0);
    const auto plan = schedule_step(st, ids, s, TierThresholds{});
    CHECK(plan.solo.size() == 1 && plan.solo[0].node == x && plan.solo[0].end - plan.solo[0].begin == 3);
    CHECK(plan.warp_cached.size() == 1 && plan.warp_cached[0].end - plan.warp_cached[0].begin == 100);
    CHECK(plan.block_cached.size() == 3);
    if (plan.block_cached.size() == 3) {
      CHECK(plan.block_cached[0].end - plan.block_cached[0].begin == 8192);
      CHECK(plan.block_cached[1].end - plan.block_cached[1].begin == 8192);
      CHECK(plan.block_cached[2].end - plan.block_cached[2].begin == 3616);
      CHECK(plan.block_cached[0].sub_task_count == 3);
    }
  }
  {  // :237-252 chain graph
    const auto s = EdgeStore::build(std::vector<TemporalEdge>{{1, 2, 1}, {2, 3, 2}}, DirectionMode::DirectedForward);
    WalkConfig c;
    c.walks_per_node = 1;
    c.walk_length = 3;
    c.bias = BiasKind::UniformIndex;
    const auto w = generate_walks(s, c);
    CHECK(w.walk_count == 2 && w.lengths[0] == 3);
    CHECK(w.node_at(0, 0) == 1 && w.time_at(0, 0) == kTimeUnset && w.node_at(0, 1) == 2 && w.time_at(0, 1) == 1);
    CHECK(w.node_at(0, 2) == 3 && w.time_at(0, 2) == 2);
  }
  {  // :294-316 scheduler neutrality + manual stepping (:393-420) == generate_walks
    const auto g = uniform_graph(40, 2000, 300, 21);
    const auto s = EdgeStore::build(g, DirectionMode::DirectedForward);
    for (BiasKind b : {BiasKind::UniformIndex, BiasKind::LinearIndex, BiasKind::ExponentialIndex,
                       BiasKind::ExponentialWeight}) {
      WalkConfig c;
      c.walks_per_node = 3;
      c.walk_length = 12;
      c.bias = b;
      c.seed = 99;
      const auto coop = generate_walks(s, c, {}, Variant::Coop);
      CHECK(coop == generate_walks(s, c, {}, Variant::CoopDirect));
      CHECK(coop == generate_walks(s, c, {}, Variant::FullWalk));
      WalkStates st;
      WalkSet manual;
      init_walks(s, c, st, manual);
      std::vector<std::uint32_t> cand(st.size());
      std::iota(cand.begin(), cand.end(), 0);
      for (;;) {
        const auto plan = schedule_step(st, cand, s, TierThresholds{});
        if (plan.empty()) break;
        TaskScratch scratch;
        for (const auto* list : {&plan.solo, &plan.warp_cached, &plan.warp_direct, &plan.block_cached,
                                 &plan.block_direct})
          for (const auto& task : *list) execute_task(task, plan, s, c, false, scratch, st, manual);
        cand = plan.walk_ids;
      }
      for (std::uint64_t w = 0; w < manual.walk_count; ++w) manual.lengths[w] = st.length[w];
      CHECK(manual == coop);
    }
  }
  {  // :450-474 sample_start_edge
    const auto s = EdgeStore::build(std::vector<TemporalEdge>{{1, 2, 5}, {3, 4, 5}, {5, 6, 9}},
                                    DirectionMode::DirectedForward);
    const auto idx = sample_start_edge(s, BiasKind::UniformIndex, 0.9, 0.0);
    CHECK(idx == 2 && s.edge_at(idx).time == 9);
    const auto e = EdgeStore::build(std::vector<TemporalEdge>{{1, 2, 5}, {3, 4, 9}, {5, 6, 12}},
                                    DirectionMode::DirectedForward);
    CHECK(e.edge_at(sample_start_edge(e, BiasKind::ExponentialIndex, 0.1, 0.0)).time == 9);
  }
  {  // :386-391, :591-597
    const auto s = EdgeStore::build(std::vector<TemporalEdge>{{1, 2, 1}, {2, 3, 2}}, DirectionMode::DirectedForward);
    WalkConfig c;
    c.direction = WalkDirection::Backward;
    CHECK_THROWS_AS(generate_walks(s, c), std::invalid_argument);
    WalkConfig big;
    big.start_mode = StartMode::Sampled;
    big.total_walks = std::uint64_t{1} << 40;
    CHECK_THROWS_AS(generate_walks(s, big), std::invalid_argument);
  }
}

static void replay_cases() {
  // test_replay.cpp:61-83 single batch == bulk
  auto stream = uniform_graph(40, 3000, 500, 7);
  std::stable_sort(stream.begin(), stream.end(), [](const auto& a, const auto& b) { return a.time < b.time; });
  WindowManager bulk({1000, DirectionMode::DirectedForward});
  bulk.ingest_batch(stream);
  WalkConfig wc;
  wc.walk_length = 10;
  wc.seed = 11;
  const auto bulk_walks = generate_walks(*bulk.snapshot(), wc);
  ReplayConfig rc;
  rc.batch_duration = 1000;
  rc.window_duration = 1000;
  rc.walk = wc;
  int batches = 0;
  bool equal = false;
  replay_stream(stream, rc, [&](const BatchRecord&, const WalkSet& w) {
    ++batches;
    equal = w == bulk_walks;
  });
  CHECK(batches == 1 && equal);
  // :26-41 batch splitting
  ReplayConfig split;
  split.batch_duration = 100;
  split.window_duration = 300;
  split.generate = false;
  auto s2 = uniform_graph(50, 5000, 999, 2);
  std::stable_sort(s2.begin(), s2.end(), [](const auto& a, const auto& b) { return a.time < b.time; });
  std::uint64_t ingested = 0;
  CHECK(replay_stream(s2, split, [&](const BatchRecord& r, const WalkSet&) { ingested += r.ingest.ingested; }) == 10);
  CHECK(ingested == s2.size());
  // B200 extension: the same stream through a one-rank ReplicaGroup equals
  // the single-GPU replay batch for batch (records, stats, walks)
  {
    ReplayConfig g = split;
    g.generate = true;
    g.walk = wc;
    std::vector<BatchRecord> r1, r2;
    std::vector<WalkSet> w1, w2;
    const auto n1 = replay_stream(s2, g, [&](const BatchRecord& r, const WalkSet& w) {
      r1.push_back(r);
      w1.push_back(w);
    });
    ReplicaGroup group(1, 0, ReplicaGroup::unique_id());
    const auto n2 = replay_stream(group, s2, g, [&](const BatchRecord& r, const WalkSet& w) {
      r2.push_back(r);
      w2.push_back(w);
    });
    CHECK(n1 == 10 && n2 == n1 && r2.size() == r1.size());
    bool same = true;
    for (std::size_t i = 0; i < r1.size() && i < r2.size(); ++i) {
      same = same && r1[i].batch_index == r2[i].batch_index && r1[i].ingest.ingested == r2[i].ingest.ingested &&
             r1[i].ingest.evicted == r2[i].ingest.evicted && r1[i].ingest.retained == r2[i].ingest.retained &&
             r1[i].walk.hops == r2[i].walk.hops && r1[i].walk.walks == r2[i].walk.walks && w1[i] == w2[i];
    }
    CHECK(same);
    WindowManager a({300, DirectionMode::DirectedForward});
    const auto& st = a.ingest_group(group, std::span<const TemporalEdge>(s2.data(), 100));
    CHECK(st.ingested == 100 && a.snapshot()->edge_count() == 100);
  }
}

static void primitive_cases() {
  // test_primitives.cpp: stable sort, RLE, partition, scan
  std::vector<std::uint64_t> keys{5, 1, 5, 3, 1, 0, 5};
  std::vector<std::uint32_t> vals{0, 1, 2, 3, 4, 5, 6};
  primitives::radix_sort_pairs(keys, vals);
  CHECK((keys == std::vector<std::uint64_t>{0, 1, 1, 3, 5, 5, 5}));
  CHECK((vals == std::vector<std::uint32_t>{5, 1, 4, 3, 0, 2, 6}));
  const auto runs = primitives::run_length_encode(keys);
  CHECK(runs.size() == 4 && runs[1].key == 1 && runs[1].start == 1 && runs[1].length == 2 && runs[3].length == 3);
  std::vector<std::uint32_t> out;
  const std::vector<std::uint8_t> flags{1, 0, 1, 0, 1};
  CHECK(primitives::partition_flagged(std::vector<std::uint32_t>{4, 3, 2, 1, 0}, flags, out) == 3);
  CHECK((out == std::vector<std::uint32_t>{4, 2, 0}));
  std::vector<std::uint64_t> in{3, 1, 4, 1, 5}, ex(5);
  CHECK(primitives::exclusive_scan(in, ex) == 14);
  CHECK((ex == std::vector<std::uint64_t>{0, 3, 4, 8, 9}));
}

// test_io.cpp:12-60 — edge files (TSV on the device)
void edge_io_cases() {
  {
    std::istringstream in("# temporal edges\n1\t2\t10\n\n3\t4\t20\n");
    const auto edges = read_edges_tsv(in);
    CHECK(edges.size() == 2);
    CHECK(edges.size() == 2 && edges[0] == (TemporalEdge{1, 2, 10}) && edges[1] == (TemporalEdge{3, 4, 20}));
    std::ostringstream out;
    write_edges_tsv(out, edges);
    CHECK(out.str() == "1\t2\t10\n3\t4\t20\n");
  }
  {
    std::istringstream missing("1\t2\t3\n4\t5\n");
    bool ok = false;
    try {
      read_edges_tsv(missing);
    } catch (const ParseError& e) {
      ok = std::string(e.what()) == "expected source<TAB>target<TAB>timestamp (line 2)" && e.line() == 2;
    }
    CHECK(ok);
    std::istringstream garbage("1\t2\tbogus\n");
    CHECK_THROWS_AS(read_edges_tsv(garbage), ParseError);
    std::istringstream negative("1\t2\t-5\n");
    CHECK_THROWS_AS(read_edges_tsv(negative), ParseError);
    std::size_t line = 0;
    try {
      std::istringstream bad("# ok\n1\t2\t3\nx\ty\tz\n");
      read_edges_tsv(bad);
    } catch (const ParseError& e) {
      line = e.line();
    }
    CHECK(line == 3);
  }
  {
    std::vector<TemporalEdge> edges;
    for (std::int64_t i = 0; i < 500; ++i) edges.push_back({(i * 7) % 50, (i * 13) % 50, i * 3});
    std::stringstream buffer;
    write_edges_binary(buffer, edges);
    CHECK(buffer.str().substr(0, 8) == "TMPW0001");
    CHECK(read_edges_binary(buffer) == edges);
    std::istringstream corrupt("XXXX0001payload");
    CHECK_THROWS_AS(read_edges_binary(corrupt), std::runtime_error);
  }
}

// test_io.cpp:62-108 — walk writers (device) and readers
void io_cases() {
  {
    WalkSet walks;
    walks.stride = 3;
    walks.walk_count = 2;
    walks.nodes = {1, 2, 3, 9, 0, 0};
    walks.times = {kTimeUnset, 5, 8, kTimeUnset, 0, 0};
    walks.lengths = {3, 1};  // the second walk never left its start
    std::ostringstream out;
    write_walks_text(out, walks);
    CHECK(out.str() == "1@- 2@5 3@8\n");
  }
  {
    std::istringstream in("1@- 2@5 3@8\n7 8 9\n");
    const auto records = read_walks_text(in);
    CHECK(records.size() == 2);
    CHECK(records[0].timed() && records[0].nodes == std::vector<NodeId>({1, 2, 3}));
    CHECK(records[0].times[0] == kTimeUnset && records[0].times[2] == 8);
    CHECK(!records[1].timed() && records[1].nodes == std::vector<NodeId>({7, 8, 9}));
    std::istringstream mixed("1@2 3 4@5\n");
    CHECK_THROWS_AS(read_walks_text(mixed), ParseError);
  }
  {
    WalkSet walks;
    walks.stride = 4;
    walks.walk_count = 3;
    walks.nodes.assign(12, 0);
    walks.times.assign(12, 0);
    walks.lengths = {4, 1, 2};
    for (std::size_t i = 0; i < 12; ++i) {
      walks.nodes[i] = static_cast<NodeId>(i * 7);
      walks.times[i] = static_cast<Timestamp>(i * 11);
    }
    // the reference zero-fills past each length; so does the device image
    for (std::uint64_t w = 0; w < 3; ++w)
      for (std::uint32_t j = walks.lengths[w]; j < 4; ++j) walks.nodes[w * 4 + j] = walks.times[w * 4 + j] = 0;
    std::stringstream buffer;
    write_walks_binary(buffer, walks);
    CHECK(buffer.str().substr(0, 8) == "TMPW0002");
    const auto parsed = read_walks_binary(buffer);
    CHECK(parsed == walks);
  }
  {  // generated walks: text image == the host formatting of the same walks
    const std::vector<TemporalEdge> edges{{1, 2, 1}, {2, 3, 2}, {3, 1, 3}, {1, 3, 4}, {2, 1, 5}};
    const auto store = EdgeStore::build(edges, DirectionMode::DirectedForward);
    WalkConfig config;
    config.walk_length = 6;
    config.walks_per_node = 3;
    const auto walks = generate_walks(store, config);
    std::ostringstream text;
    write_walks_text(text, walks);
    std::string expect;
    for (std::uint64_t w = 0; w < walks.walk_count; ++w) {
      if (walks.lengths[w] < 2) continue;
      for (std::uint32_t j = 0; j < walks.lengths[w]; ++j) {
        if (j) expect += ' ';
        const Timestamp t = walks.time_at(w, j);
        expect += std::to_string(walks.node_at(w, j)) + "@" +
                  (t == kTimeUnset || t == kTimeInfinite ? std::string("-") : std::to_string(t));
      }
      expect += '\n';
    }
    CHECK(!expect.empty() && text.str() == expect);
  }
}

// test_validity.cpp:34-190 — the auditor (check_walkset on the GPU)
void validity_cases() {
  const std::vector<TemporalEdge> edges{{1, 2, 1}, {2, 3, 2}};
  const EdgeOracle oracle(edges, false);
  {
    const std::vector<NodeId> n{1};
    const std::vector<Timestamp> t{0};
    const auto r = check_timed_walk(n, t, oracle);
    CHECK(r.valid && r.hops == 0);
  }
  {
    const std::vector<NodeId> n{1, 2, 3};
    const std::vector<Timestamp> t{0, 1, 2};
    const auto r = check_timed_walk(n, t, oracle);
    CHECK(r.valid && r.valid_hops == 2);
  }
  {
    const std::vector<TemporalEdge> tied{{1, 2, 1}, {2, 3, 1}};
    const EdgeOracle tied_oracle(tied, false);
    const std::vector<NodeId> n{1, 2, 3};
    const std::vector<Timestamp> t{0, 1, 1};
    const auto r = check_timed_walk(n, t, tied_oracle);
    CHECK(!r.valid && r.valid_hops == 1 && r.first_violation == std::optional<std::size_t>(1));
    CHECK(check_timed_walk(n, t, tied_oracle, WalkDirection::Forward, false).valid);
  }
  {
    const std::vector<NodeId> n{1, 3};
    const std::vector<Timestamp> t{0, 2};
    CHECK(!check_timed_walk(n, t, oracle).valid);
    const std::vector<NodeId> m{1, 2};
    const std::vector<Timestamp> u{kTimeUnset, 1};
    CHECK(check_timed_walk(m, u, oracle).valid);
  }
  {  // backward walks traverse stored edges in reverse
    const std::vector<TemporalEdge> chain{{1, 2, 5}, {3, 1, 2}};
    const EdgeOracle o(chain, false);
    const std::vector<NodeId> n{2, 1, 3};
    const std::vector<Timestamp> t{kTimeInfinite, 5, 2}, rising{kTimeInfinite, 2, 5};
    CHECK(check_timed_walk(n, t, o, WalkDirection::Backward).valid);
    CHECK(!check_timed_walk(n, rising, o, WalkDirection::Backward).valid);
  }
  {  // greedy untimed
    const std::vector<TemporalEdge> e1{{1, 2, 1}, {1, 2, 5}, {2, 3, 3}, {2, 3, 7}};
    const std::vector<NodeId> n{1, 2, 3};
    CHECK(check_untimed_walk_greedy(n, EdgeOracle(e1, false)).valid);
    const std::vector<TemporalEdge> e2{{1, 2, 5}, {2, 3, 3}};
    const auto r = check_untimed_walk_greedy(n, EdgeOracle(e2, false));
    CHECK(!r.valid && r.first_violation == std::optional<std::size_t>(1));
    const std::vector<NodeId> single{4};
    CHECK(check_untimed_walk_greedy(single, EdgeOracle({}, false)).valid);
  }
  {  // summarize
    std::vector<WalkCheckResult> res(10);
    for (auto& r : res) {
      r.hops = 80;
      r.valid_hops = 1;
      r.valid = false;
      r.first_violation = 0;
    }
    const auto rep = summarize(res);
    CHECK(rep.walk_percent() == 0.0 && std::abs(rep.hop_percent() - 1.25) < 1e-12);
    CHECK(rep.first_violation_per_walk.size() == 10 && summarize({}).walk_percent() == 100.0);
  }
  {  // undirected oracles accept either orientation
    const std::vector<TemporalEdge> e{{1, 2, 3}};
    CHECK(!EdgeOracle(e, false).contains(2, 1, 3));
    CHECK(EdgeOracle(e, true).contains(2, 1, 3) && EdgeOracle(e, true).contains(1, 2, 3));
    const EdgeOracle u(e, true);
    const auto* times = u.find(1, 2);
    CHECK(times && times->size() == 1 && (*times)[0] == 3);
  }
  {  // engine output audits clean end to end (the GPU check_walkset)
    std::vector<TemporalEdge> graph;
    for (std::int64_t i = 0; i < 4000; ++i) graph.push_back({(i * 37) % 60, (i * 101 + 7) % 60, (i * 13) % 500});
    const auto store = EdgeStore::build(graph, DirectionMode::DirectedForward);
    WalkConfig config;
    config.walk_length = 16;
    config.walks_per_node = 4;
    const auto walks = generate_walks(store, config);
    const EdgeOracle o(graph, false);
    const auto rep = check_walkset(walks, o);
    CHECK(rep.total_walks > 0 && rep.hop_percent() == 100.0 && rep.walk_percent() == 100.0);
    // the same walks against an oracle missing every edge of node 0: the GPU
    // audit agrees hop for hop with the single-walk rules
    std::vector<TemporalEdge> fewer;
    for (const auto& e : graph)
      if (e.source != 0) fewer.push_back(e);
    const EdgeOracle of(fewer, false);
    const auto bad = check_walkset(walks, of);
    std::vector<WalkCheckResult> host;
    for (std::uint64_t w = 0; w < walks.walk_count; ++w) {
      if (walks.lengths[w] < 2) continue;
      host.push_back(check_timed_walk(std::span<const NodeId>(walks.nodes.data() + w * walks.stride, walks.lengths[w]),
                                      std::span<const Timestamp>(walks.times.data() + w * walks.stride,
                                                                 walks.lengths[w]),
                                      of));
    }
    const auto ref = summarize(host);
    CHECK(bad.valid_hops < bad.total_hops);
    CHECK(bad.total_walks == ref.total_walks && bad.valid_walks == ref.valid_walks &&
          bad.total_hops == ref.total_hops && bad.valid_hops == ref.valid_hops &&
          bad.first_violation_per_walk == ref.first_violation_per_walk);
  }
}

// acceptance.cpp:276-294 / test_output.txt:38 — the tier-coverage input built
// by the device generator, default config, per-node starts: the reference's
// exact tier counts
void synthetic_cases() {
  const auto graph = make_hub_skewed_graph(2000, 20000, 0);
  CHECK(graph.size() == 13136 + 20000);
  const auto store = EdgeStore::build(graph, DirectionMode::DirectedForward);
  WalkStats st;
  const auto walks = generate_walks(store, WalkConfig{}, TierThresholds{}, Variant::Coop, &st);
  CHECK(st.tiers.solo == 19 && st.tiers.warp_cached == 6230 && st.tiers.warp_direct == 4 &&
        st.tiers.block_cached == 11 && st.tiers.block_direct == 1 && st.tiers.multi_block == 7);
  CHECK(make_mega_hub_graph(100, 3).size() == 100 + 64 + 1000);
  const auto ladder = make_time_ladder_graph(1000, 10, 4);
  CHECK(ladder.size() == 1000 && ladder[11].source == 1 && ladder[11].time == 1);
  const auto uni = make_uniform_graph(50, 300, 9, 2);
  CHECK(uni.size() == 300 && std::all_of(uni.begin(), uni.end(), [](const TemporalEdge& e) {
          return e.source >= 0 && e.source < 50 && e.target < 50 && e.time >= 0 && e.time <= 9;
        }));
}

// The reference's concurrency contract (window_manager.hpp:27-30): one ingest
// in flight while walk generations run over published snapshots. Thread A
// streams batches into the window while thread B repeatedly walks a snapshot
// it holds; B's walks must equal the single-threaded result, and A's final
// window must equal a sequential run's.
static void concurrency_cases() {
  const CounterRng rng(404);
  std::vector<std::vector<TemporalEdge>> batches;
  for (std::uint64_t b = 0; b < 10; ++b) {
    std::vector<TemporalEdge> e;
    for (std::uint64_t i = 0; i < 20000; ++i) {
      e.push_back({static_cast<NodeId>(rng.bits(b, i, 0) % 800), static_cast<NodeId>(rng.bits(b, i, 1) % 800),
                   static_cast<Timestamp>(b * 1000 + (i * 1000) / 20000)});
    }
    batches.push_back(std::move(e));
  }
  WindowManager seq({3000, DirectionMode::DirectedForward});
  for (const auto& b : batches) seq.ingest_batch(b);
  WalkConfig cfg;
  cfg.start_mode = StartMode::Sampled;
  cfg.total_walks = 20000;
  cfg.walk_length = 20;
  cfg.bias = BiasKind::ExponentialIndex;
  cfg.start_bias = BiasKind::UniformIndex;
  cfg.seed = 11;
  WindowManager w({3000, DirectionMode::DirectedForward});
  for (int b = 0; b < 3; ++b) w.ingest_batch(batches[b]);
  const auto held = w.snapshot();
  const WalkSet expect_full = generate_walks_fullwalk(*held, cfg);
  const WalkSet expect_coop = generate_walks(*held, cfg);
  bool walks_equal = true;
  std::thread walker([&] {
    for (int k = 0; k < 6; ++k) {
      const WalkSet a = generate_walks_fullwalk(*held, cfg);
      const WalkSet c = generate_walks(*held, cfg);
      walks_equal = walks_equal && a.nodes == expect_full.nodes && a.times == expect_full.times &&
                    c.nodes == expect_coop.nodes && c.times == expect_coop.times;
    }
  });
  std::thread ingester([&] {
    for (std::size_t b = 3; b < batches.size(); ++b) w.ingest_batch(batches[b]);
  });
  walker.join();
  ingester.join();
  CHECK(walks_equal);
  CHECK(expect_full.nodes == expect_coop.nodes && expect_full.times == expect_coop.times);
  const auto a = w.snapshot(), b = seq.snapshot();
  CHECK(a->edge_count() == b->edge_count() && a->node_count() == b->node_count());
  bool same = a->edge_count() == b->edge_count();
  for (std::size_t i = 0; same && i < a->edge_count(); i += 97) {
    const auto ea = a->edge_at(i), eb = b->edge_at(i);
    same = ea.source == eb.source && ea.target == eb.target && ea.time == eb.time;
  }
  CHECK(same);
  const WalkSet after_a = generate_walks_fullwalk(*a, cfg), after_b = generate_walks_fullwalk(*b, cfg);
  CHECK(after_a.nodes == after_b.nodes && after_a.times == after_b.times);
}

int main() {
  edge_store_cases();
  window_cases();
  sampler_cases();
  walk_cases();
  replay_cases();
  primitive_cases();
  edge_io_cases();
  io_cases();
  validity_cases();
  synthetic_cases();
  concurrency_cases();
  std::printf("%d/%d checks passed\n", g_checks - g_fail, g_checks);
  return g_fail;
}
