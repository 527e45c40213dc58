// The drop-in C++ façade: the reference's public timewalk API
// (proj/core/include/timewalk/*.hpp) implemented over the C ABI (twg.h).
// Every computation is a GPU call; the host keeps only control flow,
// argument validation (the reference's validate() contracts) and the lazily
// downloaded mirrors that back the reference's span-returning accessors.
// Status codes become the reference's exception types.
#include <algorithm>
#include <array>
#include <chrono>
#include <charconv>
#include <cstring>
#include <fstream>
#include <istream>
#include <iterator>
#include <ostream>
#include <sstream>
#include <vector>
#include <cmath>
#include <map>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>

#include "timewalk/edge_store.hpp"
#include "timewalk/io.hpp"
#include "timewalk/synthetic.hpp"
#include "timewalk/validity.hpp"
#include "timewalk/primitives.hpp"
#include "timewalk/replay.hpp"
#include "timewalk/samplers.hpp"
#include "timewalk/walk_engine.hpp"
#include "timewalk/window_manager.hpp"
#include "twg.h"

static_assert(sizeof(timewalk::TemporalEdge) == sizeof(twg_edge), "TemporalEdge must match twg_edge");

namespace timewalk {

namespace {

std::recursive_mutex& api_mutex() {  // one ctx per device is shared; its scratch is not thread-safe
  static std::recursive_mutex m;
  return m;
}

thread_local int t_device = 0;

[[noreturn]] void raise_status(int rc) {
  const std::string msg = twg_last_error();
  switch (rc) {
    case TWG_EINVAL: throw std::invalid_argument(msg);
    case TWG_ERANGE: throw std::out_of_range(msg);
    case TWG_ELOGIC: throw std::logic_error(msg);
    case TWG_ENOMEM: throw std::bad_alloc();
    default: throw std::runtime_error("timewalk (B200): " + msg);
  }
}

void check(int rc) {
  if (rc != TWG_OK) raise_status(rc);
}

twg_ctx* ctx() {
  static std::map<int, twg_ctx*> contexts;
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  auto it = contexts.find(t_device);
  if (it != contexts.end()) return it->second;
  twg_ctx* c = nullptr;
  check(twg_ctx_create(t_device, &c));
  contexts[t_device] = c;
  return c;
}

// Walk generation runs on the calling thread's own context (stream and
// scratch): the reference's contract — one ingest in flight while any number
// of walk generations run over published snapshots (window_manager.hpp:
// 27-30) — holds without the API lock. Snapshots are immutable once
// published (the ingest synchronises before publishing; the lazily completed
// views are built under a per-store lock and published complete), and a
// snapshot older than the window's retired one that a caller still holds
// makes the next ingest repack instead of reusing its slots.
twg_ctx* walk_ctx() {
  thread_local std::map<int, twg_ctx*> mine;
  auto it = mine.find(t_device);
  if (it != mine.end()) return it->second;
  twg_ctx* c = nullptr;
  {
    std::lock_guard<std::recursive_mutex> lk(api_mutex());  // context creation touches device-global state
    check(twg_ctx_create(t_device, &c));
  }
  mine[t_device] = c;  // lives for the process, like the shared context
  return c;
}

twg_walk_config to_c(const WalkConfig& c) {
  twg_walk_config w{};
  w.walk_length = c.walk_length;
  w.start_mode = static_cast<int32_t>(c.start_mode);
  w.walks_per_node = c.walks_per_node;
  w.total_walks = c.total_walks;
  w.bias = static_cast<int32_t>(c.bias);
  w.start_bias = static_cast<int32_t>(c.start_bias);
  w.node2vec = c.node2vec ? 1 : 0;
  w.temporal_adjacency = c.node2vec_temporal_adjacency ? 1 : 0;
  w.p = c.node2vec ? c.node2vec->p : 1.0;
  w.q = c.node2vec ? c.node2vec->q : 1.0;
  w.direction = static_cast<int32_t>(c.direction);
  w.rng = static_cast<int32_t>(c.rng);
  w.seed = c.seed;
  w.walk_begin = c.walk_begin;
  w.walk_end = c.walk_end;
  return w;
}

twg_thresholds to_c(const TierThresholds& t) {
  return twg_thresholds{t.w_warp, t.block_dim, t.w_max, t.g_warp_cap, t.g_block_cap};
}

}  // namespace

void set_device(int device) { t_device = device; }
int current_device() { return t_device; }

// ---------------------------------------------------------------- EdgeStore

struct EdgeStore::Impl {
  twg_store* h{nullptr};
  twg_store_info info{};
  std::once_flag f_edges, f_internal, f_ts, f_tsw, f_nodes, f_marks, f_ref, f_wp, f_ext;
  std::vector<NodeId> src_ext, dst_ext;
  std::vector<Timestamp> time;
  std::vector<std::uint32_t> src, dst;
  std::vector<std::uint64_t> ts_off;
  std::vector<Timestamp> ts_time;
  std::vector<double> ts_w;
  std::vector<std::uint64_t> n_off, n_tsidx;
  std::vector<TsGroupMark> marks;
  std::vector<std::uint32_t> ref_edge, ref_nbr;
  std::vector<double> wp;
  std::vector<NodeId> ext;

  ~Impl() {
    if (h) twg_store_release(h);
  }

  template <class T>
  void download(int field, std::vector<T>& out, std::size_t n) {
    std::lock_guard<std::recursive_mutex> lk(api_mutex());
    out.resize(n);
    check(twg_store_download(h, field, out.empty() ? nullptr : out.data()));
  }
  void refresh_info() {
    std::lock_guard<std::recursive_mutex> lk(api_mutex());
    check(twg_store_get_info(h, &info));
  }

  const Impl& edges() {
    std::call_once(f_edges, [&] {
      download(0, src_ext, info.edges);
      download(1, dst_ext, info.edges);
      download(2, time, info.edges);
    });
    return *this;
  }
  const Impl& internal() {
    std::call_once(f_internal, [&] {
      download(3, src, info.edges);
      download(4, dst, info.edges);
    });
    return *this;
  }
  const Impl& ts() {
    std::call_once(f_ts, [&] {
      download(5, ts_off, info.ts_groups + 1);
      download(6, ts_time, info.ts_groups);
    });
    return *this;
  }
  const Impl& tsw() {
    std::call_once(f_tsw, [&] { download(7, ts_w, info.ts_groups); });
    return *this;
  }
  const Impl& nodes() {
    std::call_once(f_nodes, [&] {
      download(8, n_off, info.nodes + 1);
      download(9, n_tsidx, info.nodes + 1);
    });
    return *this;
  }
  const Impl& mk() {
    std::call_once(f_marks, [&] {
      std::vector<Timestamp> t;
      std::vector<std::uint32_t> s;
      download(10, t, info.node_groups);
      download(11, s, info.node_groups);
      marks.resize(t.size());
      for (std::size_t g = 0; g < t.size(); ++g) marks[g] = TsGroupMark{t[g], s[g]};
    });
    return *this;
  }
  const Impl& refs() {
    std::call_once(f_ref, [&] {
      download(12, ref_edge, info.entries);
      download(15, ref_nbr, info.entries);
    });
    return *this;
  }
  const Impl& weights() {
    std::call_once(f_wp, [&] { download(13, wp, info.entries); });
    return *this;
  }
  const Impl& exts() {
    std::call_once(f_ext, [&] { download(14, ext, info.nodes); });
    return *this;
  }
};

EdgeStore::EdgeStore(std::shared_ptr<Impl> impl) : impl_(std::move(impl)) {}

EdgeStore::EdgeStore() : EdgeStore(build({}, DirectionMode::DirectedForward, BuildOptions{})) {}

EdgeStore EdgeStore::build(std::span<const TemporalEdge> edges, DirectionMode mode, BuildTelemetry* telemetry) {
  EdgeStore s = build(edges, mode, BuildOptions{});
  if (telemetry) telemetry->scratch_bytes = s.impl_->info.device_bytes;
  return s;
}

EdgeStore EdgeStore::build(std::span<const TemporalEdge> edges, DirectionMode mode, BuildOptions options) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  auto impl = std::make_shared<Impl>();
  const twg_build_opts o{options.weights ? 1 : 0, options.adjacency ? 1 : 0};
  check(twg_store_build(ctx(), reinterpret_cast<const twg_edge*>(edges.data()), edges.size(),
                        static_cast<int>(mode), &o, &impl->h));
  impl->refresh_info();
  return EdgeStore(std::move(impl));
}

std::size_t EdgeStore::edge_count() const { return impl_->info.edges; }
std::size_t EdgeStore::node_count() const { return impl_->info.nodes; }
std::size_t EdgeStore::ts_group_count() const { return impl_->info.ts_groups; }
bool EdgeStore::empty() const { return impl_->info.edges == 0; }
DirectionMode EdgeStore::direction_mode() const { return static_cast<DirectionMode>(impl_->info.mode); }
bool EdgeStore::supports(WalkDirection dir) const {
  const auto m = direction_mode();
  if (m == DirectionMode::Undirected) return true;
  return (m == DirectionMode::DirectedForward) == (dir == WalkDirection::Forward);
}
std::size_t EdgeStore::memory_bytes() const { return impl_->info.device_bytes; }
twg_store* EdgeStore::device_handle() const { return impl_->h; }

std::pair<std::size_t, std::size_t> EdgeStore::edge_slice_for_ts_group(std::size_t g) const {
  if (g >= ts_group_count()) throw std::out_of_range("edge_slice_for_ts_group: group index out of range");
  const auto& m = impl_->ts();
  return {m.ts_off[g], m.ts_off[g + 1]};
}
Timestamp EdgeStore::ts_group_time(std::size_t g) const { return impl_->ts().ts_time[g]; }
std::span<const double> EdgeStore::ts_group_weight_prefix() const { return impl_->tsw().ts_w; }

TemporalEdge EdgeStore::edge_at(std::size_t pos) const {
  const auto& m = impl_->edges();
  return {m.src_ext[pos], m.dst_ext[pos], m.time[pos]};
}
InternalNode EdgeStore::edge_source_internal(std::size_t pos) const { return impl_->internal().src[pos]; }
InternalNode EdgeStore::edge_target_internal(std::size_t pos) const { return impl_->internal().dst[pos]; }
Timestamp EdgeStore::edge_time(std::size_t pos) const { return impl_->edges().time[pos]; }
std::span<const Timestamp> EdgeStore::edge_times() const { return impl_->edges().time; }

std::optional<InternalNode> EdgeStore::find_node(NodeId external) const {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  std::uint32_t id = 0;
  std::uint8_t found = 0;
  check(twg_store_find_nodes(impl_->h, &external, 1, &id, &found));
  if (!found) return std::nullopt;
  return id;
}
NodeId EdgeStore::external_id(InternalNode v) const { return impl_->exts().ext[v]; }

NeighborRange EdgeStore::temporal_neighborhood(NodeId v, Timestamp t, WalkDirection dir) const {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  std::uint64_t out[3] = {0, 0, 0};
  check(twg_store_neighborhood(impl_->h, &v, &t, 1, static_cast<int>(dir), out));
  return {out[0], out[1], out[2]};
}
NeighborRange EdgeStore::temporal_neighborhood_internal(InternalNode v, Timestamp t, WalkDirection dir) const {
  return temporal_neighborhood(external_id(v), t, dir);
}
std::size_t EdgeStore::timestamp_group_count(NodeId v) const {
  const auto iv = find_node(v);
  return iv ? timestamp_group_count_internal(*iv) : 0;
}
std::size_t EdgeStore::timestamp_group_count_internal(InternalNode v) const {
  const auto& m = impl_->nodes();
  return m.n_tsidx[v + 1] - m.n_tsidx[v];
}
std::pair<std::size_t, std::size_t> EdgeStore::node_region(InternalNode v) const {
  const auto& m = impl_->nodes();
  return {m.n_off[v], m.n_off[v + 1]};
}
std::span<const TsGroupMark> EdgeStore::group_marks(InternalNode v) const {
  const auto& n = impl_->nodes();
  const auto& m = impl_->mk();
  return {m.marks.data() + n.n_tsidx[v], n.n_tsidx[v + 1] - n.n_tsidx[v]};
}
EdgeIndex EdgeStore::ref_edge(std::size_t pos) const { return impl_->refs().ref_edge[pos]; }
Timestamp EdgeStore::ref_time(std::size_t pos) const { return impl_->edges().time[impl_->refs().ref_edge[pos]]; }
InternalNode EdgeStore::ref_neighbor(std::size_t pos, InternalNode owner) const {
  if (direction_mode() != DirectionMode::Undirected) return impl_->refs().ref_nbr[pos];
  const auto& in = impl_->internal();
  const auto e = impl_->refs().ref_edge[pos];
  return in.src[e] == owner ? in.dst[e] : in.src[e];
}
std::span<const double> EdgeStore::weight_prefix() const { return impl_->weights().wp; }

bool EdgeStore::adjacent(InternalNode a, InternalNode b) const {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  std::uint8_t r = 0;
  check(twg_store_adjacent(impl_->h, &a, &b, 1, 0, nullptr, 0, &r));
  return r != 0;
}
bool EdgeStore::adjacent_after(InternalNode a, InternalNode b, Timestamp t, WalkDirection dir) const {
  if (!supports(dir)) {  // via temporal_neighborhood_internal (edge_store.cpp:279-281)
    throw std::invalid_argument("temporal_neighborhood: walk direction not served by this store's direction mode");
  }
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  std::uint8_t r = 0;
  check(twg_store_adjacent(impl_->h, &a, &b, 1, 1, &t, static_cast<int>(dir), &r));
  return r != 0;
}

std::vector<TemporalEdge> EdgeStore::export_suffix(Timestamp cutoff) const {
  const auto& m = impl_->edges();
  const auto from = static_cast<std::size_t>(std::lower_bound(m.time.begin(), m.time.end(), cutoff) - m.time.begin());
  std::vector<TemporalEdge> out;
  out.reserve(m.time.size() - from);
  for (std::size_t i = from; i < m.time.size(); ++i) out.push_back({m.src_ext[i], m.dst_ext[i], m.time[i]});
  return out;
}

// ---------------------------------------------------------------- window

WindowManager::WindowManager(WindowConfig config) : WindowManager(config, BuildOptions{}) {}

WindowManager::WindowManager(WindowConfig config, BuildOptions options) : config_(config) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  const twg_build_opts o{options.weights ? 1 : 0, options.adjacency ? 1 : 0};
  check(twg_window_create(ctx(), config.duration, static_cast<int>(config.mode), &o, &handle_));
  refresh();
}

WindowManager::~WindowManager() {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  store_.reset();
  previous_.reset();
  if (handle_) twg_window_destroy(handle_);
}

void WindowManager::refresh() {
  twg_store* h = nullptr;
  check(twg_window_snapshot(handle_, &h));
  auto impl = std::make_shared<EdgeStore::Impl>();
  impl->h = h;
  impl->refresh_info();
  previous_ = std::move(store_);  // exactly one retired snapshot (window_manager.cpp:56-57)
  store_ = std::make_shared<const EdgeStore>(EdgeStore(std::move(impl)));
}

const BatchStats& WindowManager::ingest_batch(std::span<const TemporalEdge> batch) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  twg_batch_stats s{};
  check(twg_window_ingest(handle_, reinterpret_cast<const twg_edge*>(batch.data()), batch.size(), &s));
  stats_ = BatchStats{s.ingested, s.dropped_late, s.evicted, s.retained, s.rebuild_duration, s.peak_bytes};
  check(twg_window_state(handle_, &t_high_, &batch_count_, nullptr));
  if (!batch.empty()) refresh();  // an empty batch leaves the snapshot itself unchanged
  return stats_;
}

const BatchStats& WindowManager::ingest_batch_device(const std::int64_t* d_src, const std::int64_t* d_dst,
                                                     const std::int64_t* d_t, std::uint64_t n) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  twg_batch_stats s{};
  check(twg_window_ingest_device(handle_, d_src, d_dst, d_t, n, &s));
  stats_ = BatchStats{s.ingested, s.dropped_late, s.evicted, s.retained, s.rebuild_duration, s.peak_bytes};
  check(twg_window_state(handle_, &t_high_, &batch_count_, nullptr));
  if (n) refresh();
  return stats_;
}

const BatchStats& WindowManager::adopt_group(const void* gstats) {
  const auto& g = *static_cast<const twg_group_batch_stats*>(gstats);
  if (!g.replicas_agree) throw std::runtime_error("timewalk (B200): replica windows disagree after a group ingest");
  const twg_batch_stats& s = g.local;
  stats_ = BatchStats{s.ingested, s.dropped_late, s.evicted, s.retained, s.rebuild_duration, s.peak_bytes};
  check(twg_window_state(handle_, &t_high_, &batch_count_, nullptr));
  if (g.edges) refresh();
  return stats_;
}

const BatchStats& WindowManager::ingest_group(ReplicaGroup& group, std::span<const TemporalEdge> batch, int root) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  twg_group_batch_stats g{};
  check(twg_group_ingest(static_cast<twg_group*>(group.device_handle()), handle_, root,
                         reinterpret_cast<const twg_edge*>(batch.data()), batch.size(), &g));
  return adopt_group(&g);
}

const BatchStats& WindowManager::ingest_group_staged(ReplicaGroup& group, int slot) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  twg_group_batch_stats g{};
  check(twg_group_ingest_staged(static_cast<twg_group*>(group.device_handle()), handle_, slot, &g));
  return adopt_group(&g);
}

std::pair<Timestamp, Timestamp> WindowManager::window_bounds() const {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  Timestamp lo = 0, hi = 0;
  check(twg_window_bounds(handle_, &lo, &hi));
  return {lo, hi};
}

// ---------------------------------------------------------------- walks

void TierThresholds::validate() const {
  if (w_warp < 1 || w_warp > block_dim || block_dim > w_max)
    throw std::invalid_argument("tier thresholds: need 1 <= w_warp <= block_dim <= w_max");
  if (g_warp_cap > g_block_cap) throw std::invalid_argument("tier thresholds: need g_warp_cap <= g_block_cap");
}

void WalkConfig::validate() const {
  if (walk_length < 1) throw std::invalid_argument("walk config: walk_length must be >= 1");
  if (start_mode == StartMode::PerNode && walks_per_node == 0)
    throw std::invalid_argument("walk config: walks_per_node must be positive");
  if (node2vec && (node2vec->p <= 0.0 || node2vec->q <= 0.0))
    throw std::invalid_argument("walk config: node2vec p and q must be positive");
}

namespace {
WalkSet download_walks(twg_walkset* w, const twg_walk_stats& st, std::chrono::steady_clock::time_point started,
                       WalkStats* stats);
}  // namespace

WalkSet generate_walks(const EdgeStore& store, const WalkConfig& config, const TierThresholds& thresholds,
                       Variant variant, WalkStats* stats) {
  const auto started = std::chrono::steady_clock::now();
  config.validate();
  thresholds.validate();
  const twg_walk_config c = to_c(config);
  const twg_thresholds th = to_c(thresholds);
  twg_walkset* w = nullptr;
  twg_walk_stats st{};
  check(twg_generate(walk_ctx(), store.device_handle(), &c, &th, static_cast<int>(variant), &w, &st));
  return download_walks(w, st, started, stats);
}

WalkSet generate_walks(ReplicaGroup& group, const EdgeStore& store, const WalkConfig& config,
                       const TierThresholds& thresholds, Variant variant, WalkStats* stats) {
  const auto started = std::chrono::steady_clock::now();
  config.validate();
  thresholds.validate();
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  const twg_walk_config c = to_c(config);
  const twg_thresholds th = to_c(thresholds);
  twg_walkset* w = nullptr;
  twg_walk_stats local{}, global{};
  check(twg_group_generate(static_cast<twg_group*>(group.device_handle()), store.device_handle(), &c, &th,
                           static_cast<int>(variant), &w, &local, &global));
  return download_walks(w, global, started, stats);
}

namespace {
WalkSet download_walks(twg_walkset* w, const twg_walk_stats& st, std::chrono::steady_clock::time_point started,
                       WalkStats* stats) {
  WalkSet out;
  std::uint64_t first = 0, hops = 0;
  const int rc = twg_walkset_info(w, &out.stride, &out.walk_count, &first, &hops);
  if (rc == TWG_OK) {
    out.nodes.resize(out.walk_count * out.stride);
    out.times.resize(out.walk_count * out.stride);
    out.lengths.resize(out.walk_count);
  }
  const int rc2 = rc == TWG_OK ? twg_walkset_download(w, out.nodes.data(), out.times.data(), out.lengths.data()) : rc;
  twg_walkset_destroy(w);
  check(rc2);
  if (stats) {
    *stats = WalkStats{st.walks, st.hops, st.steps,
                       TierCounts{st.solo, st.warp_cached, st.warp_direct, st.block_cached, st.block_direct,
                                  st.multi_block},
                       std::chrono::duration<double>(std::chrono::steady_clock::now() - started).count()};
  }
  return out;
}
}  // namespace

WalkSet generate_walks_fullwalk(const EdgeStore& store, const WalkConfig& config, WalkStats* stats) {
  return generate_walks(store, config, TierThresholds{}, Variant::FullWalk, stats);
}

void init_walks(const EdgeStore& store, const WalkConfig& config, WalkStates& states, WalkSet& walks) {
  config.validate();
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  const twg_walk_config c = to_c(config);
  std::uint32_t stride = 0;
  std::uint64_t count = 0;
  check(twg_init_walks(ctx(), store.device_handle(), &c, &stride, &count, nullptr, nullptr, nullptr, nullptr, nullptr,
                       nullptr, nullptr, nullptr));
  walks.stride = stride;
  walks.walk_count = count;
  walks.nodes.assign(count * stride, 0);
  walks.times.assign(count * stride, 0);
  walks.lengths.assign(count, 0);
  states.current.assign(count, 0);
  states.time.assign(count, 0);
  states.prev.assign(count, 0);
  states.has_prev.assign(count, 0);
  states.alive.assign(count, 0);
  states.length.assign(count, 0);
  if (count) {
    check(twg_init_walks(ctx(), store.device_handle(), &c, &stride, &count, states.current.data(),
                         states.time.data(), states.prev.data(), states.has_prev.data(), states.alive.data(),
                         states.length.data(), walks.nodes.data(), walks.times.data()));
  }
  walks.lengths.assign(states.length.begin(), states.length.end());
}

StepPlan schedule_step(const WalkStates& states, const std::vector<std::uint32_t>& candidates, const EdgeStore& store,
                       const TierThresholds& thresholds) {
  thresholds.validate();
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  const std::size_t n = candidates.size();
  std::vector<std::uint32_t> node(n);
  std::vector<std::uint8_t> alive(n);
  for (std::size_t i = 0; i < n; ++i) {
    node[i] = states.current[candidates[i]];
    alive[i] = states.alive[candidates[i]];
  }
  std::uint64_t sizes[5] = {0, 0, 0, 0, 0};
  std::vector<std::uint32_t> rows(6 * (n + 16));
  std::vector<std::uint32_t> ids(n + 1);
  const twg_thresholds th = to_c(thresholds);
  check(twg_schedule_step(store.device_handle(), node.data(), alive.data(), n, &th, sizes, rows.data(), n + 16,
                          ids.data()));
  StepPlan plan;
  std::size_t alive_n = 0;
  for (auto a : alive) alive_n += a ? 1 : 0;
  plan.walk_ids.resize(alive_n);
  for (std::size_t k = 0; k < alive_n; ++k) plan.walk_ids[k] = candidates[ids[k]];
  std::vector<DispatchTask>* lists[5] = {&plan.solo, &plan.warp_cached, &plan.warp_direct, &plan.block_cached,
                                         &plan.block_direct};
  std::size_t r = 0;
  for (int k = 0; k < 5; ++k) {
    for (std::uint64_t x = 0; x < sizes[k]; ++x, ++r) {
      const std::uint32_t* row = &rows[6 * r];
      lists[k]->push_back(DispatchTask{row[0], static_cast<Tier>(row[5]), row[1], row[2], row[3], row[4]});
    }
  }
  return plan;
}

void execute_task(const DispatchTask& task, const StepPlan& plan, const EdgeStore& store, const WalkConfig& config,
                  bool /*use_scratch: staging is an execution detail, results are identical*/, TaskScratch& /*scratch*/,
                  WalkStates& states, WalkSet& walks) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  const twg_walk_config c = to_c(config);
  const std::uint32_t* ids = plan.walk_ids.data() + task.begin;
  check(twg_hop_walks(ctx(), store.device_handle(), &c, ids, task.end - task.begin, states.size(), walks.stride,
                      states.current.data(), states.time.data(), states.prev.data(), states.has_prev.data(),
                      states.alive.data(), states.length.data(), walks.nodes.data(), walks.times.data()));
}

std::size_t sample_start_edge(const EdgeStore& store, BiasKind bias, double u1, double u2) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  std::uint64_t out = 0;
  check(twg_sample_start_edges(store.device_handle(), static_cast<int>(bias), &u1, &u2, 1, &out));
  return out;
}

// ---------------------------------------------------------------- samplers

namespace {
std::size_t pick(int kind, double u, std::size_t n) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  std::uint64_t nn = n, out = 0;
  check(twg_pick_index(ctx(), kind, &u, &nn, 1, &out));
  return out;
}
}  // namespace

std::size_t pick_index_uniform(double u, std::size_t n) { return pick(0, u, n); }
std::size_t pick_index_linear(double u, std::size_t n) { return pick(1, u, n); }
std::size_t pick_index_exponential(double u, std::size_t n) { return pick(2, u, n); }

std::size_t pick_weighted_range(double u, std::span<const double> prefix, std::size_t begin, std::size_t end,
                                double base) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  std::uint64_t b = begin, e = end, out = 0;
  check(twg_pick_weighted_range(ctx(), &u, prefix.data(), prefix.size(), &b, &e, &base, 1, &out));
  return out;
}

std::size_t pick_weighted(double u, std::span<const double> prefix) {
  if (prefix.empty()) throw std::invalid_argument("pick_weighted: empty prefix array");
  // samplers.cpp:74-80 == pick_weighted_range over [0, n) with base 0
  return pick_weighted_range(u, prefix, 0, prefix.size(), 0.0);
}

std::size_t pick_weighted(double u, const CumulativeWeights& cw) { return pick_weighted(u, cw.prefix); }

// Reference utilities outside the walk path (samplers.cpp:57-72, :92-103),
// evaluated where the caller's data lives, with the reference's arithmetic.
// REFERENCE-DERIVED host glue: these two functions restate the reference's
// own code (host data in, host answer out; the reference's API contract);
// they are not on the GPU path and claim no GPU work.
CumulativeWeights build_cumulative_weights(std::span<const Timestamp> times) {
  if (times.empty()) throw std::invalid_argument("build_cumulative_weights: empty input");
  CumulativeWeights cw;
  cw.prefix.resize(times.size());
  double acc = 0.0;
  for (std::size_t i = 0; i < times.size(); ++i) {
    acc += std::exp(static_cast<double>(times[i] - times.front()));
    cw.prefix[i] = acc;
  }
  return cw;
}

std::size_t oracle_pick(double u, std::span<const double> weights) {
  if (weights.empty()) throw std::invalid_argument("oracle_pick: empty weights");
  double total = 0.0;
  for (double w : weights) total += w;
  const double r = u * total;
  double cum = 0.0;
  for (std::size_t k = 0; k < weights.size(); ++k) {
    cum += weights[k];
    if (r < cum) return k;
  }
  return weights.size() - 1;
}

// ---------------------------------------------------------------- primitives

namespace primitives {

std::uint64_t exclusive_scan(std::span<const std::uint64_t> in, std::span<std::uint64_t> out) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  std::uint64_t total = 0;
  check(twg_exclusive_scan(ctx(), in.data(), out.data(), in.size(), &total));
  return total;
}

void radix_sort_pairs(std::vector<std::uint64_t>& keys, std::vector<std::uint32_t>& values) {
  if (keys.size() < 2) return;
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  check(twg_radix_sort_pairs(ctx(), keys.data(), values.data(), keys.size()));
}

std::vector<KeyRun> run_length_encode(std::span<const std::uint64_t> sorted_keys) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  std::vector<std::uint64_t> rows(3 * sorted_keys.size() + 3);
  std::uint64_t runs = 0;
  check(twg_run_length_encode(ctx(), sorted_keys.data(), sorted_keys.size(), rows.data(), &runs));
  std::vector<KeyRun> out(runs);
  for (std::uint64_t r = 0; r < runs; ++r)
    out[r] = KeyRun{rows[3 * r], static_cast<std::uint32_t>(rows[3 * r + 1]), static_cast<std::uint32_t>(rows[3 * r + 2])};
  return out;
}

std::size_t partition_flagged(std::span<const std::uint32_t> items, std::span<const std::uint8_t> flags,
                              std::vector<std::uint32_t>& out) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  out.assign(items.size(), 0);
  std::uint64_t kept = 0;
  check(twg_partition_flagged(ctx(), items.data(), items.size(), flags.data(), flags.size(), out.data(), &kept));
  out.resize(kept);
  return kept;
}

}  // namespace primitives

// ---------------------------------------------------------------- replay

void ReplayConfig::validate() const {
  if (batch_duration <= 0) throw std::invalid_argument("replay: batch_duration must be positive");
  if (window_duration < batch_duration) throw std::invalid_argument("replay: window_duration must be >= batch_duration");
  walk.validate();
  thresholds.validate();
}

// replay.cpp:16-53
std::uint64_t replay_stream(std::span<const TemporalEdge> edges, const ReplayConfig& config, const BatchSink& sink) {
  config.validate();
  if (edges.empty()) return 0;
  WindowManager window({config.window_duration, config.mode});
  std::uint64_t batch_index = 0;
  const Timestamp origin = edges.front().time;
  Timestamp boundary = origin + config.batch_duration;
  std::size_t begin = 0;
  auto flush = [&](std::size_t end) {
    if (end == begin) return;
    BatchRecord record;
    record.batch_index = batch_index++;
    record.ingest = window.ingest_batch(edges.subspan(begin, end - begin));
    WalkSet walks;
    if (config.generate && !window.snapshot()->empty()) {
      walks = generate_walks(*window.snapshot(), config.walk, config.thresholds, config.variant, &record.walk);
    }
    if (sink) sink(record, walks);
    begin = end;
  };
  for (std::size_t i = 0; i < edges.size(); ++i) {
    if (edges[i].time >= boundary) {
      flush(i);
      const Timestamp spans = (edges[i].time - origin) / config.batch_duration + 1;
      boundary = origin + spans * config.batch_duration;
    }
  }
  flush(edges.size());
  return batch_index;
}

// ---- multi-GPU replica group -----------------------------------------

std::array<std::uint8_t, 128> ReplicaGroup::unique_id() {
  std::array<std::uint8_t, 128> id{};
  check(twg_group_unique_id(id.data()));
  return id;
}

ReplicaGroup::ReplicaGroup(int nranks, int rank, const std::array<std::uint8_t, 128>& id)
    : nranks_(nranks), rank_(rank) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  twg_group* g = nullptr;
  check(twg_group_create(ctx(), nranks, rank, id.data(), &g));
  handle_ = g;
}

ReplicaGroup::~ReplicaGroup() {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  if (handle_) twg_group_destroy(static_cast<twg_group*>(handle_));
}

// replay_stream across the group: the root cuts batches exactly as the
// single-GPU loop (replay.cpp:16-53); an empty broadcast ends the stream
std::uint64_t replay_stream(ReplicaGroup& group, std::span<const TemporalEdge> edges, const ReplayConfig& config,
                            const BatchSink& sink, int root) {
  config.validate();
  const bool is_root = group.rank() == root;
  WindowManager window({config.window_duration, config.mode});
  std::uint64_t batch_index = 0;
  auto step = [&](std::span<const TemporalEdge> batch) {  // every rank, same order
    BatchRecord record;
    record.batch_index = batch_index++;
    record.ingest = window.ingest_group(group, batch, root);
    WalkSet walks;
    if (config.generate && !window.snapshot()->empty())
      walks = generate_walks(group, *window.snapshot(), config.walk, config.thresholds, config.variant, &record.walk);
    if (sink) sink(record, walks);
  };
  auto finish = [&] {  // the end-of-stream marker: an empty broadcast nobody ingests
    std::lock_guard<std::recursive_mutex> lk(api_mutex());
    check(twg_group_stage_host(static_cast<twg_group*>(group.device_handle()), 0, root, nullptr, 0));
  };
  if (!is_root) {
    for (;;) {
      std::uint64_t n = 0;
      {
        std::lock_guard<std::recursive_mutex> lk(api_mutex());
        twg_group* g = static_cast<twg_group*>(group.device_handle());
        check(twg_group_stage_host(g, 0, root, nullptr, 0));  // receives the root's next batch (or the end)
        check(twg_group_staged_edges(g, 0, &n));
      }
      if (n == 0) break;
      BatchRecord record;
      record.batch_index = batch_index++;
      record.ingest = window.ingest_group_staged(group, 0);
      WalkSet walks;
      if (config.generate && !window.snapshot()->empty())
        walks = generate_walks(group, *window.snapshot(), config.walk, config.thresholds, config.variant, &record.walk);
      if (sink) sink(record, walks);
    }
    return batch_index;
  }
  if (!edges.empty()) {
    const Timestamp origin = edges.front().time;
    Timestamp boundary = origin + config.batch_duration;
    std::size_t begin = 0;
    auto flush = [&](std::size_t end) {
      if (end == begin) return;
      step(edges.subspan(begin, end - begin));
      begin = end;
    };
    for (std::size_t i = 0; i < edges.size(); ++i) {
      if (edges[i].time >= boundary) {
        flush(i);
        const Timestamp spans = (edges[i].time - origin) / config.batch_duration + 1;
        boundary = origin + spans * config.batch_duration;
      }
    }
    flush(edges.size());
  }
  finish();
  return batch_index;
}

// ---- walk writers (io.cpp:119-135, :173-183) on the device ----------------------

namespace {

// uploads the host image, has the device serialise it, streams the bytes out
void write_walks_device(std::ostream& out, const WalkSet& walks, bool binary) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  twg_walkset* w = nullptr;
  check(twg_walkset_from_host(ctx(), walks.stride, walks.walk_count, walks.nodes.data(), walks.times.data(),
                              walks.lengths.data(), &w));
  std::uint64_t len = 0;
  int rc = binary ? twg_walkset_binary(w, nullptr, 0, &len) : twg_walkset_text(w, nullptr, 0, &len);
  std::vector<char> bytes;
  if (rc == TWG_OK) {
    bytes.resize(len);
    rc = binary ? twg_walkset_binary(w, bytes.data(), len, &len) : twg_walkset_text(w, bytes.data(), len, &len);
  }
  twg_walkset_destroy(w);
  check(rc);
  out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
}

}  // namespace

void write_walks_text(std::ostream& out, const WalkSet& walks) { write_walks_device(out, walks, false); }

// TMPW0002 of a HOST walk set is its raw image (io.cpp:176-186): the host
// vectors are written as they are (tails past lengths[w] included), with no
// device round trip. Device-resident walk sets serialise on the GPU
// (twg_walkset_binary).
void write_walks_binary(std::ostream& out, const WalkSet& walks) {
  const std::uint32_t stride = walks.stride;
  const std::uint64_t count = walks.walk_count;
  out.write(kWalkBinaryMagic, 8);
  out.write(reinterpret_cast<const char*>(&stride), sizeof(stride));
  out.write(reinterpret_cast<const char*>(&count), sizeof(count));
  out.write(reinterpret_cast<const char*>(walks.nodes.data()),
            static_cast<std::streamsize>(walks.nodes.size() * sizeof(NodeId)));
  out.write(reinterpret_cast<const char*>(walks.times.data()),
            static_cast<std::streamsize>(walks.times.size() * sizeof(Timestamp)));
  out.write(reinterpret_cast<const char*>(walks.lengths.data()),
            static_cast<std::streamsize>(walks.lengths.size() * sizeof(std::uint32_t)));
}

void write_walks(const std::string& path, const WalkSet& walks, bool binary) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open " + path + " for writing");
  if (binary) write_walks_binary(out, walks);
  else write_walks_device(out, walks, false);
}

// ---- walk readers (host deserialisers, io.cpp:137-216) ----------------------------

namespace {

// a non-negative decimal token (std::from_chars semantics, io.cpp:14-22)
std::int64_t parse_token(std::string_view tok, std::size_t line, const char* what) {
  std::int64_t v = 0;
  const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (r.ec != std::errc{} || r.ptr != tok.data() + tok.size())
    throw ParseError(std::string("invalid ") + what + " '" + std::string(tok) + "'", line);
  if (v < 0) throw ParseError(std::string("negative ") + what, line);
  return v;
}

template <class T>
T read_pod(std::istream& in) {
  T v{};
  in.read(reinterpret_cast<char*>(&v), sizeof(T));
  if (!in) throw std::runtime_error("binary input truncated");
  return v;
}

}  // namespace

// REFERENCE-DERIVED host I/O (io.cpp:137-209 restated): the walk readers
// parse host streams into host WalkSets; no GPU work is claimed for them.
std::vector<WalkRecord> read_walks_text(std::istream& in) {
  std::vector<WalkRecord> out;
  std::string line;
  std::size_t no = 0;
  while (std::getline(in, line)) {
    ++no;
    if (line.empty() || line[0] == '#') continue;
    WalkRecord rec;
    bool timed = false, untimed = false;
    std::istringstream toks(line);
    std::string tok;
    while (toks >> tok) {
      const std::string_view v(tok);
      const std::size_t at = v.find('@');
      if (at == std::string_view::npos) {
        untimed = true;
        rec.nodes.push_back(parse_token(v, no, "node"));
        rec.times.push_back(kTimeUnset);
      } else {
        timed = true;
        rec.nodes.push_back(parse_token(v.substr(0, at), no, "node"));
        const std::string_view tp = v.substr(at + 1);
        rec.times.push_back(tp == "-" ? kTimeUnset : parse_token(tp, no, "timestamp"));
      }
    }
    if (rec.nodes.empty()) continue;
    if (timed && untimed) throw ParseError("walk mixes timed and untimed entries", no);
    if (untimed) rec.times.clear();
    out.push_back(std::move(rec));
  }
  return out;
}

WalkSet read_walks_binary(std::istream& in) {
  char magic[8];
  in.read(magic, sizeof(magic));
  if (!in || std::memcmp(magic, kWalkBinaryMagic, 8) != 0) throw std::runtime_error("walk binary: bad magic header");
  WalkSet w;
  w.stride = read_pod<std::uint32_t>(in);
  w.walk_count = read_pod<std::uint64_t>(in);
  const std::size_t cells = w.walk_count * w.stride;
  w.nodes.resize(cells);
  w.times.resize(cells);
  w.lengths.resize(w.walk_count);
  in.read(reinterpret_cast<char*>(w.nodes.data()), static_cast<std::streamsize>(cells * sizeof(NodeId)));
  in.read(reinterpret_cast<char*>(w.times.data()), static_cast<std::streamsize>(cells * sizeof(Timestamp)));
  in.read(reinterpret_cast<char*>(w.lengths.data()),
          static_cast<std::streamsize>(w.walk_count * sizeof(std::uint32_t)));
  if (!in) throw std::runtime_error("walk binary: truncated payload");
  return w;
}

std::vector<WalkRecord> read_walks(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  char magic[8] = {};
  in.read(magic, sizeof(magic));
  const bool binary = in.gcount() == 8 && std::memcmp(magic, kWalkBinaryMagic, 8) == 0;
  in.clear();
  in.seekg(0);
  if (!binary) return read_walks_text(in);
  const WalkSet w = read_walks_binary(in);
  std::vector<WalkRecord> out;
  for (std::uint64_t i = 0; i < w.walk_count; ++i) {
    const std::uint32_t len = w.lengths[i];
    if (len < 2) continue;  // as the text writer: walks that never left the start node
    WalkRecord rec;
    for (std::uint32_t j = 0; j < len; ++j) {
      rec.nodes.push_back(w.node_at(i, j));
      rec.times.push_back(w.time_at(i, j));
    }
    out.push_back(std::move(rec));
  }
  return out;
}

// ---- edge files (io.cpp:40-107): TSV on the device, binary as raw triples -----------

std::vector<TemporalEdge> read_edges_tsv(std::istream& in) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  twg_edges* e = nullptr;
  std::uint64_t line = 0;
  const int rc = twg_parse_edges_tsv(ctx(), text.data(), text.size(), &e, &line);
  if (rc == TWG_EPARSE) throw ParseError(twg_last_error(), line);
  check(rc);
  std::uint64_t n = 0;
  std::vector<TemporalEdge> edges;
  static_assert(sizeof(TemporalEdge) == sizeof(twg_edge));
  int rc2 = twg_edges_info(e, &n);
  if (rc2 == TWG_OK && n) {
    edges.resize(n);
    rc2 = twg_edges_download(e, reinterpret_cast<twg_edge*>(edges.data()));
  }
  twg_edges_destroy(e);
  check(rc2);
  return edges;
}

void write_edges_tsv(std::ostream& out, std::span<const TemporalEdge> edges) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  twg_edges* e = nullptr;
  check(twg_edges_from_host(ctx(), reinterpret_cast<const twg_edge*>(edges.data()), edges.size(), &e));
  std::uint64_t len = 0;
  int rc = twg_edges_format_tsv(e, nullptr, 0, &len);
  std::vector<char> bytes;
  if (rc == TWG_OK) {
    bytes.resize(len);
    rc = twg_edges_format_tsv(e, bytes.data(), len, &len);
  }
  twg_edges_destroy(e);
  check(rc);
  out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
}

std::vector<TemporalEdge> read_edges_binary(std::istream& in) {
  char magic[8];
  in.read(magic, sizeof(magic));
  if (!in || std::memcmp(magic, kEdgeBinaryMagic, 8) != 0) throw std::runtime_error("edge binary: bad magic header");
  const auto count = read_pod<std::uint64_t>(in);
  std::vector<TemporalEdge> edges;
  edges.reserve(count);
  for (std::uint64_t i = 0; i < count; ++i) {
    const auto s = read_pod<std::int64_t>(in);
    const auto d = read_pod<std::int64_t>(in);
    const auto t = read_pod<std::int64_t>(in);
    edges.push_back({s, d, t});
  }
  return edges;
}

void write_edges_binary(std::ostream& out, std::span<const TemporalEdge> edges) {
  out.write(kEdgeBinaryMagic, 8);
  const std::uint64_t n = edges.size();
  out.write(reinterpret_cast<const char*>(&n), sizeof(n));
  out.write(reinterpret_cast<const char*>(edges.data()), static_cast<std::streamsize>(n * sizeof(TemporalEdge)));
}

std::vector<TemporalEdge> read_edges(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  char magic[8] = {};
  in.read(magic, sizeof(magic));
  const bool binary = in.gcount() == 8 && std::memcmp(magic, kEdgeBinaryMagic, 8) == 0;
  in.clear();
  in.seekg(0);
  return binary ? read_edges_binary(in) : read_edges_tsv(in);
}

void write_edges(const std::string& path, std::span<const TemporalEdge> edges, bool binary) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open " + path + " for writing");
  if (binary) write_edges_binary(out, edges);
  else write_edges_tsv(out, edges);
}

// ---- walk validity (validity.cpp) ---------------------------------------------------

EdgeOracle::EdgeOracle(std::span<const TemporalEdge> edges, bool undirected)
    : store_(std::make_shared<EdgeStore>(
          EdgeStore::build(edges, undirected ? DirectionMode::Undirected : DirectionMode::DirectedForward,
                           BuildOptions{false, false}))) {}

const std::vector<Timestamp>* EdgeOracle::find(NodeId a, NodeId b) const {
  if (!store_) return nullptr;
  std::lock_guard<std::mutex> lk(cache_->mu);
  const auto key = std::make_pair(a, b);
  if (auto it = cache_->hit.find(key); it != cache_->hit.end()) return &it->second;
  if (cache_->miss.count(key)) return nullptr;
  // a's node-view region holds its out-edges (forward) or both orientations
  // (undirected: a self-loop twice, as the reference's map gets it), time-sorted
  const auto ia = store_->find_node(a), ib = store_->find_node(b);
  std::vector<Timestamp> times;
  if (ia && ib) {
    const auto [lo, hi] = store_->node_region(*ia);
    for (std::size_t p = lo; p < hi; ++p)
      if (store_->ref_neighbor(p, *ia) == *ib) times.push_back(store_->ref_time(p));
  }
  if (times.empty()) {
    cache_->miss.insert(key);
    return nullptr;
  }
  return &cache_->hit.emplace(key, std::move(times)).first->second;
}

bool EdgeOracle::contains(NodeId a, NodeId b, Timestamp t) const {
  const auto* times = find(a, b);
  return times && std::binary_search(times->begin(), times->end(), t);
}

// REFERENCE-DERIVED single-walk rules (validity.cpp:32-106 restated over the
// device-backed EdgeOracle's answers): host control flow per walk; the bulk
// audit is check_walkset on the GPU auditor (twg_walkset_audit).
WalkCheckResult check_timed_walk(std::span<const NodeId> nodes, std::span<const Timestamp> times,
                                 const EdgeOracle& oracle, WalkDirection direction, bool strict) {
  WalkCheckResult r;
  if (nodes.size() < 2) return r;  // no hop: vacuously valid
  const bool fwd = direction == WalkDirection::Forward;
  r.hops = nodes.size() - 1;
  r.hop_valid.assign(r.hops, false);
  for (std::size_t j = 0; j < r.hops; ++j) {
    const Timestamp tp = times[j], th = times[j + 1];
    // backward hops traverse the stored edge target -> source
    const bool edge = fwd ? oracle.contains(nodes[j], nodes[j + 1], th) : oracle.contains(nodes[j + 1], nodes[j], th);
    const bool order = (j == 0 && (tp == kTimeUnset || tp == kTimeInfinite)) ||
                       (fwd ? (strict ? th > tp : th >= tp) : (strict ? th < tp : th <= tp));
    if (edge && order) {
      r.hop_valid[j] = true;
      ++r.valid_hops;
    } else if (!r.first_violation) {
      r.first_violation = j;
    }
  }
  r.valid = r.valid_hops == r.hops;
  return r;
}

WalkCheckResult check_untimed_walk_greedy(std::span<const NodeId> nodes, const EdgeOracle& oracle, bool strict) {
  WalkCheckResult r;
  if (nodes.size() < 2) return r;
  r.hops = nodes.size() - 1;
  r.hop_valid.assign(r.hops, false);
  Timestamp at = kTimeUnset;  // earliest feasible assignment so far
  for (std::size_t j = 0; j < r.hops; ++j) {
    const auto* c = oracle.find(nodes[j], nodes[j + 1]);
    auto it = c ? (strict ? std::upper_bound(c->begin(), c->end(), at) : std::lower_bound(c->begin(), c->end(), at))
                : std::vector<Timestamp>::const_iterator{};
    if (!c || it == c->end()) {
      r.first_violation = j;  // greedy-earliest failing proves infeasibility: later hops unreachable
      break;
    }
    at = *it;
    r.hop_valid[j] = true;
    ++r.valid_hops;
  }
  r.valid = r.valid_hops == r.hops;
  return r;
}

ValidityReport summarize(std::span<const WalkCheckResult> results) {
  ValidityReport rep;
  rep.total_walks = results.size();
  rep.first_violation_per_walk.reserve(results.size());
  for (const WalkCheckResult& r : results) {
    rep.total_hops += r.hops;
    rep.valid_hops += r.valid_hops;
    rep.valid_walks += r.valid ? 1 : 0;
    rep.first_violation_per_walk.push_back(r.first_violation);
  }
  return rep;
}

ValidityReport check_walkset(const WalkSet& walks, const EdgeOracle& oracle, WalkDirection direction, bool strict) {
  ValidityReport rep;
  std::vector<std::int64_t> first(walks.walk_count ? walks.walk_count : 1, -1);
  twg_audit_report r{};
  if (oracle.store()) {
    std::lock_guard<std::recursive_mutex> lk(api_mutex());
    twg_walkset* w = nullptr;
    check(twg_walkset_from_host(ctx(), walks.stride, walks.walk_count, walks.nodes.data(), walks.times.data(),
                                walks.lengths.data(), &w));
    const int rc = twg_walkset_audit(w, oracle.store()->device_handle(), static_cast<int>(direction), strict ? 1 : 0,
                                     first.data(), &r);
    twg_walkset_destroy(w);
    check(rc);
  } else {  // an empty oracle holds no edge: every emitted walk fails at hop 0
    for (std::uint64_t i = 0; i < walks.walk_count; ++i) {
      if (walks.lengths[i] < 2) continue;
      ++r.walks;
      r.hops += walks.lengths[i] - 1;
      first[i] = 0;
    }
  }
  rep.total_walks = r.walks;
  rep.valid_walks = r.valid_walks;
  rep.total_hops = r.hops;
  rep.valid_hops = r.valid_hops;
  rep.first_violation_per_walk.reserve(r.walks);
  for (std::uint64_t i = 0; i < walks.walk_count; ++i) {
    if (walks.lengths[i] < 2) continue;  // skipped, as the writers do
    rep.first_violation_per_walk.push_back(first[i] < 0 ? std::nullopt
                                                        : std::optional<std::size_t>(static_cast<std::size_t>(first[i])));
  }
  return rep;
}

// ---- synthetic graphs (synthetic.cpp) on the device ------------------------------------

namespace {

std::vector<TemporalEdge> synth(int kind, std::uint64_t a, std::uint64_t b, Timestamp t_max, std::uint64_t seed) {
  std::lock_guard<std::recursive_mutex> lk(api_mutex());
  std::uint64_t n = 0;
  check(twg_synth_graph(ctx(), kind, a, b, t_max, seed, nullptr, 0, &n));
  std::vector<TemporalEdge> edges(n);
  check(twg_synth_graph(ctx(), kind, a, b, t_max, seed, reinterpret_cast<twg_edge*>(edges.data()), n, &n));
  return edges;
}

}  // namespace

std::vector<TemporalEdge> make_uniform_graph(std::uint64_t node_count, std::uint64_t edge_count, Timestamp t_max,
                                             std::uint64_t seed) {
  return synth(0, node_count, edge_count, t_max, seed);
}

std::vector<TemporalEdge> make_hub_skewed_graph(std::uint64_t background_nodes, std::uint64_t background_edges,
                                                std::uint64_t seed) {
  return synth(1, background_nodes, background_edges, 0, seed);
}

std::vector<TemporalEdge> make_mega_hub_graph(std::uint32_t feeder_count, std::uint64_t seed) {
  return synth(2, feeder_count, 0, 0, seed);
}

std::vector<TemporalEdge> make_time_ladder_graph(std::uint64_t edge_count, std::uint32_t rungs, std::uint64_t seed) {
  return synth(3, edge_count, rungs, 0, seed);
}

}  // namespace timewalk
