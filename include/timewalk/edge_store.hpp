// Dual-index snapshot — drop-in for proj/core/include/timewalk/edge_store.hpp
// (edge_store.hpp:14-199). The index lives in GPU memory (SoA, built by the
// sm_100a kernels); the span-returning accessors read a host mirror that is
// downloaded lazily, once per field, on first use.
#pragma once

#include <memory>
#include <optional>
#include <span>
#include <utility>
#include <vector>

#include "timewalk/device.hpp"
#include "timewalk/types.hpp"

struct twg_store;

namespace timewalk {

struct NeighborRange {
  std::size_t start{};
  std::size_t end{};
  std::size_t group_count{};

  [[nodiscard]] bool empty() const { return start == end; }
  [[nodiscard]] std::size_t size() const { return end - start; }
};

struct BuildTelemetry {
  std::size_t scratch_bytes{};
};

struct TsGroupMark {
  Timestamp time{};
  std::uint32_t start{};
};

class EdgeStore {
 public:
  EdgeStore();

  static EdgeStore build(std::span<const TemporalEdge> edges, DirectionMode mode,
                         BuildTelemetry* telemetry = nullptr);
  static EdgeStore build(std::span<const TemporalEdge> edges, DirectionMode mode, BuildOptions options);

  [[nodiscard]] std::size_t edge_count() const;
  [[nodiscard]] std::size_t node_count() const;
  [[nodiscard]] std::size_t ts_group_count() const;
  [[nodiscard]] bool empty() const;
  [[nodiscard]] DirectionMode direction_mode() const;
  [[nodiscard]] bool supports(WalkDirection dir) const;

  [[nodiscard]] std::pair<std::size_t, std::size_t> edge_slice_for_ts_group(std::size_t group_index) const;
  [[nodiscard]] Timestamp ts_group_time(std::size_t group_index) const;
  [[nodiscard]] std::span<const double> ts_group_weight_prefix() const;

  [[nodiscard]] TemporalEdge edge_at(std::size_t pos) const;
  [[nodiscard]] InternalNode edge_source_internal(std::size_t pos) const;
  [[nodiscard]] InternalNode edge_target_internal(std::size_t pos) const;
  [[nodiscard]] Timestamp edge_time(std::size_t pos) const;
  [[nodiscard]] std::span<const Timestamp> edge_times() const;

  [[nodiscard]] std::optional<InternalNode> find_node(NodeId external) const;
  [[nodiscard]] NodeId external_id(InternalNode v) const;

  [[nodiscard]] NeighborRange temporal_neighborhood(NodeId v, Timestamp t, WalkDirection dir) const;
  [[nodiscard]] NeighborRange temporal_neighborhood_internal(InternalNode v, Timestamp t, WalkDirection dir) const;
  [[nodiscard]] std::size_t timestamp_group_count(NodeId v) const;
  [[nodiscard]] std::size_t timestamp_group_count_internal(InternalNode v) const;
  [[nodiscard]] std::pair<std::size_t, std::size_t> node_region(InternalNode v) const;
  [[nodiscard]] std::span<const TsGroupMark> group_marks(InternalNode v) const;
  [[nodiscard]] EdgeIndex ref_edge(std::size_t pos) const;
  [[nodiscard]] Timestamp ref_time(std::size_t pos) const;
  [[nodiscard]] InternalNode ref_neighbor(std::size_t pos, InternalNode owner) const;
  [[nodiscard]] std::span<const double> weight_prefix() const;

  [[nodiscard]] bool adjacent(InternalNode a, InternalNode b) const;
  [[nodiscard]] bool adjacent_after(InternalNode a, InternalNode b, Timestamp t, WalkDirection dir) const;

  [[nodiscard]] std::vector<TemporalEdge> export_suffix(Timestamp cutoff) const;
  [[nodiscard]] std::vector<TemporalEdge> export_edges() const { return export_suffix(kTimeUnset); }

  [[nodiscard]] std::size_t memory_bytes() const;

  // B200 extension: the C-ABI handle (for twg_* calls on this snapshot)
  [[nodiscard]] twg_store* device_handle() const;

  struct Impl;
  explicit EdgeStore(std::shared_ptr<Impl> impl);

 private:
  std::shared_ptr<Impl> impl_;
};

}  // namespace timewalk
