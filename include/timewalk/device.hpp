// B200 extensions of the timewalk API (not in the reference): device
// selection, RNG stream choice, optional-view build flags. Everything here
// has a default that reproduces the reference's behaviour exactly.
#pragma once

#include <array>
#include <cstdint>

namespace timewalk {

// Draw stream for walk generation. SplitMix is the reference's CounterRng
// (bit-exact with the unmodified reference); Philox4x32-10 keyed by
// (seed; walk, hop, ordinal) is bit-exact with the Philox-shadowed oracle.
enum class RngKind : std::uint8_t { SplitMix, Philox };

// GPU used by objects created afterwards on this thread (default 0).
void set_device(int device);
int current_device();

// Views built eagerly at EdgeStore::build / WindowManager ingest. The
// reference always builds both (edge_store.cpp:100-110, :216-250); turning
// one off defers it to first use (it is then built on the device lazily).
struct BuildOptions {
  bool weights{true};
  bool adjacency{true};
};

// Multi-GPU replica group (twg_group_* in twg.h): one process
// per GPU, created on this thread's current_device(). unique_id() is called
// by one rank and shared out of band; every rank constructs the group with
// it. Used by replay_stream(ReplicaGroup&, ...) and WindowManager::
// ingest_group / generate_walks_shard.
class ReplicaGroup {
 public:
  static std::array<std::uint8_t, 128> unique_id();
  ReplicaGroup(int nranks, int rank, const std::array<std::uint8_t, 128>& id);
  ~ReplicaGroup();
  ReplicaGroup(const ReplicaGroup&) = delete;
  ReplicaGroup& operator=(const ReplicaGroup&) = delete;
  [[nodiscard]] int size() const { return nranks_; }
  [[nodiscard]] int rank() const { return rank_; }
  [[nodiscard]] void* device_handle() const { return handle_; }  // twg_group*

 private:
  void* handle_{nullptr};
  int nranks_{1}, rank_{0};
};

}  // namespace timewalk
