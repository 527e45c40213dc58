// B200 extensions of the timewalk API (not in the reference): device
// selection, RNG stream choice, optional-view build flags. Everything here
// has a default that reproduces the reference's behaviour exactly.
#pragma once

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

}  // namespace timewalk
