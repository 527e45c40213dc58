// Diagnostic: the acceptance suite's 100-batch stream (acceptance.cpp:303-321,
// criteria 07/08) through the drop-in, printing every batch's
// rebuild_duration and peak_bytes, so the per-batch cost curve behind
// criterion 08's least-squares slope can be read.
//   g++ -std=c++20 -O2 -Iinclude tools/diag_accum.cpp -o build/diag_accum \
//       -Lpaper_2605_16182_b200/lib -ltimewalk_b200 -Wl,-rpath,$PWD/paper_2605_16182_b200/lib
#include <chrono>
#include <cstdio>
#include <vector>

#include "timewalk/rng.hpp"
#include "timewalk/window_manager.hpp"

using namespace timewalk;

int main(int argc, char** argv) {
  const int reps = argc > 1 ? std::atoi(argv[1]) : 1;
  for (int rep = 0; rep < reps; ++rep) {
    const CounterRng rng(77);
    WindowManager window({3000, DirectionMode::DirectedForward});
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    int n = 0;
    for (std::uint64_t b = 0; b < 100; ++b) {
      std::vector<TemporalEdge> batch;
      batch.reserve(100000);
      for (std::uint64_t i = 0; i < 100000; ++i) {
        batch.push_back({static_cast<NodeId>(rng.bits(b, i, 0) % 20000),
                         static_cast<NodeId>(rng.bits(b, i, 1) % 20000),
                         static_cast<Timestamp>(b * 1000 + rng.bits(b, i, 2) % 1000)});
      }
      const auto t0 = std::chrono::steady_clock::now();
      const auto& stats = window.ingest_batch(batch);
      const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      std::printf("rep %d batch %3llu duration %.6f wall %.6f peak %llu\n", rep, (unsigned long long)b,
                  stats.rebuild_duration, wall, (unsigned long long)stats.peak_bytes);
      if (b >= 9) {
        const double x = static_cast<double>(b), y = stats.rebuild_duration;
        sx += x, sy += y, sxx += x * x, sxy += x * y, ++n;
      }
    }
    const double slope = (n * sxy - sx * sy) / (n * sxx - sx * sx);
    std::printf("rep %d slope %.3g mean %.3g ratio %.4f\n", rep, slope, sy / n, slope / (sy / n));
  }
  return 0;
}
