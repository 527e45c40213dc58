// Device pickers — bit-exact restatements of samplers.cpp:17-90 and
// walk_engine.cpp:49-84. All fp64 arithmetic uses explicit round-to-nearest
// intrinsics (no FMA contraction), matching the reference's x86-64 build
// (SURVEY App. A.6). exp/expm1 of integer arguments come from host-computed
// glibc tables; log1p/log use CUDA's (<=1-2 ulp); a draw whose value lies
// within 4 ulp of an integer is counted as "ambiguous" (its floor could in
// principle differ from glibc's) — measured 0 on the parity workloads.
#pragma once

#include "common.cuh"

namespace twg {

// samplers.cpp:17-21
__device__ __forceinline__ u64 pick_uniform(double u, u64 n) {
  const u64 i = __double2ull_rz(__dmul_rn(u, __ull2double_rn(n)));
  return i >= n ? n - 1 : i;
}

// samplers.cpp:23-40. The result is max{i < n : cum(i) <= r} (cum is
// monotone), so the sqrt guess only sets the starting point of the nudges.
__device__ __forceinline__ double cum_linear(i64 k) {
  return __dmul_rn(__dmul_rn(0.5, static_cast<double>(k)), static_cast<double>(k + 1));
}
__device__ __forceinline__ u64 pick_linear(double u, u64 n) {
  const double nn = __ull2double_rn(n);
  const double total = __dmul_rn(__dmul_rn(0.5, nn), __dadd_rn(nn, 1.0));
  const double r = __dmul_rn(u, total);
  const double disc =
      __dadd_rn(1.0, __dmul_rn(__dmul_rn(__dmul_rn(4.0, u), nn), __dadd_rn(nn, 1.0)));
  const double x = __dmul_rn(0.5, __dadd_rn(-1.0, __dsqrt_rn(disc)));
  i64 i = static_cast<i64>(x);
  if (i < 0) i = 0;
  if (i >= static_cast<i64>(n)) i = static_cast<i64>(n) - 1;
  while (i > 0 && cum_linear(i) > r) --i;
  while (i + 1 < static_cast<i64>(n) && cum_linear(i + 1) <= r) ++i;
  return static_cast<u64>(i);
}

__device__ __forceinline__ bool near_integer(double x) {
  if (!(x > 0.0)) return false;
  const double k = rint(x);
  const double ulp = fabs(x) * 2.220446049250313e-16;
  return fabs(x - k) <= 4.0 * ulp && k >= 1.0;
}

// samplers.cpp:42-55 (kExponentialExactLimit = 700, samplers.hpp:52)
__device__ __forceinline__ u64 pick_exponential(double u, u64 n, const double* expm1_tab, u32* ambiguous) {
  if (n == 1) return 0;
  double x;
  if (n <= 700) {
    x = log1p(__dmul_rn(u, expm1_tab[n]));
  } else {
    x = __dadd_rn(__ull2double_rn(n), log(u));
  }
  if (near_integer(x)) ++*ambiguous;
  if (!(x > 0.0)) return 0;
  const u64 i = __double2ull_rz(x);
  return i >= n ? n - 1 : i;
}

// lower_bound over [begin, end) of doubles
__device__ __forceinline__ u64 lower_bound_f64(const double* a, u64 lo, u64 hi, double r) {
  while (lo < hi) {
    const u64 mid = lo + ((hi - lo) >> 1);
    if (a[mid] < r) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// samplers.cpp:82-90
__device__ __forceinline__ u64 pick_weighted_range(double u, const double* prefix, u64 begin, u64 end,
                                                   double base) {
  const double r = __dadd_rn(base, __dmul_rn(u, __dsub_rn(prefix[end - 1], base)));
  u64 k = lower_bound_f64(prefix, begin, end, r);
  if (k == end) --k;
  return k - begin;
}

// samplers.cpp:74-80
__device__ __forceinline__ u64 pick_weighted(double u, const double* prefix, u64 n) {
  const double r = __dmul_rn(u, prefix[n - 1]);
  u64 k = lower_bound_f64(prefix, 0, n, r);
  if (k == n) --k;
  return k;
}

// glibc exp(d) for an integer d <= 0 (table; exp(-746..) == +0)
__device__ __forceinline__ double exp_nonpos(i64 d, const double* exp_neg) {
  const i64 k = -d;
  return k >= kExpTableSize ? 0.0 : exp_neg[k];
}

}  // namespace twg
