// Device-wide data-parallel primitives for the index build and the walk
// scheduler (the sm_100a replacements of the reference's CPU primitives,
// primitives.cpp:24-148 — radix_sort_pairs, exclusive_scan,
// run_length_encode, partition_flagged — and of the CUB calls the paper's
// GPU engine uses):
//
//  * exclusive_scan: three-phase tile scan (tile sums -> recursive scan of
//    the sums -> rescan + write), input supplied by a functor so flag
//    computations fuse into the scan's loads;
//  * radix_sort_pairs: stable LSD radix sort of (u32|u64 key, u32 value),
//    8-bit digits, pass count from the key's actual bit width (the
//    reference's constant-digit skip, primitives.cpp:47-56, made static).
//    Per pass: tile histogram -> scan of the digit-major count matrix ->
//    stable tile ranking with warp match/ballot + shared-memory staging so
//    the global scatter is written in digit-contiguous, coalesced runs.
#pragma once

#include "common.cuh"

namespace twg {

constexpr int kScanBlock = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanBlock * kScanItems;

constexpr int kSortBlock = 256;
#ifndef TWG_SORT_ITEMS_WIDE
#define TWG_SORT_ITEMS_WIDE 8  // items per thread of a onesweep tile for pairs wider than 8 B
#endif
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;

// Lanes of the warp holding the same kBits-bit digit (the valid ones; an
// invalid lane only matches other invalid lanes): kBits + 1 ballots instead of
// match.any, which issues at a fraction of the ballot rate.
template <int kBits>
__device__ __forceinline__ u32 digit_peers(u32 d, bool valid) {
  const u32 vb = __ballot_sync(0xffffffffu, valid);
  u32 m = valid ? vb : ~vb;
#pragma unroll
  for (int b = 0; b < kBits; ++b) {
    const bool bit = (d >> b) & 1u;
    const u32 bal = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bal : ~bal;
  }
  return m;
}

// One atomicAdd per block of the block's sum (every thread of the block must
// call it): per-warp atomics on one word serialise at L2 when a large grid
// finishes at once.
__device__ __forceinline__ void block_atomic_add(unsigned long long* dst, u64 v) {
  __shared__ u64 s_part[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) s_part[warp] = v;
  __syncthreads();
  if (warp == 0) {
    u64 x = lane < nw ? s_part[lane] : 0ull;
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0 && x) atomicAdd(dst, static_cast<unsigned long long>(x));
  }
  __syncthreads();  // s_part may be reused by a second call
}

// ---- 1-D TMA bulk copies (cp.async.bulk) into shared memory --------------
//
// One thread arms an mbarrier with the byte count and issues the copies; the
// copy engine writes shared memory directly (no registers, no per-thread
// loads) and completes the transaction on the barrier; every thread waits on
// the barrier's phase. Addresses and sizes must be 16-B aligned.
__device__ __forceinline__ u32 smem_u32(const void* p) { return static_cast<u32>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// First k in [0, n) with key(k) >= x over a sorted key, by one warp: each
// round the 32 lanes probe 32 evenly spaced positions and keep the piece
// holding the boundary (log33 n dependent rounds instead of log2 n). Every
// lane of the warp calls it; every lane gets the answer.
template <class Key>
__device__ __forceinline__ u64 warp_lower_bound(Key key, u64 n, i64 x) {
  const u32 lane = threadIdx.x & 31;
  u64 lo = 0, hi = n;  // answer in [lo, hi]
  while (hi > lo) {
    const u64 span = hi - lo;
    const bool small = span <= 32;
    const u64 p = small ? lo + lane : lo + (static_cast<u64>(lane) + 1) * span / 33;
    const bool in = small ? lane < span : true;
    const u32 c = __popc(__ballot_sync(0xffffffffu, in && key(p) < x));
    if (small) return lo + c;
    const u64 plo = lo, pspan = span;
    auto probe = [&](u32 i) { return plo + (static_cast<u64>(i) + 1) * pspan / 33; };
    const u64 nlo = c > 0 ? probe(c - 1) + 1 : lo;
    const u64 nhi = c < 32 ? probe(c) : hi;
    lo = nlo;
    hi = nhi;
  }
  return lo;
}

// Block-wide reduction of one u64 (op: 0 add, 1 max, 2 min, 3 or); the
// result is valid in thread 0. Every thread of the block must call it.
template <int kOp>
__device__ __forceinline__ u64 block_reduce_u64(u64 v) {
  __shared__ u64 s_red[32];
  auto f = [](u64 a, u64 b) { return kOp == 0 ? a + b : kOp == 1 ? (a > b ? a : b) : kOp == 2 ? (a < b ? a : b) : (a | b); };
  for (int o = 16; o > 0; o >>= 1) v = f(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < nw ? s_red[lane] : s_red[0];
    for (int o = 16; o > 0; o >>= 1) v = f(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  __syncthreads();
  return v;
}

// ---------------------------------------------------------------- scan ----

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix, *total = block sum. blockDim.x == kScanBlock.
template <class T>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
  __shared__ T warp_sums[kScanBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T incl = warp_incl_scan(v);
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    T s = lane < kScanBlock / 32 ? warp_sums[lane] : T(0);
    s = warp_incl_scan(s);
    if (lane < kScanBlock / 32) warp_sums[lane] = s;
  }
  __syncthreads();
  const T warp_prefix = warp == 0 ? T(0) : warp_sums[warp - 1];
  *total = warp_sums[kScanBlock / 32 - 1];
  __syncthreads();
  return warp_prefix + incl - v;
}

template <class T, class In>
__global__ void __launch_bounds__(kScanBlock) k_scan_tile_sums(In in, u64 n, T* tile_sums) {
  const u64 base = static_cast<u64>(blockIdx.x) * kScanTile;
  T s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const u64 i = base + static_cast<u64>(threadIdx.x) * kScanItems + j;
    if (i < n) s += in(i);
  }
  T total;
  block_excl_scan<T>(s, &total);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

template <class T, class In>
__global__ void __launch_bounds__(kScanBlock) k_scan_tiles(In in, u64 n, const T* tile_offsets, T* out) {
  const u64 base = static_cast<u64>(blockIdx.x) * kScanTile;
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const u64 i = base + static_cast<u64>(threadIdx.x) * kScanItems + j;
    v[j] = i < n ? in(i) : T(0);
    s += v[j];
  }
  T total;
  T run = block_excl_scan<T>(s, &total) + (tile_offsets ? tile_offsets[blockIdx.x] : T(0));
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const u64 i = base + static_cast<u64>(threadIdx.x) * kScanItems + j;
    if (i < n) out[i] = run;
    run += v[j];
  }
  // out[n] = grand total, written by the block owning element n-1 (or n == 0)
  if (threadIdx.x == kScanBlock - 1 && base < n && n - base <= kScanTile) out[n] = run;
}

template <class T>
struct LoadFn {
  const T* p;
  __device__ __forceinline__ T operator()(u64 i) const { return p[i]; }
};

// out[0..n] : out[i] = sum_{j<i} in(j), out[n] = total. T = u32 or u64.
template <class T, class In>
void exclusive_scan(Ctx& ctx, In in, u64 n, T* out) {
  cudaStream_t st = ctx.stream;
  if (n == 0) {
    TWG_CUDA(cudaMemsetAsync(out, 0, sizeof(T), st));
    return;
  }
  const u64 tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles == 1) {
    k_scan_tiles<T, In><<<1, kScanBlock, 0, st>>>(in, n, nullptr, out);
    TWG_LAUNCHED(ctx);
    return;
  }
  DevBuf<T> sums(tiles + 1, st);
  k_scan_tile_sums<T, In><<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(in, n, sums.p);
  TWG_LAUNCHED(ctx);
  DevBuf<T> offs(tiles + 1, st);
  exclusive_scan<T>(ctx, LoadFn<T>{sums.p}, tiles, offs.p);
  k_scan_tiles<T, In><<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(in, n, offs.p, out);
  TWG_LAUNCHED(ctx);
}

// --------------------------------------------------------------- radix ----

// Input of a radix pass: arrays, or (first pass) a functor computing the
// (key, value) of item i from some other layout (In::key(i), In::val(i)).
template <class K, class V>
struct ArrayIn {
  const K* k;
  const V* v;
  __device__ __forceinline__ K key(u64 i) const { return k[i]; }
  __device__ __forceinline__ V val(u64 i) const { return v[i]; }
  __device__ __forceinline__ bool has_val() const { return v != nullptr; }
  __device__ __forceinline__ void prefetch_val(u64 i) const {
    if (v) prefetch_l2(v + i);
  }
  __device__ __forceinline__ K hist_key(u64 i) const { return k[i]; }
  __device__ __forceinline__ void run_fix(u64, int, int*) const {}  // input order is the sort's order
  using Item = K;  // (the kPre pass's register-held items; not used with ArrayIn)
  __device__ __forceinline__ K item(u64 i) const { return k[i]; }
  __device__ __forceinline__ K key_of(K x, u64) const { return x; }
  __device__ __forceinline__ V val_of(K, u64 i) const { return v[i]; }
};

// ---------------------------------------------------- single-pass scan ----
//
// Flag -> exclusive scan -> scatter in ONE pass over the input (decoupled
// look-back): each CTA takes a tile by ticket, scans its 2048 flags, posts
// its aggregate, resolves its global prefix from its predecessors' posts,
// and hands every item (index, exclusive prefix, flag) to the scatter
// functor. Replaces the three-kernel chains (tile sums, rescan, scatter)
// that read the input twice. The grand total lands in *total.
// look-back status words: relaxed GPU-scope atomics (the word carries flag and
// value together, nothing else is published through it), not volatile
// accesses, which compile to system-scope strong loads
__device__ __forceinline__ u64 lb_load(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void lb_store(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr u64 kLbAggregate = 1ull << 62;
constexpr u64 kLbInclusive = 2ull << 62;
constexpr u64 kLbValueMask = (1ull << 62) - 1;

// Flags are 0/1. Each warp owns 256 consecutive items (8 rounds of 32), so
// every flag load and every scatter is issued by 32 lanes for 32 consecutive
// items (coalesced); in-warp prefixes come from ballot + popc.
template <class FlagFn, class Scatter>
__global__ void __launch_bounds__(kScanBlock) k_scan_scatter(FlagFn flag, u64 n, u64* tile_state, u32* ticket,
                                                             u64* total, Scatter scatter) {
  __shared__ u32 s_tile;
  __shared__ u64 s_prefix;
  __shared__ u32 s_warp[kScanBlock / 32 + 1];
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const u64 tile = s_tile;
  const u64 base = tile * kScanTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 lt = (1u << lane) - 1u;
  const u64 wbase = base + static_cast<u64>(warp) * (32 * kScanItems);
  u32 f[kScanItems];
  u32 bal[kScanItems];
  u32 wsum = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const u64 i = wbase + j * 32 + lane;
    f[j] = i < n ? flag(i) : 0u;
  }
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    bal[j] = __ballot_sync(0xffffffffu, f[j] != 0);
    wsum += __popc(bal[j]);
  }
  if (lane == 0) s_warp[warp] = wsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    u32 acc = 0;
    for (int w = 0; w < kScanBlock / 32; ++w) {
      const u32 c = s_warp[w];
      s_warp[w] = acc;
      acc += c;
    }
    s_warp[kScanBlock / 32] = acc;
  }
  __syncthreads();
  const u32 agg = s_warp[kScanBlock / 32];
  if (warp == 0) {
    // warp-parallel decoupled look-back: 32 predecessors per round
    u64* st = tile_state;
    u64 prefix = 0;
    if (tile == 0) {
      if (lane == 0) lb_store(st, kLbInclusive | agg);
    } else {
      if (lane == 0) lb_store(st + tile, kLbAggregate | agg);
      long long p = static_cast<long long>(tile) - 1;
      while (true) {
        const long long idx = p - lane;
        u64 s = kLbInclusive;  // before tile 0: inclusive zero
        if (idx >= 0) {
          do {
            s = lb_load(st + idx);
          } while ((s >> 62) == 0);
        }
        const u32 incl = __ballot_sync(0xffffffffu, (s >> 62) == 2);
        const int stop = incl ? __ffs(incl) - 1 : 31;  // closest predecessor holding a full prefix
        u64 v = lane <= stop ? (s & kLbValueMask) : 0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        prefix += v;
        if (incl) break;
        p -= 32;
      }
      if (lane == 0) lb_store(st + tile, kLbInclusive | (prefix + agg));
    }
    if (lane == 0) {
      s_prefix = prefix;
      if (base + kScanTile >= n) *total = prefix + agg;
    }
  }
  __syncthreads();
  u64 run = s_prefix + s_warp[warp];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const u64 i = wbase + j * 32 + lane;
    if (i < n) scatter(i, run + __popc(bal[j] & lt), f[j]);
    run += __popc(bal[j]);
  }
}

// total -> *d_total (device). n == 0 writes 0.
template <class FlagFn, class Scatter>
void scan_scatter(Ctx& ctx, FlagFn flag, u64 n, u64* d_total, Scatter scatter) {
  cudaStream_t st = ctx.stream;
  if (n == 0) {
    TWG_CUDA(cudaMemsetAsync(d_total, 0, sizeof(u64), st));
    return;
  }
  const u64 tiles = (n + kScanTile - 1) / kScanTile;
  DevBuf<u64> state(tiles + 1, st);
  TWG_CUDA(cudaMemsetAsync(state.p, 0, state.bytes(), st));  // +1 word holds the ticket
  k_scan_scatter<FlagFn, Scatter><<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(
      flag, n, state.p, reinterpret_cast<u32*>(state.p + tiles), d_total, scatter);
  TWG_LAUNCHED(ctx);
}

// --------------------------------------------------------------- merge ----
//
// Merge-path merge of two sorted sequences A (na) and B (nb), A first on
// ties (stable). Keys come from functors ka(i) / kb(j) returning a type with
// operator<; the emitter receives (output index, from_a, source index, key)
// and writes whatever payload columns the caller needs. One tile of
// kMergeTile outputs per CTA: a global diagonal search per tile boundary,
// the tile's keys staged in shared memory, then a per-thread diagonal
// search and an 8-element sequential merge.
constexpr int kMergeBlock = 256;
constexpr int kMergeItems = 8;
constexpr int kMergeTile = kMergeBlock * kMergeItems;

template <class KA, class KB>
__global__ void k_merge_partition(KA ka, u64 na, KB kb, u64 nb, u64 ntiles, u64* part) {
  for (u64 t = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; t <= ntiles;
       t += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 d = t * kMergeTile < na + nb ? t * kMergeTile : na + nb;
    u64 lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
    while (lo < hi) {
      const u64 mid = (lo + hi) >> 1;
      if (kb(d - 1 - mid) < ka(mid)) hi = mid;
      else lo = mid + 1;
    }
    part[t] = lo;
  }
}

template <class K, class KA, class KB, class Emit>
__global__ void __launch_bounds__(kMergeBlock) k_merge_tiles(KA ka, u64 na, KB kb, u64 nb, const u64* part,
                                                             Emit emit) {
  __shared__ K sk[kMergeTile];
  const u64 t = blockIdx.x;
  const u64 d0 = t * kMergeTile;
  const u64 d1 = d0 + kMergeTile < na + nb ? d0 + kMergeTile : na + nb;
  const u64 a0 = part[t], a1 = part[t + 1];
  const u64 b0 = d0 - a0, b1 = d1 - a1;
  const u32 nal = static_cast<u32>(a1 - a0), nbl = static_cast<u32>(b1 - b0), tot = nal + nbl;
  {
    // all of a thread's key loads issued before any is consumed (ILP for the
    // dependent id-remap gathers inside ka)
    K tmp[kMergeItems];
#pragma unroll
    for (int r = 0; r < kMergeItems; ++r) {
      const u32 k = r * kMergeBlock + threadIdx.x;
      if (k < tot) tmp[r] = k < nal ? ka(a0 + k) : kb(b0 + (k - nal));
    }
#pragma unroll
    for (int r = 0; r < kMergeItems; ++r) {
      const u32 k = r * kMergeBlock + threadIdx.x;
      if (k < tot) sk[k] = tmp[r];
    }
  }
  __syncthreads();
  const K* A = sk;
  const K* B = sk + nal;
  const u32 dl = threadIdx.x * kMergeItems;
  u32 lo = dl > nbl ? dl - nbl : 0, hi = dl < nal ? dl : nal;
  if (dl >= tot) lo = hi = 0;
  while (lo < hi) {
    const u32 mid = (lo + hi) >> 1;
    if (B[dl - 1 - mid] < A[mid]) hi = mid;
    else lo = mid + 1;
  }
  u32 i = lo, j = dl - lo;
  K out[kMergeItems];
  u32 src[kMergeItems];
#pragma unroll
  for (int k = 0; k < kMergeItems; ++k) {
    if (dl + k < tot) {
      const bool take_a = j >= nbl || (i < nal && !(B[j] < A[i]));
      if (take_a) {
        out[k] = A[i];
        src[k] = i;  // index into the tile's A range
        ++i;
      } else {
        out[k] = B[j];
        src[k] = 0x80000000u | j;
        ++j;
      }
    }
  }
  // restage the merged tile in shared memory so the emitter's column writes
  // are issued by consecutive threads for consecutive outputs (coalesced)
  __shared__ u32 ssrc[kMergeTile];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kMergeItems; ++k) {
    if (dl + k < tot) {
      sk[dl + k] = out[k];
      ssrc[dl + k] = src[k];
    }
  }
  __syncthreads();
  for (u32 o = threadIdx.x; o < tot; o += blockDim.x) {
    const u32 s = ssrc[o];
    if (s & 0x80000000u) emit(d0 + o, false, b0 + (s & 0x7fffffffu), sk[o]);
    else emit(d0 + o, true, a0 + s, sk[o]);
  }
}

template <class K, class KA, class KB, class Emit>
void merge_path(Ctx& ctx, KA ka, u64 na, KB kb, u64 nb, Emit emit) {
  const u64 total = na + nb;
  if (total == 0) return;
  cudaStream_t st = ctx.stream;
  const u64 ntiles = (total + kMergeTile - 1) / kMergeTile;
  DevBuf<u64> part(ntiles + 1, st);
  k_merge_partition<KA, KB><<<grid_for(ntiles + 1, 256, 1u << 16), 256, 0, st>>>(ka, na, kb, nb, ntiles, part.p);
  TWG_LAUNCHED(ctx);
  k_merge_tiles<K, KA, KB, Emit><<<static_cast<unsigned>(ntiles), kMergeBlock, 0, st>>>(ka, na, kb, nb, part.p,
                                                                                        emit);
  TWG_LAUNCHED(ctx);
}

// ---------------------------------------------------------- radix sort ----
//
// Stable LSD radix sort, one kernel per 8-bit digit pass ("onesweep"): the
// digit histograms of ALL passes come from one read of the keys up front;
// each pass then takes its tiles by ticket, ranks the tile stably (warp-
// private match/ballot counters + a cross-warp scan), resolves every digit's
// global offset by a decoupled look-back over the preceding tiles' posted
// counts (one thread per digit), stages the tile in digit order in shared
// memory and writes digit-contiguous, coalesced runs. Each pass reads and
// writes the data once; no per-pass histogram kernel, no count-matrix scan.
constexpr int kMaxPasses = 8;

template <class K>
__device__ __forceinline__ u32 digit_of(K k, int shift) {
  return static_cast<u32>(k >> shift) & (kRadix - 1);
}

// hist[p * 256 + d] = items whose digit p (bits lo_bit + 8p ...) is d
template <class K, class In>
__global__ void __launch_bounds__(kSortBlock) k_radix_global_hist(In in, u64 n, int lo_bit, int passes, u32* hist) {
  __shared__ u32 h[kMaxPasses][kRadix];
  for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += kSortBlock) (&h[0][0])[i] = 0;
  __syncthreads();
  for (u64 i = blockIdx.x * static_cast<u64>(kSortBlock) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * kSortBlock) {
    const K k = in.hist_key(i);  // any item order will do for counts
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p][digit_of(k, lo_bit + p * kRadixBits)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += kSortBlock) {
    const u32 c = (&h[0][0])[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

// per pass: exclusive scan of the 256 digit counts -> digit starts (in place)
static __global__ void __launch_bounds__(kRadix) k_radix_digit_starts(u32* hist, int passes) {
  for (int p = 0; p < passes; ++p) {
    u32 total;
    const u32 c = hist[p * kRadix + threadIdx.x];
    const u32 ex = block_excl_scan<u32>(c, &total);
    __syncthreads();
    hist[p * kRadix + threadIdx.x] = ex;
    __syncthreads();
  }
}

#ifndef TWG_SORT_HOLD
#define TWG_SORT_HOLD 1
#endif
constexpr bool kSortHold = TWG_SORT_HOLD != 0;
#ifndef TWG_STAT_ITEMS
#define TWG_STAT_ITEMS 6  // the statistics pass's edges per thread (window.cu kStatItems)
#endif
constexpr int kPreItems = TWG_STAT_ITEMS;
constexpr u32 kPreRowsPerBlock = 8;  // statistics rows per k_hist_rows block when the prefixes are wanted

template <class K, class V, int Items = 0>
struct OnesweepSmem {
  static constexpr int kItems = Items ? Items : (sizeof(K) + sizeof(V) > 8 ? TWG_SORT_ITEMS_WIDE : 16);
  static constexpr int kTile = kSortBlock * kItems;
  u32 wcount[kSortBlock / 32][kRadix];
  u32 tile_start[kRadix + 1];
  u64 gstart[kRadix];
  u32 tile;
  K keys[kTile];
  V vals[kTile];
};

// kPre (the first pass of the streaming bucket sort): the tile's digit
// offsets are known up front — the exclusive prefix over the preceding tiles
// of the statistics pass's per-tile digit counts (input order, tiles of the
// same size: pre_rows[tile's k_hist_rows block] + stat_rows of the block's
// earlier tiles), corrected by the input's run_fix for the one equal-time run
// the canonical order may permute across the tile's start — so the pass has
// no look-back and no ticket.
template <class K, class V, class In, int Items = 0, bool kPre = false>
__global__ void __launch_bounds__(kSortBlock) k_radix_onesweep(In in, K* __restrict__ keys_out,
                                                               V* __restrict__ vals_out, u64 n, int shift,
                                                               const u32* __restrict__ digit_start, u64* state,
                                                               u32* ticket, const u32* __restrict__ pre_rows = nullptr,
                                                               const u32* __restrict__ stat_rows = nullptr) {
  using S = OnesweepSmem<K, V, Items>;
  constexpr int kItems = S::kItems, kTile = S::kTile, kWarps = kSortBlock / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);
  const bool has_val = in.has_val();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 lt = (1u << lane) - 1u;
  if (kPre) {
    if (threadIdx.x == 0) sm.tile = blockIdx.x;
    reinterpret_cast<int*>(sm.gstart)[threadIdx.x] = 0;  // run_fix's per-digit corrections
  } else if (threadIdx.x == 0) {
    sm.tile = atomicAdd(ticket, 1u);
  }
  for (int b = threadIdx.x; b < kWarps * kRadix; b += kSortBlock) (&sm.wcount[0][0])[b] = 0;
  __syncthreads();
  if constexpr (kPre) {
    if (warp == 0) in.run_fix(static_cast<u64>(blockIdx.x) * kTile, shift, reinterpret_cast<int*>(sm.gstart));
  }
  const u64 tile = sm.tile;
  const u64 base = tile * kTile;
  const u32 tile_n = static_cast<u32>(n - base < static_cast<u64>(kTile) ? n - base : kTile);
  // warp w owns the tile's items [w*32*kItems, ...) in kItems rounds of 32:
  // item order (warp, round, lane) == input order keeps the sort stable
  const u32 wbase = static_cast<u32>(warp) * (32 * kItems);
  K key[kItems];
  u32 rank[kItems];
  // kPre && TWG_SORT_HOLD: the input's whole item (OwnerIn: the 16-B log
  // record) stays in registers from the key load to the staging store
  [[maybe_unused]] typename In::Item held[(kPre && kSortHold) ? kItems : 1];
  if constexpr (kPre && kSortHold) {
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const u32 i = wbase + j * 32 + lane;
      if (i < tile_n) {
        held[j] = in.item(base + i);
        key[j] = in.key_of(held[j], base + i);
      } else {
        key[j] = K(0);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < kItems; ++j) {  // the payloads' DRAM fetch starts now, into L2
      const u32 i = wbase + j * 32 + lane;
      if (i < tile_n) in.prefetch_val(base + i);
    }
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const u32 i = wbase + j * 32 + lane;
      key[j] = i < tile_n ? in.key(base + i) : K(0);
    }
  }
  // kPre: this tile's digit-d offset = the prefix of its k_hist_rows block
  // (pre_rows = csum after k_csum_scan) + the statistics rows of the block's
  // tiles before it (< kPreRowsPerBlock loads in flight with the key loads)
  [[maybe_unused]] u32 pre_base = 0, pre_sum = 0;
  if constexpr (kPre) {
    const u64 blk = tile / kPreRowsPerBlock;
    pre_base = pre_rows[blk * 512 + threadIdx.x];
#pragma unroll
    for (u32 k = 0; k < kPreRowsPerBlock - 1; ++k) {
      const u64 r = blk * kPreRowsPerBlock + k;
      if (r < tile) pre_sum += stat_rows[r * 512 + threadIdx.x];
    }
  }
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const u32 i = wbase + j * 32 + lane;
    const bool valid = i < tile_n;
    const u32 d = valid ? digit_of(key[j], shift) : 0u;
    const u32 peers = digit_peers<kRadixBits>(d, valid);
    const u32 before = valid ? sm.wcount[warp][d] : 0u;
    __syncwarp();
    if (valid && (__ffs(peers) - 1) == lane) sm.wcount[warp][d] = before + __popc(peers);
    __syncwarp();
    rank[j] = before + __popc(peers & lt);
  }
  __syncthreads();
  // thread d: digit d's count in this tile, posted at once (successors wait
  // on it); the tile is staged in shared memory BEFORE this tile's own look-
  // back, so the predecessors get that long to post theirs
  const int d = threadIdx.x;
  u32 acc = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const u32 c = sm.wcount[w][d];
    sm.wcount[w][d] = acc;
    acc += c;
  }
  if (!kPre) lb_store(state + tile * kRadix + d, (tile == 0 ? kLbInclusive : kLbAggregate) | acc);
  {
    u32 total;
    sm.tile_start[d] = block_excl_scan<u32>(acc, &total);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kItems; ++j) {  // stage in digit order; payloads loaded only now
    const u32 i = wbase + j * 32 + lane;
    if (i < tile_n) {
      const u32 dg = digit_of(key[j], shift);
      const u32 pos = sm.tile_start[dg] + sm.wcount[warp][dg] + rank[j];
      sm.keys[pos] = key[j];
      if constexpr (kPre && kSortHold) sm.vals[pos] = in.val_of(held[j], base + i);
      else if (has_val) sm.vals[pos] = in.val(base + i);
    }
  }
  if (kPre) {
    const int fix = reinterpret_cast<const int*>(sm.gstart)[d];  // read before gstart is overwritten
    __syncthreads();
    sm.gstart[d] = digit_start[d] + static_cast<u64>(static_cast<i64>(pre_base + pre_sum) + fix);
  } else {
    u64 excl = 0;
    if (tile > 0) {
      // four predecessors per round: their words are requested together
      long long j = static_cast<long long>(tile) - 1;
      bool done = false;
      while (!done) {
        u64 st4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) st4[q] = j - q >= 0 ? lb_load(state + (j - q) * kRadix + d) : kLbInclusive;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (done) break;
          while ((st4[q] >> 62) == 0) st4[q] = lb_load(state + (j - q) * kRadix + d);
          excl += st4[q] & kLbValueMask;
          done = (st4[q] >> 62) == 2;
        }
        j -= 4;
      }
      lb_store(state + tile * kRadix + d, kLbInclusive | (excl + acc));
    }
    sm.gstart[d] = digit_start[d] + excl;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const u32 pos = static_cast<u32>(j) * kSortBlock + threadIdx.x;
    if (pos < tile_n) {
      const K k = sm.keys[pos];
      const u32 d = digit_of(k, shift);
      const u64 dst = sm.gstart[d] + (pos - sm.tile_start[d]);
      keys_out[dst] = k;
      if (has_val) vals_out[dst] = sm.vals[pos];
    }
  }
}

// Passes over key bits [lo_bit, bits): the first reads through `in0`, the
// rest ping-pong between (*keys, *vals) and the alt buffers; the sorted
// result ends in (*keys, *vals). Keys-only when the values are null.
// pre_hist (device, passes x 256 digit counts of the items): computed by the
// caller (the statistics pass fuses the owner-digit histogram), so the
// histogram kernel is skipped; it is consumed (turned into digit starts).
// pre_rows + stat_rows (with pre_hist; the first pass reading through `in0`):
// the statistics pass's per-tile digit rows (tiles of kPreItems * kSortBlock
// items) and the exclusive prefixes of their k_hist_rows block sums
// (k_csum_scan) — that pass runs without look-back.

template <class K, class V, class In>
void radix_sort_impl(Ctx& ctx, In in0, bool from_in, K** keys, K** keys_alt, V** vals, V** vals_alt, u64 n,
                     int bits, int lo_bit, u32* pre_hist = nullptr, const u32* pre_rows = nullptr,
                     const u32* stat_rows = nullptr) {
  using S = OnesweepSmem<K, V>;
  cudaStream_t st = ctx.stream;
  const int passes = (bits - lo_bit + kRadixBits - 1) / kRadixBits;
  if (passes > kMaxPasses) fail(TWG_EINVAL, "radix_sort_pairs: key too wide");
  const u64 tiles = (n + S::kTile - 1) / S::kTile;
  if (tiles >= (1ull << 31)) fail(TWG_EINVAL, "radix_sort_pairs: input too large");
  static const bool attr = [] {
    TWG_CUDA(cudaFuncSetAttribute(k_radix_onesweep<K, V, In>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(S))));
    TWG_CUDA(cudaFuncSetAttribute(k_radix_onesweep<K, V, ArrayIn<K, V>>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(S))));
    return true;
  }();
  (void)attr;
  using SP = OnesweepSmem<K, V, kPreItems>;
  if (pre_rows) {
    static const bool attr_pre = [] {
      TWG_CUDA(cudaFuncSetAttribute(k_radix_onesweep<K, V, In, kPreItems, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(SP))));
      return true;
    }();
    (void)attr_pre;
  }
  DevBuf<u32> own_hist;
  DevBuf<u64> state(tiles * kRadix + 1, st);  // + the ticket word
  u32* hist = pre_hist;
  if (!hist) {
    own_hist.alloc(static_cast<u64>(passes) * kRadix, st);
    hist = own_hist.p;
    TWG_CUDA(cudaMemsetAsync(hist, 0, own_hist.bytes(), st));
    const unsigned hgrid = grid_for(n, kSortBlock, static_cast<unsigned>(ctx.sm_count) * 8);
    if (from_in) k_radix_global_hist<K, In><<<hgrid, kSortBlock, 0, st>>>(in0, n, lo_bit, passes, hist);
    else k_radix_global_hist<K, ArrayIn<K, V>><<<hgrid, kSortBlock, 0, st>>>(ArrayIn<K, V>{*keys, *vals}, n, lo_bit,
                                                                              passes, hist);
    TWG_LAUNCHED(ctx);
  }
  k_radix_digit_starts<<<1, kRadix, 0, st>>>(hist, passes);
  TWG_LAUNCHED(ctx);
  u32* ticket = reinterpret_cast<u32*>(state.p + tiles * kRadix);
  for (int p = 0; p < passes; ++p) {
    const int shift = lo_bit + p * kRadixBits;
    const bool pre = p == 0 && from_in && pre_rows;  // no look-back: its state words are not read
    if (!pre) TWG_CUDA(cudaMemsetAsync(state.p, 0, state.bytes(), st));
    if (pre) {
      k_radix_onesweep<K, V, In, kPreItems, true>
          <<<static_cast<unsigned>((n + SP::kTile - 1) / SP::kTile), kSortBlock, sizeof(SP), st>>>(
              in0, *keys, *vals, n, shift, hist + p * kRadix, state.p, ticket, pre_rows, stat_rows);
    } else if (p == 0 && from_in) {
      k_radix_onesweep<K, V, In><<<static_cast<unsigned>(tiles), kSortBlock, sizeof(S), st>>>(
          in0, *keys, *vals, n, shift, hist + p * kRadix, state.p, ticket);
    } else {
      k_radix_onesweep<K, V, ArrayIn<K, V>><<<static_cast<unsigned>(tiles), kSortBlock, sizeof(S), st>>>(
          ArrayIn<K, V>{*keys, *vals}, *keys_alt, *vals_alt, n, shift, hist + p * kRadix, state.p, ticket);
      std::swap(*keys, *keys_alt);
      std::swap(*vals, *vals_alt);
    }
    TWG_LAUNCHED(ctx);
  }
}

// Stable LSD sort of (keys, vals) by key bits [lo_bit, bits). Sorted output
// lands in (*keys, *vals); the alt buffers are scratch of the same size.
// n < 2^32. Keys-only when *vals == nullptr.
template <class K, class V = u32>
void radix_sort_pairs(Ctx& ctx, K** keys, K** keys_alt, V** vals, V** vals_alt, u64 n, int bits, int lo_bit = 0) {
  if (n < 2 || bits <= lo_bit) return;
  radix_sort_impl<K, V>(ctx, ArrayIn<K, V>{*keys, *vals}, false, keys, keys_alt, vals, vals_alt, n, bits, lo_bit);
}

// Same, the first pass reading its items through `in` (sorted result in
// (*keys, *vals); n >= 1).
template <class K, class V, class In>
void radix_sort_pairs_from(Ctx& ctx, In in, K** keys, K** keys_alt, V** vals, V** vals_alt, u64 n, int bits,
                           int lo_bit, u32* pre_hist = nullptr, const u32* pre_rows = nullptr,
                           const u32* stat_rows = nullptr) {
  radix_sort_impl<K, V>(ctx, in, true, keys, keys_alt, vals, vals_alt, n, bits > lo_bit ? bits : lo_bit + 1, lo_bit,
                        pre_hist, pre_hist && stat_rows ? pre_rows : nullptr, stat_rows);
}

// Per-tile digit-count rows (rows x 2*256, the statistics pass's output)
// summed into hist (zeroed) — the fused owner-digit histogram's reduction.
// csum (optional): each block's column sums, for k_csum_scan (which then writes hist).
static __global__ void __launch_bounds__(512) k_hist_rows(const u32* rows, u64 nrows, u64 rows_per_block, u32* hist,
                                                          u32* csum = nullptr) {
  const u64 r0 = blockIdx.x * rows_per_block, r1 = min(nrows, r0 + rows_per_block);
  u32 acc = 0;
  for (u64 r = r0; r < r1; ++r) acc += rows[r * 512 + threadIdx.x];
  if (csum) csum[blockIdx.x * 512ull + threadIdx.x] = acc;  // k_csum_scan writes hist
  else if (acc) atomicAdd(&hist[threadIdx.x], acc);
}

// k_csum_scan: column d of csum (k_hist_rows' block sums, nblocks rows of 512,
// <= kCsumPer * 1024 rows) turned in place into its exclusive prefix over the
// blocks, and its total written to hist[d] (the digit histogram). Block d,
// thread t owns kCsumPer consecutive block rows.
constexpr u32 kCsumPer = 8;
static __global__ void __launch_bounds__(1024) k_csum_scan(u32* csum, u32 nblocks, u32* hist) {
  __shared__ u32 ws[32];
  const u32 t = threadIdx.x, lane = t & 31, warp = t >> 5, d = blockIdx.x;
  u32 v[kCsumPer];
  u32 mine = 0;
#pragma unroll
  for (u32 k = 0; k < kCsumPer; ++k) {
    const u32 c = t * kCsumPer + k;
    v[k] = c < nblocks ? csum[c * 512ull + d] : 0u;
  }
#pragma unroll
  for (u32 k = 0; k < kCsumPer; ++k) mine += v[k];
  u32 incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<u32>(o)) incl += y;
  }
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    u32 w = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= static_cast<u32>(o)) w += y;
    }
    ws[lane] = w;
  }
  __syncthreads();
  u32 run = (warp ? ws[warp - 1] : 0u) + incl - mine;
#pragma unroll
  for (u32 k = 0; k < kCsumPer; ++k) {
    const u32 c = t * kCsumPer + k;
    if (c < nblocks) csum[c * 512ull + d] = run;
    run += v[k];
  }
  if (t == 0) hist[d] = ws[31];
}

}  // namespace twg
