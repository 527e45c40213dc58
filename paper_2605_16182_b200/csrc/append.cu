// Streaming append ingest: the time-ordered fast path of
// WindowManager::ingest_batch (window_manager.cpp:14-62) on the shared
// EdgeLog / NodeArena representation (store.cuh).
//
// Preconditions (checked by the caller, window.cu ingest_streaming): the
// admitted batch sorts after every survivor in canonical order (the merge
// is a concatenation) and the node population is unchanged (new dense ids
// == old dense ids), so every id, every surviving entry and every surviving
// mark keeps its value. The snapshot the reference would rebuild from
// scratch is then
//   edges   = old edges [from, m) ++ sorted batch          -> a log append
//   ts view = old groups with time >= cutoff ++ batch groups -> a log append
//   node v  = v's entries with t >= cutoff ++ v's batch entries (canonical
//             order), marks likewise                          -> region append
// and the cost per batch is O(batch + V) instead of O(window):
//   1. log append of the sorted batch; ts groups of the batch by flag+scan;
//   2. batch entries stable-sorted by owner (radix), run bounds per node;
//   3. per node: eviction = galloping lower_bound(cutoff) on the region's
//      entry times and mark times; slack check; regions without room are
//      relocated (block-aggregated bump allocation), all regions when the
//      arena is replaced;
//   4. one decoupled-look-back pass over the sorted batch entries places
//      them at their region ends and numbers the new marks; a per-mark pass
//      scatters the marks; a per-node pass publishes {eb, ee, gb, ge}.
// Results are bit-identical to the full rebuild (tests compare every array
// after every batch against the oracle and the reference).
#include "primitives.cuh"
#include "window.cuh"

namespace twg {

namespace {

constexpr int kBlock = 256;
constexpr u32 kBigRegion = 2048;  // relocations larger than this get a CTA grid each
constexpr u32 kSmallRun = 32;     // batch runs up to this length: placed by one thread per node

__device__ __forceinline__ u32 owner_of(int mode, const u32* s, const u32* d, u64 j) {
  if (mode == TWG_UNDIRECTED) return (j & 1) ? d[j >> 1] : s[j >> 1];
  return mode == TWG_BACKWARD ? d[j] : s[j];
}

unsigned grid(Ctx& ctx, u64 n) { return grid_for(n, kBlock, static_cast<unsigned>(ctx.sm_count) * 16); }

// first k in [0, n) with t[k] >= x (one thread)
__global__ void k_lb_time(const i64* t, u64 n, i64 x, u64* out) {
  u64 lo = 0, hi = n;
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if (t[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  *out = lo;
}

__global__ void k_copy_cols(const u32* s, const u32* d, const i64* t, u64 n, u32* os, u32* od, i64* ot) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    os[i] = s[i];
    od[i] = d[i];
    ot[i] = t[i];
  }
}

// surviving ts groups [g_cut, Z) of the old snapshot -> a fresh log
__global__ void k_copy_groups(const u32* off, const i64* tt, u64 Z, const u64* g_cut, u32* ooff, i64* ott) {
  const u64 g0 = *g_cut;
  for (u64 g = g0 + blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; g < Z;
       g += static_cast<u64>(gridDim.x) * blockDim.x) {
    ooff[g - g0] = off[g];
    ott[g - g0] = tt[g];
  }
}

// batch group starts: the first batch edge starts a group unless it shares
// the last survivor's time
struct BatchGroupFn {
  const i64* t;
  const i64* last_survivor_t;  // null when there are no survivors
  __device__ __forceinline__ u32 operator()(u64 k) const {
    if (k == 0) return last_survivor_t ? (t[0] != *last_survivor_t ? 1u : 0u) : 1u;
    return t[k] != t[k - 1] ? 1u : 0u;
  }
};

struct BatchGroupScatter {
  const i64* t;
  u32 seq_b;
  u64 zbase;              // host-known write position, or
  const u64* zbase_dev;   // device-resident one (fresh log: Z_old - g_cut)
  u32* ts_off;
  i64* ts_time;
  __device__ __forceinline__ void operator()(u64 k, u64 g, u32 f) const {
    if (!f) return;
    const u64 z = (zbase_dev ? *zbase_dev : zbase) + g;
    ts_off[z] = seq_b + static_cast<u32>(k);
    ts_time[z] = t[k];
  }
};

__global__ void k_zbase(u64 Z, const u64* g_cut, u64* out) { *out = Z - *g_cut; }

// run bounds of the owner-sorted batch entries: [ystart[v], yend[v])
__global__ void k_runs(const u32* keys, u64 Yn, u32* ystart, u32* yend) {
  for (u64 q = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; q < Yn;
       q += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 v = keys[q];
    if (q == 0 || keys[q - 1] != v) ystart[v] = static_cast<u32>(q);
    if (q + 1 == Yn || keys[q + 1] != v) yend[v] = static_cast<u32>(q + 1);
  }
}

// first pos in [lo, hi) with ent[pos].t >= x, galloping from lo (eviction
// removes a short prefix of most regions)
__device__ __forceinline__ u32 gallop_ent(const Entry* e, u32 lo, u32 hi, i64 x) {
  if (lo >= hi || e[lo].t >= x) return lo;
  u32 prev = lo, step = 1, bound = hi;
  while (true) {  // e[prev].t < x
    const u64 nx = static_cast<u64>(prev) + step;
    if (nx >= hi) break;
    if (e[nx].t >= x) {
      bound = static_cast<u32>(nx);
      break;
    }
    prev = static_cast<u32>(nx);
    step <<= 1;
  }
  u32 a = prev + 1, b = bound;
  while (a < b) {
    const u32 mid = a + ((b - a) >> 1);
    if (e[mid].t < x) a = mid + 1;
    else b = mid;
  }
  return a;
}

__device__ __forceinline__ u32 gallop_time(const i64* t, u32 lo, u32 hi, i64 x) {
  if (lo >= hi || t[lo] >= x) return lo;
  u32 prev = lo, step = 1, bound = hi;
  while (true) {
    const u64 nx = static_cast<u64>(prev) + step;
    if (nx >= hi) break;
    if (t[nx] >= x) {
      bound = static_cast<u32>(nx);
      break;
    }
    prev = static_cast<u32>(nx);
    step <<= 1;
  }
  u32 a = prev + 1, b = bound;
  while (a < b) {
    const u32 mid = a + ((b - a) >> 1);
    if (t[mid] < x) a = mid + 1;
    else b = mid;
  }
  return a;
}

struct Reloc {
  u32 v, src_e, src_g, live, glive, dst;
};

// Per node: eviction bounds, room check, relocation plan. relocate_all ==
// repack every region into a fresh arena (rend_old == nullptr).
// scal: [0] bump (u64), [1] overflow flag, [2] relocations, [3] big relocations,
//       [10] nodes with a long batch run, [11] their batch entries
__global__ void __launch_bounds__(kBlock) k_plan(const uint4* onm, u64 V, const Entry* oent, const i64* omk_time,
                                                 const u32* rend_old, const u32* ystart, const u32* yend, i64 cutoff,
                                                 u64 cap, u32* rend_new, uint4* nm_new, u32* cur0, u32* gcur0,
                                                 Reloc* list, Reloc* big, u32* bignodes, u64* scal) {
  __shared__ u64 s_base;
  __shared__ u32 s_lbase, s_bbase, s_nbase;
  for (u64 base = static_cast<u64>(blockIdx.x) * kBlock; base < V; base += static_cast<u64>(gridDim.x) * kBlock) {
    const u64 v = base + threadIdx.x;
    const bool valid = v < V;
    uint4 o = make_uint4(0, 0, 0, 0);
    u32 y = 0, eb = 0, gb = 0, req = 0;
    bool move = false;
    if (valid) {
      o = onm[v];
      y = yend[v] - ystart[v];
      eb = gallop_ent(oent, o.x, o.y, cutoff);
      gb = gallop_time(omk_time, o.z, o.w, cutoff);
      const u32 need = (o.y - eb) + y;
      move = rend_old == nullptr || static_cast<u64>(o.y) + y > rend_old[v];
      if (move) req = need + (need >> 1) + (need ? 2u : 0u);
    }
    const bool is_big = move && req && (o.y - eb) > kBigRegion;
    const bool is_small = move && req && !is_big;
    const bool is_long = y > kSmallRun;
    u32 tot;
    const u32 off = block_excl_scan<u32>(req, &tot);  // u32: one block's slack never overflows
    u32 mtot;
    const u32 midx = block_excl_scan<u32>(is_small ? 1u : 0u, &mtot);
    u32 btot;
    const u32 bidx = block_excl_scan<u32>(is_big ? 1u : 0u, &btot);
    u32 ntot;
    const u32 nidx = block_excl_scan<u32>(is_long ? 1u : 0u, &ntot);
    u32 ytot;
    block_excl_scan<u32>(is_long ? y : 0u, &ytot);
    if (threadIdx.x == 0) {
      s_base = tot ? atomicAdd(reinterpret_cast<unsigned long long*>(&scal[0]), static_cast<unsigned long long>(tot))
                   : 0ull;
      s_lbase = mtot ? atomicAdd(reinterpret_cast<unsigned int*>(&scal[2]), mtot) : 0u;
      s_bbase = btot ? atomicAdd(reinterpret_cast<unsigned int*>(&scal[3]), btot) : 0u;
      s_nbase = ntot ? atomicAdd(reinterpret_cast<unsigned int*>(&scal[10]), ntot) : 0u;
      if (ytot) atomicAdd(reinterpret_cast<unsigned long long*>(&scal[11]), static_cast<unsigned long long>(ytot));
    }
    __syncthreads();
    if (valid) {
      const u32 live = o.y - eb, glive = o.w - gb;
      if (is_long) bignodes[s_nbase + nidx] = static_cast<u32>(v);
      if (!move) {
        cur0[v] = o.y;
        gcur0[v] = o.w;
        nm_new[v] = make_uint4(eb, 0, gb, 0);
      } else {
        const u64 dst = s_base + off;
        if (dst + req > cap) {
          atomicOr(reinterpret_cast<unsigned long long*>(&scal[1]), 1ull);
        } else {
          const u32 d = static_cast<u32>(dst);
          rend_new[v] = d + req;
          cur0[v] = d + live;
          gcur0[v] = d + glive;
          nm_new[v] = make_uint4(d, 0, d, 0);
          const Reloc r{static_cast<u32>(v), eb, gb, live, glive, d};
          if (is_big) big[s_bbase + bidx] = r;
          else if (is_small) list[s_lbase + midx] = r;
        }
      }
    }
    __syncthreads();
  }
}

// relocation copies: one warp per region (small), a CTA row per region (big)
__device__ __forceinline__ void copy_region(const Reloc& r, u32 i0, u32 stride, const Entry* oent, const i64* omt,
                                            const u32* oms, Entry* ent, i64* mt, u32* ms) {
  for (u32 i = i0; i < r.live; i += stride) ent[r.dst + i] = oent[r.src_e + i];
  for (u32 i = i0; i < r.glive; i += stride) {
    mt[r.dst + i] = omt[r.src_g + i];
    ms[r.dst + i] = oms[r.src_g + i] - r.src_e + r.dst;
  }
}

__global__ void k_relocate(const Reloc* list, const u64* scal, const Entry* oent, const i64* omt, const u32* oms,
                           Entry* ent, i64* mt, u32* ms) {
  const u32 n = static_cast<u32>(scal[2]);
  const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
  for (u64 k = (blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) >> 5; k < n; k += warps)
    copy_region(list[k], threadIdx.x & 31, 32, oent, omt, oms, ent, mt, ms);
}

__global__ void k_relocate_big(const Reloc* big, const Entry* oent, const i64* omt, const u32* oms, Entry* ent,
                               i64* mt, u32* ms) {
  copy_region(big[blockIdx.y], blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, oent, omt, oms, ent, mt,
              ms);
}

__device__ __forceinline__ u32 entry_edge(int mode, u32 j) { return mode == TWG_UNDIRECTED ? (j >> 1) : j; }

struct Rec {
  u32 src, dst;
  i64 t;
};

// the sorted batch into the log, plus a 16-byte record per edge for the
// owner-ordered gathers
__global__ void k_append_batch(const u32* s, const u32* d, const i64* t, u64 n, u32* os, u32* od, i64* ot, Rec* rec) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 a = s[i], b = d[i];
    const i64 x = t[i];
    os[i] = a;
    od[i] = b;
    ot[i] = x;
    rec[i] = Rec{a, b, x};
  }
}

__device__ __forceinline__ u32 nbr_of(int mode, const Rec& r, u32 j) {
  if (mode == TWG_FORWARD) return r.dst;
  if (mode == TWG_BACKWARD) return r.src;
  return (j & 1) ? r.src : r.dst;  // side 1 (owner dst) -> src; self-loops give the owner
}

__global__ void k_owner_keys(const u32* s, const u32* d, u64 A, int mode, u32* keys, u32* vals) {
  const u64 Yn = mode == TWG_UNDIRECTED ? 2 * A : A;
  for (u64 j = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; j < Yn;
       j += static_cast<u64>(gridDim.x) * blockDim.x) {
    keys[j] = owner_of(mode, s, d, j);
    vals[j] = static_cast<u32>(j);
  }
}

// Short runs, one thread per node: the run [ystart, yend) of the
// owner-sorted entries is already in canonical order; copy it to the region
// end, append the marks (the first merges with the last surviving mark when
// the times agree), publish {eb, ee, gb, ge}; Q += ge - gb.
__global__ void __launch_bounds__(kBlock) k_place_runs(u64 V, const u32* ystart, const u32* yend, const u32* vals,
                                                       const Rec* rec, int mode, u32 seq_b, const u32* cur0,
                                                       const u32* gcur0, Entry* ent, i64* mk_time, u32* mk_start,
                                                       uint4* nm_new, u64* q_total) {
  u64 acc = 0;
  for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 ys = ystart[v], y = yend[v] - ys;
    if (y > kSmallRun) continue;
    uint4 r = nm_new[v];
    const u32 c0 = cur0[v];
    u32 g = gcur0[v];
    bool has = c0 > r.x;
    i64 prev = has ? ent[c0 - 1].t : 0;
    for (u32 i = 0; i < y; ++i) {
      const u32 j = vals[ys + i];
      const u32 k = entry_edge(mode, j);
      const Rec b = rec[k];
      Entry e;
      e.nbr = nbr_of(mode, b, j);
      e.edge = seq_b + k;
      e.t = b.t;
      ent[c0 + i] = e;
      if (!has || b.t != prev) {
        mk_time[g] = b.t;
        mk_start[g] = c0 + i;
        ++g;
      }
      prev = b.t;
      has = true;
    }
    r.y = c0 + y;
    r.w = g;
    nm_new[v] = r;
    acc += r.w - r.z;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(reinterpret_cast<unsigned long long*>(q_total), acc);
}

__device__ __forceinline__ bool long_run(const u32* ystart, const u32* yend, u32 v) {
  return yend[v] - ystart[v] > kSmallRun;
}

// Long runs, pass A flag: q starts a new timestamp mark of its (long-run) node
struct MarkFlagFn {
  const u32* keys;
  const u32* vals;
  const Rec* rec;
  int mode;
  const u32* ystart;
  const u32* yend;
  const u32* cur0;
  const uint4* nm_new;  // .x = region begin after eviction / relocation
  const Entry* ent;
  __device__ __forceinline__ u32 operator()(u64 q) const {
    const u32 v = keys[q];
    if (!long_run(ystart, yend, v)) return 0u;
    const i64 t = rec[entry_edge(mode, vals[q])].t;
    if (q > 0 && keys[q - 1] == v) return t != rec[entry_edge(mode, vals[q - 1])].t ? 1u : 0u;
    const u32 c = cur0[v];
    return (c > nm_new[v].x && ent[c - 1].t == t) ? 0u : 1u;
  }
};

struct MarkTmp {
  i64 t;
  u32 pos;
  u32 v;
};

// Long runs, pass A scatter: place the entry at its region end, record the
// mark prefix (every q: the long runs' bounds read it)
struct PlaceScatter {
  const u32* keys;
  const u32* vals;
  const Rec* rec;
  int mode;
  u32 seq_b;
  u64 Yn;
  const u32* ystart;
  const u32* yend;
  const u32* cur0;
  Entry* ent;
  u32* mscan;
  MarkTmp* mtmp;
  __device__ __forceinline__ void operator()(u64 q, u64 g, u32 f) const {
    mscan[q] = static_cast<u32>(g);
    if (q + 1 == Yn) mscan[Yn] = static_cast<u32>(g + f);
    const u32 v = keys[q];
    if (!long_run(ystart, yend, v)) return;
    const u32 j = vals[q];
    const u32 k = entry_edge(mode, j);
    const Rec b = rec[k];
    const u32 pos = cur0[v] + static_cast<u32>(q - ystart[v]);
    Entry e;
    e.nbr = nbr_of(mode, b, j);
    e.edge = seq_b + k;
    e.t = b.t;
    ent[pos] = e;
    if (f) mtmp[g] = MarkTmp{e.t, pos, v};
  }
};

// Pass B: new marks to their region slots
__global__ void k_marks_scatter(const MarkTmp* mtmp, const u64* nmarks, const u32* ystart, const u32* mscan,
                                const u32* gcur0, i64* mk_time, u32* mk_start) {
  const u64 n = *nmarks;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const MarkTmp m = mtmp[i];
    const u32 g = gcur0[m.v] + static_cast<u32>(i) - mscan[ystart[m.v]];
    mk_time[g] = m.t;
    mk_start[g] = m.pos;
  }
}

__global__ void __launch_bounds__(kBlock) k_big_finish(const u32* nodes, u64 n, const u32* ystart, const u32* yend,
                                                       const u32* mscan, const u32* cur0, const u32* gcur0,
                                                       uint4* nm_new, u64* q_total) {
  u64 acc = 0;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 v = nodes[i];
    const u32 ys = ystart[v], ye = yend[v];
    uint4 r = nm_new[v];
    r.y = cur0[v] + (ye - ys);
    r.w = gcur0[v] + (mscan[ye] - mscan[ys]);
    nm_new[v] = r;
    acc += r.w - r.z;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(reinterpret_cast<unsigned long long*>(q_total), acc);
}

bool append_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TWG_APPEND");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

bool append_ingest_enabled() { return append_enabled(); }

Store* ingest_append(Window& w, const Store& O, std::unique_ptr<Store> s, const u32* bS, const u32* bD,
                     const i64* bT, u64 A, u64 from, i64 cutoff) {
  Ctx& ctx = *w.ctx;
  cudaStream_t st = ctx.stream;
  PhaseTimer pt(ctx, "ingest_append");
  const int mode = w.mode;
  const u64 S = O.m - from;
  const u64 m = S + A;
  const u64 V = s->V;
  const u64 sides = mode == TWG_UNDIRECTED ? 2 : 1;
  const u64 Yn = sides * A;
  s->P = sides * m;
  u64* sc = ctx.d_scalars + 32;  // 32..47 private to this path
  TWG_CUDA(cudaMemsetAsync(sc, 0, 16 * sizeof(u64), st));
  const u64* d_gcut = sc + 9;  // first surviving ts group of O
  k_lb_time<<<1, 1, 0, st>>>(O.ts_time.p, O.Z, cutoff, sc + 9);
  TWG_LAUNCHED(ctx);

  // 1. edge log + ts groups
  std::shared_ptr<EdgeLog> log = O.gapped ? O.log : nullptr;
  const bool in_place = log && log->len == O.log_first + O.m && log->len + A <= log->cap;
  const u32 seq0 = O.seq0 + static_cast<u32>(from);
  const u32 seq_b = seq0 + static_cast<u32>(S);
  u64 zbase = 0;
  const u64* zbase_dev = nullptr;
  if (in_place) {
    s->log_first = O.log_first + from;
    zbase = log->zlen;
  } else {
    auto nl = std::make_shared<EdgeLog>();
    nl->cap = m + 8 * A;
    nl->src.alloc(nl->cap, st);
    nl->dst.alloc(nl->cap, st);
    nl->t.alloc(nl->cap, st);
    nl->ts_off.alloc(nl->cap, st);
    nl->ts_time.alloc(nl->cap, st);
    nl->seq0 = seq0;
    k_copy_cols<<<grid(ctx, S), kBlock, 0, st>>>(O.e_src.p + from, O.e_dst.p + from, O.e_t.p + from, S, nl->src.p,
                                                 nl->dst.p, nl->t.p);
    TWG_LAUNCHED(ctx);
    k_copy_groups<<<grid(ctx, O.Z), kBlock, 0, st>>>(O.ts_off.p, O.ts_time.p, O.Z, d_gcut, nl->ts_off.p,
                                                     nl->ts_time.p);
    TWG_LAUNCHED(ctx);
    k_zbase<<<1, 1, 0, st>>>(O.Z, d_gcut, sc + 4);
    TWG_LAUNCHED(ctx);
    zbase_dev = sc + 4;
    nl->len = S;
    log = std::move(nl);
    s->log_first = 0;
  }
  const u64 lpos = s->log_first + S;  // log index of batch edge 0
  DevBuf<Rec> brec(A, st);  // one 16-byte gather per placed entry
  k_append_batch<<<grid(ctx, A), kBlock, 0, st>>>(bS, bD, bT, A, log->src.p + lpos, log->dst.p + lpos,
                                                  log->t.p + lpos, brec.p);
  TWG_LAUNCHED(ctx);
  scan_scatter(ctx, BatchGroupFn{bT, S ? O.e_t.p + (O.m - 1) : nullptr}, A, sc + 5,
               BatchGroupScatter{bT, seq_b, zbase, zbase_dev, log->ts_off.p, log->ts_time.p});
  pt.mark("log+ts");

  // 2. batch entries grouped by owner: stable radix sort of (owner, entry)
  //    pairs; run bounds per node
  const int vb = V > 1 ? bit_width_u64(V - 1) : 0;
  DevBuf<u32> k0(Yn, st), k1(Yn, st), v0(Yn, st), v1(Yn, st);
  u32* kp = k0.p;
  u32* ka = k1.p;
  u32* vp = v0.p;
  u32* va = v1.p;
  k_owner_keys<<<grid(ctx, Yn), kBlock, 0, st>>>(bS, bD, A, mode, kp, vp);
  TWG_LAUNCHED(ctx);
  radix_sort_pairs<u32>(ctx, &kp, &ka, &vp, &va, Yn, vb);
  DevBuf<u32> ystart(V, st), yend(V, st);
  TWG_CUDA(cudaMemsetAsync(ystart.p, 0, V * 4, st));
  TWG_CUDA(cudaMemsetAsync(yend.p, 0, V * 4, st));
  k_runs<<<grid(ctx, Yn), kBlock, 0, st>>>(kp, Yn, ystart.p, yend.p);
  TWG_LAUNCHED(ctx);
  (kp == k0.p ? k1 : k0).release();  // the pass count decides which buffer holds the result
  (vp == v0.p ? v1 : v0).release();
  pt.mark("owner_sort");

  // 3. eviction + room per node; relocation / repack
  DevBuf<u32> cur0(V, st), gcur0(V, st), bignodes(V, st);
  s->nm.alloc(V, st);
  std::shared_ptr<NodeArena> arena = O.gapped ? O.arena : nullptr;
  DevBuf<Reloc> list, big;
  u64 plan[6] = {0, 0, 0, 0, 0, 0};
  auto run_plan = [&](NodeArena& dst, const u32* rend_old) {
    TWG_CUDA(cudaMemsetAsync(sc, 0, 4 * sizeof(u64), st));
    TWG_CUDA(cudaMemsetAsync(sc + 10, 0, 2 * sizeof(u64), st));
    TWG_CUDA(cudaMemcpyAsync(sc, &dst.used, sizeof(u64), cudaMemcpyHostToDevice, st));
    k_plan<<<grid(ctx, V), kBlock, 0, st>>>(O.nm.p, V, O.ent.p, O.mk_time.p, rend_old, ystart.p, yend.p, cutoff,
                                            dst.cap, dst.rend.p, s->nm.p, cur0.p, gcur0.p, list.p, big.p,
                                            bignodes.p, sc);
    TWG_LAUNCHED(ctx);
    u64 all[12];
    read_scalars(ctx, sc, all, 12);
    for (int i = 0; i < 4; ++i) plan[i] = all[i];
    plan[4] = all[10];  // long-run nodes
    plan[5] = all[11];  // their entries
  };
  list.alloc(V, st);
  big.alloc(V, st);
  bool fresh = false;
  if (arena) {
    run_plan(*arena, arena->rend.p);
    if (plan[1]) {
      arena.reset();  // exhausted: repack below
    }
  }
  if (!arena) {
    auto na = std::make_shared<NodeArena>();
    na->V = V;
    na->cap = std::min<u64>((5 * s->P) / 2 + 4 * V + 1024, 0xffffff00ull);  // u32 positions
    na->ent.alloc(na->cap, st);
    na->mk_time.alloc(na->cap, st);
    na->mk_start.alloc(na->cap, st);
    na->rend.alloc(V, st);
    na->used = 0;
    arena = std::move(na);
    run_plan(*arena, nullptr);
    if (plan[1]) fail(TWG_ENOMEM, "ingest: node arena sized below the live regions");
    fresh = true;
  }
  arena->used = plan[0];
  if (plan[2]) {
    k_relocate<<<grid(ctx, 32 * plan[2]), kBlock, 0, st>>>(list.p, sc, O.ent.p, O.mk_time.p, O.mk_start.p,
                                                           arena->ent.p, arena->mk_time.p, arena->mk_start.p);
    TWG_LAUNCHED(ctx);
  }
  for (u64 b0 = 0; b0 < plan[3]; b0 += 65535) {
    const unsigned rows = static_cast<unsigned>(std::min<u64>(65535, plan[3] - b0));
    k_relocate_big<<<dim3(32, rows), kBlock, 0, st>>>(big.p + b0, O.ent.p, O.mk_time.p, O.mk_start.p, arena->ent.p,
                                                      arena->mk_time.p, arena->mk_start.p);
    TWG_LAUNCHED(ctx);
  }
  list.release();
  big.release();
  pt.mark(fresh ? "plan+repack" : "plan+relocate");

  // 4a. short runs (the streaming common case): one thread per node copies
  //     its run (canonical order) to the region end, appends its marks and
  //     publishes {eb, ee, gb, ge}
  k_place_runs<<<grid(ctx, V), kBlock, 0, st>>>(V, ystart.p, yend.p, vp, brec.p, mode, seq_b, cur0.p, gcur0.p,
                                                arena->ent.p, arena->mk_time.p, arena->mk_start.p, s->nm.p, sc + 7);
  TWG_LAUNCHED(ctx);
  pt.mark("place_runs");

  // 4b. long runs (hub owners): one decoupled-look-back pass over the sorted
  //     entries places them and numbers their new marks (other nodes' flags
  //     are 0), a per-mark pass scatters the marks, a per-node pass publishes
  if (plan[4]) {
    DevBuf<u32> mscan(Yn + 1, st);
    DevBuf<MarkTmp> mtmp(plan[5], st);
    scan_scatter(ctx, MarkFlagFn{kp, vp, brec.p, mode, ystart.p, yend.p, cur0.p, s->nm.p, arena->ent.p}, Yn, sc + 6,
                 PlaceScatter{kp, vp, brec.p, mode, seq_b, Yn, ystart.p, yend.p, cur0.p, arena->ent.p, mscan.p,
                              mtmp.p});
    k_marks_scatter<<<grid(ctx, plan[5]), kBlock, 0, st>>>(mtmp.p, sc + 6, ystart.p, mscan.p, gcur0.p,
                                                           arena->mk_time.p, arena->mk_start.p);
    TWG_LAUNCHED(ctx);
    k_big_finish<<<grid(ctx, plan[4]), kBlock, 0, st>>>(bignodes.p, plan[4], ystart.p, yend.p, mscan.p, cur0.p,
                                                        gcur0.p, s->nm.p, sc + 7);
    TWG_LAUNCHED(ctx);
    pt.mark("place_long_runs");
  }

  // the one closing read-back: g_cut, batch groups, Q
  u64 r[4];
  TWG_CUDA(cudaMemcpyAsync(sc + 8, d_gcut, sizeof(u64), cudaMemcpyDeviceToDevice, st));
  read_scalars(ctx, sc + 5, r, 4);  // [5] Zb, [6] marks, [7] Q, [8] g_cut
  const u64 Zb = r[0], Q = r[2], g_cut = r[3];
  const u64 Z = (O.Z - g_cut) + Zb;
  s->ts_first = in_place ? O.ts_first + g_cut : 0;
  log->len = lpos + A;
  log->zlen = s->ts_first + Z;

  s->gapped = true;
  s->seq0 = seq0;
  s->m = m;
  s->Z = Z;
  s->Q = Q;
  s->e_src.alias(log->src.p + s->log_first, m);
  s->e_dst.alias(log->dst.p + s->log_first, m);
  s->e_t.alias(log->t.p + s->log_first, m);
  s->ts_off.alias(log->ts_off.p + s->ts_first, Z);
  s->ts_time.alias(log->ts_time.p + s->ts_first, Z);
  s->ent.alias(arena->ent.p, arena->cap);
  s->mk_time.alias(arena->mk_time.p, arena->cap);
  s->mk_start.alias(arena->mk_start.p, arena->cap);
  s->log = std::move(log);
  s->arena = std::move(arena);
  s->has_weights = false;
  s->has_adjacency = false;
  return s.release();
}

}  // namespace twg
