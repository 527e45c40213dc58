// Walk output path: the reference's walk writers
// (io.cpp:119-135 write_walks_text, io.cpp:173-183 write_walks_binary)
// produced on the device, so a walk set is serialised where it lives and
// only the finished bytes cross PCIe.
//
// Text (io.cpp:119-135): one line per walk that recorded a hop (length >= 2),
// entries `node@time` separated by one space, a start sentinel (kTimeUnset /
// kTimeInfinite, io.cpp:37) printed as `node@-`, '\n' after every line;
// integers in `std::ostream <<` decimal form. Three device passes over the
// slot-major walk set: per-walk byte counts -> exclusive scan -> one thread
// per walk writes its line at its offset (reads coalesced across walks).
//
// Binary (io.cpp:173-183): "TMPW0002", u32 stride, u64 walk_count, then the
// walk-major nodes, times (i64, count x stride, zero past each length — the
// reference's zero-initialised image) and lengths (u32) — the download
// image behind a 20-byte header.
#include "primitives.cuh"
#include "walk.cuh"

namespace twg {

namespace {

constexpr int kBlock = 256;

unsigned grid(Ctx& ctx, u64 n) { return grid_for(n, kBlock, static_cast<unsigned>(ctx.sm_count) * 16); }

__device__ __forceinline__ bool sentinel(i64 t) { return t == kTimeUnset || t == kTimeInfinite; }

__device__ __forceinline__ u32 dec_len(i64 x) {  // characters of `os << x`
  u64 m = x < 0 ? static_cast<u64>(0) - static_cast<u64>(x) : static_cast<u64>(x);
  u32 n = x < 0 ? 2u : 1u;
  while (m >= 10u) {
    m /= 10u;
    ++n;
  }
  return n;
}

// writes `os << x` at p, returns the end
__device__ __forceinline__ char* put_dec(char* p, i64 x) {
  u64 m = x < 0 ? static_cast<u64>(0) - static_cast<u64>(x) : static_cast<u64>(x);
  if (x < 0) *p++ = '-';
  char buf[20];
  int k = 0;
  do {
    buf[k++] = static_cast<char>('0' + m % 10u);
    m /= 10u;
  } while (m);
  while (k) *p++ = buf[--k];
  return p;
}

struct TextSizeFn {
  const i64* nodes;  // slot-major: [slot * count + walk]
  const i64* times;
  const u32* lengths;
  u64 count;
  __device__ u64 operator()(u64 w) const {
    const u32 len = lengths[w];
    if (len < 2) return 0;  // never left the start node (io.cpp:122)
    u64 b = len;            // len - 1 separators + '\n'
    for (u32 j = 0; j < len; ++j) {
      const u64 c = static_cast<u64>(j) * count + w;
      const i64 t = times[c];
      b += dec_len(nodes[c]) + 1u + (sentinel(t) ? 1u : dec_len(t));
    }
    return b;
  }
};

__global__ void k_text_write(TextSizeFn f, const u64* offs, char* out) {
  for (u64 w = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; w < f.count;
       w += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 len = f.lengths[w];
    if (len < 2) continue;
    char* p = out + offs[w];
    for (u32 j = 0; j < len; ++j) {
      const u64 c = static_cast<u64>(j) * f.count + w;
      if (j > 0) *p++ = ' ';
      p = put_dec(p, f.nodes[c]);
      *p++ = '@';
      const i64 t = f.times[c];
      if (sentinel(t)) *p++ = '-';
      else p = put_dec(p, t);
    }
    *p = '\n';
  }
}

__global__ void k_to_slot_major(const i64* wn, const i64* wt, u64 count, u32 stride, i64* sn, i64* st) {
  const u64 cells = count * stride;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < cells;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 w = i % count, j = i / count;  // i = j * count + w: coalesced writes
    sn[i] = wn[w * stride + j];
    st[i] = wt[w * stride + j];
  }
}

}  // namespace

void walks_text(Ctx& ctx, const WalkSetDev& w, DevBuf<char>& text, u64* bytes) {
  cudaStream_t st = ctx.stream;
  const TextSizeFn f{w.nodes.p, w.times.p, w.lengths.p, w.count};
  DevBuf<u64> offs(w.count + 1, st);
  exclusive_scan<u64>(ctx, f, w.count, offs.p);
  u64 total[1];
  read_scalars(ctx, offs.p + w.count, total, 1);
  *bytes = total[0];
  text.alloc(total[0] ? total[0] : 1, st);
  if (total[0]) {
    k_text_write<<<grid(ctx, w.count), kBlock, 0, st>>>(f, offs.p, text.p);
    TWG_LAUNCHED(ctx);
  }
}

u64 walks_binary_size(const WalkSetDev& w) { return kWalkBinaryHeader + 16u * w.count * w.stride + 4u * w.count; }

void walks_from_host(Ctx& ctx, u32 stride, u64 count, const i64* nodes, const i64* times, const u32* lengths,
                     WalkSetDev& out) {
  cudaStream_t st = ctx.stream;
  const u64 cells = count * stride;
  out.ctx = &ctx;
  out.stride = stride;
  out.count = count;
  out.first = 0;
  out.nodes.alloc(cells ? cells : 1, st);
  out.times.alloc(cells ? cells : 1, st);
  out.lengths.alloc(count ? count : 1, st);
  u64 hops = 0;
  for (u64 i = 0; i < count; ++i) hops += lengths[i] > 1 ? lengths[i] - 1 : 0;
  out.hops = hops;
  if (!cells) return;
  DevBuf<i64> wn(cells, st), wt(cells, st);
  TWG_CUDA(cudaMemcpyAsync(wn.p, nodes, cells * sizeof(i64), cudaMemcpyHostToDevice, st));
  TWG_CUDA(cudaMemcpyAsync(wt.p, times, cells * sizeof(i64), cudaMemcpyHostToDevice, st));
  TWG_CUDA(cudaMemcpyAsync(out.lengths.p, lengths, count * sizeof(u32), cudaMemcpyHostToDevice, st));
  k_to_slot_major<<<grid(ctx, cells), kBlock, 0, st>>>(wn.p, wt.p, count, stride, out.nodes.p, out.times.p);
  TWG_LAUNCHED(ctx);
  TWG_CUDA(cudaStreamSynchronize(st));  // the host arrays may go away when we return
}

}  // namespace twg
