// Edge files on the device (the data format in front of the
// path): the reference's TSV reader and writer (io.cpp:40-63
// read_edges_tsv, io.cpp:65-69 write_edges_tsv).
//
// Reader. getline semantics: a line starts at 0 and after every '\n' (a
// final '\n' opens no line). Empty lines and lines starting with '#' are
// skipped, then one trailing '\r' is dropped (a line that was only "\r" is
// skipped too); a data line is `source<TAB>target<TAB>timestamp` with each
// field an std::from_chars int64 over the whole token (optional '-', digits,
// no overflow), and negative values rejected — in this order per field,
// fields left to right, the first failing line of the file reported. Device
// passes: line starts by flag + decoupled-look-back scan over the bytes; one
// thread per line classifies and parses it (adjacent threads read adjacent
// lines); flag + scan compaction of the data lines into SoA columns; the
// first error line by atomicMin. The caller re-parses that one line on the
// host for the reference's exact message.
//
// Writer. `source \t target \t time \n` per edge in `os <<` decimal: per-edge
// byte counts -> scan -> one thread per edge writes its line.
#include "primitives.cuh"
#include "walk.cuh"

namespace twg {

namespace {

constexpr int kBlock = 256;

unsigned grid(Ctx& ctx, u64 n) { return grid_for(n, kBlock, static_cast<unsigned>(ctx.sm_count) * 16); }

struct LineStartFn {
  const char* s;
  __device__ __forceinline__ u32 operator()(u64 p) const { return (p == 0 || s[p - 1] == '\n') ? 1u : 0u; }
};
__global__ void k_count_lines(const char* s, u64 bytes, unsigned long long* n) {
  u32 c = 0;
  for (u64 p = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; p < bytes;
       p += static_cast<u64>(gridDim.x) * blockDim.x)
    c += (p == 0 || s[p - 1] == '\n') ? 1u : 0u;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(n, static_cast<unsigned long long>(c));
}

struct LineStartScatter {
  u64* starts;
  __device__ __forceinline__ void operator()(u64 i, u64 g, u32 f) const {
    if (f) starts[g] = i;
  }
};

// std::from_chars(int64) over the whole token [b, e): false if empty, a
// non-digit, or out of range
__device__ bool parse_i64(const char* b, const char* e, i64* out) {
  const bool neg = b < e && *b == '-';
  if (neg) ++b;
  if (b == e) return false;
  const u64 limit = neg ? (1ull << 63) : (1ull << 63) - 1u;
  u64 m = 0;
  for (; b < e; ++b) {
    const unsigned d = static_cast<unsigned char>(*b) - static_cast<unsigned>('0');
    if (d > 9u) return false;
    if (m > (limit - d) / 10u) return false;
    m = m * 10u + d;
  }
  *out = neg ? static_cast<i64>(0ull - m) : static_cast<i64>(m);
  return true;
}

__global__ void k_parse_lines(const char* s, u64 bytes, const u64* starts, u64 L, i64* src, i64* dst, i64* tt,
                              u8* kind, unsigned long long* first_err) {
  for (u64 k = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; k < L;
       k += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 b = starts[k];
    u64 e = k + 1 < L ? starts[k + 1] - 1 : (s[bytes - 1] == '\n' ? bytes - 1 : bytes);
    u8 r = kLineSkip;
    if (e > b && s[b] != '#') {
      if (s[e - 1] == '\r') --e;
      if (e > b) {
        u64 t1 = b;
        while (t1 < e && s[t1] != '\t') ++t1;
        u64 t2 = t1 < e ? t1 + 1 : e;
        while (t2 < e && s[t2] != '\t') ++t2;
        if (t1 >= e || t2 >= e) {
          r = kLineErrTabs;
        } else {
          const char* c = s;
          const u64 fb[3] = {b, t1 + 1, t2 + 1}, fe[3] = {t1, t2, e};
          i64 v[3] = {0, 0, 0};
          r = kLineEdge;
          for (int f = 0; f < 3 && r == kLineEdge; ++f) {
            if (!parse_i64(c + fb[f], c + fe[f], &v[f])) r = static_cast<u8>(kLineErrInvalid + f);
            else if (v[f] < 0) r = static_cast<u8>(kLineErrNegative + f);
          }
          src[k] = v[0];
          dst[k] = v[1];
          tt[k] = v[2];
        }
      }
    }
    kind[k] = r;
    if (r >= kLineErrTabs) atomicMin(first_err, static_cast<unsigned long long>(k));
  }
}

struct EdgeLineFn {
  const u8* kind;
  __device__ __forceinline__ u32 operator()(u64 k) const { return kind[k] == kLineEdge ? 1u : 0u; }
};
struct EdgeLineScatter {
  const i64 *src, *dst, *tt;
  i64 *os, *od, *ot;
  __device__ __forceinline__ void operator()(u64 k, u64 g, u32 f) const {
    if (f) {
      os[g] = src[k];
      od[g] = dst[k];
      ot[g] = tt[k];
    }
  }
};

__device__ __forceinline__ u32 dec_len(i64 x) {
  u64 m = x < 0 ? 0ull - static_cast<u64>(x) : static_cast<u64>(x);
  u32 n = x < 0 ? 2u : 1u;
  while (m >= 10u) {
    m /= 10u;
    ++n;
  }
  return n;
}

__device__ __forceinline__ char* put_dec(char* p, i64 x) {
  u64 m = x < 0 ? 0ull - static_cast<u64>(x) : static_cast<u64>(x);
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

struct EdgeTextSizeFn {
  const i64 *s, *d, *t;
  __device__ __forceinline__ u64 operator()(u64 i) const { return dec_len(s[i]) + dec_len(d[i]) + dec_len(t[i]) + 3u; }
};

__global__ void k_edges_text(EdgeTextSizeFn e, u64 n, const u64* offs, char* out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    char* p = out + offs[i];
    p = put_dec(p, e.s[i]);
    *p++ = '\t';
    p = put_dec(p, e.d[i]);
    *p++ = '\t';
    p = put_dec(p, e.t[i]);
    *p = '\n';
  }
}

}  // namespace

void parse_edges_tsv(Ctx& ctx, const char* text, u64 bytes, DevBuf<i64>& src, DevBuf<i64>& dst, DevBuf<i64>& t,
                     u64* count, u64* error_line, u8* error_kind) {
  cudaStream_t st = ctx.stream;
  *count = 0;
  *error_line = 0;
  *error_kind = kLineSkip;
  if (bytes == 0) return;
  DevBuf<char> s(bytes, st);
  TWG_CUDA(cudaMemcpyAsync(s.p, text, bytes, cudaMemcpyHostToDevice, st));
  // line starts: every position 0 or after a '\n' (the lines getline yields)
  TWG_CUDA(cudaMemsetAsync(ctx.d_scalars + 24, 0, sizeof(u64), st));
  k_count_lines<<<grid(ctx, bytes), kBlock, 0, st>>>(s.p, bytes,
                                                     reinterpret_cast<unsigned long long*>(ctx.d_scalars + 24));
  TWG_LAUNCHED(ctx);
  u64 sc[1];
  read_scalars(ctx, ctx.d_scalars + 24, sc, 1);
  const u64 L = sc[0];
  DevBuf<u64> starts(L, st);
  scan_scatter(ctx, LineStartFn{s.p}, bytes, ctx.d_scalars + 24, LineStartScatter{starts.p});
  DevBuf<i64> ls(L, st), ld(L, st), lt(L, st);
  DevBuf<u8> kind(L, st);
  DevBuf<unsigned long long> err(1, st);
  TWG_CUDA(cudaMemsetAsync(err.p, 0xff, sizeof(unsigned long long), st));
  k_parse_lines<<<grid(ctx, L), kBlock, 0, st>>>(s.p, bytes, starts.p, L, ls.p, ld.p, lt.p, kind.p, err.p);
  TWG_LAUNCHED(ctx);
  unsigned long long first = 0;
  TWG_CUDA(cudaMemcpyAsync(&first, err.p, sizeof(first), cudaMemcpyDeviceToHost, st));
  TWG_CUDA(cudaStreamSynchronize(st));
  if (first != ~0ull) {  // the first bad line (1-based) and its kind
    u8 k = 0;
    TWG_CUDA(cudaMemcpy(&k, kind.p + first, 1, cudaMemcpyDeviceToHost));
    *error_line = first + 1;
    *error_kind = k;
    return;
  }
  src.alloc(L ? L : 1, st);
  dst.alloc(L ? L : 1, st);
  t.alloc(L ? L : 1, st);
  scan_scatter(ctx, EdgeLineFn{kind.p}, L, ctx.d_scalars + 25,
               EdgeLineScatter{ls.p, ld.p, lt.p, src.p, dst.p, t.p});
  read_scalars(ctx, ctx.d_scalars + 25, sc, 1);
  *count = sc[0];
}

void format_edges_tsv(Ctx& ctx, const i64* src, const i64* dst, const i64* t, u64 n, DevBuf<char>& text,
                      u64* bytes) {
  cudaStream_t st = ctx.stream;
  const EdgeTextSizeFn f{src, dst, t};
  DevBuf<u64> offs(n + 1, st);
  exclusive_scan<u64>(ctx, f, n, offs.p);
  u64 total[1];
  read_scalars(ctx, offs.p + n, total, 1);
  *bytes = total[0];
  text.alloc(total[0] ? total[0] : 1, st);
  if (n) {
    k_edges_text<<<grid(ctx, n), kBlock, 0, st>>>(f, n, offs.p, text.p);
    TWG_LAUNCHED(ctx);
  }
}

}  // namespace twg
