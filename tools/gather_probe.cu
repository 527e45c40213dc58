// Random-gather ceiling of this B200's HBM: atoms per second the memory
// system serves when threads issue independent loads of aligned atoms
// (pattern 0: uniformly random over the footprint; pattern 1: warp-coalesced
// sequential, the copy-like reference point) over footprints from L2-sized
// to far beyond L2. The walk kernel's gathers are of the random kind.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/gather_probe tools/gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int kAtom, int kIlp>
__global__ void k_gather(const int4* buf, uint64_t n_atoms, int per, uint64_t seed, int pattern, int4* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  uint64_t x = seed * 0x9e3779b97f4a7c15ull + tid * 0xbf58476d1ce4e5b9ull + 1;
  int acc = 0;
  for (int r = 0; r < per; r += kIlp) {
    int4 v[kIlp][kAtom / 16];
#pragma unroll
    for (int k = 0; k < kIlp; ++k) {
      uint64_t a;
      if (pattern == 0) {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        a = (x >> 20) & (n_atoms - 1);
      } else {
        a = ((uint64_t)(r + k) * nthr + tid) & (n_atoms - 1);
      }
      const int4* p = buf + a * (kAtom / 16);
#pragma unroll
      for (int q = 0; q < kAtom / 16; ++q) v[k][q] = __ldcg(p + q);
    }
#pragma unroll
    for (int k = 0; k < kIlp; ++k)
#pragma unroll
      for (int q = 0; q < kAtom / 16; ++q) acc ^= v[k][q].x ^ v[k][q].y ^ v[k][q].z ^ v[k][q].w;
  }
  if (acc == 0x12345) sink[0].x = acc;
}

template <int kAtom, int kIlp>
void run(const int4* buf, int4* sink, int blocks_per_sm, int sms, uint64_t span, int pattern) {
  const uint64_t n_atoms = span / kAtom;  // the footprint (a power of two)
  const int per = 64;
  const int threads = 256, blocks = sms * blocks_per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_gather<kAtom, kIlp><<<blocks, threads>>>(buf, n_atoms, per, 1, pattern, sink);
  cudaEventRecord(a);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) k_gather<kAtom, kIlp><<<blocks, threads>>>(buf, n_atoms, per, 7 + i, pattern, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const cudaError_t e = cudaGetLastError();
  const double atoms = (double)blocks * threads * per * reps;
  std::printf("{\"pattern\": \"%s\", \"footprint_GiB\": %.3f, \"atom_bytes\": %d, \"ilp\": %d, \"ctas_per_sm\": %d, "
              "\"G_atoms_per_s\": %.3f, \"GB_per_s\": %.1f, \"err\": \"%s\"}\n",
              pattern ? "sequential" : "random", span / 1073741824.0, kAtom, kIlp, blocks_per_sm,
              atoms / (ms * 1e-3) / 1e9, atoms * kAtom / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t bytes = 16ull << 30;  // 16 GiB: far beyond the 126 MB L2
  int4* buf = nullptr;
  int4* sink = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
  cudaMalloc(&sink, 64);
  cudaMemset(buf, 1, bytes);
  cudaDeviceSynchronize();
  for (int pattern : {1, 0}) {
    for (uint64_t span : {1ull << 27, 1ull << 28, 1ull << 29, 1ull << 30, 2ull << 30, 4ull << 30, 16ull << 30}) {
      run<64, 4>(buf, sink, 8, sms, span, pattern);
      if (pattern == 0) run<32, 4>(buf, sink, 8, sms, span, pattern);
    }
  }
  cudaFree(buf);
  return 0;
}
