// Microbenchmark: 32-bit atomicMax throughput on B200 vs footprint and pattern.
// Words are addressed with an 8-byte stride (like the solver's state words).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
template <int K>
__global__ void k_atom(unsigned* a, unsigned nwords, unsigned iters, unsigned mode, unsigned* sink) {
  unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned acc = 0;
  for (unsigned it = 0; it < iters; ++it) {
    unsigned old[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      unsigned idx;
      unsigned r = hash32(tid * 977u + it * 131u + k * 7u);
      if (mode == 0) idx = r % nwords;                                   // uniform random
      else idx = ((tid >> 5) * 4096u + (r & 1023u) + it * 64u) % nwords;  // clustered per warp
      old[k] = atomicMax(a + 2ull * idx + 1, r);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc += old[k];
  }
  if (acc == 0x12345678u) *sink = acc;
}
__global__ void k_load(const unsigned* a, unsigned nwords, unsigned iters, unsigned* sink) {
  unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned acc = 0;
  for (unsigned it = 0; it < iters; ++it) {
    unsigned v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcg(a + 2ull * (hash32(tid * 977u + it * 131u + k * 7u) % nwords) + 1);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k];
  }
  if (acc == 0x12345678u) *sink = acc;
}
int main() {
  unsigned* a; unsigned* sink;
  size_t maxw = 1u << 28;   // 2 GiB at 8 B stride
  cudaMalloc(&a, maxw * 8); cudaMalloc(&sink, 4); cudaMemset(a, 0, maxw * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = 148 * 8, threads = 256; unsigned iters = 64;
  for (unsigned mode = 0; mode < 2; ++mode)
    for (unsigned nw : {1u << 20, 1u << 22, 1u << 24, 1u << 26, 1u << 28}) {
      k_atom<8><<<blocks, threads>>>(a, nw, 4, mode, sink);
      cudaEventRecord(e0);
      k_atom<8><<<blocks, threads>>>(a, nw, iters, mode, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double n = (double)blocks * threads * iters * 8;
      printf("atomicMax mode=%s footprint=%7.1f MB: %.1f G atomics/s\n", mode ? "clustered" : "random", nw * 8.0 / 1e6, n / ms / 1e6);
    }
  for (unsigned nw : {1u << 22, 1u << 24, 1u << 26, 1u << 28}) {
    k_load<<<blocks, threads>>>(a, nw, 4, sink);
    cudaEventRecord(e0);
    k_load<<<blocks, threads>>>(a, nw, iters, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)blocks * threads * iters * 8;
    printf("random ld.cg footprint=%7.1f MB: %.1f G loads/s\n", nw * 8.0 / 1e6, n / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
