// Microbenchmark: grid-barrier round-trip latency on B200 for the persistent cycle kernels
// (VERDICT r01 "cut barrier cost").  Every block of a co-resident grid (256
// threads, 3 or 4 blocks per SM) crosses ITERS barriers; ns per barrier = elapsed / ITERS.
//   flat     : the solver's barrier — one atomicAdd per block on one counter, poll with ld.acquire
//   flags    : every block stores its epoch to its own 128-byte line; block 0's warps gather
//              them and store one release word that everyone polls (no same-address atomics)
//   cluster  : hardware cluster barrier (barrier.cluster) inside clusters of C blocks, then the
//              flat barrier among the cluster leaders only, then barrier.cluster again
//   redflat  : as flat, arrivals as fire-and-forget red.release.gpu.add
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 barrier.cu -o barrier
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int THREADS = 256;

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_rel_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int SLEEP>
__device__ __forceinline__ void bar_flat(unsigned long long* bar, unsigned long long target, bool red) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (red) red_rel_add(bar, 1ull);
    else { __threadfence(); atomicAdd(bar, 1ull); }
    while (ld_acq(bar) < target) if (SLEEP) __nanosleep(SLEEP);
  }
  __syncthreads();
}

template <int SLEEP>
__global__ void __launch_bounds__(THREADS) k_flat(unsigned long long* bar, int iters, int red) {
  const unsigned long long G = gridDim.x;
  for (int i = 1; i <= iters; ++i) bar_flat<SLEEP>(bar, G * i, red != 0);
}

// flags: arrival = own line; block 0 gathers with all its threads, releases one word
__global__ void __launch_bounds__(THREADS) k_flags(unsigned long long* lines, unsigned long long* rel, int iters) {
  const unsigned G = gridDim.x;
  for (int i = 1; i <= iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) st_rel(lines + 16ull * blockIdx.x, (unsigned long long)i);
    if (blockIdx.x == 0) {
      for (unsigned b = threadIdx.x; b < G; b += THREADS)
        while (ld_acq(lines + 16ull * b) < (unsigned long long)i) { }
      __syncthreads();
      if (threadIdx.x == 0) st_rel(rel, (unsigned long long)i);
    } else if (threadIdx.x == 0) {
      while (ld_acq(rel) < (unsigned long long)i) __nanosleep(32);
    }
    __syncthreads();
  }
}

// cluster: hardware barrier inside the cluster, flat barrier among cluster leaders
__global__ void __launch_bounds__(THREADS) k_cluster(unsigned long long* bar, int iters, int csize) {
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const unsigned long long L = gridDim.x / csize;
  for (int i = 1; i <= iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (rank == 0 && threadIdx.x == 0) {
      red_rel_add(bar, 1ull);
      while (ld_acq(bar) < L * (unsigned long long)i) __nanosleep(32);
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 20000;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *bar, *lines;
  cudaMalloc(&bar, 256);
  cudaMalloc(&lines, 16ull * 8 * 2048 + 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, int grid, auto launch) {
    cudaMemset(bar, 0, 256);
    cudaMemset(lines, 0, 16ull * 8 * 2048 + 1024);
    launch();  // warm-up
    cudaDeviceSynchronize();
    cudaMemset(bar, 0, 256);
    cudaMemset(lines, 0, 16ull * 8 * 2048 + 1024);
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("%-22s grid %4d: %8.0f ns per barrier %s\n", name, grid, 1e6 * ms / iters, e ? cudaGetErrorString(e) : "");
  };
  for (int per : {3, 4}) {
    const int grid = per * nsm;
    timeit("flat sleep32", grid, [&] { k_flat<32><<<grid, THREADS, 48 * 1024>>>(bar, iters, 0); });
    timeit("flat nosleep", grid, [&] { k_flat<0><<<grid, THREADS, 48 * 1024>>>(bar, iters, 0); });
    timeit("redflat sleep32", grid, [&] { k_flat<32><<<grid, THREADS, 48 * 1024>>>(bar, iters, 1); });
    timeit("flags", grid, [&] { k_flags<<<grid, THREADS, 48 * 1024>>>(lines, bar + 8, iters); });
    for (int cs : {2, 4, 8}) {
      if (grid % cs) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(THREADS);
      cfg.dynamicSmemBytes = 48 * 1024;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int maxc = 0;
      cudaOccupancyMaxActiveClusters(&maxc, (void*)k_cluster, &cfg);
      char name[64];
      snprintf(name, sizeof(name), "cluster%d (max %d)", cs, maxc);
      if (maxc * cs < grid) { printf("%-22s grid %4d: not co-resident\n", name, grid); continue; }
      timeit(name, grid, [&] { cudaLaunchKernelEx(&cfg, k_cluster, bar, iters, cs); });
    }
  }
  return 0;
}
