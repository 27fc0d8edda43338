// wcsp_gen.cuh — the seeded synthetic-instance recipe on the device:
// the same pure function of (seed, vertex, axis, channel) as the host generator
// paper_1511_06441_b200/instances.py grid_values / set_mask, written a second time
// so a rank can generate only its own slab of a 1024^3 cube in HBM instead of
// building (and slicing) 8 GB of host arrays.  No arithmetic of the method here.
//
//   sm(x) = splitmix64 finaliser of (x + 0x9E3779B97F4A7C15)
//   h     = sm(sm(seed) ^ (8 v + 2 k + c)),  c = 0: f1, 1: f2
//   value = lo + ((h >> 32) mod (hi - lo + 1)),  0 where x_k = n_k - 1 (edge absent)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace wcspk {

__host__ __device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct GenShape {
  int d;
  long long n[4];
  long long plane;   // product of all axes but the last
  long long v0;      // global index of the first generated vertex (z0 * plane)
  long long Nl;      // generated vertices ((z1 - z0) * plane)
};

// f1/f2 of the planes [z0, z1): out[k * Nl + i] for local vertex i = global v0 + i
__global__ void __launch_bounds__(256) k_gen_grid(GenShape g, unsigned long long s0, unsigned lo, unsigned span,
                                                 uint8_t* f1, uint8_t* f2) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.Nl; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long v = (unsigned long long)(g.v0 + i);
    unsigned long long stride = 1;
    for (int k = 0; k < g.d; ++k) {
      const long long xk = (long long)((v / stride) % (unsigned long long)g.n[k]);
      uint8_t a = 0, b = 0;
      if (xk != g.n[k] - 1) {
        const unsigned long long key = 8ull * v + 2ull * (unsigned long long)k;
        a = (uint8_t)(lo + (unsigned)((splitmix64(s0 ^ key) >> 32) % span));
        b = (uint8_t)(lo + (unsigned)((splitmix64(s0 ^ (key + 1ull)) >> 32) % span));
      }
      f1[(size_t)k * g.Nl + i] = a;
      f2[(size_t)k * g.Nl + i] = b;
      stride *= (unsigned long long)g.n[k];
    }
  }
}

// vertex sets of instances.set_mask: 0 face x0 = 0, 1 face x0 = n0 - 1, 2 boundary (any x_k
// extreme, the §6 protocol), 3 centre (floor(n/2) per axis), 4 corner v = 0, 5 corner v = N - 1
__global__ void __launch_bounds__(256) k_gen_mask(GenShape g, int rule, uint8_t* out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.Nl; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long v = (unsigned long long)(g.v0 + i);
    unsigned long long stride = 1;
    bool inb = false, centre = true, c0 = true, c1 = true;
    long long x0 = 0;
    for (int k = 0; k < g.d; ++k) {
      const long long xk = (long long)((v / stride) % (unsigned long long)g.n[k]);
      if (k == 0) x0 = xk;
      inb |= xk == 0 || xk == g.n[k] - 1;
      centre &= xk == g.n[k] / 2;
      c0 &= xk == 0;
      c1 &= xk == g.n[k] - 1;
      stride *= (unsigned long long)g.n[k];
    }
    bool m = false;
    switch (rule) {
      case 0: m = x0 == 0; break;
      case 1: m = x0 == g.n[0] - 1; break;
      case 2: m = inb; break;
      case 3: m = centre; break;
      case 4: m = c0; break;
      default: m = c1; break;
    }
    out[i] = m ? 1 : 0;
  }
}

}  // namespace wcspk
