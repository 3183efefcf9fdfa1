// fht_common.cuh -- shared device helpers for the sm_100a FHT kernels.
//
// Notation: a quadrant transform runs on a "frame": Hp = 2^K rows (FHT rows),
// content width wc, cyclic width W = wc + Hp, sign sigma (R4). Computation is done in
// SIGNED (unwrapped) columns: the cyclic cell x0 of a sigma=+1 quadrant is the signed start
// x0 (x0 < wc) or x0 - W (x0 >= wc); for sigma=-1 it is x0 itself (R6). Pixels outside
// [0, wc) are zero, so no modular arithmetic is needed inside the butterflies.
//
// The 2^K-row transform is split into two passes by the pre-shear identity:
//   pass 1: levels 1..m on strips of 2^m rows          -> F_m[i][j](x)   (scratch)
//   pass 2: group j = FHT_{2^L}( i -> F_m[i][j](x + sigma*j*i) ),  t = j*2^L + u
// Both passes run the same in-tile butterfly (north_star "out[t] = A[t>>1] + B[t>>1] shifted
// by ceil(t/2)"; Fig. 6).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Bounds-checked debug build (-DFHT_CHECKS=1; tools/checks_build.sh): every shared-memory access of the
// tile bodies, every plain global store and every TMA store coordinate is checked, a violation prints
// and traps. compute-sanitizer is closed on this pool; this build run over the GPU suite stands in.
#ifndef FHT_CHECKS
#define FHT_CHECKS 0
#endif
#if FHT_CHECKS
#include <cstdio>
#define FHT_CHECK(c)                                                                              \
  do {                                                                                            \
    if (!(c)) {                                                                                   \
      printf("FHT_CHECK failed %s:%d (block %d thread %d): %s\n", __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x, #c);                                                               \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define FHT_CHECK(c) \
  do {               \
  } while (0)
#endif

namespace fht {

// shared-memory access of `bytes` at generic pointer p lies inside the CTA's shared memory
__device__ __forceinline__ bool smem_in_bounds(const void* p, int bytes) {
  unsigned total;
  asm volatile("mov.u32 %0, %%total_smem_size;" : "=r"(total));
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  return a + (unsigned)bytes <= total;
}

constexpr int kMaxLog = 6;  // one pass handles <= 6 levels (64-row tiles); Hp <= 4096 in 2 passes

__host__ __device__ __forceinline__ int ceil_half(int v) { return (v + 1) >> 1; }

// Dyadic pattern offset D_{2^K, s}(y) by the bit closed form (SURVEY method summary):
// D(y) = sum_q bit_{K-1-q}(y) * ceil((s >> q) / 2). Used only for the §4/§5 range geometry.
__host__ __device__ __forceinline__ int dyadic_offset(int K, int s, int y) {
  int d = 0;
  for (int q = 0; q < K; ++q) d += ((y >> (K - 1 - q)) & 1) * (((s >> q) + 1) >> 1);
  return d;
}

template <typename T> struct AccOf;
template <> struct AccOf<uint8_t> { using type = int; };
template <> struct AccOf<int32_t> { using type = int; };
template <> struct AccOf<float> { using type = float; };

}  // namespace fht
