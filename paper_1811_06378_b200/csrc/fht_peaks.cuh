// fht_peaks.cuh -- top-k peaks of Hough planes (R25).
//
// A cell (r, c) of a plane [R][W] is a peak when it beats each of its up to 8 neighbours --
// columns cyclic (x0 is taken mod W), rows not -- where a beats b iff v(a) > v(b), or
// v(a) == v(b) and a comes first in row-major order. The k <= 32 peaks with the largest value
// (ties: smaller row-major index first) are returned per plane.
//
// Keys: (orderable value bits << 32) | (0xFFFFFFFF - index): a larger key is a better peak, 0 is
// "empty". Every warp keeps a descending list of 32 keys, one per lane.
//   k_peaks_band: one CTA per (band of rows, plane); each warp walks 32-column strips down the
//     band, keeping the centre values of rows r-1, r, r+1 in registers. Only lanes whose value
//     reaches the list's minimum load the 6 side neighbours and run the full test (after the list
//     fills this is rare), so the pass is a streaming read of the plane. The 8 warp lists are
//     merged in shared memory; the CTA writes its 32 keys.
//   k_peaks_merge: one warp per plane merges the bands' lists and decodes (value, row, col).
#pragma once
#include <cstdint>

namespace fht {
namespace pk {

constexpr int kMaxK = 32;
constexpr int kWarps = 8;
constexpr int kRowsInFlight = 8;  // rows a warp loads ahead of its test

__device__ __forceinline__ uint32_t ord_bits(float v) {
  const uint32_t u = __float_as_uint(v + 0.0f);  // -0 -> +0: equal values get equal keys
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint32_t ord_bits(int v) { return static_cast<uint32_t>(v) ^ 0x80000000u; }
__device__ __forceinline__ float unord(uint32_t o, float) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
__device__ __forceinline__ int unord(uint32_t o, int) { return static_cast<int>(o ^ 0x80000000u); }

// insert `cand` into the warp's descending list (one key per lane); cand must beat the minimum
__device__ __forceinline__ void list_insert(uint64_t& list, uint64_t cand, int lane) {
  const int pos = __popc(__ballot_sync(0xffffffffu, list > cand));
  const uint64_t up = __shfl_up_sync(0xffffffffu, list, 1);
  if (lane == pos) list = cand;
  else if (lane > pos) list = up;
}

// every lane offers `key` (0 = nothing); keys beating both the list minimum and `floor` (a key
// known to have 32 better peaks in the plane) are inserted
__device__ __forceinline__ void list_offer(uint64_t& list, uint64_t& lmin, uint64_t key, int lane,
                                           uint64_t floor = 0) {
  unsigned m = __ballot_sync(0xffffffffu, key > lmin && key > floor);
  while (m) {
    const int src = __ffs(m) - 1;
    const uint64_t cand = __shfl_sync(0xffffffffu, key, src);
    list_insert(list, cand, lane);
    lmin = __shfl_sync(0xffffffffu, list, 31);
    m &= ~(1u << src);
    m &= __ballot_sync(0xffffffffu, key > lmin);
  }
}

struct PeakArgs {
  const void* data;
  int64_t bstride, qstride, rstride;  // elements
  int nquad, R, W;
  int band, nbands;
  uint64_t* part;                     // [planes][nbands][32]
  unsigned long long* thr;            // [planes]: the largest full-list minimum any warp has seen (0 first)
  void* values;                       // [planes][k]
  int32_t* rows;                      // [planes][k]
  int32_t* cols;                      // [planes][k]
  int k, planes;
};

template <typename A>
__global__ void __launch_bounds__(kWarps * 32) k_peaks_band(const PeakArgs a) {
  __shared__ uint64_t lists[kWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int plane = blockIdx.y;
  const A* base = static_cast<const A*>(a.data) + (int64_t)(plane / a.nquad) * a.bstride +
                  (int64_t)(plane % a.nquad) * a.qstride;
  const int R = a.R, W = a.W;
  const int r0 = blockIdx.x * a.band, r1 = min(R, r0 + a.band);
  uint64_t list = 0, lmin = 0, published = 0;
  // a warp whose list is full proves 32 peaks >= its minimum: that key bounds the whole plane
  unsigned long long* gthr = a.thr + plane;
  for (int c0 = warp * 32; c0 < W; c0 += kWarps * 32) {
    const int c = c0 + lane;
    const bool valid = c < W;
    const int cl = c == 0 ? W - 1 : c - 1, cr = c + 1 >= W ? 0 : c + 1;
    bool hp = r0 > 0;
    A vp = (hp && valid) ? __ldg(base + (int64_t)(r0 - 1) * a.rstride + c) : A(0);
    A vc = valid ? __ldg(base + (int64_t)r0 * a.rstride + c) : A(0);
    for (int rb = r0; rb < r1; rb += kRowsInFlight) {
      const uint64_t floor = max(lmin, (uint64_t)__ldcg(gthr));
      // rows rb+1 .. rb+8 in flight together (one row at a time left the walk latency-bound)
      A nx[kRowsInFlight];
#pragma unroll
      for (int u = 0; u < kRowsInFlight; ++u) {
        const int rr = rb + 1 + u;
        nx[u] = (valid && rr < R && rr <= r1) ? __ldg(base + (int64_t)rr * a.rstride + c) : A(0);
      }
#pragma unroll
      for (int u = 0; u < kRowsInFlight; ++u) {
      const int r = rb + u;
      if (r >= r1) break;
      const bool hn = r + 1 < R;
      const A vn = nx[u];
      const bool cand = valid && ord_bits(vc) >= (uint32_t)(max(lmin, floor) >> 32);
      if (__any_sync(0xffffffffu, cand)) {
        uint64_t key = 0;
        if (cand) {
          const A* rowc = base + (int64_t)r * a.rstride;
          bool peak = true;
          if (W > 1) {  // same row: the left neighbour is earlier unless it wraps, the right later unless it wraps
            const A l = __ldg(rowc + cl), rt = __ldg(rowc + cr);
            peak = (c == 0 ? !(l > vc) : !(l >= vc)) && (c == W - 1 ? !(rt >= vc) : !(rt > vc));
          }
          if (peak && hp) {  // row above: every neighbour is earlier
            const A* rp = rowc - a.rstride;
            peak = !(vp >= vc) && !(__ldg(rp + cl) >= vc) && !(__ldg(rp + cr) >= vc);
          }
          if (peak && hn) {  // row below: every neighbour is later
            const A* rn = rowc + a.rstride;
            peak = !(vn > vc) && !(__ldg(rn + cl) > vc) && !(__ldg(rn + cr) > vc);
          }
          if (peak) key = ((uint64_t)ord_bits(vc) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)(r * W + c));
        }
        list_offer(list, lmin, key, lane, floor);
      }
      vp = vc;
      vc = vn;
      hp = true;
      }
      if (lane == 0 && lmin > published) {  // lmin != 0 only once the list is full
        atomicMax(gthr, (unsigned long long)lmin);
        published = lmin;
      }
    }
  }
  lists[warp][lane] = list;
  __syncthreads();
  if (warp == 0) {
    for (int w2 = 1; w2 < kWarps; ++w2) list_offer(list, lmin, lists[w2][lane], lane);
    a.part[((int64_t)plane * a.nbands + blockIdx.x) * 32 + lane] = list;
  }
}

template <typename A> struct V4Of;
template <> struct V4Of<float> { using type = float4; };
template <> struct V4Of<int> { using type = int4; };
template <typename V> __device__ __forceinline__ auto vget(const V& v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}

// 16-byte variant (W, the strides and the base a multiple of 4 elements): lane l holds columns
// c0 + 4l .. c0 + 4l + 3 of a 128-column strip, so the per-row filter, ballot and loop overhead
// is paid once per 4 cells; neighbours inside the lane come from registers.
template <typename A>
__global__ void __launch_bounds__(kWarps * 32) k_peaks_band4(const PeakArgs a) {
  using V = typename V4Of<A>::type;
  __shared__ uint64_t lists[kWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int plane = blockIdx.y;
  const A* base = static_cast<const A*>(a.data) + (int64_t)(plane / a.nquad) * a.bstride +
                  (int64_t)(plane % a.nquad) * a.qstride;
  const int R = a.R, W = a.W;
  const int r0 = blockIdx.x * a.band, r1 = min(R, r0 + a.band);
  uint64_t list = 0, lmin = 0, published = 0;
  unsigned long long* gthr = a.thr + plane;
  for (int c0 = warp * 128; c0 < W; c0 += kWarps * 128) {
    const int cb = c0 + 4 * lane;  // first column of the lane
    const bool valid = cb < W;     // W % 4 == 0: all four or none
    auto ldv = [&](int r) -> V { return *reinterpret_cast<const V*>(base + (int64_t)r * a.rstride + cb); };
    bool hp = r0 > 0;
    V vp = (hp && valid) ? ldv(r0 - 1) : V{};
    V vc = valid ? ldv(r0) : V{};
    for (int rb = r0; rb < r1; rb += kRowsInFlight) {
      const uint64_t floor = max(lmin, (uint64_t)__ldcg(gthr));
      V nx[kRowsInFlight];
#pragma unroll
      for (int u = 0; u < kRowsInFlight; ++u) {
        const int rr = rb + 1 + u;
        nx[u] = (valid && rr < R && rr <= r1) ? ldv(rr) : V{};
      }
#pragma unroll
      for (int u = 0; u < kRowsInFlight; ++u) {
        const int r = rb + u;
        if (r >= r1) break;
        const bool hn = r + 1 < R;
        const V vn = nx[u];
        const uint32_t th = (uint32_t)(max(lmin, floor) >> 32);
        unsigned cm = 0;  // candidate columns of the lane
        if (valid) {
#pragma unroll
          for (int j = 0; j < 4; ++j) cm |= (ord_bits(vget(vc, j)) >= th) ? (1u << j) : 0u;
        }
        if (__any_sync(0xffffffffu, cm != 0)) {
          const A* rowc = base + (int64_t)r * a.rstride;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint64_t key = 0;
            if (cm & (1u << j)) {
              const int c = cb + j;
              const A v = vget(vc, j);
              const int cl = c == 0 ? W - 1 : c - 1, cr = c + 1 >= W ? 0 : c + 1;
              // same row (W >= 4 here): left earlier unless it wraps, right later unless it wraps
              const A l = j > 0 ? vget(vc, j - 1) : __ldg(rowc + cl);
              const A rt = j < 3 ? vget(vc, j + 1) : __ldg(rowc + cr);
              bool peak = (c == 0 ? !(l > v) : !(l >= v)) && (c == W - 1 ? !(rt >= v) : !(rt > v));
              if (peak && hp) {
                const A* rp = rowc - a.rstride;
                const A pl = j > 0 ? vget(vp, j - 1) : __ldg(rp + cl);
                const A pr = j < 3 ? vget(vp, j + 1) : __ldg(rp + cr);
                peak = !(vget(vp, j) >= v) && !(pl >= v) && !(pr >= v);
              }
              if (peak && hn) {
                const A* rn = rowc + a.rstride;
                const A nl = j > 0 ? vget(vn, j - 1) : __ldg(rn + cl);
                const A nr = j < 3 ? vget(vn, j + 1) : __ldg(rn + cr);
                peak = !(vget(vn, j) > v) && !(nl > v) && !(nr > v);
              }
              if (peak) key = ((uint64_t)ord_bits(v) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)(r * W + c));
            }
            list_offer(list, lmin, key, lane, floor);
          }
        }
        vp = vc;
        vc = vn;
        hp = true;
      }
      if (lane == 0 && lmin > published) {
        atomicMax(gthr, (unsigned long long)lmin);
        published = lmin;
      }
    }
  }
  lists[warp][lane] = list;
  __syncthreads();
  if (warp == 0) {
    for (int w2 = 1; w2 < kWarps; ++w2) list_offer(list, lmin, lists[w2][lane], lane);
    a.part[((int64_t)plane * a.nbands + blockIdx.x) * 32 + lane] = list;
  }
}

template <typename A>
__global__ void __launch_bounds__(kWarps * 32) k_peaks_merge(const PeakArgs a) {
  const int lane = threadIdx.x & 31;
  const int plane = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (plane >= a.planes) return;
  uint64_t list = 0, lmin = 0;
  const uint64_t* p = a.part + (int64_t)plane * a.nbands * 32;
  for (int b = 0; b < a.nbands; ++b) list_offer(list, lmin, __ldg(p + b * 32 + lane), lane);
  if (lane < a.k) {
    const int64_t o = (int64_t)plane * a.k + lane;
    A v = A(0);
    int32_t r = -1, c = -1;
    if (list != 0) {
      const uint32_t idx = 0xFFFFFFFFu - (uint32_t)list;
      r = (int32_t)(idx / (uint32_t)a.W);
      c = (int32_t)(idx % (uint32_t)a.W);
      v = unord((uint32_t)(list >> 32), A(0));
    }
    static_cast<A*>(a.values)[o] = v;
    a.rows[o] = r;
    a.cols[o] = c;
  }
}

}  // namespace pk
}  // namespace fht
