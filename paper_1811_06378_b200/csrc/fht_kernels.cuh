// fht_kernels.cuh -- sm_100a kernels of the FHT hot path.
//
//   k_pass1   : SURVEY a3 -- levels 1..m of a 2^m-row strip, loaded once from the image
//               (row or transposed loads = quadrant handling by index transposition, a1),
//               optional §4 shear+scale loader (a6). Writes F_m to scratch.
//   k_pass2   : SURVEY a4 -- levels m+1..K of one group j through the pre-shear identity,
//               black-zone tiles written as zeros without loads, store addressing for the
//               QUADS / CONCAT layouts (a5) and an optional fused fhtshift (§5).
//   k_fhtshift: SURVEY a7 -- standalone per-row cyclic rotation.
//   k_range_tables : §4 per-row shear offsets e_y, scale map colmap[u] and per-row support.
#pragma once
#include "fht_common.cuh"

namespace fht {

constexpr int kThreads = 256;
constexpr int kTileX = 128;  // output columns per tile (both passes)

// ------------------------------------------------------------------------------------------
// In-tile butterfly (north_star; Fig. 6). Rows 0..R-1 of `src` hold R input
// rows; local column c holds signed x = X + c (sigma=+1) or X + TX-1-c (sigma=-1), so the
// shifted partner is always at c + ceil(t/2) ("halo" columns [TX, TX+R-1) on the right).
// After level k the block of 2^k rows starting at row r0 holds shifts t = 0..2^k-1:
//   dst[r0 + t][c] = src[r0 + (t>>1)][c] + src[r0 + 2^(k-1) + (t>>1)][c + ceil(t/2)].
// Returns the buffer holding the final R rows (shift u in row u).
// ------------------------------------------------------------------------------------------
template <int LOGR, typename A>
__device__ __forceinline__ A* tile_levels(A* src, A* dst, int pitch, int TX) {
  constexpr int R = 1 << LOGR;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll 1
  for (int k = 1; k <= LOGR; ++k) {
    const int half = 1 << (k - 1);
    const int valid = TX + R - (1 << k);  // columns still needed by the levels above
    for (int row = warp; row < R; row += nw) {
      const int t = row & ((1 << k) - 1);
      const int a = (row - t) + (t >> 1);
      const A* pa = src + a * pitch;
      const A* pb = src + (a + half) * pitch + ((t + 1) >> 1);
      A* pd = dst + row * pitch;
      for (int c = lane; c < valid; c += 32) pd[c] = pa[c] + pb[c];
    }
    __syncthreads();
    A* tmp = src;
    src = dst;
    dst = tmp;
  }
  return src;
}

__host__ __device__ constexpr int tile_pitch(int R) { return (kTileX + R - 1) | 1; }

// ------------------------------------------------------------------------------------------
// Pass 1
// ------------------------------------------------------------------------------------------
struct Pass1Args {
  const void* img;
  int64_t img_bstride, img_rstride;  // elements
  int img_rows, img_cols;            // FRAME coordinates: FHT rows / cols that hold pixels
  int transposed;                    // FHT row y = image column, FHT col x = image row
  void* scratch;                     // [z][2^m][2^L][Ws]
  int64_t scratch_zstride;
  int L;                             // log2(#strips)
  int Ws;                            // scratch row length
  int xlo[2];                        // signed x of scratch column 0, per quadrant slot
  int sigma[2];
  int nq;                            // quadrants per image in this launch (1 or 2)
  int img0;                          // first image of the chunk
  // §4 range loader (sigma = +1 only)
  int range;
  const int* e_tab;                  // [rows] shear offsets e_y
  const int* colmap;                 // [w_content]
  int w_content;
};

template <typename Tin>
__device__ __forceinline__ typename AccOf<Tin>::type load_px(const Tin* p) {
  return static_cast<typename AccOf<Tin>::type>(*p);
}

template <typename Tin, int LOGR>
__global__ void __launch_bounds__(kThreads) k_pass1(const Pass1Args a) {
  using A = typename AccOf<Tin>::type;
  constexpr int R = 1 << LOGR;
  constexpr int TX = kTileX;
  constexpr int WT = TX + R - 1;
  constexpr int pitch = tile_pitch(R);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* b0 = reinterpret_cast<A*>(smem_raw);
  A* b1 = b0 + R * pitch;

  const int z = blockIdx.z;
  const int qi = z % a.nq;
  const int img = a.img0 + z / a.nq;
  const int sigma = a.sigma[qi];
  const int strip = blockIdx.y;
  const int X = a.xlo[qi] + blockIdx.x * TX;
  const Tin* src = static_cast<const Tin*>(a.img) + (int64_t)img * a.img_bstride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;

  if (!a.transposed) {
    for (int r = warp; r < R; r += nw) {
      const int y = strip * R + r;
      const bool row_ok = y < a.img_rows;
      const Tin* prow = src + (int64_t)y * a.img_rstride;
      int e = 0;
      if (a.range && row_ok) e = a.e_tab[y];
      for (int c = lane; c < WT; c += 32) {
        const int x = sigma > 0 ? X + c : X + TX - 1 - c;
        A v = A(0);
        if (row_ok) {
          if (!a.range) {
            if (x >= 0 && x < a.img_cols) v = load_px(prow + x);
          } else {  // T(x, y) = I[y][colmap[x - e_y]] (unwrapped; R13, R14)
            const int u = x - e;
            if (u >= 0 && u < a.w_content) v = load_px(prow + a.colmap[u]);
          }
        }
        b0[r * pitch + c] = v;
      }
    }
  } else {
    // FHT row y = image column y, FHT column x = image row x: lanes run along image columns
    // (coalesced), smem pitch is odd so the column-wise smem writes are conflict-free.
    for (int c = warp; c < WT; c += nw) {
      const int x = sigma > 0 ? X + c : X + TX - 1 - c;
      const bool ok = x >= 0 && x < a.img_cols;
      const Tin* prow = src + (int64_t)x * a.img_rstride;
      for (int r = lane; r < R; r += 32) {
        const int y = strip * R + r;
        A v = A(0);
        if (ok && y < a.img_rows) v = load_px(prow + y);
        b0[r * pitch + c] = v;
      }
    }
  }
  __syncthreads();
  A* res = tile_levels<LOGR, A>(b0, b1, pitch, TX);

  A* dst = static_cast<A*>(a.scratch) + (int64_t)z * a.scratch_zstride;
  const int nstrips = 1 << a.L;
  for (int t = warp; t < R; t += nw) {
    A* drow = dst + ((int64_t)t * nstrips + strip) * a.Ws;
    for (int c = lane; c < TX; c += 32) {
      const int x = sigma > 0 ? X + c : X + TX - 1 - c;
      const int col = x - a.xlo[qi];
      if (col >= 0 && col < a.Ws) drow[col] = res[t * pitch + c];
    }
  }
}

// ------------------------------------------------------------------------------------------
// Pass 2
// ------------------------------------------------------------------------------------------
struct Pass2Args {
  const void* scratch;
  int64_t scratch_zstride;
  int Ws;
  int xlo[2];
  int sigma[2];
  int m, L;
  void* out;
  int64_t out_img_stride, out_row_stride;
  int64_t out_q_offset[2];  // element offset of the quadrant's row-0 base inside an image
  int row_base[2], row_sign[2], skip_t[2];  // output row = base + sign*t; t == skip not stored
  int W, wc, Hp;
  int xbeg[2];              // signed x of the first output column computed
  int nq, img0;
  int shift;                // fused fhtshift: 1 = quadrant rule, 2 = range rule
  int range;
  const int* start_tab;     // range: per-row unwrapped support start
  const int* len_tab;       // range: per-row support length
};

template <typename A, int LOGR>
__global__ void __launch_bounds__(kThreads) k_pass2(const Pass2Args a) {
  constexpr int R = 1 << LOGR;
  constexpr int TX = kTileX;
  constexpr int WT = TX + R - 1;
  constexpr int pitch = tile_pitch(R);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* b0 = reinterpret_cast<A*>(smem_raw);
  A* b1 = b0 + R * pitch;

  const int z = blockIdx.z;
  const int qi = z % a.nq;
  const int img = a.img0 + z / a.nq;
  const int sigma = a.sigma[qi];
  const int j = blockIdx.y;
  const int X = a.xbeg[qi] + blockIdx.x * TX;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int t0 = j << a.L;
  const int tmax = t0 + R - 1;

  A* outp = static_cast<A*>(a.out) + (int64_t)img * a.out_img_stride + a.out_q_offset[qi];

  bool zero_tile = false;
  if (!a.range) {  // black zone: sigma=+1 cells x < -t, sigma=-1 cells x >= wc + t
    zero_tile = sigma > 0 ? (X + TX - 1 < -tmax) : (X >= a.wc + tmax);
  }
  A* res = nullptr;
  if (!zero_tile) {
    const A* src = static_cast<const A*>(a.scratch) + (int64_t)z * a.scratch_zstride +
                   (int64_t)(j << a.L) * a.Ws;
    for (int i = warp; i < R; i += nw) {
      const A* srow = src + (int64_t)i * a.Ws;
      const int off = sigma * j * i - a.xlo[qi];  // pre-shear by sigma*j*i
      for (int c = lane; c < WT; c += 32) {
        const int x = sigma > 0 ? X + c : X + TX - 1 - c;
        const int col = x + off;
        b0[i * pitch + c] = (col >= 0 && col < a.Ws) ? srow[col] : A(0);
      }
    }
    __syncthreads();
    res = tile_levels<LOGR, A>(b0, b1, pitch, TX);
  }

  for (int u = warp; u < R; u += nw) {
    const int t = t0 + u;
    if (t == a.skip_t[qi]) continue;
    A* orow = outp + (int64_t)(a.row_base[qi] + a.row_sign[qi] * t) * a.out_row_stride;
    int lo, hi, k = 0;
    if (!a.range) {
      lo = a.xbeg[qi];
      hi = lo + a.W;
      if (a.shift) k = sigma > 0 ? ceil_half(a.W - a.wc + t) : ceil_half(a.W - a.wc - t);  // R11, pad = W - wc
    } else {
      lo = a.start_tab[t];
      hi = lo + a.W;
      if (a.shift) k = ceil_half(a.W - a.len_tab[t]) - lo;
    }
    for (int c = lane; c < TX; c += 32) {
      const int x = sigma > 0 ? X + c : X + TX - 1 - c;
      if (x < lo || x >= hi) continue;
      int x0 = x % a.W;
      if (x0 < 0) x0 += a.W;
      if (k) {
        x0 = (x0 + k) % a.W;
        if (x0 < 0) x0 += a.W;
      }
      orow[x0] = zero_tile ? A(0) : res[u * pitch + c];
    }
  }
}

// ------------------------------------------------------------------------------------------
// §4 tables: e_y (rows), colmap (w_content), per-row support start/len (Hp rows).
// Double arithmetic with explicit round-to-nearest intrinsics (no FMA contraction, R16).
// ------------------------------------------------------------------------------------------
struct RangeTableArgs {
  double g, alpha;
  int h, w, w_content, Hp, K;
  int* e_tab;     // [h]
  int* colmap;    // [w_content]
  int* start_tab; // [Hp]
  int* len_tab;   // [Hp]
};

__device__ __forceinline__ int shear_e(double g, int y) {
  return (int)floor(__dadd_rn(__dmul_rn(g, (double)y), 0.5));
}

// Per output row s of the range frame: start_s = min_y (e_y - D_s(y)), len_s = max - min + w'
// (R17). D_s(y) = sum over the set bits b of y of ceil((s >> (K-1-b)) / 2) (the closed form of
// dyadic_offset) is additive over the bits. One warp per row: with y = 32k + lane the low 5 bits
// are the lane (a per-lane constant) and the high bits are k (the same for the whole warp, from a
// per-warp 128-entry table). The shear offsets e_y are computed once per block (shared memory).
// Blocks [0, nsb) do kRangeRowsPerBlock rows with 8 warps; the remaining blocks write e_tab, colmap.
#ifndef FHT_RANGE_ROWS_PER_BLOCK
#define FHT_RANGE_ROWS_PER_BLOCK 8
#endif
constexpr int kRangeRowsPerBlock = FHT_RANGE_ROWS_PER_BLOCK;  // one row per warp: 512 blocks for Hp = 4096

// min / max over y < h of e_y - D_s(y) for row s, by one warp (every lane gets the result). e_s: the
// block's shared e_y table; dh: the warp's 128-entry scratch (reused: ends with __syncwarp).
__device__ __forceinline__ void row_support_warp(int K, int h, int s, const int* e_s, int* dh, int lane, int& mn,
                                                 int& mx) {
  auto wbit = [&](int bit) { return bit < K ? ((s >> (K - 1 - bit)) + 1) >> 1 : 0; };
  int dl = 0;  // bits 0..4 of y = lane
  for (int b = 0; b < 5; ++b)
    if ((lane >> b) & 1) dl += wbit(b);
  for (int k = lane; k < 128; k += 32) {  // bits 5..11 of y = k
    int d = 0;
    for (int b = 0; b < 7; ++b)
      if ((k >> b) & 1) d += wbit(5 + b);
    dh[k] = d;
  }
  __syncwarp();
  mn = INT32_MAX;
  mx = INT32_MIN;
  for (int k = 0; 32 * k < h; ++k) {
    const int y = 32 * k + lane;
    if (y < h) {
      const int v = e_s[y] - dl - dh[k];
      mn = min(mn, v);
      mx = max(mx, v);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __syncwarp();  // dh reused by the warp's next row
}
__global__ void k_range_tables(const RangeTableArgs a) {
  extern __shared__ int e_s[];          // [h]
  __shared__ int dh_s[8][128];          // per warp: D of the high bits, y >> 5
  const int nsb = (a.Hp + kRangeRowsPerBlock - 1) / kRangeRowsPerBlock;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if ((int)blockIdx.x < nsb) {
    for (int y = threadIdx.x; y < a.h; y += blockDim.x) e_s[y] = shear_e(a.g, y);
    __syncthreads();
    const int s_end = min(a.Hp, ((int)blockIdx.x + 1) * kRangeRowsPerBlock);
    int* dh = dh_s[warp];
    for (int s = blockIdx.x * kRangeRowsPerBlock + warp; s < s_end; s += nw) {
      int mn, mx;
      row_support_warp(a.K, a.h, s, e_s, dh, lane, mn, mx);
      if (lane == 0) {
        a.start_tab[s] = mn;
        a.len_tab[s] = mx - mn + a.w_content;
      }
    }
    return;
  }
  // remaining blocks: e_y and colmap
  const int idx = ((int)blockIdx.x - nsb) * blockDim.x + threadIdx.x;
  if (idx < a.h) a.e_tab[idx] = shear_e(a.g, idx);
  if (idx < a.w_content) {
    const int c = (int)floor(__ddiv_rn((double)idx + 0.5, a.alpha));
    a.colmap[idx] = min(a.w - 1, c);
  }
}

// The same tables with the per-row supports by the FHT's own block recursion, (min, max) in place of + (the host
// plan's method, fht_angle_plan): D_t of a 2^k-row block is D_{t>>1} on its top half and ceil(t/2) + D_{t>>1} on its
// bottom half, so
//   mn_k[b][t] = min(mn_{k-1}[2b][t>>1], mn_{k-1}[2b+1][t>>1] - ceil(t/2))      (mx likewise, padding rows neutral):
// Hp log2 Hp steps in block 0's shared memory ([4][Hp] ints) instead of Hp * h terms over 512 blocks (C4: 17.5 us
// of a 255 us step). The other blocks write e_tab and colmap.
constexpr int kRangeRecThreads = 512;
__global__ void __launch_bounds__(kRangeRecThreads) k_range_tables_rec(const RangeTableArgs a) {
  extern __shared__ int rec_s[];  // mn, mx, mn2, mx2: [Hp] each
  if (blockIdx.x > 0) {
    const int idx = ((int)blockIdx.x - 1) * blockDim.x + threadIdx.x;
    if (idx < a.h) a.e_tab[idx] = shear_e(a.g, idx);
    if (idx < a.w_content) {
      const int c = (int)floor(__ddiv_rn((double)idx + 0.5, a.alpha));
      a.colmap[idx] = min(a.w - 1, c);
    }
    return;
  }
  constexpr int kInf = 1 << 29;  // neutral element (padding rows); |e_y|, D < 2^28 keep it apart
  int *mn = rec_s, *mx = rec_s + a.Hp, *mn2 = rec_s + 2 * a.Hp, *mx2 = rec_s + 3 * a.Hp;
  for (int y = threadIdx.x; y < a.Hp; y += blockDim.x) {
    const int e = y < a.h ? shear_e(a.g, y) : 0;
    mn[y] = y < a.h ? e : kInf;
    mx[y] = y < a.h ? e : -kInf;
  }
  __syncthreads();
  for (int half = 1; half < a.Hp; half <<= 1) {  // level: blocks of 2 * half rows, shifts t < 2 * half
    for (int idx = threadIdx.x; idx < a.Hp; idx += blockDim.x) {
      const int t = idx & (2 * half - 1), top = (idx - t) + (t >> 1), bot = top + half;
      const int c = (t + 1) >> 1;
      mn2[idx] = min(mn[top], mn[bot] - c);
      mx2[idx] = max(mx[top], mx[bot] - c);
    }
    __syncthreads();
    int* tmp = mn; mn = mn2; mn2 = tmp;
    tmp = mx; mx = mx2; mx2 = tmp;
  }
  for (int s = threadIdx.x; s < a.Hp; s += blockDim.x) {
    a.start_tab[s] = mn[s];
    a.len_tab[s] = mx[s] - mn[s] + a.w_content;
  }
}

// ------------------------------------------------------------------------------------------
// Standalone fhtshift (R11): out[r][x] = in[r][(x - k_r) mod W].
// ------------------------------------------------------------------------------------------
struct ShiftArgs {
  const void* in;
  void* out;
  int64_t in_img_stride, in_q_stride, in_row_stride;
  int64_t out_img_stride, out_q_stride, out_row_stride;
  int rows, W, nquad;
  int64_t rows_total;   // batch * nquad * rows
  int mode, layout;     // fht_mode / fht_layout
  int quadrant;         // QUADRANT mode
  int Hp, Wp;           // quadrant row counts (QA/QB: Hp, QC/QD: Wp)
  int pad;              // QUADRANT mode: the frame's extension W - w_frame (FULL: pad = the row count)
  int row0;             // FULL/QUADS band of a sharded transform: row r is shift row0 + r
  int vec;              // 16-byte path: W, every stride a multiple of 4 elements, bases 16-B aligned
  double g;             // RANGE: shear e_y = floor(g*y + 0.5), y < h; K = log2 Hp; w' (R17 support)
  int h, K, w_content;
};

__device__ __forceinline__ int quadrant_sigma(int q) { return (q == 0 || q == 3) ? 1 : -1; }

// k(s) of output row r (R11, R17): QUADRANT / FULL (QUADS or CONCAT row attribution,
// P:111-113, R8) by the closed form, RANGE from the per-row support tables.
__device__ __forceinline__ int shift_amount(const ShiftArgs& a, int r, int qs) {
  int q, s;
  if (a.mode == 1 && a.layout == 1) {
    const int Hp = a.Hp, Wp = a.Wp;
    if (r < Hp) { q = 0; s = Hp - 1 - r; }
    else if (r < 2 * Hp - 1) { q = 1; s = r - (Hp - 1); }
    else if (r < 2 * Hp - 2 + Wp) { q = 2; s = Wp - 1 - (r - (2 * Hp - 2)); }
    else { q = 3; s = r - (2 * Hp + Wp - 3); }
  } else {
    q = a.mode == 0 ? a.quadrant : qs;
    s = r + a.row0;
  }
  const int n = (q < 2) ? a.Hp : a.Wp;
  if (s >= n) return 0;
  // R11 generic rule k = ceil((W - len)/2) - start, len = w_frame + s: ceil((pad + s)/2) for sigma=+1
  // (start = -s), ceil((pad - s)/2) for sigma=-1 (start = 0); pad = W - w_frame (full mode: n)
  const int pad = a.mode == 0 ? a.pad : n;
  int k = (quadrant_sigma(q) > 0 ? ceil_half(pad + s) : ceil_half(pad - s)) % a.W;
  return k < 0 ? k + a.W : k;
}

template <typename T> struct Vec4;
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<int> { using type = int4; };

// out = src[4c - k .. 4c - k + 3] from the aligned chunks A = chunk(c - k) and B = the next one
// (row-uniform misalignment O = (-k) mod 4)
template <int O, typename V>
__device__ __forceinline__ V rot_combine(const V& A, const V& B) {
  if constexpr (O == 0) return A;
  else if constexpr (O == 1) return V{A.y, A.z, A.w, B.x};
  else if constexpr (O == 2) return V{A.z, A.w, B.x, B.y};
  else return V{A.w, B.x, B.y, B.z};
}

// One warp rotates one row of W4 16-byte chunks: output chunk c <- source chunks ca, ca + 1
// (mod W4) with ca = (cA0 + c) mod W4. Four chunks per lane in flight before their stores.
template <int O, typename T>
__device__ __forceinline__ void shift_row_vec(const T* src, T* dst, int W4, int cA0, int lane) {
  using V = typename Vec4<T>::type;
  const V* s4 = reinterpret_cast<const V*>(src);
  V* d4 = reinterpret_cast<V*>(dst);
  int ca = cA0 + lane;
  if (ca >= W4) ca -= W4;
  for (int c0 = lane; c0 < W4; c0 += 128) {
    V o[4];
    int cu = ca;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (c0 + 32 * u < W4) {
        const V A = __ldg(s4 + cu);
        V B = A;
        if constexpr (O != 0) B = __ldg(s4 + (cu + 1 == W4 ? 0 : cu + 1));
        o[u] = rot_combine<O>(A, B);
      }
      cu += 32;
      while (cu >= W4) cu -= W4;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c0 + 32 * u < W4) __stcs(d4 + c0 + 32 * u, o[u]);
    ca = cu;
  }
}

// Standalone fhtshift (R11): out[r][x] = in[r][(x - k_r) mod W]. One warp
// per row (8 rows per block); 16-byte loads and streaming stores when everything is aligned.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_fhtshift(const ShiftArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  int k_range = 0;
  if (a.mode == 2) {
    // RANGE (R11 generic rule, R17 support): k = ceil((W' - len)/2) - start, start/len of the row by
    // the §4 table method -- e_y once per block in shared memory, then one warp per row
    extern __shared__ int e_s[];  // [h]
    __shared__ int dh_s[kThreads / 32][128];
    for (int y = threadIdx.x; y < a.h; y += blockDim.x) e_s[y] = shear_e(a.g, y);
    __syncthreads();
    if (row >= a.rows_total) return;
    int mn, mx;
    row_support_warp(a.K, a.h, (int)(row % a.rows), e_s, dh_s[threadIdx.x >> 5], lane, mn, mx);
    k_range = (ceil_half(a.W - (mx - mn + a.w_content)) - mn) % a.W;
    if (k_range < 0) k_range += a.W;
  }
  if (row >= a.rows_total) return;
  const int r = (int)(row % a.rows);
  const int64_t zq = row / a.rows;  // image * nquad + quadrant slot
  const int img = (int)(zq / a.nquad), qs = (int)(zq % a.nquad);
  const int k = a.mode == 2 ? k_range : shift_amount(a, r, qs);
  const T* src = static_cast<const T*>(a.in) + (int64_t)img * a.in_img_stride + (int64_t)qs * a.in_q_stride +
                 (int64_t)r * a.in_row_stride;
  T* dst = static_cast<T*>(a.out) + (int64_t)img * a.out_img_stride + (int64_t)qs * a.out_q_stride +
           (int64_t)r * a.out_row_stride;
  if (a.vec) {
    const int base0 = k == 0 ? 0 : a.W - k;  // source index of output column 0
    const int W4 = a.W >> 2, cA0 = base0 >> 2;
    switch (base0 & 3) {
      case 0: shift_row_vec<0>(src, dst, W4, cA0, lane); break;
      case 1: shift_row_vec<1>(src, dst, W4, cA0, lane); break;
      case 2: shift_row_vec<2>(src, dst, W4, cA0, lane); break;
      default: shift_row_vec<3>(src, dst, W4, cA0, lane); break;
    }
    return;
  }
  for (int x = lane; x < a.W; x += 32) {
    int sx = x - k;
    if (sx < 0) sx += a.W;
    FHT_CHECK(sx >= 0 && sx < a.W);
    __stcs(dst + x, __ldg(src + sx));
  }
}

// ------------------------------------------------------------------------------------------
// Fold for quadrant pads below h_frame - 1 (R22; "mod(w+h)"): the cyclic transform of
// width W = w + pad is the signed transform summed over columns congruent mod W. The signed
// transform comes from the default (pad = Hp) run, whose Wt = w + Hp columns hold every signed
// column of the window [xlo, xlo + Wt) exactly once, at x mod Wt.
// ------------------------------------------------------------------------------------------
struct FoldArgs {
  const void* tmp;
  int64_t tmp_pitch, tmp_batch;  // elements
  void* out;                     // may be NULL
  int64_t out_pitch, out_batch;
  void* outs;                    // fhtshift destination, may be NULL
  int64_t outs_pitch, outs_batch;
  int Hp, W, Wt, xlo, sigma;
  int pad;                       // W - w_frame (the fused fhtshift's R11 rule)
  int64_t total;                 // batch * Hp * W
};

template <typename T>
__global__ void __launch_bounds__(kThreads) k_fold(const FoldArgs a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.total; i += (int64_t)gridDim.x * blockDim.x) {
    const int x0 = (int)(i % a.W);
    const int64_t rs = i / a.W;
    const int s = (int)(rs % a.Hp);
    const int64_t b = rs / a.Hp;
    const T* row = static_cast<const T*>(a.tmp) + b * a.tmp_batch + (int64_t)s * a.tmp_pitch;
    // signed columns x = x0 + m W inside the window, ascending
    int x = x0 + ((a.xlo - x0) > 0 ? ((a.xlo - x0) + a.W - 1) / a.W : -((x0 - a.xlo) / a.W)) * a.W;
    T acc = T(0);
    for (; x < a.xlo + a.Wt; x += a.W) {
      int c = x % a.Wt;
      c += c < 0 ? a.Wt : 0;
      acc += row[c];
    }
    if (a.out) static_cast<T*>(a.out)[b * a.out_batch + (int64_t)s * a.out_pitch + x0] = acc;
    if (a.outs) {
      int k = (a.sigma > 0 ? ceil_half(a.pad + s) : ceil_half(a.pad - s)) % a.W;  // R11 generic rule
      k += k < 0 ? a.W : 0;
      int xs = x0 + k;
      xs -= xs >= a.W ? a.W : 0;
      FHT_CHECK(xs >= 0 && xs < a.W && k >= 0);
      static_cast<T*>(a.outs)[b * a.outs_batch + (int64_t)s * a.outs_pitch + xs] = acc;
    }
  }
}

}  // namespace fht
