// fht_tile.cuh -- v2 sm_100a kernels of the FHT hot path: register-resident warp butterflies
// (DESIGN.md §4 "v2").
//
// The 2^K-row transform is split in two passes by the pre-shear identity:
//   pass 1 (k_p1): levels 1..m of every 2^m-row strip, straight from the image -> F_m[i][j](x)
//   pass 2 (k_p2): group j: G_j[i](x) = F_m[i][j](x + sigma*j*i), levels 1..L over i -> H[j*2^L+u]
// Inside ONE CTA the same identity splits a 2^r-row tile once more (r = a + b):
//   sub-pass A: blocks of 2^a rows, butterflies in registers (warp_fht<a, VA>)
//   sub-pass B: group j' of 2^b rows read at column c + j'*i' from the A results, warp_fht<b, VB>
// so every butterfly level runs on registers with at most a few warp shuffles per row; shared
// memory is touched once per sub-pass (odd per-lane strides VA=9 / VB=7: conflict-free for any
// offset), not once per level as in v1.
//
// Window and local columns: a tile computes the 217 signed columns x = Xw + s, s in [0, 217)
// ("window index" s). The butterflies run in a local frame where the partner sits at +shift for
// both signs: c = s (sigma = +1) or c = 216 - s (sigma = -1, mirrored). Lane l owns local
// columns l*V .. l*V+V-1; lane 31 is a halo lane whose results are discarded, so every shuffle
// partner of lanes 0..30 is inside the warp (needs 2^levels - 1 <= V).
//
// Stores (measured TMA rules on this B200, tools/tma_probe.cu: a bulk tensor store needs a
// 16-byte-aligned, non-negative start column and a 128-byte-aligned shared source; the upper
// tensor bound clips): each output row is staged in shared memory at an offset chosen so that
// its destination starts on a 16-byte boundary, then written by ONE cp.async.bulk.tensor row
// store (SASS UTMASTG). Pass-1 scratch rows are always aligned. Pass-2 rows (x mod W for the
// Hough image, (x + k_t) mod W for the fused fhtshift) use a 212-wide box starting up to 3
// columns left of the tile's 208 columns (the tile computes them anyway); a cyclic-wrap
// remainder or a row-support edge (range mode) is written by a warp with coalesced st.global.
#pragma once
#include <cuda.h>
#include "fht_common.cuh"

namespace fht {
namespace v2 {

constexpr int VA = 9;            // local columns per lane, sub-pass A (odd => conflict-free)
constexpr int VB = 7;            // local columns per lane, sub-pass B (odd => conflict-free)
constexpr int WA = 32 * VA;      // 288 local input columns loaded per tile
constexpr int WC = 31 * VB;      // 217 computed window columns per tile
constexpr int IN_PITCH = WA + 1; // 289: odd pitch, conflict-free column-wise (transposed) fills
constexpr int ST_PITCH = 224;    // staging pitch (elements): 896 B rows, 128-B aligned for TMA
constexpr int TX1 = 216;         // pass-1 tile width (= its TMA box), multiple of 4
constexpr int BOX2 = 212;        // pass-2 TMA box width (multiple of 4)
constexpr int TX2 = BOX2 - 4;    // pass-2 tile stride: 208 columns owned per tile
constexpr int WO2 = 4;           // pass-2 window starts 4 columns left of the tile

template <int R> struct Split;
template <> struct Split<1> { static constexpr int a = 1, b = 0, nw = 4; };
template <> struct Split<2> { static constexpr int a = 2, b = 0, nw = 4; };
template <> struct Split<3> { static constexpr int a = 3, b = 0, nw = 4; };
template <> struct Split<4> { static constexpr int a = 2, b = 2, nw = 4; };
template <> struct Split<5> { static constexpr int a = 3, b = 2, nw = 4; };
template <> struct Split<6> { static constexpr int a = 3, b = 3, nw = 8; };

// Dynamic shared memory: the tile buffer (reused as `ndest` staging planes) + the offset table.
__host__ __device__ constexpr size_t tile_buf_elems(int R, int ndest) {
  return (size_t)(1 << R) * (IN_PITCH > ndest * ST_PITCH ? IN_PITCH : ndest * ST_PITCH);
}
__host__ __device__ constexpr size_t tile_smem_bytes(int R, int ndest) {
  return tile_buf_elems(R, ndest) * 4 + 2 * 64 * 4;
}

// ------------------------------------------------------------------------------------------
// Register butterfly (north_star "out[t] = A[t>>1] + B[t>>1] shifted by ceil(t/2)"
// Fig. 6). v[row][q] = row `row`, local column lane*V + q. After the call row t holds
// shift t of the 2^NB-row block. Partner columns beyond the lane come from lane+1 (shfl_down);
// valid for lanes 0..30 when 2^NB - 1 <= V.
// ------------------------------------------------------------------------------------------
template <int NB, int V, int K, typename A>
struct Level {
  static __device__ __forceinline__ void run(A (&v)[1 << NB][V]) {
    constexpr int HS = 1 << (K - 1);
    static_assert(HS <= V, "shift partner must be within lane+1");
    A nv[1 << NB][V];
#pragma unroll
    for (int r0 = 0; r0 < (1 << NB); r0 += 2 * HS) {
#pragma unroll
      for (int i = 0; i < HS; ++i) {
        A ext[V + HS];  // B row extended to the right: ext[e] = B(col lane*V + e)
#pragma unroll
        for (int e = 0; e < V; ++e) ext[e] = v[r0 + HS + i][e];
#pragma unroll
        for (int e = V; e < V + HS; ++e)
          ext[e] = (e <= V + i) ? __shfl_down_sync(0xffffffffu, v[r0 + HS + i][e - V], 1) : A(0);
#pragma unroll
        for (int q = 0; q < V; ++q) {
          nv[r0 + 2 * i][q] = v[r0 + i][q] + ext[q + i];          // t = 2i,   shift i
          nv[r0 + 2 * i + 1][q] = v[r0 + i][q] + ext[q + i + 1];  // t = 2i+1, shift i+1
        }
      }
    }
#pragma unroll
    for (int r = 0; r < (1 << NB); ++r)
#pragma unroll
      for (int q = 0; q < V; ++q) v[r][q] = nv[r][q];
    Level<NB, V, K + 1, A>::run(v);
  }
};
template <int NB, int V, typename A>
struct Level<NB, V, NB + 1, A> {
  static __device__ __forceinline__ void run(A (&)[1 << NB][V]) {}
};
template <int NB, int V, typename A>
__device__ __forceinline__ void warp_fht(A (&v)[1 << NB][V]) {
  Level<NB, V, 1, A>::run(v);
}

// ------------------------------------------------------------------------------------------
// In-CTA FHT of a 2^R-row tile held in `buf` ([2^R][IN_PITCH], local columns, row rho = input
// row). On return, staging plane d ([2^R][ST_PITCH] at buf + d*2^R*ST_PITCH) holds output row
// tau (= shift tau) with window index s stored at s - soff[d*64 + tau], for 0 <= that < box;
// the proxy fence for the TMA engine is done and the CTA is synchronised.
// ------------------------------------------------------------------------------------------
template <int R, typename A>
__device__ __forceinline__ void tile_fht(A* buf, int sigma, int ndest, const int* soff, int box) {
  using S = Split<R>;
  constexpr int a = S::a, b = S::b, NW = S::nw;
  constexpr int NA = 1 << a, NBk = 1 << b, NR = 1 << R;
  constexpr int TPW = (NA + NW - 1) / NW;  // sub-pass B tasks per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // sub-pass A: block blk = rows blk*2^a .. +2^a-1, in place (row blk*2^a + j' <- F_a[blk][j'])
#pragma unroll 1
  for (int blk = warp; blk < NBk; blk += NW) {
    A v[NA][VA];
    A* p = buf + (blk * NA) * IN_PITCH + lane * VA;
#pragma unroll
    for (int r = 0; r < NA; ++r)
#pragma unroll
      for (int q = 0; q < VA; ++q) v[r][q] = p[r * IN_PITCH + q];
    warp_fht<a, VA>(v);
#pragma unroll
    for (int r = 0; r < NA; ++r)
#pragma unroll
      for (int q = 0; q < VA; ++q) p[r * IN_PITCH + q] = v[r][q];
  }
  __syncthreads();

  // sub-pass B: group jp: G[i'](c) = F_a[i'][jp](c + jp*i')  (pre-shear identity, local frame)
  A w[TPW][NBk][VB];
#pragma unroll
  for (int g = 0; g < TPW; ++g) {
    const int jp = warp + g * NW;
    if (jp < NA) {
#pragma unroll
      for (int i = 0; i < NBk; ++i) {
        const A* src = buf + (i * NA + jp) * IN_PITCH + lane * VB + jp * i;
#pragma unroll
        for (int q = 0; q < VB; ++q) w[g][i][q] = src[q];
      }
      warp_fht<b, VB>(w[g]);
    }
  }
  __syncthreads();  // every read of the A results is done: reuse buf as the staging planes

  // staging: output row tau = jp*2^b + u
#pragma unroll
  for (int g = 0; g < TPW; ++g) {
    const int jp = warp + g * NW;
    if (jp < NA && lane < 31) {
#pragma unroll
      for (int u = 0; u < NBk; ++u) {
        const int tau = jp * NBk + u;
        for (int d = 0; d < ndest; ++d) {
          A* dst = buf + (d * NR + tau) * ST_PITCH;
          const int so = soff[d * 64 + tau];
#pragma unroll
          for (int q = 0; q < VB; ++q) {
            const int c = lane * VB + q;
            const int idx = (sigma > 0 ? c : (WC - 1) - c) - so;
            if (idx >= 0 && idx < box) dst[idx] = w[g][u][q];
          }
        }
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
}

// ------------------------------------------------------------------------------------------
// TMA helpers (cp.async.bulk.tensor: SASS UTMASTG)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void tma_store_row(const CUtensorMap* map, const void* smem, int col, int row) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
               :: "l"(reinterpret_cast<uint64_t>(map)), "r"(s), "r"(col), "r"(row) : "memory");
}
__device__ __forceinline__ void tma_commit_and_wait_read() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ int mod_pos(int v, int W) {
  int r = v % W;
  return r < 0 ? r + W : r;
}

// ------------------------------------------------------------------------------------------
// Pass 1
// ------------------------------------------------------------------------------------------
struct P1Slot {
  int sigma;
  int xlo, xhi;       // F_m columns computed: [xlo, xhi), xhi - xlo a multiple of 4
  int ntiles;
  int64_t srow0;      // scratch row of (j = 0, i = 0) inside one image's scratch block
};

struct P1Params {
  const void* img;
  int64_t img_bstride, img_rstride;  // elements
  int rows_avail, cols_avail;        // FRAME rows / cols backed by pixels
  int transposed;                    // FHT row y = image column (P:52 mostly-horizontal)
  int range;                         // §4 loader (sigma = +1, not transposed)
  const int* e_tab;
  const int* colmap;
  int w_content;
  int nq, img0;
  int L;                             // log2(#strips)
  int TX;                            // tile width = TMA box (multiple of 4, <= TX1)
  int64_t scratch_img_rows;          // scratch rows per image
  void* scratch;                     // same buffer as tm_scr (debug st.global path)
  int64_t scr_pitch;
  int no_tma;                        // debug: write rows with st.global instead of TMA
  P1Slot slot[4];
};

// scratch layout: row (img, slot, j, i) = img*scratch_img_rows + srow0 + j*2^L + i,
// column x - xlo holds F_m[i][j](x)  (F_m = levels 1..m of strip i, shift j).
template <typename Tin, int R>
__global__ void __launch_bounds__(Split<R>::nw * 32)
k_p1(const __grid_constant__ CUtensorMap tm_scr, const __grid_constant__ P1Params p) {
  using A = typename AccOf<Tin>::type;
  constexpr int NT = Split<R>::nw * 32;
  constexpr int NR = 1 << R;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  A* buf = reinterpret_cast<A*>(smem_raw);
  int* soff = reinterpret_cast<int*>(smem_raw + tile_buf_elems(R, 1) * 4);

  const int z = blockIdx.z;
  const int qi = z % p.nq;
  const int img = p.img0 + z / p.nq;
  const P1Slot& sl = p.slot[qi];
  const int n = blockIdx.x;
  if (n >= sl.ntiles) return;
  const int strip = blockIdx.y;
  const int TX = p.TX;
  const int X = min(sl.xlo + TX * n, sl.xhi - TX);  // tile = window start (Xw = X)
  const int sigma = sl.sigma;
  const Tin* src = static_cast<const Tin*>(p.img) + (int64_t)img * p.img_bstride;
  const int y0 = strip * NR;
  if (threadIdx.x < NR) soff[threadIdx.x] = 0;

  // ---- fill: buf[rho][c] = frame pixel (y0 + rho, x(c)), zero outside the image (a1: padding is
  // never written to HBM; quadrant handling by index transposition)
  if (!p.transposed) {
#pragma unroll 4
    for (int idx = threadIdx.x; idx < NR * WA; idx += NT) {
      const int rho = idx / WA, c = idx - rho * WA;
      const int y = y0 + rho;
      const int x = sigma > 0 ? X + c : X + (WC - 1) - c;
      A v = A(0);
      if (y < p.rows_avail) {
        if (!p.range) {
          if (x >= 0 && x < p.cols_avail) v = static_cast<A>(__ldg(src + (int64_t)y * p.img_rstride + x));
        } else {  // T(x, y) = I[y][colmap[x - e_y]]  (R13, R14)
          const int u = x - __ldg(p.e_tab + y);
          if (u >= 0 && u < p.w_content)
            v = static_cast<A>(__ldg(src + (int64_t)y * p.img_rstride + __ldg(p.colmap + u)));
        }
      }
      buf[rho * IN_PITCH + c] = v;
    }
  } else {
#pragma unroll 4
    for (int idx = threadIdx.x; idx < NR * WA; idx += NT) {
      const int c = idx / NR, rho = idx - c * NR;  // consecutive threads: consecutive image columns
      const int y = y0 + rho;
      const int x = sigma > 0 ? X + c : X + (WC - 1) - c;
      A v = A(0);
      if (y < p.rows_avail && x >= 0 && x < p.cols_avail)
        v = static_cast<A>(__ldg(src + (int64_t)x * p.img_rstride + y));
      buf[rho * IN_PITCH + c] = v;
    }
  }
  __syncthreads();
  tile_fht<R, A>(buf, sigma, 1, soff, TX);

  // ---- store F_m[strip][j] (j = tau): scratch column X - xlo is 16-byte aligned
  const int64_t rowbase = (int64_t)(img - p.img0) * p.scratch_img_rows + sl.srow0 + strip;
  const int col = X - sl.xlo;
  if (!p.no_tma) {
    if (threadIdx.x < NR) {
      const int j = threadIdx.x;
      tma_store_row(&tm_scr, buf + j * ST_PITCH, col, (int)(rowbase + ((int64_t)j << p.L)));
      tma_commit_and_wait_read();
    }
  } else {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = warp; j < NR; j += NT / 32) {
      A* drow = static_cast<A*>(p.scratch) + (rowbase + ((int64_t)j << p.L)) * p.scr_pitch + col;
      for (int c = lane; c < TX; c += 32) __stcg(drow + c, buf[j * ST_PITCH + c]);
    }
  }
}

// ------------------------------------------------------------------------------------------
// Pass 2
// ------------------------------------------------------------------------------------------
struct P2Slot {
  int sigma;
  int xlo1, xhi1;    // pass-1 columns: F_m[i][j](x') stored for x' in [xlo1, xhi1)
  int64_t srow0;
  int xbeg, xend;    // output signed column range covered by tiles (width W, or range span)
  int ntiles;
  int64_t qrow;      // output row (in the [rows_total][W] view) of quadrant row 0, per image
  int rbase, rsign, skip;  // output row = qrow + rbase + rsign*t; t == skip not stored
};

struct P2Dest {
  void* ptr;
  int64_t pitch;           // elements
  int64_t rows_per_img;
  int shifted;             // 1 = fused fhtshift (§5) destination
};

struct P2Params {
  const void* scratch;
  int64_t scr_pitch;
  int64_t scratch_img_rows;
  int nq, img0;
  int TX;                  // tile stride (columns owned per tile); TMA box = TX + 4
  int W, Hp, wc;
  int range;
  const int* start_tab;    // range: per-row support start (signed, unwrapped)
  const int* len_tab;      // range: per-row support length
  int ndest;               // 1 or 2 destinations
  int no_tma;              // debug: write rows with st.global instead of TMA
  P2Slot slot[4];
  P2Dest dest[2];
};

template <typename A, int R>
__global__ void __launch_bounds__(Split<R>::nw * 32)
k_p2(const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1,
     const __grid_constant__ P2Params p) {
  constexpr int NW = Split<R>::nw;
  constexpr int NT = NW * 32;
  constexpr int NR = 1 << R;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  A* buf = reinterpret_cast<A*>(smem_raw);
  int* soff = reinterpret_cast<int*>(smem_raw + tile_buf_elems(R, p.ndest) * 4);

  const int z = blockIdx.z;
  const int qi = z % p.nq;
  const int img = p.img0 + z / p.nq;
  const P2Slot& sl = p.slot[qi];
  const int n = blockIdx.x;
  if (n >= sl.ntiles) return;
  const int j = blockIdx.y;
  const int TX = p.TX, box = TX + WO2;
  const int X = min(sl.xbeg + TX * n, sl.xend - TX);
  const int Xw = X - WO2;  // window start: window index s <-> x = Xw + s
  const int sigma = sl.sigma;
  const int t0 = j * NR, tmax = t0 + NR - 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // per (dest, row): destination shift k, aligned start r and the staging offset (window index
  // s is staged at s - soff; staging index 0 <-> x = X - r)
  if (threadIdx.x < 2 * NR) {
    const int d = threadIdx.x / NR, tau = threadIdx.x - d * NR;
    int so = 0;
    if (d < p.ndest) {
      const int t = t0 + tau;
      int k = 0;
      if (p.dest[d].shifted) {
        if (p.range) k = (((p.W - __ldg(p.len_tab + t)) + 1) >> 1) - __ldg(p.start_tab + t);
        else k = sigma > 0 ? ceil_half(p.Hp + t) : ceil_half(p.Hp - t);
      }
      const int r = mod_pos(X + k, p.W) & 3;
      so = WO2 - r;
    }
    soff[d * 64 + tau] = so;
  }

  bool black = false;  // the whole window is outside every row's pattern support
  if (!p.range) black = sigma > 0 ? (Xw + WC - 1 < -tmax) : (Xw >= p.wc + tmax);

  if (!black) {
    const A* scr = static_cast<const A*>(p.scratch) +
                   ((int64_t)(img - p.img0) * p.scratch_img_rows + sl.srow0 + t0) * p.scr_pitch;
#pragma unroll 4
    for (int idx = threadIdx.x; idx < NR * WA; idx += NT) {
      const int i = idx / WA, c = idx - i * WA;
      const int x = sigma > 0 ? Xw + c : Xw + (WC - 1) - c;
      const int xs = x + sigma * j * i;  // G_j[i](x) = F_m[i][j](x + sigma*j*i)
      A v = A(0);
      if (xs >= sl.xlo1 && xs < sl.xhi1) v = __ldcg(scr + (int64_t)i * p.scr_pitch + (xs - sl.xlo1));
      buf[i * IN_PITCH + c] = v;
    }
    __syncthreads();
    tile_fht<R, A>(buf, sigma, p.ndest, soff, box);
  } else {
    for (int idx = threadIdx.x; idx < p.ndest * NR * ST_PITCH; idx += NT) buf[idx] = A(0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }

  // ---- stores: item = (dest d, row tau); one warp per item
  bool issued = false;
  for (int item = warp; item < p.ndest * NR; item += NW) {
    const int d = item / NR, tau = item - d * NR;
    const P2Dest& D = p.dest[d];
    const int t = t0 + tau;
    if (t == sl.skip) continue;
    const int64_t orow = (int64_t)img * D.rows_per_img + sl.qrow + sl.rbase + (int64_t)sl.rsign * t;
    // valid columns of this row: [vlo, vhi); the tile owns [X, X + TX)
    int vlo = sl.xbeg, vhi = sl.xend, k = 0;
    if (p.range) {
      vlo = __ldg(p.start_tab + t);
      vhi = vlo + p.W;
      if (D.shifted) k = (((p.W - __ldg(p.len_tab + t)) + 1) >> 1) - vlo;
    } else if (D.shifted) {
      k = sigma > 0 ? ceil_half(p.Hp + t) : ceil_half(p.Hp - t);
    }
    const int r = WO2 - soff[d * 64 + tau];
    const int xs0 = X - r;                     // x of staging index 0
    const int d0 = mod_pos(xs0 + k, p.W);      // its destination column (16-byte aligned)
    const A* srow = buf + (d * NR + tau) * ST_PITCH;
    int mlo = max(X, vlo), mhi = min(X + TX, vhi);  // columns still to write by hand
    if (!p.no_tma && xs0 >= vlo && xs0 + min(box, p.W - d0) <= vhi) {
      if (lane == 0) {
        tma_store_row(d == 0 ? &tm0 : &tm1, srow, d0, (int)orow);  // clipped at column W
        issued = true;
      }
      mlo = max(mlo, xs0 + (p.W - d0));       // the wrapped remainder, if any
    }
    if (mlo < mhi) {
      A* drow = static_cast<A*>(D.ptr) + orow * D.pitch;
      for (int x = mlo + lane; x < mhi; x += 32) {
        int col = d0 + (x - xs0);
        if (col >= p.W) col -= p.W;
        __stcs(drow + col, srow[x - xs0]);
      }
    }
  }
  if (issued) tma_commit_and_wait_read();
}

}  // namespace v2
}  // namespace fht
