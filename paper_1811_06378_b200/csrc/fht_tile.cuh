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
// ("window index" s) from the 288 input columns x(e) = Xa + e, e in [0, 288) (Xa = Xw for
// sigma = +1, Xw - 71 for sigma = -1: the halo lies on the partner side). The butterflies run in
// a local frame where the partner sits at +shift for both signs: c = e (sigma = +1) or
// c = 287 - e (sigma = -1, mirrored); window index s = c (+1) or 216 - c (-1). Lane l owns local
// columns l*V .. l*V+V-1; lane 31 is a halo lane whose results are discarded, so every shuffle
// partner of lanes 0..30 is inside the warp (needs 2^levels - 1 <= V).
//
// Bulk tensor copies (measured on this B200 by tools/tma_probe.cu): the innermost start
// coordinate must be 16-byte aligned (negative is allowed for loads, which zero-fill outside the
// tensor; stores need >= 0 and clip at the upper bound), and the shared address 128-byte aligned.
// Loads therefore start at the aligned-down column and the tile keeps a per-row offset; stores
// are staged at an offset chosen so the destination starts on a 16-byte boundary.
//   pass 1: input rows by TMA (non-transposed image with 16-byte pitch), a vectorised transposing
//           fill (transposed quadrants) or a scalar gather (angle-range loader, odd pitches);
//           scratch rows by TMA (always aligned).
//   pass 2: scratch rows by TMA (the tensor bound is the written extent, so the zero fill is the
//           "outside the pass-1 support" mask); Hough rows x mod W and, for the fused fhtshift,
//           (x + k_t) mod W by TMA from a staging row realigned per destination; a cyclic-wrap
//           remainder or a row-support edge (range mode) by a warp with coalesced st.global.
#pragma once
#include <cuda.h>

#include <type_traits>
#include <utility>

#include "fht_common.cuh"

// Compile-time variants for A/B timing (tools/build_variant.sh); defaults are the measured best.
#ifndef FHT_STAGE_ASM
#define FHT_STAGE_ASM 1   // staging: explicitly predicated st.shared (1) or C++ if (0)
#endif
#ifndef FHT_P2_DENSE
#define FHT_P2_DENSE 1    // pass-2 plain destination of interior tiles as one 2-D box (1)
#endif

#ifndef FHT_SCR_KEEP
#define FHT_SCR_KEEP 1    // pass-1 scratch stores with an L2 evict-last hint
#endif
#ifndef FHT_P2_WARPLOAD
#define FHT_P2_WARPLOAD 1 // pass 2: each warp issues and waits for the TMA loads of its own sub-pass-A blocks
#endif
#ifndef FHT_P1_WARPLOAD
#define FHT_P1_WARPLOAD 1 // pass 1 (TMA fill): same, per-block mbarriers instead of one for the tile
#endif
#ifndef FHT_OUT_EVICT_FIRST
#define FHT_OUT_EVICT_FIRST 0 // Hough-row TMA stores with an L2 evict-first hint (measured: 0 is ~0.5% faster)
#endif
#ifndef FHT_P2_BLACK
#define FHT_P2_BLACK 1    // pass 2: black-zone tiles store zeros without loads or butterflies
#endif
#ifndef FHT_P2_REVERSE_DEST
#define FHT_P2_REVERSE_DEST 1  // pass 2: store the second destination (fhtshift) first (measured ~1% faster)
#endif
#ifndef FHT_PDL
#define FHT_PDL 1         // programmatic dependent launch between the passes (griddepcontrol)
#endif
#ifndef FHT_P2_UNPRED
#define FHT_P2_UNPRED 1   // pass 2: row staging planes with slack, stored without bounds predicates
#endif
#ifndef FHT_P2_DENSE_MASK
#define FHT_P2_DENSE_MASK 1  // pass 2 dense box: the lane's in-box flags computed once for all rows
#endif
#ifndef FHT_P2_WARPSTORE
#define FHT_P2_WARPSTORE 1  // pass 2: each warp stages and stores its own 8 output rows (no CTA barrier after sub-pass B)
#endif
#ifndef FHT_ROW32
#define FHT_ROW32 1       // one TMA per 4-byte row: a [rows][cols/32][32] view, box {32, 10} = 320 columns (was 256 + 36)
#endif
#if FHT_ROW32 && !FHT_P2_WARPLOAD
#error "FHT_ROW32 needs the per-warp pass-2 loads (FHT_P2_WARPLOAD)"
#endif
#ifndef FHT_P1_STAGE2
#define FHT_P1_STAGE2 1   // pass 1: full-width tiles predicate only the last staged column
#endif

namespace fht {
namespace v2 {

// Programmatic dependent launch (PDL): a kernel launched with programmatic stream serialization
// may start while its predecessor drains; griddepcontrol.wait blocks until the predecessor grid
// has completed and its memory is visible, launch_dependents lets the successor be scheduled.
__device__ __forceinline__ void pdl_wait() {
#if FHT_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#if FHT_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// Thread groups: a tile body runs on a group of threads that synchronise among themselves. GrpAll is
// the whole CTA (__syncthreads); GrpPart<N> is N threads from `base` (a multiple of 32) with their
// own named barrier, so one CTA can run two independent tiles side by side (the pipelined kernel).
struct GrpAll {
  __device__ __forceinline__ int tid() const { return (int)threadIdx.x; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
  __device__ __forceinline__ bool sync_or(bool v) const { return __syncthreads_or(v) != 0; }
};
template <int N>
struct GrpPart {
  int base, bar;  // first thread; named barrier id (1..15; 0 is __syncthreads)
  __device__ __forceinline__ int tid() const { return (int)threadIdx.x - base; }
  __device__ __forceinline__ void sync() const { asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(N) : "memory"); }
  __device__ __forceinline__ bool sync_or(bool v) const {
    uint32_t r;
    asm volatile("{ .reg .pred p, q; setp.ne.u32 p, %1, 0; bar.red.or.pred q, %2, %3, p; selp.u32 %0, 1, 0, q; }"
                 : "=r"(r) : "r"((uint32_t)v), "r"(bar), "n"(N) : "memory");
    return r != 0;
  }
};

constexpr int VA = 9;            // local columns per lane, sub-pass A (odd => conflict-free)
constexpr int VB = 7;            // local columns per lane, sub-pass B (odd => conflict-free)
constexpr int WA = 32 * VA;      // 288 local input columns per tile
constexpr int WC = 31 * VB;      // 217 computed window columns per tile
constexpr int FA_PITCH = WA + 1; // 289: odd pitch (A results; conflict-free transposing fill)
constexpr int TMA_PITCH = 320;   // TMA-loaded 4-byte rows: 292 used, 1280-B (128-B multiple) pitch
constexpr int TMA_PITCH_U8 = 384;// TMA-loaded 1-byte rows: 304 used, 384-B pitch
constexpr int ST_PITCH = 224;    // staging pitch (elements): 896 B rows, 128-B aligned for TMA
constexpr int kStgOff = 32;      // row planes start 128 B into the buffer (a margin for row 0's out-of-box columns)
constexpr int TX1 = 216;         // pass-1 tile width (= its TMA box), multiple of 4
constexpr int BOX2 = 212;        // pass-2 store box width (multiple of 4)
constexpr int WO2 = 4;           // pass-2 window starts 4 columns left of the tile's own columns

template <int R> struct Split;
template <> struct Split<1> { static constexpr int a = 1, b = 0, nw = 4; };
template <> struct Split<2> { static constexpr int a = 2, b = 0, nw = 4; };
template <> struct Split<3> { static constexpr int a = 3, b = 0, nw = 4; };
template <> struct Split<4> { static constexpr int a = 2, b = 2, nw = 4; };
#ifndef FHT_SPLIT5_A
#define FHT_SPLIT5_A 2  // 32-row tiles: sub-pass A levels (3: 8-row A blocks + 4-row B groups; 2: 4 + 8)
#endif
template <> struct Split<5> { static constexpr int a = FHT_SPLIT5_A, b = 5 - FHT_SPLIT5_A, nw = 4; };
template <> struct Split<6> { static constexpr int a = 3, b = 3, nw = 8; };
// pass-1 scratch element: u8 input keeps F_m (<= 255 * 2^m <= 16320 for m <= 6) in uint16
template <typename Tin> struct ScrOf { using type = typename AccOf<Tin>::type; };
template <> struct ScrOf<uint8_t> { using type = uint16_t; };
template <int R> constexpr int kMinBlocks = Split<R>::nw == 4 ? 5 : 2;  // occupancy target (regs <= 102 / 128)
template <int R> constexpr int kTPW = ((1 << Split<R>::a) + Split<R>::nw - 1) / Split<R>::nw;  // B tasks/warp
// pass 2 stores per warp (FHT_P2_WARPSTORE): every warp owns one sub-pass-B group of 8 rows
template <int R> constexpr bool kWarpStore = FHT_P2_WARPSTORE && (1 << Split<R>::b) == 8 && kTPW<R> == 1 &&
                                             (1 << Split<R>::a) == Split<R>::nw && Split<R>::nw * 32 >= 2 * (1 << R);
// rows of the dense-box store (tensor map box height): a warp's 8 rows, or the whole tile
inline int p2_box_rows(int R) {
  switch (R) {
    case 5: return kWarpStore<5> ? 8 : 32;
    case 6: return kWarpStore<6> ? 8 : 64;
  }
  return 1 << R;
}

// Shared memory layout (bytes): [main buffer][u8 input tile (pass 1 u8 TMA only)][tables]
__host__ __device__ constexpr size_t main_buf_bytes(int R) { return (size_t)(1 << R) * TMA_PITCH * 4; }
__host__ __device__ constexpr size_t u8_tile_bytes(int R) { return (size_t)(1 << R) * TMA_PITCH_U8; }
// tables: [rowoff 64 ints][soff 2x64 ints][mbarrier] = 1 KB, then (pass 2) RowInfo [2][2^R], 16 B each.
// Kept small: 5 CTAs of 2^R = 32 rows must fit in 228 KB (measured: 4 CTAs/SM cost 10%).
constexpr size_t kTableBytes = 1024;
__host__ __device__ constexpr size_t p1_smem_bytes(int R, bool u8) {
  return main_buf_bytes(R) + (u8 ? u8_tile_bytes(R) : 0) + kTableBytes;
}
// §4 range loader: the strip's colmap slice staged after the tables (2 KB keeps 5 CTAs/SM at R = 5)
constexpr int kColmapStage = 512;
constexpr size_t kColmapStageBytes = kColmapStage * 4;
__host__ __device__ constexpr size_t p2_smem_bytes(int R) {
  return main_buf_bytes(R) + kTableBytes + 2 * (size_t)(1 << R) * 16;
}

// ------------------------------------------------------------------------------------------
// Register butterfly (north_star "out[t] = A[t>>1] + B[t>>1] shifted by ceil(t/2)"
// Fig. 6). v[row][q] = row `row`, local column lane*V + q. After the call row t holds
// shift t of the 2^NB-row block. Partner columns beyond the lane come from lane+1 (shfl_down);
// valid for lanes 0..30 when 2^NB - 1 <= V.
// ------------------------------------------------------------------------------------------
// ------------------------------------------------------------------------------------------
// TMA / mbarrier helpers (SASS: UTMALDG / UTMASTG, SYNCS)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tma_store_row(const CUtensorMap* map, const void* smem, int col, int row) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
               :: "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(smem)), "r"(col), "r"(row) : "memory");
}
// Hough rows are never re-read: evict-first keeps the L2 for the pass-1 scratch
__device__ __forceinline__ void tma_store_row_stream(const CUtensorMap* map, const void* smem, int col, int row) {
#if !FHT_OUT_EVICT_FIRST
  tma_store_row(map, smem, col, row);
  return;
#endif
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;"
               :: "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(smem)), "r"(col), "r"(row), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* smem, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
               :: "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
// Pass-1 scratch: keep it in L2 for pass 2 (evict-last)
__device__ __forceinline__ void tma_store_3d_keep(const CUtensorMap* map, const void* smem, int c0, int c1, int c2) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;"
               :: "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
               : "memory");
}
// 4-D pass-1 scratch box, L2 evict-last (kept for pass 2)
__device__ __forceinline__ void tma_store_4d_keep(const CUtensorMap* map, const void* smem, int c0, int c1, int c2, int c3) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4, %5}], [%1], %6;"
               :: "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
                  "l"(pol)
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* smem, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];"
               :: "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, void* smem, uint64_t* bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               :: "r"(smem_u32(smem)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, void* smem, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
               :: "r"(smem_u32(smem)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1),
                  "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_load_4d(const CUtensorMap* map, void* smem, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
               :: "r"(smem_u32(smem)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1),
                  "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// wait for the completion of the phase with parity `par` (a barrier reused across tiles alternates)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t par) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(par) : "memory");
  }
}
__device__ __forceinline__ void mbar_wait0(uint64_t* bar) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(bar)) : "memory");
  }
}

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
// In-CTA FHT of a 2^R-row tile. Input element (row rho, x-order index e) is
// src[rho*src_pitch + rowoff[rho] + e] (converted to A). Sub-pass A writes F_a in LOCAL order
// to fa[row*fa_pitch + c] (may alias src: each warp reads all its rows before writing them);
// sub-pass B leaves output row tau = jp*2^b + u, local column lane*VB + q in w[g][u][q]
// (jp = warp + g*NW). Ends with __syncthreads (fa and src are free afterwards).
// ------------------------------------------------------------------------------------------
// The loader fills v[r][q] = input (row blk*2^a + r, x-order index e) for the lane's columns,
// e = lane*VA + q (SIG = +1) or (WA - 1) - lane*VA - q (SIG = -1).
// jp_lim: sub-pass-B groups computed (rows tau < jp_lim * 2^b; the others are not needed: a pruned plan's pass 1
// stores only its first shifts)
template <int R, int SIG, typename A, typename LoadA, typename G>
__device__ __forceinline__ void tile_fht_ld(const G& grp, const LoadA& load, A* fa, int fa_pitch,
                                            A (&w)[kTPW<R>][1 << Split<R>::b][VB], int jp_lim = 1 << Split<R>::a) {
  using S = Split<R>;
  constexpr int a = S::a, b = S::b, NW = S::nw;
  constexpr int NA = 1 << a, NBk = 1 << b;
  const int warp = grp.tid() >> 5, lane = threadIdx.x & 31;

  // sub-pass A: block blk = rows blk*2^a .. +2^a-1 -> fa row blk*2^a + j' = F_a[blk][j']
#pragma unroll 1
  for (int blk = warp; blk < NBk; blk += NW) {
    A v[NA][VA];
    load(blk, v);
    warp_fht<a, VA>(v);
    A* d = fa + (blk * NA) * fa_pitch + lane * VA;
    FHT_CHECK(smem_in_bounds(d + (NA - 1) * fa_pitch + VA - 1, sizeof(A)));
#pragma unroll
    for (int r = 0; r < NA; ++r)
#pragma unroll
      for (int q = 0; q < VA; ++q) d[r * fa_pitch + q] = v[r][q];
  }
  grp.sync();

  // sub-pass B: group jp: G[i'](c) = F_a[i'][jp](c + jp*i')  (pre-shear identity, local frame)
#pragma unroll
  for (int g = 0; g < kTPW<R>; ++g) {
    const int jp = warp + g * NW;
    if (jp < NA && jp < jp_lim) {
#pragma unroll
      for (int i = 0; i < NBk; ++i) {
        const A* s = fa + (i * NA + jp) * fa_pitch + lane * VB + jp * i;
        FHT_CHECK(smem_in_bounds(s + VB - 1, sizeof(A)) && lane * VB + jp * i + VB <= fa_pitch);
#pragma unroll
        for (int q = 0; q < VB; ++q) w[g][i][q] = s[q];
      }
      warp_fht<b, VB>(w[g]);
    }
  }
  grp.sync();
}

// Input rows from shared memory: element (rho, e) at src[rho*src_pitch + rowoff[rho] + e]; with
// blk_bars, a block's rows are waited for (TMA) by the warp that reads them.
// The lane's VA = 9 consecutive narrow elements (u8 pass-1 rows, u16 pass-2 scratch rows) by 32-bit shared loads:
// the aligned words covering them (3 for 9 bytes, 5 for 9 u16), funnel-shifted by the misalignment and split with
// byte permutes -- a third (u8) / a half (u16) of the shared-memory wavefronts of one narrow load per element (these
// passes are bound by the L1 / shared-memory pipe). e[k] = element lo + k.
#ifndef FHT_NARROW_VEC
#define FHT_NARROW_VEC 1
#endif
__device__ __forceinline__ uint32_t lds_b32(uint32_t a) {  // shared-space load (a generic load would be LD, not LDS)
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");  // ordered before the in-place fa stores
  return v;
}
template <typename Tsrc>
__device__ __forceinline__ void load9_narrow(const Tsrc* lo, uint32_t (&e)[VA]) {
  const uint32_t la = smem_u32(lo);
  const uint32_t wa = la & ~3u;
  const uint32_t sh = (la & 3u) * 8u;
  if constexpr (sizeof(Tsrc) == 1) {
    const uint32_t w0 = lds_b32(wa), w1 = lds_b32(wa + 4), w2 = lds_b32(wa + 8);
    const uint32_t x0 = __funnelshift_r(w0, w1, sh), x1 = __funnelshift_r(w1, w2, sh);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      e[k] = __byte_perm(x0, 0u, 0x4440u | k);
      e[4 + k] = __byte_perm(x1, 0u, 0x4440u | k);
    }
    e[8] = (w2 >> sh) & 0xffu;
  } else {
    const uint32_t w0 = lds_b32(wa), w1 = lds_b32(wa + 4), w2 = lds_b32(wa + 8), w3 = lds_b32(wa + 12),
                   w4 = lds_b32(wa + 16);
    const uint32_t x[4] = {__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh), __funnelshift_r(w2, w3, sh),
                           __funnelshift_r(w3, w4, sh)};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      e[2 * j] = x[j] & 0xffffu;
      e[2 * j + 1] = x[j] >> 16;
    }
    e[8] = (w4 >> sh) & 0xffffu;
  }
}

template <int R, int SIG, typename A, typename Tsrc, typename G>
__device__ __forceinline__ void tile_fht(const G& grp, const Tsrc* src, int src_pitch, const int* rowoff, A* fa,
                                         int fa_pitch, A (&w)[kTPW<R>][1 << Split<R>::b][VB],
                                         uint64_t* blk_bars = nullptr, uint32_t par = 0,
                                         int jp_lim = 1 << Split<R>::a) {
  constexpr int NA = 1 << Split<R>::a;
  const int lane = threadIdx.x & 31;
  auto load = [&](int blk, A (&v)[NA][VA]) {
    if (blk_bars) mbar_wait(blk_bars + blk, (par >> blk) & 1u);  // this block's rows have landed (TMA)
#pragma unroll
    for (int r = 0; r < NA; ++r) {
      const int rho = blk * NA + r;
      const Tsrc* p = src + rho * src_pitch + rowoff[rho] + (SIG > 0 ? lane * VA : (WA - 1) - lane * VA);
      FHT_CHECK(smem_in_bounds(SIG > 0 ? p + VA - 1 : p, sizeof(Tsrc)) &&
                smem_in_bounds(SIG > 0 ? p : p - (VA - 1), sizeof(Tsrc)));
      if constexpr (FHT_NARROW_VEC && sizeof(Tsrc) < 4) {
        uint32_t e[VA];
        load9_narrow<Tsrc>(SIG > 0 ? p : p - (VA - 1), e);
#pragma unroll
        for (int q = 0; q < VA; ++q) v[r][q] = static_cast<A>(e[SIG > 0 ? q : VA - 1 - q]);
      } else {
#pragma unroll
        for (int q = 0; q < VA; ++q) v[r][q] = static_cast<A>(p[SIG > 0 ? q : -q]);
      }
    }
  };
  tile_fht_ld<R, SIG, A>(grp, load, fa, fa_pitch, w, jp_lim);
}

// Sg: the staged element type (A, or uint16_t for the u8 pipeline's pass-1 scratch)
template <int Q, typename Sg, typename A>
__device__ __forceinline__ void st_pred(uint32_t a, int idx, int box, A v) {
  if constexpr (sizeof(Sg) == 2) {
    const uint16_t bits = static_cast<uint16_t>(v);  // exact: u8 pass-1 sums are <= 255 * 2^6
    asm volatile("{ .reg .pred p; setp.lt.u32 p, %1, %2; @p st.shared.b16 [%0+%3], %4; }"
                 :: "r"(a), "r"(idx), "r"(box), "n"(Q * 2), "h"(bits) : "memory");
  } else {
    const uint32_t bits = *reinterpret_cast<const uint32_t*>(&v);
    asm volatile("{ .reg .pred p; setp.lt.u32 p, %1, %2; @p st.shared.b32 [%0+%3], %4; }"
                 :: "r"(a), "r"(idx), "r"(box), "n"(Q * 4), "r"(bits) : "memory");
  }
}
template <int SIG, typename Sg, typename A, int... Q>
__device__ __forceinline__ void st_pred_row(uint32_t a, int lo, int box, const A (&v)[VB], std::integer_sequence<int, Q...>) {
  (st_pred<Q, Sg>(a, lo + Q, box, v[SIG > 0 ? Q : VB - 1 - Q]), ...);
}

// Write the register results into a staging plane of row pitch `pitch`: output row tau, window
// index s stored at s - soff[tau] when 0 <= that < box. Explicitly predicated st.shared (one
// ISETP + one STS per element, no branches). Then fence for the TMA engine and synchronise.
// PRED = 0: no bounds predicates -- the plane has slack around every row (staging indices [-4, WC) land inside
// the pitch, row 0's negatives in a margin before the plane), so the out-of-box columns are written and never read.
// PRED = 2: soff == 0 and box >= WC - 1 (pass 1's full-width tiles): only a lane's last column can fall outside
// (window index WC - 1 = 216 of a 216-wide box), so only that store is predicated.
// PRED = 3: every row has the same soff (pass 2's dense box): the lane's 7 in-box flags are computed once and
// shared by all its rows.
template <int R, int SIG, typename A, typename Sg = A, typename G = GrpAll, int PRED = 1>
__device__ __forceinline__ void stage_rows(const G& grp, A (&w)[kTPW<R>][1 << Split<R>::b][VB], Sg* stg,
                                           const int* soff, int box, int pitch, int jp_lim = 1 << Split<R>::a) {
  using S = Split<R>;
  constexpr int NA = 1 << S::a, NBk = 1 << S::b, NW = S::nw;
  const int warp = grp.tid() >> 5, lane = threadIdx.x & 31;
  uint32_t inbox = 0;  // PRED == 3: bit q = column q of the lane is inside the box (the same for every row)
  if constexpr (PRED == 3) {
    const int lo = (SIG > 0 ? lane * VB : (WC - VB) - lane * VB) - soff[0];
#pragma unroll
    for (int q = 0; q < VB; ++q) inbox |= ((unsigned)(lo + q) < (unsigned)box ? 1u : 0u) << q;
  }
#pragma unroll
  for (int g = 0; g < kTPW<R>; ++g) {
    const int jp = warp + g * NW;
    if (jp < NA && jp < jp_lim && lane < 31) {
#pragma unroll
      for (int u = 0; u < NBk; ++u) {
        const int tau = jp * NBk + u;
        // lowest window index of the lane's 7 columns, and its staging index
        const int lo = (SIG > 0 ? lane * VB : (WC - VB) - lane * VB) - soff[tau];
        FHT_CHECK(box <= pitch && smem_in_bounds(stg + tau * pitch + box - 1, sizeof(Sg)));
        if constexpr (PRED == 3) {
          Sg* dst = stg + tau * pitch + lo;
#pragma unroll
          for (int q = 0; q < VB; ++q)
            if (inbox & (1u << q)) dst[q] = static_cast<Sg>(w[g][u][SIG > 0 ? q : VB - 1 - q]);
          continue;
        }
        if constexpr (PRED == 2) {
          Sg* dst = stg + tau * pitch + lo;
#pragma unroll
          for (int q = 0; q < VB - 1; ++q) dst[q] = static_cast<Sg>(w[g][u][SIG > 0 ? q : VB - 1 - q]);
          if (lo + VB - 1 < box) dst[VB - 1] = static_cast<Sg>(w[g][u][SIG > 0 ? VB - 1 : 0]);
          continue;
        }
        if constexpr (PRED == 0) {
          Sg* dst = stg + tau * pitch + lo;
          FHT_CHECK(lo >= -4 && lo + VB <= pitch - 4 && smem_in_bounds(dst, sizeof(Sg)));
#pragma unroll
          for (int q = 0; q < VB; ++q) dst[q] = static_cast<Sg>(w[g][u][SIG > 0 ? q : VB - 1 - q]);
          continue;
        }
#if FHT_STAGE_ASM
        const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(stg + tau * pitch + lo));
        // element q of the lane sits at staging index lo + q
        st_pred_row<SIG, Sg>(a, lo, box, w[g][u], std::make_integer_sequence<int, VB>{});
#else
        Sg* dst = stg + tau * pitch;
#pragma unroll
        for (int q = 0; q < VB; ++q)
          if ((unsigned)(lo + q) < (unsigned)box) dst[lo + q] = static_cast<Sg>(w[g][u][SIG > 0 ? q : VB - 1 - q]);
#endif
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  grp.sync();
}

// ------------------------------------------------------------------------------------------
// TMA / mbarrier helpers (SASS: UTMALDG / UTMASTG, SYNCS)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ int mod_pos(int v, int W) {
  int r = v % W;
  return r < 0 ? r + W : r;
}

// ------------------------------------------------------------------------------------------
// Pass 1
// ------------------------------------------------------------------------------------------
struct P1Slot {
  int sigma;
  int transposed;     // FHT row y = image column (P:52 mostly-horizontal quadrants)
  int xlo, xhi;       // F_m columns computed: [xlo, xhi), xhi - xlo a multiple of 4
  int ntiles;
  int64_t srow0;      // scratch row of (j = 0, i = 0) inside one image's scratch block
};

struct P1Params {
  const void* img;
  int64_t img_bstride, img_rstride;  // elements
  int img_h, img_w;                  // image rows / cols (a transposed slot swaps their roles)
  int range;                         // §4 loader (sigma = +1, not transposed)
  const int* e_tab;
  const int* colmap;
  int w_content;
  int fill_tma;                      // non-transposed rows by TMA (image base/pitch 16-B aligned)
  int fill_vec;                      // transposed fill with 16-byte (u8: 4-byte) loads
  int fill32;                        // 4-byte rows by ONE TMA each: tm_img0 is the view [img][row][col/32][32] (w % 32 == 0)
  int tfill_tma;                     // u8 transposed tiles by TMA (k_p1's tm_imgT: image, box {2^R columns, 144 rows})
  int nq, img0;
  int ntiles;                        // tiles per strip (max over slots)
  int L;                             // log2(#strips)
  int TX;                            // tile width = TMA box (multiple of 4, <= TX1)
  int64_t scratch_img_rows;          // scratch rows per image
  int z0;                            // first z (= image-in-chunk * nq + slot) of this scratch buffer
  int strip0;                        // first strip of the launch (image rows from strip0 * 2^m): a shard's strips
  int nq_log;                        // log2 nq (1, 2 or 4 slots)
  int ndst;                          // scratch destinations (P1Dst): 1, or one per rank of a sharded transform
  int jper;                          // shifts j per destination (ngroups / ndst)
  P1Slot slot[4];
};

// Where pass 1 stores F_m: ndst 4-D tensor maps [z][j][strip][column] (dims column, strip, j, z), each
// taking `jper` consecutive shifts j of the tile's box -- destination d gets j in [d*jper, (d+1)*jper).
// One destination: the local scratch. A sharded transform: one per rank, each rank's
// groups J_d, into the send buffer (then one all-to-all) or straight into the peers' receive buffers.
constexpr int kMaxDst = 8;
struct P1Dst {
  CUtensorMap m[kMaxDst];
};

// scratch layout: row (img, slot, j, i) = img*scratch_img_rows + srow0 + j*2^L + i,
// column x - xlo holds F_m[i][j](x)  (F_m = levels 1..m of strip i, shift j).
//
// The butterfly part is instantiated per sign (SIG); the fills are sign-independent (they only
// need the input origin Xa) and exist once per kernel, which keeps the kernel's code footprint
// inside the instruction cache.
constexpr int kNoRow = -2147483647 - 1;  // range fill: the row has no content in this tile

// FILL = 1 (§4 range loader, sigma = +1): tsrc holds, per row rho, the image row y0 + rho from
// column rowoff[rho] on (TMA); the transformed row T(x', y) = I[y][colmap[x' - e_y]] (P:146,
// P:152) is gathered from it through colmap, e_y = erow[rho].
// zscr: the scratch z (= buffer image x slot) the tile's F_m rows go to; smem: the group's shared memory.
template <typename Tin, int R, int SIG, typename Tsrc, int FILL = 0, typename G>
__device__ __forceinline__ void p1_tail_impl(const G grp, unsigned char* smem, const P1Dst* dst, const P1Params& p,
                                     const P1Slot& sl, int strip, int X, int zscr, const Tsrc* tsrc, int tpitch,
                                     int fa_pitch, uint64_t* bars, uint32_t par) {
  using A = typename AccOf<Tin>::type;
  using S = Split<R>;
  A* buf = reinterpret_cast<A*>(smem);
  unsigned char* tab = smem + main_buf_bytes(R) + (sizeof(Tin) == 1 ? u8_tile_bytes(R) : 0);
  // only the shifts j < ndst * jper are stored (a pruned plan's groups): sub-pass-B groups past them are skipped
  const int jp_lim = (p.ndst * p.jper + (1 << S::b) - 1) >> S::b;
  const int* rowoff = reinterpret_cast<const int*>(tab);
  const int* soff = rowoff + 64;
  A w[kTPW<R>][1 << S::b][VB];
  if constexpr (FILL == 1) {
    constexpr int NA = 1 << S::a;
    const int* erow = soff + 64;
    const int* cm_s = reinterpret_cast<const int*>(tab + kTableBytes);  // colmap[cm_lo + i]
    const int cm_lo = reinterpret_cast<const int*>(tab)[224], cm_n = reinterpret_cast<const int*>(tab)[225];
    const int lane = threadIdx.x & 31;
    auto load = [&](int blk, A (&v)[NA][VA]) {
      mbar_wait(bars + blk, (par >> blk) & 1u);
      if (cm_n <= kColmapStage) {  // every u of the strip is inside the staged slice
#pragma unroll
        for (int r = 0; r < NA; ++r) {
          const int rho = blk * NA + r;
          const int a0 = rowoff[rho], u0 = X + lane * VA - erow[rho];
#pragma unroll
          for (int q = 0; q < VA; ++q) {
            const int u = u0 + q;
            A val = A(0);
            if (a0 != kNoRow && (unsigned)u < (unsigned)p.w_content)
              val = static_cast<A>(tsrc[rho * tpitch + (cm_s[u - cm_lo] - a0)]);
            v[r][q] = val;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < NA; ++r) {
          const int rho = blk * NA + r;
          const int a0 = rowoff[rho], u0 = X + lane * VA - erow[rho];
#pragma unroll
          for (int q = 0; q < VA; ++q) {
            const int u = u0 + q;
            A val = A(0);
            if (a0 != kNoRow && (unsigned)u < (unsigned)p.w_content)
              val = static_cast<A>(tsrc[rho * tpitch + (__ldg(p.colmap + u) - a0)]);
            v[r][q] = val;
          }
        }
      }
    };
    tile_fht_ld<R, SIG, A>(grp, load, buf, fa_pitch, w, jp_lim);
  } else {
    tile_fht<R, SIG, A>(grp, tsrc, tpitch, rowoff, buf, fa_pitch, w, bars, par, jp_lim);
  }
  // dense [NR][TX] in the scratch type (u8 input: uint16), the box layout
  using Sc = typename ScrOf<Tin>::type;
  if (FHT_P1_STAGE2 && p.TX >= WC - 1)  // full-width tile (soff = 0): only the window's last column can fall outside
    stage_rows<R, SIG, A, Sc, G, 2>(grp, w, reinterpret_cast<Sc*>(buf), soff, p.TX, p.TX, jp_lim);
  else
    stage_rows<R, SIG, A, Sc>(grp, w, reinterpret_cast<Sc*>(buf), soff, p.TX, p.TX, jp_lim);
  // ---- store F_m[strip][j] for all j: per destination d ONE box {TX, 1, jper, 1} of its 4-D view
  // [z][j][strip][column] (z = image-in-chunk * nq + slot); column X - xlo is 16-B aligned
  if (grp.tid() == 0) {
    FHT_CHECK(X - sl.xlo >= 0 && X - sl.xlo + p.TX <= sl.xhi - sl.xlo && p.ndst * p.jper <= (1 << R));
    for (int d = 0; d < p.ndst; ++d) {
      const void* src = reinterpret_cast<const Sc*>(buf) + (size_t)d * p.jper * p.TX;
#if FHT_SCR_KEEP
      tma_store_4d_keep(&dst->m[d], src, X - sl.xlo, strip, 0, zscr);
#else
      tma_store_4d(&dst->m[d], src, X - sl.xlo, strip, 0, zscr);
#endif
    }
    tma_commit();
  }
  pdl_trigger();
  if (grp.tid() == 0) tma_wait_read();
}

// The tail behind a call boundary in k_p1 (one instance per sign: the kernel's code stays inside the
// instruction cache); inlined (INL) where a caller keeps state across it (the pipelined kernel).
template <typename Tin, int R, int SIG, typename Tsrc, int FILL = 0, typename G>
__device__ __noinline__ void p1_tail(const G grp, unsigned char* smem, const P1Dst* dst, const P1Params& p,
                                     const P1Slot& sl, int strip, int X, int zscr, const Tsrc* tsrc, int tpitch,
                                     int fa_pitch, uint64_t* bars, uint32_t par) {
  p1_tail_impl<Tin, R, SIG, Tsrc, FILL>(grp, smem, dst, p, sl, strip, X, zscr, tsrc, tpitch, fa_pitch, bars, par);
}

template <typename Tin, int R, typename Tsrc, int FILL = 0, bool INL = false, typename G>
__device__ __forceinline__ void p1_tail_sig(const G& grp, unsigned char* smem, int sigma, const P1Dst* dst,
                                            const P1Params& p, const P1Slot& sl, int strip, int X, int zscr,
                                            const Tsrc* tsrc, int tpitch, int fa_pitch, uint64_t* bars = nullptr,
                                            uint32_t par = 0) {
  if constexpr (INL) {
    if constexpr (FILL == 1) {
      p1_tail_impl<Tin, R, 1, Tsrc, 1>(grp, smem, dst, p, sl, strip, X, zscr, tsrc, tpitch, fa_pitch, bars, par);
    } else {
      if (sigma > 0)
        p1_tail_impl<Tin, R, 1, Tsrc, 0>(grp, smem, dst, p, sl, strip, X, zscr, tsrc, tpitch, fa_pitch, bars, par);
      else
        p1_tail_impl<Tin, R, -1, Tsrc, 0>(grp, smem, dst, p, sl, strip, X, zscr, tsrc, tpitch, fa_pitch, bars, par);
    }
  } else if constexpr (FILL == 1) {  // the range frame is sigma = +1 only
    p1_tail<Tin, R, 1, Tsrc, 1>(grp, smem, dst, p, sl, strip, X, zscr, tsrc, tpitch, fa_pitch, bars, par);
  } else {
    if (sigma > 0)
      p1_tail<Tin, R, 1, Tsrc, 0>(grp, smem, dst, p, sl, strip, X, zscr, tsrc, tpitch, fa_pitch, bars, par);
    else
      p1_tail<Tin, R, -1, Tsrc, 0>(grp, smem, dst, p, sl, strip, X, zscr, tsrc, tpitch, fa_pitch, bars, par);
  }
}

// Returns whether the tile used its per-block mbarriers (one phase each): the TMA fills. INL: the tail
// inlined (see p1_tail).
template <typename Tin, int R, bool INL = false, typename G>
__device__ __forceinline__ bool p1_body(const G& grp, unsigned char* smem_raw, const CUtensorMap* tm_img0,
                                        const CUtensorMap* tm_img1, const P1Dst* dst, const P1Params& p,
                                        const P1Slot& sl, int img, int strip, int X, int zscr,
                                        uint64_t* ext_bars = nullptr, uint32_t par = 0,
                                        const CUtensorMap* tm_imgT = nullptr) {
  using A = typename AccOf<Tin>::type;
  using S = Split<R>;
  constexpr int NT = S::nw * 32;
  constexpr int NR = 1 << R;
  const int tid = grp.tid();
  A* buf = reinterpret_cast<A*>(smem_raw);
  unsigned char* tab = smem_raw + main_buf_bytes(R) + (sizeof(Tin) == 1 ? u8_tile_bytes(R) : 0);
  int* rowoff = reinterpret_cast<int*>(tab);          // [NR]
  int* soff = rowoff + 64;                            // [NR]
  // per-block mbarriers: the tile's own (initialised here, phase 0), or the caller's persistent ones
  // (initialised once, phase parity `par` bit per block: the pipelined kernel)
  uint64_t* bar = ext_bars ? ext_bars : reinterpret_cast<uint64_t*>(tab + 768);
  const Tin* src = static_cast<const Tin*>(p.img) + (int64_t)img * p.img_bstride;
  const int y0 = (p.strip0 + strip) * NR;  // strip: the launch's (a shard's) local strip index
  const int Xa = sl.sigma > 0 ? X : X - (WA - WC);  // x of input index e = 0

  if (p.range && p.fill_tma) {
    // ---- §4 range loader by TMA (alpha >= 1: a tile row's 288 transformed columns come from at
    // most 289 consecutive image columns, colmap being a dilation): row rho = image row y0 + rho
    // from the aligned-down column of colmap[max(0, Xa - e_y)]; the transform is gathered from
    // shared memory in the sub-pass-A loader. Every warp loads its own blocks' rows.
    constexpr int AL = 16 / sizeof(Tin);
    constexpr int TP = sizeof(Tin) == 1 ? TMA_PITCH_U8 : TMA_PITCH;
    constexpr uint32_t row_bytes = sizeof(Tin) == 1 ? 256 + 48 : (256 + 36) * 4;
    constexpr int NA = 1 << S::a, NBk = 1 << S::b, NW = S::nw;
    Tin* tile = reinterpret_cast<Tin*>(sizeof(Tin) == 1 ? smem_raw + main_buf_bytes(R) : smem_raw);
    int* erow = soff + 64;
    const int warp = tid >> 5, lane = threadIdx.x & 31;
    bool any_row = false;  // some row of the tile has transformed content (the warp's blocks)
    for (int b = warp; b < NBk; b += NW) {
      const int rho = b * NA + lane, y = y0 + rho;
      int a0 = kNoRow, e = 0;
      bool ne = false;
      if (lane < NA) {
        if (y < p.img_h) {
          e = __ldg(p.e_tab + y);
          const int u0 = Xa - e;
          if (u0 < p.w_content && u0 + WA > 0) {
            a0 = __ldg(p.colmap + max(0, u0)) & ~(AL - 1);
            ne = true;
          }
        }
        rowoff[rho] = a0;
        erow[rho] = e;
        soff[rho] = 0;
      }
      const unsigned m = __ballot_sync(0xffffffffu, ne);
      any_row |= m != 0u;
      if (lane == 0) {
        if (!ext_bars) mbar_init(bar + b);
        mbar_expect_tx(bar + b, (uint32_t)__popc(m) * row_bytes);
      }
      __syncwarp();
      if (ne) {
        Tin* d = tile + rho * TP;
        tma_load_3d(tm_img0, d, bar + b, a0, y, img);
        tma_load_3d(tm_img1, d + 256, bar + b, a0 + 256, y, img);
      }
    }
    // the strip's colmap slice: e_y is monotonic in y (e_y = floor(g*y + 0.5)), so the u range of
    // the strip is [Xa - e_max, Xa + 288 - e_min) from its first and last rows; staged while the
    // row loads are in flight
    {
      int* cm_s = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(rowoff) + kTableBytes);
      int ulo = 0, n = 0;
      if (y0 < p.img_h) {
        const int ea = __ldg(p.e_tab + y0), eb = __ldg(p.e_tab + min(y0 + NR - 1, p.img_h - 1));
        ulo = max(0, Xa - max(ea, eb));
        n = max(0, min(p.w_content, Xa + WA - min(ea, eb)) - ulo);
      }
      if (n <= kColmapStage)
        for (int i = tid; i < n; i += NT) cm_s[i] = __ldg(p.colmap + ulo + i);
      if (tid == 0) {
        rowoff[224] = ulo;
        rowoff[225] = n;
      }
      if (!grp.sync_or(any_row)) {
        // no row of the tile has content (no load was issued): F_m is 0 over the whole tile
        A* z = reinterpret_cast<A*>(smem_raw);
        for (int idx = tid; idx < NR * p.TX; idx += NT) z[idx] = A(0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        grp.sync();
        if (tid == 0) {
          for (int d = 0; d < p.ndst; ++d)
            tma_store_4d_keep(&dst->m[d], z + (size_t)d * p.jper * p.TX, X - sl.xlo, strip, 0, zscr);
          tma_commit();
        }
        pdl_trigger();
        if (tid == 0) tma_wait_read();
        return true;
      }
    }
    p1_tail_sig<Tin, R, Tin, 1, INL>(grp, smem_raw, 1, dst, p, sl, strip, X, zscr, static_cast<const Tin*>(tile), TP,
                                sizeof(Tin) == 1 ? FA_PITCH : TMA_PITCH, bar, par);
    return true;
  }
  if (!sl.transposed && p.fill_tma) {
    // ---- TMA: NR image rows, columns [Xa, Xa + 288) from the 16-byte aligned column below
    constexpr int AL = 16 / sizeof(Tin);
    const int a0 = Xa & ~(AL - 1);
    constexpr int TP = sizeof(Tin) == 1 ? TMA_PITCH_U8 : TMA_PITCH;
    Tin* tile = reinterpret_cast<Tin*>(sizeof(Tin) == 1 ? smem_raw + main_buf_bytes(R) : smem_raw);
    constexpr uint32_t row_bytes = sizeof(Tin) == 1 ? 256 + 48 : (256 + 36) * 4;
#if FHT_P1_WARPLOAD
    // each warp issues (lane 0) and waits for (in tile_fht) the rows of its own sub-pass-A blocks
    constexpr int NA = 1 << S::a, NBk = 1 << S::b, NW = S::nw;
    const int warp = tid >> 5, lane = threadIdx.x & 31;
    // fill32 (4-byte rows): ONE box {32, 10} of the [img][row][col/32][32] view per row, from the 128-byte
    // aligned column a32 <= Xa: 320 columns cover the 288 the tile needs for any offset Xa - a32 < 32
    const int a32 = Xa & ~31;
    const bool f32r = sizeof(Tin) == 4 && FHT_ROW32 && p.fill32;
    for (int b = warp; b < NBk; b += NW) {
      if (lane == 0) {
        if (!ext_bars) mbar_init(bar + b);
        mbar_expect_tx(bar + b, f32r ? NA * (uint32_t)TMA_PITCH * 4 : NA * row_bytes);
        for (int rho = b * NA; rho < (b + 1) * NA; ++rho) {
          Tin* d = tile + rho * TP;
          if (f32r) {
            tma_load_4d(tm_img0, d, bar + b, 0, a32 >> 5, y0 + rho, img);
          } else {
            tma_load_3d(tm_img0, d, bar + b, a0, y0 + rho, img);
            tma_load_3d(tm_img1, d + 256, bar + b, a0 + 256, y0 + rho, img);
          }
        }
      }
      if (lane < NA) {
        rowoff[b * NA + lane] = Xa - (f32r ? a32 : a0);
        soff[b * NA + lane] = 0;
      }
    }
    __syncwarp();
    uint64_t* const bars = bar;
#else
    if (tid < NR) {
      rowoff[tid] = Xa - a0;
      soff[tid] = 0;
    }
    if (tid == 0) mbar_init(bar);
    grp.sync();
    if (tid < 32) {
      if (tid == 0) mbar_expect_tx(bar, NR * row_bytes);
      __syncwarp();
      for (int rho = tid; rho < NR; rho += 32) {
        Tin* d = tile + rho * TP;
        tma_load_3d(tm_img0, d, bar, a0, y0 + rho, img);
        tma_load_3d(tm_img1, d + 256, bar, a0 + 256, y0 + rho, img);
      }
    }
    mbar_wait0(bar);
    uint64_t* const bars = nullptr;
#endif
    if constexpr (sizeof(Tin) == 1)
      p1_tail_sig<Tin, R, Tin, 0, INL>(grp, smem_raw, sl.sigma, dst, p, sl, strip, X, zscr,
                                       static_cast<const Tin*>(tile), TP, FA_PITCH, bars, par);
    else
      p1_tail_sig<Tin, R, A, 0, INL>(grp, smem_raw, sl.sigma, dst, p, sl, strip, X, zscr,
                                     reinterpret_cast<const A*>(tile), TP, TMA_PITCH, bars, par);
    return bars != nullptr;
  }
  if (tid < NR) {
    rowoff[tid] = 0;
    soff[tid] = 0;
  }
  if (!sl.transposed || p.range) {
    // ---- scalar fill (angle-range gather T(x, y) = I[y][colmap[x - e_y]], or odd pitches), in
    // batches of CH elements per thread: every gather of a batch is in flight before its stores
    // (the colmap -> pixel chain is two dependent loads; 4 in flight per thread was latency-bound).
    // A mostly-horizontal range plan (transposed slot) gathers T(x, y) = I[colmap[x - e_y]][y]:
    // frame row y is image column y.
    const int frows = sl.transposed ? p.img_w : p.img_h;
    constexpr int ITS = (NR * WA + NT - 1) / NT;
    constexpr int CH = ITS >= 12 ? 12 : ITS;
#pragma unroll 1
    for (int it0 = 0; it0 < ITS; it0 += CH) {
      int cm[CH];
      A v[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) {  // stage 1: colmap (range) or the column index itself
        const int idx = tid + (it0 + c) * NT;
        const int rho = idx / WA, e = idx - rho * WA;
        const int y = y0 + rho, x = Xa + e;
        cm[c] = -1;
        if (it0 + c < ITS && idx < NR * WA && y < frows) {
          if (!p.range) {
            if (x >= 0 && x < p.img_w) cm[c] = x;
          } else {  // P:146; R13, R14
            const int u = x - __ldg(p.e_tab + y);
            if (u >= 0 && u < p.w_content) cm[c] = __ldg(p.colmap + u);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < CH; ++c) {  // stage 2: the pixels
        const int idx = tid + (it0 + c) * NT;
        const int rho = idx / WA;
        const int64_t off = sl.transposed ? (int64_t)cm[c] * p.img_rstride + (y0 + rho)
                                          : (int64_t)(y0 + rho) * p.img_rstride + cm[c];
        v[c] = cm[c] >= 0 ? static_cast<A>(__ldg(src + off)) : A(0);
      }
#pragma unroll
      for (int c = 0; c < CH; ++c) {  // stage 3: shared memory
        const int idx = tid + (it0 + c) * NT;
        if (it0 + c < ITS && idx < NR * WA) {
          const int rho = idx / WA, e = idx - rho * WA;
          buf[rho * FA_PITCH + e] = v[c];
        }
      }
    }
  } else if (sizeof(Tin) == 1 && NR >= 16 && tm_imgT && p.tfill_tma && !ext_bars) {
    // ---- transposed u8 tile by TMA: the image block [Xa, Xa + 288) rows x [y0, y0 + NR) columns lands dense
    // ([288][NR] bytes, zero outside the image) in the u8 tile area (two boxes of 144 rows), then each warp
    // transposes 32 consecutive image rows x 4 columns per step: one 4-byte shared load, four conflict-free
    // int column stores (FHT row y0 + c = image column, FHT column e = image row). Replaces NR/4 scattered 4-byte
    // global loads per image row (C3's transposed pass 1 took 1.8x its non-transposed one).
    uint8_t* tt = reinterpret_cast<uint8_t*>(smem_raw + main_buf_bytes(R));
    uint64_t* b0 = bar;
    if (tid == 0) {
      mbar_init(b0);
      mbar_expect_tx(b0, (uint32_t)(WA * NR));
      tma_load_3d(tm_imgT, tt, b0, y0, Xa, img);
      tma_load_3d(tm_imgT, tt + 144 * NR, b0, y0, Xa + 144, img);
    }
    grp.sync();
    mbar_wait0(b0);
    constexpr int NQ = NR >= 16 ? NR / 4 : 1;  // 4-byte words per image row
    const int lane = threadIdx.x & 31, warp = tid >> 5;
    for (int it = warp; it < (WA / 32) * NQ; it += NT / 32) {
      const int q = it % NQ, e = (it / NQ) * 32 + lane;  // image row Xa + e, columns y0 + 4q .. + 3
      const uint32_t wv = reinterpret_cast<const uint32_t*>(tt)[e * NQ + q];
      A* d = buf + (4 * q) * FA_PITCH + e;
      d[0] = static_cast<A>(wv & 0xffu);
      d[FA_PITCH] = static_cast<A>((wv >> 8) & 0xffu);
      d[2 * FA_PITCH] = static_cast<A>((wv >> 16) & 0xffu);
      d[3 * FA_PITCH] = static_cast<A>(wv >> 24);
    }
  } else if (p.fill_vec && NR >= 4) {
    // ---- transposed: FHT row y = image column, FHT column x = image row. Thread = (x, 4 y's):
    // one 16-byte (u8: 4-byte) load from image row x, 4 conflict-free column stores. All of a
    // thread's loads are issued before its first store (memory-level parallelism).
    constexpr int YQ = NR >= 4 ? NR / 4 : 1;  // threads per image row
    constexpr int IT = (WA * YQ + NT - 1) / NT;
    constexpr int ES = NT / YQ;                // image rows per iteration (NT is a multiple of YQ)
    static_assert(NT % YQ == 0, "whole image rows per iteration");
    using V4 = typename std::conditional<sizeof(Tin) == 1, uchar4,
               typename std::conditional<std::is_same<Tin, float>::value, float4, int4>::type>::type;
    // a thread's 4 image columns (yq) are fixed; its image row advances by ES per iteration: one base pointer
    // and a constant stride instead of a 64-bit multiply and the divisions per element (the fill was ~19% of
    // the 64-row pass 1's instructions)
    const int yq = tid & (YQ - 1), e0 = tid / YQ;
    const int y = y0 + 4 * yq;
    const bool yfull = y + 3 < p.img_w;
    const Tin* base = src + (int64_t)(Xa + e0) * p.img_rstride + y;
    const int64_t step = (int64_t)ES * p.img_rstride;
    // every image row of the tile inside the image: no per-iteration row check
    const bool rows_in = Xa >= 0 && Xa + WA <= p.img_h;
    V4 vals[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = e0 + it * ES, x = Xa + e;
      vals[it] = V4{};
      const Tin* ps = base + it * step;
      if (e < WA && (rows_in || (x >= 0 && x < p.img_h))) {
        if (yfull) {
          vals[it] = __ldg(reinterpret_cast<const V4*>(ps));
        } else {
          Tin t[4] = {Tin(0), Tin(0), Tin(0), Tin(0)};
          for (int k = 0; k < 3; ++k)
            if (y + k < p.img_w) t[k] = __ldg(ps + k);
          vals[it].x = t[0];
          vals[it].y = t[1];
          vals[it].z = t[2];
        }
      }
    }
    A* const dbase = buf + (4 * yq) * FA_PITCH + e0;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      if (e0 + it * ES < WA) {
        A* d = dbase + it * ES;
        d[0] = static_cast<A>(vals[it].x);
        d[FA_PITCH] = static_cast<A>(vals[it].y);
        d[2 * FA_PITCH] = static_cast<A>(vals[it].z);
        d[3 * FA_PITCH] = static_cast<A>(vals[it].w);
      }
    }
  } else {
    for (int idx = tid; idx < NR * WA; idx += NT) {
      const int e = idx / NR, rho = idx - e * NR;  // consecutive threads: consecutive image columns
      const int y = y0 + rho, x = Xa + e;
      A v = A(0);
      if (y < p.img_w && x >= 0 && x < p.img_h) v = static_cast<A>(__ldg(src + (int64_t)x * p.img_rstride + y));
      buf[rho * FA_PITCH + e] = v;
    }
  }
  grp.sync();
  p1_tail_sig<Tin, R, A, 0, INL>(grp, smem_raw, sl.sigma, dst, p, sl, strip, X, zscr, static_cast<const A*>(buf),
                                 FA_PITCH, FA_PITCH);
  return false;
}

// tm_img0: image [batch][h][w], box 1 x 1 x 256 columns; tm_img1: box 36 (u8: 48) columns;
// dst: where F_m goes (P1Dst; box {TX, 1, jper, 1} each).
template <typename Tin, int R>
__global__ void __launch_bounds__(Split<R>::nw * 32, kMinBlocks<R>)
k_p1(const __grid_constant__ CUtensorMap tm_img0, const __grid_constant__ CUtensorMap tm_img1,
     const __grid_constant__ P1Dst dst, const __grid_constant__ P1Params p,
     const __grid_constant__ CUtensorMap tm_imgT) {
  pdl_wait();  // the image may come from the previous kernel; the scratch may still be read by it
  // flat grid, quadrant slot fastest: with 148 SMs (a multiple of 4) the round-robin CTA
  // placement gives every SM CTAs of one slot, i.e. one sign and one fill path (I-cache locality)
  // grid (ntiles * nq, strips, images): no integer division (it was 4% of the kernel's instructions)
  const int qi = blockIdx.x & ((1 << p.nq_log) - 1);
  const int n = blockIdx.x >> p.nq_log;
  const int strip = blockIdx.y;
  const int img = p.img0 + blockIdx.z;
  const P1Slot& sl = p.slot[qi];
  if (n >= sl.ntiles) return;
  const int X = min(sl.xlo + p.TX * n, sl.xhi - p.TX);  // tile = window start (Xw = X)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  p1_body<Tin, R>(GrpAll{}, smem_raw, &tm_img0, &tm_img1, &dst, p, sl, img, strip, X,
                  p.z0 + (img - p.img0) * p.nq + qi, nullptr, 0, &tm_imgT);
}

// ------------------------------------------------------------------------------------------
// Pass 2
// ------------------------------------------------------------------------------------------
struct P2Slot {
  int sigma;
  int xlo1, xhi1;    // pass-1 columns: F_m[i][j](x') stored for x' in [xlo1, xhi1)
  int64_t srow0;
  int xbeg, xend;    // output signed column range covered by tiles (width W, or range span)
  int xmid;          // tiles never straddle xmid (the cyclic wrap x = 0 of sigma = +1 rows)
  int ntiles_a;      // tiles in [xbeg, xmid); the rest tile [xmid, xend)
  int ntiles;
  int64_t qrow;      // output row (in the [rows_total][W] view) of quadrant row 0, per image
  int rbase, rsign, skip;  // output row = qrow + rbase + rsign*t; t == skip not stored
};

struct P2Dest {
  void* ptr;
  int64_t pitch;           // elements
  int64_t rows_per_img;
  int64_t nrows;           // rows of the destination's [rows_total][W] view (bounds checks)
  int shifted;             // 1 = fused fhtshift (§5) destination
};

struct P2Params {
  int64_t scratch_img_rows;
  int64_t row0;            // first scratch row of this chunk's buffer
  int nq, img0;
  int nq_log;              // log2 nq
  int ntiles;              // tiles per group (max over slots)
  int m;                   // log2(#groups of the transform)
  int ngroups;             // groups launched (2^m, or ceil(rows_out / 2^L) for a pruned range plan)
  int rows_out;            // output rows t >= rows_out are neither computed for nor stored (f2)
  int TX;                  // tile stride (columns owned per tile); store box = TX + 4
  int W, Hp, wc;
  int range;
  const int* start_tab;    // range: per-row support start (signed, unwrapped)
  const int* len_tab;      // range: per-row support length
  int ndest;               // 1 or 2 destinations
  int no_tma;              // debug: write every row with st.global
  // sharded transform: groups j0 .. j0 + ngroups - 1; strip i of group j is scratch row
  // rbase(j) + (i >> logS) * strideG + (i & (2^logS - 1)) -- the chunk from rank i >> logS of a receive
  // buffer [rank][z][j_local][strip_local]. Unsharded: j0 = 0, logS = L (one chunk).
  int j0, logS;
  int64_t strideG;
  int64_t scr_rows;        // rows of the scratch tensor pass 2 reads (bounds checks)
  P2Slot slot[4];
  P2Dest dest[2];
};

struct RowInfo {  // per (destination, output row), shared memory, 16 B
  int orow;       // row in the destination's [rows_total][W] view
  int d0;         // destination column of staging index 0 (16-byte aligned); bit 30 = TMA row store
  int mlo, mhi;   // columns [mlo, mhi) left to plain stores
};
constexpr int kTmaBit = 1 << 30;

// rbase: the scratch row of (group j, strip 0); strip i is row rbase + i. smem: the group's shared memory.
// Returns whether the tile used its per-block mbarriers (every tile but a black one).
template <typename A, int R, int SIG, typename Tscr, typename G>
__device__ __forceinline__ bool p2_body(const G& grp, unsigned char* smem_raw, const CUtensorMap* tm_scr0,
                                        const CUtensorMap* tm_scr1, const CUtensorMap* tm0, const CUtensorMap* tm1,
                                        const CUtensorMap* tm0_box, const P2Params& p, const P2Slot& sl, int img,
                                        int j, int X, int own, int64_t rbase, uint64_t* ext_bars = nullptr,
                                        uint32_t par = 0) {
  using S = Split<R>;
  constexpr int NW = S::nw;
  constexpr int NT = NW * 32;
  constexpr int NR = 1 << R;
  const int tid = grp.tid();
  A* buf = reinterpret_cast<A*>(smem_raw);
  unsigned char* tab = smem_raw + main_buf_bytes(R);
  int* rowoff = reinterpret_cast<int*>(tab);                  // [64]
  int* soff = rowoff + 64;                                    // [2][64]
  // [8] per-block mbarriers: the tile's own, or the caller's persistent ones (parity bits `par`)
  uint64_t* bar = ext_bars ? ext_bars : reinterpret_cast<uint64_t*>(tab + 768);
  RowInfo* info = reinterpret_cast<RowInfo*>(tab + 1024);     // [2][NR], 16 B each
  const int TX = p.TX, box = TX + WO2;
  const int Xw = X - WO2;                        // window start: window index s <-> x = Xw + s
  const int Xa = SIG > 0 ? Xw : Xw - (WA - WC);  // x of input index e = 0
  const int t0 = j * NR, tmax = t0 + NR - 1;
  const int warp = tid >> 5, lane = threadIdx.x & 31;
  A w[kTPW<R>][1 << S::b][VB];

  bool black = false;  // the whole window is outside every row's pattern support
  if (FHT_P2_BLACK && !p.range) black = SIG > 0 ? (Xw + WC - 1 < -tmax) : (Xw >= p.wc + tmax);

  // ---- scratch rows t0 + i, column (x + sigma*j*i) - xlo1 for x = Xa + e: TMA from the
  // aligned-down column, zero outside [0, xhi1 - xlo1) = outside what pass 1 wrote. Issued first,
  // so the loads are in flight while the CTA plans its stores.
  constexpr int NA = 1 << S::a, NBk = 1 << S::b;  // sub-pass A blocks: one mbarrier each
#if FHT_P2_WARPLOAD
  // every warp issues (lane 0) and waits for the rows of its own sub-pass-A blocks blk = warp,
  // warp + NW, ...: no CTA-wide barrier between the issue and the butterflies, and the four warps
  // issue in parallel. rowoff of a block's rows is written by the warp that reads them.
  if (!black) {
    // scratch rows of Tscr: loads start at the 16-byte aligned column below (kAl elements) and
    // take 256 + kBox1 columns (kBox1 * sizeof(Tscr) a multiple of 16); row i lands at byte
    // i * TMA_PITCH * 4 of the buffer, where its fa row will be written in place
#if FHT_ROW32
    // ONE box {32, 10} per row of the scratch view [row][col/32][32] (the pass-1 span is a multiple of 32
    // columns, host side): 320 columns from the aligned-down column cover the 288 needed
    constexpr int kAl = 32;
    constexpr uint32_t kRowBytes = 320 * (uint32_t)sizeof(Tscr);
#else
    constexpr int kAl = 16 / (int)sizeof(Tscr), kBox1 = sizeof(Tscr) == 2 ? 40 : 36;
    constexpr uint32_t kRowBytes = (256 + kBox1) * (uint32_t)sizeof(Tscr);
#endif
    for (int b = warp; b < NBk; b += NW) {
      if (lane == 0) {
        if (!ext_bars) mbar_init(bar + b);
        mbar_expect_tx(bar + b, NA * kRowBytes);
        for (int i = b * NA; i < (b + 1) * NA; ++i) {
          const int a0 = (Xa + SIG * j * i - sl.xlo1) & ~(kAl - 1);
          Tscr* d = reinterpret_cast<Tscr*>(buf + i * TMA_PITCH);
          const int row = (int)(rbase + (int64_t)(i >> p.logS) * p.strideG + (i & ((1 << p.logS) - 1)));
          FHT_CHECK(row >= 0 && row < p.scr_rows);
#if FHT_ROW32
          tma_load_3d(tm_scr0, d, bar + b, 0, a0 >> 5, row);
#else
          tma_load_2d(tm_scr0, d, bar + b, a0, row);
          tma_load_2d(tm_scr1, d + 256, bar + b, a0 + 256, row);
#endif
        }
      }
      if (lane < NA) rowoff[b * NA + lane] = (Xa + SIG * j * (b * NA + lane) - sl.xlo1) & (kAl - 1);
    }
    __syncwarp();
  }
#else
  if (!black && tid == 0) {
    for (int b = 0; b < NBk; ++b) mbar_init(bar + b);
    for (int b = 0; b < NBk; ++b) {
      mbar_expect_tx(bar + b, NA * (256 + 36) * 4);
      for (int i = b * NA; i < (b + 1) * NA; ++i) {
        const int a0 = (Xa + SIG * j * i - sl.xlo1) & ~3;
        A* d = buf + i * TMA_PITCH;
        tma_load_2d(tm_scr0, d, bar + b, a0, (int)(rbase + i));
        tma_load_2d(tm_scr1, d + 256, bar + b, a0 + 256, (int)(rbase + i));
      }
    }
  }
#endif

  // ---- store plan per (destination, row): shift k, 16-byte aligned start, TMA or plain stores.
  // remw[c]: some row of plan items [32c, 32c + 32) has columns left to plain stores (one ballot per warp: the
  // items of a warp are one 32-item chunk while NT >= ndest * NR, which holds for every R)
  int* const remw = reinterpret_cast<int*>(tab + 896);
  for (int it = tid; it < p.ndest * NR; it += NT) {
    const int d = it / NR, tau = it - d * NR, t = t0 + tau;
    const P2Dest& D = p.dest[d];
    int vlo = sl.xbeg, vhi = sl.xend, k = 0;
    if (p.range) {
      vlo = __ldg(p.start_tab + t);
      vhi = vlo + p.W;
      if (D.shifted) k = (((p.W - __ldg(p.len_tab + t)) + 1) >> 1) - vlo;
    } else if (D.shifted) {
      // R11 generic rule ceil((W - len)/2) - start with len = wc + t: ceil((pad + t)/2) (sigma = +1,
      // start = -t) or ceil((pad - t)/2) (sigma = -1, start = 0), pad = W - wc
      const int pad = p.W - p.wc;
      k = SIG > 0 ? ceil_half(pad + t) : ceil_half(pad - t);
    }
    // X in [xbeg, xend), k in [0, W): one conditional add/subtract replaces the modulo (range
    // mode: k is arbitrary, keep the division)
    int v = X + k;
    if (p.range) v = mod_pos(v, p.W);
    else { v += v < 0 ? p.W : 0; v -= v >= p.W ? p.W : 0; }  // X + k in (-W, 2W) for every pad >= h - 1
    const int r = v & 3;
    const int xs0 = X - r;
    int d0 = v - r;
    d0 += d0 < 0 ? p.W : 0;
    RowInfo ri;
    ri.orow = (int)((int64_t)img * D.rows_per_img + sl.qrow + sl.rbase + (int64_t)sl.rsign * t);
    ri.d0 = d0;
    ri.mlo = max(X, vlo);
    ri.mhi = min(X + own, vhi);
    if (t == sl.skip || t >= p.rows_out) {
      ri.mhi = ri.mlo;
    } else if (!p.no_tma && xs0 >= vlo && xs0 + min(box, p.W - d0) <= vhi) {
      ri.d0 |= kTmaBit;
      ri.mlo = max(ri.mlo, xs0 + min(box, p.W - d0));  // what the box does not cover (wrap, tile end)
    }
    info[d * NR + tau] = ri;
    soff[d * 64 + tau] = WO2 - r;
    if (NT >= 2 * NR) {
      const unsigned rem = __ballot_sync(__activemask(), ri.mlo < ri.mhi);
      if ((threadIdx.x & 31) == 0) remw[it >> 5] = rem != 0u;
    }
  }
#if FHT_P2_WARPLOAD
  // the plan (info, soff) is read after tile_fht's first group barrier; a black tile has none
  if (black) grp.sync();
#else
  if (!black && tid < NR) rowoff[tid] = (Xa + SIG * j * tid - sl.xlo1) & 3;
  grp.sync();
#endif

  if (!black)
    tile_fht<R, SIG, A, Tscr, G>(grp, reinterpret_cast<const Tscr*>(buf), TMA_PITCH * 4 / (int)sizeof(Tscr), rowoff,
                                     buf, TMA_PITCH, w, bar, par);

#if FHT_P2_WARPSTORE
  if constexpr (kWarpStore<R>) {
    // ---- warp-owned stores: warp w holds output rows [8w, 8w + 8) (sub-pass-B group jp = w) and stages them in
    // its own region of the buffer, [8][box] (dense plane of destination 0) or 8 rows of ST_PITCH after a 32-element
    // margin (row planes), then issues their bulk stores itself: after the sub-pass-B barrier no CTA barrier is
    // needed, only the warp's own fence / __syncwarp and its lane 0's wait for the bulk reads before it restages.
    constexpr int RW = 8, WREG = 32 + RW * ST_PITCH;  // rows per warp; region per warp (128-byte multiple)
    const int r0 = warp * RW;
    A* const stw = buf + warp * WREG;
    bool issued = false;
    for (int dd = 0; dd < p.ndest; ++dd) {
      const int d = FHT_P2_REVERSE_DEST ? p.ndest - 1 - dd : dd;
      const P2Dest& D = p.dest[d];
      const RowInfo* inf = info + d * NR;
      const int* so = soff + d * 64;
      if (dd > 0) {
        if (lane == 0 && issued) tma_wait_read();
        __syncwarp();
      }
      const bool dense = FHT_P2_DENSE && !p.range && !D.shifted && sl.rsign == 1 && (sl.skip < t0 || sl.skip > tmax) &&
                         tmax < p.rows_out && (inf[0].d0 & kTmaBit) && inf[0].mlo >= inf[0].mhi;
      A* const stg = dense ? stw : stw + 32;
      const int pitch = dense ? box : ST_PITCH;
      if (!black) {
        const int lo0 = SIG > 0 ? lane * VB : (WC - VB) - lane * VB;  // lowest window index of the lane's columns
        if (lane < 31) {
          if (dense) {  // one aligned start for all rows: the lane's in-box flags once
            const int lo = lo0 - so[0];
            uint32_t inbox = 0;
#pragma unroll
            for (int q = 0; q < VB; ++q) inbox |= ((unsigned)(lo + q) < (unsigned)box ? 1u : 0u) << q;
#pragma unroll
            for (int u = 0; u < RW; ++u) {
              A* dst = stg + u * box + lo;
              FHT_CHECK(smem_in_bounds(stg + RW * box - 1, sizeof(A)));
#pragma unroll
              for (int q = 0; q < VB; ++q)
                if (inbox & (1u << q)) dst[q] = w[0][u][SIG > 0 ? q : VB - 1 - q];
            }
          } else {  // rows with slack: staging indices [-4, WC) stay inside the row's pitch / the margin
#pragma unroll
            for (int u = 0; u < RW; ++u) {
              A* dst = stg + u * ST_PITCH + lo0 - so[r0 + u];
              FHT_CHECK(smem_in_bounds(dst, sizeof(A)) && smem_in_bounds(dst + VB - 1, sizeof(A)));
#pragma unroll
              for (int q = 0; q < VB; ++q) dst[q] = w[0][u][SIG > 0 ? q : VB - 1 - q];
            }
          }
        }
      } else {  // a black tile's outputs are all 0
        float4* z4 = reinterpret_cast<float4*>(stg);
        for (int idx = lane; idx < (RW * pitch) >> 2; idx += 32) z4[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (dense) {
          FHT_CHECK(inf[r0].orow >= 0 && inf[r0].orow + RW <= D.nrows);
          tma_store_row_stream(tm0_box, stg, inf[0].d0 & ~kTmaBit, inf[r0].orow);  // box {box, 8}
        } else {
#pragma unroll 1
          for (int u = 0; u < RW; ++u) {
            const RowInfo ri = inf[r0 + u];
            if (ri.d0 & kTmaBit) {
              FHT_CHECK((ri.d0 & ~kTmaBit) >= 0 && (ri.d0 & ~kTmaBit) < p.W && ri.orow >= 0 && ri.orow < D.nrows);
              tma_store_row_stream(d == 0 ? tm0 : tm1, stg + u * ST_PITCH, ri.d0 & ~kTmaBit, ri.orow);  // clipped at W
            }
          }
        }
        tma_commit();
        issued = true;
      }
      // columns the boxes do not cover (the cyclic wrap, a tile's end, range row-support edges): coalesced stores
      if (remw[(d * NR + r0) >> 5]) {
#pragma unroll 1
        for (int u = 0; u < RW; ++u) {
          const RowInfo ri = inf[r0 + u];
          if (ri.mlo >= ri.mhi) continue;
          A* drow = static_cast<A*>(D.ptr) + (int64_t)ri.orow * D.pitch;
          const A* srow = stg + u * pitch;
          const int xs0 = X - (WO2 - so[dense ? 0 : r0 + u]), d0 = ri.d0 & ~kTmaBit;
          for (int x = ri.mlo + lane; x < ri.mhi; x += 32) {
            int col = d0 + (x - xs0);
            if (col >= p.W) col -= p.W;
            FHT_CHECK(col >= 0 && col < p.W && ri.orow >= 0 && ri.orow < D.nrows && x - xs0 >= 0 && x - xs0 < pitch);
            __stcs(drow + col, srow[x - xs0]);
          }
        }
      }
    }
    pdl_trigger();
    if (lane == 0 && issued) tma_wait_read();
    return !black;
  }
#endif
  // ---- stores, one destination at a time (the staging plane is reused)
  bool issued = false;
  for (int dd = 0; dd < p.ndest; ++dd) {
    const int d = FHT_P2_REVERSE_DEST ? p.ndest - 1 - dd : dd;
    const P2Dest& D = p.dest[d];
    const RowInfo* inf = info + d * NR;
    const int* so = soff + d * 64;
    if (dd > 0) {
      if (issued) tma_wait_read();
      grp.sync();
    }
    // plain destination of an interior QUADS tile: every row has the same aligned start and no
    // remainder, rows ascend -> ONE 2-D box {box, NR} from a dense [NR][box] staging plane
    const bool dense = FHT_P2_DENSE && !p.range && !D.shifted && sl.rsign == 1 && (sl.skip < t0 || sl.skip > tmax) &&
                       tmax < p.rows_out &&
                       (inf[0].d0 & kTmaBit) && inf[0].mlo >= inf[0].mhi;
    const int pitch = dense ? box : ST_PITCH;
    // the dense plane is the 2-D box itself (predicated staging); row planes start kStgOff elements in, with slack
    // around every row, and stage without predicates
    A* const stg = (dense || !FHT_P2_UNPRED) ? buf : buf + kStgOff;
    if (!black) {
      if (dense && FHT_P2_DENSE_MASK)  // one aligned start for all rows: the in-box flags once per lane
        stage_rows<R, SIG, A, A, G, 3>(grp, w, stg, so, pitch, pitch);
      else if (dense || !FHT_P2_UNPRED)
        stage_rows<R, SIG, A>(grp, w, stg, so, pitch, pitch);  // every computed column that fits the row
      else
        stage_rows<R, SIG, A, A, G, 0>(grp, w, stg, so, pitch, pitch);
    } else {  // every output of a black tile is 0 (no pattern touches a pixel)
      // 16-byte stores (both planes start 16-byte aligned; NR * pitch is a multiple of 4: pitch is)
      float4* z4 = reinterpret_cast<float4*>(stg);
      for (int idx = tid; idx < (NR * pitch) >> 2; idx += NT) z4[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      grp.sync();
    }
    if (dense) {
      if (tid == 0) {
        FHT_CHECK(inf[0].orow >= 0 && inf[0].orow + NR <= D.nrows);
        tma_store_row_stream(tm0_box, buf, inf[0].d0 & ~kTmaBit, inf[0].orow);  // box {box, NR}
        tma_commit();
        issued = true;
      }
    } else {
      if (tid < NR && (inf[tid].d0 & kTmaBit)) {  // one row store per thread
        const RowInfo ri = inf[tid];
        FHT_CHECK((ri.d0 & ~kTmaBit) >= 0 && (ri.d0 & ~kTmaBit) < p.W && ri.orow >= 0 && ri.orow < D.nrows);
        tma_store_row_stream(d == 0 ? tm0 : tm1, stg + tid * ST_PITCH, ri.d0 & ~kTmaBit, ri.orow);  // clipped at W
        tma_commit();
        issued = true;
      }
      for (int tau = warp; tau < NR; tau += NW) {
        const RowInfo ri = inf[tau];
        if (ri.mlo >= ri.mhi) continue;
        A* drow = static_cast<A*>(D.ptr) + (int64_t)ri.orow * D.pitch;
        const A* srow = stg + tau * ST_PITCH;
        const int xs0 = X - (WO2 - so[tau]), d0 = ri.d0 & ~kTmaBit;
        for (int x = ri.mlo + lane; x < ri.mhi; x += 32) {
          int col = d0 + (x - xs0);
          if (col >= p.W) col -= p.W;
          FHT_CHECK(col >= 0 && col < p.W && ri.orow >= 0 && ri.orow < D.nrows && x - xs0 >= 0 && x - xs0 < ST_PITCH);
          __stcs(drow + col, srow[x - xs0]);
        }
      }
    }
  }
  pdl_trigger();
  if (issued) tma_wait_read();
  return !black;
}

// tm_scr0: scratch, one row x 256 columns; tm_scr1: one row x 36 columns; tm0 / tm1: destinations
// (one-row boxes); tm0_box: destination 0 with box {TX + 4, 2^R} (dense interior tiles)
template <typename A, int R, typename Tscr = A>
__global__ void __launch_bounds__(Split<R>::nw * 32, kMinBlocks<R>)
k_p2(const __grid_constant__ CUtensorMap tm_scr0, const __grid_constant__ CUtensorMap tm_scr1,
     const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1,
     const __grid_constant__ CUtensorMap tm0_box, const __grid_constant__ P2Params p) {
  pdl_wait();  // pass 1 (the predecessor) has written the scratch
  // flat grid, tile fastest: CTAs running together read overlapping scratch rows (L2 reuse of
  // the 72-column halo and of the sheared rows of one group)
  // grid (ntiles, groups, images * nq): no integer division
  const int n = blockIdx.x;
  const int jl = blockIdx.y;  // the launch's group index; j = j0 + jl is the transform's
  const int j = p.j0 + jl;
  const int qi = blockIdx.z & ((1 << p.nq_log) - 1);
  const int img = p.img0 + (blockIdx.z >> p.nq_log);
  const P2Slot& sl = p.slot[qi];
  if (n >= sl.ntiles) return;
  // tile n of part [lo, hi): X = lo + TX*k, owning TX columns; the last tile of a part sits at
  // hi - (TX + 4) and owns the rest, so its 16-byte aligned store box ends inside the part
  const bool pa = n < sl.ntiles_a;
  int lo = pa ? sl.xbeg : sl.xmid, nk = pa ? sl.ntiles_a : sl.ntiles - sl.ntiles_a;
  const int hi = pa ? sl.xmid : sl.xend;
  const int k = pa ? n : n - sl.ntiles_a;
  if (p.range) {
    // §4 frame: start_s = min_y (e_y - D_s(y)) is non-increasing in s (D_s(y) is) and
    // D_s(y) <= Dmax(s) = sum_q ceil((s >> q) / 2), so no row t <= tmax of group j stores left of
    // e_min - Dmax(tmax) (e_min = xbeg + Hp - 1): the group's tiles start there
    const int tmax = (j << R) + (1 << R) - 1;
    int dm = 0;
    for (int s2 = tmax; s2 > 0; s2 >>= 1) dm += (s2 + 1) >> 1;
    lo = max(lo, sl.xbeg + p.Hp - 1 - dm);
    const int boxw = p.TX + WO2;
    nk = hi <= lo ? 0 : (hi - lo <= boxw ? 1 : 1 + (hi - lo - boxw + p.TX - 1) / p.TX);
    if (k >= nk) return;
  }
  const int X = k + 1 < nk ? lo + p.TX * k : max(lo, hi - (p.TX + WO2));
  const int own = k + 1 < nk ? p.TX : hi - X;
  // scratch row of (group j, strip 0): [z][j_local][strip] with p.logS strip bits per chunk
  const int64_t rbase = p.row0 + (int64_t)(img - p.img0) * p.scratch_img_rows + sl.srow0 + ((int64_t)jl << p.logS);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  if (sl.sigma > 0)
    p2_body<A, R, 1, Tscr>(GrpAll{}, smem_raw, &tm_scr0, &tm_scr1, &tm0, &tm1, &tm0_box, p, sl, img, j, X, own, rbase);
  else
    p2_body<A, R, -1, Tscr>(GrpAll{}, smem_raw, &tm_scr0, &tm_scr1, &tm0, &tm1, &tm0_box, p, sl, img, j, X, own, rbase);
}

// The 2^R-row pass-2 tile on a CTA pair (cluster dims {2, 1, 1}, blockIdx.x = 2 * tile + rank): half the
// shared memory and warps of k_p2<R> per CTA, so a 64-row tile keeps five CTAs of four warps per SM instead of
// two of eight ("Cluster pass 2"). Both CTAs of a pair take the same early exits.
template <int R> constexpr size_t p2c_smem_bytes() { return main_buf_bytes(R) / 2 + kTableBytes + (size_t)(1 << R) * 16; }
template <typename A, int R, typename Tscr = A>
__global__ void __launch_bounds__(Split<R>::nw * 16, 5)
k_p2c(const __grid_constant__ CUtensorMap tm_scr0, const __grid_constant__ CUtensorMap tm_scr1,
      const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1,
      const __grid_constant__ CUtensorMap tm0_box, const __grid_constant__ P2Params p) {
  pdl_wait();
  const int n = blockIdx.x >> 1;
  const int jl = blockIdx.y;
  const int j = p.j0 + jl;
  const int qi = blockIdx.z & ((1 << p.nq_log) - 1);
  const int img = p.img0 + (blockIdx.z >> p.nq_log);
  const P2Slot& sl = p.slot[qi];
  if (n >= sl.ntiles) return;
  const bool pa = n < sl.ntiles_a;
  int lo = pa ? sl.xbeg : sl.xmid, nk = pa ? sl.ntiles_a : sl.ntiles - sl.ntiles_a;
  const int hi = pa ? sl.xmid : sl.xend;
  const int k = pa ? n : n - sl.ntiles_a;
  if (p.range) {  // as k_p2
    const int tmax = (j << R) + (1 << R) - 1;
    int dm = 0;
    for (int s2 = tmax; s2 > 0; s2 >>= 1) dm += (s2 + 1) >> 1;
    lo = max(lo, sl.xbeg + p.Hp - 1 - dm);
    const int boxw = p.TX + WO2;
    nk = hi <= lo ? 0 : (hi - lo <= boxw ? 1 : 1 + (hi - lo - boxw + p.TX - 1) / p.TX);
    if (k >= nk) return;
  }
  const int X = k + 1 < nk ? lo + p.TX * k : max(lo, hi - (p.TX + WO2));
  const int own = k + 1 < nk ? p.TX : hi - X;
  const int64_t rbase = p.row0 + (int64_t)(img - p.img0) * p.scratch_img_rows + sl.srow0 + ((int64_t)jl << p.logS);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  if (sl.sigma > 0)
    p2_body<A, R, 1, Tscr, GrpAll, 2>(GrpAll{}, smem_raw, &tm_scr0, &tm_scr1, &tm0, &tm1, &tm0_box, p, sl, img, j, X,
                                      own, rbase);
  else
    p2_body<A, R, -1, Tscr, GrpAll, 2>(GrpAll{}, smem_raw, &tm_scr0, &tm_scr1, &tm0, &tm1, &tm0_box, p, sl, img, j, X,
                                       own, rbase);
}

}  // namespace v2
}  // namespace fht
