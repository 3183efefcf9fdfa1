// fht_p1p.cuh -- persistent pass 1 for 64-row strips of 4-byte images (k_p1p; DESIGN.md §4 "Persistent pass 1").
//
// k_p1 runs one tile per CTA: launch, TMA issue, DRAM latency, sub-passes A and B, staging, the scratch store and
// its drain are one dependent chain, and with two 8-warp CTAs per SM (the 80 KB plane of a 64-row tile) an SM often
// holds a single computing CTA. Here a CTA walks tiles T = blockIdx.x, + gridDim.x, ... (two CTAs per SM; gridDim.x
// is a multiple of the slot count, so a CTA stays on one quadrant slot: one sign, one fill path) and
//   * issues the NEXT tile's loads as soon as every warp holds its sub-pass-B inputs in registers (a CTA barrier
//     after sub-pass B's shared-memory reads, BEFORE its butterflies):
//     non-transposed slots one TMA box {32, 10, 8 rows} per warp (its own sub-pass-A block, its own mbarrier, phase
//     parity alternating per tile); transposed slots (FHT row = image column) four TMA boxes {32 image columns, 144
//     image rows} with the 128-byte swizzle: the block lands UNtransposed, and sub-pass A reads a lane's column e of
//     its 8 FHT rows (8 consecutive image columns = two 16-byte chunks of image row e) with two 16-byte loads -- the
//     swizzle (chunk ^ (row & 7)) makes the eight lanes of a quarter-warp, whose rows e = 9 lane + q differ mod 8,
//     hit eight different chunks: conflict-free, 18 loads per lane instead of 72. The transposition is index
//     arithmetic; a CTA barrier separates those reads from the in-place sub-pass-A stores. (4-byte
//     cp.async copies that transpose on the way in measured 1.45x slower than k_p1's vector fill.)
//   * stages the results outside the plane: every warp owns the 8 rows of its sub-pass-B group and writes them in
//     two halves through its own [4][TX] slot (3456 B), one bulk store {TX, 1, 4, 1} per half, waiting only for its
//     own previous bulk read. No CTA barrier after sub-pass B's, no drain before the next tile.
// The arithmetic is tile_fht_ld's (warp_fht on the same operands in the same order as k_p1): bit-identical results.
#pragma once
#include "fht_tile.cuh"

#ifndef FHT_P1P_HALF0_STG
#define FHT_P1P_HALF0_STG 0  // A/B (measured slower: C5 pass 1 381 vs 341 us): first half of a warp's rows: read back from its slot and stored with 16-byte st.global
#endif                       // (no bulk-read wait before the second half is staged); second half: bulk store
#ifndef FHT_P1P_TR_SPLIT
#define FHT_P1P_TR_SPLIT 1  // transposed slots: one mbarrier (and one issuing thread) per column half of the tile
#endif
#ifndef FHT_P1P_LOAD_AFTER_STORE0
#define FHT_P1P_LOAD_AFTER_STORE0 0  // measured: C5 pass 1 343 us (0) vs 354 us (1)
#endif

namespace fht {
namespace v2 {

constexpr int kP1pHalf = 4;                                                  // rows per staged half
constexpr size_t kP1pStageBytes = (size_t)8 * kP1pHalf * TX1 * 4;            // 8 warps x [4][216] x 4 B = 27648
// tail: 128 B (mbarriers), then the §4 range loader's tables: rowoff[64], erow[64], {cm_lo, cm_n}, colmap slice [512]
constexpr size_t kP1pRangeBytes = 64 * 4 + 64 * 4 + 64 + kColmapStageBytes;
__host__ __device__ constexpr size_t p1p_smem_bytes(bool range = false) {
  return main_buf_bytes(6) + kP1pStageBytes + 128 + (range ? kP1pRangeBytes : 0);
}

constexpr int kP1pBoxRows = 144;                                 // transposed slots: image rows per TMA box
constexpr uint32_t kP1pBoxBytes = kP1pBoxRows * 128;             // {32 columns, 144 rows} x 4 B = 18432 (18 x 1024)

struct P1pTile {
  int X, strip, img_l;
};

// One CTA's tiles of slot `sl` (sign SIG, transposed TR). tm_img8: the image view [img][row][col/32][32] with box
// {32, 10, 8, 1}; tm_imgS: the image [img][row][col] with box {32, 144, 1} and the 128-byte swizzle; tm_dst4: the
// scratch view [z][j][strip][column] with box {TX, 1, 4, 1}.
// RG: the §4 range loader (sigma = +1, not transposed): rows by TMA from the aligned-down column of
// colmap[max(0, Xa - e_y)] (tm_img8 / tm_imgS are then the 3-D image maps with boxes of 256 and 36 columns), the
// transform T(x', y) = I[y][colmap[x' - e_y]] gathered from shared memory in sub-pass A, as in p1_body.
template <typename Tin, int SIG, bool TR, bool RG = false>
__device__ __forceinline__ void p1p_run(unsigned char* smem, const CUtensorMap* tm_img8, const CUtensorMap* tm_imgS,
                                        const CUtensorMap* tm_dst4, const P1Params& p, const P1Slot& sl, int qi,
                                        int total, void* scr, int64_t scr_pitch) {
  using A = typename AccOf<Tin>::type;
  static_assert(sizeof(Tin) == 4 && sizeof(A) == 4, "4-byte images");
  constexpr int R = 6, NA = 1 << Split<R>::a, NR = 1 << R;
  static_assert(Split<R>::nw == 8 && NA == 8 && (1 << Split<R>::b) == 8, "one sub-pass-A block and one B group per warp");
  constexpr int PITCH = TMA_PITCH;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  A* plane = reinterpret_cast<A*>(smem);
  A* stg = reinterpret_cast<A*>(smem + main_buf_bytes(R)) + warp * (kP1pHalf * TX1);
  // non-transposed: one mbarrier per warp (its block's rows); transposed: one for the tile's four boxes
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + main_buf_bytes(R) + kP1pStageBytes) + (TR ? 8 + (FHT_P1P_TR_SPLIT ? (warp >> 2) : 0) : warp);
  const int ntq = p.ntiles << p.nq_log;
  const int G = (int)gridDim.x;

  auto decode = [&](int T, P1pTile& t) -> bool {
    const int rest = T / ntq, x = T - rest * ntq;
    const int n = x >> p.nq_log;
    if (n >= sl.ntiles) return false;
    t.X = min(sl.xlo + p.TX * n, sl.xhi - p.TX);
    t.strip = rest & ((1 << p.L) - 1);
    t.img_l = rest >> p.L;
    return true;
  };
  auto next = [&](int T, P1pTile& t) {
    do {
      T += G;
    } while (T < total && !decode(T, t));
    return T;
  };
  // §4 range tables (shared memory tail)
  int* rowoff = reinterpret_cast<int*>(smem + main_buf_bytes(R) + kP1pStageBytes + 128);  // [64] a0 or kNoRow
  int* erow = rowoff + 64;                                                                 // [64] e_y
  int* cmhdr = erow + 64;                                                                  // cm_lo, cm_n
  int* cm_s = cmhdr + 16;                                                                  // colmap[cm_lo + i]
  // loads of a tile into the plane (free: every warp is past sub-pass B's reads); RG: also the tile's tables, and
  // the return value says whether any row of the tile has content (CTA-uniform; ends with a CTA barrier)
  auto issue = [&](const P1pTile& t) -> bool {
    const int Xa = SIG > 0 ? t.X : t.X - (WA - WC);
    const int y0 = (p.strip0 + t.strip) * NR;
    const int img = p.img0 + t.img_l;
    if constexpr (RG) {
      const int rho = warp * NA + lane, y = y0 + rho;
      int a0 = kNoRow, e = 0;
      bool ne = false;
      if (lane < NA) {
        if (y < p.img_h) {
          e = __ldg(p.e_tab + y);
          const int u0 = Xa - e;
          if (u0 < p.w_content && u0 + WA > 0) {
            a0 = __ldg(p.colmap + max(0, u0)) & ~3;
            ne = true;
          }
        }
        rowoff[rho] = a0;
        erow[rho] = e;
      }
      const unsigned m = __ballot_sync(0xffffffffu, ne);
      if (lane == 0) mbar_expect_tx(bar, (uint32_t)__popc(m) * (256 + 36) * 4);
      __syncwarp();
      if (ne) {
        A* d = plane + rho * TMA_PITCH;
        tma_load_3d(tm_img8, d, bar, a0, y, img);
        tma_load_3d(tm_imgS, d + 256, bar, a0 + 256, y, img);
      }
      // the strip's colmap slice (e_y is monotonic in y: the u range comes from the first and last rows)
      int ulo = 0, n = 0;
      if (y0 < p.img_h) {
        const int ea = __ldg(p.e_tab + y0), eb = __ldg(p.e_tab + min(y0 + NR - 1, p.img_h - 1));
        ulo = max(0, Xa - max(ea, eb));
        n = max(0, min(p.w_content, Xa + WA - min(ea, eb)) - ulo);
      }
      if (n <= kColmapStage)
        for (int i = tid; i < n; i += 256) cm_s[i] = __ldg(p.colmap + ulo + i);
      if (tid == 0) {
        cmhdr[0] = ulo;
        cmhdr[1] = n;
      }
      return __syncthreads_or(m != 0u) != 0;
    } else if constexpr (!TR) {
      if (lane == 0) {
        mbar_expect_tx(bar, (uint32_t)NA * TMA_PITCH * 4);
        tma_load_4d(tm_img8, plane + warp * NA * TMA_PITCH, bar, 0, (Xa & ~31) >> 5, y0 + warp * NA, img);
      }
      return true;
    } else {
      // image rows [Xa, Xa + 288) x image columns [y0, y0 + 64): box (hb, rb) = columns y0 + 32 hb.., rows Xa + 144 rb..
#if FHT_P1P_TR_SPLIT
      // one mbarrier per column half: warps 0-3 read only the boxes of columns y0 .. y0 + 31, warps 4-7 the others
      if ((tid & 127) == 0) {
        const int hb = tid >> 7;
        mbar_expect_tx(bar, 2u * kP1pBoxBytes);
#pragma unroll
        for (int rb = 0; rb < 2; ++rb)
          tma_load_3d(tm_imgS, smem + (2 * hb + rb) * kP1pBoxBytes, bar, y0 + 32 * hb, Xa + kP1pBoxRows * rb, img);
      }
#else
      if (tid == 0) {
        mbar_expect_tx(bar, 4u * kP1pBoxBytes);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tma_load_3d(tm_imgS, smem + k * kP1pBoxBytes, bar, y0 + 32 * (k >> 1), Xa + kP1pBoxRows * (k & 1), img);
      }
#endif
      return true;
    }
  };

  if constexpr (!TR) {
    if (lane == 0) mbar_init(bar);
    __syncwarp();
  } else {
    if ((tid & (FHT_P1P_TR_SPLIT ? 127 : 255)) == 0) mbar_init(bar);
    __syncthreads();
  }
  int T = (int)blockIdx.x;
  P1pTile cur{}, nxt{};
  if (T < total && !decode(T, cur)) T = next(T, cur);
  if (T < total) {
    bool cur_any = issue(cur), nxt_any = false;
    uint32_t par = 0;
    while (true) {
      const int Tn = next(T, nxt);
      const bool more = Tn < total;
      const int Xa = SIG > 0 ? cur.X : cur.X - (WA - WC);
      A w[1][1 << Split<R>::b][VB];
      mbar_wait(bar, par);  // (a range tile without content: its warps' empty phases complete at once)
      const bool any = !RG || cur_any;  // (compile-time true outside the range loader)
      if (any) {
        // ---- sub-pass A: block = warp, rows warp * 8 + r; v[r][q] = input (row, x-order index e), e = lane * 9 + q
        // (SIG = +1) or 287 - lane * 9 - q (SIG = -1): the local frame of tile_fht_ld
        A v[NA][VA];
        if constexpr (RG) {
          const int cm_lo = cmhdr[0], cm_n = cmhdr[1];
#pragma unroll
          for (int r = 0; r < NA; ++r) {
            const int rho = warp * NA + r;
            const int a0 = rowoff[rho], u0 = cur.X + lane * VA - erow[rho];
#pragma unroll
            for (int q = 0; q < VA; ++q) {
              const int u = u0 + q;
              A val = A(0);
              if (a0 != kNoRow && (unsigned)u < (unsigned)p.w_content) {
                const int c = cm_n <= kColmapStage ? cm_s[u - cm_lo] : __ldg(p.colmap + u);
                FHT_CHECK(c - a0 >= 0 && c - a0 < 256 + 36 && (cm_n > kColmapStage || (u - cm_lo >= 0 && u - cm_lo < cm_n)));
                val = plane[rho * PITCH + (c - a0)];
              }
              v[r][q] = val;
            }
          }
        } else if constexpr (!TR) {
          const int rowoff = Xa & 31;
#pragma unroll
          for (int r = 0; r < NA; ++r) {
            const A* q0 = plane + (warp * NA + r) * PITCH + rowoff + (SIG > 0 ? lane * VA : (WA - 1) - lane * VA);
            FHT_CHECK((SIG > 0 ? q0 : q0 - (VA - 1)) >= plane + (warp * NA + r) * PITCH &&
                      (SIG > 0 ? q0 + VA : q0 + 1) <= plane + (warp * NA + r + 1) * PITCH);
#pragma unroll
            for (int q = 0; q < VA; ++q) v[r][q] = q0[SIG > 0 ? q : -q];
          }
          // in place: the warp has read all rows of its block (its own TMA box) before it overwrites them
        } else {
          // from the untransposed, swizzled block: FHT rows warp * 8 + r = image columns = chunks ch, ch + 1 of box
          // column hb; FHT column e = image row e
          const uint32_t base = smem_u32(smem) + (uint32_t)(warp >> 2) * 2u * kP1pBoxBytes;
          const uint32_t ch = (2u * (uint32_t)warp) & 7u;
#pragma unroll
          for (int q = 0; q < VA; ++q) {
            const int e = SIG > 0 ? lane * VA + q : (WA - 1) - lane * VA - q;
            const int rb = e >= kP1pBoxRows ? 1 : 0, er = e - rb * kP1pBoxRows;
            const uint32_t a0 = base + (uint32_t)rb * kP1pBoxBytes + (uint32_t)er * 128u + ((ch ^ ((uint32_t)er & 7u)) << 4);
            FHT_CHECK(e >= 0 && e < WA && (a0 & 15u) == 0 && a0 >= smem_u32(smem) &&
                      (a0 | 16u) + 16u <= smem_u32(smem) + 4u * kP1pBoxBytes);
            uint32_t x[8];
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]) : "r"(a0) : "memory");
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]) : "r"(a0 ^ 16u) : "memory");
#pragma unroll
            for (int r = 0; r < NA; ++r) {
              if constexpr (std::is_same<A, float>::value)
                v[r][q] = __uint_as_float(x[r]);
              else
                v[r][q] = static_cast<A>(x[r]);
            }
          }
          __syncthreads();  // every warp has read the block: sub-pass A's rows overwrite it
        }
        warp_fht<Split<R>::a, VA>(v);
        A* d = plane + (warp * NA) * PITCH + lane * VA;
        FHT_CHECK(d + (NA - 1) * PITCH + VA <= plane + NR * PITCH && lane * VA + VA <= PITCH);
#pragma unroll
        for (int r = 0; r < NA; ++r)
#pragma unroll
          for (int q = 0; q < VA; ++q) d[r * PITCH + q] = v[r][q];
        __syncthreads();
        // ---- sub-pass B (as tile_fht_ld): group jp = warp reads row jp of every block at column c + jp * i
#pragma unroll
        for (int i = 0; i < NA; ++i) {
          const A* sp = plane + (i * NA + warp) * PITCH + lane * VB + warp * i;
          FHT_CHECK(lane * VB + warp * i + VB <= WA && sp + VB <= plane + NR * PITCH);
#pragma unroll
          for (int q = 0; q < VB; ++q) w[0][i][q] = sp[q];
        }
      } else {  // (range) no row of the tile has content: F_m is 0 over the whole tile
#pragma unroll
        for (int i = 0; i < NA; ++i)
#pragma unroll
          for (int q = 0; q < VB; ++q) w[0][i][q] = A(0);
      }
      // The next tile's TMA loads overwrite the plane through the async proxy: each thread orders its (possibly still
      // in-flight) shared-memory reads before them with a proxy fence, the barrier makes that cumulative. Without the
      // fence the equality test failed about once in three runs (a bulk copy overtaking queued ld.shared).
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();  // every warp holds its sub-pass-B inputs in registers: the plane is free
      par ^= 1u;
#if !FHT_P1P_LOAD_AFTER_STORE0
      if (more) nxt_any = issue(nxt);  // the next tile's loads fly during the sub-pass-B butterflies and the stores
#endif
      if (any) warp_fht<Split<R>::b, VB>(w[0]);
      // ---- the warp's 8 rows tau = warp * 8 + u, in two halves through its slot
      const int Xs = cur.X - sl.xlo, zscr = p.z0 + cur.img_l * p.nq + qi;
      FHT_CHECK(Xs >= 0 && Xs + p.TX <= sl.xhi - sl.xlo && p.TX == TX1 && (Xs & 3) == 0 && zscr >= 0 &&
                cur.strip >= 0 && cur.strip < (1 << p.L));
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        if (half == 0 || !FHT_P1P_HALF0_STG) {
          if (lane == 0) tma_wait_read();  // the slot's previous bulk store has read it
          __syncwarp();
        }
        if (lane < 31) {
          const int lo = SIG > 0 ? lane * VB : (WC - VB) - lane * VB;
#pragma unroll
          for (int u = 0; u < kP1pHalf; ++u) {
            A* d = stg + u * TX1 + lo;
            // (pointer ranges, not smem_in_bounds: its %total_smem_size bound does not count the 1 KB the system
            // reserves below the dynamic window, and the slots reach the window's last kilobyte)
            FHT_CHECK(lo >= 0 && lo + VB - 1 <= TX1 && d >= stg && d + VB - 1 <= stg + kP1pHalf * TX1 &&
                      reinterpret_cast<unsigned char*>(stg + kP1pHalf * TX1) <= smem + main_buf_bytes(R) + kP1pStageBytes);
#pragma unroll
            for (int q = 0; q < VB - 1; ++q) d[q] = w[0][half * kP1pHalf + u][SIG > 0 ? q : VB - 1 - q];
            if (lo + VB - 1 < TX1) d[VB - 1] = w[0][half * kP1pHalf + u][SIG > 0 ? VB - 1 : 0];
          }
        }
        if (FHT_P1P_HALF0_STG && half == 0) {
          // rows j = warp * 8 + u of F_m[strip] at scratch row (z * 64 + j) * strips + strip, columns [Xs, Xs + TX):
          // 54 aligned 16-byte groups per row, read back from the slot (conflict-free) and stored coalesced
          __syncwarp();
          const int64_t srow = ((int64_t)zscr * NR + warp * 8) << p.L;
#pragma unroll
          for (int u0 = 0; u0 < kP1pHalf; u0 += 2) {  // two rows in flight (16 registers)
            uint4 g[2][2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const uint4* sv = reinterpret_cast<const uint4*>(stg + (u0 + u) * TX1);
              g[u][0] = sv[lane];
              if (lane < TX1 / 4 - 32) g[u][1] = sv[lane + 32];
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              uint4* gv = reinterpret_cast<uint4*>(static_cast<A*>(scr) +
                                                   (srow + ((int64_t)(u0 + u) << p.L) + cur.strip) * scr_pitch + Xs);
              gv[lane] = g[u][0];
              if (lane < TX1 / 4 - 32) gv[lane + 32] = g[u][1];
            }
          }
          __syncwarp();  // every lane has read the slot before the second half is staged
          continue;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
#if FHT_SCR_KEEP
          tma_store_4d_keep(tm_dst4, stg, Xs, cur.strip, warp * 8 + half * kP1pHalf, zscr);
#else
          tma_store_4d(tm_dst4, stg, Xs, cur.strip, warp * 8 + half * kP1pHalf, zscr);
#endif
          tma_commit();
        }
#if FHT_P1P_LOAD_AFTER_STORE0
        // A/B: the next tile's loads behind the first half's store (so that store's shared-memory read, which the
        // second half waits for, is not queued behind 80 KB of loads): slower, the loads' head start matters more
        if (half == 0 && more) nxt_any = issue(nxt);
#endif
      }
      if (!more) break;
      T = Tn;
      cur = nxt;
      cur_any = nxt_any;
    }
  }
  pdl_trigger();
  if (lane == 0) tma_wait_read();
}

template <typename Tin>
__global__ void __launch_bounds__(256, 2)
k_p1p(const __grid_constant__ CUtensorMap tm_img8, const __grid_constant__ CUtensorMap tm_imgS,
      const __grid_constant__ CUtensorMap tm_dst4, const __grid_constant__ P1Params p, int total, void* scr,
      int64_t scr_pitch) {
  pdl_wait();  // the image may come from the previous kernel; the scratch may still be read by it
  extern __shared__ __align__(1024) unsigned char smem_p1p[];  // swizzled boxes: 1024-byte aligned
  const int qi = blockIdx.x & ((1 << p.nq_log) - 1);  // gridDim.x % nq == 0: every tile of this CTA is slot qi's
  const P1Slot& sl = p.slot[qi];
  if (p.range) {  // §4 range frame: sigma = +1, not transposed; tm_img8 / tm_imgS: the 256- and 36-column row maps
    p1p_run<Tin, 1, false, true>(smem_p1p, &tm_img8, &tm_imgS, &tm_dst4, p, sl, qi, total, scr, scr_pitch);
  } else if (!sl.transposed) {
    if (sl.sigma > 0)
      p1p_run<Tin, 1, false>(smem_p1p, &tm_img8, &tm_imgS, &tm_dst4, p, sl, qi, total, scr, scr_pitch);
    else
      p1p_run<Tin, -1, false>(smem_p1p, &tm_img8, &tm_imgS, &tm_dst4, p, sl, qi, total, scr, scr_pitch);
  } else {
    if (sl.sigma > 0)
      p1p_run<Tin, 1, true>(smem_p1p, &tm_img8, &tm_imgS, &tm_dst4, p, sl, qi, total, scr, scr_pitch);
    else
      p1p_run<Tin, -1, true>(smem_p1p, &tm_img8, &tm_imgS, &tm_dst4, p, sl, qi, total, scr, scr_pitch);
  }
}

}  // namespace v2
}  // namespace fht
