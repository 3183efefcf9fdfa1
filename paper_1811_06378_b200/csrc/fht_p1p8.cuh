// fht_p1p8.cuh -- persistent pass 1 for 16-row strips of u8 images (k_p1p8; DESIGN.md §4 "Persistent pass 1").
//
// The u8 counterpart of k_p1p for the small tiles of C3-like batches (Hp = 256 / 512: m = 4, 24576 tiles of 16 rows
// for C3, each ~500 instructions per warp, so k_p1's per-CTA launch, TMA issue, load latency and store drain are most
// of a tile's life). Six 4-warp CTAs per SM walk the tiles (a CTA stays on one quadrant slot). The u8 rows land in
// their own area, apart from the int plane of sub-pass-A results, so
//   * non-transposed slots: a warp re-arms and re-issues its own TMA box {128, 4, 4 rows} of the [row][col/128][128]
//     view for the NEXT tile as soon as it has read the current rows into registers (a whole tile ahead);
//   * transposed slots: two boxes {16 image columns, 144 image rows} land untransposed ([288][16] bytes); a lane's
//     column e of its warp's 4 FHT rows is ONE 32-bit word of image row e (the transposition is index arithmetic,
//     SURVEY a1); the next tile's boxes are issued after the CTA barrier that follows everyone's reads;
//   * a warp's 4 result rows (uint16 scratch) go through its own [4][TX] slot and one bulk store
//     {TX, 1, 4, 1}; the slot's previous store was issued a tile ago, so its read-wait is free.
// The arithmetic is warp_fht on the same operands in the same order as k_p1<uint8_t, 4>: bit-identical results.
#pragma once
#include "fht_tile.cuh"
#include "fht_p1p.cuh"

namespace fht {
namespace v2 {

constexpr int kP8InPitch = 512;                                      // landing pitch of a u8 row (box {128, 4})
constexpr size_t kP8PlaneBytes = (size_t)16 * TMA_PITCH * 4;         // 20480: sub-pass-A results (int)
constexpr size_t kP8InBytes = (size_t)16 * kP8InPitch;               // 8192 (transposed: [288][16] = 4608 used)
constexpr size_t kP8SlotBytes = 1792;                                // [4][216] uint16 = 1728, 128-byte multiple
constexpr size_t kP8StageBytes = 4 * kP8SlotBytes;
__host__ __device__ constexpr size_t p1p8_smem_bytes() { return kP8PlaneBytes + kP8InBytes + kP8StageBytes + 64; }

template <int SIG, bool TR>
__device__ __forceinline__ void p1p8_run(unsigned char* smem, const CUtensorMap* tm_img128, const CUtensorMap* tm_imgT,
                                         const CUtensorMap* tm_dst4, const P1Params& p, const P1Slot& sl, int qi,
                                         int total) {
  constexpr int R = 4, NA = 4, NR = 16, NW = 4;
  static_assert(Split<R>::a == 2 && Split<R>::b == 2 && Split<R>::nw == NW, "one sub-pass-A block and one B group per warp");
  constexpr int PITCH = TMA_PITCH;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int* plane = reinterpret_cast<int*>(smem);
  uint8_t* in8 = smem + kP8PlaneBytes;
  uint16_t* stg = reinterpret_cast<uint16_t*>(smem + kP8PlaneBytes + kP8InBytes + warp * kP8SlotBytes);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kP8PlaneBytes + kP8InBytes + kP8StageBytes) + (TR ? 4 : warp);
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
  // the warp's own box (non-transposed) or the tile's two boxes (transposed, thread 0)
  auto issue = [&](const P1pTile& t) {
    const int Xa = SIG > 0 ? t.X : t.X - (WA - WC);
    const int y0 = (p.strip0 + t.strip) * NR;
    const int img = p.img0 + t.img_l;
    if constexpr (!TR) {
      if (lane == 0) {
        mbar_expect_tx(bar, (uint32_t)NA * kP8InPitch);
        tma_load_4d(tm_img128, in8 + warp * NA * kP8InPitch, bar, 0, (Xa & ~127) >> 7, y0 + warp * NA, img);
      }
    } else {
      if (tid == 0) {
        mbar_expect_tx(bar, 2u * 144u * 16u);
        tma_load_3d(tm_imgT, in8, bar, y0, Xa, img);
        tma_load_3d(tm_imgT, in8 + 144 * 16, bar, y0, Xa + 144, img);
      }
    }
  };

  if constexpr (!TR) {
    if (lane == 0) mbar_init(bar);
    __syncwarp();
  } else {
    if (tid == 0) mbar_init(bar);
    __syncthreads();
  }
  int T = (int)blockIdx.x;
  P1pTile cur{}, nxt{};
  if (T < total && !decode(T, cur)) T = next(T, cur);
  if (T < total) {
    issue(cur);
    uint32_t par = 0;
    while (true) {
      const int Tn = next(T, nxt);
      const bool more = Tn < total;
      const int Xa = SIG > 0 ? cur.X : cur.X - (WA - WC);
      int w[NA][VB];
      {
        // ---- sub-pass A: block = warp, FHT rows warp * 4 + r; v[r][q] = input at x-order index e = lane * 9 + q
        // (SIG = +1) or 287 - lane * 9 - q (SIG = -1)
        int v[NA][VA];
        mbar_wait(bar, par);
        if constexpr (!TR) {
          const int rowoff = Xa & 127;
#pragma unroll
          for (int r = 0; r < NA; ++r) {
            const uint8_t* q0 = in8 + (warp * NA + r) * kP8InPitch + rowoff + (SIG > 0 ? lane * VA : (WA - VA) - lane * VA);
            FHT_CHECK(q0 >= in8 + (warp * NA + r) * kP8InPitch && q0 + 12 <= in8 + (warp * NA + r + 1) * kP8InPitch);
            uint32_t e[VA];
            load9_narrow<uint8_t>(q0, e);
#pragma unroll
            for (int q = 0; q < VA; ++q) v[r][q] = (int)e[SIG > 0 ? q : VA - 1 - q];
          }
        } else {
          // image row e holds the warp's 4 FHT rows (image columns y0 + 4 warp ..) as one 32-bit word
#pragma unroll
          for (int q = 0; q < VA; ++q) {
            const int e = SIG > 0 ? lane * VA + q : (WA - 1) - lane * VA - q;
            FHT_CHECK(e >= 0 && e < WA);
            const uint32_t wv = lds_b32(smem_u32(in8 + e * 16 + 4 * warp));
            v[0][q] = (int)(wv & 0xffu);
            v[1][q] = (int)((wv >> 8) & 0xffu);
            v[2][q] = (int)((wv >> 16) & 0xffu);
            v[3][q] = (int)(wv >> 24);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        warp_fht<Split<R>::a, VA>(v);
        if constexpr (!TR) {
          // the warp's box is consumed (its values went through the butterflies): the next tile's rows can land, most
          // of a tile ahead; the proxy fence orders the warp's shared-memory reads before the bulk copy's writes
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (more) issue(nxt);
        }
        // every warp is past sub-pass B's reads of the previous tile (the plane is free) and, transposed, past its
        // reads of the landing block
        __syncthreads();
        if constexpr (TR) {
          if (more) issue(nxt);
        }
        int* d = plane + (warp * NA) * PITCH + lane * VA;
        FHT_CHECK(d + (NA - 1) * PITCH + VA <= plane + NR * PITCH);
#pragma unroll
        for (int r = 0; r < NA; ++r)
#pragma unroll
          for (int q = 0; q < VA; ++q) d[r * PITCH + q] = v[r][q];
      }
      __syncthreads();
      // ---- sub-pass B: group jp = warp reads row jp of every block at column c + jp * i
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        const int* sp = plane + (i * NA + warp) * PITCH + lane * VB + warp * i;
        FHT_CHECK(lane * VB + warp * i + VB <= WA && sp + VB <= plane + NR * PITCH);
#pragma unroll
        for (int q = 0; q < VB; ++q) w[i][q] = sp[q];
      }
      par ^= 1u;
      warp_fht<Split<R>::b, VB>(w);
      // ---- the warp's 4 rows tau = warp * 4 + u through its slot, as uint16 (F_m <= 255 * 16)
      const int Xs = cur.X - sl.xlo, zscr = p.z0 + cur.img_l * p.nq + qi;
      FHT_CHECK(Xs >= 0 && Xs + p.TX <= sl.xhi - sl.xlo && p.TX == TX1 && (Xs & 7) == 0 && zscr >= 0);
      if (lane == 0) tma_wait_read();  // the slot's previous bulk store (a tile ago) has read it
      __syncwarp();
      if (lane < 31) {
        const int lo = SIG > 0 ? lane * VB : (WC - VB) - lane * VB;
#pragma unroll
        for (int u = 0; u < NA; ++u) {
          uint16_t* d = stg + u * TX1 + lo;
          FHT_CHECK(lo >= 0 && d + VB - 1 <= stg + NA * TX1);
#pragma unroll
          for (int q = 0; q < VB - 1; ++q) d[q] = static_cast<uint16_t>(w[u][SIG > 0 ? q : VB - 1 - q]);
          if (lo + VB - 1 < TX1) d[VB - 1] = static_cast<uint16_t>(w[u][SIG > 0 ? VB - 1 : 0]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
#if FHT_SCR_KEEP
        tma_store_4d_keep(tm_dst4, stg, Xs, cur.strip, warp * NA, zscr);
#else
        tma_store_4d(tm_dst4, stg, Xs, cur.strip, warp * NA, zscr);
#endif
        tma_commit();
      }
      if (!more) break;
      T = Tn;
      cur = nxt;
    }
  }
  pdl_trigger();
  if (lane == 0) tma_wait_read();
}

// tm_img128: the u8 image view [img][row][col/128][128], box {128, 4, 4, 1}; tm_imgT: the image [img][row][col], box
// {16 columns, 144 rows, 1}; tm_dst4: the uint16 scratch view [z][j][strip][column], box {TX, 1, 4, 1}.
__global__ void __launch_bounds__(128, 6)
k_p1p8(const __grid_constant__ CUtensorMap tm_img128, const __grid_constant__ CUtensorMap tm_imgT,
       const __grid_constant__ CUtensorMap tm_dst4, const __grid_constant__ P1Params p, int total) {
  pdl_wait();  // the image may come from the previous kernel; the scratch may still be read by it
  extern __shared__ __align__(1024) unsigned char smem_p1p8[];
  const int qi = blockIdx.x & ((1 << p.nq_log) - 1);  // gridDim.x % nq == 0: every tile of this CTA is slot qi's
  const P1Slot& sl = p.slot[qi];
  if (!sl.transposed) {
    if (sl.sigma > 0)
      p1p8_run<1, false>(smem_p1p8, &tm_img128, &tm_imgT, &tm_dst4, p, sl, qi, total);
    else
      p1p8_run<-1, false>(smem_p1p8, &tm_img128, &tm_imgT, &tm_dst4, p, sl, qi, total);
  } else {
    if (sl.sigma > 0)
      p1p8_run<1, true>(smem_p1p8, &tm_img128, &tm_imgT, &tm_dst4, p, sl, qi, total);
    else
      p1p8_run<-1, true>(smem_p1p8, &tm_img128, &tm_imgT, &tm_dst4, p, sl, qi, total);
  }
}

}  // namespace v2
}  // namespace fht
