// fht_pipe.cuh -- the pipelined transform: ONE persistent kernel runs both passes of a square full
// transform (or of one quadrant) over a stream of units, so pass 1 of a later unit overlaps pass 2 of
// an earlier one and a unit's pass-1 scratch is read back while it is still in L2 (DESIGN.md §4,
// "Pipelined passes").
//
// Work decomposition. A unit is (a chunk of `nbu` images, one quadrant slot). Pass-1 items are the
// k_p1 tiles of a unit (levels 1..m of one 2^m-row strip x TX columns, image -> scratch), pass-2 items
// the k_p2 tiles (levels m+1..K of one group j x TX columns, scratch -> Hough rows); the two tile
// bodies are the ones the two-launch path runs (p1_body / p2_body in fht_tile.cuh). A CTA of NT
// threads runs one item at a time; an item is TPI1 = NT / G1 pass-1 tiles or TPI2 = NT / G2 pass-2
// tiles, each on its own thread group (G = the tile body's 4 or 8 warps, own named barrier, own
// shared memory), so 64-row pass-1 tiles (8 warps) and 32-row pass-2 tiles (4 warps) share one CTA
// shape.
//
// Schedule (a global queue, dequeued in order by atomicAdd): pass-1 items of units 0..D-1, then for
// every unit u a segment holding the pass-2 items of u evenly interleaved (Bresenham) with the pass-1
// items of unit u + D. Unit u's scratch lives in ring buffer u mod NBUF.
//   - a pass-2 item of u waits until all pass-1 items of u have completed (their TMA stores landed);
//   - a pass-1 item of u >= NBUF waits until all pass-2 items of u - NBUF have completed (buffer reuse).
// Both wait only on items that precede them in the queue; a dequeued item is held by a running CTA
// that completes it without waiting on anything later, so the waits always end (no co-residency
// assumption, no inter-kernel dependency: one launch).
#pragma once
#include "fht_tile.cuh"

namespace fht {
namespace v2 {

struct PipeParams {
  int nunits;     // U = nchunks * nq
  int nq;         // slots per image (units cycle through them)
  int nbu;        // images per unit (divides the batch)
  int D;          // lookahead in units (pass 1 of u + D runs beside pass 2 of u)
  int NBUF;       // scratch ring buffers (>= D + 1)
  int n1, n2;     // items per unit: pass 1 (tiles), pass 2 (ceil(tiles / TPI2))
  int t2;         // pass-2 tiles per unit
  int nstrips, ntiles1, ngroups, ntiles2, L;
  int64_t n_items;
  int64_t buf_rows;  // scratch rows of one ring buffer = nbu * Hp
  int* counters;     // [0] queue head, [1 + u] pass-1 items done of unit u, [1 + U + u] pass-2 items done
  // debug hook (FHT_PIPE_TRACE_PTR / _N, tools/pipe_trace.py): per item 4 x u64 = globaltimer at dequeue,
  // after its waits, at its end, and (smid << 32 | kind << 24 | unit); NULL = off
  unsigned long long* trace;
  int64_t trace_n;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_count(const int* p, int want) {
  if (ld_acquire(p) >= want) return;
  int ns = 32;
  while (ld_acquire(p) < want) {
    __nanosleep(ns);
    ns = ns < 256 ? 2 * ns : ns;
  }
}

// item k of the queue -> (kind 1 = pass 1 / 2 = pass 2, unit, index inside the unit)
__device__ __forceinline__ void decode_item(const PipeParams& pp, int64_t k, int& kind, int& unit, int& idx) {
  const int D = pp.D < pp.nunits ? pp.D : pp.nunits;
  const int64_t P = (int64_t)D * pp.n1;
  if (k < P) {
    kind = 1;
    unit = (int)(k / pp.n1);
    idx = (int)(k % pp.n1);
    return;
  }
  k -= P;
  const int full = pp.nunits - D;  // segments with pass-1 items of unit u + D
  const int64_t Ls = (int64_t)pp.n2 + pp.n1;
  if (k < (int64_t)full * Ls) {
    const int u = (int)(k / Ls);
    const int64_t off = k % Ls;
    const int64_t c0 = off * pp.n1 / Ls, c1 = (off + 1) * pp.n1 / Ls;  // pass-1 items before / through off
    if (c1 > c0) {
      kind = 1;
      unit = u + D;
      idx = (int)c0;
    } else {
      kind = 2;
      unit = u;
      idx = (int)(off - c0);
    }
    return;
  }
  k -= (int64_t)full * Ls;
  kind = 2;
  unit = full + (int)(k / pp.n2);
  idx = (int)(k % pp.n2);
}

template <int R1, int R2>
struct PipeShape {
  static constexpr int G1 = Split<R1>::nw * 32, G2 = Split<R2>::nw * 32;
  static constexpr int NT = G1 > G2 ? G1 : G2;
  static constexpr int TPI1 = NT / G1, TPI2 = NT / G2;
#ifndef FHT_PIPE_MINB128
#define FHT_PIPE_MINB128 5
#endif
  static constexpr int kMinBlocks = NT == 128 ? FHT_PIPE_MINB128 : 2;
};
// dynamic shared memory: the larger of the item layouts, then the persistent mbarriers
// ([TPI1][8] for pass-1 groups, [TPI2][8] for pass-2 groups; they outlive the items, whose layouts
// overlap each other)
template <int R1, int R2, bool U8>
__host__ __device__ constexpr size_t pipe_body_bytes() {
  using PS = PipeShape<R1, R2>;
  const size_t a = PS::TPI1 * p1_smem_bytes(R1, U8), b = PS::TPI2 * p2_smem_bytes(R2);
  return ((a > b ? a : b) + 127) & ~size_t(127);
}
template <int R1, int R2, bool U8>
__host__ __device__ constexpr size_t pipe_smem_bytes() {
  using PS = PipeShape<R1, R2>;
  return pipe_body_bytes<R1, R2, U8>() + (size_t)(PS::TPI1 + PS::TPI2) * 8 * sizeof(uint64_t);
}

// The tile bodies, inlined into the persistent loop. The loop keeps nothing in registers across a body
// (item, unit and the barrier parities live in shared memory), so the bodies get the register budget
// they have in k_p1 / k_p2 (a call boundary instead costs every tile a callee-saved register spill).
template <typename Tin, int R, typename G>
__device__ __forceinline__ bool p1_item(const G grp, unsigned char* smem, const CUtensorMap* tm_img0,
                                     const CUtensorMap* tm_img1, const P1Dst* dst, const P1Params& p,
                                     const P1Slot& sl, int img, int strip, int X, int zscr, uint64_t* bars,
                                     uint32_t par) {
  return p1_body<Tin, R>(grp, smem, tm_img0, tm_img1, dst, p, sl, img, strip, X, zscr, bars, par);
}
template <typename A, int R, typename Tscr, typename G>
__device__ __forceinline__ bool p2_item(const G grp, unsigned char* smem, const CUtensorMap* tm_scr0,
                                     const CUtensorMap* tm_scr1, const CUtensorMap* tm0, const CUtensorMap* tm1,
                                     const CUtensorMap* tm0_box, const P2Params& p, const P2Slot& sl, int img, int j,
                                     int X, int own, int64_t rbase, uint64_t* bars, uint32_t par) {
  if (sl.sigma > 0)
    return p2_body<A, R, 1, Tscr>(grp, smem, tm_scr0, tm_scr1, tm0, tm1, tm0_box, p, sl, img, j, X, own, rbase, bars,
                                  par);
  return p2_body<A, R, -1, Tscr>(grp, smem, tm_scr0, tm_scr1, tm0, tm1, tm0_box, p, sl, img, j, X, own, rbase, bars,
                                 par);
}

// Maps: as k_p1 (tm_img0/1, dst over the ring: [z][j][strip][column], z = buffer*nbu + image)
// and k_p2 (tm_scr0/1 rows of the ring, tm0/tm1/tm0_box destinations).
template <typename Tin, int R1, int R2>
__global__ void __launch_bounds__(PipeShape<R1, R2>::NT, PipeShape<R1, R2>::kMinBlocks)
k_pipe(const __grid_constant__ CUtensorMap tm_img0, const __grid_constant__ CUtensorMap tm_img1,
       const __grid_constant__ P1Dst dst, const __grid_constant__ CUtensorMap tm_scr0,
       const __grid_constant__ CUtensorMap tm_scr1, const __grid_constant__ CUtensorMap tm0,
       const __grid_constant__ CUtensorMap tm1, const __grid_constant__ CUtensorMap tm0_box,
       const __grid_constant__ P1Params p1, const __grid_constant__ P2Params p2,
       const __grid_constant__ PipeParams pp) {
  using A = typename AccOf<Tin>::type;
  using Tscr = typename ScrOf<Tin>::type;
  using PS = PipeShape<R1, R2>;
  constexpr int NB1 = 1 << Split<R1>::b, NB2 = 1 << Split<R2>::b;  // mbarriers (sub-pass-A blocks) per tile
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ int item_s;
  __shared__ unsigned long long tr_s[2];  // trace timestamps of the current item (debug hook)
  __shared__ uint32_t par_s[PS::NT];  // per thread: parity bits of its pass-1 group (0..15), pass-2 group (16..31)
  int* const head = pp.counters;
  int* const done1 = pp.counters + 1;
  int* const done2 = pp.counters + 1 + pp.nunits;
  uint64_t* const bars1 = reinterpret_cast<uint64_t*>(smem_raw + pipe_body_bytes<R1, R2, sizeof(Tin) == 1>());
  uint64_t* const bars2 = bars1 + PS::TPI1 * 8;
  if (threadIdx.x < (PS::TPI1 + PS::TPI2) * 8) mbar_init(bars1 + threadIdx.x);
  // phase parity of every barrier of this thread's group (a used tile advances each of its NB by one)
  par_s[threadIdx.x] = 0;
  __syncthreads();
  pdl_wait();  // the image may come from the previous kernel in the stream

  for (;;) {
    if (threadIdx.x == 0) item_s = atomicAdd(head, 1);
    __syncthreads();
    const int64_t item = item_s;
    if (pp.trace && threadIdx.x == 0) tr_s[0] = gtimer();
    if (item >= pp.n_items) break;
    int kind, unit, idx;
    decode_item(pp, item, kind, unit, idx);
    const int q = unit % pp.nq, chunk = unit / pp.nq, buf = unit % pp.NBUF;
    if (kind == 1) {
      // ---- pass 1: the ring buffer must be free (pass 2 of unit - NBUF done)
      if (threadIdx.x == 0 && unit >= pp.NBUF) {
        wait_count(done2 + (unit - pp.NBUF), pp.n2);
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      if (pp.trace && threadIdx.x == 0) tr_s[1] = gtimer();
      __syncthreads();
      const int g = threadIdx.x / PS::G1;
      const int tile = idx * PS::TPI1 + g;
      if (tile < pp.nbu * pp.nstrips * pp.ntiles1) {
        const int n = tile % pp.ntiles1, strip = (tile / pp.ntiles1) % pp.nstrips;
        const int il = tile / (pp.ntiles1 * pp.nstrips);
        const P1Slot& sl = p1.slot[q];
        if (n < sl.ntiles) {
        const int X = min(sl.xlo + p1.TX * n, sl.xhi - p1.TX);
        unsigned char* sm = smem_raw + (size_t)g * p1_smem_bytes(R1, sizeof(Tin) == 1);
        const int img = chunk * pp.nbu + il, z = buf * pp.nbu + il;
        bool used;
        const uint32_t par1 = par_s[threadIdx.x] & 0xffffu;
        if constexpr (PS::TPI1 == 1)
          used = p1_item<Tin, R1>(GrpAll{}, sm, &tm_img0, &tm_img1, &dst, p1, sl, img, strip, X, z, bars1, par1);
        else
          used = p1_item<Tin, R1>(GrpPart<PS::G1>{g * PS::G1, 1 + g}, sm, &tm_img0, &tm_img1, &dst, p1, sl, img,
                                  strip, X, z, bars1 + 8 * g, par1);
        if (used) par_s[threadIdx.x] ^= (1u << NB1) - 1u;
        // the tile's scratch box has been WRITTEN (not only read out of shared memory) before it counts
        if (threadIdx.x % PS::G1 == 0) {
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {  // re-derive the unit (nothing is kept in registers across the body)
        int kd, un, ix;
        decode_item(pp, item_s, kd, un, ix);
        red_release_add(pp.counters + 1 + un, 1);
      }
    } else {
      // ---- pass 2: every pass-1 tile of the unit has landed
      if (threadIdx.x == 0) {
        wait_count(done1 + unit, pp.n1);
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      if (pp.trace && threadIdx.x == 0) tr_s[1] = gtimer();
      __syncthreads();
      const int g = threadIdx.x / PS::G2;
      const int tile = idx * PS::TPI2 + g;
      if (tile < pp.t2) {
        const int n = tile % pp.ntiles2, j = (tile / pp.ntiles2) % pp.ngroups;
        const int il = tile / (pp.ntiles2 * pp.ngroups);
        const P2Slot& sl = p2.slot[q];
        // tile n of the slot's parts (as k_p2)
        const bool pa = n < sl.ntiles_a;
        const int lo = pa ? sl.xbeg : sl.xmid, nk = pa ? sl.ntiles_a : sl.ntiles - sl.ntiles_a;
        const int hi = pa ? sl.xmid : sl.xend;
        const int k = pa ? n : n - sl.ntiles_a;
        if (n < sl.ntiles) {
          const int X = k + 1 < nk ? lo + p2.TX * k : max(lo, hi - (p2.TX + WO2));
          const int own = k + 1 < nk ? p2.TX : hi - X;
          const int img = chunk * pp.nbu + il;
          const int64_t rbase = (int64_t)buf * pp.buf_rows + (int64_t)il * (pp.buf_rows / pp.nbu) + ((int64_t)j << R2);
          unsigned char* sm = smem_raw + (size_t)g * p2_smem_bytes(R2);
          uint64_t* bb = bars2 + 8 * g;
          bool used;
          const uint32_t par2 = par_s[threadIdx.x] >> 16;
          if constexpr (PS::TPI2 == 1)
            used = p2_item<A, R2, Tscr>(GrpAll{}, sm, &tm_scr0, &tm_scr1, &tm0, &tm1, &tm0_box, p2, sl, img, j, X, own,
                                        rbase, bb, par2);
          else
            used = p2_item<A, R2, Tscr>(GrpPart<PS::G2>{g * PS::G2, 1 + g}, sm, &tm_scr0, &tm_scr1, &tm0, &tm1,
                                        &tm0_box, p2, sl, img, j, X, own, rbase, bb, par2);
          if (used) par_s[threadIdx.x] ^= ((1u << NB2) - 1u) << 16;
        }
      }
      __syncthreads();  // every group's scratch loads have landed (mbarriers) and its staging is drained
      if (threadIdx.x == 0) {
        int kd, un, ix;
        decode_item(pp, item_s, kd, un, ix);
        red_release_add(pp.counters + 1 + pp.nunits + un, 1);
      }
    }
    if (pp.trace && threadIdx.x == 0 && item_s < pp.trace_n) {
      int kd, un, ix;
      decode_item(pp, item_s, kd, un, ix);
      unsigned long long* r = pp.trace + 4 * (int64_t)item_s;
      r[0] = tr_s[0];
      r[1] = tr_s[1];
      r[2] = gtimer();
      r[3] = ((unsigned long long)smid() << 32) | ((unsigned long long)kd << 24) | (unsigned)un;
    }
  }
  // outstanding Hough-row stores of this CTA complete before it exits (bulk stores are tracked per thread)
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace v2
}  // namespace fht
