// fht_dual.cuh -- staggered pass pairs: ONE launch runs pass 1 of batch chunk k beside pass 2 of chunk
// k - 1 ("Staggered dual launches").
//
// Why. Pass 1 is latency/issue-bound (≈0.45 of the copy bandwidth on its bytes), pass 2 is DRAM-bound on the
// Hough rows it writes; run one after the other they cannot use each other's idle resource. Two streams do not
// interleave them (the block scheduler dispatches a kernel's CTAs before the next kernel's, whatever the stream
// priority: profiles/r02/prio_ab.log), so here both passes are items of one grid, interleaved in blockIdx
// order (Bresenham), and the block scheduler keeps both kinds resident on every SM for the whole launch.
//
// Schedule over nchunks chunks (scratch buffers ping-pong by chunk parity):
//   launch 0:          k_p1(chunk 0)
//   launch k (1..n-1): k_dual = pass 1 of chunk k (buffer k&1) + pass 2 of chunk k-1 (buffer (k-1)&1)
//   launch n:          k_p2(chunk n-1)
// Every launch starts with griddepcontrol.wait (programmatic dependent launch): launch k's pass 2 reads what
// launch k-1's pass 1 wrote, and launch k's pass 1 overwrites the buffer launch k-1's pass 2 read -- both
// ordered by the completion of launch k-1. No CTA waits on another CTA (no flags, no co-residency
// assumption). The tile bodies are k_p1's and k_p2's (fht_tile.cuh), so the results are bit-identical.
//
// CTA shape: NT = max(pass-1 group, pass-2 group) threads; an item is NT / G1 pass-1 tiles or NT / G2
// pass-2 tiles, each on its own thread group with its own shared memory (as fht_pipe.cuh). The bodies are
// inlined (behind call boundaries every parameter read became a generic load; FHT_DUAL_NOINLINE=1 restores
// that variant) and both kinds of items run slot-slowest, so an SM holds one sign's code at a time.
// Measured slower than the two-launch schedule; opt-in.
#pragma once
#include "fht_pipe.cuh"

namespace fht {
namespace v2 {

#ifndef FHT_DUAL_NOINLINE
#define FHT_DUAL_NOINLINE 0
#endif
#if FHT_DUAL_NOINLINE
#define DUAL_INLINE __noinline__
#else
#define DUAL_INLINE __forceinline__  // parameters stay in the constant bank (a call takes their address: generic loads)
#endif

struct DualParams {
  int64_t n1, n2;       // pass-1 / pass-2 items of the launch
  int64_t t1, t2;       // pass-1 / pass-2 tiles (items * tiles per item, minus the ragged end)
  int ntiles1, nstrips; // pass-1 tiles per strip, strips per image
  int ntiles2, ngroups; // pass-2 tiles per group, groups
};

template <typename Tin, int R1, int R2>
struct DualShape {
  static constexpr int G1 = Split<R1>::nw * 32, G2 = Split<R2>::nw * 32;
  static constexpr int NT = G1 > G2 ? G1 : G2;
  static constexpr int TPI1 = NT / G1, TPI2 = NT / G2;
  static constexpr size_t S1 = p1_smem_bytes(R1, sizeof(Tin) == 1), S2 = p2_smem_bytes(R2);
  static constexpr size_t smem = TPI1 * S1 > TPI2 * S2 ? TPI1 * S1 : TPI2 * S2;
  static constexpr int kMinBlocks = NT == 128 ? 5 : 2;
};

template <typename Tin, int R, typename G>
__device__ DUAL_INLINE void dual_p1_tile(const G grp, unsigned char* smem, const CUtensorMap* tm_img0,
                                          const CUtensorMap* tm_img1, const P1Dst* dst, const P1Params* p, int64_t t,
                                          int64_t t1_per_slot) {
  // slot slowest (then image, strip, tile): the launch runs the slots one after another, and pass-2 items are
  // ordered the same way, so an SM holds one sign's pass-1 tail, one fill path and one sign's pass-2 body at a
  // time (the instruction cache: mixing them stalled C3's dual launch on instruction fetch, 43% of samples)
  const int64_t per_slot = t1_per_slot;
  const int qi = (int)(t / per_slot);
  const int64_t r0 = t - (int64_t)qi * per_slot;
  const int64_t per_img = (int64_t)p->ntiles << p->L;
  const int il = (int)(r0 / per_img);
  const int64_t r = r0 - (int64_t)il * per_img;
  const int strip = (int)(r / p->ntiles), n = (int)(r % p->ntiles);
  const P1Slot& sl = p->slot[qi];
  if (n >= sl.ntiles) return;
  const int X = min(sl.xlo + p->TX * n, sl.xhi - p->TX);
  p1_body<Tin, R>(grp, smem, tm_img0, tm_img1, dst, *p, sl, p->img0 + il, strip, X, p->z0 + il * p->nq + qi);
}

template <typename A, int R, int SIG, typename Tscr, typename G>
__device__ DUAL_INLINE void dual_p2_tile(const G grp, unsigned char* smem, const CUtensorMap* tm_scr0,
                                          const CUtensorMap* tm_scr1, const CUtensorMap* tm0, const CUtensorMap* tm1,
                                          const CUtensorMap* tm0_box, const P2Params* p, int qi, int il, int jl, int n) {
  const P2Slot& sl = p->slot[qi];
  const bool pa = n < sl.ntiles_a;
  const int lo = pa ? sl.xbeg : sl.xmid, nk = pa ? sl.ntiles_a : sl.ntiles - sl.ntiles_a;
  const int hi = pa ? sl.xmid : sl.xend;
  const int k = pa ? n : n - sl.ntiles_a;
  const int X = k + 1 < nk ? lo + p->TX * k : max(lo, hi - (p->TX + WO2));
  const int own = k + 1 < nk ? p->TX : hi - X;
  const int64_t rbase = p->row0 + (int64_t)il * p->scratch_img_rows + sl.srow0 + ((int64_t)jl << p->logS);
  p2_body<A, R, SIG, Tscr>(grp, smem, tm_scr0, tm_scr1, tm0, tm1, tm0_box, *p, sl, p->img0 + il, p->j0 + jl, X, own,
                           rbase);
}

template <typename Tin, int R1, int R2>
__global__ void __launch_bounds__(DualShape<Tin, R1, R2>::NT, DualShape<Tin, R1, R2>::kMinBlocks)
k_dual(const __grid_constant__ CUtensorMap tm_img0, const __grid_constant__ CUtensorMap tm_img1,
       const __grid_constant__ P1Dst dst, const __grid_constant__ CUtensorMap tm_scr0,
       const __grid_constant__ CUtensorMap tm_scr1, const __grid_constant__ CUtensorMap tm0,
       const __grid_constant__ CUtensorMap tm1, const __grid_constant__ CUtensorMap tm0_box,
       const __grid_constant__ P1Params p1, const __grid_constant__ P2Params p2,
       const __grid_constant__ DualParams dp) {
  using A = typename AccOf<Tin>::type;
  using Tscr = typename ScrOf<Tin>::type;
  using DS = DualShape<Tin, R1, R2>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  pdl_wait();  // launch k-1 complete: its scratch is written, the buffer this pass 1 overwrites is read
  const int64_t b = blockIdx.x, tot = dp.n1 + dp.n2;
  const int64_t c = b * dp.n1 / tot;  // pass-1 items before b (Bresenham interleave)
  if ((b + 1) * dp.n1 / tot > c) {
    const int g = threadIdx.x / DS::G1;
    const int64_t t = c * DS::TPI1 + g;
    if (t >= dp.t1) return;
    unsigned char* sm = smem_raw + (size_t)g * DS::S1;
    if constexpr (DS::TPI1 == 1)
      dual_p1_tile<Tin, R1>(GrpAll{}, sm, &tm_img0, &tm_img1, &dst, &p1, t, dp.t1 >> p1.nq_log);
    else
      dual_p1_tile<Tin, R1>(GrpPart<DS::G1>{g * DS::G1, 1 + g}, sm, &tm_img0, &tm_img1, &dst, &p1, t, dp.t1 >> p1.nq_log);
    return;
  }
  const int g = threadIdx.x / DS::G2;
  const int64_t t = (b - c) * DS::TPI2 + g;
  if (t >= dp.t2) return;
  // tile n fastest, then group jl, then the image, the slot slowest (as the pass-1 items)
  const int n = (int)(t % dp.ntiles2);
  const int64_t s = t / dp.ntiles2;
  const int jl = (int)(s % dp.ngroups);
  const int64_t z = s / dp.ngroups;
  const int64_t nimg2 = (dp.t2 >> p2.nq_log) / ((int64_t)dp.ngroups * dp.ntiles2);
  const int qi = (int)(z / nimg2), il = (int)(z % nimg2);
  if (n >= p2.slot[qi].ntiles) return;
  unsigned char* sm = smem_raw + (size_t)g * DS::S2;
  if constexpr (DS::TPI2 == 1) {
    if (p2.slot[qi].sigma > 0)
      dual_p2_tile<A, R2, 1, Tscr>(GrpAll{}, sm, &tm_scr0, &tm_scr1, &tm0, &tm1, &tm0_box, &p2, qi, il, jl, n);
    else
      dual_p2_tile<A, R2, -1, Tscr>(GrpAll{}, sm, &tm_scr0, &tm_scr1, &tm0, &tm1, &tm0_box, &p2, qi, il, jl, n);
  } else {
    const GrpPart<DS::G2> grp{g * DS::G2, 1 + g};
    if (p2.slot[qi].sigma > 0)
      dual_p2_tile<A, R2, 1, Tscr>(grp, sm, &tm_scr0, &tm_scr1, &tm0, &tm1, &tm0_box, &p2, qi, il, jl, n);
    else
      dual_p2_tile<A, R2, -1, Tscr>(grp, sm, &tm_scr0, &tm_scr1, &tm0, &tm1, &tm0_box, &p2, qi, il, jl, n);
  }
}

}  // namespace v2
}  // namespace fht
