// fht_pipe.cu -- instantiations and launch of the pipelined kernel (fht_pipe.cuh), in their own
// translation unit so the library's sources compile in parallel.
#include "../../include/fht.h"
#include "fht_internal.cuh"

namespace fht {
namespace detail {
namespace {

template <typename Tin, int R1, int R2>
cudaError_t launch_pipe_t(const PipeMaps& m, const v2::P1Params& a, const v2::P2Params& b, v2::PipeParams pp,
                          cudaStream_t st) {
  using PS = v2::PipeShape<R1, R2>;
  constexpr size_t smem = v2::pipe_smem_bytes<R1, R2, sizeof(Tin) == 1>();
  static std::atomic<unsigned long long> done{0};
  cudaError_t e = smem_optin(v2::k_pipe<Tin, R1, R2>, smem, done);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0, occ = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess ||
      (e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess ||
      (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, v2::k_pipe<Tin, R1, R2>, PS::NT, smem)) != cudaSuccess)
    return e;
  const int n1t = pp.nbu * pp.nstrips * pp.ntiles1;  // pass-1 tiles per unit
  pp.n1 = (n1t + PS::TPI1 - 1) / PS::TPI1;
  pp.t2 = pp.nbu * pp.ngroups * pp.ntiles2;
  pp.n2 = (pp.t2 + PS::TPI2 - 1) / PS::TPI2;
  pp.n_items = (int64_t)pp.nunits * (pp.n1 + pp.n2);
  int64_t grid = (int64_t)nsm * (occ > 0 ? occ : 1);  // persistent: one wave of resident CTAs
  if (env_int("FHT_PIPE_GRID", 0) > 0) grid = env_int("FHT_PIPE_GRID", 0);
  if (grid > pp.n_items) grid = pp.n_items;
  if (env_int("FHT_PIPE_DEBUG", 0))
    std::fprintf(stderr, "k_pipe<%d,%d>: occ %d/SM x %d SMs, grid %lld, NT %d, smem %zu, units %d (nbu %d, D %d, NBUF %d), "
                 "items %lld (n1 %d, n2 %d)\n", R1, R2, occ, nsm, (long long)grid, PS::NT, smem, pp.nunits, pp.nbu, pp.D,
                 pp.NBUF, (long long)pp.n_items, pp.n1, pp.n2);
  return launch_pdl(v2::k_pipe<Tin, R1, R2>, dim3((unsigned)grid), dim3(PS::NT), smem, st, m.img0, m.img1, m.dst,
                    m.scr0, m.scr1, m.out0, m.out1, m.out0_box, a, b, pp);
}
template <typename Tin>
cudaError_t launch_pipe_tt(int m1, int L, const PipeMaps& m, const v2::P1Params& a, const v2::P2Params& b,
                           const v2::PipeParams& pp, cudaStream_t st) {
  if (m1 == 4 && L == 4) return launch_pipe_t<Tin, 4, 4>(m, a, b, pp, st);
  if (m1 == 4 && L == 5) return launch_pipe_t<Tin, 4, 5>(m, a, b, pp, st);
  if (m1 == 5 && L == 5) return launch_pipe_t<Tin, 5, 5>(m, a, b, pp, st);
  if (m1 == 6 && L == 5) return launch_pipe_t<Tin, 6, 5>(m, a, b, pp, st);
  if (m1 == 6 && L == 6) return launch_pipe_t<Tin, 6, 6>(m, a, b, pp, st);
  return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t launch_pipe(int dtype, int m1, int L, const PipeMaps& m, const v2::P1Params& a, const v2::P2Params& b,
                        v2::PipeParams pp, cudaStream_t st) {
  if (dtype == 0) return launch_pipe_tt<uint8_t>(m1, L, m, a, b, pp, st);
  if (dtype == 1) return launch_pipe_tt<int32_t>(m1, L, m, a, b, pp, st);
  return launch_pipe_tt<float>(m1, L, m, a, b, pp, st);
}

}  // namespace detail
}  // namespace fht
