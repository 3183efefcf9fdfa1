// fht_dual.cu -- instantiations and launch of the staggered pass-pair kernel (fht_dual.cuh), in their own
// translation unit so the library's sources compile in parallel.
#include "../../include/fht.h"
#include "fht_internal.cuh"

namespace fht {
namespace detail {
namespace {

template <typename Tin, int R1, int R2>
cudaError_t launch_dual_t(const PipeMaps& m, const v2::P1Params& a, const v2::P2Params& b, v2::DualParams dp,
                          cudaStream_t st) {
  using DS = v2::DualShape<Tin, R1, R2>;
  static std::atomic<unsigned long long> done{0};
  cudaError_t e = smem_optin(v2::k_dual<Tin, R1, R2>, DS::smem, done);
  if (e != cudaSuccess) return e;
  dp.n1 = (dp.t1 + DS::TPI1 - 1) / DS::TPI1;
  dp.n2 = (dp.t2 + DS::TPI2 - 1) / DS::TPI2;
  const int64_t grid = dp.n1 + dp.n2;
  if (grid <= 0 || grid > 0x7fffffff) return cudaErrorInvalidValue;
  return launch_pdl(v2::k_dual<Tin, R1, R2>, dim3((unsigned)grid), dim3(DS::NT), DS::smem, st, m.img0, m.img1, m.dst,
                    m.scr0, m.scr1, m.out0, m.out1, m.out0_box, a, b, dp);
}
template <typename Tin>
cudaError_t launch_dual_tt(int m1, int L, const PipeMaps& m, const v2::P1Params& a, const v2::P2Params& b,
                           const v2::DualParams& dp, cudaStream_t st) {
  if (m1 == 4 && L == 5) return launch_dual_t<Tin, 4, 5>(m, a, b, dp, st);
  if (m1 == 5 && L == 5) return launch_dual_t<Tin, 5, 5>(m, a, b, dp, st);
  if (m1 == 6 && L == 5) return launch_dual_t<Tin, 6, 5>(m, a, b, dp, st);
  if (m1 == 6 && L == 6) return launch_dual_t<Tin, 6, 6>(m, a, b, dp, st);
  return cudaErrorInvalidValue;
}
}  // namespace

bool dual_split_ok(int m1, int L) { return (m1 == 4 || m1 == 5 || m1 == 6) && (L == 5 || (L == 6 && m1 == 6)); }

cudaError_t launch_dual(int dtype, int m1, int L, const PipeMaps& m, const v2::P1Params& a, const v2::P2Params& b,
                        const v2::DualParams& dp, cudaStream_t st) {
  if (dtype == 0) return launch_dual_tt<uint8_t>(m1, L, m, a, b, dp, st);
  if (dtype == 1) return launch_dual_tt<int32_t>(m1, L, m, a, b, dp, st);
  return launch_dual_tt<float>(m1, L, m, a, b, dp, st);
}

}  // namespace detail
}  // namespace fht
