// fht_internal.cuh -- host helpers shared by the translation units of libfht.so (fht_api.cu: the C ABI
// and the two-launch schedule; fht_pipe.cu: the pipelined kernel's instantiations). Not part of the ABI.
#pragma once
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "fht_dual.cuh"
#include "fht_pipe.cuh"

namespace fht {
namespace detail {

inline int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && e[0] ? std::atoi(e) : dflt;
}

// ---------------------------------------------------------------- dynamic shared memory opt-in
// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device (per-context) attribute: `done` (one
// per kernel instantiation) records, one bit per device ordinal, where it has been set, so a
// process that drives several GPUs opts in on each of them (a pure cache of device state).
template <typename K>
inline cudaError_t smem_optin(K kern, size_t bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}


// Launch with programmatic stream serialization (PDL): the kernel may be scheduled while its
// predecessor in the stream drains; it calls griddepcontrol.wait before touching memory.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = FHT_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

struct PipeMaps {
  CUtensorMap img0, img1;
  v2::P1Dst dst;
  CUtensorMap scr0, scr1, out0, out1, out0_box;
};

// k_pipe<Tin, m, L> (fht_pipe.cu): dtype 0 = u8, 1 = i32, 2 = f32. Sets the per-unit item counts and the
// persistent grid; the counters must be zero (the caller's memset).
cudaError_t launch_pipe(int dtype, int m, int L, const PipeMaps& maps, const v2::P1Params& p1,
                        const v2::P2Params& p2, v2::PipeParams pp, cudaStream_t st);

// k_dual<Tin, m, L> (fht_dual.cu): pass 1 of one chunk beside pass 2 of the previous one in one grid; sets the
// item counts from dp.t1 / dp.t2. dual_split_ok: the instantiated (m, L) pairs.
bool dual_split_ok(int m, int L);
cudaError_t launch_dual(int dtype, int m, int L, const PipeMaps& maps, const v2::P1Params& p1, const v2::P2Params& p2,
                        const v2::DualParams& dp, cudaStream_t st);

}  // namespace detail
}  // namespace fht
