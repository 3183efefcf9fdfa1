// TMA row-store probe: does a 1 x BOX box store from shared memory work with a tensor map passed
// as a __grid_constant__ kernel parameter, for several smem offsets, box widths and coordinates
// (including partially out-of-bounds boxes, negative start)? Prints one line per case.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_store(const __grid_constant__ CUtensorMap tm, int smem_off_floats, int box, int col, int row) {
  extern __shared__ __align__(1024) float sm[];
  float* s = sm + smem_off_floats;
  for (int i = threadIdx.x; i < box; i += blockDim.x) s[i] = 1000.f + i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(s));
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                 :: "l"(reinterpret_cast<uint64_t>(&tm)), "r"(sa), "r"(col), "r"(row) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

int load_main(int which);
int main(int argc, char** argv) {
  if (argc > 2 && argv[1][0] == 'L') return load_main(atoi(argv[2]));
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  int ci = -1;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  const int COLS = argc > 2 ? atoi(argv[2]) : 100;
  const int ROWS = 4, PITCH = 256;
  float* g;
  CK(cudaMalloc(&g, ROWS * PITCH * 4));
  struct Case { int off, box, col, row; };
  Case cases[] = {{0, 16, 0, 0}, {224, 16, 4, 1}, {32, 16, 4, 1}, {4, 16, 4, 1}, {0, 12, 3, 2},
                  {0, 16, 90, 3}, {0, 16, -6, 3}, {0, 48, 0, 0},
                  {0, 16, 88, 3}, {0, 16, -8, 2}, {0, 212, 0, 1}, {32, 212, 0, 1}};
  for (auto c : cases) {
    if (++ci != only && only >= 0) continue;
    CK(cudaMemset(g, 0, ROWS * PITCH * 4));
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)COLS, (cuuint64_t)ROWS};
    cuuint64_t strides[1] = {PITCH * 4};
    cuuint32_t box[2] = {(cuuint32_t)c.box, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("off %d box %d col %d: encode failed %d\n", c.off, c.box, c.col, (int)r); continue; }
    k_store<<<1, 128, 8192>>>(tm, c.off, c.box, c.col, c.row);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("off %d box %d col %d row %d: %s\n", c.off, c.box, c.col, c.row, cudaGetErrorString(e)); return 2; }
    static float h[ROWS * PITCH];
    CK(cudaMemcpy(h, g, sizeof(h), cudaMemcpyDeviceToHost));
    int first = -1, last = -1, bad = 0;
    for (int x = 0; x < PITCH; ++x) {
      const float v = h[c.row * PITCH + x];
      if (v != 0.f) { if (first < 0) first = x; last = x; if (v != 1000.f + (x - c.col)) bad = 1; }
    }
    printf("off %d box %d col %d row %d: wrote cols [%d, %d] %s\n", c.off, c.box, c.col, c.row, first, last,
           bad ? "WRONG VALUES" : "ok");
  }
  return 0;
}

// ---- load probe: 1 x BOX box load into shared memory at (col, row), OOB zero fill
__global__ void k_load(const __grid_constant__ CUtensorMap tm, int box, int col, int row, float* out) {
  extern __shared__ __align__(1024) float sm2[];
  __shared__ __align__(8) unsigned long long bar;
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  for (int i = threadIdx.x; i < box; i += blockDim.x) sm2[i] = -1.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(box * 4) : "memory");
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sm2));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 :: "r"(d), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(b), "r"(col), "r"(row) : "memory");
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(b) : "memory");
  }
  for (int i = threadIdx.x; i < box; i += blockDim.x) out[i] = sm2[i];
}

int load_main(int which) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  const int COLS = 100, ROWS = 4, PITCH = 104;
  static float h[ROWS * PITCH];
  for (int r = 0; r < ROWS; ++r) for (int x = 0; x < PITCH; ++x) h[r * PITCH + x] = r * 1000 + x;
  float *g, *o;
  CK(cudaMalloc(&g, sizeof(h)));
  CK(cudaMalloc(&o, 256 * 4));
  CK(cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice));
  struct Case { int box, col, row; };
  Case cases[] = {{16, 0, 1}, {16, 3, 1}, {16, -6, 2}, {16, 90, 3}, {32, -13, 0}, {256, -100, 2}};
  Case c = cases[which];
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)COLS, (cuuint64_t)ROWS};
  cuuint64_t strides[1] = {PITCH * 4};
  cuuint32_t boxd[2] = {(cuuint32_t)c.box, 1};
  cuuint32_t es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, boxd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("load box %d col %d: encode failed\n", c.box, c.col);
    return 1;
  }
  k_load<<<1, 128, 4096>>>(tm, c.box, c.col, c.row, o);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("load box %d col %d row %d: %s\n", c.box, c.col, c.row, cudaGetErrorString(e)); return 2; }
  float r[256];
  CK(cudaMemcpy(r, o, c.box * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < c.box; ++i) {
    const int x = c.col + i;
    const float want = (x >= 0 && x < COLS) ? c.row * 1000 + x : 0.f;
    if (r[i] != want) bad++;
  }
  printf("load box %d col %d row %d: %s (first %g last %g)\n", c.box, c.col, c.row, bad ? "WRONG" : "ok", r[0], r[c.box - 1]);
  return 0;
}
