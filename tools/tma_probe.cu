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

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  int ci = -1;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  const int COLS = argc > 2 ? atoi(argv[2]) : 100, ROWS = 4, PITCH = 256;
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
    cuuint64_t dims[2] = {COLS, ROWS};
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
