// Hardware probe: device properties, HBM write/read/copy bandwidth, L2-resident read
// bandwidth, FADD throughput. Used to size the FHT kernels.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void wr(float4* p, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) p[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}
__global__ void rd(const float4* p, size_t n, float* out) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  float acc = 0;
  for (; i < n; i += st) { float4 v = __ldcg(p + i); acc += v.x + v.y + v.z + v.w; }
  if (acc == 12345.f) out[0] = acc;
}
__global__ void cp(const float4* a, float4* b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}
__global__ void fadd(float* out, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  float b = 1e-7f * blockIdx.x, c = 2e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 += b; a1 += c; a2 += b; a3 += c; a4 += b; a5 += c; a6 += b; a7 += c;
    }
  }
  float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 0.123f) out[0] = s;
}
__global__ void iadd(int* out, int iters) {
  int a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  int b = blockIdx.x, c = 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 += b; a1 += c; a2 += b; a3 += c; a4 += b; a5 += c; a6 += b; a7 += c;
    }
  }
  int s = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
  if (s == 0x1234567) out[0] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int l2 = 0, persist = 0; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  cudaDeviceGetAttribute(&persist, cudaDevAttrMaxPersistingL2CacheSize, 0);
  printf("name=%s sms=%d cc=%d.%d l2=%d persistL2max=%d smemPerSM=%zu smemOptin=%zu regsPerSM=%d clockKHz=%d memClockKHz=%d busw=%d\n",
         p.name, p.multiProcessorCount, p.major, p.minor, l2, persist, p.sharedMemPerMultiprocessor,
         p.sharedMemPerBlockOptin, p.regsPerMultiprocessor, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  size_t big = (size_t)2 << 30;  // 2 GiB
  float4 *a, *b; float* o; CK(cudaMalloc(&a, big)); CK(cudaMalloc(&b, big)); CK(cudaMalloc(&o, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = p.multiProcessorCount * 8;
  auto timeit = [&](auto fn, int reps) { fn(); cudaEventRecord(e0); for (int r = 0; r < reps; ++r) fn(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / reps; };
  size_t n = big / 16;
  float ms = timeit([&] { wr<<<grid, 256>>>(a, n); }, 10); printf("hbm_write GB/s %.1f\n", big / ms / 1e6);
  ms = timeit([&] { rd<<<grid, 256>>>(a, n, o); }, 10); printf("hbm_read GB/s %.1f\n", big / ms / 1e6);
  ms = timeit([&] { cp<<<grid, 256>>>(a, b, n); }, 10); printf("hbm_copy GB/s %.1f (r+w)\n", 2 * big / ms / 1e6);
  for (size_t mb : {8, 16, 32, 48, 64, 96}) {
    size_t bytes = mb << 20, nn = bytes / 16;
    ms = timeit([&] { rd<<<grid, 256>>>(a, nn, o); }, 50); printf("l2_read %zuMB GB/s %.1f\n", mb, bytes / ms / 1e6);
    ms = timeit([&] { wr<<<grid, 256>>>(a, nn); }, 50); printf("l2_write %zuMB GB/s %.1f\n", mb, bytes / ms / 1e6);
  }
  int iters = 4096;
  ms = timeit([&] { fadd<<<p.multiProcessorCount * 4, 512>>>(o, iters); }, 5);
  double ops = (double)p.multiProcessorCount * 4 * 512 * iters * 16 * 8;
  printf("fadd Tops/s %.2f  per-SM-clk(at %d MHz) %.1f\n", ops / ms / 1e9, p.clockRate / 1000, ops / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3));
  ms = timeit([&] { iadd<<<p.multiProcessorCount * 4, 512>>>((int*)o, iters); }, 5);
  printf("iadd Tops/s %.2f\n", ops / ms / 1e9);
  CK(cudaDeviceSynchronize());
  return 0;
}
