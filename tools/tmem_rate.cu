// Developer probe: tcgen05.ld throughput (TMEM -> registers) per SM, by warps reading and shape.
// Each warp reads its 32-lane subpartition (warp % 4) repeatedly; reports bytes / cycle / SM.
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2505_05799_b200/csrc/sm100.cuh"
using namespace mxm;

template <int X>
__device__ __forceinline__ void ld(uint32_t a, uint32_t (&r)[32]) {
  if constexpr (X == 8)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(a));
  else if constexpr (X == 16)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(a));
  else
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                   "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(a));
}

template <int X>
__global__ void k(int iters, int nwarps, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tb);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = tb + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    for (int i = 0; i < iters; ++i) {
      uint32_t r[32];
      ld<X>(base + ((i * X + warp * 64) & 511), r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < X; ++j) acc += r[j];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

template <int X>
void run(int nwarps) {
  const int iters = 4096;
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  k<X><<<148, 512>>>(iters, nwarps, d, sink);
  cudaDeviceSynchronize();
  k<X><<<148, 512>>>(iters, nwarps, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[148];
  cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
  double bytes = (double)nwarps * iters * 32 * X * 4;
  printf("tcgen05.ld 32x32b.x%d, %2d warps: %.1f B/cycle/SM (%s)\n", X, nwarps, bytes / c[0], cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}
int main() {
  for (int w : {1, 4, 8, 16}) {
    run<8>(w);
    run<16>(w);
    run<32>(w);
  }
  return 0;
}
