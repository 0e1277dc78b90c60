// Developer probe: issue cost of cp.async.bulk (global -> smem, mbarrier complete_tx) per copy, by copy size and by
// how many lanes of one warp issue them (1 lane serially vs 4 lanes in parallel). One CTA per SM, all SMs streaming.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2505_05799_b200/csrc/sm100.cuh"
using namespace mxm;

__global__ void __launch_bounds__(128, 1) k(const uint8_t* src, int bytes, int copies, int lanes, int rounds,
                                          unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x / 32, nw = blockDim.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_mbar_init(); }
  __syncthreads();
  const uint8_t* base = src + (size_t)blockIdx.x * 8 * 1024 * 1024;
  unsigned long long issue = 0;
  const unsigned long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    uint64_t* b = &bar[r & 1];
    if (threadIdx.x == 0) mbar_arrive_expect_tx(b, (uint32_t)(bytes * copies));
    __syncthreads();
    const unsigned long long ti = clock64();
    const uint8_t* rb = base + (size_t)(r & 15) * copies * bytes;
    for (int c = warp; c < copies; c += nw) {
      if (lane == (lanes == 1 ? 0 : (c & 3)))
        bulk_load(sm + c * bytes, rb + (size_t)c * bytes, (uint32_t)bytes, b);
    }
    __syncthreads();
    issue += clock64() - ti;
    mbar_wait(b, (r >> 1) & 1);
  }
  const unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && lane == 0) { out[0] = t1 - t0; out[1] = issue; }
}

int main() {
  uint8_t* src;
  cudaMalloc(&src, (size_t)148 * 8 * 1024 * 1024);
  cudaMemset(src, 1, (size_t)148 * 8 * 1024 * 1024);
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int bytes : {256, 8192}) {
    for (int copies : {4, 8}) {
      if (bytes * copies > 190 * 1024) continue;
      for (int lanes : {1, 32, 64, 128}) {  // 1: one lane; 32: 4 lanes of one warp; 64/128: 2 / 4 warps
        const int rounds = 200;
        const int thr = lanes <= 32 ? 32 : lanes;
        k<<<148, thr, 200 * 1024>>>(src, bytes, copies, lanes == 32 ? 4 : 1, rounds, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("bytes %6d copies %d lanes %d: %7.1f cycles/round (%.1f issue) -> %.1f cycles per copy issue, %.1f B/cycle %s\n",
               bytes, copies, lanes, (double)h[0] / rounds, (double)h[1] / rounds, (double)h[1] / rounds / copies,
               (double)bytes * copies * rounds / h[0], e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
