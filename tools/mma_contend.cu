// Developer probe: tcgen05.mma (bf16 SS, N=128, 2 mats) cycles/MMA while W other warps stream STS.128 / LDS.128.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2505_05799_b200/csrc/sm100.cuh"
using namespace mxm;
__global__ void __launch_bounds__(512, 1) k(int N, int iters, int nwriters, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 196608 / 4; i += 512) ((uint32_t*)sm)[i] = 0x3c003c00u * (i & 1);
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); stop = 0; }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = tbase;
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    uint32_t idesc = idesc_bf16(N);
    uint32_t a0 = smem_u32(sm), a1 = smem_u32(sm + 16384), b = smem_u32(sm + 32768);
    unsigned long long t0 = clock64();
    if (threadIdx.x == 0) {
      for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          uint64_t bd = sw128_kmajor_desc(b + kk * 32);
          mma_bf16(tmem, sw128_kmajor_desc(a0 + kk * 32), bd, idesc, 1);
          mma_bf16(tmem + 256, sw128_kmajor_desc(a1 + kk * 32), bd, idesc, 1);
        }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      unsigned long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
      stop = 1;
    }
    __syncwarp();
  } else if (warp <= nwriters) {
    // streaming smem traffic in the upper 64 KB (not the MMA operands)
    uint4* p = (uint4*)(sm + 131072) + (threadIdx.x - 32) % 2048;
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    unsigned long long cnt = 0;
    while (!stop) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (mode == 0) p[(j * 512) % 4096] = v;
        else { uint4 t = p[(j * 512) % 4096]; v.x ^= t.x; }
      }
      cnt += 16;
    }
    if (v.x == 12345) out[1] = cnt;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16); unsigned long long h;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 2; ++mode)
    for (int N : {128, 256})
      for (int w : {0, 2, 4, 8, 15}) {
        int iters = 4000;
        k<<<sms, 512, 200 * 1024>>>(N, iters, w, mode, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%s N=%d writers=%2d: %.1f cycles/MMA (nominal %.0f)\n", mode ? "LDS" : "STS", N, w, (double)h / (iters * 8), N / 2.0);
      }
  return 0;
}
