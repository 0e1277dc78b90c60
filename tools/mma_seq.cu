// Developer probe: which per-stage control instruction slows tcgen05.mma issue? (bf16, N=128, 2 mats x 4 k)
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2505_05799_b200/csrc/sm100.cuh"
using namespace mxm;
__global__ void __launch_bounds__(128, 1) k(int iters, int v, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, cbar[4], dummy;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)sm)[i] = 0x3c003c00u * (i & 1);
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&dummy, 1); for (int i = 0; i < 4; ++i) mbar_init(&cbar[i], 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    uint32_t idesc = idesc_bf16(128);
    uint32_t a0 = smem_u32(sm), a1 = smem_u32(sm + 16384), b = smem_u32(sm + 32768);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (v & 4) mbar_wait(&dummy, 1);   // already-complete phase: returns at once
      if (v & 2) tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t bd = sw128_kmajor_desc(b + kk * 32);
        mma_bf16(tmem, sw128_kmajor_desc(a0 + kk * 32), bd, idesc, 1);
        mma_bf16(tmem + 256, sw128_kmajor_desc(a1 + kk * 32), bd, idesc, 1);
      }
      if (v & 1) mma_commit(&cbar[it & 3]);
      if (v & 8) mma_commit(&cbar[(it + 1) & 3]);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8); unsigned long long h;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* nm[] = {"plain", "+commit", "+fence", "+commit+fence", "+wait", "+wait+commit", "+wait+fence", "+wait+fence+commit", "", "+2commits", "", "+fence+2commits", "", "", "", "all+2commits"};
  for (int v : {0, 1, 2, 3, 4, 5, 6, 7, 9, 11, 15}) {
    int iters = 3000;
    k<<<sms, 128, 100 * 1024>>>(iters, v, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-22s %.1f cycles/stage of 8 MMAs (nominal 512)\n", nm[v], (double)h / iters);
  }
  return 0;
}
