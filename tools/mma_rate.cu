// Developer probe: tcgen05.mma throughput vs N from resident SMEM tiles (SS mode), one CTA per SM.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2505_05799_b200/csrc/sm100.cuh"
using namespace mxm;
__global__ void __launch_bounds__(128, 1) k(int N, int iters, int kind, int nmats, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 3 * 32768 / 4; i += 128) ((uint32_t*)sm)[i] = 0x3c003c00u * (i & 1);
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    uint32_t idesc = kind == 0 ? idesc_bf16(N) : idesc_s8(N);
    uint32_t a0 = smem_u32(sm), a1 = smem_u32(sm + 16384), b = smem_u32(sm + 65536);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t bd = sw128_kmajor_desc(b + kk * 32);
        for (int m = 0; m < nmats; ++m) {
          uint64_t ad = sw128_kmajor_desc((m ? a1 : a0) + kk * 32);
          if (kind == 0) mma_bf16(tmem + m * 256, ad, bd, idesc, 1); else mma_i8(tmem + m * 256, ad, bd, idesc, 1);
        }
      }
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
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int kind = 0; kind < 2; ++kind)
    for (int nm = 1; nm <= 2; ++nm)
      for (int N : {16, 32, 64, 128, 256}) {
        int iters = 2000;
        k<<<sms, 128, 200 * 1024>>>(N, iters, kind, nm, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        double per = (double)h / (iters * 4 * nm);
        double nominal = 128.0 * N / 256.0 / (kind ? 2 : 1);
        printf("%s mats=%d N=%3d: %.1f cycles/MMA (nominal %.0f)  -> %.0f%% of peak\n", kind ? "i8  " : "bf16", nm, N, per,
               nominal, 100 * nominal / per);
      }
  return 0;
}
