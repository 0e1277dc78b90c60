// Developer probe: per-stage time with per-stage control overhead (wait + fence + commit), issuing the
// 8 MMAs of a stage from 1 warp vs from 2 warps (4 each, separate accumulators). bf16 SS, N=128 and N=64.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2505_05799_b200/csrc/sm100.cuh"
using namespace mxm;
__global__ void __launch_bounds__(128, 1) k(int N, int iters, int two, int ovh, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[2], cb[2][4], dummy;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)sm)[i] = 0x3c003c00u * (i & 1);
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_init(&dummy, 1); for (int i = 0; i < 4; ++i) { mbar_init(&cb[0][i], 1); mbar_init(&cb[1][i], 1);} fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = tbase;
  int w = threadIdx.x / 32;
  bool active = (threadIdx.x % 32 == 0) && (w == 0 || (two && w == 1));
  if (active) {
    uint32_t idesc = idesc_bf16(N);
    uint32_t a0 = smem_u32(sm), a1 = smem_u32(sm + 16384), b = smem_u32(sm + 32768);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (ovh) { mbar_wait(&dummy, 1); mbar_wait(&dummy, 1); tc_fence_after(); }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t bd = sw128_kmajor_desc(b + kk * 32);
        if (!two || w == 0) mma_bf16(tmem, sw128_kmajor_desc(a0 + kk * 32), bd, idesc, 1);
        if (!two || w == 1) mma_bf16(tmem + 256, sw128_kmajor_desc(a1 + kk * 32), bd, idesc, 1);
      }
      if (ovh) { mma_commit(&cb[w][it & 3]); mma_commit(&cb[w][(it + 1) & 3]); }
    }
    mma_commit(&bar[w]);
    mbar_wait(&bar[w], 0);
    if (blockIdx.x == 0 && w == 0) out[0] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8); unsigned long long h;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int N : {64, 128})
    for (int ovh = 0; ovh < 2; ++ovh)
      for (int two = 0; two < 2; ++two) {
        int iters = 3000;
        k<<<sms, 128, 100 * 1024>>>(N, iters, two, ovh, d);
        if (cudaDeviceSynchronize()) { printf("err\n"); return 1; }
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("N=%3d overhead=%d warps=%d: %.1f cycles/stage (8 MMAs, nominal %d)\n", N, ovh, two ? 2 : 1, (double)h / iters, 8 * N / 2);
      }
  return 0;
}
