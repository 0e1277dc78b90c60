// Developer probe: tcgen05.mma (bf16 SS, N=128, 2 mats) cycles/MMA while warp 1 streams cp.async.bulk copies
// (global, L2-resident) into other SMEM regions at full speed.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2505_05799_b200/csrc/sm100.cuh"
using namespace mxm;
__global__ void __launch_bounds__(128, 1) k(int iters, int copy_kb, const uint8_t* src, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar, cb[2];
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 49152 / 4; i += 128) ((uint32_t*)sm)[i] = 0x3c003c00u * (i & 1);
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&cb[0], 1); mbar_init(&cb[1], 1); fence_mbar_init(); stop = 0; }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = tbase;
  int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    uint32_t idesc = idesc_bf16(128);
    uint32_t a0 = smem_u32(sm), a1 = smem_u32(sm + 16384), b = smem_u32(sm + 32768);
    unsigned long long t0 = clock64();
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
  } else if (threadIdx.x == 32 && copy_kb > 0) {
    uint32_t ph[2] = {0, 0};
    unsigned long long n = 0;
    const uint8_t* s = src + (size_t)blockIdx.x * 65536;
    for (int i = 0; !stop; ++i) {
      int j = i & 1;
      if (i >= 2) { mbar_wait(&cb[j], ph[j]); ph[j] ^= 1; }
      mbar_arrive_expect_tx(&cb[j], copy_kb * 1024);
      for (int c = 0; c < copy_kb; c += 16) bulk_load(sm + 65536 + j * 65536 + c * 1024, s + c * 1024, 16384, &cb[j]);
      ++n;
    }
    for (int j = 0; j < 2; ++j) mbar_wait(&cb[j], ph[j]);
    if (blockIdx.x == 0) out[1] = n;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16); unsigned long long h[2];
  uint8_t* src; cudaMalloc(&src, 148 * 65536); cudaMemset(src, 1, 148 * 65536);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int kb : {0, 16, 32, 64}) {
    int iters = 4000;
    k<<<sms, 128, 200 * 1024>>>(iters, kb, src, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    double cyc = (double)h[0];
    printf("bulk %2d KB batches: %.1f cycles/MMA (nominal 64); copy rate %.1f B/cycle/SM\n", kb, cyc / (iters * 8),
           kb ? (double)h[1] * kb * 1024 / cyc : 0.0);
  }
  return 0;
}
