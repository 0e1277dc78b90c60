// Developer probe: cycles per tcgen05.mma vs N for SS and TS forms (bf16 and i8), 1 issuing thread.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2505_05799_b200/csrc/sm100.cuh"
using namespace mxm;
template <int TS, int I8>
__global__ void __launch_bounds__(128, 1) k(int N, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)sm)[i] = I8 ? 0x01010101u : 0x3c003c00u * (i & 1);
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    uint32_t idesc = I8 ? idesc_s8(N) : idesc_bf16(N);
    uint32_t a0 = smem_u32(sm), b = smem_u32(sm + 32768);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t bd = sw128_kmajor_desc(b + kk * 32);
        if (TS) { if (I8) mma_i8_ts(tmem, tmem + 256 + kk * 8, bd, idesc, 1); else mma_bf16_ts(tmem, tmem + 256 + kk * 8, bd, idesc, 1); }
        else { if (I8) mma_i8(tmem, sw128_kmajor_desc(a0 + kk * 32), bd, idesc, 1); else mma_bf16(tmem, sw128_kmajor_desc(a0 + kk * 32), bd, idesc, 1); }
      }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0) out[0] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}
template <int TS, int I8> void run() {
  unsigned long long* d; cudaMalloc(&d, 8); unsigned long long h;
  cudaFuncSetAttribute(k<TS, I8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int N : {16, 32, 64, 128, 256}) {
    int iters = 4000;
    k<TS, I8><<<sms, 128, 100 * 1024>>>(N, iters, d);
    if (cudaDeviceSynchronize()) { printf("err\n"); return; }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%s %s N=%3d: %.1f cycles/MMA (nominal %.0f)\n", TS ? "TS" : "SS", I8 ? "i8  " : "bf16", N, (double)h / (iters * 4),
           128.0 * N / 256 / (I8 ? 2 : 1));
  }
}
int main() { run<0, 0>(); run<1, 0>(); run<0, 1>(); run<1, 1>(); return 0; }
