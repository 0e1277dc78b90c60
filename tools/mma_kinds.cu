// Developer probe: tcgen05.mma throughput per kind (f16 / i8 / f8f6f4) and A source (SMEM = SS, TMEM = TS), two
// accumulators alternating (the dual gate/up pattern), token width N. Prints cycles per MMA vs nominal N/2
// (M = 128, K = 32 bytes per instruction: 16 bf16 or 32 8-bit elements). One CTA per SM, one elected issuer.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2505_05799_b200/csrc/sm100.cuh"
using namespace mxm;

template <int KIND, bool TS>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint32_t at, uint64_t b, uint32_t idesc) {
  if constexpr (KIND == 0) {
    if constexpr (TS) mma_bf16_ts(d, at, b, idesc, 1); else mma_bf16(d, a, b, idesc, 1);
  } else if constexpr (KIND == 1) {
    if constexpr (TS) mma_i8_ts(d, at, b, idesc, 1); else mma_i8(d, a, b, idesc, 1);
  } else {
    if constexpr (TS) mma_f8_ts(d, at, b, idesc, 1); else mma_f8(d, a, b, idesc, 1);
  }
}

template <int KIND, bool TS>
__global__ void __launch_bounds__(384, 1) k(int N, int iters, unsigned long long* out, int ldwarps, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 3 * 16384 / 4; i += 128) ((uint32_t*)sm)[i] = 0;
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t idesc = KIND == 0 ? idesc_bf16(N) : (KIND == 1 ? idesc_s8(N) : idesc_f8(N));
  const uint32_t a0 = smem_u32(sm), a1 = smem_u32(sm + 16384), b = smem_u32(sm + 32768);
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  const int warp = threadIdx.x / 32;
  if (warp >= 4 && warp < 4 + ldwarps) {  // concurrent accumulator reads (the g128 drain pattern)
    uint32_t acc = 0;
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    int i = 0;
    while (!done) {
      uint32_t r[8];
      tmem_ld8(base + ((i * 8) & 255), r);
      tmem_ld_wait();
      for (int j = 0; j < 8; ++j) acc += r[j];
      ++i;
    }
    sink[blockIdx.x * 384 + threadIdx.x] = acc;
  }
  if (threadIdx.x < 32) {
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          mma<KIND, TS>(tmem, sw128_kmajor_desc(a0 + kk * 32), tmem + 384 + kk * 8, sw128_kmajor_desc(b + kk * 32), idesc);
          mma<KIND, TS>(tmem + 192, sw128_kmajor_desc(a1 + kk * 32), tmem + 416 + kk * 8, sw128_kmajor_desc(b + kk * 32),
                        idesc);
        }
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
    if (threadIdx.x == 0) done = 1;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int KIND, bool TS>
void run(int N, int ldw) {
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&sink, 148 * 384 * 4);
  cudaMalloc(&d, 8);
  unsigned long long h = 0;
  cudaFuncSetAttribute(k<KIND, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2000;
  k<KIND, TS><<<sms, 384, 100 * 1024>>>(N, iters, d, ldw, sink);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const char* kn[3] = {"f16 ", "i8  ", "f8  "};
  printf("%s %s N=%3d ldwarps=%d: %6.1f cycles/MMA (nominal %.0f) %s\n", kn[KIND], TS ? "TS" : "SS", N, ldw,
         (double)h / (iters * 8), N / 2.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}
int main() {
  for (int ldw : {0, 4, 8}) {
    for (int N : {64, 96}) {
      run<0, false>(N, ldw); run<0, true>(N, ldw);
      run<2, false>(N, ldw); run<2, true>(N, ldw);
    }
  }
  return 0;
}
