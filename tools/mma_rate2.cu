// Developer probe: tcgen05.mma issue variants (N=128/256 bf16, 2 mats) -> cycles per MMA.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2505_05799_b200/csrc/sm100.cuh"
using namespace mxm;
__device__ __forceinline__ void mma_nc(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
template <int V>
__global__ void __launch_bounds__(128, 1) k(int N, int iters, unsigned long long* out) {
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
  uint32_t idesc = idesc_bf16(N);
  uint32_t a0 = smem_u32(sm), a1 = smem_u32(sm + 16384), b = smem_u32(sm + 65536);
  uint64_t ad0[4], ad1[4], bd[4];
  for (int kk = 0; kk < 4; ++kk) { ad0[kk] = sw128_kmajor_desc(a0 + kk * 32); ad1[kk] = sw128_kmajor_desc(a1 + kk * 32); bd[kk] = sw128_kmajor_desc(b + kk * 32); }
  if (threadIdx.x < 32) {
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (V == 0) {  // lane 0 only, per-iteration descriptors (current kernel style)
          if (threadIdx.x == 0) {
            mma_bf16(tmem, sw128_kmajor_desc(a0 + kk * 32), sw128_kmajor_desc(b + kk * 32), idesc, 1);
            mma_bf16(tmem + 256, sw128_kmajor_desc(a1 + kk * 32), sw128_kmajor_desc(b + kk * 32), idesc, 1);
          }
        } else if (V == 1) {  // whole warp, elect
          if (elect_one()) {
            mma_bf16(tmem, ad0[kk], bd[kk], idesc, 1);
            mma_bf16(tmem + 256, ad1[kk], bd[kk], idesc, 1);
          }
          __syncwarp();
        } else if (V == 2) {  // lane 0, precomputed descriptors, no memory clobber
          if (threadIdx.x == 0) {
            mma_nc(tmem, ad0[kk], bd[kk], idesc, 1);
            mma_nc(tmem + 256, ad1[kk], bd[kk], idesc, 1);
          }
        } else {  // whole warp elect + no clobber
          if (elect_one()) {
            mma_nc(tmem, ad0[kk], bd[kk], idesc, 1);
            mma_nc(tmem + 256, ad1[kk], bd[kk], idesc, 1);
          }
        }
      }
    }
    if (threadIdx.x == 0) { mma_commit(&bar); mbar_wait(&bar, 0); }
    __syncwarp();
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}
template <int V> void run(int N) {
  unsigned long long* d; cudaMalloc(&d, 8); unsigned long long h;
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters = 2000;
  k<V><<<sms, 128, 200 * 1024>>>(N, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  double per = (double)h / (iters * 8);
  printf("variant %d N=%3d: %.1f cycles/MMA (nominal %.0f)\n", V, N, per, 128.0 * N / 256.0);
}
int main() { for (int N : {64, 128, 256}) { run<0>(N); run<1>(N); run<2>(N); run<3>(N); } return 0; }
