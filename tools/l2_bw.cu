// Developer probe: L2 read bandwidth (32 MB working set, L2-resident) and HBM read bandwidth (2 GB).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const int4* __restrict__ p, size_t n, int iters, int4* out) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      int4 v = __ldcg(p + i);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if (acc.x == 0x12345) out[0] = acc;
}
int main() {
  int4 *buf, *out;
  size_t big = (size_t)2 << 30;
  cudaMalloc(&buf, big); cudaMalloc(&out, 64); cudaMemset(buf, 1, big);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (size_t ws : {(size_t)32 << 20, (size_t)64 << 20, big}) {
    size_t n = ws / 16; int iters = ws < big ? 50 : 3;
    rd<<<sms * 4, 512>>>(buf, n, 1, out);
    cudaEventRecord(a); rd<<<sms * 4, 512>>>(buf, n, iters, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("working set %zu MB: %.1f GB/s\n", ws >> 20, (double)ws * iters / (ms * 1e-3) / 1e9);
  }
  return 0;
}
