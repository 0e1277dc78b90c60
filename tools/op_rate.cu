// op_rate.cu — per-SM issue throughput of the CUDA-core instructions the dequant / drain paths use
// (dev probe): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/op_rate tools/op_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

constexpr int kChains = 8, kIters = 4096;

template <int OP>
__global__ void rate(uint32_t* out, unsigned long long* cyc, uint32_t seed) {
  uint32_t v[kChains];
  float f[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) { v[c] = seed * (threadIdx.x + 1) + c; f[c] = (float)v[c]; }
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if constexpr (OP == 0) {  // I2F (cvt.rn.f32.s32), chained through the bits
        f[c] = (float)(int32_t)v[c]; v[c] = __float_as_uint(f[c]) ^ seed;
      } else if constexpr (OP == 1) {  // bf16x2 fma
        __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&v[c]);
        __nv_bfloat162 s = *reinterpret_cast<__nv_bfloat162*>(&seed);
        a = __hfma2(a, s, s); v[c] = *reinterpret_cast<uint32_t*>(&a);
      } else if constexpr (OP == 2) {  // lop3
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xea;" : "+r"(v[c]) : "r"(seed), "r"(0x43004300u));
      } else if constexpr (OP == 3) {  // shift
        asm volatile("shf.r.wrap.b32 %0, %0, %0, %1;" : "+r"(v[c]) : "r"(seed & 31));
      } else if constexpr (OP == 4) {  // f32x2 fma
        unsigned long long x = ((unsigned long long)v[c] << 32) | v[c], r;
        asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(r) : "l"(x));
        v[c] = (uint32_t)r ^ (uint32_t)(r >> 32);
      } else if constexpr (OP == 5) {  // fp32 fma
        f[c] = fmaf(f[c], 1.0001f, 0.5f); v[c] = __float_as_uint(f[c]);
      } else if constexpr (OP == 6) {  // iadd
        asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(seed));
      }
    }
  }
  const unsigned long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc ^= v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int threads) {
  uint32_t* out; unsigned long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  rate<OP><<<148, threads>>>(out, cyc, 0x3f813f81u);
  rate<OP><<<148, threads>>>(out, cyc, 0x3f813f81u);
  cudaDeviceSynchronize();
  unsigned long long c[148];
  cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
  double ops = (double)threads * kChains * kIters;
  printf("%-10s threads/SM %4d : %6.1f lane-ops/clk/SM (%.2f cycles per warp-instr per SMSP)\n", name, threads,
         ops / c[0], 32.0 * 4 / (ops / c[0]));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int th : {256, 512}) {
    run<0>("I2F", th); run<1>("HFMA2.BF16", th); run<2>("LOP3", th); run<3>("SHF", th);
    run<4>("FFMA2", th); run<5>("FFMA", th); run<6>("IADD", th);
  }
  return 0;
}
