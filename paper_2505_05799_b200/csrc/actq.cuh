// actq.cuh — dynamic symmetric activation quantizer, one warp per group.
// Definition (R9): amax = max|v|; amax == 0 -> s = 1, q = 0; else
//   r = fl32(qmax / amax), s = fl32(amax / qmax), q = clamp(rint(fl32(v * r)), -qmax, qmax).
// IEEE fp32 with explicit _rn intrinsics (no fast-math anywhere in this library).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace mxm {

__device__ __forceinline__ float bf16_bits_to_float(uint32_t b) { return __uint_as_float(b << 16); }

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Quantize `n` bf16 values src[0..n) (n % 256 == 0 or n == 128: each lane handles 4- or 8-element
// vectors) into dst codes, return the group scale; whole warp participates.
// src may be global (generic pointer). Uses 8-byte (4 x bf16) vector loads.
template <bool kCoherent = false>
__device__ __forceinline__ float quant_group_warp(const uint16_t* src, int8_t* __restrict__ dst, int n, int qmax,
                                                  int* qsum_out) {
  const int lane = threadIdx.x & 31;
  float amax = 0.f;
  for (int i = lane * 4; i < n; i += 128) {
    uint2 v = kCoherent ? __ldcg(reinterpret_cast<const uint2*>(src + i)) : *reinterpret_cast<const uint2*>(src + i);
    amax = fmaxf(amax, fabsf(bf16_bits_to_float(v.x & 0xFFFFu)));
    amax = fmaxf(amax, fabsf(bf16_bits_to_float(v.x >> 16)));
    amax = fmaxf(amax, fabsf(bf16_bits_to_float(v.y & 0xFFFFu)));
    amax = fmaxf(amax, fabsf(bf16_bits_to_float(v.y >> 16)));
  }
  amax = warp_max(amax);
  const float fq = (float)qmax;
  float r = 0.f, s = 1.f;
  if (amax > 0.f) {
    r = __fdiv_rn(fq, amax);
    s = __fdiv_rn(amax, fq);
  }
  int qs = 0;
  for (int i = lane * 4; i < n; i += 128) {
    uint2 v = kCoherent ? __ldcg(reinterpret_cast<const uint2*>(src + i)) : *reinterpret_cast<const uint2*>(src + i);
    float f[4] = {bf16_bits_to_float(v.x & 0xFFFFu), bf16_bits_to_float(v.x >> 16), bf16_bits_to_float(v.y & 0xFFFFu),
                  bf16_bits_to_float(v.y >> 16)};
    uint32_t packed = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float q = rintf(__fmul_rn(f[j], r));
      q = fminf(fmaxf(q, -fq), fq);
      int qi = (int)q;
      qs += qi;
      packed |= (uint32_t)(qi & 0xFF) << (8 * j);
    }
    *reinterpret_cast<uint32_t*>(dst + i) = packed;
  }
  if (qsum_out) *qsum_out = warp_sum(qs);
  return s;
}

}  // namespace mxm
