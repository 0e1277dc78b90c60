// actq.cuh — dynamic symmetric activation quantizer, one warp per group.
// Definition (R9): amax = max|v|; amax == 0 -> s = 1, q = 0; else
//   r = fl32(qmax / amax), s = fl32(amax / qmax), q = clamp(rint(fl32(v * r)), -qmax, qmax).
// IEEE fp32 with explicit _rn intrinsics (no fast-math anywhere in this library).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace mxm {

__device__ __forceinline__ float bf16_bits_to_float(uint32_t b) { return __uint_as_float(b << 16); }

// warp max of non-negative floats (|v|): their bit patterns order like the values, so one REDUX.MAX does it
__device__ __forceinline__ float warp_max(float v) {
  return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(v)));
}
__device__ __forceinline__ int warp_sum(int v) { return __reduce_add_sync(0xffffffffu, v); }

// Code byte of an integer code q (|q| <= 127): two's complement int8 (kind::i8 operands, canonical output), or
// for E4 the e4m3 byte (q<0)<<7 | |q| whose value is q * 2^-9 (|q| <= 15; kind::f8f6f4 operands of w4a4 blocks).
template <bool E4>
__device__ __forceinline__ uint32_t code_byte(int q) {
  if constexpr (E4)
    return (q < 0 ? 0x80u : 0u) | (uint32_t)(q < 0 ? -q : q);
  else
    return (uint32_t)q & 0xFFu;
}

// e4m3 (OCP FP8 E4M3) code of a value with |a| <= 448, round to nearest, ties to the even mantissa (DESIGN R25 /
// R26): exact from fp64 (the scalings by powers of two and the mantissa split are exact, rint rounds once).
__device__ __forceinline__ uint32_t e4m3_rn(double a) {
  const uint32_t sgn = signbit(a) ? 0x80u : 0u;
  const double m = fabs(a);
  uint32_t code;
  if (m < 0.015625) {  // below 2^-6: the subnormal grid m 2^9 (rounds up to code 8 = 2^-6 at the boundary)
    code = (uint32_t)rint(m * 512.0);
  } else {
    int e;
    const double f = frexp(m, &e);  // m = f 2^e, f in [0.5, 1): m = (1 + t) 2^(e-1), t = 2f - 1 exact
    uint32_t q = (uint32_t)rint((2.0 * f - 1.0) * 8.0);
    int E = e - 1 + 7;
    if (q == 8) {
      q = 0;
      ++E;
    }
    code = ((uint32_t)E << 3) | q;
  }
  if (code > 0x7Eu) code = 0x7Eu;
  return sgn | code;
}
// value of an e4m3 code (finite codes)
__device__ __forceinline__ float e4m3_value(uint32_t c) {
  const uint32_t e = (c >> 3) & 15u, m = c & 7u;
  const float v = e == 0 ? (float)m * 0.001953125f : ldexpf(1.0f + (float)m * 0.125f, (int)e - 7);
  return (c & 0x80u) ? -v : v;
}
// FP8 activation code of v under the row / group reciprocal r (R26): e4m3_rn(clamp(fl32(v r), +-448))
__device__ __forceinline__ uint32_t fp8_act_code(float v, float r) {
  const float p = fminf(fmaxf(__fmul_rn(v, r), -448.f), 448.f);
  return e4m3_rn((double)p);
}

// Quantize `n` bf16 values src[0..n) (n % 256 == 0 or n == 128: each lane handles 4- or 8-element
// vectors) into dst codes, return the group scale; whole warp participates.
// src may be global (generic pointer). Uses 8-byte (4 x bf16) vector loads.
template <bool kCoherent = false, bool E4 = false>
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
      packed |= code_byte<E4>(qi) << (8 * j);
    }
    *reinterpret_cast<uint32_t*>(dst + i) = packed;
  }
  if (qsum_out) *qsum_out = warp_sum(qs);
  return s;
}

// One whole row of d bf16 values (d % 128 == 0, d <= 128 * MAXG) quantized by one warp in groups of g
// (128, or g == d for per-token scales): the row is loaded once into registers (lane l holds elements
// 128*i + 4l .. +3 of chunk i), all loads in flight together; same arithmetic as quant_group_warp.
// Scales go to sc[gi * R], code sums (if qs != nullptr) to qs[gi * R] (group-major [g][R]).
// The hot path's gate/up input quantizer (route.cu gather) and the mxm_act_quant debug entry both call it.
// FP8 (R26): codes e4m3_rn(clamp(fl32(v r))) with qmax = 448 and r = fl32(448 / amax); code sums stay 0.
template <int MAXG, bool E4, bool FP8 = false>
__device__ __forceinline__ void quant_row_warp(const uint16_t* __restrict__ src, int8_t* __restrict__ dst, int d, int g,
                                               int qmax, float* __restrict__ sc, int32_t* __restrict__ qs,
                                               int64_t R) {
  const int lane = threadIdx.x & 31;
  const int nch = d / 128;
  uint2 v[MAXG];
#pragma unroll
  for (int i = 0; i < MAXG; ++i)
    if (i < nch) v[i] = *reinterpret_cast<const uint2*>(src + 128 * i + 4 * lane);
  auto absmax4 = [](uint2 x) {
    return fmaxf(fmaxf(fabsf(bf16_bits_to_float(x.x & 0xFFFFu)), fabsf(bf16_bits_to_float(x.x >> 16))),
                 fmaxf(fabsf(bf16_bits_to_float(x.y & 0xFFFFu)), fabsf(bf16_bits_to_float(x.y >> 16))));
  };
  const float fq = FP8 ? 448.f : (float)qmax;
  auto quant4 = [&](uint2 x, float r, int& qsum) {
    const float f[4] = {bf16_bits_to_float(x.x & 0xFFFFu), bf16_bits_to_float(x.x >> 16),
                        bf16_bits_to_float(x.y & 0xFFFFu), bf16_bits_to_float(x.y >> 16)};
    uint32_t packed = 0;
    if constexpr (FP8) {
#pragma unroll
      for (int j = 0; j < 4; ++j) packed |= fp8_act_code(f[j], r) << (8 * j);
      return packed;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float q = rintf(__fmul_rn(f[j], r));
      q = fminf(fmaxf(q, -fq), fq);
      qsum += (int)q;
      packed |= code_byte<E4>((int)q) << (8 * j);
    }
    return packed;
  };
  if (g == 128) {  // one group per 128-element chunk
#pragma unroll
    for (int i = 0; i < MAXG; ++i) {
      if (i < nch) {
        const float amax = warp_max(absmax4(v[i]));
        float r = 0.f, s = 1.f;
        if (amax > 0.f) {
          r = __fdiv_rn(fq, amax);
          s = __fdiv_rn(amax, fq);
        }
        int qsum = 0;
        *reinterpret_cast<uint32_t*>(dst + 128 * i + 4 * lane) = quant4(v[i], r, qsum);
        if (qs) qsum = warp_sum(qsum);
        if (lane == 0) {
          sc[(int64_t)i * R] = s;
          if (qs) qs[(int64_t)i * R] = qsum;
        }
      }
    }
  } else {  // per token: one group = the row
    float amax = 0.f;
#pragma unroll
    for (int i = 0; i < MAXG; ++i)
      if (i < nch) amax = fmaxf(amax, absmax4(v[i]));
    amax = warp_max(amax);
    float r = 0.f, s = 1.f;
    if (amax > 0.f) {
      r = __fdiv_rn(fq, amax);
      s = __fdiv_rn(amax, fq);
    }
    int qsum = 0;
#pragma unroll
    for (int i = 0; i < MAXG; ++i)
      if (i < nch) *reinterpret_cast<uint32_t*>(dst + 128 * i + 4 * lane) = quant4(v[i], r, qsum);
    if (qs) qsum = warp_sum(qsum);
    if (lane == 0) {
      sc[0] = s;
      if (qs) qs[0] = qsum;
    }
  }
}

}  // namespace mxm
