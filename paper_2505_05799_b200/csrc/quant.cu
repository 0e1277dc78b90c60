// quant.cu — setup kernels: weight quantizer (S0a), packer (S0b), debug dequantizer,
// and the standalone activation quantizer entry (quant_row_warp, the hot path's gate/up input quantizer).
//
// Weight quantizer Q (§2.1; 16-bit meta P:339; groups along K P:452), readings
// DESIGN.md R1-R7: fp64 arithmetic, stored scale = smallest bf16 s with c*s >= range, codes
// rint((x - z)/s) clamped. Independent of the CPU oracle; parity is checked bit-exactly.
#include <cuda_bf16.h>
#include <cstdint>

#include "actq.cuh"
#include "common.cuh"
#include "kernels.h"

namespace mxm {

__device__ __forceinline__ double bf16_bits_to_double(uint16_t b) { return (double)__uint_as_float((uint32_t)b << 16); }
__device__ __forceinline__ uint16_t double_to_bf16_rn(double d) {
  __nv_bfloat16 h = __double2bfloat16(d);  // cvt.rn.bf16.f64: single rounding
  return *reinterpret_cast<uint16_t*>(&h);
}

// smallest positive bf16 s with c*s >= D (D > 0); c*s is exact in fp64
__device__ double smallest_bf16_at_least(double D, int c) {
  uint16_t b = double_to_bf16_rn(D / (double)c);
  if (b == 0) b = 1;
  while (b > 1 && (double)c * bf16_bits_to_double((uint16_t)(b - 1)) >= D) --b;
  while ((double)c * bf16_bits_to_double(b) < D) ++b;
  return bf16_bits_to_double(b);
}

// one thread per (row, group)
__global__ void quantize_kernel(const uint16_t* __restrict__ w, int64_t N, int64_t K, int bits, int group, int sym,
                                uint8_t* __restrict__ codes, uint16_t* __restrict__ scale, uint16_t* __restrict__ zero,
                                int32_t* err) {
  const int64_t ng = K / group;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= N * ng) return;
  const int64_t n = idx / ng, gi = idx % ng;
  const uint16_t* src = w + n * K + gi * group;
  uint8_t* dst = codes + n * K + gi * group;
  bool finite = true;
  double xmin = 0, xmax = 0, amax = 0;
  for (int i = 0; i < group; ++i) {
    double x = bf16_bits_to_double(src[i]);
    if (!isfinite(x)) finite = false;
    if (i == 0) xmin = xmax = x;
    xmin = fmin(xmin, x);
    xmax = fmax(xmax, x);
    amax = fmax(amax, fabs(x));
  }
  if (!finite && err) atomicExch(err, (int32_t)MXM_E_DATA);
  double s, z = 0;
  if (bits == -8) {  // FP8 e4m3 (R25): s = smallest bf16 with 448 s >= max|w|, code = e4m3_rn(w / s)
    s = amax > 0 ? smallest_bf16_at_least(amax, 448) : 1.0;
    for (int i = 0; i < group; ++i) dst[i] = (uint8_t)e4m3_rn(__ddiv_rn(bf16_bits_to_double(src[i]), s));
    if (zero) zero[n * ng + gi] = 0;
  } else if (!sym) {
    const int c = (1 << bits) - 1;
    const double D = xmax - xmin;
    s = D > 0 ? smallest_bf16_at_least(D, c) : 1.0;
    z = xmin;
    for (int i = 0; i < group; ++i) {
      double q = rint(__ddiv_rn(__dsub_rn(bf16_bits_to_double(src[i]), z), s));
      q = fmin(fmax(q, 0.0), (double)c);
      dst[i] = (uint8_t)(int)q;
    }
    zero[n * ng + gi] = double_to_bf16_rn(z);
  } else {
    const int c = (1 << (bits - 1)) - 1;
    s = amax > 0 ? smallest_bf16_at_least(amax, c) : 1.0;
    for (int i = 0; i < group; ++i) {
      double q = rint(__ddiv_rn(bf16_bits_to_double(src[i]), s));
      q = fmin(fmax(q, (double)-c), (double)c);
      dst[i] = (uint8_t)(int8_t)(int)q;
    }
    if (zero) zero[n * ng + gi] = 0;
  }
  scale[n * ng + gi] = double_to_bf16_rn(s);
}

// ---------------------------------------------------------------- pack (docs/packed_format.md)
__device__ __forceinline__ int field_pos(bool i8kind, int pb, int i) {
  if (!i8kind) {
    if (pb == 2) return (i >> 1) + 8 * (i & 1);
    if (pb == 1) return (i >> 1) + 16 * (i & 1);
    if (pb == 4) return (i >> 1) + 4 * (i & 1);
    return i;  // pb == 8
  }
  if (pb == 4) return i < 4 ? 2 * i : 2 * (i - 4) + 1;
  return 8 * (i & 3) + (i >> 2);  // pb == 1
}

// stored value u of canonical code at (n, k)
__device__ __forceinline__ uint32_t stored_code(const PackGeom& g, const uint8_t* codes, int64_t n, int64_t k) {
  const uint8_t c = codes[n * g.K + k];
  if (g.kind == KIND_WO && !g.sym) return c;
  if (g.kind == KIND_WA_IMG) return c;  // two's complement byte
  return (uint32_t)((int)(int8_t)c + (1 << (g.w_bits - 1)));
}

// grid: (ns, rb), block: 128 threads (one per row of the chunk)
__global__ void pack_kernel(PackGeom g, const uint8_t* __restrict__ codes, const uint16_t* __restrict__ scale,
                            const uint16_t* __restrict__ zero, uint8_t* __restrict__ out) {
  const int ks = blockIdx.x, rb = blockIdx.y, r = threadIdx.x;
  const int64_t n = (int64_t)rb * 128 + r;
  const int64_t k0 = (int64_t)ks * g.ks;
  uint8_t* chunk = out + chunk_offset(g, rb, ks);
  if (g.kind == KIND_W16 || g.kind == KIND_WA_IMG || g.kind == KIND_FP8) {
    // row r: 128 bytes of K-slice; byte b at r*128 + ((b>>4 ^ r&7)<<4) + (b&15)
    const uint8_t* src = (g.kind == KIND_W16) ? codes + (n * g.K + k0) * 2 : codes + n * g.K + k0;
    for (int c = 0; c < 8; ++c) {
      uint4 v = *reinterpret_cast<const uint4*>(src + c * 16);
      *reinterpret_cast<uint4*>(chunk + r * 128 + ((c ^ (r & 7)) << 4)) = v;
    }
  } else {
    const bool i8k = kind_is_row8(g.kind);
    uint8_t* p = chunk;
    if (chunk_has_meta(g, ks)) {
      const int64_t gi = k0 / g.group, ng = g.K / g.group;
      reinterpret_cast<uint16_t*>(p)[r] = scale[n * ng + gi];
      p += 256;
      if (!g.sym) {
        reinterpret_cast<uint16_t*>(p)[r] = zero[n * ng + gi];
        p += 256;
      }
    }
    const int planes[2] = {g.w_bits == 3 ? 2 : (g.w_bits == 5 ? 4 : g.w_bits), (g.w_bits == 3 || g.w_bits == 5) ? 1 : 0};
    int shift = 0;
    for (int pi = 0; pi < 2; ++pi) {
      const int pb = planes[pi];
      if (pb == 0) break;
      const int per_word = 32 / pb, W = g.ks / per_word;
      for (int j = 0; j < W; ++j) {
        uint32_t word = 0;
        for (int ii = 0; ii < per_word; ++ii) {
          uint32_t u = (stored_code(g, codes, n, k0 + j * per_word + ii) >> shift) & ((1u << pb) - 1);
          word |= u << (field_pos(i8k, pb, ii) * pb);
        }
        reinterpret_cast<uint32_t*>(p)[j * 128 + r] = word;
      }
      p += (size_t)W * 128 * 4;
      shift += pb;
    }
  }
  if (kind_is_wa(g.kind) && ks == 0) {
    const int64_t ng = g.K / g.group;
    uint16_t* sc = reinterpret_cast<uint16_t*>(out + g.wa_scale_off);
    for (int64_t gi = 0; gi < ng; ++gi) sc[gi * g.N + n] = scale[n * ng + gi];
  }
}

// ---------------------------------------------------------------- dequantize (debug)
__device__ uint32_t read_stored_code(const PackGeom& g, const uint8_t* packed, int64_t n, int64_t k) {
  const int rb = (int)(n / 128), r = (int)(n % 128), ks = (int)(k / g.ks), i = (int)(k % g.ks);
  const uint8_t* chunk = packed + chunk_offset(g, rb, ks);
  if (g.kind == KIND_WA_IMG || g.kind == KIND_FP8) {
    const int b = i;
    return chunk[r * 128 + (((b >> 4) ^ (r & 7)) << 4) + (b & 15)];
  }
  const bool i8k = kind_is_row8(g.kind);
  const uint8_t* p = chunk + (chunk_has_meta(g, ks) ? g.meta_bytes : 0);
  const int planes[2] = {g.w_bits == 3 ? 2 : (g.w_bits == 5 ? 4 : g.w_bits), (g.w_bits == 3 || g.w_bits == 5) ? 1 : 0};
  uint32_t u = 0;
  int shift = 0;
  for (int pi = 0; pi < 2; ++pi) {
    const int pb = planes[pi];
    if (pb == 0) break;
    const int per_word = 32 / pb, W = g.ks / per_word;
    const int j = i / per_word, ii = i % per_word;
    uint32_t word = reinterpret_cast<const uint32_t*>(p)[j * 128 + r];
    u |= ((word >> (field_pos(i8k, pb, ii) * pb)) & ((1u << pb) - 1)) << shift;
    p += (size_t)W * 128 * 4;
    shift += pb;
  }
  return u;
}

__global__ void dequant_kernel(PackGeom g, const uint8_t* __restrict__ packed, float* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)g.N * g.K) return;
  const int64_t n = idx / g.K, k = idx % g.K;
  if (g.kind == KIND_W16) {
    const int rb = (int)(n / 128), r = (int)(n % 128), ks = (int)(k / 64), b = (int)(k % 64) * 2;
    const uint8_t* chunk = packed + chunk_offset(g, rb, ks);
    uint16_t v = *reinterpret_cast<const uint16_t*>(chunk + r * 128 + (((b >> 4) ^ (r & 7)) << 4) + (b & 15));
    out[idx] = bf16_bits_to_float(v);
    return;
  }
  const uint32_t u = read_stored_code(g, packed, n, k);
  const int gi = (int)(k / g.group);
  double s, z = 0;
  int q;
  if (g.kind == KIND_FP8) {
    s = bf16_bits_to_double(reinterpret_cast<const uint16_t*>(packed + g.wa_scale_off)[(int64_t)gi * g.N + n]);
    out[idx] = (float)((double)e4m3_value(u) * s);
    return;
  }
  if (kind_is_wa(g.kind)) {
    q = g.kind == KIND_WA_IMG ? (int)(int8_t)u : (int)u - (1 << (g.w_bits - 1));
    s = bf16_bits_to_double(reinterpret_cast<const uint16_t*>(packed + g.wa_scale_off)[(int64_t)gi * g.N + n]);
  } else {
    const int ksm = (int)(((int64_t)gi * g.group) / g.ks);  // chunk holding this group's meta
    const uint8_t* meta = packed + chunk_offset(g, (int)(n / 128), ksm);
    s = bf16_bits_to_double(reinterpret_cast<const uint16_t*>(meta)[n % 128]);
    if (!g.sym) z = bf16_bits_to_double(reinterpret_cast<const uint16_t*>(meta + 256)[n % 128]);
    q = g.sym ? (int)u - (1 << (g.w_bits - 1)) : (int)u;
  }
  out[idx] = (float)((double)q * s + z);
}

// ---------------------------------------------------------------- activation quantizer (debug entry)
// One warp per row, through the hot path's gate/up input quantizer (quant_row_warp, actq.cuh; route.cu gather)
// with canonical two's complement codes; rows longer than 4096 use its per-group fallback (quant_group_warp).
// The gather writes group-major [g][R] scales; here row-major [M][K/g] (stride 1 between groups of a row).
__global__ void act_quant_kernel(const uint16_t* __restrict__ v, int64_t M, int64_t K, int a_bits, int group,
                                 int8_t* __restrict__ codes, float* __restrict__ scale, int32_t* __restrict__ qsum) {
  const int64_t ng = K / group;
  const int64_t m = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (m >= M) return;
  const int qmax = (1 << (a_bits - 1)) - 1;
  if (K <= 128 * 32) {
    quant_row_warp<32, false>(v + m * K, codes + m * K, (int)K, group, qmax, scale + m * ng,
                              qsum ? qsum + m * ng : nullptr, 1);
    return;
  }
  for (int64_t gi = 0; gi < ng; ++gi) {
    int qs;
    const float s = quant_group_warp<false, false>(v + m * K + gi * group, codes + m * K + gi * group, group, qmax, &qs);
    if ((threadIdx.x & 31) == 0) {
      scale[m * ng + gi] = s;
      if (qsum) qsum[m * ng + gi] = qs;
    }
  }
}

// ---------------------------------------------------------------- host launchers
cudaError_t launch_quantize(const PackGeom& g, const void* w, void* codes, void* scale, void* zero, int32_t* err,
                            cudaStream_t st) {
  const int64_t n = (int64_t)g.N * (g.K / g.group);
  quantize_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(
      (const uint16_t*)w, g.N, g.K, g.kind == KIND_FP8 ? -8 : g.w_bits, g.group, g.sym, (uint8_t*)codes,
      (uint16_t*)scale, (uint16_t*)zero, err);
  return cudaGetLastError();
}
cudaError_t launch_pack(const PackGeom& g, const void* codes, const void* scale, const void* zero, void* out,
                        cudaStream_t st) {
  dim3 grid(g.ns, g.N / 128);
  pack_kernel<<<grid, 128, 0, st>>>(g, (const uint8_t*)codes, (const uint16_t*)scale, (const uint16_t*)zero,
                                    (uint8_t*)out);
  return cudaGetLastError();
}
cudaError_t launch_dequantize(const PackGeom& g, const void* packed, float* out, cudaStream_t st) {
  const int64_t n = (int64_t)g.N * g.K;
  dequant_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, (const uint8_t*)packed, out);
  return cudaGetLastError();
}
cudaError_t launch_act_quant(const void* v, int64_t M, int64_t K, int a_bits, int group, void* codes, float* scale,
                             int32_t* qsum, cudaStream_t st) {
  const int64_t warps = M;
  act_quant_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(
      (const uint16_t*)v, M, K, a_bits, group, (int8_t*)codes, scale, qsum);
  return cudaGetLastError();
}

}  // namespace mxm
