// gptq.cu — NEXT-4 offline weight preparation: randomized Hadamard incoherence processing and GPTQ,
// producing codes / scales / zeros in the S0a canonical format (mxm_quantize's), packable by mxm_pack.
//
// PAPER.md P:206 (§4.2.3) "we apply randomized Hadamard transformations to model weights using the incoherence
// processing used in QuaRot, then perform GPTQ-based quantization"; P:335 online rotations disabled. Readings
// DESIGN.md R22-R24 (the paper restates neither algorithm):
//   R22 Q = blockdiag_b(diag(sigma_b) H_128) / sqrt(128) on the hidden dim: W_gate Q, W_up Q, Q^T W_down.
//   R23 GPTQ (Frantar et al. 2022, Alg. 1, no act-order): H = 2 X^T X / n, dead columns, 1 % mean-diagonal damping,
//       U = upper Cholesky factor of H^-1, columns left to right in blocks of 128 with lazy batch updates.
//   R24 group parameters from the current (error-updated) weights at each group start (per channel: initial),
//       zero = largest bf16 <= x_min, scale = smallest bf16 s with c s >= x_max - zero (sym: max|x|).
// Everything in fp64 with explicit _rn intrinsics (no FMA contraction where the reading fixes an operation
// order), so the codes match the fp64 oracle's decisions.
#include <cuda_bf16.h>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace mxm {

namespace {

__device__ __forceinline__ double gbf(uint16_t b) { return (double)__uint_as_float((uint32_t)b << 16); }
__device__ __forceinline__ uint16_t bf_rn(double d) {
  __nv_bfloat16 h = __double2bfloat16(d);
  return *reinterpret_cast<uint16_t*>(&h);
}
// largest bf16 <= d (directed rounding twice in the same direction is one directed rounding)
__device__ __forceinline__ double bf_at_most(double d) {
  __nv_bfloat16 h = __float2bfloat16_rd(__double2float_rd(d));
  return (double)__bfloat162float(h);
}
// smallest positive bf16 s with c s >= D (D > 0); c s exact in fp64
__device__ double bf_at_least(double D, int c) {
  uint16_t b = bf_rn(D / (double)c);
  if (b == 0) b = 1;
  while (b > 1 && (double)c * gbf((uint16_t)(b - 1)) >= D) --b;
  while ((double)c * gbf(b) < D) ++b;
  return gbf(b);
}

// ---------------------------------------------------------------- R22: signs, FWHT-128, 1/sqrt(128), bf16 once
// one warp per 128-vector (lane l holds elements 4l..4l+3); axis 1: the vector runs along K (row n, block b);
// axis 0: along N (column k, block b)
__global__ void hadamard_kernel(const uint16_t* __restrict__ w, uint16_t* __restrict__ out, int64_t N, int64_t K,
                                const int8_t* __restrict__ sg, int axis) {
  const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  const int64_t L = axis == 1 ? K : N;  // rotated dimension
  const int64_t other = axis == 1 ? N : K;
  if (v >= other * (L / 128)) return;
  const int64_t o = v / (L / 128), b0 = (v % (L / 128)) * 128;
  auto at = [&](int i) -> int64_t { return axis == 1 ? o * K + b0 + i : (b0 + i) * K + o; };
  double x[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int i = 4 * lane + j;
    x[j] = (double)sg[b0 + i] * gbf(w[at(i)]);
  }
  // in-lane butterflies (strides 1, 2), then across lanes (strides 4 .. 64 = lane xor 1 .. 16); sums and
  // differences of bf16 values with ±1 signs are exact in fp64
  double a0 = x[0] + x[1], a1 = x[0] - x[1], a2 = x[2] + x[3], a3 = x[2] - x[3];
  x[0] = a0 + a2;
  x[1] = a1 + a3;
  x[2] = a0 - a2;
  x[3] = a1 - a3;
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const bool hi = (lane & m) != 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double y = __shfl_xor_sync(0xffffffffu, x[j], m);
      x[j] = hi ? y - x[j] : x[j] + y;
    }
  }
  const double r128 = __dsqrt_rn(128.0);  // the exact +-1 sums divided once by fl(sqrt(128)), then bf16 once
#pragma unroll
  for (int j = 0; j < 4; ++j) out[at(4 * lane + j)] = bf_rn(__ddiv_rn(x[j], r128));
}

// ---------------------------------------------------------------- R23: H = 2 X^T X / n (fp64, 32 x 32 tiles)
__global__ void hessian_kernel(const uint16_t* __restrict__ x, int64_t n, int64_t K, double* __restrict__ H) {
  __shared__ double a[32][33], b[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads, 4 outputs each
  const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  double acc[4] = {0, 0, 0, 0};
  for (int64_t r0 = 0; r0 < n; r0 += 32) {
    for (int t = ty; t < 32; t += 8) {
      const int64_t r = r0 + t;
      a[t][tx] = (r < n && i0 + tx < K) ? gbf(x[r * K + i0 + tx]) : 0.0;
      b[t][tx] = (r < n && j0 + tx < K) ? gbf(x[r * K + j0 + tx]) : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int t = 0; t < 32; ++t) {
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = __fma_rn(a[t][ty + 8 * q], b[t][tx], acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t i = i0 + ty + 8 * q, j = j0 + tx;
    if (i < K && j < K) H[i * K + j] = 2.0 * acc[q] / (double)n;
  }
}

// dead columns (H_jj == 0 -> 1), damping lambda = percdamp * mean(diag) (one block)
__global__ void damp_kernel(double* __restrict__ H, int64_t K, double percdamp, int32_t* __restrict__ dead) {
  __shared__ double part[1024];
  double s = 0;
  for (int64_t j = threadIdx.x; j < K; j += blockDim.x) {
    double h = H[j * K + j];
    const bool d = h == 0.0;
    if (d) h = 1.0;
    H[j * K + j] = h;
    dead[j] = d ? 1 : 0;
    s += h;
  }
  part[threadIdx.x] = s;
  __syncthreads();
  for (int m = blockDim.x / 2; m > 0; m >>= 1) {
    if ((int)threadIdx.x < m) part[threadIdx.x] += part[threadIdx.x + m];
    __syncthreads();
  }
  const double lam = percdamp * (part[0] / (double)K);
  for (int64_t j = threadIdx.x; j < K; j += blockDim.x) H[j * K + j] += lam;
}

// reverse (upper) Cholesky H = V V^T, right-looking from the bottom-right: step k updates the leading k x k
// block with the (unscaled) row k: A_ij -= A_ki A_kj / A_kk. Only the lower triangle (i >= j) is kept current,
// so the entries of column k above the diagonal are read as their mirror A_ki in row k.
__global__ void rchol_step_kernel(double* __restrict__ A, int64_t K, int64_t k) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = idx / k, j = idx % k;
  if (i >= k || j > i) return;
  const double akk = A[k * K + k];
  A[i * K + j] = __dsub_rn(A[i * K + j], __ddiv_rn(__dmul_rn(A[k * K + i], A[k * K + j]), akk));
}
// V (upper): V_kk = sqrt(A_kk), V_ik = A_ik / V_kk for i < k (A symmetric: read the lower triangle A_ki)
__global__ void rchol_final_kernel(const double* __restrict__ A, double* __restrict__ V, int64_t K) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= K * K) return;
  const int64_t i = idx / K, k = idx % K;
  double v = 0.0;
  if (i <= k) {
    const double vkk = __dsqrt_rn(A[k * K + k]);
    v = i == k ? vkk : __ddiv_rn(A[k * K + i], vkk);
  }
  V[i * K + k] = v;
}
// U = V^-1 (upper triangular): one block per column j, back substitution with a block-wide dot product per row
__global__ void triinv_kernel(const double* __restrict__ V, double* __restrict__ U, int64_t K) {
  const int64_t j = blockIdx.x;
  __shared__ double red[256];
  __shared__ double uj;
  for (int64_t i = threadIdx.x; i < K; i += blockDim.x) U[i * K + j] = 0.0;
  __syncthreads();
  if (threadIdx.x == 0) U[j * K + j] = 1.0 / V[j * K + j];
  __syncthreads();
  for (int64_t i = j - 1; i >= 0; --i) {
    double s = 0.0;
    for (int64_t k = i + 1 + threadIdx.x; k <= j; k += blockDim.x) s += V[i * K + k] * U[k * K + j];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int m = blockDim.x / 2; m > 0; m >>= 1) {
      if ((int)threadIdx.x < m) red[threadIdx.x] += red[threadIdx.x + m];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      uj = -red[0] / V[i * K + i];
      U[i * K + j] = uj;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- R23/R24: the column sweep
// work layout: W fp64 [N][K] (error-updated weights), Err fp64 [N][128] (the current block's scaled errors)
__global__ void gptq_init_kernel(const uint16_t* __restrict__ w, const int32_t* __restrict__ dead, int64_t N, int64_t K,
                                 double* __restrict__ W) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= N * K) return;
  W[idx] = dead[idx % K] ? 0.0 : gbf(w[idx]);
}

struct GParams {
  int bits, group, sym;
};

// group parameters of row r over columns [c0, c0 + len) of a row-major fp64 source (R24)
__device__ void params_of(const double* __restrict__ src, int64_t stride, int len, GParams g, double& s, double& z) {
  double mn = src[0], mx = src[0], am = fabs(src[0]);
  for (int i = 1; i < len; ++i) {
    const double v = src[(int64_t)i * stride];
    mn = fmin(mn, v);
    mx = fmax(mx, v);
    am = fmax(am, fabs(v));
  }
  if (g.sym) {
    const int c = (1 << (g.bits - 1)) - 1;
    s = am > 0 ? bf_at_least(am, c) : 1.0;
    z = 0.0;
  } else {
    const int c = (1 << g.bits) - 1;
    z = bf_at_most(mn);
    const double D = __dsub_rn(mx, z);
    s = D > 0 ? bf_at_least(D, c) : 1.0;
  }
}

constexpr int kGB = 128;    // GPTQ block (columns)
constexpr int kGRows = 64;  // rows per CTA of the sweep

// per-channel parameters from the initial (dead-zeroed) weights: one thread per row
__global__ void gptq_pc_params_kernel(const double* __restrict__ W, int64_t N, int64_t K, GParams g,
                                      double* __restrict__ ps, double* __restrict__ pz) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  double s, z;
  params_of(W + r * K, 1, (int)K, g, s, z);
  ps[r] = s;
  pz[r] = z;
}

// sweep of block [i1, i1 + B): one thread per row (kGRows rows per CTA), the block's columns of the CTA's rows
// in shared memory (column-major: consecutive rows -> consecutive banks), U's diagonal block broadcast from smem
__global__ void __launch_bounds__(kGRows) gptq_sweep_kernel(double* __restrict__ W, double* __restrict__ Err,
                                                            const double* __restrict__ U, int64_t N, int64_t K,
                                                            int64_t i1, int B, GParams g, const double* __restrict__ ps,
                                                            const double* __restrict__ pz, uint8_t* __restrict__ codes,
                                                            uint16_t* __restrict__ scale, uint16_t* __restrict__ zero) {
  extern __shared__ double sm[];
  double* ub = sm;                   // [B][B]
  double* wb = sm + kGB * kGB;       // [B][kGRows]
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kGRows, r = r0 + t;
  for (int i = t; i < B * B; i += kGRows) ub[i] = U[(i1 + i / B) * K + i1 + i % B];
  for (int i = 0; i < B; ++i) wb[i * kGRows + t] = r < N ? W[r * K + i1 + i] : 0.0;
  __syncthreads();
  if (r >= N) return;
  const int gsz = g.group == -1 ? (int)K : g.group;
  const int ng = (int)(K / gsz);
  double s = 0, z = 0;
  if (g.group == -1) {
    s = ps[r];
    z = pz[r];
  }
  for (int i = 0; i < B; ++i) {
    const int64_t j = i1 + i;
    if (g.group != -1 && j % gsz == 0) {  // group start inside this block (groups of 64 / 128 never straddle it)
      params_of(wb + i * kGRows + t, kGRows, gsz, g, s, z);
      scale[r * ng + j / gsz] = bf_rn(s);
      if (zero) zero[r * ng + j / gsz] = g.sym ? 0 : bf_rn(z);
    } else if (g.group == -1 && j == 0) {
      scale[r] = bf_rn(s);
      if (zero) zero[r] = g.sym ? 0 : bf_rn(z);
    }
    const double wv = wb[i * kGRows + t];
    double q, deq;
    if (g.sym) {
      const double c = (double)((1 << (g.bits - 1)) - 1);
      q = fmin(fmax(rint(__ddiv_rn(wv, s)), -c), c);
      deq = __dmul_rn(q, s);
      codes[r * K + j] = (uint8_t)(int8_t)(int)q;
    } else {
      const double c = (double)((1 << g.bits) - 1);
      q = fmin(fmax(rint(__ddiv_rn(__dsub_rn(wv, z), s)), 0.0), c);
      deq = __dadd_rn(__dmul_rn(q, s), z);
      codes[r * K + j] = (uint8_t)(int)q;
    }
    const double e = __ddiv_rn(__dsub_rn(wv, deq), ub[i * B + i]);
    Err[r * kGB + i] = e;
    for (int k = i + 1; k < B; ++k) wb[k * kGRows + t] = __dsub_rn(wb[k * kGRows + t], __dmul_rn(e, ub[i * B + k]));
  }
}

// lazy batch update W[:, i2:] -= Err[:, :B] U[i1:i2, i2:] (64-column x 16-row output tiles, fp64; the B-long
// reduction in two 64-long chunks so the static shared memory stays under 48 KB)
__global__ void gptq_update_kernel(double* __restrict__ W, const double* __restrict__ Err, const double* __restrict__ U,
                                   int64_t N, int64_t K, int64_t i1, int B) {
  __shared__ double ea[64][17], ub[64][65];
  const int64_t i2 = i1 + B;
  const int64_t c0 = i2 + (int64_t)blockIdx.x * 64, r0 = (int64_t)blockIdx.y * 16;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4 threads: 4 rows each
  double acc[4] = {0, 0, 0, 0};
  for (int k0 = 0; k0 < B; k0 += 64) {
    const int kn = B - k0 < 64 ? B - k0 : 64;
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) {
      const int rr = i % 16, kk = i / 16;
      ea[kk][rr] = (kk < kn && r0 + rr < N) ? Err[(r0 + rr) * kGB + k0 + kk] : 0.0;
    }
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
      const int cc = i % 64, kk = i / 64;
      ub[kk][cc] = (kk < kn && c0 + cc < K) ? U[(i1 + k0 + kk) * K + c0 + cc] : 0.0;
    }
    __syncthreads();
    for (int kk = 0; kk < kn; ++kk) {
      const double u = ub[kk][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = __fma_rn(ea[kk][ty + 4 * q], u, acc[q]);
    }
  }
  const int64_t c = c0 + tx;
  if (c >= K) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t rr = r0 + ty + 4 * q;
    if (rr < N) W[rr * K + c] = __dsub_rn(W[rr * K + c], acc[q]);
  }
}

}  // namespace

cudaError_t launch_hadamard(const void* w, void* out, int64_t N, int64_t K, const int8_t* signs, int axis,
                            cudaStream_t st) {
  const int64_t L = axis == 1 ? K : N, other = axis == 1 ? N : K;
  const int64_t warps = other * (L / 128);
  if (warps <= 0) return cudaSuccess;
  hadamard_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>((const uint16_t*)w, (uint16_t*)out, N, K,
                                                                        signs, axis);
  return cudaGetLastError();
}

cudaError_t launch_gptq_hessian(const void* x, int64_t n, int64_t K, double* H, cudaStream_t st) {
  dim3 grid((unsigned)((K + 31) / 32), (unsigned)((K + 31) / 32));
  hessian_kernel<<<grid, 256, 0, st>>>((const uint16_t*)x, n, K, H);
  return cudaGetLastError();
}

cudaError_t launch_gptq_prepare(double* H, int64_t K, double percdamp, double* V, double* U, int32_t* dead,
                                cudaStream_t st) {
  damp_kernel<<<1, 1024, 0, st>>>(H, K, percdamp, dead);
  for (int64_t k = K - 1; k >= 1; --k) {
    const int64_t n = k * k;
    rchol_step_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(H, K, k);
  }
  rchol_final_kernel<<<(unsigned)((K * K + 255) / 256), 256, 0, st>>>(H, V, K);
  triinv_kernel<<<(unsigned)K, 256, 0, st>>>(V, U, K);
  return cudaGetLastError();
}

cudaError_t launch_gptq_quantize(int bits, int group, int sym, const void* w, int64_t N, int64_t K, const double* U,
                                 const int32_t* dead, double* work, void* codes, void* scale, void* zero,
                                 cudaStream_t st) {
  double* W = work;
  double* Err = W + N * K;
  double* ps = Err + N * kGB;
  double* pz = ps + N;
  const GParams g{bits, group, sym};
  gptq_init_kernel<<<(unsigned)((N * K + 255) / 256), 256, 0, st>>>((const uint16_t*)w, dead, N, K, W);
  if (group == -1) gptq_pc_params_kernel<<<(unsigned)((N + 127) / 128), 128, 0, st>>>(W, N, K, g, ps, pz);
  const size_t smem = sizeof(double) * (kGB * kGB + kGB * kGRows);
  cudaError_t e = cudaFuncSetAttribute(gptq_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  for (int64_t i1 = 0; i1 < K; i1 += kGB) {
    const int B = (int)(K - i1 < kGB ? K - i1 : kGB);
    gptq_sweep_kernel<<<(unsigned)((N + kGRows - 1) / kGRows), kGRows, smem, st>>>(
        W, Err, U, N, K, i1, B, g, ps, pz, (uint8_t*)codes, (uint16_t*)scale, (uint16_t*)zero);
    if (i1 + B < K) {
      dim3 grid((unsigned)((K - i1 - B + 63) / 64), (unsigned)((N + 15) / 16));
      gptq_update_kernel<<<grid, 256, 0, st>>>(W, Err, U, N, K, i1, B);
    }
  }
  return cudaGetLastError();
}

int64_t gptq_work_doubles(int64_t N, int64_t K) { return N * K + N * kGB + 2 * N; }

}  // namespace mxm
