// gemv_probe.cu -- dev probe (not product code): how fast can a CUDA-core GEMV run a weight-only w4a16-g128
// expert at tiny m, against the tcgen05 path's measured 0.85 TB/s at m = 8 (profiles/r02/isolation_ncu.txt)?
// Sizes a "CUDA-core path for tiny-M experts" before building one into the persistent kernel.
// Layout (probe-only, not the product's packed format): q[N][K/8] uint32 (8 nibbles along k), per-row per-128
// group scale and zero (bf16, w = q*s + z), x[m][K] bf16, y[m][N] fp32. Persistent grid, one warp per output
// row, x staged once per block in shared memory; lane l of chunk c holds k = 256c + 8l .. +8.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gemv_probe tools/gemv_probe.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cmath>

template <int M>
__global__ void __launch_bounds__(256) gemv_w4(const uint32_t* __restrict__ q, const __nv_bfloat162* __restrict__ sz,
                                               const __nv_bfloat16* __restrict__ x, float* __restrict__ y, int N,
                                               int K) {
  extern __shared__ __align__(16) __nv_bfloat16 xs[];  // [M][K]
  for (int i = threadIdx.x * 8; i < M * K; i += blockDim.x * 8)
    *reinterpret_cast<uint4*>(xs + i) = *reinterpret_cast<const uint4*>(x + i);
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nch = K / 256, ng = K / 128;
  for (int n = blockIdx.x * 8 + wib; n < N; n += gridDim.x * 8) {
    const uint32_t* qr = q + (size_t)n * (K / 8);
    const __nv_bfloat162* szr = sz + (size_t)n * ng;
    float acc[M];
#pragma unroll
    for (int i = 0; i < M; ++i) acc[i] = 0.f;
    uint32_t wv[16];
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c < nch) wv[c] = __ldcs(qr + c * 32 + lane);
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      if (c >= nch) break;
      const float2 s_z = __bfloat1622float2(szr[2 * c + (lane >> 4)]);
      float w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float qf = __int_as_float(0x4B000000 | ((wv[c] >> (4 * j)) & 15u)) - 8388608.f;
        w[j] = fmaf(qf, s_z.x, s_z.y);
      }
      const int k0 = c * 256 + lane * 8;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        const uint4 xv = *reinterpret_cast<const uint4*>(xs + i * K + k0);
        const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&xv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 xf = __bfloat1622float2(xp[j]);
          acc[i] = fmaf(w[2 * j], xf.x, acc[i]);
          acc[i] = fmaf(w[2 * j + 1], xf.y, acc[i]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
      float v = acc[i];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) y[(size_t)i * N + n] = v;
    }
  }
}


// v2: 16-B weight loads (lane = 32 consecutive k of one 1024-k chunk, one group scale per chunk), two rows per
// warp in flight, nibble pairs dequantized as bf16x2 with the 0x4300 magic (w = (128 + q) s + (z - 128 s)),
// fp32 accumulation
template <int M>
__global__ void __launch_bounds__(256) gemv_w4_v2(const uint32_t* __restrict__ q, const __nv_bfloat162* __restrict__ sz,
                                                  const __nv_bfloat16* __restrict__ x, float* __restrict__ y, int N,
                                                  int K) {
  extern __shared__ __align__(16) __nv_bfloat16 xs[];  // [M][K]
  for (int i = threadIdx.x * 8; i < M * K; i += blockDim.x * 8)
    *reinterpret_cast<uint4*>(xs + i) = *reinterpret_cast<const uint4*>(x + i);
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nch = K / 1024, ng = K / 128;
  constexpr int R = 2;
  for (int n0 = (blockIdx.x * 8 + wib) * R; n0 < N; n0 += gridDim.x * 8 * R) {
    uint4 wv[R][4];
    float2 szf[R][4];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (c < nch && n0 + r < N) {
          // chunk c of row n0 + r: k = 1024 c + 32 lane .. +32 = words 128 c + 4 lane .. +4 (the probe's q layout
          // groups 8 nibbles per word along k; here the word order is re-read as 4 consecutive words per lane)
          wv[r][c] = __ldcs(reinterpret_cast<const uint4*>(q + (size_t)(n0 + r) * (K / 8) + 128 * c + 4 * lane));
          szf[r][c] = __bfloat1622float2(sz[(size_t)(n0 + r) * ng + 8 * c + lane / 4]);
        }
    float acc[R][M];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int i = 0; i < M; ++i) acc[r][i] = 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (c >= nch) break;
      const int k0 = 1024 * c + 32 * lane;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        uint4 xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = *reinterpret_cast<const uint4*>(xs + i * K + k0 + 8 * u);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const __nv_bfloat162 s2 = __float2bfloat162_rn(szf[r][c].x);
          const __nv_bfloat162 z2 = __float2bfloat162_rn(szf[r][c].y - 128.f * szf[r][c].x);
          const uint32_t words[4] = {wv[r][c].x, wv[r][c].y, wv[r][c].z, wv[r][c].w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {  // word u: k0 + 8u .. +8, nibble j = k0 + 8u + j
            const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&xv[u]);
#pragma unroll
            for (int h = 0; h < 4; ++h) {  // nibbles 2h, 2h+1 -> bf16x2 (128 + q)
              const uint32_t nb = ((words[u] >> (8 * h)) & 0xFu) | (((words[u] >> (8 * h + 4)) & 0xFu) << 16);
              uint32_t b2 = nb | 0x43004300u;
              const __nv_bfloat162 wq = __hfma2(*reinterpret_cast<__nv_bfloat162*>(&b2), s2, z2);
              const float2 wf = __bfloat1622float2(wq), xf = __bfloat1622float2(xp[h]);
              acc[r][i] = fmaf(wf.x, xf.x, fmaf(wf.y, xf.y, acc[r][i]));
            }
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int i = 0; i < M; ++i) {
        float v = acc[r][i];
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && n0 + r < N) y[(size_t)i * N + n0 + r] = v;
      }
  }
}

template <int M, bool V2>
static void run(int N, int K, const uint32_t* dq, const __nv_bfloat162* dsz, const __nv_bfloat16* dx, float* dy,
                const std::vector<uint32_t>& hq, const std::vector<__nv_bfloat162>& hsz,
                const std::vector<__nv_bfloat16>& hx, char* flush, size_t flush_bytes) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = (size_t)M * K * 2;
  auto kfn = V2 ? gemv_w4_v2<M> : gemv_w4<M>;
  cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, 256, smem);
  const int grid = nsm * (per_sm > 0 ? per_sm : 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f, sum = 0.f;
  const int reps = 20;
  for (int r = 0; r < reps + 3; ++r) {
    cudaMemsetAsync(flush, r, flush_bytes);  // L2 flush between launches
    cudaEventRecord(a);
    kfn<<<grid, 256, smem>>>(dq, dsz, dx, dy, N, K);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 3) {
      best = fminf(best, ms);
      sum += ms;
    }
  }
  // check 64 rows against a host fp64 reference of the same formula
  std::vector<float> hy((size_t)M * N);
  cudaMemcpy(hy.data(), dy, hy.size() * 4, cudaMemcpyDeviceToHost);
  double maxrel = 0.0;
  for (int t = 0; t < 64; ++t) {
    const int n = (int)((t * 2654435761u) % (unsigned)N);
    for (int i = 0; i < M; ++i) {
      double ref = 0.0, mag = 0.0;
      for (int k = 0; k < K; ++k) {
        const uint32_t word = hq[(size_t)n * (K / 8) + (k / 256) * 32 + (k % 256) / 8];
        const int qv = (word >> (4 * (k % 8))) & 15;
        const float2 s_z = __bfloat1622float2(hsz[(size_t)n * (K / 128) + k / 128]);
        const double w = (double)qv * s_z.x + s_z.y;
        const double xv = (double)__bfloat162float(hx[(size_t)i * K + k]);
        ref += w * xv;
        mag += fabs(w * xv);
      }
      maxrel = fmax(maxrel, fabs(hy[(size_t)i * N + n] - ref) / (mag + 1e-30));
    }
  }
  const double bytes = (double)N * K / 2 + (double)N * (K / 128) * 4 + (double)M * K * 2 + (double)M * N * 4;
  printf("%s m=%d grid=%d: best %.2f us, mean %.2f us, %.2f TB/s (best), max |err|/sum|terms| %.2e\n", V2 ? "v2" : "v1", M, grid,
         best * 1e3, sum / reps * 1e3, bytes / (best * 1e-3) / 1e12, maxrel);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 14336, K = argc > 2 ? atoi(argv[2]) : 4096;
  if (K % 256 || K > 4096) {
    printf("K must be a multiple of 256, <= 4096\n");
    return 1;
  }
  std::vector<uint32_t> hq((size_t)N * (K / 8));
  std::vector<__nv_bfloat162> hsz((size_t)N * (K / 128));
  std::vector<__nv_bfloat16> hx((size_t)8 * K);
  uint64_t st = 12345;
  auto rnd = [&]() {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    return (uint32_t)(st >> 32);
  };
  for (auto& v : hq) v = rnd();
  for (auto& v : hsz)
    v = __floats2bfloat162_rn(0.01f + (rnd() % 1000) * 1e-5f, -0.08f + (rnd() % 1000) * 1e-5f);
  for (auto& v : hx) v = __float2bfloat16(((int)(rnd() % 2001) - 1000) * 1e-3f);
  uint32_t* dq;
  __nv_bfloat162* dsz;
  __nv_bfloat16* dx;
  float* dy;
  char* flush;
  const size_t flush_bytes = (size_t)256 << 20;
  cudaMalloc(&dq, hq.size() * 4);
  cudaMalloc(&dsz, hsz.size() * 4);
  cudaMalloc(&dx, hx.size() * 2);
  cudaMalloc(&dy, (size_t)8 * N * 4);
  cudaMalloc(&flush, flush_bytes);
  cudaMemcpy(dq, hq.data(), hq.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dsz, hsz.data(), hsz.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  printf("w4a16-g128 CUDA-core GEMV, N=%d K=%d, weights %.1f MB, L2 flushed per launch\n", N, K,
         (double)N * K / 2 / 1e6);
  run<1, false>(N, K, dq, dsz, dx, dy, hq, hsz, hx, flush, flush_bytes);
  run<2, false>(N, K, dq, dsz, dx, dy, hq, hsz, hx, flush, flush_bytes);
  run<4, false>(N, K, dq, dsz, dx, dy, hq, hsz, hx, flush, flush_bytes);
  run<8, false>(N, K, dq, dsz, dx, dy, hq, hsz, hx, flush, flush_bytes);
  run<1, true>(N, K, dq, dsz, dx, dy, hq, hsz, hx, flush, flush_bytes);
  run<2, true>(N, K, dq, dsz, dx, dy, hq, hsz, hx, flush, flush_bytes);
  run<4, true>(N, K, dq, dsz, dx, dy, hq, hsz, hx, flush, flush_bytes);
  const cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
