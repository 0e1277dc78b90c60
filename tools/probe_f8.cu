// Developer probe: tcgen05.mma kind::f8f6f4 (e4m3 x e4m3 -> f32) as an exact small-integer GEMM.
// A (TMEM, TS form, or SMEM image, SS form) holds bytes 0..15 = nibble codes u; as e4m3 such a byte is the
// subnormal/first-binade value u * 2^-9 (linear in u). B (SMEM, SW128 K-major) holds sign-magnitude bytes
// (s << 7) | |q|, |q| <= 15, i.e. q * 2^-9. D must equal 2^-18 * sum_k u_k q_k EXACTLY (integer sums < 2^24).
// Also checks the worst-case magnitude (all u = 15, q = +-15) over K = 128 * nst. Not part of the product.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../paper_2505_05799_b200/csrc/sm100.cuh"
using namespace mxm;

__device__ __forceinline__ void tst32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
               "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
               "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
               "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
               "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
__host__ __device__ constexpr uint32_t idesc_f8(uint32_t n) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}
// ts: A from TMEM; else A from smem (canonical SW128 image after the B stages)
__global__ void k(const uint32_t* A, const uint8_t* Aimg, const uint8_t* Bimg, int N, int nst, int ts, uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  int r = threadIdx.x;
  uint8_t* sB = sm;
  uint8_t* sA = sm + nst * N * 128;
  for (int i = threadIdx.x; i < nst * N * 128 / 4; i += 128) ((uint32_t*)sB)[i] = ((const uint32_t*)Bimg)[i];
  if (!ts)
    for (int i = threadIdx.x; i < nst * 16384 / 4; i += 128) ((uint32_t*)sA)[i] = ((const uint32_t*)Aimg)[i];
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = tb;
  const uint32_t lane_base = (uint32_t)((r / 32) * 32) << 16;
  for (int s0 = 0; s0 < nst; s0 += 4) {  // A ring of 4 stages at columns 256..383
    if (ts) {
      for (int s = s0; s < s0 + 4 && s < nst; ++s) {
        uint32_t v[32];
        for (int j = 0; j < 32; ++j) v[j] = A[(s * 128 + r) * 32 + j];
        tst32(tmem + lane_base + 256 + (s - s0) * 32, v);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (threadIdx.x == 0) {
      for (int s = s0; s < s0 + 4 && s < nst; ++s)
        for (int kk = 0; kk < 4; ++kk) {
          uint64_t bd = sw128_kmajor_desc(smem_u32(sB + s * N * 128) + kk * 32);
          uint32_t acc = (s | kk) != 0;
          if (ts) {
            uint32_t at = tmem + 256 + (s - s0) * 32 + kk * 8;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}"
                         ::"r"(tmem), "r"(at), "l"(bd), "r"(idesc_f8(N)), "r"(acc));
          } else {
            uint64_t ad = sw128_kmajor_desc(smem_u32(sA + s * 16384) + kk * 32);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc_f8(N)), "r"(acc));
          }
        }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, (s0 / 4) & 1);
    tc_fence_after();
    __syncthreads();
  }
  for (int c = 0; c < N; c += 16) {
    uint32_t o[16];
    tmem_ld16(tmem + lane_base + c, o);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[r * N + c + j] = o[j];
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

// pattern 0: random u in [0,15], q in [-15,15]; 1: worst case u = 15, q = +15; 2: u = 15, q = -15 / +15 by row
int run(int N, int nst, int ts, int pattern) {
  int K = 128 * nst;
  std::vector<uint8_t> A(128 * K), B(N * K);
  std::vector<int> qa(N * K);
  srand(11 + N + nst + pattern);
  for (size_t i = 0; i < A.size(); ++i) A[i] = pattern ? 15 : (uint8_t)(rand() % 16);
  for (int n = 0; n < N; ++n)
    for (int kk = 0; kk < K; ++kk) {
      int q = pattern == 0 ? rand() % 31 - 15 : (pattern == 1 ? 15 : ((n & 1) ? -15 : 15));
      qa[n * K + kk] = q;
      B[(size_t)n * K + kk] = (uint8_t)((q < 0 ? 0x80 : 0) | (q < 0 ? -q : q));
    }
  std::vector<uint32_t> Aw(nst * 128 * 32);
  for (int s = 0; s < nst; ++s) for (int r = 0; r < 128; ++r) for (int j = 0; j < 32; ++j)
    memcpy(&Aw[(s * 128 + r) * 32 + j], &A[(size_t)r * K + s * 128 + 4 * j], 4);
  std::vector<uint8_t> Aimg(nst * 16384);
  for (int s = 0; s < nst; ++s) for (int r = 0; r < 128; ++r) for (int b = 0; b < 128; ++b)
    Aimg[s * 16384 + r * 128 + (((b >> 4) ^ (r & 7)) << 4) + (b & 15)] = A[(size_t)r * K + s * 128 + b];
  std::vector<uint8_t> Bimg(nst * N * 128);
  for (int s = 0; s < nst; ++s) for (int r = 0; r < N; ++r) for (int b = 0; b < 128; ++b)
    Bimg[s * N * 128 + r * 128 + (((b >> 4) ^ (r & 7)) << 4) + (b & 15)] = B[(size_t)r * K + s * 128 + b];
  uint32_t *dA, *dO; uint8_t *dB, *dAi;
  cudaMalloc(&dA, Aw.size() * 4); cudaMalloc(&dB, Bimg.size()); cudaMalloc(&dAi, Aimg.size()); cudaMalloc(&dO, 128 * N * 4);
  cudaMemcpy(dA, Aw.data(), Aw.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bimg.data(), Bimg.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dAi, Aimg.data(), Aimg.size(), cudaMemcpyHostToDevice);
  int smem = 1024 + nst * N * 128 + (ts ? 0 : nst * 16384);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<1, 128, smem>>>(dA, dAi, dB, N, nst, ts, dO);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<uint32_t> o(128 * N);
  cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  double me = 0;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) {
    long long ref = 0;
    for (int kk = 0; kk < K; ++kk) ref += (long long)A[(size_t)m * K + kk] * qa[n * K + kk];
    float f; memcpy(&f, &o[m * N + n], 4);
    double got = (double)f * 262144.0;
    double err = fabs(got - (double)ref);
    me = err > me ? err : me;
    if (err != 0) ++bad;
  }
  printf("f8 %s N=%d K=%d pattern=%d maxerr=%g bad=%ld %s\n", ts ? "TS" : "SS", N, K, pattern, me, bad, bad ? "FAIL" : "OK");
  cudaFree(dA); cudaFree(dB); cudaFree(dAi); cudaFree(dO);
  return bad != 0;
}
int main() {
  int f = 0;
  f += run(64, 1, 1, 0);
  f += run(64, 1, 0, 0);
  f += run(96, 4, 1, 0);
  f += run(32, 28, 1, 0);
  f += run(16, 28, 1, 1);
  f += run(16, 28, 1, 2);
  f += run(16, 96, 1, 1);
  f += run(128, 2, 0, 0);
  printf(f ? "F8 PROBE FAILED\n" : "F8 PROBE OK\n");
  return f;
}
