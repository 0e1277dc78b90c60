// Developer probe: tcgen05.mma with A from TMEM (TS form). A row r = TMEM lane r; for one K-stage of 128 bytes
// per row, 32 consecutive 32-bit columns hold the row's bytes in order (bf16: element k in column k/2, low half
// = even k). Checks D = A * B^T against a CPU reference for kind::f16 and kind::i8.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../paper_2505_05799_b200/csrc/sm100.cuh"
using namespace mxm;
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
               "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
               "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
               "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
               "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
__device__ __forceinline__ void mma_ts(int kind, uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  if (kind == 0)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                 ::"r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
                 ::"r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}
__global__ void k(const uint32_t* A /*[128][32] words per stage*/, const void* dummy,
                  const uint8_t* Bimg /*N x 128B swizzled*/, int N, int nst, int kind, uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  int r = threadIdx.x;  // lane / row
  for (int i = threadIdx.x; i < nst * N * 128 / 4; i += 128) ((uint32_t*)sm)[i] = ((const uint32_t*)Bimg)[i];
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = tb;
  const uint32_t lane_base = (uint32_t)((r / 32) * 32) << 16;
  for (int s = 0; s < nst; ++s) {
    uint32_t v[32];
    for (int j = 0; j < 32; ++j) v[j] = A[(s * 128 + r) * 32 + j];
    tmem_st32(tmem + lane_base + 256 + s * 32, v);  // A stages at columns 256.. (accumulator at 0)
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) {
    uint32_t idesc = kind == 0 ? idesc_bf16(N) : idesc_s8(N);
    for (int s = 0; s < nst; ++s)
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t bd = sw128_kmajor_desc(smem_u32(sm + s * N * 128) + kk * 32);
        mma_ts(kind, tmem, tmem + 256 + s * 32 + kk * 8, bd, idesc, (s | kk) != 0);
      }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t o[16];
    tmem_ld16(tmem + lane_base + c, o);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[r * N + c + j] = o[j];
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}
static float bf(uint16_t b) { uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f; }
static uint16_t tobf(float f) { uint32_t u; memcpy(&u, &f, 4); u += 0x7FFF + ((u >> 16) & 1); return u >> 16; }
int run(int kind, int N, int nst) {
  int esz = kind == 0 ? 2 : 1, KS = 128 / esz, K = KS * nst;
  std::vector<uint8_t> A(128 * K * esz), B(N * K * esz);
  srand(7 + kind + N);
  for (size_t i = 0; i < A.size() / esz; ++i) { if (kind == 0) { uint16_t v = tobf((rand() % 2001 - 1000) / 500.f); memcpy(&A[2 * i], &v, 2); } else A[i] = (uint8_t)(rand() % 255 - 127); }
  for (size_t i = 0; i < B.size() / esz; ++i) { if (kind == 0) { uint16_t v = tobf((rand() % 2001 - 1000) / 500.f); memcpy(&B[2 * i], &v, 2); } else B[i] = (uint8_t)(rand() % 255 - 127); }
  // A words: stage s, row r, word j = bytes [s*128 + 4j, +4) of row r
  std::vector<uint32_t> Aw(nst * 128 * 32);
  for (int s = 0; s < nst; ++s) for (int r = 0; r < 128; ++r) for (int j = 0; j < 32; ++j) memcpy(&Aw[(s * 128 + r) * 32 + j], &A[(size_t)r * K * esz + s * 128 + 4 * j], 4);
  std::vector<uint8_t> Bimg(nst * N * 128);
  for (int s = 0; s < nst; ++s) for (int r = 0; r < N; ++r) for (int b = 0; b < 128; ++b) Bimg[s * N * 128 + r * 128 + (((b >> 4) ^ (r & 7)) << 4) + (b & 15)] = B[(size_t)r * K * esz + s * 128 + b];
  uint32_t *dA, *dO; uint8_t* dB;
  cudaMalloc(&dA, Aw.size() * 4); cudaMalloc(&dB, Bimg.size()); cudaMalloc(&dO, 128 * N * 4);
  cudaMemcpy(dA, Aw.data(), Aw.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dB, Bimg.data(), Bimg.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<1, 128, 100 * 1024>>>(dA, nullptr, dB, N, nst, kind, dO);
  cudaError_t e = cudaDeviceSynchronize(); if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<uint32_t> o(128 * N); cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
  long bad = 0; double me = 0;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) {
    double ref = 0;
    for (int kk = 0; kk < K; ++kk) {
      if (kind == 0) { uint16_t a, b; memcpy(&a, &A[((size_t)m * K + kk) * 2], 2); memcpy(&b, &B[((size_t)n * K + kk) * 2], 2); ref += (double)bf(a) * bf(b); }
      else ref += (double)(int8_t)A[(size_t)m * K + kk] * (int8_t)B[(size_t)n * K + kk];
    }
    double got; if (kind == 0) { float f; memcpy(&f, &o[m * N + n], 4); got = f; } else got = (int32_t)o[m * N + n];
    double err = fabs(got - ref); me = err > me ? err : me;
    if (kind ? err != 0 : err > 1e-2 * (1 + fabs(ref))) ++bad;
  }
  printf("TS kind=%d N=%d K=%d maxerr=%g bad=%ld %s\n", kind, N, K, me, bad, bad ? "FAIL" : "OK");
  return bad != 0;
}
int main() { int f = 0; f += run(0, 128, 2); f += run(0, 64, 1); f += run(1, 128, 2); f += run(1, 32, 1); printf(f ? "TS PROBE FAILED\n" : "TS PROBE OK\n"); return f; }
