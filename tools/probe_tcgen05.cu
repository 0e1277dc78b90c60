// Developer probe: validates the sm100.cuh descriptor / TMA / TMEM encodings on one tile.
//   D[128 x N] = A[128 x K] * B[N x K]^T   for kind::f16 (bf16) and kind::i8 (s8, u8 x s8)
// A is bulk-copied from a host-built canonical SW128 K-major image; B arrives by TMA
// (SWIZZLE_128B). Prints max error vs a CPU reference. Not part of the product.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../paper_2505_05799_b200/csrc/sm100.cuh"

using namespace mxm;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

// kind: 0 bf16, 1 s8xs8, 2 u8xs8
__global__ void probe_kernel(const uint8_t* a_img, int a_stage_bytes, const __grid_constant__ CUtensorMap bmap,
                             int N, int nstages, int kind, uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                       // nstages * 16 KB
  uint8_t* sB = smem + nstages * 16384;     // nstages * N*128
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  if (threadIdx.x == 32) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    uint32_t bytes = nstages * (16384 + N * 128);
    mbar_arrive_expect_tx(&bar_load, bytes);
    for (int s = 0; s < nstages; ++s) {
      bulk_load(sA + s * 16384, a_img + s * a_stage_bytes, 16384, &bar_load);
      tma_load_2d(sB + s * N * 128, &bmap, &bar_load, s * (kind == 0 ? 64 : 128), 0);
    }
    mbar_wait(&bar_load, 0);
    tc_fence_after();
    uint32_t idesc = kind == 0 ? idesc_bf16(N) : idesc_s8(N, kind == 1, true);
    for (int s = 0; s < nstages; ++s) {
      for (int k = 0; k < 4; ++k) {
        uint64_t ad = sw128_kmajor_desc(smem_u32(sA + s * 16384) + k * 32);
        uint64_t bd = sw128_kmajor_desc(smem_u32(sB + s * N * 128) + k * 32);
        if (kind == 0)
          mma_bf16(tmem, ad, bd, idesc, (s | k) != 0);
        else
          mma_i8(tmem, ad, bd, idesc, (s | k) != 0);
      }
    }
    mma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  int lane_base = (warp % 4) * 32;
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + (uint32_t(lane_base) << 16) + c, r);
    tmem_ld_wait();
    int row = lane_base + threadIdx.x % 32;
    for (int j = 0; j < 16; ++j) out[row * N + c + j] = r[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static float bf2f(uint16_t b) {
  uint32_t u = uint32_t(b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return uint16_t(u >> 16);
}

int run(int kind, int N, int nstages) {
  int esz = kind == 0 ? 2 : 1;
  int KS = 128 / esz;  // elements per stage
  int K = KS * nstages;
  std::vector<uint8_t> A(128 * K * esz), B(N * K * esz);
  srand(1234 + kind * 10 + N);
  for (size_t i = 0; i < A.size() / esz; ++i) {
    if (kind == 0) {
      uint16_t v = f2bf((rand() % 2001 - 1000) / 1000.0f);
      memcpy(&A[i * 2], &v, 2);
    } else if (kind == 1) {
      A[i] = uint8_t(int8_t(rand() % 255 - 127));
    } else {
      A[i] = uint8_t(rand() % 256);
    }
  }
  for (size_t i = 0; i < B.size() / esz; ++i) {
    if (kind == 0) {
      uint16_t v = f2bf((rand() % 2001 - 1000) / 1000.0f);
      memcpy(&B[i * 2], &v, 2);
    } else {
      B[i] = uint8_t(int8_t(rand() % 255 - 127));
    }
  }
  // canonical SW128 K-major image of A, per stage
  std::vector<uint8_t> img(nstages * 16384);
  for (int s = 0; s < nstages; ++s)
    for (int r = 0; r < 128; ++r)
      for (int b = 0; b < 128; ++b) {
        int c = b / 16, w = b % 16;
        int dst = s * 16384 + r * 128 + ((c ^ (r % 8)) * 16) + w;
        img[dst] = A[(size_t)r * K * esz + s * 128 + b];
      }
  uint8_t *dimg, *dB;
  uint32_t* dout;
  CK(cudaMalloc(&dimg, img.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dout, 128 * N * 4));
  CK(cudaMemcpy(dimg, img.data(), img.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
  cuuint64_t strides[1] = {(cuuint64_t)K * esz};
  cuuint32_t box[2] = {(cuuint32_t)KS, (cuuint32_t)N};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = get_encode()(&map, kind == 0 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
                             dB, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    printf("encode failed %d\n", cr);
    return 1;
  }
  int smem = 1024 + nstages * (16384 + N * 128);
  CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe_kernel<<<1, 128, smem>>>(dimg, 16384, map, N, nstages, kind, dout);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<uint32_t> out(128 * N);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0;
  long bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) {
        if (kind == 0) {
          uint16_t a, b;
          memcpy(&a, &A[((size_t)m * K + k) * 2], 2);
          memcpy(&b, &B[((size_t)n * K + k) * 2], 2);
          ref += (double)bf2f(a) * bf2f(b);
        } else {
          int av = kind == 1 ? int(int8_t(A[(size_t)m * K + k])) : int(A[(size_t)m * K + k]);
          ref += double(av) * int(int8_t(B[(size_t)n * K + k]));
        }
      }
      double got;
      if (kind == 0) {
        float f;
        memcpy(&f, &out[m * N + n], 4);
        got = f;
      } else {
        got = double(int32_t(out[m * N + n]));
      }
      double e = fabs(got - ref);
      if (e > maxerr) maxerr = e;
      if (kind != 0 && e != 0) ++bad;
      if (kind == 0 && e > 1e-2 * (1 + fabs(ref))) ++bad;
    }
  printf("probe kind=%d N=%d K=%d : maxerr=%g bad=%ld %s\n", kind, N, K, maxerr, bad, bad ? "FAIL" : "OK");
  cudaFree(dimg);
  cudaFree(dB);
  cudaFree(dout);
  return bad ? 1 : 0;
}

int main() {
  int fails = 0;
  fails += run(0, 64, 2);
  fails += run(0, 16, 1);
  fails += run(0, 128, 3);
  fails += run(1, 64, 2);
  fails += run(1, 32, 1);
  fails += run(2, 128, 2);
  printf(fails ? "PROBE FAILED\n" : "PROBE OK\n");
  return fails;
}
