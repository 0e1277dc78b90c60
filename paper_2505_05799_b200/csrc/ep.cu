// ep.cu — expert-parallel dispatch / combine index kernels.
//
// Eq. 2 is a sum over experts, so the block shards by experts: rank r owns routed experts
// [r*E/G, (r+1)*E/G). A token is sent once to every destination rank that hosts at least one of its
// routed experts (deduplicated), carrying its k (local expert id | -1, weight) pairs. The NCCL
// all-to-all itself is issued by the host runtime (torch.distributed on ProcessGroupNCCL); these kernels
// build the send buffers and combine the returned partial sums in a fixed (destination-rank) order.
#include <cuda_bf16.h>
#include <cstdint>

#include "actq.cuh"
#include "common.cuh"
#include "kernels.h"

namespace mxm {

// one block per destination rank r: stable positions of the tokens that have an expert on r
__global__ void ep_route_kernel(const int32_t* __restrict__ ids, int64_t T, int k, int E, int G,
                                int32_t* __restrict__ dest_counts, int32_t* __restrict__ pos, int32_t* err) {
  const int r = blockIdx.x;
  const int epr = E / G;
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t base = 0; base < T; base += blockDim.x) {
    const int64_t t = base + threadIdx.x;
    int has = 0;
    if (t < T) {
      for (int j = 0; j < k; ++j) {
        const int e = ids[t * k + j];
        if (e < -1 || e >= E) {
          if (err && r == 0) atomicExch(err, (int32_t)MXM_E_DATA);
          continue;
        }
        if (e >= 0 && e / epr == r) has = 1;
      }
    }
    // block-wide exclusive scan of `has`
    const unsigned m = __ballot_sync(0xffffffffu, has);
    const int in_warp = __popc(m & ((1u << lane) - 1));
    if (lane == 0) wsum[warp] = __popc(m);
    __syncthreads();
    int before = 0;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    int total = 0;
    for (int w = 0; w < nw; ++w) total += wsum[w];
    if (t < T) pos[t * G + r] = has ? carry + before + in_warp : -1;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) dest_counts[r] = carry;
}

// one warp per (token, destination) pair: copy the row and its local (id, weight) metadata
__global__ void ep_pack_kernel(const uint16_t* __restrict__ x, int64_t T, int d, const int32_t* __restrict__ ids,
                               const float* __restrict__ w, int k, int E, int G, const int32_t* __restrict__ pos,
                               const int32_t* __restrict__ dest_off, uint16_t* __restrict__ sx, int32_t* __restrict__ sids,
                               float* __restrict__ sw, int32_t* __restrict__ ssrc) {
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (gw >= T * G) return;
  const int64_t t = gw / G;
  const int r = (int)(gw % G);
  const int p = pos[t * G + r];
  if (p < 0) return;
  const int64_t row = (int64_t)dest_off[r] + p;
  const uint4* src = reinterpret_cast<const uint4*>(x + t * d);
  uint4* dst = reinterpret_cast<uint4*>(sx + row * d);
  for (int i = lane; i < d / 8; i += 32) dst[i] = src[i];
  const int epr = E / G;
  if (lane < k) {
    const int e = ids[t * k + lane];
    const bool mine = e >= 0 && e < E && e / epr == r;
    sids[row * k + lane] = mine ? e - r * epr : -1;
    sw[row * k + lane] = mine ? w[t * k + lane] : 0.f;
  }
  if (lane == 0) ssrc[row] = (int32_t)t;
}

// y[t] = bf16( sum_r back[dest_off[r] + pos[t, r]] (r ascending) + ysh[t] )
__global__ void ep_combine_kernel(const uint16_t* __restrict__ back, const int32_t* __restrict__ pos,
                                  const int32_t* __restrict__ dest_off, int G, int64_t T, int d,
                                  const uint16_t* __restrict__ ysh, uint16_t* __restrict__ y) {
  const int64_t t = blockIdx.x;
  for (int c = threadIdx.x; c < d / 8; c += blockDim.x) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int r = 0; r < G; ++r) {
      const int p = pos[t * G + r];
      if (p < 0) continue;
      const uint4 v = reinterpret_cast<const uint4*>(back + ((int64_t)dest_off[r] + p) * d)[c];
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[2 * i] += bf16_bits_to_float(wv[i] & 0xFFFFu);
        acc[2 * i + 1] += bf16_bits_to_float(wv[i] >> 16);
      }
    }
    if (ysh) {
      const uint4 v = reinterpret_cast<const uint4*>(ysh + t * d)[c];
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[2 * i] += bf16_bits_to_float(wv[i] & 0xFFFFu);
        acc[2 * i + 1] += bf16_bits_to_float(wv[i] >> 16);
      }
    }
    uint32_t out[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
      out[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    reinterpret_cast<uint4*>(y + t * d)[c] = make_uint4(out[0], out[1], out[2], out[3]);
  }
}

cudaError_t launch_ep_route(const int32_t* ids, int64_t T, int k, int E, int G, int32_t* dest_counts, int32_t* pos,
                            int32_t* err, cudaStream_t st) {
  ep_route_kernel<<<G, 1024, 0, st>>>(ids, T, k, E, G, dest_counts, pos, err);
  return cudaGetLastError();
}
cudaError_t launch_ep_pack(const void* x, int64_t T, int d, const int32_t* ids, const float* w, int k, int E, int G,
                           const int32_t* pos, const int32_t* dest_off, void* sx, int32_t* sids, float* sw,
                           int32_t* ssrc, cudaStream_t st) {
  if (T == 0) return cudaSuccess;
  const int64_t warps = T * G;
  ep_pack_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>((const uint16_t*)x, T, d, ids, w, k, E, G, pos,
                                                                        dest_off, (uint16_t*)sx, sids, sw, ssrc);
  return cudaGetLastError();
}
// sync-free EP constants on the device (no host staging): dest_off[r] = r * C, the shared experts' ids
// sid[t, s] = s and unit weights
__global__ void ep_fill_kernel(int32_t* __restrict__ dest_off, int G, int64_t C, int32_t* __restrict__ sid,
                               float* __restrict__ ones, int64_t T, int S) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= G) dest_off[i] = (int32_t)(i * C);
  if (i < T * S) {
    sid[i] = (int32_t)(i % S);
    ones[i] = 1.0f;
  }
}
cudaError_t launch_ep_fill(int32_t* dest_off, int G, int64_t C, int32_t* sid, float* ones, int64_t T, int S,
                           cudaStream_t st) {
  const int64_t n = (T * S > G + 1) ? T * S : G + 1;
  ep_fill_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(dest_off, G, C, sid, ones, T, S);
  return cudaGetLastError();
}
cudaError_t launch_ep_combine(const void* back, const int32_t* pos, const int32_t* dest_off, int G, int64_t T, int d,
                              const void* ysh, void* y, cudaStream_t st) {
  if (T == 0) return cudaSuccess;
  ep_combine_kernel<<<(unsigned)T, 128, 0, st>>>((const uint16_t*)back, pos, dest_off, G, T, d, (const uint16_t*)ysh,
                                                 (uint16_t*)y);
  return cudaGetLastError();
}

}  // namespace mxm
