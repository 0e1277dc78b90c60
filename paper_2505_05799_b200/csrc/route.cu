// route.cu — step S1 (route preparation) and S2 (activation quantize + gather) and S8 (combine).
//
// S1: histogram of the T*k expert ids, exclusive scan, stable (t, j)-ordered placement
//     (the GPU form of "each expert is processed individually": rows of one expert are
//     contiguous). Shared experts (always active) occupy rows [s*T, (s+1)*T) first; routed rows
//     follow at S*T + offsets[e].
// S2: per route row, the block inputs of its expert's gate/up: a bf16 copy (weight-only schemes)
//     and/or int8 codes + fp32 scales of the dynamic activation quantizer.
// S8: y[t] = sum_j O[row(t, j)] + sum_s O[s*T + t]  (Eq. 2; w_e already applied), fixed order.
#include <cuda_bf16.h>
#include <cstdint>

#include "actq.cuh"
#include "common.cuh"
#include "kernels.h"

namespace mxm {

constexpr int kRouteChunk = 256;  // one placement round per block: 96 blocks at T*k = 24576
constexpr int kMaxExperts = 1024;

// ---- S1a: per-chunk histograms; invalid ids -> error word
__global__ void route_count_kernel(const int32_t* __restrict__ ids, int64_t n, int E, int32_t* __restrict__ chunk_hist,
                                   int32_t* err) {
  __shared__ int32_t hist[kMaxExperts];
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRouteChunk;
  for (int i = threadIdx.x; i < kRouteChunk; i += blockDim.x) {
    const int64_t r = base + i;
    if (r >= n) break;
    const int e = ids[r];
    if (e >= 0 && e < E)
      atomicAdd(&hist[e], 1);
    else if (e != -1 && err)
      atomicExch(err, (int32_t)MXM_E_DATA);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) chunk_hist[(int64_t)blockIdx.x * E + e] = hist[e];
}

// ---- S1b: one warp per expert: exclusive scan of its per-chunk counts (lane = contiguous chunk range)
__global__ void route_scan_kernel(int32_t* __restrict__ chunk_hist, int nchunks, int E, int32_t* __restrict__ counts) {
  const int e = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (e >= E) return;
  const int per = (nchunks + 31) / 32;
  const int c0 = min(nchunks, lane * per), c1 = min(nchunks, c0 + per);
  int32_t sum = 0;
  for (int c = c0; c < c1; ++c) sum += chunk_hist[(int64_t)c * E + e];
  int32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int32_t run = incl - sum;
  for (int c = c0; c < c1; ++c) {
    const int32_t h = chunk_hist[(int64_t)c * E + e];
    chunk_hist[(int64_t)c * E + e] = run;  // becomes the chunk's base within expert e
    run += h;
  }
  if (lane == 31 && counts) counts[e] = incl;
}

// exclusive scan of counts[0..E) (E <= 256) into smem `off` by a 256-thread block; returns the total
__device__ int32_t block_scan_counts(const int32_t* __restrict__ counts, int E, int32_t* off, int32_t* wtot) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int32_t v = t < E ? counts[t] : 0;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wtot[w] = x;
  __syncthreads();
  int32_t before = 0, total = 0;
  for (int i = 0; i < 8; ++i) {
    if (i < w) before += wtot[i];
    total += wtot[i];
  }
  if (t < E) off[t] = before + x - v;
  __syncthreads();
  return total;
}

// ---- S1c: stable placement within chunk (warp match + per-warp counts)
__global__ void route_place_kernel(const int32_t* __restrict__ ids, const float* __restrict__ topk_w, int64_t n, int k,
                                   int E, int S, int64_t T, const int32_t* __restrict__ chunk_base,
                                   const int32_t* __restrict__ counts, int32_t* __restrict__ offsets,
                                   int32_t* __restrict__ v_off, int32_t* __restrict__ perm,
                                   int32_t* __restrict__ row_src, float* __restrict__ row_w,
                                   int32_t* __restrict__ row_exp, int32_t* __restrict__ inv) {
  __shared__ int32_t base[kMaxExperts];
  __shared__ int32_t wcnt[8][kMaxExperts / 4];  // 8 warps; E <= 256 in this path
  __shared__ int32_t wtot[8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  // expert offsets (every block recomputes the E-scan; block 0 publishes offsets / v_off)
  const int32_t total = block_scan_counts(counts, E, base, wtot);
  const int64_t row_base = row_src ? (int64_t)S * T : 0;  // routed rows follow the S*T shared-expert rows
  if (blockIdx.x == 0) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      if (offsets) offsets[e] = base[e];
      if (v_off) v_off[e] = (int32_t)row_base + base[e];
    }
    if (threadIdx.x == 0) {
      if (offsets) offsets[E] = total;
      if (v_off) {
        v_off[E + S] = (int32_t)row_base + total;  // end of routed rows
        for (int s = 0; s < S; ++s) v_off[E + s] = (int32_t)(s * T);
      }
    }
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) base[e] += chunk_base[(int64_t)blockIdx.x * E + e];
  const int64_t c0 = (int64_t)blockIdx.x * kRouteChunk;
  for (int sub = 0; sub < kRouteChunk; sub += 256) {
    for (int i = threadIdx.x; i < 8 * E; i += blockDim.x) wcnt[i / E][i % E] = 0;
    __syncthreads();
    const int64_t r = c0 + sub + threadIdx.x;
    int e = -1;
    if (r < n) e = ids[r];
    if (e >= E || e < 0) e = -1;
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(peers & ((1u << lane) - 1));
    if (e >= 0 && rank == 0) wcnt[warp][e] = __popc(peers);
    __syncthreads();
    if (e >= 0) {
      int pos = base[e] + rank;
      for (int w = 0; w < warp; ++w) pos += wcnt[w][e];
      if (perm) perm[pos] = (int32_t)r;
      const int64_t row = row_base + pos;
      if (row_src) {
        row_src[row] = (int32_t)(r / k);
        row_w[row] = topk_w[r];
        row_exp[row] = e;
        inv[r] = (int32_t)row;
      }
    } else if (r < n && inv) {
      inv[r] = -1;
    }
    __syncthreads();
    for (int ee = threadIdx.x; ee < E; ee += blockDim.x) {
      int s = 0;
      for (int w = 0; w < 8; ++w) s += wcnt[w][ee];
      base[ee] += s;
    }
    __syncthreads();
  }
}

// ---- shared-expert rows
__global__ void route_shared_kernel(int64_t T, int E, int S, const float* __restrict__ shared_w,
                                    int32_t* __restrict__ row_src, float* __restrict__ row_w, int32_t* __restrict__ row_exp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T * S) return;
  const int64_t s = i / T, t = i % T;
  row_src[i] = (int32_t)t;
  row_w[i] = shared_w ? shared_w[t * S + s] : 1.0f;
  row_exp[i] = E + (int32_t)s;
}

// ---- S2: one warp per route row: gather / quantize the gate/up inputs of the row's expert
// QUANT: the layer has weight-activation input slots (the row-in-registers quantizer needs ~124 registers;
// an all-weight-only layer launches the copy-only instantiation at full occupancy)
template <bool QUANT>
__global__ void gather_quant_kernel(const uint16_t* __restrict__ x, int d, const int32_t* __restrict__ row_src,
                                    const int32_t* __restrict__ row_exp, const int32_t* __restrict__ v_off, int V,
                                    const ExpertDesc* __restrict__ ex,
                                    int64_t R, uint16_t* __restrict__ Xb, int8_t* __restrict__ XqA, float* __restrict__ XsA,
                                    int8_t* __restrict__ XqB, float* __restrict__ XsB, int32_t* __restrict__ XcA,
                                    int32_t* __restrict__ XcB, uint32_t* __restrict__ hmax) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (row >= R) return;
  if (row >= v_off[V]) return;  // rows past the last valid route are unused
  const int v = row_exp[row];
  if (lane == 0 && hmax) hmax[row] = 0u;
  const ExpertDesc& E = ex[v];
  const uint16_t* src = x + (int64_t)row_src[row] * d;
  for (int b = 0; b < 2; ++b) {
    const LinDesc& L = E.blk[b];
    if (b == 1 && E.blk[1].in_slot == E.blk[0].in_slot) break;
    if (L.in_slot == 0) {
      const uint4* __restrict__ s4 = reinterpret_cast<const uint4*>(src);
      uint4* __restrict__ d4 = reinterpret_cast<uint4*>(Xb + row * d);
#pragma unroll 4
      for (int i = lane; i < d / 8; i += 32) d4[i] = s4[i];
    } else if constexpr (QUANT) {
      int8_t* q = (L.in_slot == 1 ? XqA : XqB) + row * d;
      float* sc = (L.in_slot == 1 ? XsA : XsB) + row;  // group-major [g][R]
      int32_t* qs = (L.in_slot == 1 ? XcA : XcB) + row;
      const int g = L.a_group == -1 ? d : L.a_group;
      const int qmax = (1 << (L.a_bits - 1)) - 1;
      const bool e4 = kind_is_w4a4(L.geo.kind);  // w4a4: e4m3 small-integer codes for kind::f8f6f4 (common.cuh)
      if (d <= 128 * 32 && (g == 128 || g == d)) {  // whole row in registers, all loads in flight
        if (kind_is_fp8(L.geo.kind))
          quant_row_warp<32, false, true>(src, q, d, g, qmax, sc, qs, R);
        else if (e4)
          quant_row_warp<32, true>(src, q, d, g, qmax, sc, qs, R);
        else
          quant_row_warp<32, false>(src, q, d, g, qmax, sc, qs, R);
      } else {
        for (int gi = 0; gi < d / g; ++gi) {
          int qsum = 0;
          const float s = e4 ? quant_group_warp<false, true>(src + gi * g, q + gi * g, g, qmax, &qsum)
                             : quant_group_warp<false, false>(src + gi * g, q + gi * g, g, qmax, &qsum);
          if (lane == 0) {
            sc[gi * R] = s;
            qs[gi * R] = qsum;
          }
        }
      }
    }
  }
}

// ---- S2, token-major: one warp per (token, input format). The dynamic quantizer's result depends only on the
// token's row and the format (a_bits, group, code encoding), not on the expert, so each token is quantized once
// per format in use ("dynamically quantized at runtime according to the corresponding allocated scheme")
// and the codes / scales / code sums are stored to every route row of the token whose gate or up block reads
// that format (k routed rows via inv[], S shared rows s*T + t). Same arithmetic as quant_row_warp (DESIGN R9):
// every stored row is bit-identical to the row-major kernel's. Format a_bits 16 = the bf16 row copy (Xb).
template <int MAXG>
#ifndef MXM_GATHER_MINB
#define MXM_GATHER_MINB 4  // resident 256-thread blocks per SM the register budget is sized for
#endif
#ifndef MXM_GATHER_PASS
#define MXM_GATHER_PASS 8  // 128-element chunks per register pass (8, 16 measured: profiles/r02/ab_experiments.txt ab18)
#endif
__global__ void __launch_bounds__(256, MXM_GATHER_MINB) gather_tok_kernel(
    const uint16_t* __restrict__ x, int d, int64_t T, int k, int S, int E, const int32_t* __restrict__ inv,
    const int32_t* __restrict__ row_exp, const ExpertDesc* __restrict__ ex, ActFormats fm, int64_t R,
    uint16_t* __restrict__ Xb, int8_t* __restrict__ XqA, float* __restrict__ XsA, int8_t* __restrict__ XqB,
    float* __restrict__ XsB, int32_t* __restrict__ XcA, int32_t* __restrict__ XcB, uint32_t* __restrict__ hmax) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (w >= T * fm.n) return;
  const int64_t t = w / fm.n;
  const int f = (int)(w % fm.n);
  const int fb = fm.a_bits[f], fg = fm.a_group[f];
  const int fe = fm.e4[f];  // code encoding: 0 two's complement, 1 w4a4 e4m3 small integers, 2 FP8 e4m3 (R26)
  // lane j < k + S resolves route j of the token: its row and the slots (1 / 2) of gate / up that read format f
  int64_t row = -1;
  int sl0 = -1, sl1 = -1;  // slot written for the gate / up input (-1: another format)
  if (lane < k + S) {
    row = lane < k ? (int64_t)inv[t * k + lane] : (int64_t)(lane - k) * T + t;
    if (row >= 0) {
      const int v = lane < k ? row_exp[row] : E + (lane - k);
      const LinDesc& L0 = ex[v].blk[0];
      const LinDesc& L1 = ex[v].blk[1];
      auto match = [&](const LinDesc& L) {
        if (L.in_slot == 0) return fb == 16;
        return fb == L.a_bits && fg == L.a_group && fe == (kind_is_fp8(L.geo.kind) ? 2 : (kind_is_w4a4(L.geo.kind) ? 1 : 0));
      };
      if (match(L0)) sl0 = L0.in_slot;
      if (L1.in_slot != L0.in_slot && match(L1)) sl1 = L1.in_slot;
    }
  }
  const unsigned todo = __ballot_sync(0xffffffffu, sl0 >= 0 || sl1 >= 0);
  if (todo == 0) return;
  const int nch = d / 128;
  const uint16_t* src = x + t * d;
  // the row in passes of kPass 128-element chunks: the register tile (3 x kPass words) fits 64 registers, so 4
  // blocks stay resident per SM instead of 2 -- the kernel is latency-bound (ncu: 25 % occupancy, issue 28 %)
  constexpr int kPass = MAXG < MXM_GATHER_PASS ? MAXG : MXM_GATHER_PASS;
  auto load_chunk = [&](int i) { return *reinterpret_cast<const uint2*>(src + 128 * i + 4 * lane); };
  if (fb == 16) {  // bf16 copy into every weight-only / 16-bit route row of the token
    for (int c0 = 0; c0 < nch; c0 += kPass) {
      uint2 v[kPass];
#pragma unroll
      for (int i = 0; i < kPass; ++i)
        if (c0 + i < nch) v[i] = load_chunk(c0 + i);
      for (unsigned m = todo; m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        const int64_t r = __shfl_sync(0xffffffffu, row, j);
        uint16_t* dst = Xb + r * d;
#pragma unroll
        for (int i = 0; i < kPass; ++i)
          if (c0 + i < nch) *reinterpret_cast<uint2*>(dst + 128 * (c0 + i) + 4 * lane) = v[i];
      }
    }
    for (unsigned m = todo; m; m &= m - 1) {
      const int j = __ffs(m) - 1;
      const int64_t r = __shfl_sync(0xffffffffu, row, j);
      const int g0 = __shfl_sync(0xffffffffu, sl0, j);
      if (lane == 0 && g0 >= 0 && hmax) hmax[r] = 0u;
    }
    return;
  }
  const float fq = fe == 2 ? 448.f : (float)((1 << (fb - 1)) - 1);
  auto absmax4 = [](uint2 a) {
    return fmaxf(fmaxf(fabsf(bf16_bits_to_float(a.x & 0xFFFFu)), fabsf(bf16_bits_to_float(a.x >> 16))),
                 fmaxf(fabsf(bf16_bits_to_float(a.y & 0xFFFFu)), fabsf(bf16_bits_to_float(a.y >> 16))));
  };
  auto quant4 = [&](uint2 a, float r, int& qsum) {
    const float fv[4] = {bf16_bits_to_float(a.x & 0xFFFFu), bf16_bits_to_float(a.x >> 16),
                         bf16_bits_to_float(a.y & 0xFFFFu), bf16_bits_to_float(a.y >> 16)};
    uint32_t packed = 0;
    if (fe == 2) {
#pragma unroll
      for (int j = 0; j < 4; ++j) packed |= fp8_act_code(fv[j], r) << (8 * j);
      return packed;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float q = rintf(__fmul_rn(fv[j], r));
      q = fminf(fmaxf(q, -fq), fq);
      qsum += (int)q;
      packed |= (fe ? code_byte<true>((int)q) : code_byte<false>((int)q)) << (8 * j);
    }
    return packed;
  };
  float my_s = 1.f;  // g128: lane i holds group i's scale and code sum; per token: the row's
  int my_qs = 0;
  // per token: the row maximum first (a load-only pass; the quantizing pass re-reads the row from L1)
  float r_row = 0.f;
  int qsum_row = 0;
  if (fg != 128) {
    float amax = 0.f;
    for (int i = 0; i < nch; ++i) amax = fmaxf(amax, absmax4(load_chunk(i)));
    amax = warp_max(amax);
    if (amax > 0.f) {
      r_row = __fdiv_rn(fq, amax);
      my_s = __fdiv_rn(amax, fq);
    }
  }
  for (int c0 = 0; c0 < nch; c0 += kPass) {
    uint2 v[kPass];
#pragma unroll
    for (int i = 0; i < kPass; ++i)
      if (c0 + i < nch) v[i] = load_chunk(c0 + i);
    uint32_t code[kPass];
    if (fg == 128) {
      // the pass's group maxima (independent reductions), then lane c divides for group c only (two IEEE
      // divisions per lane instead of a dependent chain of 2 per group), r broadcast per group
      float my_amax = 0.f;
#pragma unroll
      for (int i = 0; i < kPass; ++i) {
        if (c0 + i < nch) {
          const float amax = warp_max(absmax4(v[i]));
          if (lane == c0 + i) my_amax = amax;
        }
      }
      float r_l = 0.f;
      if (my_amax > 0.f) {
        r_l = __fdiv_rn(fq, my_amax);
        my_s = __fdiv_rn(my_amax, fq);
      }
#pragma unroll
      for (int i = 0; i < kPass; ++i) {
        if (c0 + i < nch) {
          const float r = __shfl_sync(0xffffffffu, r_l, c0 + i);
          int qsum = 0;
          code[i] = quant4(v[i], r, qsum);
          qsum = warp_sum(qsum);
          if (lane == c0 + i) my_qs = qsum;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < kPass; ++i)
        if (c0 + i < nch) code[i] = quant4(v[i], r_row, qsum_row);
    }
    for (unsigned m = todo; m; m &= m - 1) {
      const int j = __ffs(m) - 1;
      const int64_t r = __shfl_sync(0xffffffffu, row, j);
      const int g0 = __shfl_sync(0xffffffffu, sl0, j), g1 = __shfl_sync(0xffffffffu, sl1, j);
      for (int b = 0; b < 2; ++b) {
        const int slot = b == 0 ? g0 : g1;
        if (slot < 1) continue;
        int8_t* q = (slot == 1 ? XqA : XqB) + r * d;
#pragma unroll
        for (int i = 0; i < kPass; ++i)
          if (c0 + i < nch) *reinterpret_cast<uint32_t*>(q + 128 * (c0 + i) + 4 * lane) = code[i];
      }
    }
  }
  if (fg != 128) my_qs = warp_sum(qsum_row);
  const int ng = fg == 128 ? nch : 1;
  for (unsigned m = todo; m; m &= m - 1) {
    const int j = __ffs(m) - 1;
    const int64_t r = __shfl_sync(0xffffffffu, row, j);
    const int g0 = __shfl_sync(0xffffffffu, sl0, j), g1 = __shfl_sync(0xffffffffu, sl1, j);
    for (int b = 0; b < 2; ++b) {
      const int slot = b == 0 ? g0 : g1;
      if (slot < 1) continue;
      float* sc = (slot == 1 ? XsA : XsB) + r;  // group-major [g][R]
      int32_t* qs = (slot == 1 ? XcA : XcB) + r;
      if (lane < ng) {
        sc[(int64_t)lane * R] = my_s;
        qs[(int64_t)lane * R] = my_qs;
      }
    }
    if (lane == 0 && g0 >= 0 && hmax) hmax[r] = 0u;
  }
}

// ---- S8: combine, one block per token; all k + S source rows are resolved first so their loads overlap
__global__ void combine_kernel(const uint16_t* __restrict__ O, int d, int64_t T, int k, int S,
                               const int32_t* __restrict__ inv, uint16_t* __restrict__ y) {
  const int64_t t = blockIdx.x;
  __shared__ int32_t rows[64];
  if (threadIdx.x < k + S) {
    const int j = threadIdx.x;
    rows[j] = j < k ? inv[t * k + j] : (int32_t)((j - k) * T + t);  // routed rows, then shared rows
  }
  __syncthreads();
  const int n = k + S;
  auto add = [](float (&acc)[8], uint4 u) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[2 * i] += bf16_bits_to_float(w[i] & 0xFFFFu);
      acc[2 * i + 1] += bf16_bits_to_float(w[i] >> 16);
    }
  };
  for (int c = threadIdx.x; c < d / 8; c += blockDim.x) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    constexpr int kBatch = 8;  // loads in flight per thread before the (fixed-order) sum
    for (int j0 = 0; j0 < n; j0 += kBatch) {
      uint4 v[kBatch];
#pragma unroll
      for (int j = 0; j < kBatch; ++j) {
        v[j] = make_uint4(0, 0, 0, 0);
        if (j0 + j < n && rows[j0 + j] >= 0)
          v[j] = __ldcs(reinterpret_cast<const uint4*>(O + (int64_t)rows[j0 + j] * d) + c);
      }
#pragma unroll
      for (int j = 0; j < kBatch; ++j)
        if (j0 + j < n && rows[j0 + j] >= 0) add(acc, v[j]);
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

// ---------------------------------------------------------------- host launchers
int64_t route_scratch_bytes(int64_t n_routes, int E) {
  const int64_t nch = (n_routes + kRouteChunk - 1) / kRouteChunk;
  return ((nch * E * 4) + 255) / 256 * 256;
}

cudaError_t launch_route_prep(const int32_t* ids, const float* topk_w, int64_t T, int k, int E, int S,
                              const float* shared_w, int32_t* counts, int32_t* offsets, int32_t* v_off, int32_t* perm,
                              int32_t* row_src, float* row_w, int32_t* row_exp, int32_t* inv, int32_t* err,
                              void* scratch, cudaStream_t st) {
  if (E > 256) return cudaErrorInvalidValue;
  const int64_t n = T * k;
  const int nch = (int)((n + kRouteChunk - 1) / kRouteChunk);
  int32_t* hist = reinterpret_cast<int32_t*>(scratch);
  if (nch > 0) {
    route_count_kernel<<<nch, 256, 0, st>>>(ids, n, E, hist, err);
  }
  route_scan_kernel<<<(E + 7) / 8, 256, 0, st>>>(hist, nch, E, counts);
  route_place_kernel<<<nch > 0 ? nch : 1, 256, 0, st>>>(ids, topk_w, n, k, E, S, T, hist, counts, offsets, v_off,
                                                        perm, row_src, row_w, row_exp, inv);
  if (row_src && S > 0 && T > 0) {
    route_shared_kernel<<<(unsigned)((T * S + 255) / 256), 256, 0, st>>>(T, E, S, shared_w, row_src, row_w, row_exp);
  }
  return cudaGetLastError();
}

cudaError_t launch_gather_quant(const void* x, int d, const int32_t* row_src, const int32_t* row_exp,
                                const int32_t* v_off, int V,
                                const ExpertDesc* ex, int64_t R, void* Xb, void* XqA, float* XsA, void* XqB, float* XsB,
                                int32_t* XcA, int32_t* XcB, uint32_t* hmax, cudaStream_t st) {
  if (R <= 0) return cudaSuccess;
  if (XqA != nullptr || XqB != nullptr)
    gather_quant_kernel<true><<<(unsigned)((R * 32 + 255) / 256), 256, 0, st>>>(
        (const uint16_t*)x, d, row_src, row_exp, v_off, V, ex, R, (uint16_t*)Xb, (int8_t*)XqA, XsA, (int8_t*)XqB, XsB,
        XcA, XcB, hmax);
  else
    gather_quant_kernel<false><<<(unsigned)((R * 32 + 255) / 256), 256, 0, st>>>(
        (const uint16_t*)x, d, row_src, row_exp, v_off, V, ex, R, (uint16_t*)Xb, (int8_t*)XqA, XsA, (int8_t*)XqB, XsB,
        XcA, XcB, hmax);
  return cudaGetLastError();
}

cudaError_t launch_gather_tok(const void* x, int d, int64_t T, int k, int S, int E, const int32_t* inv,
                              const int32_t* row_exp, const ExpertDesc* ex, const ActFormats& fm, int64_t R, void* Xb,
                              void* XqA, float* XsA, void* XqB, float* XsB, int32_t* XcA, int32_t* XcB, uint32_t* hmax,
                              cudaStream_t st) {
  if (T <= 0 || fm.n <= 0) return cudaSuccess;
  const int64_t warps = T * fm.n;
  gather_tok_kernel<32><<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(
      (const uint16_t*)x, d, T, k, S, E, inv, row_exp, ex, fm, R, (uint16_t*)Xb, (int8_t*)XqA, XsA, (int8_t*)XqB,
      XsB, XcA, XcB, hmax);
  return cudaGetLastError();
}

cudaError_t launch_combine(const void* O, int d, int64_t T, int k, int S, const int32_t* inv, void* y,
                           cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  combine_kernel<<<(unsigned)T, 128, 0, st>>>((const uint16_t*)O, d, T, k, S, inv, (uint16_t*)y);
  return cudaGetLastError();
}

}  // namespace mxm
