// gemm.cu — steps S4-S7: the persistent heterogeneous-tile mixed-precision group-GEMM.
//
// One launch, one CTA per SM (grid = #SMs), dynamic task queue built by plan.cu in LPT order
// (P:231). Each task is a 128-output-channel tile of one linear block of one expert over one
// m-tile of that expert's routed tokens ("swap-AB": weights are the MMA's A operand with
// M = 128 channels, tokens are B with N = 16..128):
//   phase 0: gate & up (same scheme -> one K loop sharing the token tile; else two K loops),
//            fused SwiGLU epilogue h = bf16(silu(g) * u)   (Eq. 1; DESIGN R15/R16)
//   phase 1: dynamic per-token / per-128-group quantization of h for weight-activation downs
//   phase 2: down, epilogue o * w_e -> bf16 (Eq. 2)
// Warp roles ("micro-kernels ... CTA-index independent", "same number of warps"):
//   warp 0      producer: queue pop, dependency wait, bulk copy of packed weight chunks, TMA of tokens
//   warp 1      MMA issuer: tcgen05.mma kind::f16 (weight-only / bf16) or kind::i8 (weight-activation)
//   warp 2      TMEM allocator (512 columns = 4 accumulator buffers of 128 columns)
//   warps 4-7   transform: packed codes -> bf16 (dequant, weight-only) or s8 (w4/w5 unpack) A tiles
//   warps 8-15  epilogue (2 warpgroups split the token columns): TMEM -> scales -> SwiGLU / w_e -> HBM
// Weight-activation g128 blocks drain the int32 accumulator every 128-K group (the group scales
// s_w[n,g] s_a[m,g] differ per group; "W4A4-g128 ... strict adherence to 128 quantization
// group"), ping-ponging between TMEM buffers so the tensor core keeps running.
#include <cuda_bf16.h>
#include <cstdint>

#include "actq.cuh"
#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace mxm {

constexpr int kStages = 3;
constexpr int kRing = 4;
constexpr int kAccBufs = 4;
constexpr int kThreads = 512;
constexpr int kRawBytes = 10752;
constexpr int kTileBytes = 16384;

constexpr int kOffA = 0;
constexpr int kOffB = kOffA + kStages * 2 * kTileBytes;
constexpr int kOffRaw = kOffB + kStages * kTileBytes;
constexpr int kOffCtl = kOffRaw + kStages * 2 * kRawBytes;
constexpr int kCtlBytes = 512;
constexpr int kSmemBytes = kOffCtl + kCtlBytes + 1024;

struct Ctl {
  uint64_t full[kStages], empty[kStages], aready[kStages];
  uint64_t accf[kAccBufs], acce[kAccBufs];
  uint64_t tfull[kRing], tempty[kRing];
  Task ring[kRing];
  uint32_t tmem_base;
};
static_assert(sizeof(Ctl) <= kCtlBytes, "ctl");

struct SubLoop {
  const LinDesc* mat[2];
  int nmats, bmap, ns, i8, xform, g128;
};

__device__ __forceinline__ SubLoop make_sl(const LinDesc* a, const LinDesc* b, int bmap) {
  SubLoop s;
  s.mat[0] = a;
  s.mat[1] = b;
  s.nmats = b ? 2 : 1;
  s.bmap = bmap;
  s.ns = a->geo.ns;
  s.i8 = kind_is_i8(a->geo.kind);
  s.xform = kind_needs_transform(a->geo.kind);
  s.g128 = s.i8 && a->geo.group == 128;
  return s;
}

__device__ __forceinline__ int build_subloops(const Task& t, const ExpertDesc* __restrict__ ex, SubLoop* sl) {
  const ExpertDesc& e = ex[t.expert];
  if (t.phase == 0) {
    if (e.same_gu) {
      sl[0] = make_sl(&e.blk[0], &e.blk[1], e.blk[0].in_slot);
      return 1;
    }
    sl[0] = make_sl(&e.blk[0], nullptr, e.blk[0].in_slot);
    sl[1] = make_sl(&e.blk[1], nullptr, e.blk[1].in_slot);
    return 2;
  }
  sl[0] = make_sl(&e.blk[2], nullptr, 3 + e.blk[2].in_slot);
  return 1;
}

__device__ __forceinline__ int nt_index(int nt) { return nt <= 16 ? 0 : (nt <= 32 ? 1 : (nt <= 64 ? 2 : 3)); }

// ---------------------------------------------------------------- transforms (one thread per A row)
__device__ __forceinline__ uint32_t bf2_sub(uint32_t a, uint32_t b) {
  __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&a), y = *reinterpret_cast<__nv_bfloat162*>(&b);
  __nv_bfloat162 r = __hsub2(x, y);
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t bf2_fma(uint32_t a, uint32_t b, uint32_t c) {
  __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&a), y = *reinterpret_cast<__nv_bfloat162*>(&b),
                 z = *reinterpret_cast<__nv_bfloat162*>(&c);
  __nv_bfloat162 r = __hfma2(x, y, z);
  return *reinterpret_cast<uint32_t*>(&r);
}
// (128 + u_even, 128 + u_odd) as bf16x2 -> q*s + z rounded once to bf16 (q = u - off)
__device__ __forceinline__ uint32_t deq_pair(uint32_t fields, uint32_t off2, uint32_t s2, uint32_t z2) {
  return bf2_fma(bf2_sub(fields | 0x43004300u, off2), s2, z2);
}

__device__ __forceinline__ void xform_wo(const uint8_t* __restrict__ raw, uint8_t* __restrict__ A, const PackGeom& g,
                                         int ks, int r, uint32_t& s2, uint32_t& z2) {
  const uint8_t* codes = raw;
  if (chunk_has_meta(g, ks)) {
    const uint32_t sb = reinterpret_cast<const uint16_t*>(raw)[r];
    s2 = sb | (sb << 16);
    if (!g.sym) {
      const uint32_t zb = reinterpret_cast<const uint16_t*>(raw + 256)[r];
      z2 = zb | (zb << 16);
    } else {
      z2 = 0;
    }
    codes += g.meta_bytes;
  }
  const uint32_t* w = reinterpret_cast<const uint32_t*>(codes);
  uint8_t* dst = A + r * 128;
  const int sw = r & 7;
  const uint32_t off = g.sym ? (1u << (g.w_bits - 1)) : 0u;
  const uint32_t off2 = (0x4300u | off) * 0x10001u;
  if (g.w_bits == 4) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t word = w[j * 128 + r];
      uint4 o;
      o.x = deq_pair(word & 0x000F000Fu, off2, s2, z2);
      o.y = deq_pair((word >> 4) & 0x000F000Fu, off2, s2, z2);
      o.z = deq_pair((word >> 8) & 0x000F000Fu, off2, s2, z2);
      o.w = deq_pair((word >> 12) & 0x000F000Fu, off2, s2, z2);
      *reinterpret_cast<uint4*>(dst + ((j ^ sw) << 4)) = o;
    }
  } else if (g.w_bits == 2) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t word = w[j * 128 + r];
      uint4 o0, o1;
      o0.x = deq_pair(word & 0x00030003u, off2, s2, z2);
      o0.y = deq_pair((word >> 2) & 0x00030003u, off2, s2, z2);
      o0.z = deq_pair((word >> 4) & 0x00030003u, off2, s2, z2);
      o0.w = deq_pair((word >> 6) & 0x00030003u, off2, s2, z2);
      o1.x = deq_pair((word >> 8) & 0x00030003u, off2, s2, z2);
      o1.y = deq_pair((word >> 10) & 0x00030003u, off2, s2, z2);
      o1.z = deq_pair((word >> 12) & 0x00030003u, off2, s2, z2);
      o1.w = deq_pair((word >> 14) & 0x00030003u, off2, s2, z2);
      *reinterpret_cast<uint4*>(dst + (((2 * j) ^ sw) << 4)) = o0;
      *reinterpret_cast<uint4*>(dst + (((2 * j + 1) ^ sw) << 4)) = o1;
    }
  } else if (g.w_bits == 3) {
    const uint32_t* wh = w + 4 * 128;
    const uint32_t h0 = wh[r], h1 = wh[128 + r];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t word = w[j * 128 + r];
      const uint32_t hw = ((j >> 1) ? h1 : h0) >> (8 * (j & 1));
      uint32_t p[8];
#pragma unroll
      for (int t = 0; t < 8; ++t)
        p[t] = deq_pair(((word >> (2 * t)) & 0x00030003u) | (((hw >> t) & 0x00010001u) << 2), off2, s2, z2);
      *reinterpret_cast<uint4*>(dst + (((2 * j) ^ sw) << 4)) = make_uint4(p[0], p[1], p[2], p[3]);
      *reinterpret_cast<uint4*>(dst + (((2 * j + 1) ^ sw) << 4)) = make_uint4(p[4], p[5], p[6], p[7]);
    }
  } else {  // 8-bit: fp32 path (128 + u is not exact in bf16 for u >= 128)
    const float sf = __uint_as_float(s2 << 16), zf = __uint_as_float(z2 << 16), fo = (float)off;
#pragma unroll 4
    for (int c = 0; c < 8; ++c) {
      uint32_t o[4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t word = w[(2 * c + h) * 128 + r];
        float f[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) f[b] = (__uint_as_float(0x4B000000u | ((word >> (8 * b)) & 0xFFu)) - 8388608.f) - fo;
        __nv_bfloat162 lo = __floats2bfloat162_rn(fmaf(f[0], sf, zf), fmaf(f[1], sf, zf));
        __nv_bfloat162 hi = __floats2bfloat162_rn(fmaf(f[2], sf, zf), fmaf(f[3], sf, zf));
        o[2 * h] = *reinterpret_cast<uint32_t*>(&lo);
        o[2 * h + 1] = *reinterpret_cast<uint32_t*>(&hi);
      }
      *reinterpret_cast<uint4*>(dst + ((c ^ sw) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

__device__ __forceinline__ uint32_t to_s8_4(uint32_t u, uint32_t bias) { return (u + bias) ^ 0x80808080u; }

__device__ __forceinline__ void xform_wa(const uint8_t* __restrict__ raw, uint8_t* __restrict__ A, const PackGeom& g,
                                         int r) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(raw);
  uint8_t* dst = A + r * 128;
  const int sw = r & 7;
  if (g.w_bits == 4) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t w0 = w[(2 * c) * 128 + r], w1 = w[(2 * c + 1) * 128 + r];
      uint4 o;
      o.x = to_s8_4(w0 & 0x0F0F0F0Fu, 0x78787878u);
      o.y = to_s8_4((w0 >> 4) & 0x0F0F0F0Fu, 0x78787878u);
      o.z = to_s8_4(w1 & 0x0F0F0F0Fu, 0x78787878u);
      o.w = to_s8_4((w1 >> 4) & 0x0F0F0F0Fu, 0x78787878u);
      *reinterpret_cast<uint4*>(dst + ((c ^ sw) << 4)) = o;
    }
  } else {  // w5: 4-bit plane (16 words) + 1-bit plane (4 words)
    const uint32_t* wh = w + 16 * 128;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint32_t o[4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 2 * c + h;
        const uint32_t word = w[j * 128 + r];
        const uint32_t hb = wh[(j >> 2) * 128 + r];
        const int t0 = 2 * (j & 3);
        const uint32_t lo = (word & 0x0F0F0F0Fu) | (((hb >> t0) & 0x01010101u) << 4);
        const uint32_t hi = ((word >> 4) & 0x0F0F0F0Fu) | (((hb >> (t0 + 1)) & 0x01010101u) << 4);
        o[2 * h] = to_s8_4(lo, 0x70707070u);
        o[2 * h + 1] = to_s8_4(hi, 0x70707070u);
      }
      *reinterpret_cast<uint4*>(dst + ((c ^ sw) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// ---------------------------------------------------------------- epilogue helpers
__device__ __forceinline__ float silu_f(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

__device__ __forceinline__ float bf16f(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }

__device__ __forceinline__ uint16_t f2bf(float f) {
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}

// ---------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(kThreads, 1) moe_gemm_kernel(const __grid_constant__ GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Ctl& ctl = *reinterpret_cast<Ctl*>(smem + kOffCtl);
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  auto tileA = [&](int s, int m) { return smem + kOffA + (s * 2 + m) * kTileBytes; };
  auto tileB = [&](int s) { return smem + kOffB + s * kTileBytes; };
  auto tileRaw = [&](int s, int m) { return smem + kOffRaw + (s * 2 + m) * kRawBytes; };

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&ctl.full[i], 1);
      mbar_init(&ctl.empty[i], 1);
      mbar_init(&ctl.aready[i], 4);
    }
    for (int i = 0; i < kAccBufs; ++i) {
      mbar_init(&ctl.accf[i], 1);
      mbar_init(&ctl.acce[i], 8);
    }
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&ctl.tfull[i], 1);
      mbar_init(&ctl.tempty[i], 13);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&ctl.tmem_base);
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 5; ++i)
      for (int j = 0; j < 4; ++j) prefetch_tmap(&p.tmap[i][j]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl.tmem_base;
  const int n_tasks = p.meta[0];

  if (warp == 0) {
    // =========================== producer
    if (lane == 0) {
      uint32_t stage = 0, sphase = 0;
      for (uint32_t it = 0;; ++it) {
        const uint32_t slot = it % kRing, rphase = (it / kRing) & 1;
        const int idx = atomicAdd(&p.meta[5], 1);
        Task t;
        if (idx < n_tasks) {
          t = p.tasks[idx];
        } else {
          t.phase = 255;
        }
        mbar_wait(&ctl.tempty[slot], rphase ^ 1);
        ctl.ring[slot] = t;
        mbar_arrive(&ctl.tfull[slot]);
        if (t.phase == 255) break;
        if (t.phase == 1) continue;
        if (t.phase == 2) {
          const ExpertDesc& e = p.ex[t.expert];
          const bool wa = kind_is_i8(e.blk[2].geo.kind);
          const int* ctr = (wa ? p.hq_done : p.p1_done) + t.gid;
          const int need = wa ? p.grp_nq[t.gid] : p.grp_n1[t.gid];
          while (ld_acquire_gpu(ctr) < need) __nanosleep(64);
          fence_proxy_async_global();
        }
        SubLoop sl[2];
        const int nsl = build_subloops(t, p.ex, sl);
        const int nti = nt_index(t.nt);
        for (int si = 0; si < nsl; ++si) {
          const SubLoop& s = sl[si];
          const CUtensorMap* map = &p.tmap[s.bmap][nti];
          for (int ks = 0; ks < s.ns; ++ks) {
            mbar_wait(&ctl.empty[stage], sphase ^ 1);
            uint32_t bytes = (uint32_t)t.nt * 128u;
            uint32_t cb[2];
            for (int m = 0; m < s.nmats; ++m) {
              const PackGeom& g = s.mat[m]->geo;
              cb[m] = (uint32_t)g.code_bytes + (chunk_has_meta(g, ks) ? (uint32_t)g.meta_bytes : 0u);
              bytes += cb[m];
            }
            mbar_arrive_expect_tx(&ctl.full[stage], bytes);
            for (int m = 0; m < s.nmats; ++m) {
              const LinDesc& L = *s.mat[m];
              const uint8_t* src = L.packed + chunk_offset(L.geo, t.ntile, ks);
              bulk_load(s.xform ? tileRaw(stage, m) : tileA(stage, m), src, cb[m], &ctl.full[stage]);
            }
            tma_load_2d(tileB(stage), map, &ctl.full[stage], ks * (s.i8 ? 128 : 64), t.row0);
            if (++stage == kStages) {
              stage = 0;
              sphase ^= 1;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // =========================== MMA issuer
    if (lane == 0) {
      uint32_t stage = 0, sphase = 0, abuf = 0;
      uint32_t acc_uses[kAccBufs] = {0, 0, 0, 0};
      uint32_t ar_uses[kStages] = {0, 0, 0};
      for (uint32_t it = 0;; ++it) {
        const uint32_t slot = it % kRing, rphase = (it / kRing) & 1;
        mbar_wait(&ctl.tfull[slot], rphase);
        const Task t = ctl.ring[slot];
        mbar_arrive(&ctl.tempty[slot]);
        if (t.phase == 255) break;
        if (t.phase == 1) continue;
        SubLoop sl[2];
        const int nsl = build_subloops(t, p.ex, sl);
        for (int si = 0; si < nsl; ++si) {
          const SubLoop& s = sl[si];
          const int nbuf = (s.nmats == 2 && !s.g128) ? 2 : 1;
          const uint32_t idesc = s.i8 ? idesc_s8(t.nt) : idesc_bf16(t.nt);
          uint32_t bufs[2] = {0, 0};
          for (int ks = 0; ks < s.ns; ++ks) {
            const bool ev_start = s.g128 || ks == 0, ev_end = s.g128 || ks == s.ns - 1;
            if (ev_start) {
              for (int b = 0; b < nbuf; ++b) {
                bufs[b] = abuf;
                mbar_wait(&ctl.acce[abuf], (acc_uses[abuf] & 1) ^ 1);
                ++acc_uses[abuf];
                abuf = (abuf + 1) % kAccBufs;
              }
            }
            mbar_wait(&ctl.full[stage], sphase);
            if (s.xform) {
              mbar_wait(&ctl.aready[stage], ar_uses[stage] & 1);
              ++ar_uses[stage];
            }
            tc_fence_after();
            const uint32_t bbase = smem_u32(tileB(stage));
            for (int m = 0; m < s.nmats; ++m) {
              const uint32_t col = nbuf == 2 ? bufs[m] * 128u : bufs[0] * 128u + (uint32_t)m * 64u;
              const uint32_t abase = smem_u32(tileA(stage, m));
              const bool first = s.g128 || ks == 0;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint64_t ad = sw128_kmajor_desc(abase + k * 32);
                const uint64_t bd = sw128_kmajor_desc(bbase + k * 32);
                const uint32_t acc = (first && k == 0) ? 0u : 1u;
                if (s.i8)
                  mma_i8(tmem + col, ad, bd, idesc, acc);
                else
                  mma_bf16(tmem + col, ad, bd, idesc, acc);
              }
            }
            mma_commit(&ctl.empty[stage]);
            if (ev_end)
              for (int b = 0; b < nbuf; ++b) mma_commit(&ctl.accf[bufs[b]]);
            if (++stage == kStages) {
              stage = 0;
              sphase ^= 1;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 8) {
    // =========================== transform warpgroup
    const int r = threadIdx.x - 128;
    uint32_t stage = 0, sphase = 0;
    for (uint32_t it = 0;; ++it) {
      const uint32_t slot = it % kRing, rphase = (it / kRing) & 1;
      mbar_wait(&ctl.tfull[slot], rphase);
      const Task t = ctl.ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl.tempty[slot]);
      if (t.phase == 255) break;
      if (t.phase == 1) continue;
      SubLoop sl[2];
      const int nsl = build_subloops(t, p.ex, sl);
      for (int si = 0; si < nsl; ++si) {
        const SubLoop& s = sl[si];
        uint32_t s2[2] = {0, 0}, z2[2] = {0, 0};
        for (int ks = 0; ks < s.ns; ++ks) {
          if (s.xform) {
            mbar_wait(&ctl.full[stage], sphase);
            for (int m = 0; m < s.nmats; ++m) {
              const PackGeom& g = s.mat[m]->geo;
              if (s.i8)
                xform_wa(tileRaw(stage, m), tileA(stage, m), g, r);
              else
                xform_wo(tileRaw(stage, m), tileA(stage, m), g, ks, r, s2[m], z2[m]);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&ctl.aready[stage]);
          }
          if (++stage == kStages) {
            stage = 0;
            sphase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 8) {
    // =========================== epilogue (2 warpgroups)
    const int ew = warp - 8, wg = ew >> 2, q = warp & 3;
    const int l = q * 32 + lane;  // output channel within the tile == TMEM lane
    uint32_t abuf = 0;
    uint32_t acc_uses[kAccBufs] = {0, 0, 0, 0};
    for (uint32_t it = 0;; ++it) {
      const uint32_t slot = it % kRing, rphase = (it / kRing) & 1;
      mbar_wait(&ctl.tfull[slot], rphase);
      const Task t = ctl.ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl.tempty[slot]);
      if (t.phase == 255) break;
      const ExpertDesc& E = p.ex[t.expert];
      if (t.phase == 1) {
        // ---- dynamic quantization of h for a weight-activation down block (rows of one 32-row chunk)
        if (ew == 0 && lane == 0) {
          const int need = p.grp_n1[t.gid];
          while (ld_acquire_gpu(p.p1_done + t.gid) < need) __nanosleep(64);
        }
        named_bar_sync(1, 256);
        const LinDesc& L = E.blk[2];
        const int K = E.inter;
        const int g = L.a_group == -1 ? K : L.a_group;
        const int qmax = (1 << (L.a_bits - 1)) - 1;
        const int sub0 = t.ntile * 32;
        for (int rr = ew; rr < 32; rr += 8) {
          const int local = sub0 + rr;
          if (local >= t.rows) break;
          const int64_t row = (int64_t)t.row0 + local;
          const uint16_t* src = p.H + row * p.f_max;
          int8_t* dst = p.Hq + row * p.f_max;
          for (int gi = 0; gi < K / g; ++gi) {
            const float s = quant_group_warp<true>(src + gi * g, dst + gi * g, g, qmax, nullptr);
            if (lane == 0) p.Hs[row * (p.f_max / 128) + gi] = s;
          }
        }
        named_bar_sync(1, 256);
        if (ew == 0 && lane == 0) {
          __threadfence();
          atomicAdd(p.hq_done + t.gid, 1);
          atomicAdd(p.meta + 6, 1);
        }
        continue;
      }
      SubLoop sl[2];
      const int nsl = build_subloops(t, p.ex, sl);
      const bool reg_mode = nsl == 2 || sl[0].g128;
      const int half = t.nt >> 1;
      const int col0 = wg * half;
      const int n = t.ntile * 128 + l;
      const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
      float acc[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) acc[i] = 0.f;
      const float* xs = t.phase == 0 ? p.xs[E.blk[0].in_slot] : p.Hs;
      const int xs_stride = t.phase == 0 ? p.d / 128 : p.f_max / 128;

      for (int si = 0; si < nsl; ++si) {
        const SubLoop& s = sl[si];
        const int nbuf = (s.nmats == 2 && !s.g128) ? 2 : 1;
        const int nev = s.g128 ? s.ns : 1;
        const float* xs_s = (t.phase == 0) ? p.xs[s.mat[0]->in_slot] : p.Hs;
        for (int ev = 0; ev < nev; ++ev) {
          uint32_t bufs[2] = {0, 0};
          for (int b = 0; b < nbuf; ++b) {
            bufs[b] = abuf;
            abuf = (abuf + 1) % kAccBufs;
          }
          for (int b = 0; b < nbuf; ++b) {
            mbar_wait(&ctl.accf[bufs[b]], acc_uses[bufs[b]] & 1);
            ++acc_uses[bufs[b]];
          }
          tc_fence_after();
          // per-mat weight scale (weight-activation) for this event's group
          float sw[2] = {1.f, 1.f};
          if (s.i8) {
            const int gi = s.g128 ? ev : 0;
            for (int m = 0; m < s.nmats; ++m) {
              const LinDesc& L = *s.mat[m];
              sw[m] = bf16f(reinterpret_cast<const uint16_t*>(L.packed + L.geo.wa_scale_off)[(int64_t)gi * L.geo.N + n]);
            }
          }
          const int gi = s.g128 ? ev : 0;
          if (!reg_mode) {
            // ---- streaming epilogue: one drain event for the whole task
#pragma unroll 1
            for (int c = 0; c < half; c += 8) {
              uint32_t va[8], vb[8];
              const uint32_t cbase = (uint32_t)(col0 + c);
              const uint32_t colA = nbuf == 2 ? bufs[0] * 128u : bufs[0] * 128u;
              tmem_ld8(lane_addr + colA + cbase, va);
              if (s.nmats == 2) tmem_ld8(lane_addr + bufs[1] * 128u + cbase, vb);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int col = col0 + c + j;
                if (col >= t.rows) break;
                const int64_t row = (int64_t)t.row0 + col;
                float sa = 1.f;
                if (s.i8) sa = __ldg(xs_s + row * xs_stride + gi);
                if (t.phase == 0) {
                  float g, u;
                  if (s.i8) {
                    g = (float)(int32_t)va[j] * (sw[0] * sa);
                    u = (float)(int32_t)vb[j] * (sw[1] * sa);
                  } else {
                    g = __uint_as_float(va[j]);
                    u = __uint_as_float(vb[j]);
                  }
                  p.H[row * p.f_max + n] = f2bf(silu_f(g) * u);
                } else {
                  float o = s.i8 ? (float)(int32_t)va[j] * (sw[0] * sa) : __uint_as_float(va[j]);
                  o *= __ldg(p.row_w + row);
                  p.O[row * p.d + n] = f2bf(o);
                }
              }
            }
          } else {
            // ---- register-accumulating epilogue (g128 drains / hetero gate-up)
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              if (c * 8 < half) {
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                  if (m < s.nmats) {
                    uint32_t v[8];
                    const uint32_t colm = nbuf == 2 ? bufs[m] * 128u : bufs[0] * 128u + (uint32_t)m * 64u;
                    tmem_ld8(lane_addr + colm + (uint32_t)(col0 + c * 8), v);
                    tmem_ld_wait();
                    // destination: dual (phase 0): gate -> acc[0..31], up -> acc[32..63]; single: acc[0..63]
                    const int slot_m = (t.phase == 0) ? ((nsl == 2 ? si : m) * 32) : 0;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                      const int col = col0 + c * 8 + j;
                      float val;
                      if (s.i8) {
                        const float sa = col < t.rows ? __ldg(xs_s + ((int64_t)t.row0 + col) * xs_stride + gi) : 0.f;
                        val = (float)(int32_t)v[j] * (sw[m] * sa);
                      } else {
                        val = __uint_as_float(v[j]);
                      }
                      const int ai = slot_m + c * 8 + j;
                      if (ai < 64) acc[ai] += val;
                    }
                  }
                }
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0)
            for (int b = 0; b < nbuf; ++b) mbar_arrive(&ctl.acce[bufs[b]]);
        }
      }
      if (reg_mode) {
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          if (c < half) {
            const int col = col0 + c;
            if (col < t.rows) {
              const int64_t row = (int64_t)t.row0 + col;
              if (t.phase == 0) {
                if (c < 32) p.H[row * p.f_max + n] = f2bf(silu_f(acc[c]) * acc[32 + c]);
              } else {
                p.O[row * p.d + n] = f2bf(acc[c] * __ldg(p.row_w + row));
              }
            }
          }
        }
      }
      if (t.phase == 0) {
        named_bar_sync(1, 256);
        if (ew == 0 && lane == 0) {
          __threadfence();
          atomicAdd(p.p1_done + t.gid, 1);
        }
      }
      if (ew == 0 && lane == 0) atomicAdd(p.meta + 6, 1);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

cudaError_t launch_moe_gemm(const GemmParams& prm, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(moe_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  moe_gemm_kernel<<<grid, kThreads, kSmemBytes, st>>>(prm);
  return cudaGetLastError();
}

}  // namespace mxm
