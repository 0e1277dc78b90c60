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
//   warp 1      TMEM allocator (512 columns = 4 accumulator buffers of 128 columns) and MMA issuer:
//               tcgen05.mma kind::f16 (weight-only / bf16) or kind::i8 (weight-activation)
//   warps 4-7   transform: packed codes -> bf16 (dequant, weight-only) or s8 (w4/w5 unpack) A tiles
//   warps 8-15  epilogue (2 warpgroups split the token columns): TMEM -> scales -> SwiGLU / w_e -> HBM
// Weight-activation g128 blocks drain the int32 accumulator every 128-K group (the group scales
// s_w[n,g] s_a[m,g] differ per group; "W4A4-g128 ... strict adherence to 128 quantization
// group"), ping-ponging between TMEM buffers so the tensor core keeps running.
#include <cuda_bf16.h>
#include <cstdint>
#include <mutex>
#include <type_traits>

#include "actq.cuh"
#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace mxm {

#ifndef MXM_STAGES
#define MXM_STAGES 4
#endif
#ifndef MXM_TILE_KB
#define MXM_TILE_KB 16
#endif
#ifndef MXM_SSLOTS
#define MXM_SSLOTS 8
#endif
#ifndef MXM_LANE_ARRIVE
#define MXM_LANE_ARRIVE 0  // 1: every lane arrives on the g128 scale-slot barriers (round-1 protocol)
#endif
constexpr int kStages = MXM_STAGES;
constexpr int kRing = 4;
// TMEM (512 columns): two accumulator buffers of 192 columns at [0, 384) -- a dual tile (gate | up, or two
// 128-channel down tiles) of up to 96 tokens fits one buffer, so every task is double-buffered against the
// next one's MMAs -- and a 2-slot A ring at [384, 512) for TS-form MMAs (dequantized weights; per slot
// 2 mats x 32 columns), decoupled from the 4 smem stages by its own ready / empty barriers.
// MXM_ASLOTS=3 (2 x 160 accumulator columns, 80-token tiles, 3 A slots) was measured slower on every
// config (DSV2 GEMM 0.93 -> 1.09 ms): the smaller tiles cost more than the deeper A ring saves.
constexpr int kAccBufs = MXM_ACC_BUFS;
constexpr int kASlots = MXM_ASLOTS;
constexpr int kAccCols = kAccBufs == 3 ? 128 : (kASlots == 3 ? 160 : 192);  // 2x160+3x64 = 2x192+2x64 = 3x128+2x64
constexpr int kMat1Col = kAccCols / 2;               // column offset of mat 1 inside an accumulator buffer
constexpr int kTmemA = kAccBufs * kAccCols;
static_assert(kTmemA + 64 * kASlots == 512, "TMEM partition");
static_assert(kMat1Col == MXM_DUAL_TILE, "dual token tile (common.cuh) must match the accumulator buffer");
constexpr int kThreads = 640;  // 20 warps: producer, MMA issuer, 2 scale staging, 4 transform, 8 epilogue, 4 transform
constexpr int kXfWarps = 8;     // transform warps 4..7 (K half 0) and 16..19 (K half 1); one A row per thread
constexpr int kTileBytes = MXM_TILE_KB * 1024;
constexpr int kSlotBytes = 3 * kTileBytes;  // per stage: token tile B | mat 0 (raw codes or A image) | mat 1

constexpr int kOffCtl = kStages * kSlotBytes;
constexpr int kCtlBytes = 8192;
// scale ring for weight-activation g128 stages (one 128-K group each): the producer bulk-copies the group's
// weight scales (128 bf16 per mat) and activation scales (the m-tile's rows of the group-major [g][R]
// array, from the 16-byte-aligned floor) next to the stage's operands; the epilogue drains the event's
// accumulator against them, then releases the slot.
constexpr int kSSlots = MXM_SSLOTS;
// scale slot of one g128 drain event, written by the staging warp (stage_scales) from global memory: [0,256) mat-0
// s_w | [256,512) mat-1 s_w (bf16 per channel) | [512,1024) per token column drain factor a (s_a, or s_a 2^18 for
// w4a4) | [1024,1536) w4a4 offset correction b = -8 s_a sum(q_a); 16-B aligned from column 0 so the epilogue reads
// the factors as broadcast float4s
constexpr int kSSlotBytes = 1536;
constexpr int kSlotA = 512, kSlotB = 1024;
constexpr int kOffScale = kOffCtl + kCtlBytes;
constexpr int kSmemBytes = kOffScale + kSSlots * kSSlotBytes + 1024;

struct Ctl {
  uint64_t full[kStages], empty[kStages];
  uint64_t aready[kASlots], aempty[kASlots];
  uint64_t sfull[kSSlots], sempty[kSSlots], sready[kSSlots];
  uint64_t accf[kAccBufs], acce[kAccBufs];
  uint64_t tfull[kRing], tempty[kRing];
  Task ring[kRing];
  uint32_t tmem_base;
  int red_last;  // split-K: this CTA's slice arrived last (epilogue broadcast)
  uint32_t colmax[2][2][4][8];  // [buffer][warpgroup][lane quarter][column] for the fused g128 h-quant
  alignas(16) float cw[8][3][64];  // per epilogue warp and token column (broadcast reads): [0] activation scale
                                   // of the current drain event (w4a4: s_a * 2^18), [1] route weight,
                                   // [2] w4a4 offset correction -8 s_a sum(q_a) of the event
  int32_t colsum[2][2][4][8];      // [buffer][warpgroup][lane quarter][column]: fused g128 h-quant code sums (w4a4)
};
static_assert(sizeof(Ctl) <= kCtlBytes, "ctl");

struct SubLoop {
  const LinDesc* mat[2];
  int tile[2];                           // 128-channel output tile of each mat
  int nmats, bmap, ns, i8, f8, xform, g128;  // i8: W-A (8-bit operands); f8: kind::f8f6f4 (w4a4 or FP8)
  int w4;                                     // w4a4 (nibble-offset accumulators: a = s_a 2^18, correction b)
                                              // xform: bit m set = mat m needs the packed->A transform
  int ks0, ks1;                           // stage range (a split-K slice of a down task, else [0, ns))
};

__device__ __forceinline__ SubLoop make_sl(const LinDesc* a, const LinDesc* b, int bmap, int tile0, int tile1) {
  SubLoop s;
  s.mat[0] = a;
  s.mat[1] = b;
  s.tile[0] = tile0;
  s.tile[1] = tile1;
  s.nmats = b ? 2 : 1;
  s.bmap = bmap;
  s.ns = a->geo.ns;
  s.i8 = kind_is_wa(a->geo.kind);
  s.f8 = kind_is_f8(a->geo.kind);
  s.w4 = kind_is_w4a4(a->geo.kind);
  s.xform = (kind_needs_transform(a->geo.kind) ? 1 : 0) | ((b && kind_needs_transform(b->geo.kind)) ? 2 : 0);
  s.g128 = s.i8 && a->geo.group == 128;
  s.ks0 = 0;
  s.ks1 = s.ns;
  return s;
}

// phase 0: gate & up share the token tile (one sub-loop when dual); phase 2: a task covers down tiles
// (2j, 2j+1) as two mats sharing the h tile when down_pair() (common.cuh), else tile j alone
__device__ __forceinline__ int build_subloops(const Task& t, const ExpertDesc* __restrict__ ex, int d, int S,
                                              SubLoop* sl) {
  const ExpertDesc& e = ex[t.expert];
  const int tile = task_tile(t);
  if (t.phase == 0) {
    if (e.dual) {
      sl[0] = make_sl(&e.blk[0], &e.blk[1], e.blk[0].in_slot, t.ntile, t.ntile);
      return 1;
    }
    sl[0] = make_sl(&e.blk[0], nullptr, e.blk[0].in_slot, t.ntile, t.ntile);
    sl[1] = make_sl(&e.blk[1], nullptr, e.blk[1].in_slot, t.ntile, t.ntile);
    return 2;
  }
  const int nd = d / 128;
  if (down_pair(e, t.nt, nd)) {
    const int j0 = 2 * tile;
    const bool two = j0 + 1 < nd;
    sl[0] = make_sl(&e.blk[2], two ? &e.blk[2] : nullptr, 3 + e.blk[2].in_slot, j0, j0 + 1);
  } else {
    sl[0] = make_sl(&e.blk[2], nullptr, 3 + e.blk[2].in_slot, tile, tile);
  }
  if (S > 1 && down_splittable(e)) split_range(sl[0].ns, S, task_slice(t), sl[0].ks0, sl[0].ks1);
  return 1;
}

__device__ __forceinline__ int nt_index(int nt) { return nt <= 16 ? 0 : (nt <= 32 ? 1 : (nt <= 64 ? 2 : 3)); }  // box 16/32/64/dual

// activation scales of group g for rows [row0, row0 + nt): 16-byte-aligned source span and element offset
__device__ __forceinline__ const float* ascale_span(const float* base, int64_t R, int g, int row0, uint32_t& off) {
  const float* p = base + (int64_t)g * R + row0;
  off = (uint32_t)(((uintptr_t)p & 15u) >> 2);
  return p - off;
}

#ifdef MXM_DEBUG_NAN
// first non-finite value seen: [site, expert, phase, ntile, ks, row0, block, extra] at prof[148*16 ..]
__device__ unsigned long long g_nan_info[8];
__device__ __forceinline__ void nan_note(unsigned long long*, int site, const Task& t, int ks, int extra) {
  unsigned long long* info = g_nan_info;
  if (atomicCAS(info, 0ull, (unsigned long long)site) == 0ull) {
    info[1] = t.expert; info[2] = t.phase; info[3] = t.ntile; info[4] = ks; info[5] = t.row0; info[6] = blockIdx.x;
    info[7] = (unsigned long long)(unsigned)extra;
  }
}
__device__ __forceinline__ bool bf2_nonfinite(uint32_t v) {
  return ((v >> 7) & 0xFFu) == 0xFFu || ((v >> 23) & 0xFFu) == 0xFFu;
}
#endif
#ifdef MXM_TRACE
// per-stage event timestamps of CTA 0 (diagnostic build): [event][index], see tools/diag_trace.py
constexpr int kTrN = 2048;
__device__ unsigned long long g_tr[13][kTrN];
#define TR(ev, idx) do { if (blockIdx.x == 0 && (idx) < kTrN) g_tr[ev][idx] = clock64(); } while (0)
#else
#define TR(ev, idx) do { } while (0)
#endif
#ifdef MXM_TRACE_TASKS
// per-task timeline of CTA 0 and per-CTA start / end / counts (diagnostic build): tools/diag_tasks.py
constexpr int kTtN = 4096, kTtCta = 160;
__device__ unsigned long long g_tt[2][kTtN];   // [0] clock64 at task fetch, [1] phase | stages << 8 | nt << 32
__device__ unsigned long long g_cta[kTtCta][4];  // globaltimer start, end, tasks, stages
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif
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
#ifdef MXM_ABL_XF_RAW  // timing diagnostic: raw (128 + u) codes, no scale / zero (numerically wrong)
  return fields;
#endif
  return bf2_fma(bf2_sub(fields, off2), s2, z2);
}
// codes of one pair at bits (sh, sh+16) of `word`, widths given by `mask`, as (128+u) bf16x2 (one LOP3)
__device__ __forceinline__ uint32_t pair_fields(uint32_t word, int sh, uint32_t mask) {
  return and_or(word >> sh, mask, 0x43004300u);
}

// Weight-only dequant of one half-stage of one A row (thread r = TMEM lane r): the H-th 32 of the stage's
// 64 K elements -> 16 words o[] in K order (o[j] = elements 2j, 2j+1), written to the TMEM A ring with one
// tcgen05.st (two transform warpgroups split every stage by K halves).
// `hm`: this stage starts a group, so the chunk begins with scale[128] (and zero[128] if asymmetric).
template <int BITS, int H>
__device__ __forceinline__ void xform_wo(const uint8_t* __restrict__ raw, bool hm, int meta_bytes, bool sym,
                                         uint32_t off2, int r, uint32_t& s2, uint32_t& z2, uint32_t (&o)[16]) {
  const uint8_t* codes = raw;
  if (hm) {
    const uint32_t sb = reinterpret_cast<const uint16_t*>(raw)[r];
    s2 = sb | (sb << 16);
    if (!sym) {
      const uint32_t zb = reinterpret_cast<const uint16_t*>(raw + 256)[r];
      z2 = zb | (zb << 16);
    } else {
      z2 = 0;
    }
    codes += meta_bytes;
  }
  const uint32_t* w = reinterpret_cast<const uint32_t*>(codes);
  if constexpr (BITS == 4) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t word = w[(4 * H + j) * 128 + r];
#pragma unroll
      for (int t = 0; t < 4; ++t) o[4 * j + t] = deq_pair(pair_fields(word, 4 * t, 0x000F000Fu), off2, s2, z2);
    }
  } else if constexpr (BITS == 2) {
    // pair t sits at bits (2t, 2t+16). Masked in place at mantissa bit 2*tau (tau = 0, 1, 2) the bf16 field
    // reads 128 + u * 4^tau, so only the words >> 6 and >> 12 are shifted (2 SHF per 8 pairs instead of 7);
    // (128 + u 4^tau - (128 + off 4^tau)) * (s 4^-tau) + z is the same exact q*s + z, rounded once (HFMA2).
    // s 4^-tau is an exact bf16 for any normal s (power-of-two scaling).
    const uint32_t offb = off2 & 0x007F007Fu;
    const uint32_t offs[3] = {off2, 0x43004300u | (offb << 2), 0x43004300u | (offb << 4)};
    uint32_t ss[3];
    {
      __nv_bfloat162 sv = *reinterpret_cast<const __nv_bfloat162*>(&s2);
      const uint32_t q4 = 0x3E803E80u, q16 = 0x3D803D80u;  // 0.25, 0.0625
      __nv_bfloat162 a = __hmul2(sv, *reinterpret_cast<const __nv_bfloat162*>(&q4));
      __nv_bfloat162 b = __hmul2(sv, *reinterpret_cast<const __nv_bfloat162*>(&q16));
      ss[0] = s2;
      ss[1] = *reinterpret_cast<uint32_t*>(&a);
      ss[2] = *reinterpret_cast<uint32_t*>(&b);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t word = w[(2 * H + j) * 128 + r];
      const uint32_t ws[3] = {word, word >> 6, word >> 12};
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int src = t < 6 ? t / 3 : 2;
        const int tau = t < 6 ? t % 3 : t - 6;
        const uint32_t fields = and_or(ws[src], 0x00030003u << (2 * tau), 0x43004300u);
        o[8 * j + t] = deq_pair(fields, offs[tau], ss[tau], z2);
      }
    }
  } else if constexpr (BITS == 3) {
    const uint32_t hw2 = w[(4 + H) * 128 + r];  // high-bit plane word covering low-plane words 2H, 2H+1
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t word = w[(2 * H + j) * 128 + r];
      const uint32_t hw = hw2 >> (8 * j);
#pragma unroll
      for (int t = 0; t < 8; ++t)
        o[8 * j + t] = deq_pair(and_or(word >> (2 * t), 0x00030003u, (((hw >> t) & 0x00010001u) << 2) | 0x43004300u),
                                off2, s2, z2);
    }
  } else {  // 8-bit: 128 + u is not exact in bf16 for u >= 128. q s + z is exact in fp64 (q s has 16 significant
            // bits), so one rounding to bf16 gives R5's bf16_rne(q s + z); an fp32 sum would round twice
    const double sd = (double)__uint_as_float(s2 << 16), zd = (double)__uint_as_float(z2 << 16);
    const int fo = (int)(off2 & 0xFFu);
    auto deq = [&](uint32_t u) { return __double2bfloat16(fma((double)((int)u - fo), sd, zd)); };
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t word = w[(8 * H + j) * 128 + r];
      __nv_bfloat162 lo, hi;
      lo.x = deq(word & 0xFFu);
      lo.y = deq((word >> 8) & 0xFFu);
      hi.x = deq((word >> 16) & 0xFFu);
      hi.y = deq(word >> 24);
      o[2 * j] = *reinterpret_cast<uint32_t*>(&lo);
      o[2 * j + 1] = *reinterpret_cast<uint32_t*>(&hi);
    }
  }
}

template <int H>
__device__ __forceinline__ void xform_wo_any(int bits, const uint8_t* raw, bool hm, int mb, bool sym, uint32_t off2,
                                             int r, uint32_t& s2, uint32_t& z2, uint32_t (&o)[16]) {
  switch (bits) {
    case 2:
      xform_wo<2, H>(raw, hm, mb, sym, off2, r, s2, z2, o);
      break;
    case 3:
      xform_wo<3, H>(raw, hm, mb, sym, off2, r, s2, z2, o);
      break;
    case 4:
      xform_wo<4, H>(raw, hm, mb, sym, off2, r, s2, z2, o);
      break;
    default:
      xform_wo<8, H>(raw, hm, mb, sym, off2, r, s2, z2, o);
      break;
  }
}

__device__ __forceinline__ uint32_t to_s8_4(uint32_t u, uint32_t bias) { return (u + bias) ^ 0x80808080u; }

// W-A w4/w5 unpack of one half-stage of one row: 64 of the stage's 128 codes -> s8, o[j] = bytes 4j..4j+3
// w4a4 (kind::f8f6f4) unpack of one half-stage of one row: the offset-binary nibbles u = q + 8 zero-extended
// to bytes, which the MMA reads as the e4m3 values u * 2^-9 (common.cuh KIND_WA_F8): one AND per 4 codes
template <int H>
__device__ __forceinline__ void xform_f8(const uint8_t* __restrict__ raw, int r, uint32_t (&o)[16]) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(raw);
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const uint32_t word = w[(8 * H + jj) * 128 + r];
    o[2 * jj] = word & 0x0F0F0F0Fu;
    o[2 * jj + 1] = (word >> 4) & 0x0F0F0F0Fu;
  }
}

template <int BITS, int H>
__device__ __forceinline__ void xform_wa(const uint8_t* __restrict__ raw, int r, uint32_t (&o)[16]) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(raw);
  const uint32_t* wh = w + 16 * 128;
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int j = 8 * H + jj;
    const uint32_t word = w[j * 128 + r];
    if constexpr (BITS == 4) {
      o[2 * jj] = to_s8_4(word & 0x0F0F0F0Fu, 0x78787878u);
      o[2 * jj + 1] = to_s8_4((word >> 4) & 0x0F0F0F0Fu, 0x78787878u);
    } else {
      const uint32_t hb = wh[(j >> 2) * 128 + r];
      const int t0 = 2 * (j & 3);
      const uint32_t lo = (word & 0x0F0F0F0Fu) | (((hb >> t0) & 0x01010101u) << 4);
      const uint32_t hi = ((word >> 4) & 0x0F0F0F0Fu) | (((hb >> (t0 + 1)) & 0x01010101u) << 4);
      o[2 * jj] = to_s8_4(lo, 0x70707070u);
      o[2 * jj + 1] = to_s8_4(hi, 0x70707070u);
    }
  }
}

// one transform warpgroup's share (K half H) of one stage: both mats -> TMEM A ring (each mat's tcgen05.st
// is issued as soon as it is unpacked, so it overlaps the next mat's unpack)
template <int H>
__device__ __forceinline__ void xform_stage(const SubLoop& s, const uint8_t* x0, const uint8_t* x1, uint32_t tA, int r,
                                            bool hmA, bool hmB, int bitsA, int bitsB, int mbA, int mbB, bool symA,
                                            bool symB, uint32_t offA, uint32_t offB, bool xa, bool xb, uint32_t& sa,
                                            uint32_t& za, uint32_t& sb, uint32_t& zb, uint32_t (&o)[16]) {
  if (s.f8) {
    if (xa) {
      xform_f8<H>(x0, r, o);
      tmem_st16(tA + 16 * H, o);
    }
    if (xb) {
      xform_f8<H>(x1, r, o);
      tmem_st16(tA + 32 + 16 * H, o);
    }
  } else if (s.i8) {
    if (xa) {
      xform_wa<5, H>(x0, r, o);
      tmem_st16(tA + 16 * H, o);
    }
    if (xb) {
      xform_wa<5, H>(x1, r, o);
      tmem_st16(tA + 32 + 16 * H, o);
    }
  } else {
    if (xa) {
      xform_wo_any<H>(bitsA, x0, hmA, mbA, symA, offA, r, sa, za, o);
      tmem_st16(tA + 16 * H, o);
    }
    if (xb) {
      xform_wo_any<H>(bitsB, x1, hmB, mbB, symB, offB, r, sb, zb, o);
      tmem_st16(tA + 32 + 16 * H, o);
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

// broadcast the per-column value preloaded by lane (idx & 31) of register lo (idx < 32) / hi
__device__ __forceinline__ float colval(float lo, float hi, int idx) {
  return __shfl_sync(0xffffffffu, idx < 32 ? lo : hi, idx & 31);
}

// packed fp32x2 helpers (sm_100a FFMA2 / FMUL2 / FADD2)
__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(r);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}

// One drain event of the register-accumulating epilogue for HALF token columns of this warpgroup.
// acc2 holds 64 fp32 accumulators as 32 pairs: dual gate/up -> gate cols in pairs [0,16), up in [16,32);
// single -> cols in pairs [0,32). i8: acc += int32 * (s_w * s_a[col]) ; bf16-kind: acc += fp32.
// `sa` is this warp's smem copy of the event's activation scales (broadcast reads, no shuffles).
// SMALL (g128 groups: |int32| <= 128*127*127 < 2^22): exact int->float by the 2^23+2^22 magic add
// (IADD + FADD on the full-rate pipes instead of the quarter-rate I2F).
// I8 / TWO / SMALL are template parameters: with run-time flags the compiler if-converts both conversion
// paths and the mat-1 work into predicated instructions that still take issue slots
// F8 (w4a4, kind::f8f6f4): the accumulator is f32 = 2^-18 sum (q_w + 8) q_a exactly; with a = s_a 2^18 and
// b = -8 s_a sum(q_a) per token column (sa[], sa[128 + col]) the event adds s_w * (acc * a + b): two FFMA2, no I2F.
template <int HALF, int DST0, bool I8, bool TWO, bool SMALL, bool F8 = false>
__device__ __forceinline__ void drain_event(float2 (&acc2)[32], uint32_t addrA, uint32_t addrB, float sw0, float sw1,
                                            const float* sa) {
  constexpr int CH = 8;  // 16-wide staging + 64 accumulators exceeds the 128-register epilogue budget (spills)
  constexpr int NCH = HALF / CH;
  constexpr float kMagic = 12582912.f;  // 2^23 + 2^22
#ifdef MXM_F8_MATWISE
  if constexpr (I8 && F8 && HALF == 32) {
    // mat by mat: all 32 columns of a mat in one TMEM load (one round trip per mat), factors as broadcast float4s
#pragma unroll
    for (int m = 0; m < (TWO ? 2 : 1); ++m) {
      uint32_t xv[32];
      tmem_ld32(m == 0 ? addrA : addrB, xv);
      const float2 swm = m == 0 ? make_float2(sw0, sw0) : make_float2(sw1, sw1);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 a4 = *reinterpret_cast<const float4*>(sa + 4 * q);
        const float4 b4 = *reinterpret_cast<const float4*>(sa + 128 + 4 * q);
        const int dst = (m == 0 ? DST0 : 16) + 2 * q;
        acc2[dst] = ffma2(ffma2(make_float2(__uint_as_float(xv[4 * q]), __uint_as_float(xv[4 * q + 1])),
                                make_float2(a4.x, a4.y), make_float2(b4.x, b4.y)), swm, acc2[dst]);
        acc2[dst + 1] = ffma2(ffma2(make_float2(__uint_as_float(xv[4 * q + 2]), __uint_as_float(xv[4 * q + 3])),
                                    make_float2(a4.z, a4.w), make_float2(b4.z, b4.w)), swm, acc2[dst + 1]);
      }
    }
    return;
  }
#endif
#ifdef MXM_F8_2CH
  if constexpr (I8 && F8 && HALF % 16 == 0) {
    // two 8-column chunks per round trip: both chunks' TMEM loads (both mats) issued together
#pragma unroll
    for (int c = 0; c < HALF / 16; ++c) {
      const int c0 = c * 16;
      uint32_t xa[2][8], xb[2][8];
#pragma unroll
      for (int j = 0; j < 8; ++j) xb[0][j] = xb[1][j] = 0u;
      tmem_ld8(addrA + c0, xa[0]);
      tmem_ld8(addrA + c0 + 8, xa[1]);
      if constexpr (TWO) {
        tmem_ld8(addrB + c0, xb[0]);
        tmem_ld8(addrB + c0 + 8, xb[1]);
      }
      tmem_ld_wait();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const float4 a4 = *reinterpret_cast<const float4*>(sa + c0 + 8 * h + 4 * q);
          const float4 b4 = *reinterpret_cast<const float4*>(sa + 128 + c0 + 8 * h + 4 * q);
          const int dst = (c0 + 8 * h + 4 * q) / 2;
          const float2 a01 = make_float2(a4.x, a4.y), a23 = make_float2(a4.z, a4.w);
          const float2 b01 = make_float2(b4.x, b4.y), b23 = make_float2(b4.z, b4.w);
          acc2[DST0 + dst] = ffma2(ffma2(make_float2(__uint_as_float(xa[h][4 * q]), __uint_as_float(xa[h][4 * q + 1])),
                                         a01, b01), make_float2(sw0, sw0), acc2[DST0 + dst]);
          acc2[DST0 + dst + 1] = ffma2(ffma2(make_float2(__uint_as_float(xa[h][4 * q + 2]),
                                                         __uint_as_float(xa[h][4 * q + 3])), a23, b23),
                                       make_float2(sw0, sw0), acc2[DST0 + dst + 1]);
          if constexpr (TWO) {
            acc2[16 + dst] = ffma2(ffma2(make_float2(__uint_as_float(xb[h][4 * q]), __uint_as_float(xb[h][4 * q + 1])),
                                         a01, b01), make_float2(sw1, sw1), acc2[16 + dst]);
            acc2[16 + dst + 1] = ffma2(ffma2(make_float2(__uint_as_float(xb[h][4 * q + 2]),
                                                         __uint_as_float(xb[h][4 * q + 3])), a23, b23),
                                       make_float2(sw1, sw1), acc2[16 + dst + 1]);
          }
        }
      }
    }
    return;
  }
#endif
  if constexpr (I8 && F8) {
    // per chunk of FCH columns: both mats' TMEM loads and the chunk's factors (a, b: broadcast float4s) in
    // flight together, one wait, then 2 FFMA2 per element pair (no cross-chunk software pipelining: at 128
    // registers ptxas serialises it anyway, and one round trip per chunk is what that costs)
#ifndef MXM_F8_CH
#define MXM_F8_CH 8
#endif
    constexpr int FCH = (HALF % MXM_F8_CH == 0) ? MXM_F8_CH : 8;
#pragma unroll
    for (int c = 0; c < HALF / FCH; ++c) {
      const int c0 = c * FCH;
      uint32_t xa[FCH], xb[FCH];
#pragma unroll
      for (int j = 0; j < FCH; ++j) xb[j] = 0u;
      if constexpr (FCH == 16) {
        tmem_ld16(addrA + c0, xa);
        if constexpr (TWO) tmem_ld16(addrB + c0, xb);
      } else {
        tmem_ld8(addrA + c0, *reinterpret_cast<uint32_t(*)[8]>(xa));
        if constexpr (TWO) tmem_ld8(addrB + c0, *reinterpret_cast<uint32_t(*)[8]>(xb));
      }
      float2 ac[FCH / 2], bc[FCH / 2];
#pragma unroll
      for (int q = 0; q < FCH / 4; ++q) {
        const float4 a4 = *reinterpret_cast<const float4*>(sa + c0 + 4 * q);
        const float4 b4 = *reinterpret_cast<const float4*>(sa + 128 + c0 + 4 * q);
        ac[2 * q] = make_float2(a4.x, a4.y);
        ac[2 * q + 1] = make_float2(a4.z, a4.w);
        bc[2 * q] = make_float2(b4.x, b4.y);
        bc[2 * q + 1] = make_float2(b4.z, b4.w);
      }
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < FCH; j += 2) {
        const int col = c0 + j;
        const float2 fa = make_float2(__uint_as_float(xa[j]), __uint_as_float(xa[j + 1]));
#ifdef MXM_ABL_DRAIN_1FMA  // timing diagnostic: one FFMA2 per element pair (numerically wrong)
        acc2[DST0 + col / 2] = ffma2(fa, ac[j / 2], acc2[DST0 + col / 2]);
        if constexpr (TWO)
          acc2[16 + col / 2] = ffma2(make_float2(__uint_as_float(xb[j]), __uint_as_float(xb[j + 1])), ac[j / 2],
                                     acc2[16 + col / 2]);
        continue;
#endif
        acc2[DST0 + col / 2] = ffma2(ffma2(fa, ac[j / 2], bc[j / 2]), make_float2(sw0, sw0), acc2[DST0 + col / 2]);
        if constexpr (TWO) {
          const float2 fb = make_float2(__uint_as_float(xb[j]), __uint_as_float(xb[j + 1]));
          acc2[16 + col / 2] = ffma2(ffma2(fb, ac[j / 2], bc[j / 2]), make_float2(sw1, sw1), acc2[16 + col / 2]);
        }
      }
    }
    return;
  }
  // software-pipelined: chunk c+1's TMEM loads are in flight while chunk c is scaled and accumulated
  uint32_t va[2][CH], vb[2][CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) vb[0][j] = vb[1][j] = 0u;
#ifdef MXM_ABL_DRAIN_LD  // diagnostic: no TMEM loads (operands = lane-dependent constants)
#define tmem_ld8(a, r) do { for (int _j = 0; _j < 8; ++_j) (r)[_j] = (a) + _j; } while (0)
#define tmem_ld_wait_regs(a, b) do { } while (0)
#endif
  tmem_ld8(addrA, va[0]);
  if constexpr (TWO) tmem_ld8(addrB, vb[0]);
  tmem_ld_wait_regs(va[0], vb[0]);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int cur = c & 1;
    if (c + 1 < NCH) {
      tmem_ld8(addrA + (c + 1) * CH, va[cur ^ 1]);
      if constexpr (TWO) tmem_ld8(addrB + (c + 1) * CH, vb[cur ^ 1]);
    }
    const int c0 = c * CH;
#ifdef MXM_ABL_DRAIN_MATH  // diagnostic: loads only, one integer add per element
    if (true) {
#pragma unroll
      for (int j = 0; j < CH; j += 2) {
        const int col = c0 + j;
        acc2[DST0 + col / 2].x = __int_as_float(__float_as_int(acc2[DST0 + col / 2].x) + (int)(va[cur][j] + vb[cur][j]));
      }
    } else
#endif
    if constexpr (I8) {
#pragma unroll
      for (int j = 0; j < CH; j += 2) {
        const int col = c0 + j;
        const float4 sa4 = *reinterpret_cast<const float4*>(sa + (col & ~3));  // 16-B aligned, broadcast
        const float2 sac = (col & 2) ? make_float2(sa4.z, sa4.w) : make_float2(sa4.x, sa4.y);
        float2 fa, fb;
#ifndef MXM_MAGIC_I2F
#define MXM_MAGIC_I2F 0  // 1: every conversion by the 2^23+2^22 add (A/B alternative)
#endif
#ifndef MXM_SPLIT_I2F
#define MXM_SPLIT_I2F 0  // 1: mat 1 converts with the magic add (measured slower: the FMA pipe is the drain limit)
#endif
        // I2FP.F32.S32 issues at 1/4 rate (32 lanes/clk/SM, tools/op_rate.cu) on its own pipe, the magic add
        // costs an IADD + FADD2 on the FMA pipe that FMUL2 / FFMA2 already load: mat 0 converts with I2FP,
        // mat 1 with the magic add, so both pipes share the drain (exact: |acc| < 2^22 for a 128-K group)
        if constexpr (MXM_SPLIT_I2F && !MXM_MAGIC_I2F && SMALL && TWO) {
          fa = make_float2((float)(int32_t)va[cur][j], (float)(int32_t)va[cur][j + 1]);
          fb = fadd2(make_float2(__int_as_float((int32_t)vb[cur][j] + 0x4B400000),
                                 __int_as_float((int32_t)vb[cur][j + 1] + 0x4B400000)),
                     make_float2(-kMagic, -kMagic));
        } else if constexpr (MXM_MAGIC_I2F && SMALL) {
          fa = fadd2(make_float2(__int_as_float((int32_t)va[cur][j] + 0x4B400000),
                                 __int_as_float((int32_t)va[cur][j + 1] + 0x4B400000)),
                     make_float2(-kMagic, -kMagic));
          fb = fadd2(make_float2(__int_as_float((int32_t)vb[cur][j] + 0x4B400000),
                                 __int_as_float((int32_t)vb[cur][j + 1] + 0x4B400000)),
                     make_float2(-kMagic, -kMagic));
        } else {
          fa = make_float2((float)(int32_t)va[cur][j], (float)(int32_t)va[cur][j + 1]);
          fb = make_float2((float)(int32_t)vb[cur][j], (float)(int32_t)vb[cur][j + 1]);
        }
        acc2[DST0 + col / 2] = ffma2(fa, fmul2(make_float2(sw0, sw0), sac), acc2[DST0 + col / 2]);
        if constexpr (TWO) acc2[16 + col / 2] = ffma2(fb, fmul2(make_float2(sw1, sw1), sac), acc2[16 + col / 2]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < CH; j += 2) {
        const int col = c0 + j;
        acc2[DST0 + col / 2] =
            fadd2(acc2[DST0 + col / 2], make_float2(__uint_as_float(va[cur][j]), __uint_as_float(va[cur][j + 1])));
        if constexpr (TWO)
          acc2[16 + col / 2] =
              fadd2(acc2[16 + col / 2], make_float2(__uint_as_float(vb[cur][j]), __uint_as_float(vb[cur][j + 1])));
      }
    }
    if (c + 1 < NCH) tmem_ld_wait_regs(va[cur ^ 1], vb[cur ^ 1]);
  }
#ifdef MXM_ABL_DRAIN_LD
#undef tmem_ld8
#undef tmem_ld_wait_regs
#endif
}

template <int DST0, bool I8, bool TWO, bool SMALL, bool F8>
__device__ __forceinline__ void drain_half(int half, float2 (&acc2)[32], uint32_t addrA, uint32_t addrB, float sw0,
                                           float sw1, const float* sa) {
  // two mats: tiles of <= 64 tokens (half <= 32). One mat: also a g128 W-A down of an expert whose gate/up
  // allow 96-token tiles (single-mat down, half 48); half 64 keeps the 128-token case total
  if (half == 8) {
    drain_event<8, DST0, I8, TWO, SMALL, F8>(acc2, addrA, addrB, sw0, sw1, sa);
  } else if (half == 16) {
    drain_event<16, DST0, I8, TWO, SMALL, F8>(acc2, addrA, addrB, sw0, sw1, sa);
  } else if (half == 32 || TWO || DST0 != 0) {
    drain_event<32, DST0, I8, TWO, SMALL, F8>(acc2, addrA, addrB, sw0, sw1, sa);
  } else if constexpr (!TWO && DST0 == 0) {
    if (half == 40)
      drain_event<40, 0, I8, false, SMALL, F8>(acc2, addrA, addrB, sw0, sw1, sa);
    else if (half == 48)
      drain_event<48, 0, I8, false, SMALL, F8>(acc2, addrA, addrB, sw0, sw1, sa);
    else
      drain_event<64, 0, I8, false, SMALL, F8>(acc2, addrA, addrB, sw0, sw1, sa);
  }
}

// i8 && small: W-A g128 events (dual or single mat); i8 && !small / bf16: one mat of a heterogeneous
// gate/up pair (never two mats). f8: w4a4 (kind::f8f6f4 accumulators, drain_event F8)
template <int DST0>
__device__ __forceinline__ void drain_event_any(int half, float2 (&acc2)[32], uint32_t addrA, uint32_t addrB, bool i8,
                                                bool f8, bool two, bool small, float sw0, float sw1, const float* sa) {
  if (f8) {
    if (two) {
      if constexpr (DST0 == 0) drain_half<0, true, true, true, true>(half, acc2, addrA, addrB, sw0, sw1, sa);
    } else {
      drain_half<DST0, true, false, true, true>(half, acc2, addrA, addrB, sw0, sw1, sa);
    }
  } else if (i8 && small) {
    if (two) {
      if constexpr (DST0 == 0) drain_half<0, true, true, true, false>(half, acc2, addrA, addrB, sw0, sw1, sa);
    } else {
      drain_half<DST0, true, false, true, false>(half, acc2, addrA, addrB, sw0, sw1, sa);
    }
  } else if (i8) {
    drain_half<DST0, true, false, false, false>(half, acc2, addrA, addrB, sw0, sw1, sa);
  } else {
    drain_half<DST0, false, false, false, false>(half, acc2, addrA, addrB, sw0, sw1, sa);
  }
}

// H / Hq row layout (api.cu make_layout): shared-expert rows [0, h_srows) at stride f_s, then the routed rows
// at stride f_r, so the workspace holds sum over rows of that row's expert width instead of R x max(f, f_s)
__device__ __forceinline__ int64_t h_off(const GemmParams& p, int64_t row) {
  return row < p.h_srows ? row * p.f_s : p.h_rbase + (row - p.h_srows) * p.f_r;
}
__device__ __forceinline__ int64_t h_ld(const GemmParams& p, int64_t row) { return row < p.h_srows ? p.f_s : p.f_r; }

// h for 8 token columns [colc, colc+8) of output channel n (= this thread's TMEM lane), already rounded to
// bf16 (hb, DESIGN R16), in the form the down block consumes (dmode): 0 bf16 H; 1 bf16 H + row max|h| via
// atomicMax (per-token W-A down, quantized later in one pass); 2 fused per-128-group quantization: the group
// is exactly this tile's 128 channels, so codes + scale are produced here (DESIGN R9).
// nv = valid columns from colc (rows of the m-tile), hrow = &H[row0 + colc][n] (h_off / h_ld: the row's region).
template <bool DUMP = false>
__device__ __forceinline__ void emit_h8(const GemmParams& p, const Task& t, int dmode, int qmax, int n, int colc, int nv,
                                     const uint16_t (&hb)[8], Ctl& ctl, int wg, int q, int lane, uint32_t& rbuf) {
  const int64_t row0 = (int64_t)t.row0 + colc;
  if (dmode >= 2) {  // 2: int8 codes (w5a5 / w8a8 g128 down), 3: e4m3 codes + group code sums (w4a4 g128 down),
                     // 4: FP8 e4m3 codes (FP8 g128 down)
    if constexpr (DUMP) {  // test build: also keep the bf16 h the fused quantizer consumed (bit-exact h-quant test)
      uint16_t* hrow = p.H + h_off(p, row0) + n;
      const int64_t ld = h_ld(p, row0);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < nv) hrow[(int64_t)j * ld] = hb[j];
    }
    uint32_t m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = __reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(bf16f(hb[j]))));
    if (lane == 0)
#pragma unroll
      for (int j = 0; j < 8; ++j) ctl.colmax[rbuf][wg][q][j] = m[j];
    named_bar_sync(2 + wg, 128);
    // lanes 0..7 derive column (lane)'s reciprocal / scale once (IEEE division, DESIGN R9), then broadcast
    const float fq = dmode == 4 ? 448.f : (float)qmax;  // 4: FP8 e4m3 codes (R26)
    float r_l = 0.f, sc_l = 1.f;
    if (lane < 8) {
      const uint32_t a = max(max(ctl.colmax[rbuf][wg][0][lane], ctl.colmax[rbuf][wg][1][lane]),
                             max(ctl.colmax[rbuf][wg][2][lane], ctl.colmax[rbuf][wg][3][lane]));
      const float amax = __uint_as_float(a);
      if (amax > 0.f) {
        r_l = __fdiv_rn(fq, amax);
        sc_l = __fdiv_rn(amax, fq);
      }
      if (q == 0 && lane < nv) p.Hs[row0 + lane + (int64_t)t.ntile * p.hs_stride] = sc_l;
    }
    int8_t* hq = p.Hq + h_off(p, row0) + n;
    const int64_t hld = h_ld(p, row0);
    int qi[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float r = __shfl_sync(0xffffffffu, r_l, j);
      if (dmode == 4) {
        qi[j] = 0;
        if (j < nv) hq[(int64_t)j * hld] = (int8_t)fp8_act_code(bf16f(hb[j]), r);
        continue;
      }
      qi[j] = (int)fminf(fmaxf(rintf(__fmul_rn(bf16f(hb[j]), r)), -fq), fq);
      if (j < nv) hq[(int64_t)j * hld] = (int8_t)(dmode == 3 ? code_byte<true>(qi[j]) : code_byte<false>(qi[j]));
    }
    if (dmode == 3) {  // sum of the group's codes per token column: warp sums, then the 4 warps of the warpgroup
      int cs[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) cs[j] = __reduce_add_sync(0xffffffffu, qi[j]);
      if (lane == 0)
#pragma unroll
        for (int j = 0; j < 8; ++j) ctl.colsum[rbuf][wg][q][j] = cs[j];
      named_bar_sync(2 + wg, 128);  // (double-buffered by rbuf: the next write of this buffer is 2 barriers away)
      if (q == 0 && lane < 8 && lane < nv)
        p.Hc[row0 + lane + (int64_t)t.ntile * p.hs_stride] = ctl.colsum[rbuf][wg][0][lane] +
                                                              ctl.colsum[rbuf][wg][1][lane] +
                                                              ctl.colsum[rbuf][wg][2][lane] +
                                                              ctl.colsum[rbuf][wg][3][lane];
    }
    rbuf ^= 1;
    return;
  }
  uint16_t* hrow = p.H + h_off(p, row0) + n;
  const int64_t ld = h_ld(p, row0);
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (j < nv) hrow[(int64_t)j * ld] = hb[j];
  if (dmode == 1) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t m = __reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(bf16f(hb[j]))));
      if (lane == 0 && j < nv) atomicMax(p.hmax + row0 + j, m);
    }
  }
}

// Test build only (mxm_debug_moe_group_gemm_dump): copy the raw 32-bit accumulators of one drain event -- this
// warpgroup's `half` token columns starting at TMEM column addrA (mat 0) / addrB (mat 1) -- to p.dump, before
// the drain consumes them: gate / up (j = 0, 1) at ((j * d/128 + g) * R + row) * f_max + n, down (j = 2) at
// 2 * (d/128) * R * f_max + (g * R + row) * d + n.
__device__ __forceinline__ int64_t dump_index(const GemmParams& p, int j, int g, int64_t row, int n) {
  const int64_t R = p.hs_stride;
  const int64_t gu = (int64_t)(p.d / 128) * R * p.f_max;
  return j < 2 ? (((int64_t)j * (p.d / 128) + g) * R + row) * p.f_max + n : 2 * gu + ((int64_t)g * R + row) * p.d + n;
}
__device__ __forceinline__ void dump_event(const GemmParams& p, uint32_t addrA, uint32_t addrB, bool two, int jA,
                                           int jB, int g, int nA, int nB, int64_t row0, int half, int nvalid) {
  for (int c = 0; c < half; c += 8) {
    uint32_t va[8], vb[8];
    tmem_ld8(addrA + c, va);
    if (two) tmem_ld8(addrB + c, vb);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (c + j < nvalid) {
        const int64_t row = row0 + c + j;
        p.dump[dump_index(p, jA, g, row, nA)] = va[j];
        if (two) p.dump[dump_index(p, jB, g, row, nB)] = vb[j];
      }
    }
  }
}

// wait with optional cycle accounting (debug profiling of the stage pipeline)
__device__ __forceinline__ void twait(uint64_t* bar, uint32_t parity, unsigned long long& acc, bool on) {
  if (!on) {
    mbar_wait(bar, parity);
    return;
  }
  const unsigned long long t0 = clock64();
  mbar_wait(bar, parity);
  acc += clock64() - t0;
}

struct MmaState {
  uint32_t stage, sphase, abuf, acc_ph, aidx;  // aidx: TS stages so far (A slot = aidx % kASlots)
  int nev;                                      // drain events committed (trace index, diagnostic build)
  int ntr;                                      // stages issued (trace index, diagnostic build)
};

// One sub-loop of MMAs (all K stages of one or two mats sharing the token tile), specialised on the MMA
// kind and the number of mats so the issue loop has no runtime kind branches.
__device__ __forceinline__ uint32_t bcast(uint32_t v) { return __shfl_sync(0xffffffffu, v, 0); }

// One sub-loop of MMAs (all K stages of one or two mats sharing the token tile), specialised on the MMA
// kind, the number of mats and the A-operand source (MODE 0: both A images in smem (SS); 1: all A in the
// TMEM ring (TS); 2: per-mat at run time). Executed by the whole MMA warp with warp-uniform operands
// (broadcast from lane 0) and the tcgen05 instructions inside one elect.sync block per stage: this keeps the
// operands in uniform registers (no per-lane "waterfall" loop around each MMA). The issue queue is shallow,
// so every instruction between two stages' MMAs is a tensor-core bubble: the smem descriptors are built once
// per sub-loop and advanced by one add per MMA (start address field += 32 B >> 4 per K step).
// MK: MMA kind 0 = kind::f16 (bf16), 1 = kind::i8 (s8 x s8), 2 = kind::f8f6f4 (e4m3 x e4m3, w4a4)
template <int MK, bool TWO, int MODE>
__device__ __forceinline__ void mma_subloop(Ctl& ctl, uint8_t* smem, uint32_t tmem, uint32_t ns, uint32_t g128,
                                            uint32_t xform, uint32_t nt, MmaState& st, unsigned long long (&pc)[16],
                                            bool prof_on) {
  const uint32_t idesc = MK == 1 ? idesc_s8(nt) : (MK == 2 ? idesc_f8(nt) : idesc_bf16(nt));
  // descriptor words: lo = start>>4 | LBO 1 << 16 ; hi = SBO 1024>>4 | version 1 << 14 | SWIZZLE_128B 2 << 29
  const uint32_t lo0 = ((smem_u32(smem) >> 4) & 0x3FFFu) | (1u << 16);
  constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);
  constexpr uint32_t kSlotLo = kSlotBytes >> 4, kTileLo = kTileBytes >> 4;
  const bool ts0 = MODE == 1 || (MODE == 2 && (xform & 1) != 0);
  const bool ts1 = MODE == 1 || (MODE == 2 && (xform & 2) != 0);
  const bool any_ts = MODE == 1 || (MODE == 2 && xform != 0);
  auto desc = [](uint32_t lo) { return ((uint64_t)kHi << 32) | lo; };
  uint32_t b0 = 0;
  for (uint32_t ks = 0; ks < ns; ++ks) {
    const bool ev_start = g128 || ks == 0, ev_end = g128 || ks == ns - 1;
    if (ev_start) {
      b0 = st.abuf;
      if ((threadIdx.x & 31) == 0) TR(10, st.nev);
      twait(&ctl.acce[b0], ((st.acc_ph >> b0) & 1) ^ 1, pc[4], prof_on);
      if ((threadIdx.x & 31) == 0) TR(11, st.nev);
      st.acc_ph ^= 1u << b0;
      st.abuf = st.abuf + 1 == kAccBufs ? 0 : st.abuf + 1;
    }
    const uint32_t stage = st.stage;
    const uint32_t d0 = tmem + b0 * (uint32_t)kAccCols;
    const uint32_t d1 = d0 + (uint32_t)kMat1Col;
    const uint32_t blo = lo0 + stage * kSlotLo;
    const uint32_t aslot = st.aidx % kASlots;
    const uint32_t at0 = tmem + kTmemA + aslot * 64u;
    // one wait per stage: a TS stage's A slot is ready only after the transform saw the stage's data
    if (any_ts) {
      twait(&ctl.aready[aslot], (st.aidx / kASlots) & 1, pc[6], prof_on);
    } else {
      twait(&ctl.full[stage], st.sphase, pc[5], prof_on);
    }
#if defined(MXM_PROF_SUBLOOP) && defined(MXM_DEBUG_COUNTERS)
    const unsigned long long t_f = prof_on ? clock64() : 0ull;
    tc_fence_after();
    if (prof_on) pc[14] += clock64() - t_f;
#else
    tc_fence_after();
#endif
    const unsigned long long t_iss = prof_on ? clock64() : 0ull;
    if ((threadIdx.x & 31) == 0) TR(3, st.ntr);
    if (elect_one()) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t acc = (k == 0 && ev_start) ? 0u : 1u;
        const uint64_t bd = desc(blo + 2 * k);
        if constexpr (MK == 2) {
          if (ts0) mma_f8_ts(d0, at0 + k * 8, bd, idesc, acc); else mma_f8(d0, desc(blo + kTileLo + 2 * k), bd, idesc, acc);
          if constexpr (TWO) {
            if (ts1) mma_f8_ts(d1, at0 + 32 + k * 8, bd, idesc, acc);
            else mma_f8(d1, desc(blo + 2 * kTileLo + 2 * k), bd, idesc, acc);
          }
        } else if constexpr (MK == 1) {
          if (ts0) mma_i8_ts(d0, at0 + k * 8, bd, idesc, acc); else mma_i8(d0, desc(blo + kTileLo + 2 * k), bd, idesc, acc);
          if constexpr (TWO) {
            if (ts1) mma_i8_ts(d1, at0 + 32 + k * 8, bd, idesc, acc);
            else mma_i8(d1, desc(blo + 2 * kTileLo + 2 * k), bd, idesc, acc);
          }
        } else {
          if (ts0) mma_bf16_ts(d0, at0 + k * 8, bd, idesc, acc);
          else mma_bf16(d0, desc(blo + kTileLo + 2 * k), bd, idesc, acc);
          if constexpr (TWO) {
            if (ts1) mma_bf16_ts(d1, at0 + 32 + k * 8, bd, idesc, acc);
            else mma_bf16(d1, desc(blo + 2 * kTileLo + 2 * k), bd, idesc, acc);
          }
        }
      }
      // TS stage: the transform warps finished reading the smem stage before aready, so the MMA thread
      // arrives for them on the stage's empty barrier (they arrive themselves only on weight-image stages)
      if (any_ts) mbar_arrive_cnt(&ctl.empty[stage], kXfWarps);
      mma_commit(&ctl.empty[stage]);
      if (any_ts) mma_commit(&ctl.aempty[aslot]);
      if (ev_end) mma_commit(&ctl.accf[b0]);
    }
    if (ev_end) {
      if ((threadIdx.x & 31) == 0) TR(12, st.nev);  // (trace build: event-indexed commit time)
      ++st.nev;
    }
    __syncwarp();
    if (prof_on) {
      pc[11] += clock64() - t_iss;
      pc[13] += 1;
    }
    if ((threadIdx.x & 31) == 0) TR(4, st.ntr);
    ++st.ntr;
    if (any_ts) ++st.aidx;
    if (++st.stage == kStages) {
      st.stage = 0;
      st.sphase ^= 1;
    }
  }
}

template <int MK, bool TWO>
__device__ __forceinline__ void mma_subloop_mode(Ctl& ctl, uint8_t* smem, uint32_t tmem, uint32_t ns, uint32_t g128,
                                                 uint32_t xform, uint32_t nt, MmaState& st,
                                                 unsigned long long (&pc)[16], bool prof_on) {
  const uint32_t all = TWO ? 3u : 1u;
  if (xform == 0)
    mma_subloop<MK, TWO, 0>(ctl, smem, tmem, ns, g128, xform, nt, st, pc, prof_on);
  else if ((xform & all) == all)
    mma_subloop<MK, TWO, 1>(ctl, smem, tmem, ns, g128, xform, nt, st, pc, prof_on);
  else
    mma_subloop<MK, TWO, 2>(ctl, smem, tmem, ns, g128, xform, nt, st, pc, prof_on);
}

// ---------------------------------------------------------------- the kernel
// SPLIT: the launch may cut downs into K-slices (tiny T, workspace has the partial buffer). A separate
// instantiation, so the split-K bookkeeping costs the large-T kernel no registers.
// The per-stage copies of one task's sub-loops, split over two warps because each cp.async.bulk / TMA issue
// occupies its warp for ~100-190 cycles (tools/copy_issue.cu): ROLE 0 (producer, warp 0): the stage's
// expect_tx and mat 0's packed chunk (+ its copied group meta); ROLE 1 (warp 2): the dependency wait of
// phase-2 tasks, mat 1's chunk and the token tile (TMA). Both walk the same stage / parity sequence and wait
// for the same `empty` phase; a copy may land before the expect_tx (the transaction count may go negative).
#ifndef MXM_HELPER_SLEEP
#define MXM_HELPER_SLEEP 0
#endif
template <int ROLE, bool SPLIT>
__device__ __forceinline__ void copy_task(const GemmParams& p, const Task& t, Ctl& ctl, uint8_t* smem,
                                          uint32_t& stage, uint32_t& sphase, int n_split,
                                          unsigned long long (&pc)[16], bool prof_on, int& n_tr_p) {
  if (ROLE == 1 && t.phase == 2) {
    const ExpertDesc& e = p.ex[t.expert];
    // per-token W-A downs wait for the h-quant pass; all others only for the gate/up tiles
    const bool wa_pt = kind_is_wa(e.blk[2].geo.kind) && e.blk[2].geo.group != 128;
    const int* ctr = (wa_pt ? p.hq_done : p.p1_done) + t.gid;
    const int need = wa_pt ? p.grp_nq[t.gid] : p.grp_n1[t.gid];
    const unsigned long long td = prof_on ? clock64() : 0ull;
    while (ld_acquire_gpu(ctr) < need) __nanosleep(64);
    if (prof_on) pc[2] += clock64() - td;
    fence_proxy_async_global();
  }
  SubLoop sl[2];
  const int nsl = build_subloops(t, p.ex, p.d, n_split, sl);
  const int nti = nt_index(t.nt);
  for (int si = 0; si < nsl; ++si) {
    const SubLoop s = sl[si];
    // h inputs of a down (maps 3, 4): shared rows use the shared-region maps (5, 6), routed rows their own
    // region's maps with region-relative row coordinates
    int bm = s.bmap, trow = t.row0;
    if (bm >= 3) {
      if (t.row0 < p.h_srows)
        bm += 2;
      else
        trow = (int)(t.row0 - p.h_srows);
    }
    const CUtensorMap* map = &p.tmap[bm][nti];
    // per-mat chunk streams (gate and up may differ in bits / group / format)
    const PackGeom& g0 = s.mat[0]->geo;
    const PackGeom& g1 = s.mat[s.nmats - 1]->geo;
    const uint32_t cb0 = (uint32_t)g0.code_bytes, mb0 = (uint32_t)g0.meta_bytes;
    const uint32_t cb1 = (uint32_t)g1.code_bytes, mb1 = (uint32_t)g1.meta_bytes;
    const int gst0 = g0.group / g0.ks, gst1 = g1.group / g1.ks;
    const int ksb = SPLIT ? s.ks0 : 0, kse = SPLIT ? s.ks1 : s.ns;
    const uint8_t* src0 = s.mat[0]->packed + (SPLIT ? chunk_offset(g0, s.tile[0], ksb) : (int64_t)s.tile[0] * g0.rb_bytes);
    const uint8_t* src1 = s.nmats == 2 ? s.mat[1]->packed + (SPLIT ? chunk_offset(g1, s.tile[1], ksb)
                                                                      : (int64_t)s.tile[1] * g1.rb_bytes)
                                       : nullptr;
    const int kstep = s.i8 ? 128 : 64;
    int gc0 = SPLIT ? ksb % gst0 : 0, gc1 = SPLIT ? ksb % gst1 : 0;
    // a split-K slice that starts inside a weight-only group: its first stage is laid out as a group
    // start, [group meta (copied from the group-start chunk) | codes], so the transform needs no case
    const uint8_t* gm0 = (SPLIT && gc0 != 0 && g0.kind == KIND_WO)
                             ? s.mat[0]->packed + chunk_offset(g0, s.tile[0], ksb - gc0) : nullptr;
    const uint8_t* gm1 = (SPLIT && src1 && gc1 != 0 && g1.kind == KIND_WO)
                             ? s.mat[1]->packed + chunk_offset(g1, s.tile[1], ksb - gc1) : nullptr;
    for (int ks = ksb; ks < kse; ++ks) {
      const uint32_t c0 = cb0 + (gc0 == 0 ? mb0 : 0u);
      const uint32_t c1 = src1 ? cb1 + (gc1 == 0 ? mb1 : 0u) : 0u;
      const uint32_t e0 = SPLIT && gm0 ? mb0 : 0u, e1 = SPLIT && gm1 ? mb1 : 0u;
      if (++gc0 == gst0) gc0 = 0;
      if (++gc1 == gst1) gc1 = 0;
      if (ROLE == 1) {  // off the transform warps' issue slots: poll with a short sleep (4 stages of slack)
        while (!mbar_try_wait(&ctl.empty[stage], sphase ^ 1))
          if (MXM_HELPER_SLEEP) __nanosleep(MXM_HELPER_SLEEP);
      } else {
        twait(&ctl.empty[stage], sphase ^ 1, pc[1], prof_on);
      }
      uint8_t* slot = smem + stage * kSlotBytes;
#ifndef MXM_COPY_SPLIT
#define MXM_COPY_SPLIT 2  // 1: warp 2 issues mat 1 + token tile; 2 (measured best): warp 2 issues only the token tile
#endif
      const bool mat1_here = (ROLE == 0) == (MXM_COPY_SPLIT == 2);
      if (ROLE == 0) {
        TR(0, n_tr_p);
        mbar_arrive_expect_tx(&ctl.full[stage], (uint32_t)t.nt * 128u + c0 + c1 + e0 + e1);
        if (e0) bulk_load(slot + kTileBytes, gm0, e0, &ctl.full[stage]);
        bulk_load(slot + kTileBytes + e0, src0, c0, &ctl.full[stage]);
        ++n_tr_p;
      }
      if (src1 && mat1_here) {
        if (e1) bulk_load(slot + 2 * kTileBytes, gm1, e1, &ctl.full[stage]);
        bulk_load(slot + 2 * kTileBytes + e1, src1, c1, &ctl.full[stage]);
      }
      if (ROLE == 1) tma_load_2d(slot, map, &ctl.full[stage], ks * kstep, trow);
      src0 += c0;
      gm0 = nullptr;
      if (src1) {
        src1 += c1;
        gm1 = nullptr;
      }
      if (++stage == kStages) {
        stage = 0;
        sphase ^= 1;
      }
    }
  }
}

// Scale staging for one weight-activation g128 sub-loop (warp 3): per 128-K group, once the epilogue released the
// scale slot (sempty), the drain factors of the group -- per channel s_w of each mat, per token column
// a = s_a (s_a 2^18 for w4a4) and b = -8 s_a sum(q_a) -- read straight from global memory (no bulk copies on the
// producer's path) and written 16-B aligned into the slot, then sready.
__device__ __forceinline__ void stage_scales(const GemmParams& p, const Task& t, const SubLoop& s, Ctl& ctl,
                                             uint8_t* smem, uint32_t& xsidx, int lane, unsigned long long (&pc)[16],
                                             bool prof_on) {
  const float* xs_t = (t.phase == 0) ? p.xs[s.mat[0]->in_slot] : p.Hs;
  const int32_t* xc_t = (t.phase == 0) ? p.xc[s.mat[0]->in_slot] : p.Hc;
  const uint16_t* w0 = reinterpret_cast<const uint16_t*>(s.mat[0]->packed + s.mat[0]->geo.wa_scale_off) +
                       s.tile[0] * 128;
  const uint16_t* w1 = s.nmats == 2 ? reinterpret_cast<const uint16_t*>(s.mat[1]->packed + s.mat[1]->geo.wa_scale_off) +
                                          s.tile[1] * 128
                                    : nullptr;
  for (int ks = 0; ks < s.ns; ++ks) {
    // this group's values (loads in flight before the slot wait; loading 4 or 8 groups ahead through a register
    // ring was measured no faster / slower: profiles/r02/ab_experiments.txt)
    const uint2 sw0 = *reinterpret_cast<const uint2*>(w0 + (int64_t)ks * s.mat[0]->geo.N + 4 * lane);
    const uint2 sw1 = w1 ? *reinterpret_cast<const uint2*>(w1 + (int64_t)ks * s.mat[1]->geo.N + 4 * lane)
                         : make_uint2(0, 0);
    float sa[3] = {0.f, 0.f, 0.f};
    int qs[3] = {0, 0, 0};
#pragma unroll
    for (int h = 0; h < 3; ++h) {
      const int c = lane + 32 * h;
      if (c < t.rows) {
        sa[h] = __ldcg(xs_t + (int64_t)ks * p.hs_stride + t.row0 + c);
        if (s.w4) qs[h] = __ldcg(xc_t + (int64_t)ks * p.hs_stride + t.row0 + c);
      }
    }
    const uint32_t ss = xsidx & (kSSlots - 1);
    twait(&ctl.sempty[ss], ((xsidx / kSSlots) & 1) ^ 1, pc[8], prof_on);
    uint8_t* slotp = smem + kOffScale + ss * kSSlotBytes;
    reinterpret_cast<uint2*>(slotp)[lane] = sw0;
    reinterpret_cast<uint2*>(slotp + 256)[lane] = sw1;
#pragma unroll
    for (int h = 0; h < 3; ++h) {
      const int c = lane + 32 * h;
      if (c < (int)t.nt) {
        reinterpret_cast<float*>(slotp + kSlotA)[c] = s.w4 ? sa[h] * 262144.f : sa[h];
        reinterpret_cast<float*>(slotp + kSlotB)[c] = s.w4 ? __fmul_rn(-8.f * (float)qs[h], sa[h]) : 0.f;
      }
    }
#if MXM_LANE_ARRIVE
    mbar_arrive(&ctl.sready[ss]);  // every lane releases its own slot writes
#else
    __syncwarp();  // orders every lane's slot writes before lane 0's release
    if (lane == 0) mbar_arrive(&ctl.sready[ss]);
#endif
    ++xsidx;
  }
}

// DUMP: test-only instantiation that also copies every weight-activation accumulator to p.dump (and the bf16 h
// of fused-quantized downs to p.H) for the bit-exact accumulator tests; never launched by mxm_moe_group_gemm.
template <bool SPLIT, bool DUMP>
__global__ void __launch_bounds__(kThreads, 1) moe_gemm_kernel(const __grid_constant__ GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  // keep the pointer in the shared window (no uintptr_t round trip) so tile accesses compile to LDS/STS
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Ctl& ctl = *reinterpret_cast<Ctl*>(smem + kOffCtl);
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  auto tileB = [&](int s) { return smem + s * kSlotBytes; };
  auto tileX = [&](int s, int m) { return smem + s * kSlotBytes + (1 + m) * kTileBytes; };  // raw codes / A image

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&ctl.full[i], 1);
      // a stage is refilled only after the MMA consumed it AND every transform warp passed it: the transform
      // skips weight-image (SS) stages, and without its arrival it could run more than a ring cycle ahead of the
      // producer and pass a full-barrier parity wait one phase early (stale operands)
#ifndef MXM_EMPTY_XF
#define MXM_EMPTY_XF 1  // 0 only for timing A/B on layers without weight-image stages (unsafe otherwise)
#endif
      mbar_init(&ctl.empty[i], MXM_EMPTY_XF ? 1 + kXfWarps : 1);
    }
    for (int i = 0; i < kASlots; ++i) {
      mbar_init(&ctl.aready[i], kXfWarps);
      mbar_init(&ctl.aempty[i], 1);
    }
    for (int i = 0; i < kSSlots; ++i) {
      mbar_init(&ctl.sfull[i], 1);
      mbar_init(&ctl.sempty[i], MXM_LANE_ARRIVE ? 256 : 8);  // lane 0 of every epilogue warp (after __syncwarp)
      mbar_init(&ctl.sready[i], MXM_LANE_ARRIVE ? 32 : 1);   // lane 0 of the scale-staging warp 3
    }
    for (int i = 0; i < kAccBufs; ++i) {
      mbar_init(&ctl.accf[i], 1);
      mbar_init(&ctl.acce[i], 8);
    }
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&ctl.tfull[i], 1);
      mbar_init(&ctl.tempty[i], 1 + kXfWarps + 8 + 2);  // producer, transform, epilogue, scale staging
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&ctl.tmem_base);
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 7; ++i)
      for (int j = 0; j < 4; ++j) prefetch_tmap(&p.tmap[i][j]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl.tmem_base;
  const int n_tasks = p.meta[0];
#define n_split (SPLIT ? p.meta[7] : 1)  // split-K slices of splittable downs (plan; common.cuh)
  // wait-site cycle counters: compiled in only for the diagnostic build (tools/diag_waits.py); in the
  // product build they fold away (they would otherwise pin 32 registers in every role)
#ifdef MXM_DEBUG_COUNTERS
  const bool prof_on = p.prof != nullptr;
#else
  constexpr bool prof_on = false;
#endif
  unsigned long long pc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) pc[i] = 0;
  const unsigned long long t_start = clock64();

  // register rebalancing from the launch-time 96 per thread: setmaxnreg.inc only draws on what .dec released,
  // so the budget must balance exactly: 128 x (96-64) + 256 x (96-80) = 256 x (128-96)
#ifndef MXM_REG_LO
#define MXM_REG_LO 64
#define MXM_REG_XF 80
#define MXM_REG_HI 128
#endif
  static_assert(MXM_REG_LO == 0 || 128 * (96 - MXM_REG_LO) + 256 * (96 - MXM_REG_XF) >= 256 * (MXM_REG_HI - 96),
                "setmaxnreg budget");
  if (warp < 4) {
#if MXM_REG_LO > 0
  regs_dec<MXM_REG_LO>();
#endif
  if (warp == 0) {
    // =========================== producer
    if (lane == 0) {
      uint32_t stage = 0, sphase = 0;
      int n_tr_p = 0;
      for (uint32_t it = 0;; ++it) {
        const uint32_t slot = it % kRing, rphase = (it / kRing) & 1;
        const int idx = atomicAdd(&p.meta[5], 1);
        Task t;
        if (idx < n_tasks) {
          t = p.tasks[idx];
        } else {
          t.phase = 255;
        }
        twait(&ctl.tempty[slot], rphase ^ 1, pc[0], prof_on);
        ctl.ring[slot] = t;
        mbar_arrive(&ctl.tfull[slot]);
        if (t.phase == 255) break;
        if (t.phase == 1) continue;
        copy_task<0, SPLIT>(p, t, ctl, smem, stage, sphase, n_split, pc, prof_on, n_tr_p);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // =========================== MMA issuer (whole warp; one elected lane issues; one stream per SM)
    const uint32_t tm = bcast(tmem);
    uint32_t stage = 0, sphase = 0, abuf = 0;
    uint32_t acc_ph = 0;  // bit b: parity of the next wait on acce[b] (phase bits, no local arrays)
    uint32_t aidx = 0;    // TS stages issued so far (A-ring slot and parity)
    int ntr_m = 0, nev_m = 0;
#ifdef MXM_TRACE_TASKS
    const unsigned long long tt_start = gtimer();
    unsigned long long tt_tasks = 0, tt_stages = 0;
#endif
    for (uint32_t it = 0;; ++it) {
      const uint32_t slot = it % kRing, rphase = (it / kRing) & 1;
      twait(&ctl.tfull[slot], rphase, pc[3], prof_on);
      const Task t = ctl.ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl.tempty[slot]);
      const uint32_t phase = bcast(t.phase);
#ifdef MXM_TRACE_TASKS
      if (phase == 255 && lane == 0 && blockIdx.x < kTtCta) {
        g_cta[blockIdx.x][0] = tt_start;
        g_cta[blockIdx.x][1] = gtimer();
        g_cta[blockIdx.x][2] = tt_tasks;
        g_cta[blockIdx.x][3] = tt_stages;
      }
#endif
      if (phase == 255) break;
      if (phase == 1) continue;
      SubLoop sl[2];
      const int nsl = (int)bcast((uint32_t)build_subloops(t, p.ex, p.d, n_split, sl));
      const uint32_t nt = bcast(t.nt);
#ifdef MXM_TRACE_TASKS
      {
        unsigned long long nst = 0;
        for (int si = 0; si < nsl; ++si) nst += (unsigned long long)(SPLIT ? sl[si].ks1 - sl[si].ks0 : sl[si].ns);
        if (blockIdx.x == 0 && lane == 0 && tt_tasks < kTtN) {
          g_tt[0][tt_tasks] = clock64();
          g_tt[1][tt_tasks] = phase | (nst << 8) | ((unsigned long long)nt << 32) |
                              ((unsigned long long)sl[0].g128 << 48);
        }
        ++tt_tasks;
        tt_stages += nst;
      }
#endif
      for (int si = 0; si < nsl; ++si) {
        const SubLoop s = sl[si];
        const uint32_t ns = bcast((uint32_t)(SPLIT ? s.ks1 - s.ks0 : s.ns)), g128 = bcast((uint32_t)s.g128);
        const uint32_t xf = bcast((uint32_t)s.xform);
        const uint32_t i8 = bcast((uint32_t)s.i8), f8 = bcast((uint32_t)s.f8), two = bcast((uint32_t)(s.nmats == 2));
        MmaState st{stage, sphase, abuf, acc_ph, aidx, nev_m, ntr_m};
#if defined(MXM_PROF_SUBLOOP) && defined(MXM_DEBUG_COUNTERS)
        const unsigned long long t_sl = prof_on ? clock64() : 0ull;
#endif
        if (f8) {
          if (two)
            mma_subloop_mode<2, true>(ctl, smem, tm, ns, g128, xf, nt, st, pc, prof_on);
          else
            mma_subloop_mode<2, false>(ctl, smem, tm, ns, g128, xf, nt, st, pc, prof_on);
        } else if (i8) {
          if (two)
            mma_subloop_mode<1, true>(ctl, smem, tm, ns, g128, xf, nt, st, pc, prof_on);
          else
            mma_subloop_mode<1, false>(ctl, smem, tm, ns, g128, xf, nt, st, pc, prof_on);
        } else {
          if (two)
            mma_subloop_mode<0, true>(ctl, smem, tm, ns, g128, xf, nt, st, pc, prof_on);
          else
            mma_subloop_mode<0, false>(ctl, smem, tm, ns, g128, xf, nt, st, pc, prof_on);
        }
#if defined(MXM_PROF_SUBLOOP) && defined(MXM_DEBUG_COUNTERS)
        if (prof_on) pc[12] += clock64() - t_sl;
#endif
        stage = st.stage;
        sphase = st.sphase;
        abuf = st.abuf;
        acc_ph = st.acc_ph;
        aidx = st.aidx;
        nev_m = st.nev;
        ntr_m = st.ntr;
      }
    }
    __syncwarp();
  } else {
    // =========================== warp 2: second copy issuer (mat 1 + token tile, copy_task ROLE 1);
    // warp 3: scale staging of weight-activation g128 groups (stage_scales)
    uint32_t stage = 0, sphase = 0, xsidx = 0;
    int n_tr_h = 0;
    for (uint32_t it = 0;; ++it) {
      const uint32_t slot = it % kRing, rphase = (it / kRing) & 1;
      twait(&ctl.tfull[slot], rphase, pc[7], prof_on);
      const Task t = ctl.ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl.tempty[slot]);
      if (t.phase == 255) break;
      if (t.phase == 1) continue;
      if (warp == 2) {
        if (lane == 0) copy_task<1, SPLIT>(p, t, ctl, smem, stage, sphase, n_split, pc, prof_on, n_tr_h);
        __syncwarp();
        continue;
      }
      SubLoop sl[2];
      const int nsl = build_subloops(t, p.ex, p.d, n_split, sl);
      bool any_g128 = false;
      for (int si = 0; si < nsl; ++si) any_g128 |= sl[si].g128 != 0;
      if (!any_g128) continue;
      if (t.phase == 2) {  // h scales / sums come from this kernel's gate/up epilogues of the m-tile
        if (lane == 0) {
          while (ld_acquire_gpu(p.p1_done + t.gid) < p.grp_n1[t.gid]) __nanosleep(64);
        }
        __syncwarp();
      }
      for (int si = 0; si < nsl; ++si)
        if (sl[si].g128) stage_scales(p, t, sl[si], ctl, smem, xsidx, lane, pc, prof_on);
    }
    __syncwarp();
  }
  } else if ((warp >= 4 && warp < 8) || warp >= 16) {
    // =========================== transform: two warpgroups, each one K half of every stage, one A row per thread
#if MXM_REG_LO > 0
    regs_dec<MXM_REG_XF>();
#endif
    const int r = threadIdx.x & 127;
    const int xh = warp >= 16;
    uint32_t stage = 0, sphase = 0, aidx = 0;
    for (uint32_t it = 0;; ++it) {
      const uint32_t slot = it % kRing, rphase = (it / kRing) & 1;
      twait(&ctl.tfull[slot], rphase, pc[7], prof_on);
      const Task t = ctl.ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl.tempty[slot]);
      if (t.phase == 255) break;
      if (t.phase == 1) continue;
      SubLoop sl[2];
      const int nsl = build_subloops(t, p.ex, p.d, n_split, sl);
      for (int si = 0; si < nsl; ++si) {
        const SubLoop s = sl[si];
        const bool two = s.nmats == 2;
        const PackGeom& ga = s.mat[0]->geo;
        const PackGeom& gb = s.mat[s.nmats - 1]->geo;
        const int bitsA = ga.w_bits, bitsB = gb.w_bits;
        const bool symA = ga.sym != 0, symB = gb.sym != 0;
        const int mbA = ga.meta_bytes, mbB = gb.meta_bytes;
        const int gstA = ga.group / ga.ks, gstB = gb.group / gb.ks;
        const uint32_t offA = (0x4300u | (symA ? (1u << (bitsA - 1)) : 0u)) * 0x10001u;
        const uint32_t offB = (0x4300u | (symB ? (1u << (bitsB - 1)) : 0u)) * 0x10001u;
        const bool xa = (s.xform & 1) != 0, xb = two && (s.xform & 2) != 0;
        uint32_t sa = 0, za = 0, sb = 0, zb = 0;
        int gca = 0, gcb = 0;  // a split-K slice's first stage is laid out as a group start (producer)
        for (int ks = SPLIT ? s.ks0 : 0; ks < (SPLIT ? s.ks1 : s.ns); ++ks) {
          const bool hmA = gca == 0, hmB = gcb == 0;
          if (++gca == gstA) gca = 0;
          if (++gcb == gstB) gcb = 0;
          if (!s.xform) {
            twait(&ctl.full[stage], sphase, pc[8], prof_on);
            __syncwarp();
            if (MXM_EMPTY_XF && lane == 0) mbar_arrive(&ctl.empty[stage]);
          } else {
            const uint32_t aslot = aidx % kASlots;
            twait(&ctl.aempty[aslot], ((aidx / kASlots) & 1) ^ 1, pc[8], prof_on);  // MMA done with the slot
            twait(&ctl.full[stage], sphase, pc[8], prof_on);
            if (threadIdx.x == 128) TR(1, (int)aidx);
            tc_fence_after();
            // dequantized / unpacked rows go to the TMEM A ring (lane = row); one tcgen05.st per mat and K half,
            // mat 0's store in flight while mat 1 is unpacked
            const uint32_t tA = tmem + ((uint32_t)(r & ~31) << 16) + kTmemA + aslot * 64u;
            uint32_t o[16];
#ifdef MXM_ABL_XFORM
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = 0x3f803f80u;
            tmem_st16(tA + 16 * xh, o);
            if (two) tmem_st16(tA + 32 + 16 * xh, o);
            if (0)
#endif
            if (xh)
              xform_stage<1>(s, tileX(stage, 0), tileX(stage, 1), tA, r, hmA, hmB, bitsA, bitsB, mbA, mbB, symA, symB,
                             offA, offB, xa, xb, sa, za, sb, zb, o);
            else
              xform_stage<0>(s, tileX(stage, 0), tileX(stage, 1), tA, r, hmA, hmB, bitsA, bitsB, mbA, mbB, symA, symB,
                             offA, offB, xa, xb, sa, za, sb, zb, o);
#ifdef MXM_DEBUG_NAN
            if (!s.i8 && ((xa && (bf2_nonfinite(sa) || bf2_nonfinite(za))) || (xb && (bf2_nonfinite(sb) || bf2_nonfinite(zb)))))
              nan_note(p.prof, 1, t, ks, (int)(sa ^ (sb << 16)));
#endif
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&ctl.aready[aslot]);
            if (threadIdx.x == 128) TR(2, (int)aidx);
            ++aidx;
          }
          if (++stage == kStages) {
            stage = 0;
            sphase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 8 && warp < 16) {
    // =========================== epilogue (2 warpgroups)
#if MXM_REG_LO > 0
    regs_inc<MXM_REG_HI>();
#endif
    const int ew = warp - 8, wg = ew >> 2, q = warp & 3;
    const int l = q * 32 + lane;  // output channel within the tile == TMEM lane
    uint32_t abuf = 0, acc_ph = 0, rbuf = 0, sidx = 0;
    int n_tr_e = 0;
    (void)n_tr_e;
    for (uint32_t it = 0;; ++it) {
      const uint32_t slot = it % kRing, rphase = (it / kRing) & 1;
      twait(&ctl.tfull[slot], rphase, pc[9], prof_on);
      const Task t = ctl.ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl.tempty[slot]);
      if (t.phase == 255) break;
      const ExpertDesc& E = p.ex[t.expert];
      if (t.phase == 1) {
        // ---- dynamic quantization of h for a weight-activation down block (rows of one 32-row chunk)
        if (ew == 0 && lane == 0) {
          const int need = p.grp_n1[t.gid];
          const unsigned long long td = prof_on ? clock64() : 0ull;
          while (ld_acquire_gpu(p.p1_done + t.gid) < need) __nanosleep(64);
          if (prof_on) pc[14] += clock64() - td;
        }
        named_bar_sync(1, 256);
        // per-token W-A down: the row max |h| was accumulated by the phase-0 epilogues (atomicMax);
        // one vectorized pass quantizes the row (r = fl32(qmax/amax), s = fl32(amax/qmax), DESIGN R9)
        const LinDesc& L = E.blk[2];
        const int K = E.inter;
        const bool fp8 = kind_is_fp8(L.geo.kind);  // FP8 down: e4m3 codes (R26), qmax 448
        const float fq = fp8 ? 448.f : (float)((1 << (L.a_bits - 1)) - 1);
        const int sub0 = t.ntile * 32;
        for (int rr = ew; rr < 32; rr += 8) {
          const int local = sub0 + rr;
          if (local >= t.rows) break;
          const int64_t row = (int64_t)t.row0 + local;
          const float amax = __uint_as_float(__ldcg(p.hmax + row));
          const float r = amax > 0.f ? __fdiv_rn(fq, amax) : 0.f;
          const float sc = amax > 0.f ? __fdiv_rn(amax, fq) : 1.f;
          const uint4* src = reinterpret_cast<const uint4*>(p.H + h_off(p, row));
          uint2* dst = reinterpret_cast<uint2*>(p.Hq + h_off(p, row));
          // kU 16-byte loads in flight per lane before any store (a single load per iteration leaves this pass
          // latency-bound at a few GB/s per SM)
          constexpr int kU = 8;
          const int n8 = K / 8;
          const bool e4 = kind_is_w4a4(L.geo.kind);  // w4a4 down: e4m3 codes + the row's code sum
          int qsum = 0;
          for (int i0 = lane; i0 < n8; i0 += 32 * kU) {
            uint4 v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) v[u] = i0 + 32 * u < n8 ? __ldcg(src + i0 + 32 * u) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
              uint32_t o[2] = {0, 0};
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const float x = bf16f((uint16_t)(w[e >> 1] >> (16 * (e & 1))));
                if (fp8) {
                  o[e >> 2] |= fp8_act_code(x, r) << (8 * (e & 3));
                  continue;
                }
                const int qv = (int)fminf(fmaxf(rintf(__fmul_rn(x, r)), -fq), fq);
                if (i0 + 32 * u < n8) qsum += qv;
                o[e >> 2] |= (e4 ? code_byte<true>(qv) : code_byte<false>(qv)) << (8 * (e & 3));
              }
              if (i0 + 32 * u < n8) dst[i0 + 32 * u] = make_uint2(o[0], o[1]);
            }
          }
          if (e4) qsum = warp_sum(qsum);
          if (lane == 0) {
            p.Hs[row] = sc;  // per-token: group 0 of the group-major [g][R] layout
            if (e4) p.Hc[row] = qsum;
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
      const int nsl = build_subloops(t, p.ex, p.d, n_split, sl);
      const bool reg_mode = nsl == 2 || sl[0].g128;
      const int half = t.nt >> 1;
      const int col0 = wg * half;
      const int nvalid = t.rows - col0;                          // columns of this warpgroup with a real row
      const int n = sl[0].tile[0] * 128 + l;                     // mat 0's output channel
      const int n1 = sl[0].tile[nsl == 1 ? 1 : 0] * 128 + l;     // mat 1's (paired down tiles)
      const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
      float* cw_sa = ctl.cw[ew][0];
      float* cw_rw = ctl.cw[ew][1];
      float* cw_sb = ctl.cw[ew][2];
      const int cl = col0 + lane, ch = col0 + 32 + lane;
      const bool vlo = lane < half && cl < t.rows, vhi = 32 + lane < half && ch < t.rows;
      if (t.phase == 2) {  // route weights of this warp's columns, read back as broadcast float4s
        __syncwarp();
        cw_rw[lane] = vlo ? __ldg(p.row_w + t.row0 + cl) : 0.f;
        cw_rw[32 + lane] = vhi ? __ldg(p.row_w + t.row0 + ch) : 0.f;
        __syncwarp();
      }
      const LinDesc& Ld = E.blk[2];
      const int dmode = !kind_is_wa(Ld.geo.kind) ? 0
                        : (Ld.geo.group == 128 ? (kind_is_fp8(Ld.geo.kind) ? 4 : (kind_is_w4a4(Ld.geo.kind) ? 3 : 2)) : 1);
      const int dqmax = (1 << (Ld.a_bits - 1)) - 1;
      if (!reg_mode) {
        // ======== streaming epilogue: one drain event for the whole task (dual phase 0, or phase 2)
        const SubLoop s = sl[0];
        const bool split = SPLIT && s.ks1 - s.ks0 != s.ns;
        const int slice = task_slice(t);
        const bool two = s.nmats == 2;
        const float* xs_s = (t.phase == 0) ? p.xs[s.mat[0]->in_slot] : p.Hs;  // group-major [g][R]
        const int32_t* xc_s = (t.phase == 0) ? p.xc[s.mat[0]->in_slot] : p.Hc;
        float sw0 = 1.f, sw1 = 1.f, sa_lo = 1.f, sa_hi = 1.f;
        int qs_lo = 0, qs_hi = 0;
        if (s.i8 && t.phase == 0) {  // x-scales / weight scales exist before this kernel: load before the wait
          const uint16_t* wsc0 = reinterpret_cast<const uint16_t*>(s.mat[0]->packed + s.mat[0]->geo.wa_scale_off);
          const uint16_t* wsc1 = reinterpret_cast<const uint16_t*>(s.mat[s.nmats - 1]->packed +
                                                                  s.mat[s.nmats - 1]->geo.wa_scale_off);
          sw0 = bf16f(__ldg(wsc0 + n));
          sw1 = bf16f(__ldg(wsc1 + n1));
          sa_lo = vlo ? __ldg(xs_s + (int64_t)t.row0 + cl) : 0.f;
          sa_hi = vhi ? __ldg(xs_s + (int64_t)t.row0 + ch) : 0.f;
          if (s.w4) {
            qs_lo = vlo ? __ldg(xc_s + (int64_t)t.row0 + cl) : 0;
            qs_hi = vhi ? __ldg(xc_s + (int64_t)t.row0 + ch) : 0;
          }
        }
        const uint32_t b0 = abuf;
        abuf = abuf + 1 == kAccBufs ? 0 : abuf + 1;
        twait(&ctl.accf[b0], (acc_ph >> b0) & 1, pc[10], prof_on);
        if (threadIdx.x == 256) TR(5, n_tr_e);
        acc_ph ^= 1u << b0;
        tc_fence_after();
        if (s.i8 && t.phase != 0) {  // h-scales are written by this kernel: read after the MMA consumed Hq
          const uint16_t* wsc0 = reinterpret_cast<const uint16_t*>(s.mat[0]->packed + s.mat[0]->geo.wa_scale_off);
          sw0 = bf16f(__ldg(wsc0 + n));
          sw1 = bf16f(__ldg(wsc0 + n1));
          sa_lo = vlo ? __ldcg(xs_s + (int64_t)t.row0 + cl) : 0.f;
          sa_hi = vhi ? __ldcg(xs_s + (int64_t)t.row0 + ch) : 0.f;
          if (s.w4) {
            qs_lo = vlo ? __ldcg(xc_s + (int64_t)t.row0 + cl) : 0;
            qs_hi = vhi ? __ldcg(xc_s + (int64_t)t.row0 + ch) : 0;
          }
        }
        if (s.i8) {
          __syncwarp();
          if (s.w4) {  // w4a4: acc * (s_a 2^18) - 8 s_a sum(q_a); the correction once per K (slice 0 of a split)
            const bool corr = !split || slice == 0;
            cw_sa[lane] = sa_lo * 262144.f;
            cw_sa[32 + lane] = sa_hi * 262144.f;
            cw_sb[lane] = corr ? __fmul_rn(-8.f * (float)qs_lo, sa_lo) : 0.f;
            cw_sb[32 + lane] = corr ? __fmul_rn(-8.f * (float)qs_hi, sa_hi) : 0.f;
          } else if (s.f8) {  // FP8: acc is the sum over e4m3 values, acc * s_a
            cw_sa[lane] = sa_lo;
            cw_sa[32 + lane] = sa_hi;
            cw_sb[lane] = 0.f;
            cw_sb[32 + lane] = 0.f;
          } else {
            cw_sa[lane] = sa_lo;
            cw_sa[32 + lane] = sa_hi;
          }
          __syncwarp();
        }
        const uint32_t colA = b0 * (uint32_t)kAccCols;
        const uint32_t colB = colA + (uint32_t)kMat1Col;
        if constexpr (DUMP) {
          if (s.i8)
            dump_event(p, lane_addr + colA + (uint32_t)col0, lane_addr + colB + (uint32_t)col0, two,
                       t.phase == 0 ? 0 : 2, t.phase == 0 ? 1 : 2, 0, n, t.phase == 0 ? n : n1,
                       (int64_t)t.row0 + col0, half, nvalid);
        }
        const float2 swa = make_float2(sw0, sw0), swb = make_float2(sw1, sw1);
#ifndef MXM_ABL_EPI
        // specialised on (W-A, two mats, phase 0): with run-time flags the compiler predicates both variants
        auto stream = [&](auto i8_c, auto two_c, auto p0_c, auto f8_c) {
        constexpr bool I8 = decltype(i8_c)::value, TWO = decltype(two_c)::value, P0 = decltype(p0_c)::value;
        constexpr bool F8 = decltype(f8_c)::value;
#pragma unroll 1
        for (int c = 0; c < half; c += 8) {
          uint32_t va[8], vb[8];
          const uint32_t cbase = (uint32_t)(col0 + c);
          tmem_ld8(lane_addr + colA + cbase, va);
          if constexpr (TWO) tmem_ld8(lane_addr + colB + cbase, vb);
          tmem_ld_wait();
          float fa[8], fb[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            fa[j] = __uint_as_float(va[j]);
            fb[j] = TWO ? __uint_as_float(vb[j]) : 0.f;
          }
          if constexpr (I8 && F8) {  // w4a4: s_w * (acc * a + b) per column (a, b broadcast from smem)
            const float4 x0 = *reinterpret_cast<const float4*>(cw_sa + c);
            const float4 x1 = *reinterpret_cast<const float4*>(cw_sa + c + 4);
            const float4 y0 = *reinterpret_cast<const float4*>(cw_sb + c);
            const float4 y1 = *reinterpret_cast<const float4*>(cw_sb + c + 4);
            const float2 a2s[4] = {make_float2(x0.x, x0.y), make_float2(x0.z, x0.w), make_float2(x1.x, x1.y),
                                   make_float2(x1.z, x1.w)};
            const float2 b2s[4] = {make_float2(y0.x, y0.y), make_float2(y0.z, y0.w), make_float2(y1.x, y1.y),
                                   make_float2(y1.z, y1.w)};
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
              const float2 a2 = fmul2(ffma2(make_float2(fa[j], fa[j + 1]), a2s[j / 2], b2s[j / 2]), swa);
              fa[j] = a2.x; fa[j + 1] = a2.y;
              if constexpr (TWO) {
                const float2 b2 = fmul2(ffma2(make_float2(fb[j], fb[j + 1]), a2s[j / 2], b2s[j / 2]), swb);
                fb[j] = b2.x; fb[j + 1] = b2.y;
              }
            }
          } else if constexpr (I8) {  // per-column activation scale: broadcast smem reads
            const float4 x0 = *reinterpret_cast<const float4*>(cw_sa + c);
            const float4 x1 = *reinterpret_cast<const float4*>(cw_sa + c + 4);
            const float2 s2[4] = {make_float2(x0.x, x0.y), make_float2(x0.z, x0.w), make_float2(x1.x, x1.y),
                                  make_float2(x1.z, x1.w)};
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
              const float2 a2 = fmul2(make_float2((float)(int32_t)va[j], (float)(int32_t)va[j + 1]), fmul2(swa, s2[j / 2]));
              fa[j] = a2.x; fa[j + 1] = a2.y;
              if constexpr (TWO) {
                const float2 b2 =
                    fmul2(make_float2((float)(int32_t)vb[j], (float)(int32_t)vb[j + 1]), fmul2(swb, s2[j / 2]));
                fb[j] = b2.x; fb[j + 1] = b2.y;
              }
            }
          }
#ifdef MXM_DEBUG_NAN
          for (int j = 0; j < 8; ++j)
            if (c + j < nvalid && (!isfinite(fa[j]) || (TWO && !isfinite(fb[j]))))
              nan_note(p.prof, t.phase == 0 ? 2 : 3, t, c + j, (int)__float_as_uint(isfinite(fa[j]) ? fb[j] : fa[j]));
#endif
          if constexpr (P0) {
            uint16_t hb[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) hb[j] = f2bf(silu_f(fa[j]) * fb[j]);
            emit_h8<DUMP>(p, t, dmode, dqmax, n, col0 + c, nvalid - c, hb, ctl, wg, q, lane, rbuf);
          } else if (split) {  // split-K slice: fp32 partial sums (reduced below by the last slice)
            float* q0 = p.P + ((int64_t)slice * kSplitRows + t.row0 + col0 + c) * p.d + n;
            float* q1 = p.P + ((int64_t)slice * kSplitRows + t.row0 + col0 + c) * p.d + n1;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (c + j < nvalid) {
                __stcg(q0 + (int64_t)j * p.d, fa[j]);
                if constexpr (TWO) __stcg(q1 + (int64_t)j * p.d, fb[j]);
              }
            }
          } else {
            const float4 r0 = *reinterpret_cast<const float4*>(cw_rw + c);
            const float4 r1 = *reinterpret_cast<const float4*>(cw_rw + c + 4);
            const float rw[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
            uint16_t* o0 = p.O + ((int64_t)t.row0 + col0 + c) * p.d + n;
            uint16_t* o1 = p.O + ((int64_t)t.row0 + col0 + c) * p.d + n1;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (c + j < nvalid) {
                o0[(int64_t)j * p.d] = f2bf(fa[j] * rw[j]);
                if constexpr (TWO) o1[(int64_t)j * p.d] = f2bf(fb[j] * rw[j]);
              }
            }
          }
        }
        };
        using Tt = std::true_type;
        using Ft = std::false_type;
        if (t.phase == 0) {
          if (s.f8) { if (two) stream(Tt{}, Tt{}, Tt{}, Tt{}); else stream(Tt{}, Ft{}, Tt{}, Tt{}); }
          else if (s.i8) { if (two) stream(Tt{}, Tt{}, Tt{}, Ft{}); else stream(Tt{}, Ft{}, Tt{}, Ft{}); }
          else { if (two) stream(Ft{}, Tt{}, Tt{}, Ft{}); else stream(Ft{}, Ft{}, Tt{}, Ft{}); }
        } else {
          if (s.f8) { if (two) stream(Tt{}, Tt{}, Ft{}, Tt{}); else stream(Tt{}, Ft{}, Ft{}, Tt{}); }
          else if (s.i8) { if (two) stream(Tt{}, Tt{}, Ft{}, Ft{}); else stream(Tt{}, Ft{}, Ft{}, Ft{}); }
          else { if (two) stream(Ft{}, Tt{}, Ft{}, Ft{}); else stream(Ft{}, Ft{}, Ft{}, Ft{}); }
        }
#endif
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctl.acce[b0]);
        if (threadIdx.x == 256) TR(6, n_tr_e);
        ++n_tr_e;
        if (split) {
          // the last-arriving slice of this (m-tile, down tile) sums the slices' partials in slice order
          named_bar_sync(1, 256);
          if (ew == 0 && lane == 0) {
            __threadfence();
            const int old = atomicAdd(p.red_cnt + (int64_t)t.gid * (p.d / 128) + task_tile(t), 1);
            ctl.red_last = old == n_split - 1;
            __threadfence();
          }
          named_bar_sync(1, 256);
          if (ctl.red_last) {
            const bool two = s.nmats == 2;
            for (int c = 0; c < half; ++c) {
              if (c >= nvalid) break;
              const int64_t row = (int64_t)t.row0 + col0 + c;
              float a0 = 0.f, a1 = 0.f;
              for (int q2 = 0; q2 < n_split; ++q2) {
                const float* pr = p.P + ((int64_t)q2 * kSplitRows + row) * p.d;
                a0 += __ldcg(pr + n);
                if (two) a1 += __ldcg(pr + n1);
              }
              const float rw = cw_rw[c];
              p.O[row * p.d + n] = f2bf(a0 * rw);
              if (two) p.O[row * p.d + n1] = f2bf(a1 * rw);
            }
          }
        }
      } else {
        // ======== register-accumulating epilogue (g128 drains / hetero gate-up sub-loops)
        float2 acc2[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) acc2[i] = make_float2(0.f, 0.f);
        for (int si = 0; si < nsl; ++si) {
          const SubLoop s = sl[si];
          const bool two = s.nmats == 2;
          const int nev = s.g128 ? s.ns : 1;
          const float* xs_s = (t.phase == 0) ? p.xs[s.mat[0]->in_slot] : p.Hs;  // group-major [g][R]
          const uint16_t* wsc0 = reinterpret_cast<const uint16_t*>(s.mat[0]->packed + s.mat[0]->geo.wa_scale_off);
          const uint16_t* wsc1 =
              two ? reinterpret_cast<const uint16_t*>(s.mat[1]->packed + s.mat[1]->geo.wa_scale_off) : wsc0;
          const float* xs_lo = xs_s + (int64_t)t.row0 + cl;
          const float* xs_hi = xs_s + (int64_t)t.row0 + ch;
          const int32_t* xc_s = (t.phase == 0) ? p.xc[s.mat[0]->in_slot] : p.Hc;
          const int64_t gs = p.hs_stride;
          // g128: per-event scales come through the scale ring. Per-channel: phase 0 reads scales written
          // before this kernel (read-only path, before the wait); phase 2 reads h-scales written by this
          // kernel after the accumulator wait, through L2 (ld.cg)
          const bool pre = t.phase == 0;
          float nsw0 = 1.f, nsw1 = 1.f, nsa_lo = 1.f, nsa_hi = 1.f;
          int nqs_lo = 0, nqs_hi = 0;
          if (s.i8 && !s.g128) {  // per-channel (one event): scales from global memory
            if (pre) {
              nsw0 = bf16f(__ldg(wsc0 + n));
              if (two) nsw1 = bf16f(__ldg(wsc1 + n1));
              nsa_lo = vlo ? __ldg(xs_lo) : 0.f;
              nsa_hi = vhi ? __ldg(xs_hi) : 0.f;
              if (s.w4) {
                nqs_lo = vlo ? __ldg(xc_s + (int64_t)t.row0 + cl) : 0;
                nqs_hi = vhi ? __ldg(xc_s + (int64_t)t.row0 + ch) : 0;
              }
            }
          }
          for (int ev = 0; ev < nev; ++ev) {
            float sw0 = nsw0, sw1 = nsw1;
            const uint32_t b0 = abuf;
            abuf = abuf + 1 == kAccBufs ? 0 : abuf + 1;
            twait(&ctl.accf[b0], (acc_ph >> b0) & 1, pc[10], prof_on);
            if (threadIdx.x == 256) TR(5, n_tr_e);
            acc_ph ^= 1u << b0;
            tc_fence_after();
            const float* sa_ev = cw_sa;
            uint32_t ss = 0;
            if (s.g128) {  // g128 event: the group's scales arrived in the scale ring with the stage
              ss = sidx & (kSSlots - 1);
              twait(&ctl.sready[ss], (sidx / kSSlots) & 1, pc[10], prof_on);  // factors staged by the transform
#ifndef MXM_TRACE_PRODUCER
              if (threadIdx.x == 256) TR(7, n_tr_e);
#endif
              const uint8_t* slotp = smem + kOffScale + ss * kSSlotBytes;
              sw0 = bf16f(reinterpret_cast<const uint16_t*>(slotp)[l]);
              if (two) sw1 = bf16f(reinterpret_cast<const uint16_t*>(slotp + 256)[l]);
              sa_ev = reinterpret_cast<const float*>(slotp + kSlotA) + col0;  // b at sa_ev + (kSlotB - kSlotA) / 4
            } else if (s.i8) {
              if (!pre) {  // h-scales are written by this kernel: read after the MMA consumed Hq (ld.cg)
                sw0 = bf16f(__ldg(wsc0 + n));
                if (two) sw1 = bf16f(__ldg(wsc1 + n1));
                nsa_lo = vlo ? __ldcg(xs_lo) : 0.f;
                nsa_hi = vhi ? __ldcg(xs_hi) : 0.f;
                if (s.w4) {
                  nqs_lo = vlo ? __ldcg(xc_s + (int64_t)t.row0 + cl) : 0;
                  nqs_hi = vhi ? __ldcg(xc_s + (int64_t)t.row0 + ch) : 0;
                }
              }
              __syncwarp();
              if (s.w4) {
                cw_sa[lane] = nsa_lo * 262144.f;
                cw_sa[32 + lane] = nsa_hi * 262144.f;
                cw_sb[lane] = __fmul_rn(-8.f * (float)nqs_lo, nsa_lo);
                cw_sb[32 + lane] = __fmul_rn(-8.f * (float)nqs_hi, nsa_hi);
              } else if (s.f8) {  // FP8
                cw_sa[lane] = nsa_lo;
                cw_sa[32 + lane] = nsa_hi;
                cw_sb[lane] = 0.f;
                cw_sb[32 + lane] = 0.f;
              } else {
                cw_sa[lane] = nsa_lo;
                cw_sa[32 + lane] = nsa_hi;
              }
              __syncwarp();
            }
            const uint32_t colA = b0 * (uint32_t)kAccCols;
            const uint32_t colB = colA + (uint32_t)kMat1Col;
            const bool dst_hi = t.phase == 0 && nsl == 2 && si == 1;  // hetero: the up sub-loop
            const uint32_t aA = lane_addr + colA + (uint32_t)col0, aB = lane_addr + colB + (uint32_t)col0;
            if constexpr (DUMP) {
              if (s.i8) {
                const int jA = t.phase != 0 ? 2 : (nsl == 2 ? si : 0);
                const int jB = t.phase != 0 ? 2 : 1;
                dump_event(p, aA, aB, two, jA, jB, s.g128 ? ev : 0, n, t.phase == 0 ? n : n1,
                           (int64_t)t.row0 + col0, half, nvalid);
              }
            }
#ifndef MXM_ABL_EPI
#ifndef MXM_TRACE_PRODUCER
            if (threadIdx.x == 256) TR(8, n_tr_e);
#endif
            const unsigned long long t_dr = prof_on ? clock64() : 0ull;
            if (dst_hi)
              drain_event_any<16>(half, acc2, aA, aB, s.i8, s.f8, false, s.g128, sw0, sw1, sa_ev);
            else
              drain_event_any<0>(half, acc2, aA, aB, s.i8, s.f8, two, s.g128, sw0, sw1, sa_ev);
            if (prof_on) pc[12] += clock64() - t_dr;  // register-accumulating drain time (diagnostic build)
#ifndef MXM_TRACE_PRODUCER
            if (threadIdx.x == 256) TR(9, n_tr_e);
#endif
#endif
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&ctl.acce[b0]);
            // the warp's slot reads are ordered before lane 0's release by the __syncwarp above (one arrival per
            // warp: per-lane arrivals serialise on the barrier word)
            if (s.g128 && (MXM_LANE_ARRIVE || lane == 0)) mbar_arrive(&ctl.sempty[ss]);
            if (threadIdx.x == 256) TR(6, n_tr_e);
            ++n_tr_e;
            if (s.g128) ++sidx;
          }
        }
        const float* acc = reinterpret_cast<const float*>(acc2);
        if (t.phase == 0) {
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            if (cc * 8 < half) {
              uint16_t hb[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) hb[j] = f2bf(silu_f(acc[cc * 8 + j]) * acc[32 + cc * 8 + j]);
              emit_h8<DUMP>(p, t, dmode, dqmax, n, col0 + cc * 8, nvalid - cc * 8, hb, ctl, wg, q, lane, rbuf);
            }
          }
        } else {
          const bool two = sl[0].nmats == 2;  // paired down tiles: mat 1 in acc[32..63]
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) {
            if (cc * 8 < half) {
              const float4 r0 = *reinterpret_cast<const float4*>(cw_rw + cc * 8);
              const float4 r1 = *reinterpret_cast<const float4*>(cw_rw + cc * 8 + 4);
              const float rw[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
              uint16_t* o0 = p.O + ((int64_t)t.row0 + col0 + cc * 8) * p.d + n;
              uint16_t* o1 = p.O + ((int64_t)t.row0 + col0 + cc * 8) * p.d + n1;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                if (cc * 8 + j < nvalid) {
                  o0[(int64_t)j * p.d] = f2bf(acc[cc * 8 + j] * rw[j]);
                  if (two && cc < 4) o1[(int64_t)j * p.d] = f2bf(acc[32 + cc * 8 + j] * rw[j]);
                }
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
  if (prof_on && lane == 0 && (warp == 0 || warp == 1 || warp == 4 || warp == 8)) {
    // one representative thread per role: producer (0-2), MMA (3-6, 13), transform (7-8), epilogue (9-10, 14)
    unsigned long long* dst = p.prof + (size_t)blockIdx.x * 16;
    for (int i = 0; i < 15; ++i)
      if (pc[i]) atomicAdd(dst + i, pc[i]);
    if (warp == 0) atomicAdd(dst + 15, clock64() - t_start);
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

#ifdef MXM_TRACE
cudaError_t debug_trace(unsigned long long* out) { return cudaMemcpyFromSymbol(out, g_tr, sizeof(g_tr)); }
#endif
#ifdef MXM_TRACE_TASKS
cudaError_t debug_trace_tasks(unsigned long long* tt, unsigned long long* cta) {
  cudaError_t e = cudaMemcpyFromSymbol(tt, g_tt, sizeof(g_tt));
  return e != cudaSuccess ? e : cudaMemcpyFromSymbol(cta, g_cta, sizeof(g_cta));
}
#endif
#ifdef MXM_DEBUG_NAN
cudaError_t debug_nan_info(unsigned long long* out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_nan_info, sizeof(g_nan_info));
  if (e == cudaSuccess && reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_nan_info, z, sizeof(z));
  }
  return e;
}
#endif
cudaError_t launch_moe_gemm(const GemmParams& prm, int grid, cudaStream_t st) {
  // the dynamic-smem opt-in is per device: remember it per device ordinal (first use on each GPU)
  static std::mutex mu;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr_set[dev]) {
      e = cudaFuncSetAttribute(moe_gemm_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(moe_gemm_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(moe_gemm_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
      if (e != cudaSuccess) return e;
      attr_set[dev] = true;
    }
  }
  if (prm.dump != nullptr)
    moe_gemm_kernel<false, true><<<grid, kThreads, kSmemBytes, st>>>(prm);
  else if (prm.P != nullptr)
    moe_gemm_kernel<true, false><<<grid, kThreads, kSmemBytes, st>>>(prm);
  else
    moe_gemm_kernel<false, false><<<grid, kThreads, kSmemBytes, st>>>(prm);
  return cudaGetLastError();
}

}  // namespace mxm
