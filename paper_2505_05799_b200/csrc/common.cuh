// common.cuh — structures shared by the host runtime and the device kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/mxmoe.h"

namespace mxm {

constexpr int kNumSms = 148;
#ifndef MXM_ASLOTS
#define MXM_ASLOTS 2  // TMEM A-ring depth of the group-GEMM (gemm.cu); sets the dual token tile below
#endif
#ifndef MXM_ACC_BUFS
#define MXM_ACC_BUFS 2  // TMEM accumulator buffers (3: 64-token dual tiles, one more MMA/epilogue overlap stage)
#endif
#define MXM_DUAL_TILE (MXM_ACC_BUFS == 3 ? 64 : (MXM_ASLOTS == 3 ? 80 : 96))  // max tokens of a dual m-tile
constexpr int kRowsPerTile = 128;  // output channels per tile (UMMA M)

// Packed-format kinds (docs/packed_format.md)
enum Kind : int8_t {
  KIND_W16 = 0,     // F16 image chunks (bf16 pass-through)
  KIND_WO = 1,      // F16 row-word chunks, weight-only w2/w3/w4/w8 -> dequant to bf16
  KIND_WA_ROW = 2,  // I8 row-word chunks, w5a5 -> unpack to s8, tcgen05 kind::i8
  KIND_WA_IMG = 3,  // I8 image chunks, w8a8, tcgen05 kind::i8
  KIND_WA_F8 = 4,   // I8 row-word chunks (same bytes as KIND_WA_ROW w4), w4a4 -> nibble bytes read as e4m3 by
                    // tcgen05 kind::f8f6f4: byte u in [0,15] is the e4m3 value u * 2^-9 (subnormal / first binade,
                    // linear in u), activation codes are e4m3 (q<0)<<7 | |q| = q * 2^-9, so the f32 accumulator
                    // is 2^-18 * sum (q_w + 8) q_a exactly (integer sums < 2^24; tools/probe_f8.cu)
  KIND_FP8 = 5,     // I8 image chunks of e4m3 weight codes (MXM_FMT_E4M3), tcgen05 kind::f8f6f4 from smem (SS),
                    // e4m3 activation codes; the f32 accumulator is sum q_w q_a over e4m3 values (R25/R26)
};

// weight-activation kinds: 8-bit MMA operands, 128-element K stages, per-group / per-channel scale drains
__host__ __device__ inline bool kind_is_wa(int k) { return k >= KIND_WA_ROW; }
// kinds multiplied by tcgen05.mma kind::f8f6f4 (w4a4 and FP8)
__host__ __device__ inline bool kind_is_f8(int k) { return k == KIND_WA_F8 || k == KIND_FP8; }
// w4a4 on the fp8 tensor core: nibble-offset accumulators (drain factor a = s_a 2^18, correction b)
__host__ __device__ inline bool kind_is_w4a4(int k) { return k == KIND_WA_F8; }
__host__ __device__ inline bool kind_is_fp8(int k) { return k == KIND_FP8; }
// row-word packed 8-bit-operand kinds (nibble + bit planes, unpacked by the transform warps)
__host__ __device__ inline bool kind_is_row8(int k) { return k == KIND_WA_ROW || k == KIND_WA_F8; }
__host__ __device__ inline bool kind_needs_transform(int k) { return k == KIND_WO || kind_is_row8(k); }

// Geometry of one packed linear block W[N, K].
struct PackGeom {
  int32_t N, K;
  int8_t kind, w_bits, a_bits, sym;
  int32_t group;        // effective group (K for per-channel)
  int32_t ks;           // stage elements (64 F16, 128 I8)
  int32_t ns;           // stages = K / ks
  int32_t code_bytes;   // code bytes per chunk
  int32_t meta_bytes;   // meta bytes at a group-start chunk (WO only)
  int64_t rb_bytes;     // bytes per 128-row block
  int64_t wa_scale_off; // byte offset of the I8 weight-scale array [K/g][N]
  int64_t total_bytes;
};

__host__ __device__ inline int64_t chunk_offset(const PackGeom& g, int rb, int ks) {
  const int64_t starts = ((int64_t)ks * g.ks + g.group - 1) / g.group;  // group starts before stage ks
  return (int64_t)rb * g.rb_bytes + (int64_t)ks * g.code_bytes + (g.kind == KIND_WO ? starts * g.meta_bytes : 0);
}
__host__ __device__ inline bool chunk_has_meta(const PackGeom& g, int ks) {
  return g.kind == KIND_WO && ((int64_t)ks * g.ks) % g.group == 0;
}

// Device descriptor of one linear block inside a layer.
struct LinDesc {
  const uint8_t* packed;
  PackGeom geo;
  int32_t in_slot;   // gate/up: 0 = bf16 X, 1 = i8 slot A, 2 = i8 slot B; down: 0 = bf16 H, 1 = i8 H
  int32_t a_bits, a_group;
};

// One (virtual) expert: routed experts 0..E-1, then shared experts.
struct ExpertDesc {
  LinDesc blk[3];
  int32_t inter;      // f of this expert
  int32_t dual;       // gate and up run as one K loop sharing the token tile (same MMA kind and input slot)
  int32_t shared;     // 1 = shared expert (all tokens)
  int32_t pad;
  float cost[4];      // measured cost of one m-tile group at token tiles 16 / 32 / 64 / dual (ms; 0 = analytic)
};

// Task descriptor (16 bytes), produced by the plan kernel, consumed by the persistent kernel.
struct Task {
  uint16_t expert;
  uint8_t phase;   // 0 gate/up, 1 h-quant, 2 down, 255 stop
  uint8_t nt;      // token tile (16/32/64/128); h-quant: sub-chunk index
  int32_t row0;    // first route row of the m-tile (group)
  uint16_t rows;   // valid rows in the m-tile
  uint16_t ntile;  // 128-channel output tile index (h-quant: unused)
  int32_t gid;     // m-tile group id (dependency counters)
};
static_assert(sizeof(Task) == 16, "task size");

// Split-K of phase-2 (down) tasks: when a launch has fewer down tasks than SMs (tiny T, e.g.
// Mixtral T <= 256) each down task of a streaming-epilogue expert is cut into S <= kSplitMax K-slices (meta[7]);
// slices write fp32 partials, the last-arriving slice reduces them in fixed slice order (deterministic).
// A phase-2 task's ntile holds the tile (pair) index in bits 0-9 and the slice in bits 10-13.
#ifndef MXM_SPLIT_MAX
#define MXM_SPLIT_MAX 4
#endif
constexpr int kSplitMax = MXM_SPLIT_MAX;
#ifndef MXM_SPLIT_ROWS
#define MXM_SPLIT_ROWS 512
#endif
constexpr int kSplitRows = MXM_SPLIT_ROWS;  // split only when the launch has <= this many route rows (0: never)
__host__ __device__ inline int task_tile(const Task& t) { return t.phase == 2 ? (t.ntile & 0x3FF) : t.ntile; }
__host__ __device__ inline int task_slice(const Task& t) { return t.phase == 2 ? (t.ntile >> 10) : 0; }
__host__ __device__ inline bool down_splittable(const ExpertDesc& e) {
  return !(kind_is_wa(e.blk[2].geo.kind) && e.blk[2].geo.group == 128);  // g128 W-A downs drain per group
}
// stage range [ks0, ks1) of slice `sl` of S over ns stages (slices of an even number of stages so a g128 / g64
// weight-only group never straddles two slices)
__host__ __device__ inline void split_range(int ns, int S, int sl, int& ks0, int& ks1) {
  const int per = (((ns + S - 1) / S) + 1) & ~1;
  ks0 = sl * per;
  ks1 = ks0 + per < ns ? ks0 + per : ns;
}

// Token-tile cap of an expert's m-tiles: dual gate/up tiles of up to MXM_DUAL_TILE tokens fit one TMEM
// accumulator buffer (2 x 160 columns next to a 3-slot A ring); register-accumulated tiles (g128 W-A dual, or gate and up as two sub-loops) keep
// 64 columns per warpgroup half in registers -> 64 tokens.
#ifndef MXM_REG_TILE
#define MXM_REG_TILE 64  // token-tile cap of register-accumulated (g128 W-A / two-sub-loop) m-tiles
#endif
__host__ __device__ inline int tile_cap(const ExpertDesc& e) {
  const bool reg = !e.dual || (kind_is_wa(e.blk[0].geo.kind) && e.blk[0].geo.group == 128);
  return reg ? MXM_REG_TILE : MXM_DUAL_TILE;
}
// Down tasks pair two 128-channel output tiles (two mats sharing the h tile) unless the down is a g128
// W-A block whose register-accumulated drain would exceed 64 columns per thread.
__host__ __device__ inline bool down_pair(const ExpertDesc& e, int nt, int nd) {
  const bool g128 = kind_is_wa(e.blk[2].geo.kind) && e.blk[2].geo.group == 128;
  return nd >= 2 && !(g128 && nt > 64);
}
__host__ __device__ inline int down_tasks(const ExpertDesc& e, int nt, int nd) {
  return down_pair(e, nt, nd) ? (nd + 1) / 2 : nd;
}

}  // namespace mxm

namespace mxm {
// Validate a scheme for W[N, K] and fill its packed geometry. Returns MXM_OK or MXM_E_CONFIG.
__host__ __device__ inline mxm_status make_geom(const mxm_scheme& s, int64_t N, int64_t K, PackGeom* g) {
  if (N <= 0 || K <= 0 || N % 128 != 0 || N > (1 << 24) || K > (1 << 24)) return MXM_E_CONFIG;
  if (s.fmt != MXM_FMT_INT && s.fmt != MXM_FMT_E4M3) return MXM_E_CONFIG;
  if (s.fmt == MXM_FMT_E4M3 && s.a_bits == 16) return MXM_E_CONFIG;
  PackGeom r{};
  r.N = (int32_t)N;
  r.K = (int32_t)K;
  r.w_bits = (int8_t)s.w_bits;
  r.a_bits = (int8_t)s.a_bits;
  r.sym = (int8_t)(s.symmetric ? 1 : 0);
  if (s.w_bits == 16) {
    if (s.a_bits != 16) return MXM_E_CONFIG;
    r.kind = KIND_W16;
    r.ks = 64;
    r.group = (int32_t)K;
    r.sym = 1;
  } else if (s.a_bits == 16) {
    if (!(s.w_bits == 2 || s.w_bits == 3 || s.w_bits == 4 || s.w_bits == 8)) return MXM_E_CONFIG;
    if (!(s.w_group == -1 || s.w_group == 64 || s.w_group == 128)) return MXM_E_CONFIG;
    r.kind = KIND_WO;
    r.ks = 64;
    r.group = s.w_group == -1 ? (int32_t)K : s.w_group;
  } else if (s.fmt == MXM_FMT_E4M3) {
    if (s.w_bits != 8 || s.a_bits != 8 || !s.symmetric) return MXM_E_CONFIG;
    if (!(s.w_group == -1 || s.w_group == 128) || s.a_group != s.w_group) return MXM_E_CONFIG;
    r.kind = KIND_FP8;
    r.ks = 128;
    r.group = s.w_group == -1 ? (int32_t)K : s.w_group;
  } else {
    if (s.a_bits != s.w_bits || !s.symmetric) return MXM_E_CONFIG;
    if (!(s.w_bits == 4 || s.w_bits == 5 || s.w_bits == 8)) return MXM_E_CONFIG;
    if (!(s.w_group == -1 || s.w_group == 128) || s.a_group != s.w_group) return MXM_E_CONFIG;
    r.kind = s.w_bits == 8 ? KIND_WA_IMG : (s.w_bits == 4 ? KIND_WA_F8 : KIND_WA_ROW);
    r.ks = 128;
    r.group = s.w_group == -1 ? (int32_t)K : s.w_group;
  }
  if (K % r.ks != 0 || K % r.group != 0) return MXM_E_CONFIG;
  r.ns = (int32_t)(K / r.ks);
  r.code_bytes = r.kind == KIND_W16 ? 16384 : 128 * r.ks * s.w_bits / 8;
  r.meta_bytes = r.kind == KIND_WO ? (r.sym ? 256 : 512) : 0;
  const int64_t ng = K / r.group;
  r.rb_bytes = (int64_t)r.ns * r.code_bytes + (r.kind == KIND_WO ? ng * r.meta_bytes : 0);
  r.wa_scale_off = (N / 128) * r.rb_bytes;
  r.total_bytes = r.wa_scale_off + (kind_is_wa(r.kind) ? ng * N * 2 : 0);
  *g = r;
  return MXM_OK;
}
}  // namespace mxm
