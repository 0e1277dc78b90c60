// plan.cu — step S3: build the tile task list of one MoE block on the device.
//
// The paper's runtime cost model approximates block time by the serial time of all tiles over the
// SMs and its scheduler "prioritizes computationally intensive tiles" (greedy makespan,
// P:231; Graham's bound). Here: every (expert, m-tile) group contributes f/128 gate+up tiles
// (phase 1), ceil(rows/32) h-quantization sub-tasks when its down block is weight-activation, and
// its down tasks (phase 2): pairs of 128-channel tiles (down_pair, common.cuh) or single tiles.
// Groups are ordered by estimated per-tile cost, descending (LPT); the whole phase-1 list precedes the h-quant list which precedes phase 2, so the dynamic queue
// of the persistent kernel can never deadlock on a dependency.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace mxm {

constexpr int kPlanThreads = 1024;
#ifndef MXM_NMAJOR_MIN_GROUPS
#define MXM_NMAJOR_MIN_GROUPS 2  // experts with at least this many full m-tiles are emitted n-tile-major (0 = off)
#endif
#ifndef MXM_BAND_MB
#define MXM_BAND_MB 32  // n-tile-major emission in bands of m-tiles whose input rows total <= this many MiB (0: one band)
#endif
constexpr int kMaxV = 256;

// one 16-byte store per task: the plan is a single block whose scattered task stores bound it (4-byte field
// stores issued 4 L2 transactions per lane and task: Q2 plan 239 us, ncu profiles/r02/ncu_plan_q2.txt)
__device__ __forceinline__ void st_task(Task* dst, const Task& t) {
  uint4 u;
  memcpy(&u, &t, sizeof(u));
  *reinterpret_cast<uint4*>(dst) = u;
}

// m-tiles per band of an n-tile-major expert: its input rows (row_bytes each, nt rows per m-tile) stay in L2 while
// every n-tile of the band runs; at least 2 m-tiles, at most the expert's nf full m-tiles
__device__ __forceinline__ int band_groups(int64_t row_bytes, int nt, int nf) {
  if (MXM_BAND_MB <= 0) return nf;
  const int64_t b = ((int64_t)MXM_BAND_MB << 20) / (row_bytes * nt > 0 ? row_bytes * nt : 1);
  return (int)(b < 2 ? 2 : (b > nf ? nf : b));
}
// queue slot of (m-tile i, n-task j) inside an expert's block of nf x n tasks: bands of B m-tiles, n-tile-major
// within a band
__device__ __forceinline__ int64_t band_pos(int i, int j, int nf, int n, int B) {
  const int b = i / B, ii = i - b * B, Bb = min(B, nf - b * B);
  return (int64_t)b * B * n + (int64_t)j * Bb + ii;
}

// exclusive block-wide scan of one int per thread (kPlanThreads threads); returns the block total
__device__ int block_excl_scan(int v, int* warp_tot, int* out_total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  const int base = w > 0 ? warp_tot[w - 1] : 0;
  const int total = warp_tot[31];
  __syncthreads();
  *out_total = total;
  return base + x - v;
}

__device__ __forceinline__ int pow2_index(int nt) { return nt <= 16 ? 0 : (nt <= 32 ? 1 : (nt <= 64 ? 2 : 3)); }

// token tile of an m-tile with m rows: 16 / 32 / 64 / MXM_DUAL_TILE (the TMA boxes, MMA N)
__device__ __forceinline__ int pow2_tile(int m) {
  return m <= 16 ? 16 : (m <= 32 ? 32 : (m <= 64 ? 64 : MXM_DUAL_TILE));
}

// LPT key of one m-tile group: the measured cost (mxm_profile_tile_costs, "pre-profiled ... costs") when the
// layer carries one, else an analytic estimate (MMA cycles at the kind's rate vs operand bytes over a per-SM feed)
__device__ __forceinline__ float tile_cost(const ExpertDesc& e, int d, int nt) {
  const int ni = pow2_index(nt);
  if (e.cost[ni] > 0.f) return e.cost[ni] * 1e6f;  // ms -> ns-scale units; only the order matters
  const LinDesc& g = e.blk[0];
  const float rate = kind_is_wa(g.geo.kind) ? 8192.f : 4096.f;  // MAC / cycle / SM
  const float mma = 2.f * 128.f * (float)nt * (float)d / rate;
  const float wbytes = 2.f * 128.f * (float)d * (float)g.geo.w_bits / 8.f;
  const float bbytes = (float)nt * (float)d * (kind_is_wa(g.geo.kind) ? 1.f : 2.f);
  const float mem = (wbytes + bbytes) / 24.f;
  return fmaxf(mma, mem) + 400.f;
}

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(const ExpertDesc* __restrict__ ex, int V, int E, int64_t T,
                                                            int d, const int32_t* __restrict__ v_off, int g_max,
                                                            int64_t task_cap, Task* __restrict__ tasks,
                                                            int32_t* __restrict__ meta, int32_t* __restrict__ grp_n1,
                                                            int32_t* __restrict__ grp_nq, int32_t* __restrict__ p1_done,
                                                            int32_t* __restrict__ hq_done, int32_t* __restrict__ red_cnt) {
  __shared__ int s_cap[kMaxV], s_nfull[kMaxV], s_rem[kMaxV], s_base[kMaxV], s_ragid[kMaxV];
  __shared__ float s_cf[kMaxV], s_cr[kMaxV];
  __shared__ int s_order[kMaxV];
  __shared__ int s_G, s_full;
  int32_t* grp_n2 = hq_done;  // per-group down-task count (scratch: hq_done is zeroed after the scan)
  const int tid = threadIdx.x;
  if (tid < V) {
    const ExpertDesc& e = ex[tid];
    int cnt;
    if (tid < E)
      cnt = ((tid + 1 < E) ? v_off[tid + 1] : v_off[V]) - v_off[tid];
    else
      cnt = (int)T;
    const int cap = tile_cap(e);
    int nfull = 0, rem = 0;
    if (cnt > cap) {
      nfull = cnt / cap;
      rem = cnt % cap;
    } else {
      rem = cnt;
    }
    s_cap[tid] = cap;
    s_nfull[tid] = nfull;
    s_rem[tid] = rem;
    s_cf[tid] = tile_cost(e, d, cap);
    s_cr[tid] = rem > 0 ? tile_cost(e, d, pow2_tile(rem)) : 0.f;
  }
  __syncthreads();
  // LPT order (parallel rank sort, V <= 256): experts with full tiles by full-tile cost desc (ties: lower
  // id) form the first groups; then every ragged / small group ordered by its own cost desc
  if (tid < V) {
    const int v = tid;
    int rf = 0, rr = 0;
    for (int u = 0; u < V; ++u) {
      if (s_nfull[u] > 0 && (s_cf[u] > s_cf[v] || (s_cf[u] == s_cf[v] && u < v))) ++rf;
      if (s_rem[u] > 0 && (s_cr[u] > s_cr[v] || (s_cr[u] == s_cr[v] && u < v))) ++rr;
    }
    s_order[v] = (s_nfull[v] > 0) ? rf : -1;  // rank among experts with full tiles
    s_ragid[v] = (s_rem[v] > 0) ? rr : -1;    // rank among ragged groups
  }
  __syncthreads();
  if (tid == 0) {
    int rank_to_v[kMaxV];
    int nf = 0, nr = 0;
    for (int v = 0; v < V; ++v) {
      if (s_order[v] >= 0) {
        rank_to_v[s_order[v]] = v;
        ++nf;
      }
      if (s_ragid[v] >= 0) ++nr;
    }
    int base = 0;
    for (int i = 0; i < nf; ++i) {
      s_base[rank_to_v[i]] = base;
      base += s_nfull[rank_to_v[i]];
    }
    s_full = base;
    s_G = base + nr;
  }
  __syncthreads();
  if (tid < V && s_ragid[tid] >= 0) s_ragid[tid] += s_full;
  __syncthreads();
  const int G = s_G;
  if (G > g_max) {
    if (tid == 0) meta[0] = -1;  // capacity error (host sizes the workspace so this cannot happen)
    return;
  }
  // group table (row0 | rows | nt | v) in the tail of `tasks`'s companion arrays: store in meta-relative arrays
  int32_t* grp_v = meta + 8;
  int32_t* grp_row0 = grp_v + g_max;
  int32_t* grp_rows = grp_row0 + g_max;
  int32_t* grp_nt = grp_rows + g_max;
  if (tid < V) {
    const int v = tid;
    const ExpertDesc& e = ex[v];
    // h-quant pass only for per-token W-A downs (g128 downs are quantized in the gate/up epilogue)
    const bool wa_down = kind_is_wa(e.blk[2].geo.kind) && e.blk[2].geo.group != 128;
    for (int i = 0; i < s_nfull[v]; ++i) {
      const int g = s_base[v] + i;
      grp_v[g] = v;
      grp_row0[g] = v_off[v] + i * s_cap[v];
      grp_rows[g] = s_cap[v];
      grp_nt[g] = s_cap[v];
      grp_n1[g] = e.inter / 128;
      grp_nq[g] = wa_down ? (s_cap[v] + 31) / 32 : 0;
      grp_n2[g] = down_tasks(e, s_cap[v], d / 128);
    }
    if (s_rem[v] > 0) {
      const int g = s_ragid[v];
      grp_v[g] = v;
      grp_row0[g] = v_off[v] + s_nfull[v] * s_cap[v];
      grp_rows[g] = s_rem[v];
      grp_nt[g] = pow2_tile(s_rem[v]);
      grp_n1[g] = e.inter / 128;
      grp_nq[g] = wa_down ? (s_rem[v] + 31) / 32 : 0;
      grp_n2[g] = down_tasks(e, pow2_tile(s_rem[v]), d / 128);
    }
  }
  __syncthreads();
  for (int g = tid; g < G; g += kPlanThreads) p1_done[g] = 0;
  // prefix sums of per-group task counts (3 phases); each thread owns a contiguous gid range
  const int per = (G + kPlanThreads - 1) / kPlanThreads;
  const int g0 = min(G, tid * per), g1 = min(G, g0 + per);
  int c1 = 0, cq = 0, c2 = 0;
  for (int g = g0; g < g1; ++g) {
    c1 += grp_n1[g];
    cq += grp_nq[g];
    c2 += grp_n2[g];
  }
  __shared__ int s_wt[32];
  int t1, tq, t2;
  // phase totals (the per-group offsets are scanned again per emission round below)
  block_excl_scan(c1, s_wt, &t1);
  block_excl_scan(cq, s_wt, &tq);
  block_excl_scan(c2, s_wt, &t2);
  // split-K of the downs when they cannot fill the SMs (common.cuh); red_cnt == nullptr: not allowed.
  // One slice count S for every splittable down of the launch (the last-arriver reduce counts S arrivals), so
  // S must give every splittable expert a non-empty last slice (experts may differ in ns: shared_inter != inter)
  // and the shortest one at least 2 stages.
  __shared__ int s_minns, s_ok;
  if (tid == 0) s_minns = 1 << 30;
  __syncthreads();
  const bool splittable_v = tid < V && down_splittable(ex[tid]);
  if (splittable_v) atomicMin(&s_minns, ex[tid].blk[2].geo.ns);
  __syncthreads();
  int S = 1;
  if (red_cnt != nullptr && t2 > 0 && t2 < kNumSms && s_minns < (1 << 30)) {
    for (S = min(kSplitMax, (kNumSms + t2 - 1) / t2); S > 1; --S) {
      if (tid == 0) s_ok = 1;
      __syncthreads();
      if (splittable_v) {
        int a, b;
        split_range(ex[tid].blk[2].geo.ns, S, S - 1, a, b);
        const int need = ex[tid].blk[2].geo.ns == s_minns ? 2 : 1;
        if (b - a < need) atomicAnd(&s_ok, 0);
      }
      __syncthreads();
      const int ok = s_ok;
      __syncthreads();
      if (ok) break;
    }
  }
  if (S > 1) {
    const int nd = d / 128;
    c2 = 0;
    for (int g = g0; g < g1; ++g) {
      if (down_splittable(ex[grp_v[g]])) grp_n2[g] *= S;
      c2 += grp_n2[g];
    }
    block_excl_scan(c2, s_wt, &t2);
    for (int i = tid; i < G * nd; i += kPlanThreads) red_cnt[i] = 0;
  }
  const int64_t total = (int64_t)t1 + tq + t2;
  if (tid == 0) {
    meta[0] = total <= task_cap ? (int32_t)total : -1;
    meta[1] = t1;
    meta[2] = tq;
    meta[3] = t2;
    meta[4] = G;
    meta[5] = 0;  // queue head
    meta[6] = 0;  // executed-task counter (debug)
    meta[7] = S;  // split-K slices of splittable down tasks
  }
  if (total > task_cap) return;
  // emission in rounds of kPlanThreads consecutive groups, one per thread (per-round scans give each group's
  // offsets; the queue is the same as a per-thread contiguous range would write): consecutive lanes own
  // consecutive m-tiles, so the n-tile-major blocks of large experts are written as contiguous 512-B runs
  int64_t b1 = 0, bq = 0, b2 = 0;  // tasks of the groups of earlier rounds, per phase
  for (int r0 = 0; r0 < G; r0 += kPlanThreads) {
    const int g = r0 + tid;
    const bool own = g < G;
    int rt1, rtq, rt2;
    const int x1 = block_excl_scan(own ? grp_n1[g] : 0, s_wt, &rt1);
    const int xq = block_excl_scan(own ? grp_nq[g] : 0, s_wt, &rtq);
    const int x2 = block_excl_scan(own ? grp_n2[g] : 0, s_wt, &rt2);
    if (own) {
      int64_t o1 = b1 + x1, oq = (int64_t)t1 + bq + xq, o2 = (int64_t)t1 + tq + b2 + x2;
      Task t;
      const int v = grp_v[g];
      t.expert = (uint16_t)v;
      t.row0 = grp_row0[g];
      t.rows = (uint16_t)grp_rows[g];
      t.nt = (uint8_t)grp_nt[g];
      t.gid = g;
      // an expert with many full m-tiles (e.g. a shared expert over all T tokens) is emitted n-tile-major
      // within its (contiguous) block of full groups: CTAs running side by side then share one weight tile
      // in L2 and stream different token tiles, instead of sharing a token tile and each streaming its own
      // weight tile (a large expert's weights do not fit in L2 and were re-read from HBM per m-tile)
      // A shared expert over all T tokens has more input rows than L2 holds next to the other experts' traffic
      // (Qwen2-57B: 16384 x 3584 codes for gate/up, 16384 x 20480 h codes for the down), so its m-tiles are
      // banded: n-tile-major within bands of m-tiles whose rows fit in MXM_BAND_MB (band_groups)
      const int nf = s_nfull[v], i = g - s_base[v];
      const bool nmajor = MXM_NMAJOR_MIN_GROUPS > 0 && nf >= MXM_NMAJOR_MIN_GROUPS && i >= 0 && i < nf;
      const int n1 = grp_n1[g], n2 = grp_n2[g];
      const ExpertDesc& ev = ex[v];
      const int64_t rb1 = (int64_t)d * (ev.blk[0].in_slot == 0 ? 2 : 1) +
                          (ev.blk[1].in_slot != ev.blk[0].in_slot ? (int64_t)d * (ev.blk[1].in_slot == 0 ? 2 : 1) : 0);
      const int64_t rb2 = (int64_t)ev.inter * (ev.blk[2].in_slot == 0 ? 2 : 1);
      const int B1 = band_groups(rb1, t.nt, nf), B2 = band_groups(rb2, t.nt, nf);
      t.phase = 0;
      for (int j = 0; j < n1; ++j) {
        t.ntile = (uint16_t)j;
        st_task(&tasks[nmajor ? o1 - (int64_t)i * n1 + band_pos(i, j, nf, n1, B1) : o1 + j], t);
      }
      o1 += n1;
      t.phase = 1;
      for (int j = 0; j < grp_nq[g]; ++j) {
        t.ntile = (uint16_t)j;  // 32-row sub-chunk index
        st_task(&tasks[oq++], t);
      }
      t.phase = 2;
      const int S_g = (S > 1 && down_splittable(ex[v])) ? S : 1;
      for (int j = 0; j < n2; ++j) {
        t.ntile = (uint16_t)((j / S_g) | ((j % S_g) << 10));  // down tile (or pair) index | K-slice << 10
        st_task(&tasks[nmajor ? o2 - (int64_t)i * n2 + band_pos(i, j, nf, n2, B2) : o2 + j], t);
      }
      o2 += n2;
    }
    b1 += rt1;
    bq += rtq;
    b2 += rt2;
  }
  __syncthreads();  // every thread has read its grp_n2 entries before the scratch is cleared
  for (int g = tid; g < G; g += kPlanThreads) hq_done[g] = 0;
}

cudaError_t launch_plan(const ExpertDesc* ex, int V, int E, int64_t T, int d, const int32_t* v_off, int g_max,
                        int64_t task_cap, Task* tasks, int32_t* meta, int32_t* grp_n1, int32_t* grp_nq,
                        int32_t* p1_done, int32_t* hq_done, int32_t* red_cnt, cudaStream_t st) {
  if (V > kMaxV) return cudaErrorInvalidValue;
  plan_kernel<<<1, kPlanThreads, 0, st>>>(ex, V, E, T, d, v_off, g_max, task_cap, tasks, meta, grp_n1, grp_nq, p1_done,
                                          hq_done, red_cnt);
  return cudaGetLastError();
}

}  // namespace mxm
