// plan.cu — step S3: build the tile task list of one MoE block on the device.
//
// The paper's runtime cost model approximates block time by the serial time of all tiles over the
// SMs and its scheduler "prioritizes computationally intensive tiles" (greedy makespan,
// P:231; Graham's bound). Here: every (expert, m-tile) group contributes f/128 gate+up tiles
// (phase 1), ceil(rows/32) h-quantization sub-tasks when its down block is weight-activation, and
// d/128 down tiles (phase 2). Groups are ordered by estimated per-tile cost, descending (LPT);
// the whole phase-1 list precedes the h-quant list which precedes phase 2, so the dynamic queue
// of the persistent kernel can never deadlock on a dependency.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace mxm {

constexpr int kPlanThreads = 1024;
constexpr int kMaxV = 256;

__device__ __forceinline__ int pow2_tile(int m) {
  return m <= 16 ? 16 : (m <= 32 ? 32 : (m <= 64 ? 64 : 128));
}

__device__ __forceinline__ float tile_cost(const ExpertDesc& e, int d, int nt) {
  const LinDesc& g = e.blk[0];
  const float rate = kind_is_i8(g.geo.kind) ? 8192.f : 4096.f;  // MAC / cycle / SM
  const float mma = 2.f * 128.f * (float)nt * (float)d / rate;
  const float wbytes = 2.f * 128.f * (float)d * (float)g.geo.w_bits / 8.f;
  const float bbytes = (float)nt * (float)d * (kind_is_i8(g.geo.kind) ? 1.f : 2.f);
  const float mem = (wbytes + bbytes) / 24.f;
  return fmaxf(mma, mem) + 400.f;
}

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(const ExpertDesc* __restrict__ ex, int V, int E, int64_t T,
                                                            int d, const int32_t* __restrict__ v_off, int g_max,
                                                            int64_t task_cap, Task* __restrict__ tasks,
                                                            int32_t* __restrict__ meta, int32_t* __restrict__ grp_n1,
                                                            int32_t* __restrict__ grp_nq, int32_t* __restrict__ p1_done,
                                                            int32_t* __restrict__ hq_done) {
  __shared__ int s_cnt[kMaxV], s_cap[kMaxV], s_nfull[kMaxV], s_rem[kMaxV], s_base[kMaxV], s_ragid[kMaxV];
  __shared__ float s_cf[kMaxV], s_cr[kMaxV];
  __shared__ int s_order[kMaxV];
  __shared__ int s_G, s_full;
  __shared__ int64_t s_part[3][kPlanThreads];
  const int tid = threadIdx.x;
  if (tid < V) {
    const ExpertDesc& e = ex[tid];
    int cnt;
    if (tid < E)
      cnt = ((tid + 1 < E) ? v_off[tid + 1] : v_off[V]) - v_off[tid];
    else
      cnt = (int)T;
    const bool reg_dual = !e.same_gu || (kind_is_i8(e.blk[0].geo.kind) && e.blk[0].geo.group == 128);
    const int cap = reg_dual ? 64 : 128;
    int nfull = 0, rem = 0;
    if (cnt > cap) {
      nfull = cnt / cap;
      rem = cnt % cap;
    } else {
      rem = cnt;
    }
    s_cnt[tid] = cnt;
    s_cap[tid] = cap;
    s_nfull[tid] = nfull;
    s_rem[tid] = rem;
    s_cf[tid] = tile_cost(e, d, cap);
    s_cr[tid] = rem > 0 ? tile_cost(e, d, pow2_tile(rem)) : 0.f;
  }
  __syncthreads();
  if (tid == 0) {
    // LPT order: experts with full tiles by full-tile cost desc (ties: lower id), then ragged groups
    int n = 0;
    for (int v = 0; v < V; ++v)
      if (s_nfull[v] > 0) s_order[n++] = v;
    for (int i = 1; i < n; ++i) {  // insertion sort, V <= 256
      const int v = s_order[i];
      int j = i - 1;
      while (j >= 0 && (s_cf[s_order[j]] < s_cf[v] || (s_cf[s_order[j]] == s_cf[v] && s_order[j] > v))) {
        s_order[j + 1] = s_order[j];
        --j;
      }
      s_order[j + 1] = v;
    }
    int base = 0;
    for (int i = 0; i < n; ++i) {
      s_base[s_order[i]] = base;
      base += s_nfull[s_order[i]];
    }
    s_full = base;
    n = 0;
    for (int v = 0; v < V; ++v)
      if (s_rem[v] > 0) s_order[n++] = v;
    for (int i = 1; i < n; ++i) {
      const int v = s_order[i];
      int j = i - 1;
      while (j >= 0 && (s_cr[s_order[j]] < s_cr[v] || (s_cr[s_order[j]] == s_cr[v] && s_order[j] > v))) {
        s_order[j + 1] = s_order[j];
        --j;
      }
      s_order[j + 1] = v;
    }
    for (int i = 0; i < n; ++i) s_ragid[s_order[i]] = base + i;
    s_G = base + n;
  }
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
    const bool wa_down = kind_is_i8(e.blk[2].geo.kind);
    for (int i = 0; i < s_nfull[v]; ++i) {
      const int g = s_base[v] + i;
      grp_v[g] = v;
      grp_row0[g] = v_off[v] + i * s_cap[v];
      grp_rows[g] = s_cap[v];
      grp_nt[g] = s_cap[v];
      grp_n1[g] = e.inter / 128;
      grp_nq[g] = wa_down ? (s_cap[v] + 31) / 32 : 0;
    }
    if (s_rem[v] > 0) {
      const int g = s_ragid[v];
      grp_v[g] = v;
      grp_row0[g] = v_off[v] + s_nfull[v] * s_cap[v];
      grp_rows[g] = s_rem[v];
      grp_nt[g] = pow2_tile(s_rem[v]);
      grp_n1[g] = e.inter / 128;
      grp_nq[g] = wa_down ? (s_rem[v] + 31) / 32 : 0;
    }
  }
  __syncthreads();
  for (int g = tid; g < G; g += kPlanThreads) {
    p1_done[g] = 0;
    hq_done[g] = 0;
  }
  // prefix sums of per-group task counts (3 phases); each thread owns a contiguous gid range
  const int per = (G + kPlanThreads - 1) / kPlanThreads;
  const int g0 = min(G, tid * per), g1 = min(G, g0 + per);
  int64_t c1 = 0, cq = 0, c2 = 0;
  for (int g = g0; g < g1; ++g) {
    c1 += grp_n1[g];
    cq += grp_nq[g];
    c2 += d / 128;
  }
  s_part[0][tid] = c1;
  s_part[1][tid] = cq;
  s_part[2][tid] = c2;
  __syncthreads();
  if (tid == 0) {
    int64_t r[3] = {0, 0, 0};
    for (int i = 0; i < kPlanThreads; ++i)
      for (int p = 0; p < 3; ++p) {
        const int64_t v = s_part[p][i];
        s_part[p][i] = r[p];
        r[p] += v;
      }
    const int64_t total = r[0] + r[1] + r[2];
    meta[0] = total <= task_cap ? (int32_t)total : -1;
    meta[1] = (int32_t)r[0];
    meta[2] = (int32_t)r[1];
    meta[3] = (int32_t)r[2];
    meta[4] = G;
    meta[5] = 0;  // queue head
    meta[6] = 0;  // executed-task counter (debug)
    s_part[1][kPlanThreads - 1] += 0;
    s_G = (int)r[0];
    s_full = (int)(r[0] + r[1]);
  }
  __syncthreads();
  if (meta[0] < 0) return;
  int64_t o1 = s_part[0][tid], oq = (int64_t)s_G + s_part[1][tid], o2 = (int64_t)s_full + s_part[2][tid];
  for (int g = g0; g < g1; ++g) {
    Task t;
    t.expert = (uint16_t)grp_v[g];
    t.row0 = grp_row0[g];
    t.rows = (uint16_t)grp_rows[g];
    t.nt = (uint8_t)grp_nt[g];
    t.gid = g;
    t.phase = 0;
    for (int j = 0; j < grp_n1[g]; ++j) {
      t.ntile = (uint16_t)j;
      tasks[o1++] = t;
    }
    t.phase = 1;
    for (int j = 0; j < grp_nq[g]; ++j) {
      t.ntile = (uint16_t)j;  // 32-row sub-chunk index
      tasks[oq++] = t;
    }
    t.phase = 2;
    for (int j = 0; j < d / 128; ++j) {
      t.ntile = (uint16_t)j;
      tasks[o2++] = t;
    }
  }
}

cudaError_t launch_plan(const ExpertDesc* ex, int V, int E, int64_t T, int d, const int32_t* v_off, int g_max,
                        int64_t task_cap, Task* tasks, int32_t* meta, int32_t* grp_n1, int32_t* grp_nq,
                        int32_t* p1_done, int32_t* hq_done, cudaStream_t st) {
  if (V > kMaxV) return cudaErrorInvalidValue;
  plan_kernel<<<1, kPlanThreads, 0, st>>>(ex, V, E, T, d, v_off, g_max, task_cap, tasks, meta, grp_n1, grp_nq, p1_done,
                                          hq_done);
  return cudaGetLastError();
}

}  // namespace mxm
