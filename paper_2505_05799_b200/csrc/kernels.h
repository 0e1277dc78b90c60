// kernels.h — host-callable launchers of the device kernels (internal to libmxmoe).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "common.cuh"

namespace mxm {

struct GemmParams {
  // B sources {Xb, XqA, XqB, H routed, Hq routed, H shared, Hq shared} x token tile {16, 32, 64, 96}
  CUtensorMap tmap[7][4];
  const ExpertDesc* ex;
  const Task* tasks;
  int32_t* meta;  // [0] n_tasks, [5] queue head, [6] executed tasks
  int32_t* p1_done;
  int32_t* hq_done;
  const int32_t* grp_n1;
  const int32_t* grp_nq;
  const float* xs[3];  // activation scales of the gate/up input slots (index 1, 2), group-major [g][R]
  const int32_t* xc[3];  // code sums of the gate/up input slots (index 1, 2), group-major [g][R] (w4a4 correction)
  int32_t* Hc;           // code sums of h, group-major [g][R]
  uint16_t* H;
  int8_t* Hq;
  float* Hs;           // h scales, group-major [g][R]
  int64_t hs_stride;   // R: rows of the workspace (stride between activation-scale groups)
  uint32_t* hmax;  // per route row: max |h| (fp32 bits) for per-token W-A downs (order-independent atomicMax)
  uint16_t* O;
  const float* row_w;
  float* P;          // split-K fp32 partials [kSplitMax][kSplitRows][d] (nullptr: no split-K this launch)
  int32_t* red_cnt;  // split-K arrival counters [group][d/128]
  int d, f_max;
  // H / Hq rows in two regions: shared rows [0, h_srows) at row stride f_s, then routed rows at stride f_r
  // (element offset of the routed region h_rbase = h_srows * f_s); gemm.cu h_off
  int64_t h_srows, h_rbase;
  int f_s, f_r;
  unsigned long long* prof;  // optional [grid][16] cycle counters per wait site (nullptr = off)
  // test-only accumulator dump (mxm_debug_moe_group_gemm_dump; nullptr in the product launch): the raw 32-bit
  // accumulator of every weight-activation drain event (layout: gemm.cu dump_index)
  uint32_t* dump;
};

cudaError_t launch_quantize(const PackGeom& g, const void* w, void* codes, void* scale, void* zero, int32_t* err,
                            cudaStream_t st);
cudaError_t launch_pack(const PackGeom& g, const void* codes, const void* scale, const void* zero, void* out,
                        cudaStream_t st);
cudaError_t launch_dequantize(const PackGeom& g, const void* packed, float* out, cudaStream_t st);
cudaError_t launch_act_quant(const void* v, int64_t M, int64_t K, int a_bits, int group, void* codes, float* scale,
                             int32_t* qsum, cudaStream_t st);

int64_t route_scratch_bytes(int64_t n_routes, int E);
cudaError_t launch_route_prep(const int32_t* ids, const float* topk_w, int64_t T, int k, int E, int S,
                              const float* shared_w, int32_t* counts, int32_t* offsets, int32_t* v_off, int32_t* perm,
                              int32_t* row_src, float* row_w, int32_t* row_exp, int32_t* inv, int32_t* err,
                              void* scratch, cudaStream_t st);
// NEXT-4 offline preparation (gptq.cu)
cudaError_t launch_hadamard(const void* w, void* out, int64_t N, int64_t K, const int8_t* signs, int axis,
                            cudaStream_t st);
cudaError_t launch_gptq_hessian(const void* x, int64_t n, int64_t K, double* H, cudaStream_t st);
cudaError_t launch_gptq_prepare(double* H, int64_t K, double percdamp, double* V, double* U, int32_t* dead,
                                cudaStream_t st);
cudaError_t launch_gptq_quantize(int bits, int group, int sym, const void* w, int64_t N, int64_t K, const double* U,
                                 const int32_t* dead, double* work, void* codes, void* scale, void* zero,
                                 cudaStream_t st);
int64_t gptq_work_doubles(int64_t N, int64_t K);
// distinct gate/up input formats of a layer (token-major gather): a_bits 16 = bf16 copy, else the dynamic
// quantizer's (a_bits, a_group (-1 per token / 128), e4m3 codes)
struct ActFormats {
  int n;
  int a_bits[6], a_group[6], e4[6];
};
cudaError_t launch_gather_tok(const void* x, int d, int64_t T, int k, int S, int E, const int32_t* inv,
                              const int32_t* row_exp, const ExpertDesc* ex, const ActFormats& fm, int64_t R, void* Xb,
                              void* XqA, float* XsA, void* XqB, float* XsB, int32_t* XcA, int32_t* XcB, uint32_t* hmax,
                              cudaStream_t st);
cudaError_t launch_gather_quant(const void* x, int d, const int32_t* row_src, const int32_t* row_exp,
                                const int32_t* v_off, int V, const ExpertDesc* ex, int64_t R, void* Xb, void* XqA,
                                float* XsA, void* XqB, float* XsB, int32_t* XcA, int32_t* XcB, uint32_t* hmax,
                                cudaStream_t st);
cudaError_t launch_combine(const void* O, int d, int64_t T, int k, int S, const int32_t* inv, void* y,
                           cudaStream_t st);
cudaError_t launch_plan(const ExpertDesc* ex, int V, int E, int64_t T, int d, const int32_t* v_off, int g_max,
                        int64_t task_cap, Task* tasks, int32_t* meta, int32_t* grp_n1, int32_t* grp_nq,
                        int32_t* p1_done, int32_t* hq_done, int32_t* red_cnt, cudaStream_t st);
cudaError_t launch_moe_gemm(const GemmParams& prm, int grid, cudaStream_t st);
cudaError_t launch_ep_route(const int32_t* ids, int64_t T, int k, int E, int G, int32_t* dest_counts, int32_t* pos,
                            int32_t* err, cudaStream_t st);
cudaError_t launch_ep_pack(const void* x, int64_t T, int d, const int32_t* ids, const float* w, int k, int E, int G,
                           const int32_t* pos, const int32_t* dest_off, void* sx, int32_t* sids, float* sw,
                           int32_t* ssrc, cudaStream_t st);
cudaError_t launch_ep_fill(int32_t* dest_off, int G, int64_t C, int32_t* sid, float* ones, int64_t T, int S,
                           cudaStream_t st);
cudaError_t launch_ep_combine(const void* back, const int32_t* pos, const int32_t* dest_off, int G, int64_t T, int d,
                              const void* ysh, void* y, cudaStream_t st);

}  // namespace mxm
