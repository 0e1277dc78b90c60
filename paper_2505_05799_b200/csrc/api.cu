// api.cu — the C ABI (include/mxmoe.h): host-side validation, layer descriptor table, workspace
// carving, TMA tensor maps and the launch sequence of the hot path (S1 route-prep -> S2 act-quant
// + gather -> S3 plan -> S4-S7 persistent group-GEMM -> S8 combine), all on the caller's stream.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mxmoe.h"
#include "common.cuh"
#include "kernels.h"

using namespace mxm;

namespace {
thread_local std::string g_err;

mxm_status fail(mxm_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
mxm_status cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return MXM_E_CUDA;
}
#define MXM_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool encode_2d(CUtensorMap* m, const void* base, bool bf16, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const uint32_t esz = bf16 ? 2 : 1;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * esz};
  cuuint32_t box[2] = {128u / esz, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
                  const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// SM count of the current device (cached per device ordinal)
int num_sms() {
  static std::mutex mu;
  static int n[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return kNumSms;
  std::lock_guard<std::mutex> lk(mu);
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : kNumSms;
  }
  return n[dev];
}

int64_t align256(int64_t x) { return (x + 255) / 256 * 256; }
// A/B switch from the environment (e.g. MXM_GATHER_ROWS=1: the row-major S2 gather)
bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && *v && *v != '0';
}
}  // namespace

struct mxm_layer {
  int E, S, V, d, f, fs, f_max;
  int device;  // CUDA device of the descriptor table (calls must run with it current)
  std::vector<ExpertDesc> ex;
  ExpertDesc* ex_dev;
  bool need_xb, need_xqa, need_xqb, need_hq;
  ActFormats fm;  // distinct gate/up input formats (token-major gather); fm.n = 0: row-major gather
  // optional per-stage timing: kProfEv events per slot recorded around the launches of a call
  int prof_n = 0;
  void* prof_counters = nullptr;  // device [grid][16] u64 wait-site cycle counters (debug)
  int64_t prof_calls = 0;
  std::vector<cudaEvent_t> prof_ev;
  // S3 (plan) depends only on S1's offsets, so it runs on a side stream concurrently with S2 (gather):
  // fork / join with events on the caller's stream (graph-capturable); created on first use
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::mutex side_mu;  // the fork / join events are per layer: concurrent calls serialise this section
  // tensor maps of the token-tile operands of the last call (guarded by side_mu): re-encoded only when the
  // workspace, T or top_k change (20 cuTensorMapEncodeTiled calls cost tens of us, a tenth of a T = 1 step)
  const void* tm_ws = nullptr;
  int64_t tm_T = -1;
  int tm_k = 0;
  CUtensorMap tm[7][4];
  ~mxm_layer() {
    for (auto e : prof_ev) cudaEventDestroy(e);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
  }
};
static constexpr int kProfEv = 6;  // start | route | gather | plan | gemm | combine

// workspace layout for T tokens, k routes
struct WsLayout {
  int64_t R, g_max, task_cap;
  int64_t err, route_scratch, counts, v_off, row_src, row_w, row_exp, inv;
  int64_t Xb, XqA, XsA, XqB, XsB, H, Hq, Hs, hmax, O;
  int64_t XcA, XcB, Hc;  // per-(group, row) code sums of e4m3-coded (w4a4) inputs, group-major [g][R] int32
  int64_t tasks, meta, grp_n1, grp_nq, p1_done, hq_done, P, red_cnt;
  int64_t total;
};

static WsLayout make_layout(const mxm_layer* l, int64_t T, int k) {
  WsLayout w{};
  const int64_t R = T * k + T * l->S;
  w.R = R;
  w.g_max = (R + 15) / 16 + l->V + 1;
  w.task_cap = w.g_max * (l->f_max / 128 + 4 + l->d / 128);
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    int64_t at = o;
    o += align256(bytes > 0 ? bytes : 1);
    return at;
  };
  w.err = take(256);
  w.route_scratch = take(route_scratch_bytes(T * k, l->E));
  w.counts = take(4 * (l->E + 1));
  w.v_off = take(4 * (l->V + 1));
  w.row_src = take(4 * R);
  w.row_w = take(4 * R);
  w.row_exp = take(4 * R);
  w.inv = take(4 * T * k);
  w.Xb = l->need_xb ? take(2 * R * l->d) : -1;
  w.XqA = l->need_xqa ? take(R * l->d) : -1;
  w.XsA = l->need_xqa ? take(4 * R * (l->d / 128)) : -1;
  w.XqB = l->need_xqb ? take(R * l->d) : -1;
  w.XsB = l->need_xqb ? take(4 * R * (l->d / 128)) : -1;
  // h rows in two regions (gemm.cu h_off): the T*S shared rows at the shared width, the T*k routed rows at the
  // routed width (R x max width would hold 4.5x the bytes at Qwen2-57B: f_s 20480 vs f 2560)
  const int64_t h_elems = T * l->S * l->fs + T * k * l->f;
  w.H = take(2 * h_elems);
  w.Hq = l->need_hq ? take(h_elems) : -1;
  w.Hs = l->need_hq ? take(4 * R * (l->f_max / 128)) : -1;
  w.hmax = l->need_hq ? take(4 * R) : -1;
  w.XcA = l->need_xqa ? take(4 * R * (l->d / 128)) : -1;
  w.XcB = l->need_xqb ? take(4 * R * (l->d / 128)) : -1;
  w.Hc = l->need_hq ? take(4 * R * (l->f_max / 128)) : -1;
  w.O = take(2 * R * l->d);
  w.tasks = take(16 * w.task_cap);
  w.meta = take(4 * (8 + 4 * w.g_max));
  w.grp_n1 = take(4 * w.g_max);
  w.grp_nq = take(4 * w.g_max);
  w.p1_done = take(4 * w.g_max);
  w.hq_done = take(4 * w.g_max);
  const bool split = R <= kSplitRows;  // split-K only at tiny T (bounded partial buffer)
  w.P = split ? take((int64_t)4 * kSplitMax * kSplitRows * l->d) : -1;
  w.red_cnt = split ? take(4 * w.g_max * (l->d / 128)) : -1;
  w.total = o;
  return w;
}

extern "C" {

const char* mxm_last_error(void) { return g_err.c_str(); }
const char* mxm_version(void) { return "mxmoe-b200 0.1 (sm_100a)"; }

mxm_status mxm_scheme_check(const mxm_scheme* s, int64_t N, int64_t K) {
  if (!s) return fail(MXM_E_CONFIG, "null scheme");
  PackGeom g;
  if (make_geom(*s, N, K, &g) != MXM_OK) return fail(MXM_E_CONFIG, "unsupported scheme/shape");
  return MXM_OK;
}

mxm_status mxm_quant_sizes(const mxm_scheme* s, int64_t N, int64_t K, int64_t* codes_bytes, int64_t* scale_bytes,
                           int64_t* zero_bytes, int64_t* packed_bytes) {
  if (!s) return fail(MXM_E_CONFIG, "null scheme");
  PackGeom g;
  if (make_geom(*s, N, K, &g) != MXM_OK) return fail(MXM_E_CONFIG, "unsupported scheme/shape");
  const int64_t ng = K / g.group;
  if (codes_bytes) *codes_bytes = s->w_bits == 16 ? N * K * 2 : N * K;
  if (scale_bytes) *scale_bytes = s->w_bits == 16 ? 0 : N * ng * 2;
  if (zero_bytes) *zero_bytes = (s->w_bits == 16 || g.sym) ? 0 : N * ng * 2;
  if (packed_bytes) *packed_bytes = g.total_bytes;
  return MXM_OK;
}

double mxm_storage_bits_per_weight(const mxm_scheme* s, int64_t K) {
  if (!s) return 0.0;
  if (s->w_bits == 16) return 16.0;
  const double g = s->w_group == -1 ? (double)K : (double)s->w_group;
  const bool sym = s->symmetric || s->a_bits != 16;
  return s->w_bits + (sym ? 1.0 : 2.0) * 16.0 / g;
}

mxm_status mxm_quantize(const mxm_scheme* s, const void* w, int64_t N, int64_t K, void* codes, void* scale, void* zero,
                        int32_t* err, mxm_stream stream) {
  if (!s || !w || !codes || !scale) return fail(MXM_E_CONFIG, "null argument");
  if (s->w_bits == 16) return fail(MXM_E_CONFIG, "w16 has nothing to quantize");
  PackGeom g;
  if (make_geom(*s, N, K, &g) != MXM_OK) return fail(MXM_E_CONFIG, "unsupported scheme/shape");
  if (!g.sym && !zero) return fail(MXM_E_CONFIG, "asymmetric scheme needs a zero buffer");
  MXM_CUDA(launch_quantize(g, w, codes, scale, zero, err, (cudaStream_t)stream));
  return MXM_OK;
}

// ---------------------------------------------------------------- NEXT-4 offline preparation (gptq.cu)
mxm_status mxm_hadamard_rotate(const void* w, void* out, int64_t N, int64_t K, const int8_t* signs, int32_t axis,
                               mxm_stream stream) {
  if (!w || !out || !signs) return fail(MXM_E_CONFIG, "null argument");
  if (N <= 0 || K <= 0 || (axis != 0 && axis != 1)) return fail(MXM_E_CONFIG, "bad shape / axis");
  if ((axis == 1 ? K : N) % 128 != 0) return fail(MXM_E_CONFIG, "rotated dimension must be a multiple of 128");
  if (w == out) return fail(MXM_E_CONFIG, "in-place rotation is not supported");
  MXM_CUDA(launch_hadamard(w, out, N, K, signs, axis, (cudaStream_t)stream));
  return MXM_OK;
}

mxm_status mxm_gptq_hessian(const void* x, int64_t n, int64_t K, double* H, mxm_stream stream) {
  if (!x || !H) return fail(MXM_E_CONFIG, "null argument");
  if (n <= 0 || K <= 0) return fail(MXM_E_CONFIG, "bad shape");
  MXM_CUDA(launch_gptq_hessian(x, n, K, H, (cudaStream_t)stream));
  return MXM_OK;
}

mxm_status mxm_gptq_prepare(double* H, int64_t K, double percdamp, double* scratch, double* U, int32_t* dead,
                            mxm_stream stream) {
  if (!H || !scratch || !U || !dead) return fail(MXM_E_CONFIG, "null argument");
  if (K <= 0 || !(percdamp >= 0.0)) return fail(MXM_E_CONFIG, "bad K / damping");
  MXM_CUDA(launch_gptq_prepare(H, K, percdamp, scratch, U, dead, (cudaStream_t)stream));
  return MXM_OK;
}

int64_t mxm_gptq_work_bytes(int64_t N, int64_t K) { return 8 * gptq_work_doubles(N, K); }

mxm_status mxm_gptq_quantize(const mxm_scheme* s, const void* w, int64_t N, int64_t K, const double* U,
                             const int32_t* dead, double* work, void* codes, void* scale, void* zero,
                             mxm_stream stream) {
  if (!s || !w || !U || !dead || !work || !codes || !scale) return fail(MXM_E_CONFIG, "null argument");
  if (s->w_bits == 16) return fail(MXM_E_CONFIG, "w16 has nothing to quantize");
  PackGeom g;
  if (make_geom(*s, N, K, &g) != MXM_OK) return fail(MXM_E_CONFIG, "unsupported scheme/shape");
  if (s->w_group != -1 && s->w_group != 64 && s->w_group != 128) return fail(MXM_E_CONFIG, "group must be 64 / 128 / -1");
  if (!g.sym && !zero) return fail(MXM_E_CONFIG, "asymmetric scheme needs a zero buffer");
  MXM_CUDA(launch_gptq_quantize(s->w_bits, s->w_group, g.sym ? 1 : 0, w, N, K, U, dead, work, codes, scale, zero,
                                (cudaStream_t)stream));
  return MXM_OK;
}

mxm_status mxm_pack(const mxm_scheme* s, const void* codes, const void* scale, const void* zero, int64_t N, int64_t K,
                    void* packed, mxm_stream stream) {
  if (!s || !codes || !packed) return fail(MXM_E_CONFIG, "null argument");
  PackGeom g;
  if (make_geom(*s, N, K, &g) != MXM_OK) return fail(MXM_E_CONFIG, "unsupported scheme/shape");
  if (s->w_bits != 16 && !scale) return fail(MXM_E_CONFIG, "null scale");
  if (g.kind == KIND_WO && !g.sym && !zero) return fail(MXM_E_CONFIG, "null zero");
  MXM_CUDA(launch_pack(g, codes, scale, zero, packed, (cudaStream_t)stream));
  return MXM_OK;
}

mxm_status mxm_dequantize(const mxm_scheme* s, const void* packed, int64_t N, int64_t K, float* out,
                          mxm_stream stream) {
  if (!s || !packed || !out) return fail(MXM_E_CONFIG, "null argument");
  PackGeom g;
  if (make_geom(*s, N, K, &g) != MXM_OK) return fail(MXM_E_CONFIG, "unsupported scheme/shape");
  MXM_CUDA(launch_dequantize(g, packed, out, (cudaStream_t)stream));
  return MXM_OK;
}

mxm_status mxm_act_quant(const void* v, int64_t M, int64_t K, int32_t a_bits, int32_t a_group, void* codes,
                         float* scale, int32_t* qsum, mxm_stream stream) {
  if (!v || !codes || !scale) return fail(MXM_E_CONFIG, "null argument");
  if (!(a_bits == 4 || a_bits == 5 || a_bits == 8)) return fail(MXM_E_CONFIG, "a_bits must be 4, 5 or 8");
  const int64_t g = a_group == -1 ? K : a_group;
  if (M < 0 || K <= 0 || K % 128 != 0 || !(a_group == -1 || a_group == 128)) return fail(MXM_E_CONFIG, "bad shape");
  if (M == 0) return MXM_OK;
  MXM_CUDA(launch_act_quant(v, M, K, a_bits, (int)g, codes, scale, qsum, (cudaStream_t)stream));
  return MXM_OK;
}

mxm_status mxm_route_scratch_bytes(int64_t T, int32_t k, int32_t E, int64_t* bytes) {
  if (!bytes || E <= 0 || E > 256 || k <= 0 || k > 32 || T < 0) return fail(MXM_E_CONFIG, "bad E/k/T");
  *bytes = route_scratch_bytes(T * k, E);
  return MXM_OK;
}

mxm_status mxm_route_prep(const int32_t* topk_ids, int64_t T, int32_t k, int32_t E, int32_t* counts, int32_t* offsets,
                          int32_t* perm, int32_t* err, void* scratch, int64_t scratch_bytes, mxm_stream stream) {
  if (!topk_ids || !counts || !offsets || !perm) return fail(MXM_E_CONFIG, "null argument");
  if (E <= 0 || E > 256 || k <= 0 || k > 32 || T < 0) return fail(MXM_E_CONFIG, "bad E/k/T");
  if (scratch_bytes < route_scratch_bytes(T * k, E)) return fail(MXM_E_CONFIG, "scratch too small");
  MXM_CUDA(launch_route_prep(topk_ids, nullptr, T, k, E, 0, nullptr, counts, offsets, nullptr, perm, nullptr, nullptr,
                             nullptr, nullptr, err, scratch, (cudaStream_t)stream));
  return MXM_OK;
}

mxm_status mxm_layer_desc_bytes(const mxm_layer_desc* d, int64_t* bytes) {
  if (!d || !bytes) return fail(MXM_E_CONFIG, "null argument");
  *bytes = (int64_t)sizeof(ExpertDesc) * (d->n_routed + d->n_shared);
  return MXM_OK;
}

mxm_status mxm_layer_init(const mxm_layer_desc* d, void* desc_dev, int64_t desc_bytes, const void* tile_costs,
                          mxm_layer** out) {
  if (!d || !d->blocks || !desc_dev || !out) return fail(MXM_E_CONFIG, "null argument");
  const int E = d->n_routed, S = d->n_shared, V = E + S;
  if (E <= 0 || E > 256 || S < 0 || S > 32 || V > 256) return fail(MXM_E_CONFIG, "expert count out of range");
  if (d->hidden <= 0 || d->hidden % 128 || d->inter <= 0 || d->inter % 128) return fail(MXM_E_CONFIG, "hidden/inter % 128");
  if (S > 0 && (d->shared_inter <= 0 || d->shared_inter % 128)) return fail(MXM_E_CONFIG, "shared_inter % 128");
  if (desc_bytes < (int64_t)sizeof(ExpertDesc) * V) return fail(MXM_E_CONFIG, "descriptor buffer too small");
  auto* l = new mxm_layer();
  l->E = E;
  l->S = S;
  l->V = V;
  l->d = d->hidden;
  l->f = d->inter;
  l->fs = S > 0 ? d->shared_inter : 0;
  l->f_max = l->f > l->fs ? l->f : l->fs;
  l->need_xb = l->need_xqa = l->need_xqb = l->need_hq = false;
  l->ex.resize(V);
  for (int v = 0; v < V; ++v) {
    ExpertDesc& e = l->ex[v];
    memset(&e, 0, sizeof(e));
    const int f = v < E ? l->f : l->fs;
    e.inter = f;
    e.shared = v >= E;
    for (int j = 0; j < 3; ++j) {
      const mxm_linear& b = d->blocks[v * 3 + j];
      const int64_t N = j < 2 ? f : l->d, K = j < 2 ? l->d : f;
      if (!b.packed) {
        delete l;
        return fail(MXM_E_CONFIG, "null packed block");
      }
      PackGeom g;
      if (make_geom(b.scheme, N, K, &g) != MXM_OK) {
        delete l;
        char buf[160];
        snprintf(buf, sizeof buf, "expert %d block %d: unsupported scheme w%d a%d g%d for [%lld, %lld]", v, j,
                 b.scheme.w_bits, b.scheme.a_bits, b.scheme.w_group, (long long)N, (long long)K);
        return fail(MXM_E_CONFIG, buf);
      }
      if (g.kind == KIND_FP8 && j < 2 && l->d > 4096) {  // the FP8 input quantizer keeps the row in registers
        delete l;
        return fail(MXM_E_CONFIG, "FP8 gate/up blocks need hidden <= 4096");
      }
      e.blk[j].packed = reinterpret_cast<const uint8_t*>(b.packed);
      e.blk[j].geo = g;
      e.blk[j].a_bits = b.scheme.a_bits;
      e.blk[j].a_group = b.scheme.a_bits == 16 ? -1 : b.scheme.a_group;
    }
    const mxm_scheme& sg = d->blocks[v * 3 + 0].scheme;
    const mxm_scheme& su = d->blocks[v * 3 + 1].scheme;
    // input slots
    const bool gwa = sg.a_bits != 16, uwa = su.a_bits != 16;
    e.blk[0].in_slot = gwa ? 1 : 0;
    if (!uwa)
      e.blk[1].in_slot = 0;
    else if (gwa && sg.a_bits == su.a_bits && e.blk[0].a_group == e.blk[1].a_group && sg.fmt == su.fmt)
      e.blk[1].in_slot = 1;
    else
      e.blk[1].in_slot = gwa ? 2 : 1;
    e.blk[2].in_slot = d->blocks[v * 3 + 2].scheme.a_bits != 16 ? 1 : 0;
    // gate and up share one K loop (and the token tile) when they use the same MMA kind and input:
    // any two bf16-kind blocks (w16 / weight-only of any bits and group), or identical W-A schemes
    e.dual = (!gwa && !uwa) || (gwa && uwa && e.blk[1].in_slot == 1 && sg.w_bits == su.w_bits &&
                                sg.w_group == su.w_group && sg.fmt == su.fmt);
    for (int j = 0; j < 2; ++j) {
      if (e.blk[j].in_slot == 0) l->need_xb = true;
      if (e.blk[j].in_slot == 1) l->need_xqa = true;
      if (e.blk[j].in_slot == 2) l->need_xqb = true;
    }
    if (e.blk[2].in_slot == 1) l->need_hq = true;
  }
  // distinct gate/up input formats: the token-major gather quantizes each token once per format
  {
    ActFormats fm{};
    bool ok = l->d % 128 == 0 && l->d <= 4096 && S <= 8;
    for (int v = 0; v < V && ok; ++v) {
      for (int j = 0; j < 2 && ok; ++j) {
        const LinDesc& L = l->ex[v].blk[j];
        const int b = L.in_slot == 0 ? 16 : L.a_bits, g = L.in_slot == 0 ? 0 : L.a_group;
        const int e4 = L.in_slot == 0 ? 0 : (kind_is_fp8(L.geo.kind) ? 2 : (kind_is_w4a4(L.geo.kind) ? 1 : 0));
        if (L.in_slot != 0 && g != 128 && g != -1) ok = false;
        int i = 0;
        while (i < fm.n && !(fm.a_bits[i] == b && fm.a_group[i] == g && fm.e4[i] == e4)) ++i;
        if (i == fm.n) {
          if (fm.n == 6) {
            ok = false;
          } else {
            fm.a_bits[i] = b;
            fm.a_group[i] = g;
            fm.e4[i] = e4;
            ++fm.n;
          }
        }
      }
    }
    if (!ok) fm.n = 0;
    l->fm = fm;
  }
  if (tile_costs) {  // measured per-(expert, token tile) m-tile group costs (mxm_profile_tile_costs), ms
    const float* c = reinterpret_cast<const float*>(tile_costs);
    for (int v = 0; v < V; ++v)
      for (int i = 0; i < 4; ++i) l->ex[v].cost[i] = c[v * 4 + i] > 0.f ? c[v * 4 + i] : 0.f;
  }
  cudaError_t ce = cudaMemcpy(desc_dev, l->ex.data(), sizeof(ExpertDesc) * V, cudaMemcpyHostToDevice);
  if (ce != cudaSuccess) {
    delete l;
    return cuda_fail(ce, "cudaMemcpy(desc)");
  }
  l->ex_dev = reinterpret_cast<ExpertDesc*>(desc_dev);
  cudaGetDevice(&l->device);
  *out = l;
  return MXM_OK;
}

void mxm_layer_free(mxm_layer* l) { delete l; }

mxm_status mxm_workspace_bytes(const mxm_layer* l, int64_t max_tokens, int32_t top_k, int64_t* bytes) {
  if (!l || !bytes || max_tokens < 0 || top_k <= 0 || top_k > 32) return fail(MXM_E_CONFIG, "bad argument");
  *bytes = make_layout(l, max_tokens, top_k).total;
  return MXM_OK;
}

}  // extern "C"

// The launch sequence of one MoE block; `dump` != nullptr selects the test-only accumulator-dump kernel
// (mxm_debug_moe_group_gemm_dump) and disables split-K so every accumulator is a whole-K (or whole-group) sum.
// Tile-cost profiling (mxm_profile_tile_costs) runs the same sequence on one CTA (grid = 1) without split-K and
// brackets the persistent GEMM launch with its own events.
struct RunOpts {
  int grid = 0;  // 0: one CTA per SM
  bool no_split = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

static mxm_status run_group_gemm(const mxm_layer* l, const void* x, int64_t T, int32_t k, const int32_t* topk_ids,
                                 const float* topk_w, const float* shared_w, void* y, void* ws, int64_t ws_bytes,
                                 mxm_stream stream, uint32_t* dump, const RunOpts& opt = RunOpts()) {
  const bool no_split = dump != nullptr || opt.no_split;
  if (!l || !ws || (T > 0 && (!x || !topk_ids || !topk_w || !y))) return fail(MXM_E_CONFIG, "null argument");
  if (k <= 0 || k > 32 || T < 0) return fail(MXM_E_CONFIG, "bad top_k / T");
  const WsLayout w = make_layout(l, T, k);
  if (ws_bytes < w.total) return fail(MXM_E_CONFIG, "workspace too small");
  if (w.R >= (1LL << 31) || w.task_cap >= (1LL << 31)) return fail(MXM_E_CONFIG, "too many tokens");
  {
    int dev = -1;
    MXM_CUDA(cudaGetDevice(&dev));
    if (dev != l->device) return fail(MXM_E_CONFIG, "layer was initialised on another device");
  }
  if (T == 0) return MXM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* b = reinterpret_cast<uint8_t*>(ws);
  auto P = [&](int64_t off) -> void* { return off < 0 ? nullptr : (void*)(b + off); };
  int32_t* err = (int32_t*)P(w.err);
  int32_t* v_off = (int32_t*)P(w.v_off);
  int32_t* row_src = (int32_t*)P(w.row_src);
  float* row_w = (float*)P(w.row_w);
  int32_t* row_exp = (int32_t*)P(w.row_exp);
  int32_t* inv = (int32_t*)P(w.inv);

  cudaEvent_t* pev = nullptr;
  if (l->prof_n > 0) {
    mxm_layer* ml = const_cast<mxm_layer*>(l);
    pev = &ml->prof_ev[(size_t)(ml->prof_calls % ml->prof_n) * kProfEv];
    ++ml->prof_calls;
  }
  auto mark = [&](int i) {
    if (pev) cudaEventRecord(pev[i], st);
  };
  mark(0);
  MXM_CUDA(cudaMemsetAsync(err, 0, 4, st));
  // S1 route prep
  MXM_CUDA(launch_route_prep(topk_ids, topk_w, T, k, l->E, l->S, shared_w, (int32_t*)P(w.counts), nullptr, v_off,
                             nullptr, row_src, row_w, row_exp, inv, err, P(w.route_scratch), st));
  mark(1);
  // S3 plan on the side stream (needs only S1's offsets), concurrent with S2 on the caller's stream
  mxm_layer* ml = const_cast<mxm_layer*>(l);
  std::lock_guard<std::mutex> side_lock(ml->side_mu);
  if (!ml->side) {
    MXM_CUDA(cudaStreamCreateWithFlags(&ml->side, cudaStreamNonBlocking));
    MXM_CUDA(cudaEventCreateWithFlags(&ml->ev_fork, cudaEventDisableTiming));
    MXM_CUDA(cudaEventCreateWithFlags(&ml->ev_join, cudaEventDisableTiming));
  }
  MXM_CUDA(cudaEventRecord(ml->ev_fork, st));
  MXM_CUDA(cudaStreamWaitEvent(ml->side, ml->ev_fork, 0));
  MXM_CUDA(launch_plan(l->ex_dev, l->V, l->E, T, l->d, v_off, (int)w.g_max, w.task_cap, (Task*)P(w.tasks),
                       (int32_t*)P(w.meta), (int32_t*)P(w.grp_n1), (int32_t*)P(w.grp_nq), (int32_t*)P(w.p1_done),
                       (int32_t*)P(w.hq_done), no_split ? nullptr : (int32_t*)P(w.red_cnt), ml->side));
  MXM_CUDA(cudaEventRecord(ml->ev_join, ml->side));
  // S2 activation quantize + gather
  if (l->fm.n > 0 && k + l->S <= 32 && !getenv_flag("MXM_GATHER_ROWS")) {
    MXM_CUDA(launch_gather_tok(x, l->d, T, k, l->S, l->E, inv, row_exp, l->ex_dev, l->fm, w.R, P(w.Xb), P(w.XqA),
                               (float*)P(w.XsA), P(w.XqB), (float*)P(w.XsB), (int32_t*)P(w.XcA), (int32_t*)P(w.XcB),
                               (uint32_t*)P(w.hmax), st));
  } else {
    MXM_CUDA(launch_gather_quant(x, l->d, row_src, row_exp, v_off, l->V, l->ex_dev, w.R, P(w.Xb), P(w.XqA),
                                 (float*)P(w.XsA), P(w.XqB), (float*)P(w.XsB), (int32_t*)P(w.XcA),
                                 (int32_t*)P(w.XcB), (uint32_t*)P(w.hmax), st));
  }
  mark(2);
  MXM_CUDA(cudaStreamWaitEvent(st, ml->ev_join, 0));
  mark(3);  // the plan's time beyond the gather's (usually ~0)
  // S4-S7 persistent group GEMM
  GemmParams prm;
  memset(&prm, 0, sizeof(prm));
  const uint32_t boxes[4] = {16, 32, 64, MXM_DUAL_TILE};
  // H / Hq: routed region (maps 3, 4: rows T*k at width f, after the shared region) and shared region (maps 5,
  // 6: rows T*S at width f_s), gemm.cu h_off
  const int64_t srows = T * l->S, rrows = T * k, rbase = srows * l->fs;
  const void* srcs[7] = {P(w.Xb), P(w.XqA), P(w.XqB), w.H >= 0 ? (void*)((char*)P(w.H) + 2 * rbase) : nullptr,
                         w.Hq >= 0 ? (void*)((char*)P(w.Hq) + rbase) : nullptr, srows > 0 ? P(w.H) : nullptr,
                         srows > 0 && w.Hq >= 0 ? P(w.Hq) : nullptr};
  const bool isbf[7] = {true, false, false, true, false, true, false};
  const uint64_t cols[7] = {(uint64_t)l->d, (uint64_t)l->d, (uint64_t)l->d, (uint64_t)l->f, (uint64_t)l->f,
                            (uint64_t)l->fs, (uint64_t)l->fs};
  const uint64_t rows[7] = {(uint64_t)w.R, (uint64_t)w.R, (uint64_t)w.R, (uint64_t)rrows, (uint64_t)rrows,
                            (uint64_t)srows, (uint64_t)srows};
  if (ml->tm_ws != ws || ml->tm_T != T || ml->tm_k != k) {
    ml->tm_ws = nullptr;
    for (int i = 0; i < 7; ++i) {
      if (!srcs[i]) continue;
      for (int j = 0; j < 4; ++j)
        if (!encode_2d(&ml->tm[i][j], srcs[i], isbf[i], cols[i], rows[i], boxes[j]))
          return fail(MXM_E_CUDA, "cuTensorMapEncodeTiled failed");
    }
    ml->tm_ws = ws;
    ml->tm_T = T;
    ml->tm_k = k;
  }
  for (int i = 0; i < 7; ++i)
    if (srcs[i]) memcpy(&prm.tmap[i][0], &ml->tm[i][0], sizeof(ml->tm[i]));
  prm.h_srows = srows;
  prm.h_rbase = rbase;
  prm.f_s = l->fs;
  prm.f_r = l->f;
  prm.ex = l->ex_dev;
  prm.tasks = (const Task*)P(w.tasks);
  prm.meta = (int32_t*)P(w.meta);
  prm.p1_done = (int32_t*)P(w.p1_done);
  prm.hq_done = (int32_t*)P(w.hq_done);
  prm.grp_n1 = (const int32_t*)P(w.grp_n1);
  prm.grp_nq = (const int32_t*)P(w.grp_nq);
  prm.xs[0] = nullptr;
  prm.xs[1] = (const float*)P(w.XsA);
  prm.xs[2] = (const float*)P(w.XsB);
  prm.xc[0] = nullptr;
  prm.xc[1] = (const int32_t*)P(w.XcA);
  prm.xc[2] = (const int32_t*)P(w.XcB);
  prm.Hc = (int32_t*)P(w.Hc);
  prm.H = (uint16_t*)P(w.H);
  prm.Hq = (int8_t*)P(w.Hq);
  prm.Hs = (float*)P(w.Hs);
  prm.hs_stride = w.R;
  prm.hmax = (uint32_t*)P(w.hmax);
  prm.O = (uint16_t*)P(w.O);
  prm.row_w = row_w;
  prm.P = no_split ? nullptr : (float*)P(w.P);
  prm.red_cnt = no_split ? nullptr : (int32_t*)P(w.red_cnt);
  prm.dump = dump;
  prm.d = l->d;
  prm.f_max = l->f_max;
  prm.prof = reinterpret_cast<unsigned long long*>(l->prof_counters);
  if (opt.ev0) MXM_CUDA(cudaEventRecord(opt.ev0, st));
  MXM_CUDA(launch_moe_gemm(prm, opt.grid > 0 ? opt.grid : num_sms(), st));
  if (opt.ev1) MXM_CUDA(cudaEventRecord(opt.ev1, st));
  mark(4);
  // S8 combine
  MXM_CUDA(launch_combine(P(w.O), l->d, T, k, l->S, inv, y, st));
  mark(5);
  return MXM_OK;
}

extern "C" {

mxm_status mxm_moe_group_gemm(const mxm_layer* l, const void* x, int64_t T, int32_t k, const int32_t* topk_ids,
                              const float* topk_w, const float* shared_w, void* y, void* ws, int64_t ws_bytes,
                              mxm_stream stream) {
  return run_group_gemm(l, x, T, k, topk_ids, topk_w, shared_w, y, ws, ws_bytes, stream, nullptr);
}

mxm_status mxm_debug_acc_bytes(const mxm_layer* l, int64_t T, int32_t k, int64_t* bytes) {
  if (!l || !bytes || T < 0 || k <= 0 || k > 32) return fail(MXM_E_CONFIG, "bad argument");
  // gate / up: [2][d/128][R][f_max]; down: [f_max/128][R][d]  (uint32)
  const int64_t R = make_layout(l, T, k).R;
  *bytes = (int64_t)4 * (2 * (l->d / 128) * R * l->f_max + (l->f_max / 128) * R * l->d);
  return MXM_OK;
}

mxm_status mxm_debug_moe_group_gemm_dump(const mxm_layer* l, const void* x, int64_t T, int32_t k,
                                         const int32_t* topk_ids, const float* topk_w, const float* shared_w, void* y,
                                         void* ws, int64_t ws_bytes, void* acc, int64_t acc_bytes, mxm_stream stream) {
  int64_t need = 0;
  mxm_status s = mxm_debug_acc_bytes(l, T, k, &need);
  if (s != MXM_OK) return s;
  if (!acc || acc_bytes < need) return fail(MXM_E_CONFIG, "accumulator dump buffer too small");
  return run_group_gemm(l, x, T, k, topk_ids, topk_w, shared_w, y, ws, ws_bytes, stream, (uint32_t*)acc);
}

static constexpr int kProfTiles[4] = {16, 32, 64, MXM_DUAL_TILE};

mxm_status mxm_profile_scratch_bytes(const mxm_layer* l, int64_t* bytes) {
  if (!l || !bytes) return fail(MXM_E_CONFIG, "null argument");
  const int64_t T = MXM_DUAL_TILE;
  *bytes = make_layout(l, T, 1).total + align256(2 * T * l->d) * 2 + align256(4 * T) * 2;
  return MXM_OK;
}

mxm_status mxm_profile_tile_costs(const mxm_layer* l, void* scratch, int64_t scratch_bytes, float* costs,
                                  mxm_stream stream) {
  if (!l || !scratch || !costs) return fail(MXM_E_CONFIG, "null argument");
  int64_t need = 0;
  mxm_status s = mxm_profile_scratch_bytes(l, &need);
  if (s != MXM_OK) return s;
  if (scratch_bytes < need) return fail(MXM_E_CONFIG, "profile scratch too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t Tm = MXM_DUAL_TILE;
  uint8_t* b = reinterpret_cast<uint8_t*>(scratch);
  const int64_t wsb = make_layout(l, Tm, 1).total;
  void* ws = b;
  void* x = b + wsb;
  void* y = b + wsb + align256(2 * Tm * l->d);
  int32_t* ids = reinterpret_cast<int32_t*>(b + wsb + 2 * align256(2 * Tm * l->d));
  float* w = reinterpret_cast<float*>(b + wsb + 2 * align256(2 * Tm * l->d) + align256(4 * Tm));
  // inputs: zeros (tile cost does not depend on the values), unit route weights
  MXM_CUDA(cudaMemsetAsync(x, 0, 2 * Tm * l->d, st));
  std::vector<float> ones(Tm, 1.f);
  MXM_CUDA(cudaMemcpyAsync(w, ones.data(), 4 * Tm, cudaMemcpyHostToDevice, st));
  cudaEvent_t e0, e1;
  MXM_CUDA(cudaEventCreate(&e0));
  MXM_CUDA(cudaEventCreate(&e1));
  RunOpts opt;
  opt.grid = 1;  // single-CTA runs: the cost of one SM working through the group's tiles
  opt.no_split = true;
  opt.ev0 = e0;
  opt.ev1 = e1;
  std::vector<int32_t> hid(Tm);
  auto timed = [&](int64_t T, int32_t id, float* ms) -> mxm_status {
    for (int64_t t = 0; t < T; ++t) hid[t] = id;
    MXM_CUDA(cudaMemcpyAsync(ids, hid.data(), 4 * T, cudaMemcpyHostToDevice, st));
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      mxm_status r = run_group_gemm(l, x, T, 1, ids, w, nullptr, y, ws, wsb, stream, nullptr, opt);
      if (r != MXM_OK) return r;
      MXM_CUDA(cudaEventSynchronize(e1));
      float m = 0.f;
      MXM_CUDA(cudaEventElapsedTime(&m, e0, e1));
      best = m < best ? m : best;
    }
    *ms = best;
    return MXM_OK;
  };
  mxm_status r = MXM_OK;
  for (int ni = 0; ni < 4 && r == MXM_OK; ++ni) {
    float base = 0.f;  // shared experts only (every token routed nowhere)
    r = timed(kProfTiles[ni], -1, &base);
    for (int v = 0; v < l->E && r == MXM_OK; ++v) {
      const int T = kProfTiles[ni] < tile_cap(l->ex[v]) ? kProfTiles[ni] : tile_cap(l->ex[v]);
      float t = 0.f;
      r = timed(T, v, &t);
      costs[v * 4 + ni] = t - base > 1e-6f ? t - base : 1e-6f;
    }
    for (int v = l->E; v < l->V; ++v) costs[v * 4 + ni] = base / (float)l->S;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return r;
}

mxm_status mxm_layer_set_tile_costs(mxm_layer* l, const float* costs) {
  if (!l) return fail(MXM_E_CONFIG, "null layer");
  for (int v = 0; v < l->V; ++v)
    for (int i = 0; i < 4; ++i) l->ex[v].cost[i] = costs && costs[v * 4 + i] > 0.f ? costs[v * 4 + i] : 0.f;
  MXM_CUDA(cudaMemcpy(l->ex_dev, l->ex.data(), sizeof(ExpertDesc) * l->V, cudaMemcpyHostToDevice));
  return MXM_OK;
}

mxm_status mxm_debug_workspace_layout(const mxm_layer* l, int64_t T, int32_t k, int64_t* off) {
  if (!l || !off || T < 0 || k <= 0 || k > 32) return fail(MXM_E_CONFIG, "bad argument");
  const WsLayout w = make_layout(l, T, k);
  const int64_t v[MXM_WS_N] = {w.row_src, w.row_w, w.row_exp, w.inv, w.Xb, w.XqA, w.XsA, w.XqB, w.XsB,
                               w.H, w.Hq, w.Hs, w.O, w.v_off, w.R, l->f_max, w.XcA, w.XcB, w.Hc,
                               w.tasks, w.meta, w.g_max};
  for (int i = 0; i < MXM_WS_N; ++i) off[i] = v[i];
  return MXM_OK;
}

mxm_status mxm_layer_profile(mxm_layer* l, int32_t n_slots) {
  if (!l || n_slots < 0 || n_slots > 100000) return fail(MXM_E_CONFIG, "bad argument");
  for (auto e : l->prof_ev) cudaEventDestroy(e);
  l->prof_ev.clear();
  l->prof_n = 0;
  l->prof_calls = 0;
  l->prof_ev.resize((size_t)n_slots * kProfEv);
  for (auto& e : l->prof_ev) MXM_CUDA(cudaEventCreate(&e));
  l->prof_n = n_slots;
  return MXM_OK;
}

mxm_status mxm_layer_profile_read(mxm_layer* l, float* ms, int32_t n, int32_t* n_recorded) {
  if (!l || !ms || !n_recorded) return fail(MXM_E_CONFIG, "null argument");
  const int64_t rec = l->prof_calls < l->prof_n ? l->prof_calls : l->prof_n;
  const int64_t m = rec < n ? rec : n;
  for (int64_t i = 0; i < m; ++i) {
    cudaEvent_t* e = &l->prof_ev[(size_t)i * kProfEv];
    MXM_CUDA(cudaEventSynchronize(e[kProfEv - 1]));
    for (int j = 0; j < kProfEv - 1; ++j) MXM_CUDA(cudaEventElapsedTime(&ms[i * (kProfEv - 1) + j], e[j], e[j + 1]));
  }
  *n_recorded = (int32_t)m;
  return MXM_OK;
}

mxm_status mxm_layer_debug_counters(mxm_layer* l, void* dev_buf) {
  if (!l) return fail(MXM_E_CONFIG, "null layer");
#ifndef MXM_DEBUG_COUNTERS
  if (dev_buf) return fail(MXM_E_CONFIG, "library built without MXM_DEBUG_COUNTERS (see tools/diag_waits.py)");
#endif
  l->prof_counters = dev_buf;
  return MXM_OK;
}

int32_t mxm_kernels_per_call(const mxm_layer* l) { return l ? 7 + (l->S > 0 ? 1 : 0) : 0; }

mxm_status mxm_ep_route(const int32_t* topk_ids, int64_t T, int32_t k, int32_t E, int32_t G, int32_t* dest_counts,
                        int32_t* pos, int32_t* err, mxm_stream stream) {
  if (!topk_ids || !dest_counts || !pos) return fail(MXM_E_CONFIG, "null argument");
  if (G <= 0 || G > 64 || E % G != 0 || k <= 0 || k > 32 || T < 0) return fail(MXM_E_CONFIG, "bad E/G/k/T");
  MXM_CUDA(launch_ep_route(topk_ids, T, k, E, G, dest_counts, pos, err, (cudaStream_t)stream));
  return MXM_OK;
}

mxm_status mxm_ep_pack(const void* x, int64_t T, int32_t d, const int32_t* topk_ids, const float* topk_w, int32_t k,
                       int32_t E, int32_t G, const int32_t* pos, const int32_t* dest_offsets, void* send_x,
                       int32_t* send_ids, float* send_w, int32_t* send_src, mxm_stream stream) {
  if (!x || !topk_ids || !topk_w || !pos || !dest_offsets || !send_x || !send_ids || !send_w || !send_src)
    return fail(MXM_E_CONFIG, "null argument");
  if (G <= 0 || E % G != 0 || d % 8 != 0 || k > 32) return fail(MXM_E_CONFIG, "bad shape");
  MXM_CUDA(launch_ep_pack(x, T, d, topk_ids, topk_w, k, E, G, pos, dest_offsets, send_x, send_ids, send_w, send_src,
                          (cudaStream_t)stream));
  return MXM_OK;
}

mxm_status mxm_ep_combine(const void* back, const int32_t* pos, const int32_t* dest_offsets, int32_t G, int64_t T,
                          int32_t d, const void* y_shared, void* y, mxm_stream stream) {
  if (!back || !pos || !dest_offsets || !y) return fail(MXM_E_CONFIG, "null argument");
  if (G <= 0 || d % 8 != 0) return fail(MXM_E_CONFIG, "bad shape");
  MXM_CUDA(launch_ep_combine(back, pos, dest_offsets, G, T, d, y_shared, y, (cudaStream_t)stream));
  return MXM_OK;
}

mxm_status mxm_poll_device_error(const mxm_layer* l, const void* ws, mxm_stream stream, int32_t* code) {
  if (!l || !ws || !code) return fail(MXM_E_CONFIG, "null argument");
  int32_t v = 0;
  MXM_CUDA(cudaMemcpyAsync(&v, ws, 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  MXM_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  MXM_CUDA(cudaMemsetAsync(const_cast<void*>(ws), 0, 4, (cudaStream_t)stream));
  *code = v ? MXM_E_DATA : MXM_OK;
  return MXM_OK;
}

mxm_status mxm_debug_task_stats(const mxm_layer* l, const void* ws, int64_t T, int32_t top_k, mxm_stream stream,
                                int32_t* n_tasks, int32_t* n_executed) {
  if (!l || !ws || !n_tasks || !n_executed || top_k <= 0) return fail(MXM_E_CONFIG, "null argument");
  const WsLayout w = make_layout(l, T, top_k);
  int32_t meta[8];
  MXM_CUDA(cudaMemcpyAsync(meta, (const uint8_t*)ws + w.meta, sizeof(meta), cudaMemcpyDeviceToHost,
                           (cudaStream_t)stream));
  MXM_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  *n_tasks = meta[0];
  *n_executed = meta[6];
  return MXM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- expert parallelism through the C ABI (step S9)
// v1 of SURVEY §8(e): NCCL all-to-all of per-destination counts (one host sync for the split sizes), grouped
// ncclSend / ncclRecv all-to-all-v of the deduplicated token rows with their local (id, weight) metadata, the local
// routed group-GEMM, the reverse all-to-all-v of the partial outputs, the shared experts on the own tokens, and
// the fixed-order combine. The communicator is borrowed (never destroyed here).
struct mxm_ep {
  mxm_layer* local = nullptr;
  mxm_layer* shared = nullptr;
  ncclComm_t comm = nullptr;
  int G = 1, rank = 0, E = 0;
  int mode = MXM_EP_V1;  // MXM_EP_SYNC_FREE: fixed-capacity exchange, no host sync (mxm_ep_set_mode)
};

namespace {
struct EpLayout {
  int64_t err, dest_counts, recv_counts, dest_off, pos, send_x, send_ids, send_w, send_src, recv_x, recv_ids, recv_w,
      recv_y, back, sid, ones, y_sh, ws_local, ws_shared, total, ws_local_bytes, ws_shared_bytes;
};
EpLayout ep_layout(const mxm_ep* ep, int64_t T, int k, int64_t max_recv) {
  EpLayout w{};
  const int64_t G = ep->G, d = ep->local->d, S = ep->shared ? ep->shared->E : 0;
  // v1 sends at most min(k, G) rows per token in total; sync-free reserves T rows for every destination
  const int64_t max_send = ep->mode == MXM_EP_SYNC_FREE ? T * G : T * (k < G ? k : G);
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = o;
    o += align256(bytes > 0 ? bytes : 1);
    return at;
  };
  w.err = take(256);
  w.dest_counts = take(4 * G);
  w.recv_counts = take(4 * G);
  w.dest_off = take(4 * (G + 1));
  w.pos = take(4 * T * G);
  w.send_x = take(2 * max_send * d);
  w.send_ids = take(4 * max_send * k);
  w.send_w = take(4 * max_send * k);
  w.send_src = take(4 * max_send);
  w.recv_x = take(2 * max_recv * d);
  w.recv_ids = take(4 * max_recv * k);
  w.recv_w = take(4 * max_recv * k);
  w.recv_y = take(2 * max_recv * d);
  w.back = take(2 * max_send * d);
  w.sid = take(4 * T * (S > 0 ? S : 1));
  w.ones = take(4 * T * (S > 0 ? S : 1));
  w.y_sh = take(2 * T * d);
  w.ws_local_bytes = make_layout(ep->local, max_recv, k).total;
  w.ws_local = take(w.ws_local_bytes);
  w.ws_shared_bytes = S > 0 ? make_layout(ep->shared, T, (int)S).total : 0;
  w.ws_shared = take(w.ws_shared_bytes);
  w.total = o;
  return w;
}
mxm_status nccl_fail(ncclResult_t r, const char* where) {
  g_err = std::string(where) + ": " + ncclGetErrorString(r);
  return MXM_E_NCCL;
}
#define MXM_NCCL(call)                                  \
  do {                                                  \
    ncclResult_t _r = (call);                           \
    if (_r != ncclSuccess) return nccl_fail(_r, #call); \
  } while (0)
}  // namespace

extern "C" {

mxm_status mxm_ep_init(mxm_layer* local, mxm_layer* shared, void* nccl_comm, int32_t n_global_experts, mxm_ep** out) {
  if (!local || !nccl_comm || !out) return fail(MXM_E_CONFIG, "null argument");
  if (local->S != 0) return fail(MXM_E_CONFIG, "the local layer holds routed experts only (shared go in `shared`)");
  if (shared && (shared->S != 0 || shared->d != local->d)) return fail(MXM_E_CONFIG, "shared layer mismatch");
  auto* ep = new mxm_ep();
  ep->comm = reinterpret_cast<ncclComm_t>(nccl_comm);
  ncclResult_t r = ncclCommCount(ep->comm, &ep->G);
  if (r == ncclSuccess) r = ncclCommUserRank(ep->comm, &ep->rank);
  if (r != ncclSuccess) {
    delete ep;
    return nccl_fail(r, "ncclCommCount/UserRank");
  }
  if (n_global_experts <= 0 || n_global_experts % ep->G != 0 || local->E != n_global_experts / ep->G) {
    delete ep;
    return fail(MXM_E_CONFIG, "local layer must hold n_global_experts / world_size routed experts");
  }
  ep->local = local;
  ep->shared = shared;
  ep->E = n_global_experts;
  *out = ep;
  return MXM_OK;
}

void mxm_ep_free(mxm_ep* ep) { delete ep; }

mxm_status mxm_ep_poll_device_error(const mxm_ep* ep, const void* ws, mxm_stream stream, int32_t* code) {
  if (!ep || !ws || !code) return fail(MXM_E_CONFIG, "null argument");
  int32_t v = 0;  // the EP workspace starts with its error word (bad expert ids seen by the dispatch)
  MXM_CUDA(cudaMemcpyAsync(&v, ws, 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  MXM_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  MXM_CUDA(cudaMemsetAsync(const_cast<void*>(ws), 0, 4, (cudaStream_t)stream));
  *code = v ? MXM_E_DATA : MXM_OK;
  return MXM_OK;
}

mxm_status mxm_ep_workspace_bytes(const mxm_ep* ep, int64_t T, int32_t k, int64_t max_recv_rows, int64_t* bytes) {
  if (!ep || !bytes || T < 0 || k <= 0 || k > 32 || max_recv_rows < 0) return fail(MXM_E_CONFIG, "bad argument");
  *bytes = ep_layout(ep, T, k, max_recv_rows).total;
  return MXM_OK;
}

mxm_status mxm_ep_set_mode(mxm_ep* ep, int32_t mode) {
  if (!ep || (mode != MXM_EP_V1 && mode != MXM_EP_SYNC_FREE)) return fail(MXM_E_CONFIG, "bad EP handle / mode");
  ep->mode = mode;
  return MXM_OK;
}

mxm_status mxm_ep_moe_group_gemm(mxm_ep* ep, const void* x, int64_t T, int32_t k, const int32_t* topk_ids,
                                 const float* topk_w, const float* shared_w, void* y, void* ws, int64_t ws_bytes,
                                 int64_t max_recv_rows, mxm_stream stream) {
  if (!ep || !ws || (T > 0 && (!x || !topk_ids || !topk_w || !y))) return fail(MXM_E_CONFIG, "null argument");
  if (k <= 0 || k > 32 || T < 0) return fail(MXM_E_CONFIG, "bad top_k / T");
  const EpLayout w = ep_layout(ep, T, k, max_recv_rows);
  if (ws_bytes < w.total) return fail(MXM_E_CONFIG, "EP workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* b = reinterpret_cast<uint8_t*>(ws);
  auto P = [&](int64_t off) -> void* { return (void*)(b + off); };
  const int G = ep->G, d = ep->local->d, S = ep->shared ? ep->shared->E : 0;
  int32_t* dest_counts = (int32_t*)P(w.dest_counts);
  int32_t* recv_counts = (int32_t*)P(w.recv_counts);
  int32_t* pos = (int32_t*)P(w.pos);
  if (ep->mode == MXM_EP_SYNC_FREE) {
    // fixed capacity C = T rows per destination (a token goes to a rank at most once): equal-count exchanges, no
    // host read of any count; rows no token fills carry expert id -1 (no route) and are skipped by the local layer
    const int64_t C = T, R = (int64_t)G * T;
    if (R > max_recv_rows) return fail(MXM_E_CONFIG, "sync-free EP needs max_recv_rows >= G * T");
    int32_t* dest_off = (int32_t*)P(w.dest_off);
    MXM_CUDA(launch_ep_route(topk_ids, T, k, ep->E, G, dest_counts, pos, (int32_t*)P(w.err), st));
    MXM_CUDA(launch_ep_fill(dest_off, G, C, (int32_t*)P(w.sid), (float*)P(w.ones), T, S, st));
    MXM_CUDA(cudaMemsetAsync(P(w.send_ids), 0xFF, 4 * R * k, st));  // -1: no route
    MXM_CUDA(cudaMemsetAsync(P(w.send_w), 0, 4 * R * k, st));
    MXM_CUDA(launch_ep_pack(x, T, d, topk_ids, topk_w, k, ep->E, G, pos, dest_off, P(w.send_x),
                            (int32_t*)P(w.send_ids), (float*)P(w.send_w), (int32_t*)P(w.send_src), st));
    MXM_NCCL(ncclGroupStart());
    for (int r = 0; r < G; ++r) {
      MXM_NCCL(ncclSend((uint16_t*)P(w.send_x) + r * C * d, (size_t)(C * d), ncclBfloat16, r, ep->comm, st));
      MXM_NCCL(ncclSend((int32_t*)P(w.send_ids) + r * C * k, (size_t)(C * k), ncclInt32, r, ep->comm, st));
      MXM_NCCL(ncclSend((float*)P(w.send_w) + r * C * k, (size_t)(C * k), ncclFloat32, r, ep->comm, st));
      MXM_NCCL(ncclRecv((uint16_t*)P(w.recv_x) + r * C * d, (size_t)(C * d), ncclBfloat16, r, ep->comm, st));
      MXM_NCCL(ncclRecv((int32_t*)P(w.recv_ids) + r * C * k, (size_t)(C * k), ncclInt32, r, ep->comm, st));
      MXM_NCCL(ncclRecv((float*)P(w.recv_w) + r * C * k, (size_t)(C * k), ncclFloat32, r, ep->comm, st));
    }
    MXM_NCCL(ncclGroupEnd());
    if (R > 0) {
      mxm_status s = run_group_gemm(ep->local, P(w.recv_x), R, k, (const int32_t*)P(w.recv_ids),
                                    (const float*)P(w.recv_w), nullptr, P(w.recv_y), P(w.ws_local),
                                    w.ws_local_bytes, stream, nullptr);
      if (s != MXM_OK) return s;
    }
    MXM_NCCL(ncclGroupStart());
    for (int r = 0; r < G; ++r) {
      MXM_NCCL(ncclSend((uint16_t*)P(w.recv_y) + r * C * d, (size_t)(C * d), ncclBfloat16, r, ep->comm, st));
      MXM_NCCL(ncclRecv((uint16_t*)P(w.back) + r * C * d, (size_t)(C * d), ncclBfloat16, r, ep->comm, st));
    }
    MXM_NCCL(ncclGroupEnd());
    void* y_sh = nullptr;
    if (S > 0 && T > 0) {
      y_sh = P(w.y_sh);
      mxm_status s = run_group_gemm(ep->shared, x, T, S, (const int32_t*)P(w.sid),
                                    shared_w ? shared_w : (const float*)P(w.ones), nullptr, y_sh, P(w.ws_shared),
                                    w.ws_shared_bytes, stream, nullptr);
      if (s != MXM_OK) return s;
    }
    if (T > 0) MXM_CUDA(launch_ep_combine(P(w.back), pos, dest_off, G, T, d, y_sh, y, st));
    return MXM_OK;
  }
  // 1. per-destination deduplicated counts and slots, exchanged
  MXM_CUDA(launch_ep_route(topk_ids, T, k, ep->E, G, dest_counts, pos, (int32_t*)P(w.err), st));
  MXM_NCCL(ncclGroupStart());
  for (int r = 0; r < G; ++r) {
    MXM_NCCL(ncclSend(dest_counts + r, 1, ncclInt32, r, ep->comm, st));
    MXM_NCCL(ncclRecv(recv_counts + r, 1, ncclInt32, r, ep->comm, st));
  }
  MXM_NCCL(ncclGroupEnd());
  std::vector<int32_t> sc(G), rc(G);
  MXM_CUDA(cudaMemcpyAsync(sc.data(), dest_counts, 4 * G, cudaMemcpyDeviceToHost, st));
  MXM_CUDA(cudaMemcpyAsync(rc.data(), recv_counts, 4 * G, cudaMemcpyDeviceToHost, st));
  MXM_CUDA(cudaStreamSynchronize(st));  // v1: the split sizes of the all-to-all-v live on the host
  std::vector<int64_t> so(G + 1, 0), ro(G + 1, 0);
  for (int r = 0; r < G; ++r) {
    so[r + 1] = so[r] + sc[r];
    ro[r + 1] = ro[r] + rc[r];
  }
  const int64_t S_send = so[G], R = ro[G];
  if (R > max_recv_rows) return fail(MXM_E_CONFIG, "received rows exceed max_recv_rows");
  std::vector<int32_t> so32(G + 1);
  for (int r = 0; r <= G; ++r) so32[r] = (int32_t)so[r];
  int32_t* dest_off = (int32_t*)P(w.dest_off);
  MXM_CUDA(cudaMemcpyAsync(dest_off, so32.data(), 4 * (G + 1), cudaMemcpyHostToDevice, st));
  // 2. send buffers (rows by (destination, token)) and the all-to-all-v of rows / local ids / weights
  MXM_CUDA(launch_ep_pack(x, T, d, topk_ids, topk_w, k, ep->E, G, pos, dest_off, P(w.send_x), (int32_t*)P(w.send_ids),
                          (float*)P(w.send_w), (int32_t*)P(w.send_src), st));
  MXM_NCCL(ncclGroupStart());
  for (int r = 0; r < G; ++r) {
    if (sc[r]) {
      MXM_NCCL(ncclSend((uint16_t*)P(w.send_x) + so[r] * d, (size_t)sc[r] * d, ncclBfloat16, r, ep->comm, st));
      MXM_NCCL(ncclSend((int32_t*)P(w.send_ids) + so[r] * k, (size_t)sc[r] * k, ncclInt32, r, ep->comm, st));
      MXM_NCCL(ncclSend((float*)P(w.send_w) + so[r] * k, (size_t)sc[r] * k, ncclFloat32, r, ep->comm, st));
    }
    if (rc[r]) {
      MXM_NCCL(ncclRecv((uint16_t*)P(w.recv_x) + ro[r] * d, (size_t)rc[r] * d, ncclBfloat16, r, ep->comm, st));
      MXM_NCCL(ncclRecv((int32_t*)P(w.recv_ids) + ro[r] * k, (size_t)rc[r] * k, ncclInt32, r, ep->comm, st));
      MXM_NCCL(ncclRecv((float*)P(w.recv_w) + ro[r] * k, (size_t)rc[r] * k, ncclFloat32, r, ep->comm, st));
    }
  }
  MXM_NCCL(ncclGroupEnd());
  // 3. the local routed experts on the received rows
  if (R > 0) {
    mxm_status s = run_group_gemm(ep->local, P(w.recv_x), R, k, (const int32_t*)P(w.recv_ids),
                                  (const float*)P(w.recv_w), nullptr, P(w.recv_y), P(w.ws_local), w.ws_local_bytes,
                                  stream, nullptr);
    if (s != MXM_OK) return s;
  }
  // 4. partial outputs back to their source ranks, in send order
  MXM_NCCL(ncclGroupStart());
  for (int r = 0; r < G; ++r) {
    if (rc[r]) MXM_NCCL(ncclSend((uint16_t*)P(w.recv_y) + ro[r] * d, (size_t)rc[r] * d, ncclBfloat16, r, ep->comm, st));
    if (sc[r]) MXM_NCCL(ncclRecv((uint16_t*)P(w.back) + so[r] * d, (size_t)sc[r] * d, ncclBfloat16, r, ep->comm, st));
  }
  MXM_NCCL(ncclGroupEnd());
  // 5. shared experts on the own tokens (top-k = S, every token routed to all of them with weight shared_w)
  void* y_sh = nullptr;
  if (S > 0 && T > 0) {
    std::vector<int32_t> sid((size_t)T * S);
    for (int64_t t = 0; t < T; ++t)
      for (int s2 = 0; s2 < S; ++s2) sid[(size_t)t * S + s2] = s2;
    MXM_CUDA(cudaMemcpyAsync(P(w.sid), sid.data(), 4 * T * S, cudaMemcpyHostToDevice, st));
    const float* swp = shared_w;
    if (!swp) {
      std::vector<float> ones((size_t)T * S, 1.f);
      MXM_CUDA(cudaMemcpyAsync(P(w.ones), ones.data(), 4 * T * S, cudaMemcpyHostToDevice, st));
      MXM_CUDA(cudaStreamSynchronize(st));  // host staging buffers go out of scope
      swp = (const float*)P(w.ones);
    } else {
      MXM_CUDA(cudaStreamSynchronize(st));
    }
    y_sh = P(w.y_sh);
    mxm_status s = run_group_gemm(ep->shared, x, T, S, (const int32_t*)P(w.sid), swp, nullptr, y_sh, P(w.ws_shared),
                                  w.ws_shared_bytes, stream, nullptr);
    if (s != MXM_OK) return s;
  }
  // 6. fixed-order combine over destinations + shared
  if (T > 0) MXM_CUDA(launch_ep_combine(P(w.back), pos, dest_off, G, T, d, y_sh, y, st));
  (void)S_send;
  return MXM_OK;
}

}  // extern "C"

#ifdef MXM_DEBUG_NAN
namespace mxm { cudaError_t debug_nan_info(unsigned long long* out, bool reset); }
extern "C" int mxm_debug_nan_info(unsigned long long* out) { return (int)mxm::debug_nan_info(out, true); }
#endif

#ifdef MXM_TRACE_TASKS
namespace mxm { cudaError_t debug_trace_tasks(unsigned long long* tt, unsigned long long* cta); }
extern "C" int mxm_debug_trace_tasks(unsigned long long* tt, unsigned long long* cta) {
  return (int)mxm::debug_trace_tasks(tt, cta);
}
#endif

#ifdef MXM_TRACE
namespace mxm { cudaError_t debug_trace(unsigned long long* out); }
extern "C" int mxm_debug_trace(unsigned long long* out) { return (int)mxm::debug_trace(out); }
#endif
