/* mxmoe.h — C ABI of the B200-native MxMoE mixed-precision MoE group-GEMM.
 *
 * The operations follow the paper's statement of the problem (arXiv 2505.05799,
 * /root/reference/PAPER.md, cited "P:<line>"):
 *   - uniform min-max quantization of a linear block (§2.1) at a per-block
 *     bit-width / group size / symmetry (per-linear-block allocation, §4.2.1);
 *   - a mixed-precision Group-GEMM that runs every expert's gate/up/down linear block,
 *     each at its own precision, over the routed token groups (§2.2, §4.3),
 *     computing the MoE block F = Σ_e W_down^e(σ(W_gate^e X_e) ⊙ W_up^e X_e) ⊙ w_e
 *     (Eq. 1, Eq. 2), with activations quantized dynamically at runtime
 *     for weight-activation schemes.
 * Exact numerical definitions (rounding, scale round-up, fp32 activation quantizer)
 * are the readings listed in DESIGN.md §2.
 *
 * Conventions (all entry points):
 *   - Tensor pointers are CUDA DEVICE pointers OWNED BY THE CALLER unless the parameter
 *     says "host". The library never allocates device memory and never frees caller memory.
 *   - Calls marked [async] enqueue work on `stream` and return without synchronizing;
 *     [sync] calls may block the host.
 *   - Errors are returned, never thrown: MXM_E_CONFIG (unsupported scheme/shape; nothing is
 *     launched), MXM_E_DATA (bad data detected on device; surfaced by mxm_poll_device_error),
 *     MXM_E_CUDA (a CUDA call failed; see mxm_last_error()).
 *   - Row-major layouts; bf16 is IEEE bfloat16 bit patterns (uint16).
 */
#ifndef MXMOE_H
#define MXMOE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { MXM_OK = 0, MXM_E_CONFIG = 3, MXM_E_DATA = 4, MXM_E_CUDA = 5, MXM_E_NCCL = 6 } mxm_status;

/* Quantization scheme `wxay_gz_{sym,asym}` (PAPER.md P:92 caption of fig:motivation).
 *   w_bits    2,3,4,8 (weight-only) | 4,5,8 (weight-activation) | 16 (bf16 pass-through)
 *   a_bits    16 = weight-only; otherwise == w_bits (w4a4, w5a5, w8a8)
 *   w_group   -1 = per-channel, else 64 or 128 (weight-only), 128 (weight-activation); divides K
 *   a_group   weight-activation: == w_group (-1 = per-token); weight-only: ignored
 *   symmetric 1 = scale only; 0 = scale + zero-point (weight-only only)                        */
typedef struct {
  int32_t w_bits, a_bits, w_group, a_group, symmetric;
  int32_t fmt; /* MXM_FMT_INT (0): integer codes (the paper's uniform quantizer); MXM_FMT_E4M3 (1): FP8
                * e4m3 codes for weights and activations (NEXT-4 "FP8 as an extra hardware-supported scheme",
                * readings R25/R26), w_bits = a_bits = 8, symmetric, w_group = a_group in {-1, 128} */
} mxm_scheme;
enum { MXM_FMT_INT = 0, MXM_FMT_E4M3 = 1 };

typedef void* mxm_stream; /* a cudaStream_t */

enum { MXM_GATE = 0, MXM_UP = 1, MXM_DOWN = 2 };

/* ---------------------------------------------------------------- metadata [sync, host only] */
/* MXM_OK if the scheme is supported for a block W[N, K]; MXM_E_CONFIG otherwise. */
mxm_status mxm_scheme_check(const mxm_scheme* s, int64_t N, int64_t K);
/* Sizes in bytes of the canonical quantizer outputs and of the packed buffer (docs/packed_format.md). */
mxm_status mxm_quant_sizes(const mxm_scheme* s, int64_t N, int64_t K, int64_t* codes_bytes, int64_t* scale_bytes,
                           int64_t* zero_bytes, int64_t* packed_bytes);
/* w + (1 sym | 2 asym)·16/g with g = K for per-channel (3.25 / 2.25 for w3/w2-g128-asym). */
double mxm_storage_bits_per_weight(const mxm_scheme* s, int64_t K);

/* ---------------------------------------------------------------- setup [async]
 * Quantize W[N, K] (bf16, K contiguous) group-wise along K with the min-max rule:
 *   codes  [N, K] uint8 (asym, q in [0, 2^b-1]) or int8 (sym, |q| <= 2^(b-1)-1)
 *   scale  [N, K/g] bf16, the smallest bf16 s with (2^b-1)s >= max-min (asym) or (2^(b-1)-1)s >= max|x|
 *   zero   [N, K/g] bf16 = group min (asym); may be NULL when symmetric
 * fp64 arithmetic; results are bit-exact with the CPU oracle. w_bits = 16 is rejected (nothing to quantize).
 * A non-finite weight sets the device error word (MXM_E_DATA) if `err` is non-NULL (int32, device). */
mxm_status mxm_quantize(const mxm_scheme* s, const void* w_bf16, int64_t N, int64_t K, void* codes, void* scale,
                        void* zero, int32_t* err, mxm_stream stream);
/* Pack canonical codes/scale/zero into the native layout (docs/packed_format.md); `packed` has
 * mxm_quant_sizes(...).packed_bytes bytes. For w_bits = 16, `codes` is the bf16 weight and
 * scale/zero are ignored. */
mxm_status mxm_pack(const mxm_scheme* s, const void* codes, const void* scale, const void* zero, int64_t N, int64_t K,
                    void* packed, mxm_stream stream);
/* Test/debug: dequantize a packed block to float32 w_out[N, K] = q·s + z exactly (q·s sym). */
mxm_status mxm_dequantize(const mxm_scheme* s, const void* packed, int64_t N, int64_t K, float* w_out,
                          mxm_stream stream);

/* ---- NEXT-4: offline weight preparation (§4.2.3 "randomized Hadamard transformations ... using the
 * incoherence processing used in QuaRot, then ... GPTQ-based quantization"; "We disabled online rotations").
 * Readings DESIGN.md R22-R24. Not on the hot path: they produce the codes / scales / zeros mxm_pack consumes.
 * All arithmetic fp64; every pointer is device memory owned by the caller; async on `stream`. */
/* R22: out = W Q (axis 1: rotate along K, gate / up blocks) or Q^T W (axis 0: along N, down blocks) with
 * Q = blockdiag(diag(signs) H_128) / sqrt(128); w, out bf16 [N, K] row-major (not aliased), signs int8 (+-1) of
 * the rotated length (K or N, a multiple of 128). Each output is the fp64 result rounded once to bf16. */
mxm_status mxm_hadamard_rotate(const void* w_bf16, void* out_bf16, int64_t N, int64_t K, const int8_t* signs,
                               int32_t axis, mxm_stream stream);
/* R23: H[K, K] (fp64, row-major) = 2 X^T X / n over calibration rows x_bf16 [n, K]. */
mxm_status mxm_gptq_hessian(const void* x_bf16, int64_t n, int64_t K, double* H, mxm_stream stream);
/* R23 set-up: dead columns (H_jj = 0 -> 1, dead[j] = 1), damping H += percdamp mean(diag H) I, then U[K, K]
 * (fp64, row-major, upper) = the upper Cholesky factor of H^-1 (U^T U = H^-1) via the reverse Cholesky factor V
 * (H = V V^T) and U = V^-1. H is overwritten (scratch); `scratch` holds K*K doubles. MXM_E_CONFIG on bad args. */
mxm_status mxm_gptq_prepare(double* H, int64_t K, double percdamp, double* scratch, double* U, int32_t* dead,
                            mxm_stream stream);
/* Bytes of the fp64 work buffer mxm_gptq_quantize needs for an [N, K] block. */
int64_t mxm_gptq_work_bytes(int64_t N, int64_t K);
/* R23 / R24: GPTQ of one linear block w_bf16 [N, K] against U (from mxm_gptq_prepare on the block's input
 * Hessian): columns left to right in blocks of 128, lazy batch updates, group parameters from the current weights
 * at each group start (per channel: the initial weights). Output in mxm_quantize's canonical format: codes
 * [N, K] (u8 asymmetric / s8 symmetric), scale and zero bf16 [N, K/g] (zero may be NULL for symmetric). Weight-only
 * schemes of any bits, or the weight side of a W-A scheme; w_group in {64, 128, -1}. */
mxm_status mxm_gptq_quantize(const mxm_scheme* s, const void* w_bf16, int64_t N, int64_t K, const double* U,
                             const int32_t* dead, double* work, void* codes, void* scale, void* zero,
                             mxm_stream stream);

/* Test/debug: the dynamic activation quantizer of the hot path on v[M, K] bf16:
 *   codes [M, K] int8, scale [M, K/ga] float32, qsum [M, K/ga] int32 (may be NULL).
 *   r = fl32(qmax/amax), s = fl32(amax/qmax), q = clamp(rint(fl32(v·r)), ±qmax); amax = 0 -> s = 1, q = 0. */
mxm_status mxm_act_quant(const void* v_bf16, int64_t M, int64_t K, int32_t a_bits, int32_t a_group, void* codes,
                         float* scale, int32_t* qsum, mxm_stream stream);

/* Test/debug: the hot path's route preparation (step S1). topk_ids int32[T, k] (-1 = none).
 *   counts  int32[E]      routes per expert
 *   offsets int32[E + 1]  exclusive scan of counts
 *   perm    int32[T*k]    perm[p] = t*k + j of the route at sorted position p (stable in (t, j) order);
 *                         entries >= offsets[E] are left untouched
 *   err     int32 device word, set to MXM_E_DATA for an id outside [-1, E) (that route is skipped) */
/* [sync] device scratch bytes mxm_route_prep needs for T tokens, top-k k, E experts. */
mxm_status mxm_route_scratch_bytes(int64_t T, int32_t k, int32_t E, int64_t* bytes);
mxm_status mxm_route_prep(const int32_t* topk_ids, int64_t T, int32_t k, int32_t E, int32_t* counts,
                          int32_t* offsets, int32_t* perm, int32_t* err, void* scratch, int64_t scratch_bytes,
                          mxm_stream stream);

/* ---------------------------------------------------------------- layer (the per-block precision table)
 * blocks: host array [(n_routed + n_shared) * 3], order (expert-major) gate, up, down; gate/up are [inter, hidden]
 * (routed) or [shared_inter, hidden] (shared); down is [hidden, inter]. `packed` are device buffers from mxm_pack,
 * which must stay alive while the layer is used. Shared experts see every token (weight shared_w or 1).
 * Limits (MXM_E_CONFIG otherwise): 1 <= n_routed <= 256, 0 <= n_shared <= 32, n_routed + n_shared <= 256,
 * hidden, inter, shared_inter multiples of 128. */
typedef struct {
  mxm_scheme scheme;
  const void* packed;
} mxm_linear;
typedef struct {
  int32_t n_routed, n_shared, hidden, inter, shared_inter;
  const mxm_linear* blocks;
} mxm_layer_desc;
typedef struct mxm_layer mxm_layer;

/* [sync] device bytes needed for the layer's descriptor table. */
mxm_status mxm_layer_desc_bytes(const mxm_layer_desc* d, int64_t* bytes);
/* [sync] validate every block, upload the descriptor table into desc_dev (caller-owned device buffer of
 * mxm_layer_desc_bytes bytes), return a host handle. tile_costs: NULL = analytic LPT cost model, else a HOST
 * float array [(n_routed + n_shared) * 4]: the measured cost (ms) of one m-tile group of each expert at token
 * tiles 16 / 32 / 64 / 96 (the output of mxm_profile_tile_costs; entries <= 0 fall back to the analytic model).
 * The planner orders m-tile groups by this cost, longest first (greedy LPT, "pre-profiled single-tile
 * runtime costs"). */
mxm_status mxm_layer_init(const mxm_layer_desc* d, void* desc_dev, int64_t desc_bytes, const void* tile_costs,
                          mxm_layer** out);
void mxm_layer_free(mxm_layer* l);
/* [sync] workspace bytes for calls with up to max_tokens tokens and top_k routes per token. */
mxm_status mxm_workspace_bytes(const mxm_layer* l, int64_t max_tokens, int32_t top_k, int64_t* bytes);

/* [async] The mixed-precision MoE group-GEMM (the hot path):
 *   x        bf16 [T, hidden]
 *   topk_ids int32 [T, top_k], -1 = no route; duplicates allowed (each contributes)
 *   topk_w   float32 [T, top_k] routing weights (used as given)
 *   shared_w float32 [T, n_shared] or NULL (= 1.0)
 *   y        bf16 [T, hidden] (output; fully overwritten)
 *   workspace device buffer of >= mxm_workspace_bytes(l, T, top_k) bytes, exclusive to this call.
 * One persistent launch runs all gate/up/down tiles of all experts (LPT-ordered task queue);
 * route-prep, activation quantize+gather, planning and the top-k combine are separate short launches.
 * Deterministic: identical inputs give bitwise identical y. */
mxm_status mxm_moe_group_gemm(const mxm_layer* l, const void* x, int64_t T, int32_t top_k, const int32_t* topk_ids,
                              const float* topk_w, const float* shared_w, void* y, void* workspace, int64_t ws_bytes,
                              mxm_stream stream);
/* Tile-cost profiling (the cost model and scheduler use pre-profiled single-tile runtime costs).
 * [sync] bytes of the caller-owned device scratch mxm_profile_tile_costs needs (a workspace for 96 tokens plus
 * its inputs and output). */
mxm_status mxm_profile_scratch_bytes(const mxm_layer* l, int64_t* bytes);
/* [sync] measure, on this GPU, the cost of one m-tile group of every expert at each token tile (16, 32, 64, 96;
 * capped at the expert's largest tile): the persistent group-GEMM is launched on ONE CTA over zero inputs routed
 * to that expert only (split-K off), timed with CUDA events, best of 3, minus the same run with no routed token
 * (shared experts only; their cost is that run divided by n_shared). costs: HOST float [(n_routed+n_shared)*4], ms. */
mxm_status mxm_profile_tile_costs(const mxm_layer* l, void* scratch, int64_t scratch_bytes, float* costs,
                                  mxm_stream stream);
/* [sync] replace the layer's tile-cost table (HOST float [(n_routed+n_shared)*4], ms; NULL = analytic model). */
mxm_status mxm_layer_set_tile_costs(mxm_layer* l, const float* costs);

/* [sync] read (and clear) the device error word of the last call using `workspace`: *code = MXM_OK or MXM_E_DATA. */
mxm_status mxm_poll_device_error(const mxm_layer* l, const void* workspace, mxm_stream stream, int32_t* code);
/* Test/debug [sync]: number of tile tasks (gate/up, h-quant, down) the planner emitted in the last call
 * on `workspace` (made with these T, top_k) and the number the persistent kernel executed (must be equal:
 * every task runs exactly once). */
mxm_status mxm_debug_task_stats(const mxm_layer* l, const void* workspace, int64_t T, int32_t top_k,
                                mxm_stream stream, int32_t* n_tasks, int32_t* n_executed);

/* Profiling (bench / tests): record CUDA events around every launch of the next calls in a ring of
 * n_slots calls (0 disables). [sync] allocation. */
mxm_status mxm_layer_profile(mxm_layer* l, int32_t n_slots);
/* [sync] per-stage device milliseconds of the recorded calls, ms[i*5 + s] for stage s =
 * route-prep, act-quant+gather, plan, persistent group-GEMM, combine (oldest ring slot first is NOT
 * guaranteed: slot i = call i mod n_slots). */
mxm_status mxm_layer_profile_read(mxm_layer* l, float* ms, int32_t n, int32_t* n_recorded);
/* Debug: accumulate per-CTA cycle counters of the persistent kernel's wait sites into dev_buf
 * (uint64 [num_SMs][16], caller-zeroed; NULL disables). Slots: 0 producer ring-slot wait, 1 producer
 * stage-free wait, 2 producer dependency wait, 3-6 MMA waits (task, accumulator, data, transform),
 * 7-8 transform waits (task, data), 9-10 epilogue waits (task, accumulator), 13 MMA stages issued,
 * 14 h-quant dependency wait, 15 kernel cycles. Only a library built with -DMXM_DEBUG_COUNTERS records
 * them (the product build compiles the counters out); otherwise a non-NULL dev_buf is MXM_E_CONFIG. */
mxm_status mxm_layer_debug_counters(mxm_layer* l, void* dev_buf);
/* Number of library kernels one mxm_moe_group_gemm call launches (route x3-4, gather, plan, GEMM, combine). */
int32_t mxm_kernels_per_call(const mxm_layer* l);

/* ---------------------------------------------------------------- test-only introspection of the hot path
 * Byte offsets (into the workspace of a call with T tokens, top_k routes) of the intermediate buffers the
 * hot path writes, so that tests can compare them with the oracle after a real mxm_moe_group_gemm call.
 * off[MXM_WS_N]; -1 = not allocated for this layer. Route rows: R = T*top_k + T*n_shared (shared experts'
 * rows s*T + t first, then routed rows sorted by expert, stable in (t, j)).
 *   ROW_SRC int32[R] source token   ROW_W f32[R] route weight   ROW_EXP int32[R] expert   INV int32[T*k]
 *   XB bf16[R][hidden]          gathered bf16 gate/up input (weight-only / bf16 experts)
 *   XQA/XQB int8[R][hidden]     activation codes of input slots A/B (two's complement for a5/a8; for a4 the
 *                               e4m3 byte (q<0)<<7 | |q|, whose value is q * 2^-9)
 *   XSA/XSB f32[G][R]           activation scales, group-major (G = hidden/128, or 1 per-token)
 *   XCA/XCB int32[G][R]         per-group sum of the a4 codes (offset-binary correction of w4a4 blocks)
 *   H bf16, HQ int8: h rows in two regions, the T*n_shared shared rows [T*S][shared_inter] first, then the
 *                               T*k routed rows [T*k][inter] (row r >= T*S at (T*S*shared_inter + (r-T*S)*inter))
 *   HS f32[G][R]  HC int32[G][R]  scales / code sums of h (G = F/128, F = max inter, entry F_MAX)
 *   O bf16[R][hidden]           per-route down output o * w_e
 *   V_OFF int32[E+S+1] first row of each (virtual) expert;  R and F_MAX are values, not offsets.
 *   TASKS 16-byte records {u16 expert, u8 phase, u8 nt, i32 row0, u16 rows, u16 ntile, i32 gid} in queue order
 *   META int32: [0] tasks, [1..3] tasks per phase, [4] m-tile groups G, [5] queue head, [6] executed, [7] split-K
 *                slices, then the group table grp_v / grp_row0 / grp_rows / grp_nt, G_MAX entries each;
 *                G_MAX is a value. */
enum {
  MXM_WS_ROW_SRC = 0, MXM_WS_ROW_W, MXM_WS_ROW_EXP, MXM_WS_INV, MXM_WS_XB, MXM_WS_XQA, MXM_WS_XSA, MXM_WS_XQB,
  MXM_WS_XSB, MXM_WS_H, MXM_WS_HQ, MXM_WS_HS, MXM_WS_O, MXM_WS_V_OFF, MXM_WS_R, MXM_WS_F_MAX, MXM_WS_XCA,
  MXM_WS_XCB, MXM_WS_HC, MXM_WS_TASKS, MXM_WS_META, MXM_WS_G_MAX, MXM_WS_N
};
mxm_status mxm_debug_workspace_layout(const mxm_layer* l, int64_t T, int32_t top_k, int64_t* off);
/* [sync] bytes of the accumulator dump buffer of mxm_debug_moe_group_gemm_dump for T tokens and top_k. */
mxm_status mxm_debug_acc_bytes(const mxm_layer* l, int64_t T, int32_t top_k, int64_t* bytes);
/* [async] mxm_moe_group_gemm (same arguments and result) through a test-only instantiation of the persistent
 * kernel that also stores, before each drain, the raw 32-bit accumulator of every weight-activation block:
 *   acc uint32: gate / up [2][hidden/128][R][F], then down [F/128][R][hidden] (F = max inter): element
 *   [j][g][row][n] = accumulator of block j (0 gate, 1 up, 2 down) over K-group g (g = 0 for per-channel
 *   blocks) for route row `row`, output channel n.
 *   i8-kind blocks (w5a5, w8a8): the int32 sum_k q_w q_a. f8-kind blocks (w4a4): the fp32 bits of
 *   2^-18 * sum_k (q_w + 8) q_a (exact). Entries of other blocks are left untouched.
 * Split-K is disabled, so every accumulator covers the whole group (or the whole K). For weight-activation
 * downs quantized in the gate/up epilogue (g128) the bf16 h is also written to the H buffer. */
mxm_status mxm_debug_moe_group_gemm_dump(const mxm_layer* l, const void* x, int64_t T, int32_t top_k,
                                         const int32_t* topk_ids, const float* topk_w, const float* shared_w, void* y,
                                         void* workspace, int64_t ws_bytes, void* acc, int64_t acc_bytes,
                                         mxm_stream stream);

/* ---------------------------------------------------------------- expert parallelism
 * Rank r of G owns routed experts [r*E/G, (r+1)*E/G); tokens stay on their source rank. The host runtime
 * exchanges counts and rows with NCCL all-to-all(v) (torch.distributed on ProcessGroupNCCL); these calls
 * build the send buffers and combine the returned partial sums. All pointers are device pointers.
 *
 * [async] per destination rank: how many of this rank's T tokens have >= 1 routed expert there (dedup),
 *   dest_counts int32[G]; pos int32[T, G] = stable slot of token t in destination r's block, or -1. */
mxm_status mxm_ep_route(const int32_t* topk_ids, int64_t T, int32_t k, int32_t E, int32_t G, int32_t* dest_counts,
                        int32_t* pos, int32_t* err, mxm_stream stream);
/* [async] send rows ordered by (destination, token): send_x bf16 [S, d] (S = sum dest_counts), send_ids int32
 *   [S, k] local expert ids (id - r*E/G) or -1 for experts hosted elsewhere, send_w f32 [S, k], send_src int32 [S].
 *   dest_offsets int32[G+1] = exclusive scan of dest_counts (device). */
mxm_status mxm_ep_pack(const void* x, int64_t T, int32_t d, const int32_t* topk_ids, const float* topk_w, int32_t k,
                       int32_t E, int32_t G, const int32_t* pos, const int32_t* dest_offsets, void* send_x,
                       int32_t* send_ids, float* send_w, int32_t* send_src, mxm_stream stream);
/* [async] y[t] = bf16( sum over destinations r ascending of back[dest_offsets[r] + pos[t, r]] + y_shared[t] );
 *   back bf16 [S, d] = partial block outputs returned in send order; y_shared bf16 [T, d] or NULL. */
mxm_status mxm_ep_combine(const void* back, const int32_t* pos, const int32_t* dest_offsets, int32_t G, int64_t T,
                          int32_t d, const void* y_shared, void* y, mxm_stream stream);

/* ---------------------------------------------------------------- expert parallelism through the C ABI
 * One MoE layer sharded by experts over an NCCL communicator (Eq. 2 is a sum over experts,
 * P:71-73). `local`: this rank's routed experts [rank*E/G, (rank+1)*E/G) as a layer with n_shared = 0; `shared`:
 * the replicated shared experts as a layer of n_shared "routed" experts with n_shared = 0 (or NULL). nccl_comm is
 * a ncclComm_t borrowed from the caller (e.g. torch's ProcessGroupNCCL._comm_ptr()); it is never destroyed here.
 * [sync] create / [sync] free: */
typedef struct mxm_ep mxm_ep;
mxm_status mxm_ep_init(mxm_layer* local, mxm_layer* shared, void* nccl_comm, int32_t n_global_experts, mxm_ep** out);
void mxm_ep_free(mxm_ep* ep);
/* [sync] workspace bytes for T own tokens, top_k routes and at most max_recv_rows rows received from all ranks
 * (<= world_size * T; each token is sent once per destination rank hosting one of its experts). */
mxm_status mxm_ep_workspace_bytes(const mxm_ep* ep, int64_t T, int32_t top_k, int64_t max_recv_rows, int64_t* bytes);
/* Same arguments and result as mxm_moe_group_gemm with GLOBAL expert ids, for this rank's T tokens: the counts are
 * exchanged with NCCL (one host synchronisation for the all-to-all-v split sizes, v1), rows + local (id, weight)
 * are dispatched with grouped ncclSend/ncclRecv, the local group-GEMM runs on the received rows, the partial
 * outputs return, the shared experts run on the own tokens, and y = bf16(sum over destination ranks ascending of
 * the returned partials + shared), fixed order. MXM_E_CONFIG if more than max_recv_rows rows arrive;
 * MXM_E_NCCL on a communicator error. Every rank of the communicator must call it (collective). */
mxm_status mxm_ep_moe_group_gemm(mxm_ep* ep, const void* x, int64_t T, int32_t top_k, const int32_t* topk_ids,
                                 const float* topk_w, const float* shared_w, void* y, void* workspace, int64_t ws_bytes,
                                 int64_t max_recv_rows, mxm_stream stream);
/* [sync] dispatch mode of the handle (NEXT-1 step; default MXM_EP_V1 as above). MXM_EP_SYNC_FREE: no host
 * synchronisation at all -- every rank reserves T rows per destination (a token goes to a rank at most once), the
 * exchanges use fixed equal counts, rows no token fills carry expert id -1 (no route, skipped by the local layer),
 * the shared experts' ids / unit weights are written by a kernel. Requires the same T on every rank and
 * max_recv_rows >= world_size * T (else MXM_E_CONFIG). The valid rows reach the local layer in the same relative
 * order as in v1, so y is bitwise identical; the padding travels over the links. MXM_E_CONFIG on a bad mode. */
enum { MXM_EP_V1 = 0, MXM_EP_SYNC_FREE = 1 };
mxm_status mxm_ep_set_mode(mxm_ep* ep, int32_t mode);
/* [sync] read and clear the EP workspace's error word (bad expert ids in topk_ids -> MXM_E_DATA). */
mxm_status mxm_ep_poll_device_error(const mxm_ep* ep, const void* workspace, mxm_stream stream, int32_t* code);

/* Thread-local message for the last error returned on this thread. */
const char* mxm_last_error(void);
/* Library version string. */
const char* mxm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MXMOE_H */
