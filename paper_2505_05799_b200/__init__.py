"""B200-native MxMoE mixed-precision MoE group-GEMM — thin torch binding over libmxmoe.so.

Every function marshals torch CUDA tensors into the C ABI of include/mxmoe.h and runs on
torch's current stream. All computation happens in the CUDA kernels of csrc/; nothing here
computes (there is no CPU or eager fallback).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import torch

from . import _lib
from ._lib import MxmError, check, load  # noqa: F401

__all__ = ["Scheme", "quantize", "pack", "quantize_pack", "dequantize", "act_quant", "route_prep", "MoELayer",
           "storage_bits_per_weight", "quant_sizes", "MxmError"]


@dataclass(frozen=True)
class Scheme:
    """`wxay_gz_{sym,asym}`: a_bits 16 = weight-only; w_bits 16 = bf16."""

    w_bits: int
    a_bits: int = 16
    w_group: int = -1
    a_group: int = -1
    symmetric: bool = False
    fmt: int = 0  # 0 integer codes, 1 FP8 e4m3 (MXM_FMT_E4M3)

    def c(self) -> _lib.mxm_scheme:
        return _lib.mxm_scheme(self.w_bits, self.a_bits, self.w_group, self.a_group, 1 if self.symmetric else 0,
                               self.fmt)

    @staticmethod
    def of(s) -> "Scheme":
        return s if isinstance(s, Scheme) else Scheme(s.w_bits, s.a_bits, s.w_group, s.a_group, bool(s.symmetric),
                                                      int(getattr(s, "fmt", 0)))


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def quant_sizes(scheme, N: int, K: int) -> Tuple[int, int, int, int]:
    s = Scheme.of(scheme).c()
    cb, sb, zb, pb = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    check(load().mxm_quant_sizes(C.byref(s), N, K, C.byref(cb), C.byref(sb), C.byref(zb), C.byref(pb)))
    return cb.value, sb.value, zb.value, pb.value


def storage_bits_per_weight(scheme, K: int) -> float:
    s = Scheme.of(scheme).c()
    return load().mxm_storage_bits_per_weight(C.byref(s), K)


def quantize(scheme, w: torch.Tensor, err: Optional[torch.Tensor] = None):
    """W[N,K] bf16 (cuda) -> (codes uint8/int8 [N,K], scale bf16 [N,K/g], zero bf16 [N,K/g] or None)."""
    sch = Scheme.of(scheme)
    N, K = w.shape
    assert w.dtype == torch.bfloat16 and w.is_cuda and w.is_contiguous()
    g = K if sch.w_group == -1 else sch.w_group
    codes = torch.empty(N, K, dtype=torch.int8 if sch.symmetric or sch.a_bits != 16 else torch.uint8, device=w.device)
    scale = torch.empty(N, K // g, dtype=torch.bfloat16, device=w.device)
    zero = None if (sch.symmetric or sch.a_bits != 16) else torch.empty(N, K // g, dtype=torch.bfloat16,
                                                                           device=w.device)
    s = sch.c()
    check(load().mxm_quantize(C.byref(s), _ptr(w), N, K, _ptr(codes), _ptr(scale), _ptr(zero), _ptr(err), _stream()))
    return codes, scale, zero


def pack(scheme, codes: torch.Tensor, scale, zero, N: int, K: int) -> torch.Tensor:
    sch = Scheme.of(scheme)
    _, _, _, pb = quant_sizes(sch, N, K)
    out = torch.empty(pb, dtype=torch.uint8, device=codes.device)
    s = sch.c()
    check(load().mxm_pack(C.byref(s), _ptr(codes), _ptr(scale), _ptr(zero), N, K, _ptr(out), _stream()))
    return out


def quantize_pack(scheme, w: torch.Tensor) -> torch.Tensor:
    sch = Scheme.of(scheme)
    N, K = w.shape
    if sch.w_bits == 16:
        return pack(sch, w.contiguous(), None, None, N, K)
    codes, scale, zero = quantize(sch, w)
    return pack(sch, codes, scale, zero, N, K)


def dequantize(scheme, packed: torch.Tensor, N: int, K: int) -> torch.Tensor:
    out = torch.empty(N, K, dtype=torch.float32, device=packed.device)
    s = Scheme.of(scheme).c()
    check(load().mxm_dequantize(C.byref(s), _ptr(packed), N, K, _ptr(out), _stream()))
    return out


def hadamard_rotate(w: torch.Tensor, signs: torch.Tensor, axis: int) -> torch.Tensor:
    """R22 (mxm_hadamard_rotate): W Q (axis 1, along K) or Q^T W (axis 0, along N); w bf16 [N, K], signs int8 +-1."""
    assert w.dtype == torch.bfloat16 and w.is_cuda and w.is_contiguous() and w.dim() == 2
    assert signs.dtype == torch.int8 and signs.is_cuda and signs.is_contiguous()
    assert signs.numel() == (w.shape[1] if axis == 1 else w.shape[0])
    out = torch.empty_like(w)
    check(load().mxm_hadamard_rotate(_ptr(w), _ptr(out), w.shape[0], w.shape[1], _ptr(signs), axis, _stream()))
    return out


def gptq_hessian(x: torch.Tensor) -> torch.Tensor:
    """R23 (mxm_gptq_hessian): H = 2 X^T X / n, fp64 [K, K], from calibration rows x bf16 [n, K]."""
    assert x.dtype == torch.bfloat16 and x.is_cuda and x.is_contiguous() and x.dim() == 2
    n, K = x.shape
    H = torch.empty(K, K, dtype=torch.float64, device=x.device)
    check(load().mxm_gptq_hessian(_ptr(x), n, K, _ptr(H), _stream()))
    return H


def gptq_prepare(H: torch.Tensor, percdamp: float = 0.01):
    """R23 (mxm_gptq_prepare): (U fp64 [K, K] upper, U^T U = (H + damping)^-1; dead int32 [K]). H is consumed."""
    assert H.dtype == torch.float64 and H.is_cuda and H.is_contiguous()
    K = H.shape[0]
    U = torch.empty(K, K, dtype=torch.float64, device=H.device)
    scratch = torch.empty(K, K, dtype=torch.float64, device=H.device)
    dead = torch.empty(K, dtype=torch.int32, device=H.device)
    check(load().mxm_gptq_prepare(_ptr(H), K, float(percdamp), _ptr(scratch), _ptr(U), _ptr(dead), _stream()))
    return U, dead


def gptq_quantize(scheme, w: torch.Tensor, U: torch.Tensor, dead: torch.Tensor):
    """R23/R24 (mxm_gptq_quantize): GPTQ codes / scale / zero of w bf16 [N, K] in mxm_quantize's format."""
    sch = Scheme.of(scheme)
    N, K = w.shape
    assert w.dtype == torch.bfloat16 and w.is_cuda and w.is_contiguous()
    assert U.dtype == torch.float64 and U.shape == (K, K) and dead.dtype == torch.int32 and dead.numel() == K
    g = K if sch.w_group == -1 else sch.w_group
    sym = sch.symmetric or sch.a_bits != 16
    codes = torch.empty(N, K, dtype=torch.int8 if sym else torch.uint8, device=w.device)
    scale = torch.empty(N, K // g, dtype=torch.bfloat16, device=w.device)
    zero = None if sym else torch.empty(N, K // g, dtype=torch.bfloat16, device=w.device)
    work = torch.empty(load().mxm_gptq_work_bytes(N, K), dtype=torch.uint8, device=w.device)
    s = sch.c()
    check(load().mxm_gptq_quantize(C.byref(s), _ptr(w), N, K, _ptr(U), _ptr(dead), _ptr(work), _ptr(codes),
                                   _ptr(scale), _ptr(zero), _stream()))
    return codes, scale, zero


def act_quant(v: torch.Tensor, a_bits: int, a_group: int = -1):
    """Dynamic activation quantizer on v[M,K] bf16 -> (codes int8, scale f32 [M,K/g], qsum int32)."""
    M, K = v.shape
    g = K if a_group == -1 else a_group
    codes = torch.empty(M, K, dtype=torch.int8, device=v.device)
    scale = torch.empty(M, K // g, dtype=torch.float32, device=v.device)
    qsum = torch.empty(M, K // g, dtype=torch.int32, device=v.device)
    check(load().mxm_act_quant(_ptr(v), M, K, a_bits, a_group, _ptr(codes), _ptr(scale), _ptr(qsum), _stream()))
    return codes, scale, qsum


def route_prep(topk_ids: torch.Tensor, E: int):
    """Step S1 on its own: (counts int32[E], offsets int32[E+1], perm int32[T*k], err int32[1])."""
    T, k = topk_ids.shape
    dev = topk_ids.device
    counts = torch.zeros(E, dtype=torch.int32, device=dev)
    offsets = torch.zeros(E + 1, dtype=torch.int32, device=dev)
    perm = torch.full((T * k,), -1, dtype=torch.int32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    nb = C.c_int64(0)
    check(load().mxm_route_scratch_bytes(T, k, E, C.byref(nb)))
    scratch = torch.empty(max(256, nb.value), dtype=torch.uint8, device=dev)
    check(load().mxm_route_prep(_ptr(topk_ids.contiguous()), T, k, E, _ptr(counts), _ptr(offsets), _ptr(perm),
                                _ptr(err), _ptr(scratch), scratch.numel(), _stream()))
    return counts, offsets, perm, err


class MoELayer:
    """A quantized MoE layer: the per-(expert, block) precision table + packed weights on the GPU.

    blocks: list over experts (routed then shared) of 3 (scheme, packed uint8 tensor) pairs
    (gate, up, down), packed with `quantize_pack`.
    """

    def __init__(self, n_routed: int, n_shared: int, hidden: int, inter: int, shared_inter: int,
                 blocks: Sequence[Sequence[Tuple[Scheme, torch.Tensor]]], device="cuda"):
        lib = load()
        self.n_routed, self.n_shared, self.hidden, self.inter, self.shared_inter = (n_routed, n_shared, hidden, inter,
                                                                                     shared_inter)
        V = n_routed + n_shared
        assert len(blocks) == V and all(len(b) == 3 for b in blocks)
        self._packed = [p for b in blocks for (_, p) in b]  # keep alive
        self.schemes = [[Scheme.of(s) for (s, _) in b] for b in blocks]
        arr = (_lib.mxm_linear * (3 * V))()
        for v in range(V):
            for j in range(3):
                s, p = blocks[v][j]
                arr[3 * v + j].scheme = Scheme.of(s).c()
                arr[3 * v + j].packed = p.data_ptr()
        self._desc = _lib.mxm_layer_desc(n_routed, n_shared, hidden, inter, shared_inter, arr)
        self._arr = arr
        nb = C.c_int64()
        check(lib.mxm_layer_desc_bytes(C.byref(self._desc), C.byref(nb)))
        self._desc_dev = torch.empty(nb.value, dtype=torch.uint8, device=device)
        h = C.c_void_p()
        check(lib.mxm_layer_init(C.byref(self._desc), _ptr(self._desc_dev), nb.value, None, C.byref(h)))
        self._h = h
        self._ws = None

    @classmethod
    def from_weights(cls, n_routed: int, n_shared: int, hidden: int, inter: int, shared_inter: int,
                     weights: Sequence[Sequence[torch.Tensor]], table: Sequence[Sequence[Scheme]]) -> "MoELayer":
        """Quantize + pack every (expert, block) on the GPU (mxm_quantize / mxm_pack) and build the layer.

        weights[v] = (W_gate [f, d], W_up [f, d], W_down [d, f]) bf16 CUDA tensors; table[v] = 3 schemes.
        """
        blocks = []
        for v in range(n_routed + n_shared):
            blocks.append([(Scheme.of(table[v][j]), quantize_pack(table[v][j], weights[v][j].contiguous()))
                           for j in range(3)])
        return cls(n_routed, n_shared, hidden, inter, shared_inter, blocks, device=weights[0][0].device)

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None and self._h.value:
                load().mxm_layer_free(self._h)
        except Exception:
            pass

    def workspace_bytes(self, T: int, top_k: int) -> int:
        nb = C.c_int64()
        check(load().mxm_workspace_bytes(self._h, T, top_k, C.byref(nb)))
        return nb.value

    def workspace(self, T: int, top_k: int) -> torch.Tensor:
        nb = self.workspace_bytes(T, top_k)
        if self._ws is None or self._ws.numel() < nb:
            self._ws = torch.empty(nb, dtype=torch.uint8, device=self._desc_dev.device)
        return self._ws

    def _check_args(self, x, topk_ids, topk_w, shared_w, out):
        # every tensor is read as raw memory by the kernels: check dtype, shape, contiguity and device here
        dev = self._desc_dev.device
        T = x.shape[0]
        assert x.dtype == torch.bfloat16 and x.is_contiguous() and tuple(x.shape) == (T, self.hidden), "x [T, hidden] bf16"
        assert topk_ids.dtype == torch.int32 and topk_ids.is_contiguous() and topk_ids.dim() == 2 \
            and topk_ids.shape[0] == T, "topk_ids [T, k] int32 contiguous"
        k = topk_ids.shape[1]
        assert topk_w.dtype == torch.float32 and topk_w.is_contiguous() and tuple(topk_w.shape) == (T, k), \
            "topk_w [T, k] float32 contiguous"
        if shared_w is not None:
            assert shared_w.dtype == torch.float32 and shared_w.is_contiguous() and \
                tuple(shared_w.shape) == (T, self.n_shared), "shared_w [T, n_shared] float32 contiguous"
        if out is not None:
            assert out.dtype == torch.bfloat16 and out.is_contiguous() and tuple(out.shape) == (T, self.hidden)
        for t in (x, topk_ids, topk_w, shared_w, out):
            assert t is None or t.device == dev, "all tensors on the layer's device"
        return T, k

    def __call__(self, x: torch.Tensor, topk_ids: torch.Tensor, topk_w: torch.Tensor,
                 shared_w: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                 workspace: Optional[torch.Tensor] = None) -> torch.Tensor:
        T, k = self._check_args(x, topk_ids, topk_w, shared_w, out)
        if out is None:
            out = torch.empty(T, self.hidden, dtype=torch.bfloat16, device=x.device)
        ws = workspace if workspace is not None else self.workspace(T, k)
        check(load().mxm_moe_group_gemm(self._h, _ptr(x), T, k, _ptr(topk_ids), _ptr(topk_w), _ptr(shared_w),
                                        _ptr(out), _ptr(ws), ws.numel(), _stream()))
        return out

    # ---------------------------------------------------------------- test-only introspection
    def workspace_layout(self, T: int, top_k: int) -> dict:
        """Byte offsets of the hot path's intermediate buffers (mxm_debug_workspace_layout; -1 = absent)."""
        off = (C.c_int64 * len(_lib.WS_NAMES))()
        check(load().mxm_debug_workspace_layout(self._h, T, top_k, off))
        return {n: int(off[i]) for i, n in enumerate(_lib.WS_NAMES)}

    def call_dump(self, x, topk_ids, topk_w, shared_w=None):
        """mxm_moe_group_gemm through the accumulator-dump kernel: (y, workspace, acc_gu, acc_down).

        acc_gu int32 [2, hidden/128, R, F] (gate, up), acc_down int32 [F/128, R, hidden]; raw 32-bit words.
        """
        T, k = self._check_args(x, topk_ids, topk_w, shared_w, None)
        nb = C.c_int64()
        check(load().mxm_debug_acc_bytes(self._h, T, k, C.byref(nb)))
        lay = self.workspace_layout(T, k)
        R, F, d = lay["R"], lay["f_max"], self.hidden
        acc = torch.zeros(nb.value // 4, dtype=torch.int32, device=x.device)
        ws = torch.zeros(self.workspace_bytes(T, k), dtype=torch.uint8, device=x.device)
        y = torch.empty(T, self.hidden, dtype=torch.bfloat16, device=x.device)
        check(load().mxm_debug_moe_group_gemm_dump(self._h, _ptr(x), T, k, _ptr(topk_ids), _ptr(topk_w),
                                                   _ptr(shared_w), _ptr(y), _ptr(ws), ws.numel(), _ptr(acc),
                                                   nb.value, _stream()))
        n_gu = 2 * (d // 128) * R * F
        return y, ws, acc[:n_gu].view(2, d // 128, R, F), acc[n_gu:].view(F // 128, R, d)

    def profile_tile_costs(self):
        """Measured m-tile group costs (ms) [V, 4] for token tiles 16/32/64/96 (mxm_profile_tile_costs)."""
        import numpy as np
        nb = C.c_int64()
        check(load().mxm_profile_scratch_bytes(self._h, C.byref(nb)))
        scratch = torch.empty(nb.value, dtype=torch.uint8, device=self._desc_dev.device)
        V = self.n_routed + self.n_shared
        out = (C.c_float * (4 * V))()
        check(load().mxm_profile_tile_costs(self._h, _ptr(scratch), nb.value, out, _stream()))
        return np.frombuffer(out, dtype=np.float32).reshape(V, 4).copy()

    def set_tile_costs(self, costs):
        """Use a measured cost table [V, 4] (ms) as the planner's LPT key (None: the analytic model)."""
        import numpy as np
        if costs is None:
            check(load().mxm_layer_set_tile_costs(self._h, None))
            return
        arr = np.ascontiguousarray(costs, dtype=np.float32).reshape(-1)
        assert arr.size == 4 * (self.n_routed + self.n_shared)
        check(load().mxm_layer_set_tile_costs(self._h, arr.ctypes.data_as(C.c_void_p)))

    def profile(self, n_slots: int):
        """Record per-stage CUDA events for the next calls (ring of n_slots calls)."""
        check(load().mxm_layer_profile(self._h, n_slots))

    def profile_read(self, n: int):
        """[n_recorded, 5] stage milliseconds: route, gather, plan, gemm, combine."""
        import numpy as np
        buf = (C.c_float * (5 * n))()
        got = C.c_int32()
        check(load().mxm_layer_profile_read(self._h, buf, n, C.byref(got)))
        return np.frombuffer(buf, dtype=np.float32).reshape(n, 5)[: got.value].copy()

    def debug_counters(self, buf: Optional[torch.Tensor]):
        """Attach (or detach with None) a zeroed uint64 device buffer [num_SMs, 16] of wait-site cycle counters."""
        check(load().mxm_layer_debug_counters(self._h, _ptr(buf)))

    @property
    def kernels_per_call(self) -> int:
        return int(load().mxm_kernels_per_call(self._h))

    def poll_error(self, workspace: Optional[torch.Tensor] = None) -> int:
        code = C.c_int32()
        ws = workspace if workspace is not None else self._ws
        check(load().mxm_poll_device_error(self._h, _ptr(ws), _stream(), C.byref(code)))
        return code.value

    def task_stats(self, T: int, top_k: int, workspace: Optional[torch.Tensor] = None) -> Tuple[int, int]:
        a, b = C.c_int32(), C.c_int32()
        ws = workspace if workspace is not None else self._ws
        check(load().mxm_debug_task_stats(self._h, _ptr(ws), T, top_k, _stream(), C.byref(a), C.byref(b)))
        return a.value, b.value
