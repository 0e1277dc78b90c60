"""Expert-parallel MoE block over a torch.distributed process group.

Eq. 2 is a sum over experts, so the block shards by experts: rank r of G owns
routed experts [r·E/G, (r+1)·E/G); tokens stay data-parallel on their source rank; shared experts
are replicated and run on each rank's own tokens.

Per call, v1 (one NCCL all-to-all for counts, then all-to-all-v for rows; host sync for split sizes):
  1. mxm_ep_route   per-destination dedup counts + stable slots        (kernel)
  2. all_to_all     counts                                              (NCCL)
  3. mxm_ep_pack    send rows + local (expert id, weight) metadata      (kernel)
  4. all_to_all_v   rows, ids, weights                                  (NCCL)
  5. local routed layer on the received rows (mxm_moe_group_gemm)       (kernels)
  6. all_to_all_v   partial outputs back, in send order                 (NCCL)
  7. shared experts on the own tokens (mxm_moe_group_gemm, top-k = S)   (kernels)
  8. mxm_ep_combine fixed-order sum over destinations + shared          (kernel)
Sync-free mode (NEXT-1 step, the default): no host read of any count. A token goes to a destination rank at
most once (the dispatch is deduplicated per destination), so every rank reserves C = T rows per destination:
the all-to-alls use fixed equal splits, padding rows carry expert id -1 (no route, skipped by the local layer's
route preparation and gather), and the reverse exchange and combine use the fixed offsets r * C. The valid rows
reach the local layer in the same relative order as in v1, so the result is bitwise identical (tests). Cost:
the padding travels (G * T rows each way instead of the routed ones); all ranks must pass the same T.
Index math and arithmetic run in libmxmoe kernels; this module only sizes buffers and issues the
collectives. `ops` and the two layers are injectable so the orchestration can be exercised with the
gloo backend on CPU (tests/test_ep_gloo.py).
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional, Sequence

import torch
import torch.distributed as dist

from . import MoELayer, Scheme, _ptr, _stream, check, load


class CudaEpOps:
    """The libmxmoe EP kernels (device tensors)."""

    def __init__(self):
        self.err = None  # device error word of the dispatch (bad expert ids -> MXM_E_DATA), see poll_error

    def route(self, ids: torch.Tensor, E: int, G: int):
        T, k = ids.shape
        counts = torch.zeros(G, dtype=torch.int32, device=ids.device)
        pos = torch.empty(T, G, dtype=torch.int32, device=ids.device)
        if self.err is None:
            self.err = torch.zeros(1, dtype=torch.int32, device=ids.device)
        check(load().mxm_ep_route(_ptr(ids), T, k, E, G, _ptr(counts), _ptr(pos), _ptr(self.err), _stream()))
        return counts, pos

    def poll_error(self) -> int:
        if self.err is None:
            return 0
        v = int(self.err.item())
        self.err.zero_()
        return v

    def pack(self, x, ids, w, pos, dest_off, E, G, S_total):
        T, k = ids.shape
        d = x.shape[1]
        dev = x.device
        sx = torch.empty(S_total, d, dtype=torch.bfloat16, device=dev)
        sids = torch.full((S_total, k), -1, dtype=torch.int32, device=dev)  # rows no token fills: no route
        sw = torch.zeros(S_total, k, dtype=torch.float32, device=dev)
        ssrc = torch.empty(S_total, dtype=torch.int32, device=dev)
        check(load().mxm_ep_pack(_ptr(x), T, d, _ptr(ids), _ptr(w), k, E, G, _ptr(pos), _ptr(dest_off), _ptr(sx),
                                 _ptr(sids), _ptr(sw), _ptr(ssrc), _stream()))
        return sx, sids, sw, ssrc

    def combine(self, back, pos, dest_off, G, ysh, T, d):
        y = torch.empty(T, d, dtype=torch.bfloat16, device=pos.device)
        check(load().mxm_ep_combine(_ptr(back), _ptr(pos), _ptr(dest_off), G, T, d, _ptr(ysh), _ptr(y), _stream()))
        return y


class ExpertParallelMoE:
    """One MoE layer sharded by experts over `group` (rank r owns routed experts [r·E/G, (r+1)·E/G))."""

    def __init__(self, n_routed: int, hidden: int, local_layer: Callable, shared_layer: Optional[Callable],
                 n_shared: int, group=None, ops=None, sync_free: bool = True):
        self.group = group
        self.sync_free = sync_free
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if n_routed % self.G:
            raise ValueError("n_routed must be divisible by the expert-parallel world size")
        self.E, self.S, self.d = n_routed, n_shared, hidden
        self.local, self.shared = local_layer, shared_layer
        self.ops = ops if ops is not None else CudaEpOps()

    @classmethod
    def from_weights(cls, n_routed: int, n_shared: int, hidden: int, inter: int, shared_inter: int,
                     weights: Sequence[Sequence[torch.Tensor]], table, group=None,
                     sync_free: bool = True) -> "ExpertParallelMoE":
        """weights/table cover all routed experts then the shared ones (as in MoELayer.from_weights);
        only this rank's experts (and the shared ones) are quantized and kept."""
        G, r = dist.get_world_size(group), dist.get_rank(group)
        epr = n_routed // G
        lo = r * epr
        local = MoELayer.from_weights(epr, 0, hidden, inter, 0, weights[lo:lo + epr],
                                      [[Scheme.of(s) for s in row] for row in table[lo:lo + epr]])
        shared = None
        if n_shared:
            shared = MoELayer.from_weights(n_shared, 0, hidden, shared_inter, 0, weights[n_routed:],
                                           [[Scheme.of(s) for s in row] for row in table[n_routed:]])
        return cls(n_routed, hidden, local, shared, n_shared, group, sync_free=sync_free)

    def _a2a(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits):
        dist.all_to_all_single(out, inp.contiguous(), out_splits, in_splits, group=self.group)

    def __call__(self, x: torch.Tensor, topk_ids: torch.Tensor, topk_w: torch.Tensor,
                 shared_w: Optional[torch.Tensor] = None) -> torch.Tensor:
        T, k = topk_ids.shape
        G, E, d, dev = self.G, self.E, self.d, x.device
        counts, pos = self.ops.route(topk_ids, E, G)
        if self.sync_free:
            return self._call_sync_free(x, topk_ids, topk_w, shared_w, pos)
        recv_counts = torch.empty_like(counts)
        dist.all_to_all_single(recv_counts, counts, group=self.group)
        send_splits = counts.tolist()  # host sync (v1): split sizes of the all-to-all-v
        recv_splits = recv_counts.tolist()
        dest_off_l = [0]
        for c in send_splits:
            dest_off_l.append(dest_off_l[-1] + c)
        dest_off = torch.tensor(dest_off_l, dtype=torch.int32, device=dev)
        sx, sids, sw, _ = self.ops.pack(x, topk_ids, topk_w, pos, dest_off, E, G, dest_off_l[-1])
        R = sum(recv_splits)
        rx = torch.empty(R, d, dtype=x.dtype, device=dev)
        rids = torch.empty(R, k, dtype=torch.int32, device=dev)
        rw = torch.empty(R, k, dtype=torch.float32, device=dev)
        self._a2a(rx, sx, recv_splits, send_splits)
        self._a2a(rids, sids, recv_splits, send_splits)
        self._a2a(rw, sw, recv_splits, send_splits)
        ry = self.local(rx, rids, rw) if R > 0 else torch.empty(0, d, dtype=x.dtype, device=dev)
        back = torch.empty(dest_off_l[-1], d, dtype=x.dtype, device=dev)
        self._a2a(back, ry, send_splits, recv_splits)
        return self.ops.combine(back, pos, dest_off, G, self._shared_out(x, shared_w, T), T, d)

    def _shared_out(self, x, shared_w, T):
        if not self.S:
            return None
        dev = x.device
        sid = torch.arange(self.S, dtype=torch.int32, device=dev).repeat(T, 1)
        swt = shared_w if shared_w is not None else torch.ones(T, self.S, dtype=torch.float32, device=dev)
        return self.shared(x, sid, swt.contiguous())

    def _call_sync_free(self, x, topk_ids, topk_w, shared_w, pos):
        """Fixed capacity C = T rows per destination: equal-split all-to-alls, no host sync (module docstring)."""
        T, k = topk_ids.shape
        G, E, d, dev = self.G, self.E, self.d, x.device
        cap = T
        dest_off = torch.arange(G + 1, dtype=torch.int32, device=dev) * cap
        sx, sids, sw, _ = self.ops.pack(x, topk_ids, topk_w, pos, dest_off, E, G, G * cap)
        rx = torch.empty(G * cap, d, dtype=x.dtype, device=dev)
        rids = torch.empty(G * cap, k, dtype=torch.int32, device=dev)
        rw = torch.empty(G * cap, k, dtype=torch.float32, device=dev)
        self._a2a(rx, sx, None, None)
        self._a2a(rids, sids, None, None)
        self._a2a(rw, sw, None, None)
        ry = self.local(rx, rids, rw) if G * cap > 0 else torch.empty(0, d, dtype=x.dtype, device=dev)
        back = torch.empty(G * cap, d, dtype=x.dtype, device=dev)
        self._a2a(back, ry, None, None)
        return self.ops.combine(back, pos, dest_off, G, self._shared_out(x, shared_w, T), T, d)


class CAbiExpertParallelMoE:
    """The same expert-parallel block through the library's own C ABI (mxm_ep_init / mxm_ep_moe_group_gemm):
    counts, rows and partial outputs move with NCCL inside libmxmoe on torch's communicator (_comm_ptr()),
    so a call is one library entry point per rank."""

    def __init__(self, local: MoELayer, shared: Optional[MoELayer], n_routed: int, group=None,
                 sync_free: bool = True):
        from torch.distributed.distributed_c10d import _get_default_group
        pg = group if group is not None else _get_default_group()
        comm = pg._get_backend(torch.device("cuda"))._comm_ptr()
        self.local, self.shared, self.E = local, shared, n_routed
        self.G = dist.get_world_size(group)
        h = C.c_void_p()
        check(load().mxm_ep_init(local._h, shared._h if shared is not None else None, C.c_void_p(comm), n_routed,
                                 C.byref(h)))
        self._h = h
        self._ws = None
        self.sync_free = sync_free
        check(load().mxm_ep_set_mode(h, 1 if sync_free else 0))  # MXM_EP_SYNC_FREE / MXM_EP_V1

    @classmethod
    def from_weights(cls, n_routed: int, n_shared: int, hidden: int, inter: int, shared_inter: int,
                     weights, table, group=None) -> "CAbiExpertParallelMoE":
        py = ExpertParallelMoE.from_weights(n_routed, n_shared, hidden, inter, shared_inter, weights, table, group)
        return cls(py.local, py.shared, n_routed, group)

    def set_sync_free(self, on: bool):
        check(load().mxm_ep_set_mode(self._h, 1 if on else 0))
        self.sync_free = on

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None and self._h.value:
                load().mxm_ep_free(self._h)
        except Exception:
            pass

    def workspace(self, T: int, k: int, max_recv: int) -> torch.Tensor:
        nb = C.c_int64()
        check(load().mxm_ep_workspace_bytes(self._h, T, k, max_recv, C.byref(nb)))
        if self._ws is None or self._ws.numel() < nb.value:
            self._ws = torch.zeros(nb.value, dtype=torch.uint8, device="cuda")
        return self._ws

    def __call__(self, x: torch.Tensor, topk_ids: torch.Tensor, topk_w: torch.Tensor,
                 shared_w: Optional[torch.Tensor] = None, max_recv: Optional[int] = None) -> torch.Tensor:
        T, k = topk_ids.shape
        assert x.dtype == torch.bfloat16 and x.is_contiguous() and topk_ids.dtype == torch.int32
        assert topk_ids.is_contiguous() and topk_w.dtype == torch.float32 and topk_w.is_contiguous()
        max_recv = self.G * T if max_recv is None else max_recv
        ws = self.workspace(T, k, max_recv)
        y = torch.empty(T, self.local.hidden, dtype=torch.bfloat16, device=x.device)
        check(load().mxm_ep_moe_group_gemm(self._h, _ptr(x), T, k, _ptr(topk_ids), _ptr(topk_w), _ptr(shared_w),
                                           _ptr(y), _ptr(ws), ws.numel(), max_recv, _stream()))
        return y

    def poll_error(self) -> int:
        code = C.c_int32()
        check(load().mxm_ep_poll_device_error(self._h, _ptr(self._ws), _stream(), C.byref(code)))
        return code.value
