"""Tensor-parallel paged LoRA for the hidden-dim-sharded configuration
(BASELINE configs[4]: Llama-2-70B q/v at 2/4/8 GPUs).

The S-LoRA scheme for a column-parallel base projection: TP rank i of N

  1. shrinks its rows [i·r/N, (i+1)·r/N) of every adapter:
     v_part = x · A[rows_i]ᵀ                         (plora_bgmv_tp_shrink)
  2. all-gathers v_part over the TP group (NCCL over NVLink; a T·r/N fp32
     message per rank, 4-32 KiB in total at cfg5)
  3. expands into its output-column shard:
     y[:, cols_i] += scale · v · Bᵀ[:, cols_i]       (plora_bgmv_tp_expand)

x is replicated across the group (the input of a column-parallel layer) and
y is the rank's output shard.  The reference has no multi-GPU path
(SPEC.md:8); the math is PAPER.md:64-69.  Every rank's pool holds the full
adapter pages; each rank reads only its shard (1/N of the adapter bytes).
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional, Sequence

import torch

from . import _native as N
from .lora import BatchPlan, current_stream_handle


def tp_shard_rows(plan: BatchPlan, tp_size: int) -> int:
    """Row stride (floats) of a v_part buffer: ceil(max rank / tp_size)."""
    return int(N.lib().plora_tp_shard_rows(plan.handle, tp_size))


def bgmv_tp_shrink(plan: BatchPlan, layer: int, proj: int, tp_rank: int, tp_size: int,
                   x: torch.Tensor, v_part: torch.Tensor, stream: int | None = None) -> torch.Tensor:
    """v_part[t, j] = x[t] · A_{a(t)}[tp_rank·r/N + j]ᵀ (fp32, [T, rs])."""
    if not (x.is_cuda and v_part.is_cuda) or v_part.dtype != torch.float32:
        raise N.ValidationError("x and v_part must be CUDA tensors, v_part float32")
    if x.dim() != 2 or x.stride(1) != 1 or not v_part.is_contiguous():
        raise N.ValidationError("x must be 2-D with unit column stride; v_part contiguous")
    rs = tp_shard_rows(plan, tp_size)
    if v_part.numel() < plan.n_tokens * rs:
        raise N.ValidationError("v_part smaller than n_tokens x shard rows")
    s = current_stream_handle(x.device) if stream is None else stream
    N.check(N.lib().plora_bgmv_tp_shrink(plan.handle, layer, proj, tp_rank, tp_size, x.data_ptr(),
                                         x.stride(0), v_part.data_ptr(), s))
    return v_part


def bgmv_tp_expand(plan: BatchPlan, layer: int, proj: int, tp_rank: int, tp_size: int,
                   v_gathered: torch.Tensor, y_shard: torch.Tensor, scale: float = 1.0,
                   stream: int | None = None) -> torch.Tensor:
    """y_shard += scale · v · Bᵀ[:, cols of tp_rank]; v_gathered is [N, T, rs]."""
    if not (v_gathered.is_cuda and y_shard.is_cuda) or v_gathered.dtype != torch.float32:
        raise N.ValidationError("v_gathered and y_shard must be CUDA tensors, v float32")
    if not v_gathered.is_contiguous() or y_shard.dim() != 2 or y_shard.stride(1) != 1:
        raise N.ValidationError("v_gathered contiguous; y_shard 2-D with unit column stride")
    rs = tp_shard_rows(plan, tp_size)
    if v_gathered.numel() < tp_size * plan.n_tokens * rs:
        raise N.ValidationError("v_gathered smaller than tp_size x n_tokens x shard rows")
    s = current_stream_handle(y_shard.device) if stream is None else stream
    N.check(N.lib().plora_bgmv_tp_expand(plan.handle, layer, proj, tp_rank, tp_size,
                                         v_gathered.data_ptr(), y_shard.data_ptr(),
                                         y_shard.stride(0), C.c_float(scale), s))
    return y_shard


def bgmv_tp_shrink_push(plan: BatchPlan, layer: int, proj: int, tp_rank: int, tp_size: int,
                        x: torch.Tensor, peer_v_gathered: Sequence[int], peer_flags: Sequence[int],
                        stream: int | None = None) -> None:
    """The shrink with the all-gather fused in: this rank's v rows are stored
    straight into every rank's v_gathered (device pointers, peer memory over
    NVLink: peer_v_gathered[d] is rank d's [tp_size, T, rs] fp32 buffer), then
    slot tp_rank of every rank's flag array (peer_flags[d]: rank d's [tp_size]
    uint32 counters) is incremented by one."""
    if len(peer_v_gathered) != tp_size or len(peer_flags) != tp_size:
        raise N.ValidationError("one v_gathered buffer and one flag per TP rank")
    if not x.is_cuda or x.dim() != 2 or x.stride(1) != 1:
        raise N.ValidationError("x must be a 2-D CUDA tensor with unit column stride")
    vp = (C.c_void_p * tp_size)(*peer_v_gathered)
    fp = (C.c_void_p * tp_size)(*peer_flags)
    s = current_stream_handle(x.device) if stream is None else stream
    N.check(N.lib().plora_bgmv_tp_shrink_push(plan.handle, layer, proj, tp_rank, tp_size, x.data_ptr(),
                                              x.stride(0), vp, fp, s))


def bgmv_tp_expand_wait(plan: BatchPlan, layer: int, proj: int, tp_rank: int, tp_size: int,
                        v_gathered: torch.Tensor, flags: torch.Tensor, y_shard: torch.Tensor,
                        scale: float = 1.0, stream: int | None = None) -> torch.Tensor:
    """The expand of the fused path: waits (on the device) until every slot of
    ``flags`` (this rank's [tp_size] arrival counters) shows this call's
    shrink_push of that rank, consumes them, and y_shard += scale · v ·
    Bᵀ[:, cols of tp_rank]."""
    if not (v_gathered.is_cuda and y_shard.is_cuda and flags.is_cuda):
        raise N.ValidationError("v_gathered, flags and y_shard must be CUDA tensors")
    if flags.numel() < tp_size or flags.element_size() != 4:
        raise N.ValidationError("flags must hold tp_size 32-bit counters")
    if not v_gathered.is_contiguous() or y_shard.dim() != 2 or y_shard.stride(1) != 1:
        raise N.ValidationError("v_gathered contiguous; y_shard 2-D with unit column stride")
    rs = tp_shard_rows(plan, tp_size)
    if v_gathered.numel() < tp_size * plan.n_tokens * rs:
        raise N.ValidationError("v_gathered smaller than tp_size x n_tokens x shard rows")
    s = current_stream_handle(y_shard.device) if stream is None else stream
    N.check(N.lib().plora_bgmv_tp_expand_wait(plan.handle, layer, proj, tp_rank, tp_size,
                                              v_gathered.data_ptr(), flags.data_ptr(),
                                              y_shard.data_ptr(), y_shard.stride(0), C.c_float(scale), s))
    return y_shard


def _all_gather(out: torch.Tensor, inp: torch.Tensor, group) -> None:
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
    else:  # gloo: list form (same rank-major result)
        dist.all_gather(list(out.unbind(0)), inp, group=group)


class TensorParallelLoRA:
    """One TP rank's paged LoRA for a column-parallel projection.

    ``forward(layer, proj, x, y_shard)`` runs shrink -> all-gather -> expand
    on the current stream.  ``shrink`` / ``expand`` / ``all_gather`` default
    to the sm_100a kernels and torch.distributed; they are injectable so the
    orchestration (buffer shapes, gathered layout, rank bookkeeping) can be
    exercised on CPU ranks with gloo in tests.
    """

    def __init__(self, plan, tp_rank: int, tp_size: int, group=None,
                 shrink: Optional[Callable] = None, expand: Optional[Callable] = None,
                 all_gather: Optional[Callable] = None, shard_rows: Optional[int] = None,
                 n_tokens: Optional[int] = None, device=None, force_split: bool = False,
                 allgather: str = "nccl"):
        """force_split: run the shrink / expand halves even at tp_size 1
        (timing of the per-rank kernels; otherwise one rank uses the fused
        data-parallel op).  allgather: "nccl" (shrink, NCCL all-gather,
        expand) or "fused" (the shrink stores its rows straight into every
        rank's gathered buffer over NVLink peer memory — torch symmetric
        memory — and the expand waits on per-rank arrival flags; no
        collective call)."""
        if tp_size < 1 or not 0 <= tp_rank < tp_size:
            raise N.ValidationError("tp_rank must be in [0, tp_size)")
        if allgather not in ("nccl", "fused"):
            raise N.ValidationError("allgather must be 'nccl' or 'fused'")
        self.allgather = allgather
        self._calls = 0
        self._fcap = 0
        self.plan, self.tp_rank, self.tp_size, self.group = plan, tp_rank, tp_size, group
        self.force_split = force_split
        self._shrink = shrink or bgmv_tp_shrink
        self._expand = expand or bgmv_tp_expand
        self._gather = all_gather or (lambda out, inp: _all_gather(out, inp, group))
        # fixed sizes only when injected (emulated ranks); otherwise they follow
        # the plan, which BatchPlan.update may change between calls
        self._fixed_rs, self._fixed_t = shard_rows, n_tokens
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._buf = torch.empty(0, dtype=torch.float32, device=self.device)
        self._gbuf = torch.empty(0, dtype=torch.float32, device=self.device)
        self._views()

    def _views(self):
        """v_part [T, rs] and v_gathered [N, T, rs] as contiguous prefix views
        of the buffers, sized from the plan as it is now: the expand kernel
        reads rank block i at i·T·rs of the CURRENT plan, so the gathered
        layout must be rebuilt whenever T or rs changes."""
        rs = self._fixed_rs if self._fixed_rs is not None else tp_shard_rows(self.plan, self.tp_size)
        t = self._fixed_t if self._fixed_t is not None else self.plan.n_tokens
        need = max(t * rs, 1)
        if self._buf.numel() < need:
            self._buf = torch.empty(need, dtype=torch.float32, device=self.device)
            self._gbuf = torch.empty(self.tp_size * need, dtype=torch.float32, device=self.device)
        self.rs, self.n_tokens = rs, t
        self.v_gathered = self._gbuf[:self.tp_size * t * rs].view(self.tp_size, t, rs)
        # one rank: the shrink writes the "gathered" buffer directly (no copy)
        self.v_part = self.v_gathered[0] if self.tp_size == 1 else self._buf[:t * rs].view(t, rs)

    def _fused_buffers(self):
        """Two v_gathered buffers (call parity) and the [tp_size] arrival
        flags, addressable by every rank: local tensors for one rank, torch
        symmetric memory (peer pointers over NVLink) across ranks."""
        cap = max(self.n_tokens * self.rs, 1)
        if cap <= self._fcap:
            return
        n = self.tp_size
        if n == 1:
            self._fv = torch.zeros(2 * cap, dtype=torch.float32, device=self.device)
            self._ff = torch.zeros(n, dtype=torch.int32, device=self.device)
            self._peer_v, self._peer_f = [self._fv.data_ptr()], [self._ff.data_ptr()]
        else:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm
            self._fv = symm.empty(2 * n * cap, dtype=torch.float32, device=self.device)
            self._ff = symm.empty(n, dtype=torch.int32, device=self.device)
            self._ff.zero_()
            group = self.group if self.group is not None else dist.group.WORLD
            hv, hf = symm.rendezvous(self._fv, group), symm.rendezvous(self._ff, group)
            self._peer_v, self._peer_f = list(hv.buffer_ptrs), list(hf.buffer_ptrs)
            torch.cuda.synchronize(self.device)
            dist.barrier(group=group)  # every rank's flags are zero before any push
        self._fcap = cap

    def _forward_fused(self, layer, proj, x, y_shard, scale):
        self._views()
        self._fused_buffers()
        n, t, rs, cap = self.tp_size, self.n_tokens, self.rs, self._fcap
        par = self._calls & 1
        off = par * n * cap * 4  # bytes: this call's buffer in every rank's pair
        bgmv_tp_shrink_push(self.plan, layer, proj, self.tp_rank, n, x,
                            [p + off for p in self._peer_v], self._peer_f)
        vg = self._fv[par * n * cap: par * n * cap + n * t * rs].view(n, t, rs)
        bgmv_tp_expand_wait(self.plan, layer, proj, self.tp_rank, n, vg, self._ff, y_shard, scale)
        self._calls += 1
        return y_shard

    def forward(self, layer: int, proj: int, x: torch.Tensor, y_shard: torch.Tensor,
                scale: float = 1.0) -> torch.Tensor:
        if self.allgather == "fused" and (self.tp_size > 1 or self.force_split):
            return self._forward_fused(layer, proj, x, y_shard, scale)
        if self.tp_size == 1 and self._shrink is bgmv_tp_shrink and not self.force_split:
            # one rank holds every row and column: no collective, so the fused
            # data-parallel op applies the whole LoRA in one launch
            from .lora import bgmv
            return bgmv(self.plan, layer, proj, x, y_shard, scale)
        self._views()
        self._shrink(self.plan, layer, proj, self.tp_rank, self.tp_size, x, self.v_part)
        if self.tp_size > 1:
            self._gather(self.v_gathered, self.v_part)
        return self._expand(self.plan, layer, proj, self.tp_rank, self.tp_size, self.v_gathered,
                            y_shard, scale)

    __call__ = forward
