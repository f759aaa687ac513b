"""Device-side paged multi-LoRA: the HBM adapter store and the paged LoRA
forward op (BGMV decode / SGMV prefill), over the C ABI in include/plora.h.

PyTorch is used for device memory and streams only; every kernel lives in
libplora.so.  There is no CPU or torch fallback: without the library (or a
GPU) these calls raise.

Reference anchors: the paged LoRA forward op is what the reference bills as
``cost_model.prefill_ms`` / ``step_ms`` (include/lorasim/cost_model.hpp:32-40,
src/engine.cpp:355,510); math PAPER.md:64-69; pages and tables
src/memory.cpp:7-89.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from .memory import PagePool, Relocation

_DTYPES = {torch.bfloat16: N.PLORA_BF16, torch.float32: N.PLORA_F32}


@dataclass(frozen=True)
class ModelShape:
    """Adapted matrices of the base model: n_layers × len(d_in) projections.

    In-adapter layout: for layer l, projection p (in order) one block
    [A (r × d_in[p]) | Bᵀ (r × d_out[p])], row-major.  The adapter's size is
    exactly param_count · bytes_per_param (src/adapter.cpp:22-26,52-59).
    """
    n_layers: int
    d_in: tuple[int, ...]
    d_out: tuple[int, ...]
    dtype: torch.dtype = torch.bfloat16

    @staticmethod
    def llama7b_qv(dtype: torch.dtype = torch.bfloat16) -> "ModelShape":
        """Llama-2-7B q/v: 32 layers × {q, v}, 4096 → 4096 (adapter.hpp:15-23)."""
        return ModelShape(32, (4096, 4096), (4096, 4096), dtype)

    @staticmethod
    def llama70b_qv(dtype: torch.dtype = torch.bfloat16) -> "ModelShape":
        """Llama-2-70B q/v: 80 layers; q 8192 → 8192, v 8192 → 1024 (GQA)."""
        return ModelShape(80, (8192, 8192), (8192, 1024), dtype)

    @property
    def n_proj(self) -> int:
        return len(self.d_in)

    @property
    def esize(self) -> int:
        return 2 if self.dtype == torch.bfloat16 else 4

    def to_c(self) -> N.plora_model:
        if self.dtype not in _DTYPES:
            raise N.ValidationError(f"unsupported dtype {self.dtype}")
        m = N.plora_model()
        m.n_layers = self.n_layers
        m.n_proj = self.n_proj
        for i, (a, b) in enumerate(zip(self.d_in, self.d_out)):
            m.d_in[i] = a
            m.d_out[i] = b
        m.dtype = _DTYPES[self.dtype]
        return m

    def adapter_bytes(self, rank: int) -> int:
        m = self.to_c()
        return N.lib().plora_model_adapter_bytes(C.byref(m), rank)

    def block_offset(self, rank: int, layer: int, proj: int) -> int:
        m = self.to_c()
        return N.lib().plora_model_block_offset(C.byref(m), rank, layer, proj)


def pack_adapter(shape: ModelShape, A: Sequence[Sequence[torch.Tensor]],
                 B: Sequence[Sequence[torch.Tensor]]) -> torch.Tensor:
    """Logical byte image of one adapter from A[l][p] (r × d_in) and
    B[l][p] (d_out × r), laid out as the kernels read it.  Returns uint8 (CPU)."""
    parts = []
    for l in range(shape.n_layers):
        for p in range(shape.n_proj):
            a = A[l][p].to(shape.dtype).contiguous()
            bt = B[l][p].to(shape.dtype).t().contiguous()
            parts.append(a.reshape(-1))
            parts.append(bt.reshape(-1))
    flat = torch.cat(parts).cpu()
    return flat.view(torch.uint8)


def current_stream_handle(device: int | torch.device | None = None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class AdapterStore:
    """The page pool's physical pages backed by one HBM arena, with a device
    page table and adapter directory (include/plora.h, device store)."""

    def __init__(self, pool: PagePool, shape: ModelShape, max_adapters: int, device: int = 0):
        self.pool = pool  # keep the pool alive for the store's lifetime
        self.shape = shape
        self.device = device
        m = shape.to_c()
        h = C.c_void_p()
        N.check(N.lib().plora_store_create(pool.handle, device, C.byref(m), max_adapters,
                                           C.byref(h)))
        self._h = h
        self._lib = N.lib()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.plora_store_destroy(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def arena_ptr(self) -> int:
        return self._lib.plora_store_arena(self._h) or 0

    def register(self, adapter: int, rank: int) -> None:
        N.check(self._lib.plora_store_register(self._h, adapter, rank))

    def rank(self, adapter: int) -> int:
        r = C.c_uint32()
        N.check(self._lib.plora_store_rank(self._h, adapter, C.byref(r)))
        return r.value

    def write_pages(self, adapter: int, host: torch.Tensor, mode: int = N.PLORA_COPY_CE,
                    stream: int | None = None) -> None:
        """Page-scatter the adapter's logical bytes into its pages.  `host` is a
        contiguous CPU tensor (pinned for async copies; required for
        PLORA_COPY_SM) or, with PLORA_COPY_CE, a CUDA tensor on the store's
        device (D2D scatter)."""
        if not host.is_contiguous():
            raise N.ValidationError("write_pages needs a contiguous tensor")
        if host.device.type != "cpu" and (mode != N.PLORA_COPY_CE or
                                          host.device != torch.device("cuda", self.device)):
            raise N.ValidationError("device sources need PLORA_COPY_CE on the store's device")
        nbytes = host.numel() * host.element_size()
        s = current_stream_handle(self.device) if stream is None else stream
        N.check(self._lib.plora_store_write_pages(self._h, adapter, host.data_ptr(), nbytes,
                                                  mode, s))

    def read_pages(self, adapter: int, nbytes: int, stream: int | None = None) -> torch.Tensor:
        out = torch.empty(nbytes, dtype=torch.uint8)
        s = current_stream_handle(self.device) if stream is None else stream
        N.check(self._lib.plora_store_read_pages(self._h, adapter, out.data_ptr(), nbytes, s))
        return out

    def publish(self, adapter: int, stream: int | None = None) -> None:
        s = current_stream_handle(self.device) if stream is None else stream
        N.check(self._lib.plora_store_publish(self._h, adapter, s))

    def retire(self, adapter: int, stream: int | None = None) -> None:
        s = current_stream_handle(self.device) if stream is None else stream
        N.check(self._lib.plora_store_retire(self._h, adapter, s))

    def is_published(self, adapter: int) -> bool:
        return bool(self._lib.plora_store_is_published(self._h, adapter))

    def apply_relocations(self, relocs: Sequence[Relocation], stream: int | None = None) -> None:
        arr = (N.plora_reloc * max(len(relocs), 1))()
        for i, r in enumerate(relocs):
            arr[i] = N.plora_reloc(r.adapter, r.logical, r.src, r.dst)
        s = current_stream_handle(self.device) if stream is None else stream
        N.check(self._lib.plora_store_apply_relocations(self._h, arr, len(relocs), s))

    def load(self, adapter: int, rank: int, host: torch.Tensor, mode: int = N.PLORA_COPY_CE,
             weight_bytes: int | None = None) -> None:
        """register + PagePool.alloc + page scatter + publish (a demand load)."""
        from .memory import AllocStatus
        self.register(adapter, rank)
        nbytes = weight_bytes if weight_bytes is not None else self.shape.adapter_bytes(rank)
        st = self.pool.alloc(adapter, nbytes)
        if st != AllocStatus.ok:
            raise MemoryError(f"page pool out of memory loading adapter {adapter}")
        self.write_pages(adapter, host, mode)
        self.publish(adapter)


class BatchPlan:
    """Tokens grouped by adapter for one batch; reused by every (layer, proj)
    call of the step.  ``token_adapter`` is a host sequence (-1 = no LoRA)."""

    def __init__(self, store: AdapterStore, token_adapter, stream: int | None = None):
        self.store = store
        arr = self._as_i32(token_adapter)
        h = C.c_void_p()
        s = current_stream_handle(store.device) if stream is None else stream
        N.check(N.lib().plora_plan_create(store.handle, arr.ctypes.data_as(C.POINTER(C.c_int32)),
                                          len(arr), s, C.byref(h)))
        self._h = h
        self._lib = N.lib()
        self.n_tokens = len(arr)

    @staticmethod
    def _as_i32(token_adapter) -> np.ndarray:
        if isinstance(token_adapter, torch.Tensor):
            token_adapter = token_adapter.cpu().numpy()
        return np.ascontiguousarray(np.asarray(token_adapter, dtype=np.int32))

    def update(self, token_adapter, stream: int | None = None) -> None:
        arr = self._as_i32(token_adapter)
        s = current_stream_handle(self.store.device) if stream is None else stream
        N.check(self._lib.plora_plan_update(self._h, arr.ctypes.data_as(C.POINTER(C.c_int32)),
                                            len(arr), s))
        self.n_tokens = len(arr)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.plora_plan_destroy(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @property
    def num_segments(self) -> int:
        return self._lib.plora_plan_num_segments(self._h)


def _check_io(plan: BatchPlan, proj: int, x: torch.Tensor, y: torch.Tensor):
    shape = plan.store.shape
    for name, t in (("x", x), ("y", y)):
        if not t.is_cuda:
            raise N.ValidationError(f"{name} must be a CUDA tensor")
        if t.dtype != shape.dtype:
            raise N.ValidationError(f"{name} dtype {t.dtype} != store dtype {shape.dtype}")
        if t.dim() != 2 or t.stride(1) != 1:
            raise N.ValidationError(f"{name} must be 2-D with unit column stride")
    if x.shape[0] < plan.n_tokens or y.shape[0] < plan.n_tokens:
        raise N.ValidationError("x/y have fewer rows than the plan's tokens")
    if x.shape[1] != shape.d_in[proj] or y.shape[1] != shape.d_out[proj]:
        raise N.ValidationError("x/y widths do not match the projection")


def bgmv(plan: BatchPlan, layer: int, proj: int, x: torch.Tensor, y: torch.Tensor,
         scale: float = 1.0, stream: int | None = None) -> torch.Tensor:
    """y += scale · (x · Aᵀ) · Bᵀ per token (decode path; fp32 intermediate)."""
    _check_io(plan, proj, x, y)
    s = current_stream_handle(x.device) if stream is None else stream
    N.check(N.lib().plora_bgmv(plan.handle, layer, proj, x.data_ptr(), x.stride(0),
                               y.data_ptr(), y.stride(0), scale, s))
    return y


def bgmv_layer(plan: BatchPlan, layer: int, x: torch.Tensor, ys: Sequence[torch.Tensor],
               scale: float = 1.0, stream: int | None = None) -> Sequence[torch.Tensor]:
    """Every projection of `layer` at once: ys[p] += scale · (x · A_pᵀ) · B_pᵀ
    (the projections read the same x, e.g. q and v of an attention block)."""
    shape = plan.store.shape
    if len(ys) != shape.n_proj:
        raise N.ValidationError(f"bgmv_layer needs {shape.n_proj} outputs, got {len(ys)}")
    for p, y in enumerate(ys):
        _check_io(plan, p, x, y)
    ptrs = (C.c_void_p * shape.n_proj)(*[y.data_ptr() for y in ys])
    strides = (C.c_uint64 * shape.n_proj)(*[y.stride(0) for y in ys])
    s = current_stream_handle(x.device) if stream is None else stream
    N.check(N.lib().plora_bgmv_layer(plan.handle, layer, x.data_ptr(), x.stride(0), ptrs, strides,
                                     scale, s))
    return ys


def bgmv_layers(plan: BatchPlan, layer0: int, x: torch.Tensor, ys: Sequence[torch.Tensor],
                scale: float = 1.0, stream: int | None = None) -> Sequence[torch.Tensor]:
    """Layers [layer0, layer0 + n) of bgmv_layer in one launch, n = x.shape[0]:
    x is [n, T, d_in] (layer i's rows at x[i]), ys[p] is [n, T, d_out[p]].
    For inputs that are all ready at once; bit-identical to n bgmv_layer calls."""
    shape = plan.store.shape
    if len(ys) != shape.n_proj:
        raise N.ValidationError(f"bgmv_layers needs {shape.n_proj} outputs, got {len(ys)}")
    if x.dim() != 3 or any(y.dim() != 3 or y.shape[0] != x.shape[0] for y in ys):
        raise N.ValidationError("bgmv_layers: x and every y must be [n_layers, T, d]")
    for p, y in enumerate(ys):
        _check_io(plan, p, x[0], y[0])
    n = x.shape[0]
    ptrs = (C.c_void_p * shape.n_proj)(*[y.data_ptr() for y in ys])
    strides = (C.c_uint64 * shape.n_proj)(*[y.stride(1) for y in ys])
    lstrides = (C.c_uint64 * shape.n_proj)(*[y.stride(0) for y in ys])
    s = current_stream_handle(x.device) if stream is None else stream
    N.check(N.lib().plora_bgmv_layers(plan.handle, layer0, n, x.data_ptr(), x.stride(1),
                                      x.stride(0), ptrs, strides, lstrides, scale, s))
    return ys


def sgmv(plan: BatchPlan, layer: int, proj: int, x: torch.Tensor, y: torch.Tensor,
         scale: float = 1.0, stream: int | None = None) -> torch.Tensor:
    """y += scale · (x · Aᵀ) · Bᵀ per token (prefill path, tensor cores)."""
    _check_io(plan, proj, x, y)
    s = current_stream_handle(x.device) if stream is None else stream
    N.check(N.lib().plora_sgmv(plan.handle, layer, proj, x.data_ptr(), x.stride(0),
                               y.data_ptr(), y.stride(0), scale, s))
    return y


def sgmv_layer(plan: BatchPlan, layer: int, x: torch.Tensor, ys: Sequence[torch.Tensor],
               scale: float = 1.0, stream: int | None = None) -> Sequence[torch.Tensor]:
    """Prefill path for every projection of `layer`: ys[p] += scale · (x · A_pᵀ) · B_pᵀ;
    two projections of equal shape share each x chunk of the shrink and one
    expand launch."""
    shape = plan.store.shape
    if len(ys) != shape.n_proj:
        raise N.ValidationError(f"sgmv_layer needs {shape.n_proj} outputs, got {len(ys)}")
    for p, y in enumerate(ys):
        _check_io(plan, p, x, y)
    ptrs = (C.c_void_p * shape.n_proj)(*[y.data_ptr() for y in ys])
    strides = (C.c_uint64 * shape.n_proj)(*[y.stride(0) for y in ys])
    s = current_stream_handle(x.device) if stream is None else stream
    N.check(N.lib().plora_sgmv_layer(plan.handle, layer, x.data_ptr(), x.stride(0), ptrs, strides,
                                     scale, s))
    return ys


def sgmv_fused(plan: BatchPlan, layer: int, proj: int, x: torch.Tensor, w0: torch.Tensor,
               y: torch.Tensor, scale: float = 1.0, stream: int | None = None) -> torch.Tensor:
    """y = x · W0ᵀ + scale · (x · Aᵀ) · Bᵀ per token: the base projection with the
    paged LoRA fused in (prefill, tensor cores); w0 is the base weight
    [d_out, d_in], y is overwritten."""
    _check_io(plan, proj, x, y)
    if not w0.is_cuda or w0.dtype != torch.bfloat16 or w0.dim() != 2 or w0.stride(1) != 1:
        raise N.ValidationError("w0 must be a 2-D bf16 CUDA tensor with unit column stride")
    if w0.shape[0] != y.shape[1] or w0.shape[1] != x.shape[1]:
        raise N.ValidationError("w0 must be [d_out, d_in]")
    s = current_stream_handle(x.device) if stream is None else stream
    N.check(N.lib().plora_sgmv_fused(plan.handle, layer, proj, x.data_ptr(), x.stride(0),
                                     w0.data_ptr(), w0.stride(0), y.data_ptr(), y.stride(0),
                                     scale, s))
    return y


def sgmv_fused_layer(plan: BatchPlan, layer: int, x: torch.Tensor, w0s: Sequence[torch.Tensor],
                     ys: Sequence[torch.Tensor], scale: float = 1.0,
                     stream: int | None = None) -> Sequence[torch.Tensor]:
    """ys[p] = x · W0_pᵀ + scale · (x · A_pᵀ) · B_pᵀ for every projection of
    `layer`: one shrink for all (x read once), then one fused GEMM each."""
    shape = plan.store.shape
    if len(ys) != shape.n_proj or len(w0s) != shape.n_proj:
        raise N.ValidationError(f"sgmv_fused_layer needs {shape.n_proj} weights and outputs")
    for p, (w0, y) in enumerate(zip(w0s, ys)):
        _check_io(plan, p, x, y)
        if not w0.is_cuda or w0.dtype != torch.bfloat16 or w0.dim() != 2 or w0.stride(1) != 1:
            raise N.ValidationError("w0 must be a 2-D bf16 CUDA tensor with unit column stride")
        if w0.shape[0] != y.shape[1] or w0.shape[1] != x.shape[1]:
            raise N.ValidationError("w0 must be [d_out, d_in]")
    n = shape.n_proj
    wp = (C.c_void_p * n)(*[w.data_ptr() for w in w0s])
    ws = (C.c_uint64 * n)(*[w.stride(0) for w in w0s])
    yp = (C.c_void_p * n)(*[y.data_ptr() for y in ys])
    yst = (C.c_uint64 * n)(*[y.stride(0) for y in ys])
    s = current_stream_handle(x.device) if stream is None else stream
    N.check(N.lib().plora_sgmv_fused_layer(plan.handle, layer, x.data_ptr(), x.stride(0), wp, ws, yp,
                                           yst, scale, s))
    return ys


def kernel_launch_count() -> int:
    return N.lib().plora_kernel_launch_count()
