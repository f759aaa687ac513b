"""Seeded synthetic inputs for BASELINE.json's configs.

  x, y0 ~ N(0, 1); A ~ N(0, 1/d_in); B ~ N(0, 1/r); cast to the store dtype.
  Seeds: data 1234, token->adapter assignment 5678, pool churn 20240611.
  Page tables come from a churn prologue (allocate all adapters in key order,
  free the even keys, re-allocate them) so tables are scattered and
  non-contiguous, as in SURVEY Appendix A.

Shared by tests/, bench.py and oracle/make_golden.py so every consumer sees
identical bytes.  Generation happens with torch generators on the requested
device; CPU generation is the reference for golden fixtures.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .lora import ModelShape
from .memory import AllocStatus, PagePool

SEED_DATA = 1234
SEED_ASSIGN = 5678
SEED_CHURN = 20240611


@dataclass
class DecodeConfig:
    """One BASELINE config's per-call shape."""
    name: str
    shape: ModelShape
    ranks: list[int]           # rank of adapter key k
    tokens_per_adapter: int
    page_bytes: int
    pool_factor: float = 2.0   # arena = factor × catalog bytes

    @property
    def n_adapters(self) -> int:
        return len(self.ranks)

    @property
    def n_tokens(self) -> int:
        return self.n_adapters * self.tokens_per_adapter


def cfg1(dtype=torch.bfloat16, n_layers: int = 32) -> DecodeConfig:
    """CPU-oracle config: 16 adapters (even -> r8, odd -> r16), 64 decode tokens,
    2 KiB pages (BASELINE.json configs[0])."""
    shape = ModelShape(n_layers, (4096, 4096), (4096, 4096), dtype)
    return DecodeConfig("cfg1", shape, [8 if a % 2 == 0 else 16 for a in range(16)], 4, 2048)


def cfg2(dtype=torch.bfloat16, n_layers: int = 32, page_bytes: int = 2048) -> DecodeConfig:
    """Decode BGMV: 256 tokens over 128 adapters, r = [8,16,32,64][a % 4]
    (BASELINE.json configs[1])."""
    shape = ModelShape(n_layers, (4096, 4096), (4096, 4096), dtype)
    return DecodeConfig("cfg2", shape, [(8, 16, 32, 64)[a % 4] for a in range(128)], 2,
                        page_bytes)


def cfg3(dtype=torch.bfloat16, n_layers: int = 32, page_bytes: int = 2048,
         n_segments: int = 32, seg_tokens: int = 512) -> DecodeConfig:
    """Prefill SGMV: 32 segments × 512 tokens, r = [16,64,128][s % 3]
    (BASELINE.json configs[2]); adapter s serves segment s."""
    shape = ModelShape(n_layers, (4096, 4096), (4096, 4096), dtype)
    return DecodeConfig("cfg3", shape, [(16, 64, 128)[s % 3] for s in range(n_segments)],
                        seg_tokens, page_bytes)


def cfg5(dtype=torch.bfloat16, n_layers: int = 80, page_bytes: int = 2048,
         n_adapters: int = 128) -> DecodeConfig:
    """Tensor-parallel decode at Llama-2-70B q/v shapes (q 8192 -> 8192, v
    8192 -> 1024 GQA): 256 tokens over 128 adapters, r = [8,16,64][a % 3]
    (BASELINE.json configs[4])."""
    return DecodeConfig("cfg5", ModelShape.llama70b_qv(dtype),
                        [(8, 16, 64)[a % 3] for a in range(n_adapters)], 2, page_bytes)


def segment_assignment(n_segments: int, seg_tokens: int):
    """Prefill batch: segment s = tokens [s·L, (s+1)·L) of adapter s (contiguous runs)."""
    return np.repeat(np.arange(n_segments, dtype=np.int32), seg_tokens)


def token_assignment(n_adapters: int, tokens_per_adapter: int, seed: int = SEED_ASSIGN):
    """Each adapter gets tokens_per_adapter tokens, in shuffled order."""
    ta = np.repeat(np.arange(n_adapters, dtype=np.int32), tokens_per_adapter)
    rng = np.random.default_rng(seed)
    rng.shuffle(ta)
    return ta


def build_pool(cfg: DecodeConfig) -> PagePool:
    """Churn prologue: allocate all, free even keys, re-allocate them."""
    sizes = [cfg.shape.adapter_bytes(r) for r in cfg.ranks]
    total_pages = int(sum(-(-s // cfg.page_bytes) for s in sizes) * cfg.pool_factor)
    pool = PagePool(cfg.page_bytes, total_pages)
    for a, s in enumerate(sizes):
        assert pool.alloc(a, s) == AllocStatus.ok
    for a in range(0, cfg.n_adapters, 2):
        pool.free(a)
    for a in range(0, cfg.n_adapters, 2):
        assert pool.alloc(a, sizes[a]) == AllocStatus.ok
    return pool


def adapter_image(shape: ModelShape, rank: int, key: int, seed: int = SEED_DATA,
                  device: str | torch.device = "cpu") -> torch.Tensor:
    """Logical bytes of adapter `key` (layout of ModelShape): returns a flat
    tensor of shape.dtype on `device`."""
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1_000_003 + key)
    n = shape.adapter_bytes(rank) // shape.esize
    flat = torch.randn(n, generator=g, device=device, dtype=torch.float32)
    off = 0
    for _ in range(shape.n_layers):
        for p in range(shape.n_proj):
            na, nb = rank * shape.d_in[p], rank * shape.d_out[p]
            flat[off:off + na] *= 1.0 / np.sqrt(shape.d_in[p])
            flat[off + na:off + na + nb] *= 1.0 / np.sqrt(rank)
            off += na + nb
    return flat.to(shape.dtype)


def activations(n_tokens: int, d: int, dtype, which: str, seed: int = SEED_DATA,
                device: str | torch.device = "cpu", salt: int = 0) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed + {"x": 1, "y": 2}[which] * 7919 + salt * 104729)
    return torch.randn(n_tokens, d, generator=g, device=device, dtype=torch.float32).to(dtype)
