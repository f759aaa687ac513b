"""ORACLE ONLY — the CPU arm of bench.py (`--impl reference` and the
`cpu_baseline` leg): the paged LoRA decode step of BASELINE configs[1] run on
the host cores by the C restatement (oracle/lora_oracle.c), with every page
table produced by the reference's own lorasim::PagePool (oracle/_ref/libref.so,
src/memory.cpp:18-38) and adapter sizes from the reference's own LoraDims
(src/adapter.cpp:12-26).

Nothing here imports or loads the product package (paper_2512_20210_b200 /
libplora.so): the arm measures the reference-side CPU path only.

Workload (identical to bench.py's GPU arm): Llama-7B q/v (d = k = 4096,
32 layers x 2 projections = 64 (layer, proj) calls per decode step), 128
adapters with r = [8,16,32,64][a % 4], 256 tokens (2 per adapter, shuffled),
2 KiB pages, tables scattered by the churn prologue (allocate all, free the
even keys, re-allocate them).  x, y ~ N(0,1); A ~ N(0, 1/d_in);
B ~ N(0, 1/r); bf16.
"""
from __future__ import annotations

import os
import platform
import time

import numpy as np

from . import lora as OL
from . import ref as R

D = 4096
RANKS_CFG2 = [(8, 16, 32, 64)[a % 4] for a in range(128)]
SEED_DATA, SEED_ASSIGN = 1234, 5678


def cpu_model_name() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def adapter_bytes(rank: int, n_layers: int) -> int:
    """The reference's LoraDims::param_count (d = k = 4096, 2 adapted
    matrices per layer) x 2 bytes per bf16 parameter (adapter.cpp:52-59)."""
    return R.param_count(D, D, rank, 2 * n_layers, 2) * 2


def token_assignment(n_adapters: int, per: int, seed: int = SEED_ASSIGN) -> np.ndarray:
    ta = np.repeat(np.arange(n_adapters, dtype=np.int32), per)
    np.random.default_rng(seed).shuffle(ta)
    return ta


def _bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16 bits (finite inputs: 32-bit arithmetic)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32)
    return ((u + (0x7FFF + ((u >> 16) & 1))) >> 16).astype(np.uint16)


class CpuDecodeStep:
    """The cfg2 catalog in a host arena laid out by the reference PagePool."""

    def __init__(self, n_layers: int = 32, ranks=RANKS_CFG2, page_bytes: int = 2048,
                 pool_factor: float = 1.25, nthreads: int | None = None, seed: int = SEED_DATA):
        self.L, self.ranks, self.P = n_layers, list(ranks), page_bytes
        self.nthreads = nthreads or os.cpu_count() or 1
        sizes = [adapter_bytes(r, n_layers) for r in self.ranks]
        total = int(sum(-(-s // page_bytes) for s in sizes) * pool_factor)
        pool = R.RefPagePool(page_bytes, total)
        for a, s in enumerate(sizes):  # churn prologue -> scattered tables
            assert pool.alloc(a, s) == 0
        for a in range(0, len(sizes), 2):
            pool.free(a)
        for a in range(0, len(sizes), 2):
            assert pool.alloc(a, sizes[a]) == 0
        pool.check_invariants()
        self.tables = {a: pool.table(a) for a in range(len(sizes))}
        self.arena = np.zeros(total * page_bytes, np.uint8)
        rng = np.random.default_rng(seed)
        for a, r in enumerate(self.ranks):
            # per (layer, proj) block: A (r x 4096) ~ N(0, 1/4096), Bt (r x 4096) ~ N(0, 1/r)
            blk = rng.standard_normal((n_layers * 2, 2, r * D), dtype=np.float32)
            blk[:, 0] *= 1.0 / np.sqrt(D)
            blk[:, 1] *= 1.0 / np.sqrt(r)
            OL.scatter_pages(self.arena, page_bytes, self.tables[a], _bf16_bits(blk.reshape(-1)))
        self.m = OL.model(n_layers, (D, D), (D, D), 2)
        self.ta = token_assignment(len(self.ranks), 2)
        T = len(self.ta)
        self.x = _bf16_bits(rng.standard_normal((n_layers, T, D), dtype=np.float32))
        self.y = _bf16_bits(rng.standard_normal((n_layers * 2, T, D), dtype=np.float32))
        self.rank_of = dict(enumerate(self.ranks))
        self.prepared = OL.PreparedTables(self.tables, self.rank_of)

    @property
    def n_tokens(self) -> int:
        return len(self.ta)

    def call(self, layer: int, proj: int) -> None:
        OL.paged_lora_apply(self.m, self.arena, self.P, self.prepared, None, layer, proj,
                            self.x[layer], self.y[layer * 2 + proj], self.ta,
                            nthreads=self.nthreads)

    def step(self) -> None:
        """One decode step: all 64 (layer, proj) calls."""
        for layer in range(self.L):
            for proj in range(2):
                self.call(layer, proj)

    def sample_calls(self, target_s: float, max_calls: int = 64):
        """Seconds per call over a bounded sample of calls (layer, proj cycled)."""
        n, t0 = 0, time.perf_counter()
        while n < max_calls:
            self.call((n // 2) % self.L, n % 2)
            n += 1
            if time.perf_counter() - t0 >= target_s:
                break
        return (time.perf_counter() - t0) / n, n
