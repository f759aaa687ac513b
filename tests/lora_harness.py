"""Shared harness for the paged-LoRA parity tests: builds a store from a
synth config and computes the CPU oracle on identical inputs and tables."""
from __future__ import annotations

import numpy as np
import torch

from oracle import lora as OL
from paper_2512_20210_b200 import synth
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, ModelShape

# Tolerances (BASELINE.json north_star): normwise max|y_gpu - y_oracle| / max|y_oracle|
TOL_BF16 = 1e-2
# the default bf16 decode op (bgmv_warp.cu) is two launches per call: shrink, expand
BGMV_BF16_LAUNCHES = 2
TOL_F32 = 1e-5


def to_np_bits(t: torch.Tensor) -> np.ndarray:
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16).copy()
    return t.numpy().astype(np.float32).copy()


def to_f32(a: np.ndarray) -> np.ndarray:
    return OL.bf16_bits_to_f32(a) if a.dtype == np.uint16 else a.astype(np.float32)


def delta_rel_err(y_gpu: torch.Tensor, y_ref: np.ndarray, y0: torch.Tensor) -> float:
    """Normwise error of the LoRA delta alone: max|Δy_gpu - Δy_ref| / max|Δy_ref|
    (y0 subtracted in fp64), so a systematic error in the delta cannot hide
    under |y0|."""
    g = to_f32(to_np_bits(y_gpu)).astype(np.float64)
    r = to_f32(y_ref).astype(np.float64)
    b = to_f32(to_np_bits(y0)).astype(np.float64)
    return float(np.abs((g - b) - (r - b)).max() / max(np.abs(r - b).max(), 1e-30))


def rel_err(y_gpu: torch.Tensor, y_ref: np.ndarray) -> float:
    g = to_f32(to_np_bits(y_gpu)).astype(np.float64)
    r = to_f32(y_ref).astype(np.float64)
    return float(np.abs(g - r).max() / max(np.abs(r).max(), 1e-30))


class Setup:
    """Store + host arena image for one synth config."""

    def __init__(self, cfg: synth.DecodeConfig, device: int = 0, copy_mode: int = 0,
                 pool=None):
        self.cfg = cfg
        self.shape = cfg.shape
        self.pool = pool if pool is not None else synth.build_pool(cfg)
        self.store = AdapterStore(self.pool, cfg.shape, max_adapters=cfg.n_adapters,
                                  device=device)
        P = cfg.page_bytes
        self.arena = np.zeros(self.pool.total_pages() * P, np.uint8)
        self.images = {}
        for a, r in enumerate(cfg.ranks):
            img = synth.adapter_image(cfg.shape, r, a)
            self.images[a] = img
            self.store.register(a, r)
            host = img.view(torch.uint8)
            if copy_mode == 1:
                host = host.pin_memory()
            self.store.write_pages(a, host, mode=copy_mode)
            self.store.publish(a)
            OL.scatter_pages(self.arena, P, self.pool.table(a), to_np_bits(img))
        torch.cuda.synchronize()
        self.m = OL.model(cfg.shape.n_layers, cfg.shape.d_in, cfg.shape.d_out, cfg.shape.esize)

    @classmethod
    def on_device(cls, cfg: synth.DecodeConfig, device: int = 0, pool=None):
        """Full-size configs: images generated on the GPU (torch CUDA
        generator), scattered device-to-device, and copied once to the host
        arena the oracle reads — no host copy of the images is kept."""
        self = cls.__new__(cls)
        self.cfg, self.shape = cfg, cfg.shape
        self.pool = pool if pool is not None else synth.build_pool(cfg)
        self.store = AdapterStore(self.pool, cfg.shape, max_adapters=cfg.n_adapters,
                                  device=device)
        P = cfg.page_bytes
        self.arena = np.zeros(self.pool.total_pages() * P, np.uint8)
        self.images = {}
        for a, r in enumerate(cfg.ranks):
            img = synth.adapter_image(cfg.shape, r, a, device=f"cuda:{device}")
            self.store.register(a, r)
            self.store.write_pages(a, img.view(torch.uint8))
            self.store.publish(a)
            OL.scatter_pages(self.arena, P, self.pool.table(a), to_np_bits(img))
            del img
        torch.cuda.synchronize()
        self.m = OL.model(cfg.shape.n_layers, cfg.shape.d_in, cfg.shape.d_out, cfg.shape.esize)
        return self

    def tables(self):
        return {a: self.pool.table(a) for a in range(self.cfg.n_adapters)}

    def oracle(self, layer, proj, x: torch.Tensor, y0: torch.Tensor, token_adapter,
               scale=1.0, v_bf16=False, nthreads=8) -> np.ndarray:
        xb, yb = to_np_bits(x), to_np_bits(y0)
        OL.paged_lora_apply(self.m, self.arena, self.cfg.page_bytes, self.tables(),
                            dict(enumerate(self.cfg.ranks)), layer, proj, xb, yb,
                            token_adapter, scale=scale, v_bf16=v_bf16, nthreads=nthreads)
        return yb
