"""Diagnostics: plora_sgmv time at cfg3 shapes (32 runs x 512 tokens,
Llama-7B q) as a function of a uniform adapter rank — separates the x / y
streams (rank independent) from the weight gathers (proportional to rank)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, sgmv  # noqa: E402

for r in (16, 64, 128):
    cfg = synth.DecodeConfig("sweep", synth.cfg3().shape.__class__(2, (4096, 4096), (4096, 4096)),
                             [r] * 32, 512, 2048)
    pool = synth.build_pool(cfg)
    store = AdapterStore(pool, cfg.shape, 32)
    for a in range(32):
        store.register(a, r)
        store.write_pages(a, synth.adapter_image(cfg.shape, r, a, device="cuda").view(torch.uint8))
        store.publish(a)
    ta = synth.segment_assignment(32, 512)
    plan = BatchPlan(store, ta)
    x = torch.randn(len(ta), 4096, device="cuda").to(torch.bfloat16)
    y = torch.randn(len(ta), 4096, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        sgmv(plan, 1, 0, x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        sgmv(plan, 1, 0, x, y)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 100
    print(f"rank {r}: {us:.1f} us per call ({(3 * 16384 * 4096 * 2 + 32 * r * 8192 * 2) / us / 1e3:.0f} GB/s)")
    del plan, store, pool
