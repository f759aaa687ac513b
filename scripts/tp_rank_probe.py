"""Diagnostics: one rank's TP halves at TP = 8 (cfg5 shapes, q projection)
for an ncu capture: rank 0's shrink and expand, v_gathered from every rank's
shrink filled once beforehand."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan  # noqa: E402
from paper_2512_20210_b200.tp import bgmv_tp_expand, bgmv_tp_shrink, tp_shard_rows  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = synth.cfg5(n_layers=2)
pool = synth.build_pool(cfg)
store = AdapterStore(pool, cfg.shape, cfg.n_adapters)
for a, r in enumerate(cfg.ranks):
    store.register(a, r)
    store.write_pages(a, synth.adapter_image(cfg.shape, r, a, device="cuda").view(torch.uint8))
    store.publish(a)
ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
plan = BatchPlan(store, ta)
T = len(ta)
x = torch.randn(T, 8192, device="cuda").to(torch.bfloat16)
y = torch.randn(T, 8192 // N, device="cuda").to(torch.bfloat16)
rs = tp_shard_rows(plan, N)
vg = torch.stack([bgmv_tp_shrink(plan, 1, 0, i, N, x, torch.zeros(T, rs, device="cuda")) for i in range(N)]).contiguous()
vp = torch.zeros(T, rs, device="cuda")
for _ in range(5):
    bgmv_tp_shrink(plan, 1, 0, 0, N, x, vp)
    bgmv_tp_expand(plan, 1, 0, 0, N, vg, y, 0.5)
torch.cuda.synchronize()
print("ok")
