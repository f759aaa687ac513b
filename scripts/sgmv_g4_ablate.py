"""Diagnostics: the SGMV shrink's A-row gathers split between TMA gather4
(TMA unit) and 16-byte cp.async (LSU): flags 16384 all gather4, 4096 one
group of four in four by cp.async, 0 (default) every other group, 8192 three
in four, 2048 all cp.async; timed for the layer call
(plora_sgmv_layer) and its shrink alone (flag 8: no expand), at cfg3."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, sgmv_layer  # noqa: E402

cfg = synth.cfg3(n_layers=2)
pool = synth.build_pool(cfg)
store = AdapterStore(pool, cfg.shape, 32)
for a, ra in enumerate(cfg.ranks):
    store.register(a, ra)
    store.write_pages(a, synth.adapter_image(cfg.shape, ra, a, device="cuda").view(torch.uint8))
    store.publish(a)
plan = BatchPlan(store, synth.segment_assignment(32, 512))
x = torch.randn(32 * 512, 4096, device="cuda").to(torch.bfloat16)
ys = [torch.randn(32 * 512, 4096, device="cuda").to(torch.bfloat16) for _ in range(2)]
for g4 in (16384, 4096, 0, 8192, 2048):  # 0 = the default (half by cp.async)
    for name, extra in (("layer call", 0), ("shrink only", 40), ("expand no y", 64), ("expand no B", 128)):
        N.check(N.lib().plora_debug_set_sgmv_flags(g4 | extra))
        for _ in range(3):
            sgmv_layer(plan, 1, x, ys)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            sgmv_layer(plan, 1, x, ys)
        e1.record()
        torch.cuda.synchronize()
        print(f"g4 flags {g4:5d} {name:14s} {e0.elapsed_time(e1) * 50:.1f} us")
N.check(N.lib().plora_debug_set_sgmv_flags(0))
