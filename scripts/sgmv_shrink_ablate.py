"""Diagnostics: SGMV layer call (plora_sgmv_layer, cfg3) and its shrink under
ablation flags (plora_debug_set_sgmv_flags): 8 no expand, 32 no reduction,
1 no A gather, 2 no MMA, 4 no x load, 16 no epilogue."""
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
tag = os.environ.get("PLORA_LIB", "default").split("/")[-1]
for name, fl in (("layer call", 0), ("shrink+reduce", 8), ("shrink only", 40), ("shrink no A", 41),
                 ("shrink no x", 44), ("shrink no MMA", 42), ("shrink nothing", 40 | 1 | 2 | 4 | 16)):
    N.check(N.lib().plora_debug_set_sgmv_flags(fl))
    for _ in range(3):
        sgmv_layer(plan, 1, x, ys)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        sgmv_layer(plan, 1, x, ys)
    e1.record()
    torch.cuda.synchronize()
    print(f"{tag:24s} {name:16s} {e0.elapsed_time(e1) * 50:.1f} us")
N.check(N.lib().plora_debug_set_sgmv_flags(0))
