"""A/B of the tiled SGMV expand's y epilogue at cfg3 (layer call): coalesced
read-modify-write (default) vs TMA reduce-add (flag 1 << 21).  Compares y
and times the layer call."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, sgmv_layer  # noqa: E402

RADD = 1 << 21
cfg = synth.cfg3(n_layers=2)
pool = synth.build_pool(cfg)
store = AdapterStore(pool, cfg.shape, 32)
for a, ra in enumerate(cfg.ranks):
    store.register(a, ra)
    store.write_pages(a, synth.adapter_image(cfg.shape, ra, a, device="cuda").view(torch.uint8))
    store.publish(a)
plan = BatchPlan(store, synth.segment_assignment(32, 512))
x = torch.randn(32 * 512, 4096, device="cuda").to(torch.bfloat16)
y0 = torch.randn(32 * 512, 4096, device="cuda").to(torch.bfloat16)
z0 = torch.randn(32 * 512, 4096, device="cuda").to(torch.bfloat16)
outs = {}
for name, flags in (("reduce-add", RADD), ("coalesced", 0)):
    N.check(N.lib().plora_debug_set_sgmv_flags(flags))
    y, z = y0.clone(), z0.clone()
    sgmv_layer(plan, 1, x, [y, z])
    torch.cuda.synchronize()
    outs[name] = (y, z)
for p in range(2):
    a, b = outs["reduce-add"][p].float(), outs["coalesced"][p].float()
    print(f"proj {p}: differing elements {(a != b).float().mean().item():.2e}, max |diff| {(a - b).abs().max().item():.3e}")
y, z = y0.clone(), z0.clone()
for rep in range(2):
    for name, flags in (("reduce-add", RADD), ("coalesced", 0)):
        N.check(N.lib().plora_debug_set_sgmv_flags(flags))
        for _ in range(3):
            sgmv_layer(plan, 1, x, [y, z])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            sgmv_layer(plan, 1, x, [y, z])
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:12s} layer call {e0.elapsed_time(e1) * 50:.1f} us")
N.check(N.lib().plora_debug_set_sgmv_flags(0))
