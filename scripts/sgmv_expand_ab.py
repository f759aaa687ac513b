"""A/B of the SGMV expand kernels at cfg3 (layer call, both projections):
the tiled expand (default) vs the persistent expand (debug flag 1 << 20).  Checks the two give bit-identical y, then times the layer call and
the expand parts with shrink-side diagnostics flags (results wrong meanwhile)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, sgmv_layer  # noqa: E402

PERS = 1 << 20
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
for name, flags in (("tiled", 0), ("persistent", PERS)):
    N.check(N.lib().plora_debug_set_sgmv_flags(flags))
    y, z = y0.clone(), z0.clone()
    sgmv_layer(plan, 1, x, [y, z])
    torch.cuda.synchronize()
    outs[name] = (y, z)
same = all(torch.equal(a, b) for a, b in zip(outs["tiled"], outs["persistent"]))
print("bit-identical y:", same)

y, z = y0.clone(), z0.clone()
for rep in range(2):
    for name, flags in (("tiled layer call", 0), ("persistent layer call", PERS),
                        ("tiled, expand no y", 64), ("persistent, expand no y", PERS | 64),
                        ("tiled, expand nothing", 448), ("persistent, expand nothing", PERS | 448),
                        ("shrink+reduce only", 8)):
        N.check(N.lib().plora_debug_set_sgmv_flags(flags))
        for _ in range(3):
            sgmv_layer(plan, 1, x, [y, z])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            sgmv_layer(plan, 1, x, [y, z])
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:28s} {e0.elapsed_time(e1) * 50:.1f} us")
N.check(N.lib().plora_debug_set_sgmv_flags(0))
