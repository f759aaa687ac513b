"""Diagnostics: SGMV shrink time at cfg3 with parts of its pipeline switched
off (plora_debug_set_sgmv_flags; results are wrong meanwhile) — tells which
stream (x tiles, paged weight gathers, MMAs) bounds the kernel."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, sgmv  # noqa: E402

ranks = [int(a) for a in sys.argv[1:]] or [0]
for r in ranks:
    cfg = synth.cfg3(n_layers=2)
    if r:
        cfg = synth.DecodeConfig("ablate", cfg.shape, [r] * 32, 512, 2048)
    pool = synth.build_pool(cfg)
    store = AdapterStore(pool, cfg.shape, 32)
    for a, ra in enumerate(cfg.ranks):
        store.register(a, ra)
        store.write_pages(a, synth.adapter_image(cfg.shape, ra, a, device="cuda").view(torch.uint8))
        store.publish(a)
    plan = BatchPlan(store, synth.segment_assignment(32, 512))
    x = torch.randn(32 * 512, 4096, device="cuda").to(torch.bfloat16)
    y = torch.randn(32 * 512, 4096, device="cuda").to(torch.bfloat16)
    for name, flags in (("full op", 0), ("shrink only", 8), ("shrink, no gather", 9), ("shrink, no MMA", 10),
                        ("shrink, no x", 12), ("shrink, x only", 11), ("shrink, gather only", 14),
                        ("shrink, nothing", 15), ("shrink, no reduction", 40), ("shrink, no epilogue", 24),
                        ("shrink, nothing at all", 31), ("expand, no y", 64), ("expand, no B", 128),
                        ("expand, no MMA", 256), ("expand, only y", 384), ("expand, nothing", 448),
                        ("expand prologue only", 512)):
        N.check(N.lib().plora_debug_set_sgmv_flags(flags))
        for _ in range(3):
            sgmv(plan, 1, 0, x, y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            sgmv(plan, 1, 0, x, y)
        e1.record()
        torch.cuda.synchronize()
        print(f"rank {r or 'cfg3'} {name:22s} {e0.elapsed_time(e1) * 50:.1f} us")
    N.check(N.lib().plora_debug_set_sgmv_flags(0))
    del plan, store, pool
