"""Diagnostics: one-launch-per-layer decode step (plora_bgmv_layer x 32) with
and without the hybrid pair per layer (plora_debug_set_hybrid_per_layer)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, bgmv_layer  # noqa: E402


def main():
    cfg = synth.cfg2()
    pool = synth.build_pool(cfg)
    store = AdapterStore(pool, cfg.shape, cfg.n_adapters)
    for a, r in enumerate(cfg.ranks):
        store.register(a, r)
        store.write_pages(a, synth.adapter_image(cfg.shape, r, a, device="cuda").view(torch.uint8))
        store.publish(a)
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    T = len(ta)
    x = torch.randn(32, T, 4096, device="cuda").to(torch.bfloat16)
    y = torch.randn(32, 2, T, 4096, device="cuda").to(torch.bfloat16)
    plan = BatchPlan(store, ta)
    for on in (0, 1):
        N.check(N.lib().plora_debug_set_hybrid_per_layer(on))
        step = lambda: [bgmv_layer(plan, l, x[l], [y[l, 0], y[l, 1]]) for l in range(32)]  # noqa: E731
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"hybrid per layer {on}: {ms * 1e3 / 32:.1f} us per layer = "
              f"{136314880 / (ms / 32 / 1e3) / 1e9 / 6449.4:.3f} of the HBM roofline")
    N.check(N.lib().plora_debug_set_hybrid_per_layer(0))


if __name__ == "__main__":
    main()
