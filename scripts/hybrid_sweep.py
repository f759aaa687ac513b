"""Diagnostics: decode-step time of the hybrid launch (plora_bgmv_layers) vs
the streaming share factor (plora_debug_set_hybrid_share)."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, bgmv_layers  # noqa: E402


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
    for f in [float(v) for v in sys.argv[1:]] or [0.8, 0.9, 0.95, 1.0, 1.05, 1.1, 1.2]:
        N.check(N.lib().plora_debug_set_hybrid_share(f))
        plan = BatchPlan(store, ta)
        info = (C.c_double * 4)()
        N.check(N.lib().plora_debug_plan_hybrid(plan.handle, info))
        g = torch.cuda.CUDAGraph()
        for _ in range(3):
            bgmv_layers(plan, 0, x, [y[:, 0], y[:, 1]])
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            bgmv_layers(plan, 0, x, [y[:, 0], y[:, 1]])
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"factor {f:.2f}: share {info[1]:.3f} of rows, {int(info[2])} clusters + {int(info[3])} CTAs: "
              f"{ms * 1e3:.1f} us per step = {4362076160 / (ms / 1e3) / 1e9 / 6449.4:.3f} of the HBM roofline")
    N.check(N.lib().plora_debug_set_hybrid_share(0.95))


if __name__ == "__main__":
    main()
