"""Diagnostics: item timeline of one single-layer decode call (plora_bgmv_layer,
cfg2 shapes) on the warp-item kernels: per warp item its start / end
(%globaltimer), shrink items then expand items.  Prints the phase spans,
item-duration percentiles, and a concurrency profile."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, bgmv_layer  # noqa: E402

cfg = synth.cfg2(n_layers=2)
pool = synth.build_pool(cfg)
store = AdapterStore(pool, cfg.shape, cfg.n_adapters)
for a, r in enumerate(cfg.ranks):
    store.register(a, r)
    store.write_pages(a, synth.adapter_image(cfg.shape, r, a, device="cuda").view(torch.uint8))
    store.publish(a)
ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
plan = BatchPlan(store, ta)
x = torch.randn(256, 4096, device="cuda").to(torch.bfloat16)
ys = [torch.randn(256, 4096, device="cuda").to(torch.bfloat16) for _ in range(2)]
for _ in range(5):
    bgmv_layer(plan, 1, x, ys)
buf = torch.zeros(2 * 8192, dtype=torch.int64, device="cuda")
N.check(N.lib().plora_debug_set_trace(buf.data_ptr(), buf.numel() * 8))
torch.cuda.synchronize()
for rep in range(3):
    buf.zero_()
    bgmv_layer(plan, 1, x, ys)  # previous call's kernels in flight: like a per-layer step
    bgmv_layer(plan, 1, x, ys)
    torch.cuda.synchronize()
    t = buf.view(-1, 2).cpu().numpy()
    live = np.nonzero(t[:, 0])[0]
    ns_end = 960 if len(live) else 0
    S = t[: ns_end][t[: ns_end, 0] > 0]
    E = t[ns_end:][t[ns_end:, 0] > 0]
    t0 = S[:, 0].min()
    print(f"--- rep {rep}: S items {len(S)}  E items {len(E)}")
    print(f"S start {0:.1f} .. {(S[:,0].max()-t0)/1e3:.2f} us, end {(S[:,1].min()-t0)/1e3:.2f} .. {(S[:,1].max()-t0)/1e3:.2f} us")
    print(f"E start {(E[:,0].min()-t0)/1e3:.2f} .. {(E[:,0].max()-t0)/1e3:.2f} us, end {(E[:,1].min()-t0)/1e3:.2f} .. {(E[:,1].max()-t0)/1e3:.2f} us")
    for nm, X in (("S", S), ("E", E)):
        d = (X[:, 1] - X[:, 0]) / 1e3
        print(f"{nm} item us: p10 {np.percentile(d,10):.2f} p50 {np.percentile(d,50):.2f} p90 {np.percentile(d,90):.2f} max {d.max():.2f}")
    end = max(S[:, 1].max(), E[:, 1].max())
    grid = np.arange(t0, end, 1000)
    cs = [(np.sum((S[:, 0] <= g) & (S[:, 1] > g)), np.sum((E[:, 0] <= g) & (E[:, 1] > g))) for g in grid]
    print("us : S-active E-active  " + "  ".join(f"{i}:{a}/{b}" for i, (a, b) in enumerate(cs)))
N.check(N.lib().plora_debug_set_trace(None, 0))
