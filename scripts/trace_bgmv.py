"""Diagnostics: per-unit device timeline of one bf16 BGMV call (cfg2 shape).

python scripts/trace_bgmv.py   (on a GPU box) -> prints latency / compute /
idle statistics per unit kind and writes gpurun_out/trace_bgmv.npz.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, bgmv  # noqa: E402


def main():
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
    y = torch.randn(256, 4096, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        bgmv(plan, 1, 0, x, y)
    ctas, units = 148, 64
    buf = torch.zeros(ctas * units * 8, dtype=torch.int64, device="cuda")
    N.check(N.lib().plora_debug_set_trace(buf.data_ptr(), buf.numel() * 8))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bgmv(plan, 1, 0, x, y)
    e1.record()
    torch.cuda.synchronize()
    N.check(N.lib().plora_debug_set_trace(None, 0))
    t = buf.view(ctas, units, 8).cpu().numpy().astype(np.int64)
    issued, ready, done, kind = t[..., 0], t[..., 1], t[..., 2], t[..., 3]
    top, prewait, postwait = t[..., 4], t[..., 5], t[..., 6]
    valid = issued > 0
    t0 = issued[valid].min()
    print(f"call {e0.elapsed_time(e1) * 1e3:.1f} us (event), span {(done[valid].max() - t0) / 1e3:.1f} us")
    exp = (kind >> 32) == 1
    nbytes = kind & 0xffffffff
    for name, m in (("shrink", valid & ~exp), ("expand", valid & exp)):
        lat = (ready - issued)[m] / 1e3
        comp = (done - ready)[m] / 1e3
        print(f"{name}: n={m.sum()} bytes/unit={nbytes[m].mean():.0f} "
              f"issue->ready med {np.median(lat):.2f} p90 {np.percentile(lat, 90):.2f} us; "
              f"ready->done med {np.median(comp):.2f} p90 {np.percentile(comp, 90):.2f} us")
    # consumer idle: time between done(k-1) and ready(k)
    gaps = []
    for c in range(ctas):
        v = valid[c]
        d, r = done[c][v], ready[c][v]
        if len(d) > 1:
            gaps.append(np.clip(r[1:] - d[:-1], 0, None).sum() / max(d[-1] - r[0], 1))
    print(f"consumer waiting fraction (median over CTAs): {np.median(gaps):.2f}")
    first_issue = (issued[:, 0] - t0) / 1e3
    print(f"first issue per CTA: med {np.median(first_issue):.2f} max {first_issue.max():.2f} us")
    end = np.array([done[c][valid[c]].max() - t0 for c in range(ctas) if valid[c].any()]) / 1e3
    print(f"CTA end: min {end.min():.1f} med {np.median(end):.1f} max {end.max():.1f} us")
    # issue lead: how far ahead of consumption the producer runs (units)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.savez(os.path.join(ROOT, "gpurun_out", "trace_bgmv.npz"), trace=t)
    for c in (0, 77):
        v = valid[c]
        rows = [tuple(int((z - t0) / 100) / 10 for z in (a, b, cc, d))
                for a, b, cc, d in zip(top[c][v], prewait[c][v], postwait[c][v], issued[c][v])]
        print(f"CTA {c} producer (loop top, pre-wait, post-wait, issued) us:", rows[:16])
    for c in (0, 1, 77):
        v = valid[c]
        rows = [(int((i - t0) / 1e3 * 10) / 10, int((r - t0) / 1e3 * 10) / 10,
                 int((d - t0) / 1e3 * 10) / 10, int(k >> 32))
                for i, r, d, k in zip(issued[c][v], ready[c][v], done[c][v], kind[c][v])]
        print(f"CTA {c}: (issue, ready, done, expand) us:", rows[:24])


if __name__ == "__main__":
    main()
