"""Diagnostics: per-stage device timeline of the streaming bf16 BGMV
(bgmv_stream.cu) for one cfg2 layer launch (plora_bgmv_layer).

Trace fields per (CTA, stage), SM clocks: 0 producer issued (after the slot
was free), 1 consumers saw the data, 2 consumers released the slot,
3 (an E item's first stage of this producer) cycles spent waiting on the
job's S-item counter."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, bgmv_layer  # noqa: E402

S = 512


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
    ys = [torch.randn(256, 4096, device="cuda").to(torch.bfloat16) for _ in range(2)]
    call = lambda: bgmv_layer(plan, 1, x, ys)  # noqa: E731
    flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    N.check(N.lib().plora_debug_set_bgmv_flags(flags))
    print("flags", flags)
    for _ in range(3):
        call()
    ctas = 148
    buf = torch.zeros(ctas * S * 12, dtype=torch.int64, device="cuda")
    N.check(N.lib().plora_debug_set_trace(buf.data_ptr(), buf.numel() * 8))
    torch.cuda.synchronize()
    call()
    torch.cuda.synchronize()
    N.check(N.lib().plora_debug_set_trace(None, 0))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        call()
    e1.record()
    torch.cuda.synchronize()
    print(f"untraced {e0.elapsed_time(e1) * 1e3 / 20:.1f} us/launch")
    t = buf.view(ctas, S, 12).cpu().numpy().astype(np.float64) / 1.965e3  # us
    for c in range(ctas):
        v = t[c, :, 1] > 0
        if not v.any():
            continue
    issued, seen, done, wait = t[..., 0], t[..., 1], t[..., 2], t[..., 3]
    valid = (seen > 0) & (done > 0) & (issued > 0)
    base = np.where(valid, issued, np.inf).min(axis=1, keepdims=True)
    lat = (seen - issued)[valid]
    proc = (done - seen)[valid]
    print(f"stages per CTA: {valid.sum(axis=1).min()}..{valid.sum(axis=1).max()}")
    print(f"issue->seen latency us: median {np.median(lat):.2f} p90 {np.percentile(lat, 90):.2f}")
    print(f"seen->released us: median {np.median(proc):.3f} p90 {np.percentile(proc, 90):.3f}")
    span = (np.where(valid, done, 0).max(axis=1) - base[:, 0])
    print(f"CTA span us: min {span.min():.1f} median {np.median(span):.1f} max {span.max():.1f}")
    w = wait[wait > 0]
    print(f"counter waits: n={len(w)} median {np.median(w) / 1.0 if len(w) else 0:.2f} us "
          f"p90 {np.percentile(w, 90) if len(w) else 0:.2f} max {w.max() if len(w) else 0:.2f}")
    kind = buf.view(ctas, S, 12)[..., 8].cpu().numpy()
    for kk, name in ((0, "S mid"), (1, "S last"), (2, "S first"), (4, "E mid"), (5, "E last"),
                     (6, "E first"), (7, "E first+last")):
        m = (kind == kk) & valid
        if m.any():
            x = (done - seen)[m]
            print(f"consumer {name}: n={m.sum()} seen->released median {np.median(x):.3f} "
                  f"p90 {np.percentile(x, 90):.3f} us")
    m = valid & (t[..., 10] > 0) & (t[..., 11] > 0)
    if m.any():
        print(f"S: seen -> math start median {np.median((t[..., 10] - seen)[m]):.3f} us; math "
              f"median {np.median((t[..., 11] - t[..., 10])[m]):.3f} us; math end -> released "
              f"median {np.median((done - t[..., 11])[m]):.3f} us")
    m = valid & (t[..., 9] > 0)
    if m.any():
        print(f"E: seen -> math done median {np.median((t[..., 9] - seen)[m]):.3f} us; "
              f"math done -> released median {np.median((done - t[..., 9])[m]):.3f} us")

    def d(a, b):
        m = (t[..., a] > 0) & (t[..., b] > 0)
        x = (t[..., b] - t[..., a])[m]
        if not len(x):
            return "n/a"
        return f"median {np.median(x):.3f} p90 {np.percentile(x, 90):.3f}"
    print("producer: before slot wait -> slot free", d(4, 0))
    print("producer: slot free -> copies issued", d(0, 5))
    for c in (0, 70):
        v = valid[c]
        print(f"CTA {c}: stage kind issue seen released (us from the CTA's first issue)")
        for k in range(S):
            if v[k]:
                print(f"  {k:3d} {int(kind[c, k]):d} {issued[c, k] - base[c, 0]:7.2f} "
                      f"{seen[c, k] - base[c, 0]:7.2f} {done[c, k] - base[c, 0]:7.2f}")
            if k > 60:
                break
    np.savez(os.path.join(ROOT, "gpurun_out", "trace_stream.npz"), t=t)


if __name__ == "__main__":
    main()
