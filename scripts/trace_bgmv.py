"""Diagnostics: launch geometry and per-chunk device timeline of one bf16
BGMV call (cfg2 shape) on the cluster kernel.

python scripts/trace_bgmv.py   (on a GPU box) -> prints the plan geometry,
per-CTA chunk timings and writes gpurun_out/trace_bgmv.npz.

Trace fields per (CTA, chunk k), SM clock cycles (shown as us at 1.965 GHz;
comparable within a CTA only):
  0 consumer: chunk data landed     1 consumer: partial v sent
  2 consumer: exchange complete     3 consumer: expand done, slot released
  4 producer: before slot wait      5 producer: slot free (issuing)
  6 producer: lookahead landed      (k = 63: 6 CTA start, 7 CTA end)
  8 shrink: MMAs done   9 shrink: partial barrier passed   10 expand: v built
  11 expand: MMAs done  12 page warp 0: copies issued      13 (unused)
  14 shrink: before the chunk wait  15 shrink: job x landed, barrier armed
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import (AdapterStore, BatchPlan, bgmv, bgmv_layer,  # noqa: E402
                                        bgmv_layers)

K = 64


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
    fused = "--layer" in sys.argv  # q and v in one launch (plora_bgmv_layer)
    geom = (C.c_uint32 * 8)()
    N.check(N.lib().plora_debug_plan_geom(plan.handle, 0, geom))
    names = ("cs", "ks", "ns", "a_slots", "b_slots", "smem", "clusters", "chunks")
    print("geometry:", dict(zip(names, list(geom))))
    x = torch.randn(256, 4096, device="cuda").to(torch.bfloat16)
    y = torch.randn(256, 4096, device="cuda").to(torch.bfloat16)
    y2 = torch.randn(256, 4096, device="cuda").to(torch.bfloat16)
    call = (lambda: bgmv_layer(plan, 1, x, [y, y2])) if fused else (lambda: bgmv(plan, 1, 0, x, y))
    if "--layers" in sys.argv:  # both layers in one launch (plora_bgmv_layers)
        xl = torch.randn(2, 256, 4096, device="cuda").to(torch.bfloat16)
        yl = torch.randn(2, 2, 256, 4096, device="cuda").to(torch.bfloat16)
        call = lambda: bgmv_layers(plan, 0, xl, [yl[:, 0], yl[:, 1]])  # noqa: E731
    for _ in range(3):
        call()
    ctas = geom[0] * geom[6]
    buf = torch.zeros(ctas * K * 16, dtype=torch.int64, device="cuda")
    N.check(N.lib().plora_debug_set_trace(buf.data_ptr(), buf.numel() * 8))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    call()
    e1.record()
    torch.cuda.synchronize()
    N.check(N.lib().plora_debug_set_trace(None, 0))
    # untraced timing of the same call
    for _ in range(3):
        call()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    for _ in range(20):
        call()
    e3.record()
    torch.cuda.synchronize()
    t = buf.view(ctas, K, 16).cpu().numpy().astype(np.int64)
    start = t[:, K - 1, 6]
    t0 = start.min()
    t = (t / 1.965).astype(np.int64)  # cycles -> ns
    start = t[:, K - 1, 6]
    t0 = start.min()
    rel = lambda v: (v - t0) / 1e3  # noqa: E731
    print(f"call {e0.elapsed_time(e1) * 1e3:.1f} us traced; untraced {e2.elapsed_time(e3) * 1e3 / 20:.1f} "
          f"us/call; CTA duration min/med/max {(t[:, K - 1, 7] - start).min() / 1e3:.1f}/"
          f"{np.median(t[:, K - 1, 7] - start) / 1e3:.1f}/{(t[:, K - 1, 7] - start).max() / 1e3:.1f} us")
    valid = t[..., 0] > 0
    d_ready = np.diff(np.where(valid, t[..., 0], np.nan), axis=1) / 1e3
    print(f"chunk-to-chunk (data ready) median {np.nanmedian(d_ready):.2f} us, p90 "
          f"{np.nanpercentile(d_ready, 90):.2f}")
    xch = (t[..., 2] - t[..., 1])[valid & (t[..., 2] > 0)] / 1e3
    print(f"exchange wait (sent -> all partials, next iter) median {np.median(xch):.2f} us")
    tstart = t[:, K - 1, 6].copy()
    t[:, K - 1, :] = 0
    wait_slot = (t[..., 5] - t[..., 4])[t[..., 4] > 0] / 1e3
    # page warp 0 takes every other chunk of its ring
    m = (t[:, 2::2, 6] > 0) & (t[:, :-2:2, 5] > 0)
    work = (t[:, 2::2, 6] - t[:, :-2:2, 5])[m] / 1e3
    pre = (t[..., 4] - t[..., 6])[(t[..., 4] > 0) & (t[..., 6] > 0)] / 1e3
    print(f"producer: issue work (slot free -> its next chunk's lookahead landed) median {np.median(work):.2f} us; "
          f"lookahead-landed -> slot wait start median {np.median(pre):.2f} us")
    land = (t[..., 0] - t[..., 5])[(t[..., 0] > 0) & (t[..., 5] > 0)] / 1e3
    print(f"data latency (issued -> consumer saw it) median {np.median(land):.2f} us")
    first_ready = np.array([(t[c, 0, 0] - tstart[c]) for c in range(ctas) if t[c, 0, 0] > 0]) / 1e3
    print(f"first chunk ready after CTA start: median {np.median(first_ready):.2f} max {first_ready.max():.2f} us")
    nchunks = (t[..., 0] > 0).sum(axis=1)
    print(f"chunks per CTA min/med/max {nchunks.min()}/{int(np.median(nchunks))}/{nchunks.max()}")
    print(f"producer slot wait median {np.median(wait_slot):.2f} us, p90 {np.percentile(wait_slot, 90):.2f}")
    def med(a, b):
        m = (t[..., a] > 0) & (t[..., b] > 0)
        return np.median((t[..., b] - t[..., a])[m]) / 1e3
    print(f"shrink: wait {med(14, 0):.2f} | hdr->x ready {med(0, 15):.2f} | MMAs {med(15, 8):.2f} | barrier {med(8, 9):.2f} | "
          f"sum+send {med(9, 1):.2f} us")
    print(f"expand: xchg->v built {med(2, 10):.2f} | MMAs {med(10, 11):.2f} | y+barrier {med(11, 3):.2f} us")
    print(f"page warp 0: slot free -> issued {med(5, 12):.2f} us")
    for c in (0, 1, 2, 3, ctas // 2):
        v = valid[c]
        c0 = tstart[c]
        rows = [tuple(round((z - c0) / 1e3, 2) for z in (t[c, k, 5], t[c, k, 0], t[c, k, 1], t[c, k, 2], t[c, k, 3]))
                for k in range(K) if v[k]]
        print(f"CTA {c} (issue, ready, sent, xchg, done) us:", rows[:20])
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.savez(os.path.join(ROOT, "gpurun_out", "trace_bgmv.npz"), trace=t, geom=np.array(list(geom)))


if __name__ == "__main__":
    main()
