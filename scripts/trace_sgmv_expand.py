"""Diagnostics: per-block device timeline of the persistent SGMV expand
(sgmv.cu) for one cfg3 layer call.  Fields per (CTA, block k), SM clocks:
0 gather saw its stage free, 1 gathers issued, 2 MMA saw the Bᵀ block,
3 MMA saw the accumulator free (issues), 4 epilogue saw the accumulator,
5 TMEM loaded, 6 staged (reduce-add issued), 7 epilogue loop top (staging
buffer free).  argv[1]: sgmv debug flags (e.g. 448: nothing moved)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, sgmv_layer  # noqa: E402

K = 128
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
for flags in [int(a) for a in sys.argv[1:]] or [0]:
    N.check(N.lib().plora_debug_set_sgmv_flags(flags | (1 << 20)))  # the persistent expand
    for _ in range(3):
        sgmv_layer(plan, 1, x, ys)
    buf = torch.zeros(148 * K * 8, dtype=torch.int64, device="cuda")
    N.check(N.lib().plora_debug_set_trace(buf.data_ptr(), buf.numel() * 8))
    torch.cuda.synchronize()
    sgmv_layer(plan, 1, x, ys)
    torch.cuda.synchronize()
    N.check(N.lib().plora_debug_set_trace(None, 0))
    t = buf.view(148, K, 8).cpu().numpy().astype(np.int64)
    print(f"=== flags {flags}")
    for cta in (0, 73, 147):
        tt = t[cta]
        n = int((tt[:, 3] > 0).sum())
        t0 = tt[0, 0]
        print(f"cta {cta}: {n} blocks traced; span {(tt[n-1, 6] - t0) if n else 0} cycles")
        print("  k   gfree  gissue  mmaB  mmaAcc  epiAcc  tmemld  staged  epitop   (cycles from block 0's gfree)")
        for k in list(range(0, 12)) + list(range(n - 4, n)):
            if k < 0 or k >= n:
                continue
            print(f"  {k:3d} " + " ".join(f"{(tt[k, f] - t0) if tt[k, f] else -1:7d}" for f in (0, 1, 2, 3, 4, 5, 6, 7)))
        d = np.diff(tt[:n, 3])
        print(f"  MMA issue interval: median {np.median(d):.0f}, mean {d.mean():.0f} cycles")
        for name, a_, b_ in (("gfree->mmaB", 0, 2), ("mmaAcc->epiAcc", 3, 4), ("epiAcc->tmemld", 4, 5),
                             ("tmemld->staged", 5, 6), ("epitop->epiAcc", 7, 4), ("gissue->mmaB", 1, 2)):
            dd = tt[:n, b_] - tt[:n, a_]
            print(f"  {name:16s} median {np.median(dd):.0f} cycles")
N.check(N.lib().plora_debug_set_sgmv_flags(0))
