"""Diagnostics: time one cfg2 layer launch of the bf16 decode op under
ablation flags (plora_debug_set_bgmv_flags: 1 = consumers skip the math,
2 = no weight copies) and with the cluster kernel (plora_debug_set_bgmv_impl 1),
plus the 32-layer launch (plora_bgmv_layers)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, bgmv_layer, bgmv_layers  # noqa: E402


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


def main():
    cfg = synth.cfg2(n_layers=32)
    pool = synth.build_pool(cfg)
    store = AdapterStore(pool, cfg.shape, cfg.n_adapters)
    for a, r in enumerate(cfg.ranks):
        store.register(a, r)
        store.write_pages(a, synth.adapter_image(cfg.shape, r, a, device="cuda").view(torch.uint8))
        store.publish(a)
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    plan = BatchPlan(store, ta)
    x = torch.randn(32, 256, 4096, device="cuda").to(torch.bfloat16)
    y = torch.randn(32, 2, 256, 4096, device="cuda").to(torch.bfloat16)
    per_layer = lambda: [bgmv_layer(plan, l, x[l], [y[l, 0], y[l, 1]]) for l in range(32)]  # noqa: E731
    multi = lambda: bgmv_layers(plan, 0, x, [y[:, 0], y[:, 1]])  # noqa: E731
    alg = 136314880
    flag_sets = [int(f) for f in os.environ.get("ABLATE_FLAGS", "0,1,2").split(",")]
    for impl in (1, 0):  # 1 streaming, 0 clusters (+ the hybrid streaming share for the 32-layer launch)
        N.check(N.lib().plora_debug_set_bgmv_impl(impl))
        plan.update(ta)  # the hybrid split is decided at plan build
        for pf in (1, 0):  # L2 prefetch of the streaming kernel's weight rows
            N.check(N.lib().plora_debug_set_stream_prefetch(pf))
            for flags in (flag_sets if impl == 1 else (0,)):
                N.check(N.lib().plora_debug_set_bgmv_flags(flags))
                a = timeit(per_layer, 5) / 32
                b = timeit(multi, 5) / 32
                print(f"impl {impl} prefetch {pf} flags {flags}: per-layer launch {a:.1f} us "
                      f"({alg / a / 1e3:.0f} GB/s), 32-layer launch {b:.1f} us/layer ({alg / b / 1e3:.0f} GB/s)")
    N.check(N.lib().plora_debug_set_stream_prefetch(0))
    N.check(N.lib().plora_debug_set_bgmv_flags(0))
    N.check(N.lib().plora_debug_set_bgmv_impl(0))


if __name__ == "__main__":
    main()
