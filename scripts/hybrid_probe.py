"""Diagnostics: can the 16 SMs the cluster decode kernel leaves idle carry a
share of the decode step?  Splits the cfg2 batch by adapter into a cluster
share (132 SMs) and a streaming-kernel share (16 CTAs), and times each alone
and both concurrently on two streams (one 32-layer launch each)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import _native as N, synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, bgmv_layers  # noqa: E402


def main():
    frac = float(sys.argv[1]) if len(sys.argv) > 1 else 0.093
    cfg = synth.cfg2()
    pool = synth.build_pool(cfg)
    store = AdapterStore(pool, cfg.shape, cfg.n_adapters)
    for a, r in enumerate(cfg.ranks):
        store.register(a, r)
        store.write_pages(a, synth.adapter_image(cfg.shape, r, a, device="cuda").view(torch.uint8))
        store.publish(a)
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    # adapters for the streaming share: largest first until `frac` of the weight bytes
    order = sorted(range(cfg.n_adapters), key=lambda a: -cfg.ranks[a])
    total = sum(cfg.ranks)
    sb, acc = set(), 0
    for a in order:
        if acc + cfg.ranks[a] <= frac * total:
            sb.add(a)
            acc += cfg.ranks[a]
    ta_a = np.where(np.isin(ta, list(sb)), -1, ta).astype(np.int32)
    ta_b = np.where(np.isin(ta, list(sb)), ta, -1).astype(np.int32)
    plan_a = BatchPlan(store, ta_a)
    N.check(N.lib().plora_debug_set_stream_ctas(16))
    plan_b = BatchPlan(store, ta_b)
    N.check(N.lib().plora_debug_set_stream_ctas(0))
    T = len(ta)
    x = torch.randn(32, T, 4096, device="cuda").to(torch.bfloat16)
    y = torch.randn(32, 2, T, 4096, device="cuda").to(torch.bfloat16)
    sa, sb_ = torch.cuda.Stream(), torch.cuda.Stream()

    def run_a(stream):
        N.check(N.lib().plora_debug_set_bgmv_impl(0))
        bgmv_layers(plan_a, 0, x, [y[:, 0], y[:, 1]], stream=stream.cuda_stream)

    def run_b(stream):
        N.check(N.lib().plora_debug_set_bgmv_impl(1))
        bgmv_layers(plan_b, 0, x, [y[:, 0], y[:, 1]], stream=stream.cuda_stream)
        N.check(N.lib().plora_debug_set_bgmv_impl(0))

    def timeit(fn, n=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        e0.record(cur)
        for _ in range(n):
            sa.wait_stream(cur)
            sb_.wait_stream(cur)
            fn()
            cur.wait_stream(sa)
            cur.wait_stream(sb_)
        e1.record(cur)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    alg = 4362076160
    ta_ms = timeit(lambda: run_a(sa))
    tb_ms = timeit(lambda: run_b(sb_))
    both_ab = timeit(lambda: (run_a(sa), run_b(sb_)))
    both_ba = timeit(lambda: (run_b(sb_), run_a(sa)))
    print(f"stream share {acc / total:.3f} of weight bytes ({len(sb)} adapters)")
    print(f"cluster alone {ta_ms * 1e3:.1f} us; stream(16 CTAs) alone {tb_ms * 1e3:.1f} us")
    for name, ms in (("both, cluster first", both_ab), ("both, stream first", both_ba)):
        print(f"{name}: {ms * 1e3:.1f} us per step = {alg / (ms / 1e3) / 1e9 / 6449.4:.3f} of the HBM roofline")


if __name__ == "__main__":
    main()
