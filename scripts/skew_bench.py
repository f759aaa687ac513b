"""Decode BGMV on a skewed batch: 128 adapters at Llama-7B
widths, Zipf token counts with one hot adapter holding many tokens, versus the
uniform cfg2-like batch of the same size.  Prints per-call time and the
algorithmic bytes (each adapter's block once + x + y RMW), so the GB/s shows
whether hot adapters' weights are re-streamed.  Run under ncu with
`-k regex:bgmv` for DRAM bytes."""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2512_20210_b200 import synth  # noqa: E402
from paper_2512_20210_b200.lora import (AdapterStore, BatchPlan, ModelShape, bgmv,  # noqa: E402
                                        bgmv_layer)
from test_parity_full_gpu import skewed_assignment  # noqa: E402


def main():
    hot = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    shape = ModelShape(32, (4096, 4096), (4096, 4096), torch.bfloat16)
    ranks = [(8, 16, 32, 64, 128)[a % 5] for a in range(128)]
    cfg = synth.DecodeConfig("skew", shape, ranks, 1, 2048)
    pool = synth.build_pool(cfg)
    store = AdapterStore(pool, shape, 128)
    for a, r in enumerate(ranks):
        store.register(a, r)
        store.write_pages(a, synth.adapter_image(shape, r, a, device="cuda").view(torch.uint8))
        store.publish(a)
    from paper_2512_20210_b200 import _native as N
    impl = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    route = int(sys.argv[4]) if len(sys.argv) > 4 else 16  # many-token adapters -> SGMV (0: off)
    N.check(N.lib().plora_debug_set_bgmv_impl(impl))
    N.check(N.lib().plora_debug_set_route_tokens(route))
    out = {"impl": impl, "route_min_tokens": route}
    for name, ta in (("skewed", skewed_assignment(hot=hot)),
                     ("uniform", synth.token_assignment(128, 4))):
        T = len(ta)
        used = sorted(set(int(a) for a in ta))
        wbytes = sum(ranks[a] * (4096 + 4096) * 2 for a in used)
        alg = wbytes + T * 4096 * 2 + 2 * T * 4096 * 2
        plan = BatchPlan(store, ta)
        x = torch.randn(32, T, 4096, device="cuda").to(torch.bfloat16)
        y = torch.randn(64, T, 4096, device="cuda").to(torch.bfloat16)
        for _ in range(3):
            for l in range(32):
                bgmv_layer(plan, l, x[l], [y[2 * l], y[2 * l + 1]])
        torch.cuda.synchronize()
        times = []
        for _ in range(iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for l in range(32):
                bgmv_layer(plan, l, x[l], [y[2 * l], y[2 * l + 1]])
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 32)
        ms = statistics.median(times)
        counts = np.bincount(ta, minlength=128)
        out[name] = {"tokens": T, "max_tokens_per_adapter": int(counts.max()),
                     "alg_bytes_per_layer_launch": 2 * alg - T * 4096 * 2,
                     "us_per_layer_launch": ms * 1e3,
                     "gbs": (2 * alg - T * 4096 * 2) / (ms / 1e3) / 1e9}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
