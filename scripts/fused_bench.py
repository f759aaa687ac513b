"""Diagnostics: the fused prefill op (plora_sgmv_fused) at BASELINE config 3
shapes (32 segments × 512 tokens, r = 16/64/128, Llama-7B q 4096 -> 4096)
against cuBLAS base GEMM (torch.matmul) + plora_sgmv, CUDA events, 20 reps."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_20210_b200 import synth  # noqa: E402
from paper_2512_20210_b200.lora import AdapterStore, BatchPlan, sgmv, sgmv_fused  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    cfg = synth.cfg3(n_layers=2)
    pool = synth.build_pool(cfg)
    store = AdapterStore(pool, cfg.shape, cfg.n_adapters)
    for a, r in enumerate(cfg.ranks):
        store.register(a, r)
        store.write_pages(a, synth.adapter_image(cfg.shape, r, a, device="cuda").view(torch.uint8))
        store.publish(a)
    ta = synth.segment_assignment(32, 512)
    plan = BatchPlan(store, ta)
    T = len(ta)
    x = torch.randn(T, 4096, device="cuda").to(torch.bfloat16)
    w0 = (torch.randn(4096, 4096, device="cuda") / 64).to(torch.bfloat16)
    y = torch.empty(T, 4096, device="cuda", dtype=torch.bfloat16)
    flops = 2.0 * T * 4096 * 4096 + sum(2.0 * 512 * r * (4096 + 4096) for r in cfg.ranks)
    peak = 1681.2e12
    t_f = timeit(lambda: sgmv_fused(plan, 1, 0, x, w0, y, 1.0))
    t_g = timeit(lambda: torch.matmul(x, w0.t(), out=y))
    t_u = timeit(lambda: (torch.matmul(x, w0.t(), out=y), sgmv(plan, 1, 0, x, y, 1.0)))
    print(f"fused {t_f:.1f} us = {flops / t_f / 1e6:.0f} TFLOP/s ({flops / t_f / 1e-6 / peak:.1%} of "
          f"{peak / 1e12:.0f})")
    print(f"cuBLAS base GEMM alone {t_g:.1f} us = {2.0 * T * 4096 * 4096 / t_g / 1e6:.0f} TFLOP/s")
    print(f"cuBLAS GEMM + plora_sgmv {t_u:.1f} us")
    y2 = torch.matmul(x, w0.t())
    sgmv(plan, 1, 0, x, y2, 1.0)
    sgmv_fused(plan, 1, 0, x, w0, y, 1.0)
    torch.cuda.synchronize()
    print("max |fused - (GEMM + sgmv)| / max|ref|:",
          ((y.float() - y2.float()).abs().max() / y2.float().abs().max()).item())


if __name__ == "__main__":
    main()
