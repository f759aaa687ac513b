"""Small paged-LoRA calls for compute-sanitizer (memcheck / racecheck /
synccheck): the cluster BGMV (per projection and fused per layer), the SGMV
(per projection, per layer, fused with the base GEMM) and the TP halves on a
2-layer cfg1 store.

compute-sanitizer --tool memcheck python scripts/sanitize.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from lora_harness import Setup  # noqa: E402
from paper_2512_20210_b200 import synth  # noqa: E402
from paper_2512_20210_b200.lora import BatchPlan, bgmv, bgmv_layer, sgmv, sgmv_fused, sgmv_layer  # noqa: E402
from paper_2512_20210_b200.tp import bgmv_tp_expand, bgmv_tp_shrink, tp_shard_rows  # noqa: E402


def main():
    cfg = synth.cfg1(n_layers=2)
    s = Setup(cfg)
    ta = synth.token_assignment(cfg.n_adapters, cfg.tokens_per_adapter)
    T = len(ta)
    x = torch.randn(T, 4096, device="cuda").to(torch.bfloat16)
    ys = [torch.randn(T, 4096, device="cuda").to(torch.bfloat16) for _ in range(2)]
    plan = BatchPlan(s.store, ta)
    bgmv(plan, 1, 0, x, ys[0])
    bgmv_layer(plan, 0, x, ys)
    seg = synth.segment_assignment(4, 160)  # runs of 160 tokens: full and partial tiles
    xs = torch.randn(len(seg), 4096, device="cuda").to(torch.bfloat16)
    yss = torch.randn(len(seg), 4096, device="cuda").to(torch.bfloat16)
    sgmv(BatchPlan(s.store, seg), 1, 1, xs, yss)
    seg2 = synth.segment_assignment(3, 300)  # runs of 300: tile pairs sharing the weight chunks
    xs2 = torch.randn(len(seg2), 4096, device="cuda").to(torch.bfloat16)
    ys2 = torch.randn(len(seg2), 4096, device="cuda").to(torch.bfloat16)
    sgmv(BatchPlan(s.store, seg2), 1, 0, xs2, ys2)
    plan2 = BatchPlan(s.store, seg2)
    sgmv_layer(plan2, 1, xs2, [ys2, ys2.clone()])  # both projections from one x chunk
    w0 = torch.randn(4096, 4096, device="cuda").to(torch.bfloat16)
    sgmv_fused(plan2, 0, 0, xs2, w0, torch.empty_like(ys2))  # base GEMM + LoRA K-steps
    rs = tp_shard_rows(plan, 2)
    vp = torch.empty(2, T, rs, device="cuda")
    for i in range(2):
        bgmv_tp_shrink(plan, 0, 0, i, 2, x, vp[i])
    for i in range(2):
        bgmv_tp_expand(plan, 0, 0, i, 2, vp, ys[0][:, i * 2048:(i + 1) * 2048])
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
